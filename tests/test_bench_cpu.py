"""bench.py on the CPU: the reference arm (`--impl reference`, the
reference's CPU path — the oracle port with the reference's compiled
butterfly) prints one JSON line with the contract's keys, and the C2 / C3 /
C5 size lists cover BASELINE configs[1] / [2] / [4]."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "GFLOP/s"
    assert line["cpu_baseline"]["kind"] in ("port", "reference") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_bench_size_lists_match_baseline_configs():
    sys.path.insert(0, ROOT)
    import bench
    assert [1 << e for e in bench.SIZES] == [8 << i for i in range(11)]          # C2: 2^3 .. 2^13
    assert [1 << e for e in bench.C3_SIZES] == [1 << e for e in range(20, 26)]  # C3: 2^20 .. 2^25
    assert bench.C5_SIZES == list(range(10, 26))                                 # C5: 2^10 .. 2^25
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert bench.METRIC == base["metric"]
