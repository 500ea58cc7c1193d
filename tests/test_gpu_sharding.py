"""The sharded protected path end to end on the GPU: two gloo ranks sharing
cuda:0 each run ``run_protected_sharded`` on their group-aligned slice (a
fault on rank 1's slice), and the merged report is the single-process report
byte for byte; outputs concatenate to the single-process outputs bitwise.
Also: surplus ranks with empty slices ("replicas only") and a degenerate
batch whose flags overflow the device record list."""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT, random_batch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(n, b):
    x = random_batch(np.random.default_rng([7, n]), (b, n), np.complex64)
    return x


def _worker(rank, world, port, n, b, fault, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2405_02520_b200 import build_twiddles, make_plan
    from paper_2405_02520_b200.abft import DetectionConfig, Scheme
    from paper_2405_02520_b200.fault_lab import BitFlipInjector, FaultSpec
    from paper_2405_02520_b200.fft_core import fit_group_size
    from paper_2405_02520_b200.sharding import run_protected_sharded, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    x = _case(n, b)
    plan = fit_group_size(make_plan(n, "fp32", batch=b), b)
    s0, s1 = shard_range(b, plan.bs, world, rank)
    inj = BitFlipInjector(FaultSpec(0, *fault)) if fault else None
    out, rep, cnt = run_protected_sharded(plan, build_twiddles(plan), torch.from_numpy(x[s0:s1]).cuda(),
                                          s0, Scheme.TWO_SIDED_GROUP, DetectionConfig(1e-4), injector=inj)
    q.put((rank, s0, out.cpu().numpy(), rep.to_json(), rep.max_rel_discrepancy,
           inj.fired if inj else None))
    dist.destroy_process_group()


def _sharded(world, n, b, fault):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, b, fault, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _single(n, b, fault):
    from paper_2405_02520_b200 import build_twiddles, make_plan, run_protected
    from paper_2405_02520_b200.abft import DetectionConfig, Scheme
    from paper_2405_02520_b200.fault_lab import BitFlipInjector, FaultSpec
    from paper_2405_02520_b200.fft_core import fit_group_size
    x = _case(n, b)
    plan = fit_group_size(make_plan(n, "fp32", batch=b), b)
    inj = BitFlipInjector(FaultSpec(0, *fault)) if fault else None
    out, rep, _ = run_protected(plan, build_twiddles(plan), torch.from_numpy(x).cuda(),
                                Scheme.TWO_SIDED_GROUP, DetectionConfig(1e-4), injector=inj)
    return out.cpu().numpy(), rep


@pytest.mark.parametrize("n,b,fault", [
    (1024, 64, (45, 300, "im", 30)),     # bs 1 (planner row 2^10): 64 groups, fault on rank 1
    (4096, 64, (40, 17, "re", 29)),      # bs 16: 4 groups, fault in rank 1's first group
    (2**15, 32, (20, 1000, "re", 28)),   # multi-pass, bs 16: 2 groups
])
def test_sharded_report_equals_single_process(n, b, fault):
    ref_out, ref_rep = _single(n, b, fault)
    res = _sharded(2, n, b, fault)
    for rank, s0, out, rep_json, mx, fired in res:
        assert rep_json == ref_rep.to_json()  # byte for byte on every rank
        assert mx == ref_rep.max_rel_discrepancy
        assert fired is True  # fired on rank 1 only, known on both
        np.testing.assert_array_equal(out, ref_out[s0:s0 + out.shape[0]])
    assert json.loads(ref_rep.to_json())["corrected"][0]["signal"] == fault[0]


def test_surplus_ranks_get_empty_slices():
    # 32 signals in two groups of 16 over 3 ranks: rank 2 has nothing to do
    ref_out, ref_rep = _single(4096, 32, (3, 5, "im", 30))
    res = _sharded(3, 4096, 32, (3, 5, "im", 30))
    assert res[2][2].shape == (0, 4096)
    for rank, s0, out, rep_json, mx, fired in res:
        assert rep_json == ref_rep.to_json()


def test_degenerate_batch_reports_every_flag():
    """An all-zero batch flags every signal (0/0 -> inf, pipeline.py:118-121).
    Past the device record list (2^16) the flags go through the overflow
    mask; the report still lists them all and nothing raises."""
    from paper_2405_02520_b200 import build_twiddles, make_plan, run_protected
    from paper_2405_02520_b200.abft import DetectionConfig, Scheme
    from paper_2405_02520_b200.fft_core import fit_group_size
    n, b = 8, 100_000
    plan = fit_group_size(make_plan(n, "fp32", batch=b), b)
    x = torch.zeros((b, n), dtype=torch.complex64, device="cuda")
    out, rep, _ = run_protected(plan, build_twiddles(plan), x, Scheme.TWO_SIDED_GROUP, DetectionConfig(1e-4))
    assert len(rep.flagged) == b
    assert [f["signal"] for f in rep.flagged] == list(range(b))
    assert rep.unrecoverable == list(range(b // plan.bs))
    assert rep.max_rel_discrepancy == float("inf")
    assert torch.count_nonzero(out).item() == 0
    # host (numpy) batch through the streaming path
    out2, rep2, _ = run_protected(plan, build_twiddles(plan), np.zeros((b, n), np.complex64),
                                  Scheme.TWO_SIDED_GROUP, DetectionConfig(1e-4))
    assert rep2.to_json() == rep.to_json()
