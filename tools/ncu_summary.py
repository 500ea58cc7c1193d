"""Summarise .ncu-rep captures into a small markdown table for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [...] > profiles/ncu_rNN.md

Per kernel: duration, SM clock, DRAM bytes read/written (traffic), DRAM
throughput %, L1TEX %, issue-slot %, occupancy, registers, and the split of
L1TEX wavefronts between global loads and shared memory.
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "smsp__cycles_elapsed.avg.per_second": "sm_clock",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_pct",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "wf_shared",
    "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum": "wf_global_ld",
    "smsp__inst_executed.sum": "inst",
}


PIPE_PREFIXES = ("sm__pipe_", "sm__inst_executed_pipe_")


def read_pipes(path):
    """Per kernel: every pipe-utilisation metric of the capture
    (sm__pipe_*_cycles_active / sm__inst_executed_pipe_* as % of peak), e.g.
    the FP64 pipe for the double-precision kernels."""
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[0], rows[2:]
    res = []
    for row in data:
        d = dict(zip(hdr, row))
        pipes = {}
        for k, v in d.items():
            if (k.startswith(PIPE_PREFIXES) and k.endswith("pct_of_peak_sustained_active")
                    and not any(t in k for t in (".max.", ".min.", ".sum."))):
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                if x >= 0.5:
                    pipes[k.replace(".avg.pct_of_peak_sustained_active", "")] = x
        res.append((d.get("Kernel Name", "?")[:90], pipes))
    return res


def read(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for row in data:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "?")[:90]}
        for k, name in WANT.items():
            if k in d:
                rec[name] = (d[k], u.get(k, ""))
        res.append(rec)
    return res


def fmt(v):
    try:
        x = float(str(v[0]).replace(",", ""))
    except (ValueError, TypeError):
        return str(v[0])
    unit = v[1]
    if unit in ("byte",):
        return f"{x / 2**20:.1f} MiB"
    if unit in ("nsecond", "ns"):
        return f"{x / 1e3:.1f} us"
    if unit in ("hz", "Hz", "cycle/second"):
        return f"{x / 1e9:.2f} GHz"
    if x >= 1e6:
        return f"{x:.3g}"
    return f"{x:.4g}"


def main():
    cols = ["duration", "sm_clock", "dram_read", "dram_write", "dram_pct", "l1tex_pct", "issue_pct",
            "occupancy_pct", "regs", "block", "grid", "wf_global_ld", "wf_shared", "inst"]
    print("| report | kernel | " + " | ".join(cols) + " |")
    print("|" + "---|" * (len(cols) + 2))
    for path in sys.argv[1:]:
        for rec in read(path):
            vals = [fmt(rec[c]) if c in rec else "" for c in cols]
            print(f"| {path.split('/')[-1]} | `{rec['kernel']}` | " + " | ".join(vals) + " |")
    print()
    print("Pipe utilisation (% of peak sustained, >= 0.5 %):")
    print()
    for path in sys.argv[1:]:
        for kern, pipes in read_pipes(path):
            top = ", ".join(f"{k} {v:.1f}" for k, v in sorted(pipes.items(), key=lambda kv: -kv[1]))
            print(f"- {path.split('/')[-1]} `{kern}`: {top}")


if __name__ == "__main__":
    main()
