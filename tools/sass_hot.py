"""Per-opcode instruction / stall-sample breakdown of one kernel from an
ncu report (source page, SASS view).

    python tools/sass_hot.py report.ncu-rep [--top 30]
"""
import argparse
import collections
import csv
import io
import subprocess


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    return hdr, rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--lines", type=int, default=0, help="also print the N hottest instructions")
    a = ap.parse_args()
    hdr, rows = load(a.rep)
    ix = {h: i for i, h in enumerate(hdr)}
    ops = collections.defaultdict(lambda: [0, 0])
    tot_i = tot_s = 0
    hot = []
    for r in rows:
        if r[:3] == hdr[:3]:
            break  # the next kernel's section (captures with -c > 1): first kernel only
        if len(r) < len(hdr) or not r[ix["Instructions Executed"]].strip().isdigit():
            continue
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        ins = int(r[ix["Instructions Executed"]] or 0)
        smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ops[op][0] += ins
        ops[op][1] += smp
        tot_i += ins
        tot_s += smp
        hot.append((smp, r[ix["Address"]], src))
    print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s}")
    for op, (i, s) in sorted(ops.items(), key=lambda x: -x[1][0])[:a.top]:
        print(f"{op:12s} {i:12d} {100 * i / tot_i:5.1f}%  samples {100 * s / max(tot_s, 1):5.1f}%")
    for smp, addr, src in sorted(hot, reverse=True)[:a.lines]:
        print(f"{smp:7d} {addr} {src}")


if __name__ == "__main__":
    main()
