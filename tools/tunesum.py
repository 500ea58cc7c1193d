"""Compact table of tools/tune.py JSON results: per (prec, logn) every variant's
ms with ABFT off / on and the fraction of the HBM peak (ABFT on); '*' marks the
best ABFT-on time, '=' the current codegen choice.

    python tools/tunesum.py gpurun_out/tune_r02_fp32.json [more.json ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_02520_b200 import codegen  # noqa: E402

PEAK = 6539.9
rows = []
for f in sys.argv[1:]:
    rows += json.load(open(f))
by = {}
for r in rows:
    by.setdefault((r["prec"], r["logn"]), []).append(r)
for (p, l), rs in sorted(by.items()):
    best = min(rs, key=lambda r: r["ms_on"])
    cur = codegen.SINGLE_CHOICE[p].get(l, 0)
    cands = codegen.SINGLE_CANDIDATES[p][l]
    for r in rs:
        c = cands[r["variant"]]
        mark = ("*" if r is best else " ") + ("=" if r["variant"] == cur else " ")
        print(f"{p} {l:2d} v{r['variant']:<2d}{mark} E{c['e']:<2d} {str(c['radices']):16s} thr{c['threads']:<4d} "
              f"minb{c['minb']} st{c['stage']}  off {r['ms_off']:.4f}  on {r['ms_on']:.4f}  "
              f"frac {r['gbs_on'] / PEAK:.3f}  abft {100 * (r['ms_on'] / r['ms_off'] - 1):+.1f}%")
