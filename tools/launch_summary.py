"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv`) of a
bench command: per kernel the launch count, mean duration, share of the
summed kernel time and mean DRAM bytes per launch. Writes a markdown table
and a JSON with the ABFT-on single kernels' traffic (read by bench.py for
`roofline.traffic`).

    python tools/launch_summary.py gpurun_out/launches.csv profiles/launches_r01.md profiles/traffic_r01.json
"""
import collections
import csv
import json
import re
import sys


def main():
    src, md_out, js_out = sys.argv[1:4]
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.defaultdict(dict)
    for r in rows:
        per[r[ix["ID"]]]["name"] = r[ix["Kernel Name"]]
        val = float(r[ix["Metric Value"]].replace(",", ""))
        per[r[ix["ID"]]][r[ix["Metric Name"]]] = val
    # full-batch launches only for the traffic figure (the e2e leg of the
    # bench launches the same kernels on 32 MiB chunks)
    full = collections.defaultdict(list)
    for d in per.values():
        full[re.sub(r"\(.*", "", d["name"])].append(
            d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0))
    agg = collections.OrderedDict()
    for lid, d in per.items():
        name = re.sub(r"\(.*", "", d["name"])
        a = agg.setdefault(name, dict(n=0, t=0.0, b=0.0))
        a["n"] += 1
        a["t"] += d.get("gpu__time_duration.sum", 0.0)
        a["b"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["t"] for a in agg.values())
    lines = ["| kernel | launches | mean us | share of kernel time | mean DRAM bytes / launch |",
             "|---|---|---|---|---|"]
    traffic = {}
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        mean_b = a["b"] / a["n"]
        lines.append(f"| `{name[:120]}` | {a['n']} | {a['t'] / a['n'] / 1e3:.1f} | "
                     f"{100 * a['t'] / tot:.1f} % | {mean_b:.4g} |")
        m = re.search(r"fft_single_kernel<float, (\d+), \d+, \d+, 1,", name)
        if m:
            big = [b for b in full[name] if b >= 0.5 * max(full[name])]
            traffic[m.group(1)] = sum(big) / len(big)
    open(md_out, "w").write("\n".join(lines) + "\n")
    json.dump({"dram_bytes_per_launch_by_n": traffic, "source": src}, open(js_out, "w"), indent=1)
    print("\n".join(lines[:25]))


if __name__ == "__main__":
    main()
