"""Per-pass kernel times of the multi-pass transforms (ncu launch list):
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file X \
        python tools/profile_single.py --prec P --logn L --reps 1
then: python tools/pass_times.py X  -> per kernel us, GB/s (algorithmic 2 x batch bytes)."""
import csv
import re
import sys


def main():
    for path in sys.argv[1:]:
        rows = [r for r in csv.reader(open(path)) if len(r) > 10]
        hdr, rows = rows[0], rows[1:]
        ix = {h: i for i, h in enumerate(hdr)}
        per = {}
        for r in rows:
            d = per.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})
            d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
        for lid in sorted(per, key=int):
            d = per[lid]
            us = d.get("gpu__time_duration.sum", 0) / 1e3
            by = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
            name = re.sub(r"\(.*", "", d["name"]).replace("void tfft::", "")
            print(f"{path.split('/')[-1]:28s} {us:9.1f} us  dram {by / 1e9:6.3f} GB  {by / us / 1e3 if us else 0:7.0f} GB/s  {name[:90]}")


if __name__ == "__main__":
    main()
