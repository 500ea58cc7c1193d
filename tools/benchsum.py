"""Print the key fields of a bench.py JSON line (the last JSON line of a log)."""
import json
import sys

line = [l for l in open(sys.argv[1]) if l.startswith("{")][-1]
d = json.loads(line)
for k in ["value", "ms_per_step", "hbm_gbs", "host_gap_ms_per_step", "abft_overhead_pct", "vs_cufft",
          "gpu_launches", "clocks", "fault_counters"]:
    print(k, d.get(k))
print("roofline", d.get("roofline"))
if "e2e" in d:
    print("e2e", d["e2e"].get("value"), "cpu", d.get("cpu_baseline", {}).get("value"))
for s in d.get("sweep", []):
    print({k: s[k] for k in s if k in ("n", "ms_abft_on", "ms_abft_off", "ms_cufft", "frac", "frac_abft_on",
                                      "abft_overhead_pct", "vs_cufft", "hbm_gbs")})
c3 = d.get("c3")
if c3:
    print("c3", c3["value"], c3["roofline"], c3.get("clocks"))
    for s in c3["sweep"]:
        print(s["n"], s["ms_abft_on"], s["ms_abft_off"], s["frac_per_executed_pass"], s["abft_overhead_pct"])
