"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections
import csv
import sys

path = sys.argv[1]
lines = [ln for ln in open(path) if ln.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    name = r[i_name].split("(")[0].replace("rsa::<unnamed>::", "")
    agg.setdefault(name, []).append(float(r[i_val].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':58s} {'launches':>8s} {'mean_us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:58]:58s} {len(v):8d} {sum(v) / len(v) / 1e3:9.2f} {sum(v) / tot:6.3f}")
