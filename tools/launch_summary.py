"""Summarise an `ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum] --csv`
launch list by kernel: launches, mean device time, share of the listed time, DRAM bytes per launch."""
import collections
import csv
import sys

path = sys.argv[1]
lines = [ln for ln in open(path) if ln.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
i_id, i_name = hdr.index("ID"), hdr.index("Kernel Name")
i_metric, i_unit, i_val = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
launch = collections.OrderedDict()
for r in rows[1:]:
    name = r[i_name].split("(")[0].replace("rsa::<unnamed>::", "").replace("void ", "")
    d = launch.setdefault(r[i_id], {"name": name})
    d[r[i_metric]] = float(r[i_val].replace(",", "")) * scale.get(r[i_unit], 1.0)
agg = collections.OrderedDict()
for d in launch.values():
    a = agg.setdefault(d["name"], {"n": 0, "us": 0.0, "rd": 0.0, "wr": 0.0})
    a["n"] += 1
    a["us"] += d.get("gpu__time_duration.sum", 0.0)
    a["rd"] += d.get("dram__bytes_read.sum", 0.0)
    a["wr"] += d.get("dram__bytes_write.sum", 0.0)
tot = sum(a["us"] for a in agg.values())
print(f"{'kernel':52s} {'launches':>8s} {'mean_us':>9s} {'share':>6s} {'MB_rd/launch':>13s} {'MB_wr/launch':>13s}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
    n = a["n"]
    print(f"{k[:52]:52s} {n:8d} {a['us'] / n:9.2f} {a['us'] / tot:6.3f} {a['rd'] / n / 1e6:13.1f} {a['wr'] / n / 1e6:13.1f}")
