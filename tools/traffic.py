"""DRAM traffic of one solve's combine levels from an ncu launch list
(`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv python tools/one_solve.py CFG`), for bench.py's roofline.traffic.
Usage: python tools/traffic.py launches.csv CFG > profiles/traffic_cfgCFG.json
Combine kernels = every launch of the LAST solve between the leaf step and the
recovery walk (narrow / skeleton / refinement / finalize)."""
import csv, json, sys
from collections import OrderedDict

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0,
         "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
path, cfg = sys.argv[1], int(sys.argv[2])
lines = [l for l in open(path) if l.startswith('"')]
recs = OrderedDict()
for r in csv.DictReader(lines):
    d = recs.setdefault(r["ID"], {"name": r["Kernel Name"].split("(")[0].replace("void ", "")})
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNITS.get(r["Metric Unit"], 1)
launches = list(recs.values())
start = max(i for i, d in enumerate(launches) if "nx_kernel" in d["name"])
launches = launches[start:]
comb = [d for d in launches
        if not any(t in d["name"] for t in ("nx_kernel", "leaf_wstar", "virtual_wstar", "walk_",
                                            "assemble"))]
by = OrderedDict()
for d in comb:
    k = d["name"].replace("lcsg::", "").split("<")[0]
    e = by.setdefault(k, {"launches": 0, "us": 0.0, "read_bytes": 0.0, "write_bytes": 0.0})
    e["launches"] += 1
    e["us"] += d["gpu__time_duration.sum"]
    e["read_bytes"] += d["dram__bytes_read.sum"]
    e["write_bytes"] += d["dram__bytes_write.sum"]
rd = sum(d["dram__bytes_read.sum"] for d in comb)
wr = sum(d["dram__bytes_write.sum"] for d in comb)
print(json.dumps({
    "config": cfg, "source": path.split("/")[-1],
    "note": "ncu --clock-control none launch list of one solve (cold-cache, serialised launches)",
    "combine_launches": len(comb), "combine_us_serialised": sum(d["gpu__time_duration.sum"] for d in comb),
    "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes": rd + wr,
    "by_kernel": by}, indent=1))
