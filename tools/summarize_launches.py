"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
tools/one_solve.py: per-kernel totals and the in-order launch list of the
LAST solve (from its nx_kernel launch on)."""
import csv, sys
from collections import OrderedDict

rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for rec in csv.DictReader(lines):
    if rec["Metric Name"] != "gpu__time_duration.sum":
        continue
    ns = float(rec["Metric Value"].replace(",", ""))
    if rec["Metric Unit"] == "us":
        ns *= 1e3
    elif rec["Metric Unit"] == "ms":
        ns *= 1e6
    rows.append((rec["Kernel Name"], rec["Grid Size"], rec["Block Size"], ns))
starts = [i for i, r in enumerate(rows) if r[0].startswith("nx_kernel")]
rows = rows[starts[-1]:] if starts else rows
short = lambda k: k.split("(")[0].replace("void ", "").replace("lcsg::", "")
tot = OrderedDict()
for k, g, b, ns in rows:
    e = tot.setdefault(short(k), [0.0, 0])
    e[0] += ns; e[1] += 1
total = sum(r[3] for r in rows)
print(f"one solve: {len(rows)} launches, {total / 1e3:.1f} us summed (cold-cache, serialised)")
print(f"{'kernel':48s} {'launches':>8s} {'us':>10s} {'share':>6s}")
for k, (ns, cnt) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:48s} {cnt:8d} {ns / 1e3:10.1f} {100 * ns / total:5.1f}%")
print("\nin order:")
for k, g, b, ns in rows:
    print(f"{short(k):48s} grid {g:>16s} block {b:>12s} {ns / 1e3:9.1f} us")
