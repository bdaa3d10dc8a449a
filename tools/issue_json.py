"""Issue-slot utilisation of the combine kernels for bench.py's roofline.issue_active:
reads the `smsp__issue_active` of one `ncu --set full` capture per kernel
(tools/ncu_summary.py text files) and weights them by the kernels' shares of
the launch list (tools/summarize_launches.py output).
Usage: python tools/issue_json.py launches_summary.txt label=summary.txt ... > profiles/issue_cfg5.json
A label is the kernel-name prefix it stands for in the launch list."""
import json, re, sys

summary = open(sys.argv[1]).read().split("in order:")[0].splitlines()[2:]
shares = {}
for line in summary:
    m = re.match(r"(.+?)\s+(\d+)\s+([\d.]+)\s+([\d.]+)%", line)
    if m:
        shares[m.group(1).strip()] = float(m.group(3))
kernels, wsum, tsum = {}, 0.0, 0.0
for arg in sys.argv[2:]:
    label, path = arg.split("=", 1)
    txt = open(path).read()
    pct = float(re.search(r"smsp__issue_active\S*\s+([\d.]+)", txt.replace(",", "")).group(1))
    us = sum(v for k, v in shares.items() if label in k)
    kernels[label] = {"issue_active_pct": round(pct, 1), "share_us": round(us, 1),
                      "source": path.split("/")[-1]}
    wsum += pct * us
    tsum += us
print(json.dumps({
    "note": "smsp__issue_active.avg.pct_of_peak_sustained_active of the combine kernels (one ncu "
            "--set full capture per kernel, cfg5), time-weighted by the launch-list shares",
    "kernels": kernels, "weighted_issue_active_pct": round(wsum / max(tsum, 1e-9), 1),
    "covered_us": round(tsum, 1), "all_launches_us": round(sum(shares.values()), 1)}, indent=1))
