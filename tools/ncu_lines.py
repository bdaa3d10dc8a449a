"""Per-source-line warp instructions / thread instructions / stall samples of
one kernel from an ncu report (--page source --print-source cuda,sass).
Usage: python tools/ncu_lines.py report.ncu-rep [top N]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kfilter = sys.argv[3] if len(sys.argv) > 3 else None  # e.g. regex:narrow_combine_kernel<8
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kfilter:
    cmd += ["--kernel-id", kfilter] if kfilter.startswith(":") else ["-k", kfilter]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = []
fname = "?"
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No", "Function Name") and r[2] == "-":
        try:
            rows.append((fname, int(r[0]), r[1].strip()[:90], float(r[7] or 0), float(r[8] or 0),
                         float(r[4] or 0)))
        except ValueError:
            pass
ti = sum(x[4] for x in rows) or 1
wi = sum(x[3] for x in rows) or 1
st = sum(x[5] for x in rows) or 1
print(f"warp inst {wi:.4g}  thread inst {ti:.4g}  stall samples {st:.0f}")
print(f"{'file:line':24s} {'warp%':>6s} {'thr%':>6s} {'stall%':>6s}  source")
for f, ln, src, w, t, s in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{f + ':' + str(ln):24s} {100 * w / wi:6.2f} {100 * t / ti:6.2f} {100 * s / st:6.2f}  {src}")
