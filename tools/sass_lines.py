"""Per-source-line instruction and stall shares of one kernel: joins an ncu
SASS source page (--page source --csv --print-source sass) with nvdisasm
--print-line-info output of the same cubin function.
Usage: python tools/sass_lines.py page.csv cubin_li.sass source.cu [N] [func-substring]
(cubin_li.sass = nvdisasm --print-line-info -c of the whole cubin; the
function is cut from its label to the next function label)"""
import collections, csv, re, sys

page, li, src_path = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
func = sys.argv[5] if len(sys.argv) > 5 else None
lines = open(li).read().split("\n")
if func:
    labels = [i for i, l in enumerate(lines) if re.match(r"^_Z\w+:$", l)]
    start = next(i for i in labels if func in lines[i])
    end = next((i for i in labels if i > start), len(lines))
    lines = lines[start:end]
cur, off2line = None, {}
for l in lines:
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        cur = int(m.group(2)) if m.group(1).endswith(src_path.split("/")[-1]) else -int(m.group(2))
    m2 = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m2 and cur is not None:
        off2line[int(m2.group(1), 16)] = cur
rows = list(csv.reader(open(page)))
hdr, data = rows[1], rows[2:]
ia, sa, ad, ti = (hdr.index(k) for k in ("Instructions Executed", "Warp Stall Sampling (All Samples)",
                                          "Address", "Thread Instructions Executed"))
base = int(data[0][ad], 16)
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for r in data:
    ln = off2line.get(int(r[ad], 16) - base, -1)
    agg[ln][0] += float(r[ia] or 0)
    agg[ln][1] += float(r[sa] or 0)
    agg[ln][2] += float(r[ti] or 0)
tot = sum(v[0] for v in agg.values()) or 1
st = sum(v[1] for v in agg.values()) or 1
src = open(src_path).read().split("\n")
print(f"total warp instructions {tot:.4g}, stall samples {st:.0f}")
for ln, (e, s, t) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    text = src[ln - 1].strip()[:70] if 0 < ln <= len(src) else "(other file)"
    print(f"{ln:5d} instr {100 * e / tot:5.1f}% thr/inst {t / max(e, 1):4.1f} stall {100 * s / st:5.1f}%  {text}")
