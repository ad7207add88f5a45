"""Per-CUDA-source-line totals from `ncu -i rep --page source --csv --print-source cuda,sass`
(executed warp instructions and stall samples).  python tools/src_lines.py <csv> [top]"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, cur_line, cur_src = "?", None, ""
agg = collections.defaultdict(lambda: [0, 0, ""])
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a CUDA source line row
        cur_line, cur_src = r[0], r[1]
    try:
        e = int(r[hdr.index("Instructions Executed")] or 0); s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    key = (fname, cur_line)
    agg[key][0] += e; agg[key][1] += s; agg[key][2] = cur_src
te = sum(v[0] for v in agg.values()) or 1; ts = sum(v[1] for v in agg.values()) or 1
print(f"total exec {te}, stall samples {ts}")
for (f, l), (e, s, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*e/te:5.1f}% exec {100*s/ts:5.1f}% stall {f}:{l}: {src.strip()[:90]}")
