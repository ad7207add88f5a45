"""Summarise an ncu `--page source --csv --print-source sass` export: per kernel, the
instruction-class mix (executed warp instructions) and the hottest instructions by stall
samples.   python tools/sass_hot.py <source.csv[.gz]> [kernel-substring] [top]"""
import collections, csv, gzip, io, re, sys

path = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read()
blocks = re.split(r'^"Kernel Name","', txt, flags=re.M)[1:]
for b in blocks:
    name = b.split('"', 1)[0]
    if want not in name:
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    hdr = rows[0]
    si, ss, se = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    mix, tot_s, tot_e = collections.Counter(), 0, 0
    hot = []
    for r in rows[1:]:
        if len(r) <= se:
            continue
        op = r[si].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        o = o.split(".")[0]
        e = int(r[se] or 0); s = int(r[ss] or 0)
        mix[o] += e; tot_e += e; tot_s += s
        hot.append((s, r[si].strip()))
    print(f"== {name[:100]}  executed warp-instr {tot_e}, stall samples {tot_s}")
    print("   mix: " + ", ".join(f"{k} {100*v/tot_e:.1f}%" for k, v in mix.most_common(18)))
    for s, src in sorted(hot, reverse=True)[:top]:
        print(f"   {100*s/max(tot_s,1):5.1f}%  {src}")
