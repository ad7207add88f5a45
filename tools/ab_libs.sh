#!/bin/bash
# A/B library variants on the GPU box: bash tools/ab_libs.sh def var/X/libkvtier_b200.so ...
# ("def" = the in-tree build); one bench per variant ($AB_ARGS, default 20 steps of config 3),
# per-kernel split printed.
cp paper_2506_20187_b200/lib/libkvtier_b200.so /tmp/def.so
for v in "$@"; do
  if [ "$v" = def ]; then cp /tmp/def.so paper_2506_20187_b200/lib/libkvtier_b200.so; else cp "$v" paper_2506_20187_b200/lib/libkvtier_b200.so; fi
  echo -n "$v: "
  python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-parity --sub "" ${AB_ARGS:-} 2>/dev/null | python -c '
import json, sys
d = json.loads(sys.stdin.read())
print("ms/step %.3f" % d["ms_per_step"], {k: round(v["ms_per_step"], 3) for k, v in d["per_kernel"].items()})'
done
cp /tmp/def.so paper_2506_20187_b200/lib/libkvtier_b200.so
