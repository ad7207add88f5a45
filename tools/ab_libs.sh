#!/bin/bash
# A/B library variants on the GPU box: bash tools/ab_libs.sh def var/lib_X.so ...
# ("def" = the in-tree build); one 30-step bench per variant, per-kernel split printed.
cp paper_2506_20187_b200/lib/libkvtier_b200.so /tmp/def.so
for v in "$@"; do
  if [ "$v" = def ]; then cp /tmp/def.so paper_2506_20187_b200/lib/libkvtier_b200.so; else cp "$v" paper_2506_20187_b200/lib/libkvtier_b200.so; fi
  echo -n "$v: "
  python bench.py --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | python -c '
import json, sys
d = json.loads(sys.stdin.read())
print("ms/step %.3f" % d["ms_per_step"], {k: round(v["ms_per_step"], 3) for k, v in d["per_kernel"].items()}, d["self_check_max_rel_diff"])'
done
cp /tmp/def.so paper_2506_20187_b200/lib/libkvtier_b200.so
