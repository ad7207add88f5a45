#!/bin/bash
# A/B library variants of the selector by phase timing: bash tools/ab_phases.sh def var/X/lib.so ...
cp paper_2506_20187_b200/lib/libkvtier_b200.so /tmp/def.so
for v in "$@"; do
  if [ "$v" = def ]; then cp /tmp/def.so paper_2506_20187_b200/lib/libkvtier_b200.so; else cp "$v" paper_2506_20187_b200/lib/libkvtier_b200.so; fi
  echo "== $v"
  python tools/select_phases.py ${PHASE_ARGS:---layers-probe 0,2} 2>&1 | tail -18
done
cp /tmp/def.so paper_2506_20187_b200/lib/libkvtier_b200.so
