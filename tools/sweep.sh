#!/bin/bash
# Throughput sweep for DESIGN §7: context and batch at INT4, planted and random KV.
# One JSON line per point -> gpurun_out/sweep/*.json, a summary table on stdout.
mkdir -p gpurun_out/sweep
run() {  # name, args...
  local name=$1; shift
  timeout 900 python bench.py --steps 20 --no-cpu-baseline --sub "" "$@" > gpurun_out/sweep/$name.json 2> gpurun_out/sweep/$name.err
  python - "$name" <<'PY'
import json, sys
name = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/sweep/{name}.json").read().strip().splitlines()[-1])
    pk = {k: round(v["ms_per_step"], 2) for k, v in d["per_kernel"].items()}
    print(f"| {name} | {d['ms_per_step']:.2f} | {d['value']:.1f} | {d['e2e']['value']:.1f} | "
          f"{d['roofline']['frac']:.2f} | {d.get('candidate_fraction')} | {pk} |")
except Exception as e:  # noqa: BLE001
    print(f"| {name} | failed: {e} |")
PY
}
for c in 16384 32768 65536 131072; do run ctx${c}_b8 --ctx $c --batch 8; done
for b in 1 2 4 16; do run ctx65536_b$b --ctx 65536 --batch $b; done
run ctx65536_b8_random --ctx 65536 --batch 8 --data random
run ctx32768_b4_bf16_random --ctx 32768 --batch 4 --dtype bf16 --data random
