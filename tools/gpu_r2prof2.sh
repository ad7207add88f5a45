# Round-2 evidence: launch list + ncu --set full of the config-3 step's kernels (INT4), the
# kv_quant capture, and the host-tier fetch kernel.  Outputs exported on the box.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2}
export KVT_PROFILE_RANGE=1
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --sub ''"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}_int4.csv python bench.py --dtype int4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --sub "" > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"score|attn|bounds|select|plan|qprep" -s 12 -c 6 \
  -o gpurun_out/full_${TAG}_int4 -f python bench.py --dtype int4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --sub "" > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'kv_quant_kernel' -c 2 -o gpurun_out/full_${TAG}_quant -f \
  python tools/microbench.py quant --lanes 64 --n 16384 > gpurun_out/ncu_quant.log 2>&1; echo "quant rc=$?"
python tools/microbench.py quant > gpurun_out/quant_micro.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tier_fetch|tier_touch|tier_hist|attn_ring' -s 40 -c 4 -o gpurun_out/full_${TAG}_tier -f \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --sub hosttier --ht-ctx 65536 --ht-batch 2 > gpurun_out/ncu_tier.log 2>&1; echo "tier rc=$?"
for r in gpurun_out/full_${TAG}_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.source.csv 2>/dev/null; gzip -f $b.source.csv
  rm -f $r
done
gzip -f gpurun_out/launches_${TAG}_*.csv
du -sh gpurun_out
