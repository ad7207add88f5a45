# ncu evidence for bench.py (INT4 config 3 + bf16): launch list (cold, serialised) and
# --set full captures of each hot kernel on a layer >= 2 launch.  Never a bench number.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r1}
ARGS=${ARGS:-"--steps 2 --warmup 3 --no-cpu-baseline --no-e2e"}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_${TAG}_int4.csv python bench.py $ARGS > gpurun_out/ncu_launch_int4.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_${TAG}_bf16.csv python bench.py --dtype bf16 --batch 4 $ARGS > gpurun_out/ncu_launch_bf16.log 2>&1; echo "launch bf16 rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'score_i4mma_kernel|attn_i4_kernel|bounds_tma_kernel|topk_select3_kernel|plan_kernel|qprep_kernel|kv_quant_kernel' \
  -s 60 -c 7 -o gpurun_out/full_${TAG}_int4 -f python bench.py $ARGS > gpurun_out/ncu_full_int4.log 2>&1; echo "full rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'score_tma_kernel|attn_split16_kernel' \
  -s 10 -c 2 -o gpurun_out/full_${TAG}_bf16 -f python bench.py --dtype bf16 --batch 4 $ARGS > gpurun_out/ncu_full_bf16.log 2>&1; echo "full bf16 rc=$?"
ls -la gpurun_out
# export on the box (gpurun copies back <= 64 MiB): raw + source pages as CSV, drop big reports
for r in gpurun_out/full_${TAG}_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.source.csv 2>/dev/null
  gzip -f $b.source.csv
  sz=$(stat -c %s $r); if [ $sz -gt 20000000 ]; then rm -f $r; fi
done
gzip -f gpurun_out/launches_${TAG}_*.csv
du -sh gpurun_out; ls -la gpurun_out
