# Round-2 profiling: gather-pattern microbench (+ DRAM bytes per variant) and ncu --set full
# captures of layer 2's select and attention launches in the config-3 bench step.
set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o /tmp/gather_bench tools/gather_bench.cu
/tmp/gather_bench 4 1 > gpurun_out/gather_bench.txt 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --csv \
  --log-file gpurun_out/gather_bench_ncu.csv /tmp/gather_bench 4 1 > /dev/null 2>&1
export KVT_PROFILE_RANGE=1
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"${KREGEX:-select|attn}" -s ${SKIP:-4} -c ${COUNT:-2} \
  -o gpurun_out/full_${TAG:-r2a} -f python bench.py --dtype int4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --sub "" > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
for r in gpurun_out/full_${TAG:-r2a}*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.source.csv 2>/dev/null; gzip -f $b.source.csv
  sz=$(stat -c %s $r); if [ $sz -gt 15000000 ]; then rm -f $r; fi
done
cat gpurun_out/gather_bench.txt
du -sh gpurun_out
