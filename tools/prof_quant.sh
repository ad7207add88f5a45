mkdir -p gpurun_out
python tools/microbench.py quant dequant
ncu --set full --clock-control none --import-source on -k regex:'kv_quant_kernel|kv_dequant_kernel' -c 2 -o gpurun_out/full_quant -f python tools/microbench.py quant dequant --lanes 64 --n 16384 > /dev/null 2>&1
ncu -i gpurun_out/full_quant.ncu-rep --page raw --csv > gpurun_out/full_quant.raw.csv
ncu -i gpurun_out/full_quant.ncu-rep --page details --csv > gpurun_out/full_quant.details.csv
rm -f gpurun_out/full_quant.ncu-rep
timeout 600 python -m pytest tests/test_gpu_int4.py tests/test_tier.py -x -q 2>&1 | tail -3
