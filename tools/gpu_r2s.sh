# End-of-round evidence after the score epilogue change: default bench (config 3 + reference arm),
# step launch list, ncu --set full of layer 2's score launch.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_int4.json 2> gpurun_out/bench_int4.err; echo "bench rc=$?"
timeout 900 python bench.py --kv-heads 8 --ctx 131072 --batch 16 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
TAG=r2s DTS=int4 KREGEX=score SKIP=2 COUNT=1 bash tools/gpu_prof.sh
