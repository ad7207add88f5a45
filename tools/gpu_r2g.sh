# Evidence after the paired-head GQA bounds: config 4 bench line, its step launch list and an
# ncu --set full capture of layer 2's bounds launch.
set -x
mkdir -p gpurun_out
[ -n "$SKIP_BENCH" ] || timeout 900 python bench.py --kv-heads 8 --ctx 131072 --batch 16 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
TAG=r2g DTS=int4 KREGEX=bounds SKIP=2 COUNT=1 ARGS="--kv-heads 8 --ctx 131072 --batch 16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --sub none" bash tools/gpu_prof.sh
