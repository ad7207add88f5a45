# Round evidence: full bench (default INT4 config 3 + bf16 B=4), smoke, ncu launch lists and
# full captures of each hot kernel (layer >= 2) -> gpurun_out/
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_int4.json 2> gpurun_out/bench_int4.err; echo "bench rc=$?"
timeout 900 python bench.py --dtype bf16 --batch 4 --no-cpu-baseline > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err; echo "bench bf16 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
TAG=${TAG:-r1} KREGEX="score|attn|bounds|select|plan|qprep" SKIP=${SKIP:-12} COUNT=${COUNT:-6} bash tools/gpu_prof.sh
