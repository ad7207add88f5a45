# Round-2 validation: -m gpu suite, smoke, default bench, reference arm -> gpurun_out/
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout ${TEST_TO:-1500} python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/r2_gputests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"
if [ -z "$NOBENCH" ]; then
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo "ref rc=$?"
fi
tail -15 gpurun_out/r2_gputests.log; cat gpurun_out/r2_smoke.log; cat gpurun_out/r2_bench.json; tail -5 gpurun_out/r2_bench.err; cat gpurun_out/r2_bench_ref.json
