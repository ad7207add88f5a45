# Iteration helper: selected GPU tests ($TESTS), then bench lines ($BENCHES, ';'-separated arg lists)
set -x
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then timeout ${TEST_TO:-900} python -m pytest $TESTS -x -q -p no:cacheprovider > gpurun_out/iter_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/iter_tests.log; fi
IFS=';' read -ra BL <<< "$BENCHES"
i=0
for b in "${BL[@]}"; do
  timeout 900 python bench.py $b > gpurun_out/iter_bench_$i.json 2> gpurun_out/iter_bench_$i.err; echo "bench $i rc=$?"
  python - "$i" <<'PY'
import json, sys
i = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/iter_bench_{i}.json").read().strip().splitlines()[-1])
    pk = {k: round(v["ms_per_step"], 3) for k, v in d.get("per_kernel", {}).items()}
    print(i, d["config"]["workload"], "tok/s", round(d["value"], 1), "ms", round(d["ms_per_step"], 3), "e2e", round(d.get("e2e", {}).get("value", 0), 1), pk, "parity", d.get("parity", {}).get("set_mismatches"), d.get("parity", {}).get("max_rel_err"), "frac", round(d["roofline"]["frac"], 3), d["roofline"]["kernel"])
except Exception as e:
    print(i, "parse error", e); print(open(f"gpurun_out/iter_bench_{i}.err").read()[-3000:])
PY
  i=$((i+1))
done
