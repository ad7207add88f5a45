# quick GPU loop: full -m gpu suite, then short benches (INT4 config 3, bf16 B=4) with per-stage ms
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -${TAILN:-4}
for X in "${BENCH1:---dtype int4}" "${BENCH2:---dtype bf16 --batch 4}"; do
  python bench.py $X --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(d['config']['workload'], 'ms/step %.3f' % d['ms_per_step'], 'tok/s %.1f' % d['value'], {k: (round(v['ms_per_step'],3), round(v['gbs'] or 0)) for k,v in d['per_kernel'].items()})"
done
