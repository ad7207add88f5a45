# Config 4 (LLaMA-3-8B GQA, 128K, B = 16, INT4): per-lane vs union attention A/B + ncu of layer 2's GQA kernels
set -x
mkdir -p gpurun_out
KVT_GQA_UNION=0 timeout 600 python bench.py --kv-heads 8 --ctx 131072 --batch 16 --steps 10 --no-cpu-baseline --no-e2e --sub "" > gpurun_out/c4_lane.json 2>gpurun_out/c4_lane.err; echo rc=$?
KVT_GQA_UNION=1 timeout 600 python bench.py --kv-heads 8 --ctx 131072 --batch 16 --steps 10 --no-cpu-baseline --no-e2e --sub "" > gpurun_out/c4_union.json 2>gpurun_out/c4_union.err; echo rc=$?
export KVT_PROFILE_RANGE=1 KVT_GQA_UNION=1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"gqa" -s 4 -c 2 -o gpurun_out/full_c4u -f python bench.py --kv-heads 8 --ctx 131072 --batch 16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --sub "" > gpurun_out/ncu_c4u.log 2>&1; echo rc=$?
for r in gpurun_out/full_c4*.ncu-rep; do b=${r%.ncu-rep}; ncu -i $r --page raw --csv > $b.raw.csv; ncu -i $r --page source --csv --print-source sass > $b.source.csv; gzip -f $b.source.csv; rm -f $r; done
for f in c4_lane c4_union; do python - $f <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["ms_per_step"],3), {k:(round(v["ms_per_step"],3), round(v["gbs"] or 0)) for k,v in d["per_kernel"].items()}, d.get("parity",{}).get("set_mismatches"), d.get("parity",{}).get("max_rel_err"))
PY
done
python profiles/summarize.py raw gpurun_out/full_c4u.raw.csv | head -14
