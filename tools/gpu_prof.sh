# ncu evidence for bench.py's decode step (KVT_PROFILE_RANGE=1 + --profile-from-start off:
# only the timed region's launches).  Launch list (cold, serialised) and --set full
# captures of each hot kernel.  Never a bench number.  Outputs are exported on the box
# (gpurun copies back <= 64 MiB).
set -x
mkdir -p gpurun_out
TAG=${TAG:-r1}
ARGS=${ARGS:-"--steps 1 --warmup 3 --no-cpu-baseline --no-e2e"}
export KVT_PROFILE_RANGE=1
for DT in ${DTS:-int4 bf16}; do
  if [ $DT = bf16 ]; then X="--dtype bf16 --batch 4"; else X="--dtype int4"; fi
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_${DT}.csv python bench.py $X $ARGS > gpurun_out/ncu_launch_${DT}.log 2>&1; echo "launch $DT rc=$?"
  timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"${KREGEX:-score|attn|bounds|select|plan|qprep}" -s ${SKIP:-64} -c ${COUNT:-6} \
    -o gpurun_out/full_${TAG}_${DT} -f python bench.py $X $ARGS > gpurun_out/ncu_full_${DT}.log 2>&1; echo "full $DT rc=$?"
done
for r in gpurun_out/full_${TAG}_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.source.csv 2>/dev/null; gzip -f $b.source.csv
  sz=$(stat -c %s $r); if [ $sz -gt 15000000 ]; then rm -f $r; fi
done
gzip -f gpurun_out/launches_${TAG}_*.csv
du -sh gpurun_out
