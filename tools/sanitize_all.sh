#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py -> gpurun_out/sanitize_*.log
mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $t python tools/sanitize.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|SYNCCHECK SUMMARY|sanitize run ok|Error|error" gpurun_out/sanitize_$t.log | head -5
done
