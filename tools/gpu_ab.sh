# A/B: var/base (previous build) vs the in-tree build, config 3 twice interleaved, then config 4;
# then the INT4 / decoder GPU tests on the in-tree build.
set -x
bash tools/ab_libs.sh var/base/libkvtier_b200.so def var/base/libkvtier_b200.so def
AB_ARGS="--kv-heads 8 --ctx 131072 --batch 16" bash tools/ab_libs.sh var/base/libkvtier_b200.so def
timeout 900 python -m pytest tests -m gpu -x -q -k "int4 or decoder or i4" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab.log
