# A/B: var/base (previous build) vs the in-tree build: config 3 twice interleaved, 64K B = 1;
# then the selection / decoder GPU tests on the in-tree build.
set -x
bash tools/ab_libs.sh var/base/libkvtier_b200.so def var/base/libkvtier_b200.so def
AB_ARGS="--batch 1" bash tools/ab_libs.sh var/base/libkvtier_b200.so def
timeout 900 python -m pytest tests -m gpu -x -q -k "${AB_TESTS:-plan or select or decoder or dropin or kernels}" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab.log
