# A/B: var/base vs the in-tree build at config 3 (x2), 64K B = 1 and config 4; selection tests.
set -x
bash tools/ab_libs.sh var/base/libkvtier_b200.so def var/base/libkvtier_b200.so def
AB_ARGS="--batch 1" bash tools/ab_libs.sh var/base/libkvtier_b200.so def
AB_ARGS="--kv-heads 8 --ctx 131072 --batch 16" bash tools/ab_libs.sh var/base/libkvtier_b200.so def
timeout 900 python -m pytest tests -m gpu -x -q -k "${AB_TESTS:-plan or select or decoder or dropin or kernels or gqa}" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab.log
