# A/B at config 4 (GQA) and config 3: var/base vs the in-tree build; then GQA / bounds GPU tests.
set -x
AB_ARGS="--kv-heads 8 --ctx 131072 --batch 16" bash tools/ab_libs.sh var/base/libkvtier_b200.so def var/base/libkvtier_b200.so def
[ -n "$NO_CFG3" ] || bash tools/ab_libs.sh var/base/libkvtier_b200.so def
timeout 900 python -m pytest tests -m gpu -x -q -k "${AB_TESTS:-gqa or bound or decoder or shard or tier}" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab.log
