set -x
bash tools/ab_libs.sh var/base/libkvtier_b200.so var/s4/libkvtier_b200.so var/base/libkvtier_b200.so var/s4/libkvtier_b200.so
