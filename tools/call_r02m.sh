set -u
T=r02m
export EXTRA=""
bash tools/ab2.sh $T "r256 r512 r128s4 r128ms32" "c4_10m c3_1m"
