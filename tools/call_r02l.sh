set -u
T=r02l
export EXTRA=""
bash tools/ab2.sh $T "b2 b2r64 r64 r128 r64w512" "c4_10m c3_1m"
