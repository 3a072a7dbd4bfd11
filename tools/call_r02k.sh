set -u
T=r02k
export EXTRA=""
bash tools/ab2.sh $T "default ad0 ad0w128 fill4k r16 r64" "c4_10m c3_1m"
