set -u
T=r02n
export EXTRA=""
bash tools/ab2.sh $T "r1k r4k" "c4_10m"
bash tools/ab2.sh $T "r32 r512 r4k" "c5_set c7552"
