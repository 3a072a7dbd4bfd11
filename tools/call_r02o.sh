set -u
T=r02o
export EXTRA=""
bash tools/ab2.sh $T "default colreg" "c4_10m c3_1m"
EXTRA="--chunk-events 8192" SUF=_m8k bash tools/ab2.sh $T "default" "c4_10m c3_1m"
EXTRA="--chunk-events 32768" SUF=_m32k bash tools/ab2.sh $T "default" "c4_10m c3_1m"
