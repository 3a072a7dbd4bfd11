set -u
T=r02q
export EXTRA=""
bash tools/ab2.sh $T "default r32ms256 r64ms256 r128 r32" "c4_10m c4_mini"
EXTRA="--ncycles 60000" SUF=_60k bash tools/ab2.sh $T "default r32ms256 r64ms256 r128 r32" "c4_mini"
EXTRA="--ncycles 60000 --wcv 1" SUF=_60kw1 bash tools/ab2.sh $T "default r32ms256 r64ms256 r128 r32" "c4_mini"
