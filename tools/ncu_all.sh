#!/bin/bash
# one --set full capture per product kernel at benchmark-like sizes (run under gpurun)
#   bash tools/ncu_all.sh TAG
set -e
TAG=${1:-r01}
mkdir -p gpurun_out
for w in c2 c3 c4 c1; do python tools/prof_one.py $w 2 > gpurun_out/plain_${w}_${TAG}.log 2>&1; done
ncu --set full --clock-control none --import-source on -k regex:"bad_patch" -s 1 -c 1 -o gpurun_out/ncu_c2_${TAG} -f python tools/prof_one.py c2 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sift|project" -s 2 -c 2 -o gpurun_out/ncu_c3_${TAG} -f python tools/prof_one.py c3 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"warp_nn|bad_patch|sift|project" -s 4 -c 4 -o gpurun_out/ncu_c4_${TAG} -f python tools/prof_one.py c4 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"integral|bad_image" -s 3 -c 3 -o gpurun_out/ncu_c1_${TAG} -f python tools/prof_one.py c1 2 > /dev/null 2>&1
echo done
