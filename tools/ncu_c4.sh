#!/bin/bash
# ncu evidence for the configs[4] step (run under gpurun from the repo root).
#   1. the plain command must exit 0 first (B200_PROFILING.md)
#   2. launch list with device times (cold-cache, serialised: compare SHARES)
#   3. one --set full capture of each kernel of one timed step (256,000 keypoints: 64 images)
# 64 images x 4000 keypoints = 256,000 keypoints = one internal chunk per step; each step
# launches warp_nn, bad_patch, zero_invalid, sift, project, zero_invalid.  -s 12 skips the
# 3 warm-up steps of the 4 filtered kernels.
set -e
TAG=${1:-r01}
CMD="python bench.py --images 64 --steps 2 --warmup 3 --no-cpu-baseline --no-per-config --e2e-images 1"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_${TAG}.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"warp_nn|bad_patch|sift|project" \
    -s 12 -c 4 -o gpurun_out/prof_${TAG} -f $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo done
