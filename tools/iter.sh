#!/bin/bash
# One build -> measure iteration on the GPU box (run under gpurun):
#   bash tools/iter.sh TAG "pytest -k expr" "kbench workloads" "ncu workloads"
# e.g. bash tools/iter.sh r02b "patch or warped" c2,c4 "c2"
TAG=$1; TESTS=${2:-}; KB=${3:-c2}; NCU=${4:-}
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -k "$TESTS" > gpurun_out/pytest_${TAG}.log 2>&1
  echo "pytest rc=$? $(tail -1 gpurun_out/pytest_${TAG}.log)"
fi
timeout 600 python tools/kbench.py --which $KB --reps 20 > gpurun_out/kbench_${TAG}.jsonl 2>&1
echo "kbench rc=$?"; cat gpurun_out/kbench_${TAG}.jsonl
for w in $NCU; do
  case $w in
    c2) k='regex:bad_patch'; n=1;;
    c3) k='regex:sift|project'; n=2;;
    c4) k='regex:warp_nn|bad_patch|sift|project'; n=4;;
    c1) k='regex:integral|bad_image'; n=3;;
  esac
  timeout 900 ncu --set full --clock-control none --import-source on -k "$k" -s $n -c $n -o gpurun_out/ncu_${w}_${TAG} -f \
    python tools/prof_one.py $w 2 > gpurun_out/ncu_${w}_${TAG}.log 2>&1
  echo "ncu $w rc=$?"
done
