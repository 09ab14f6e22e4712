#!/bin/bash
# One gpurun call that refreshes the round's evidence (run from the repo root under gpurun):
#   bash tools/evidence.sh r02x
# GPU tests, the default bench line, per-workload kernel timings, the configs[4] launch list and
# --set full captures (c4 step, c2, c3, c1, the matcher m1), and the parity report.  Outputs in gpurun_out/.
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi_${TAG}.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu_${TAG}.log)"
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
timeout 600 python tools/kbench.py --reps 20 > gpurun_out/kbench_${TAG}.jsonl 2>&1
echo "kbench rc=$?"
timeout 900 bash tools/ncu_c4.sh ${TAG} > /dev/null 2>&1
echo "ncu c4 rc=$?"
for w in c2 c3 c1 m1; do
  case $w in
    c2) k='regex:bad_patch'; n=1;;
    c3) k='regex:sift|project'; n=2;;
    c1) k="regex:integral|bad_image"; n=4;;
    m1) k='regex:match_kernel'; n=1;;
  esac
  timeout 600 ncu --set full --clock-control none --import-source on -k "$k" -s $n -c $n -o gpurun_out/ncu_${w}_${TAG} -f \
    python tools/prof_one.py $w 2 > gpurun_out/ncu_${w}_${TAG}.log 2>&1
  echo "ncu $w rc=$?"
done
timeout 900 python tools/parity_report.py --out gpurun_out/parity_${TAG}.json > gpurun_out/parity_${TAG}.log 2>&1
echo "parity rc=$?"
