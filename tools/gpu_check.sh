#!/bin/bash
# One gpurun call: GPU parity tests, default bench line, per-workload kernel timings, ncu.
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh r01a'
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi_${TAG}.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
timeout 300 python tools/kbench.py > gpurun_out/kbench_${TAG}.jsonl 2>&1
echo "kbench rc=$?"
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 bash tools/ncu_c4.sh ${TAG}
  echo "ncu rc=$?"
fi
tail -3 gpurun_out/pytest_gpu_${TAG}.log
cat gpurun_out/bench_${TAG}.json
cat gpurun_out/kbench_${TAG}.jsonl
