#!/bin/bash
# Image-path iteration under gpurun: image-BAD parity (normal + debug build), kbench c1/c0,
# optional ncu capture.  bash tools/c1_run.sh TAG [ncu]
mkdir -p gpurun_out
T=${1:-c1}
timeout 900 python -m pytest tests -m gpu -q -x -k "bad and not patch" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_$T.log)"
BINDESC_DEBUG=1 timeout 900 python -m pytest tests -m gpu -q -x -k "bad and not patch" > gpurun_out/pytest_${T}d.log 2>&1; echo "pytest dbg rc=$? $(tail -1 gpurun_out/pytest_${T}d.log)"
timeout 300 python tools/kbench.py --which c1,c0 --reps 20 > gpurun_out/kbench_$T.jsonl 2>&1; echo kb rc=$?; cat gpurun_out/kbench_$T.jsonl
true
[ -n "$2" ] && { timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:integral|bad_image' -s 4 -c 4 -o gpurun_out/ncu_c1_$T -f \
    python tools/prof_one.py c1 2 > gpurun_out/ncu_c1_$T.log 2>&1; echo ncu rc=$?; }
true
