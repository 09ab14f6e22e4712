#!/bin/bash
# Patch-kernel iteration under gpurun: patch parity (normal + debug build), kbench c2/c4, and with a
# second argument an ncu --set full capture of the c2 patch kernel.  bash tools/tc_run.sh TAG [ncu]
mkdir -p gpurun_out
T=${1:-tc}
timeout 600 python -m pytest tests -m gpu -q -x -k "patch or warped" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_$T.log)"
BINDESC_DEBUG=1 timeout 600 python -m pytest tests -m gpu -q -x -k "patch" > gpurun_out/pytest_${T}d.log 2>&1; echo "pytest dbg rc=$? $(tail -1 gpurun_out/pytest_${T}d.log)"
timeout 300 python tools/kbench.py --which c2,c4 --reps 20 > gpurun_out/kbench_$T.jsonl 2>&1; echo kb rc=$?; cat gpurun_out/kbench_$T.jsonl
[ -n "$2" ] && { timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:bad_patch' -s 1 -c 1 -o gpurun_out/ncu_c2_$T -f \
    python tools/prof_one.py c2 2 > gpurun_out/ncu_c2_$T.log 2>&1; echo ncu rc=$?; }
true
