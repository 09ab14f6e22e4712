#!/bin/bash
# Full GPU suite, the debug-build BAD subset and one default bench line under gpurun.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_full_tc.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_full_tc.log)"
BINDESC_DEBUG=1 timeout 900 python -m pytest tests -m gpu -q -x -k "patch or bad or warped" > gpurun_out/pytest_full_tcd.log 2>&1; echo "pytest dbg rc=$? $(tail -1 gpurun_out/pytest_full_tcd.log)"
timeout 600 python bench.py > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_tc.json
