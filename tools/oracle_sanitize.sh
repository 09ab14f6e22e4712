#!/bin/bash
# The CPU oracle's pin tests under AddressSanitizer + UndefinedBehaviorSanitizer:
# the oracle is rebuilt as oracle/liboracle_san.so with -fsanitize=address,undefined and the
# runtime is preloaded into the Python process.  Any report aborts the run (UBSan: no recover).
#   bash tools/oracle_sanitize.sh [pytest -k expression]
set -e
cd "$(dirname "$0")/.."
export BINDESC_ORACLE_SANITIZE=1
export ASAN_OPTIONS=detect_leaks=0:abort_on_error=1
export UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1
export LD_PRELOAD="$(gcc -print-file-name=libasan.so):$(gcc -print-file-name=libubsan.so)"
python -m pytest tests -q -m "not gpu" -k "${1:-oracle or synth}" -p no:cacheprovider
