#!/bin/bash
# The CPU oracle's pins under AddressSanitizer + UndefinedBehaviorSanitizer
# (compute-sanitizer is closed on the GPU pool; this covers the host C code).
cd "$(dirname "$0")/.."
export ORACLE_SANITIZE=1 ASAN_OPTIONS=detect_leaks=0:abort_on_error=1 UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1
export LD_PRELOAD="$(gcc -print-file-name=libasan.so)"
exec python -m pytest tests/test_oracle_pins.py tests/test_batch_policy.py tests/test_next4.py -q -p no:cacheprovider "$@"
