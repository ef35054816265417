#!/bin/bash
# The oracle's CPU test suite against an AddressSanitizer + UndefinedBehaviorSanitizer build
# of gse_oracle.c.  Output: profiles/sanitizer_r02/oracle_asan_ubsan.log
set -u
cd "$(dirname "$0")/.."
mkdir -p profiles/sanitizer_r02
ASAN_LIB=$(gcc -print-file-name=libasan.so)
UBSAN_LIB=$(gcc -print-file-name=libubsan.so)
ORACLE_SANITIZE=1 python -c "import oracle; oracle.build(force=True)"
ORACLE_SANITIZE=1 LD_PRELOAD="$ASAN_LIB $UBSAN_LIB" ASAN_OPTIONS=detect_leaks=0:abort_on_error=1 \
  UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1 \
  timeout 1800 python -m pytest tests/test_oracle_codec.py tests/test_oracle_spmv_solvers.py \
  tests/test_oracle_half.py tests/test_oracle_sampling.py tests/test_oracle_krylov16.py -q -p no:cacheprovider \
  > profiles/sanitizer_r02/oracle_asan_ubsan.log 2>&1
echo "rc=$?" >> profiles/sanitizer_r02/oracle_asan_ubsan.log
tail -3 profiles/sanitizer_r02/oracle_asan_ubsan.log
