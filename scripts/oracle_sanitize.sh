# Host sanitizers over the oracle: AddressSanitizer + UBSan build of
# oracle/tc_oracle.c, every CPU pin test run through it.  Usage: bash scripts/oracle_sanitize.sh
set -e
export TC_ORACLE_SANITIZE=1
export ASAN_OPTIONS=detect_leaks=0:abort_on_error=1
export UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1
export OMP_NUM_THREADS=4
LD_PRELOAD=$(gcc -print-file-name=libasan.so):$(gcc -print-file-name=libubsan.so) \
    python -m pytest tests/test_oracle_pins.py tests/test_oracle_pins_next.py -q -p no:cacheprovider "$@"
