#!/bin/bash
# Sanitizer substitute (compute-sanitizer is closed on this pool): the whole GPU
# test suite and tools/sanitize_cases.py on the CHECKING build (every device
# allocation poisoned with 0xff bytes = NaN / -1, device bounds checks that trap).
TAG=${1:-chk}
OUT=gpurun_out/$TAG; mkdir -p $OUT
cp paper_1009_4975_b200/libtomesh.so /tmp/lib_keep.so
cp ab/lib_debug.so paper_1009_4975_b200/libtomesh.so
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_checking_build.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_checking_build.log
timeout 600 python tools/sanitize_cases.py > $OUT/cases_checking_build.log 2>&1; echo "cases rc=$?" >> $OUT/cases_checking_build.log
# determinism under repetition (a data race shows up as run-to-run differences)
timeout 600 python tools/repeat_check.py > $OUT/repeat_checking_build.log 2>&1; echo "repeat rc=$?" >> $OUT/repeat_checking_build.log
cp /tmp/lib_keep.so paper_1009_4975_b200/libtomesh.so
tail -3 $OUT/pytest_checking_build.log; tail -3 $OUT/cases_checking_build.log; tail -8 $OUT/repeat_checking_build.log
