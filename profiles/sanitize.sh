#!/bin/bash
# compute-sanitizer over a small slice of the parity tests (memcheck, then racecheck on the shared-memory kernels)
sel='(field_kernel and (desk64 or field21 or closed-four) and (None-None-None-None or 3-4-1 or 1-8-0 or 1-4-1-48)) or (test_golden_digests) or (negative_zero) or (pair_kernel and desk64) or (rebuild_with_more) or (position_ordered and (desk64 or closed-ped3)) or (rebuild_skips and pairs-list)'
compute-sanitizer --tool memcheck --error-exitcode 9 --target-processes all python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "$sel" 2>&1 | tail -8
echo "memcheck exit ${PIPESTATUS[0]}"
compute-sanitizer --tool racecheck --racecheck-report analysis --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "(field_kernel and desk64 and (None-None-None-None or 3-4-1 or 1-4-1-48)) or (pair_kernel and desk64) or (position_ordered and desk64)" 2>&1 | tail -12
echo "racecheck exit ${PIPESTATUS[0]}"
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_api.py -x -q -m gpu -k "band_swapped and (desk64-2 or field35)" 2>&1 | tail -4
echo "memcheck(band) exit ${PIPESTATUS[0]}"
