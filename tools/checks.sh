#!/bin/bash
# GPU box: the GPU parity tests against a -DPD_CHECKS build of libpd (device bounds asserts on the on-chip arrays:
# removed-slot list, plane / vertex slots and triplets, queue slots, tier-1 topology records).  compute-sanitizer
# is closed on this GPU pool, so this is the memory-safety evidence for code changed after profiles/r2_sanitizer.md.
#   bash tools/checks.sh  -> gpurun_out/checks.log
mkdir -p gpurun_out
[ -f paper_2605_06408_b200/libpd_checks.so ] || python tools/ab.py build checks PD_CHECKS > /dev/null
PD_LIB=paper_2605_06408_b200/libpd_checks.so timeout 1800 python -m pytest tests -m gpu -q -x \
    -k "not full_size_sampled" > gpurun_out/checks.log 2>&1
echo "rc=$?" >> gpurun_out/checks.log
tail -3 gpurun_out/checks.log
