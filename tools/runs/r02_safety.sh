#!/bin/bash
# Round 2, first GPU contact after the loopback rework (the r02 GPU faults came from
# loopback ranks freeing regions peers still stored into; fixed by the region
# refcount + abort-gated kernels). compute-sanitizer memcheck first: an invalid
# access is reported by the tool instead of reaching the MMU. Stop at the first
# finding; only then the plain runs.
set -u
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for w in 2 4 8; do
  TMO=60 PINNED=1 W=$w N=24 timeout 900 $S --tool memcheck --error-exitcode 9 --print-limit 20 \
      python tools/dbg/lb_seq.py > gpurun_out/r02_memcheck_lbseq_w$w.log 2>&1
  rc=$?
  echo "memcheck lb_seq W=$w rc=$rc"; tail -4 gpurun_out/r02_memcheck_lbseq_w$w.log
  [ $rc -ne 0 ] && exit $rc
done
for w in 2 8; do
  PINNED=1 W=$w N=80 timeout 300 python tools/dbg/lb_seq.py > gpurun_out/r02_lbseq_w$w.log 2>&1
  rc=$?; echo "lb_seq W=$w rc=$rc"; tail -2 gpurun_out/r02_lbseq_w$w.log
  [ $rc -ne 0 ] && exit $rc
done
exit 0
