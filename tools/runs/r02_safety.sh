#!/bin/bash
# Round 2, first GPU contact after the loopback rework (the r02 GPU faults came from
# loopback ranks freeing regions peers still stored into; fixed by the region
# refcount + abort-gated kernels). compute-sanitizer memcheck first: an invalid
# access is reported by the tool instead of reaching the MMU. Stop at the first
# finding; only then the plain runs.
set -u
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
# 0. the C ABI alone (no Python / PyTorch): tools/lb_abi (built here if missing)
[ -x tools/lb_abi ] || nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/lb_abi.cu \
    -Lpaper_1902_00465_b200 -lrp -Xlinker -rpath,'$ORIGIN/../paper_1902_00465_b200' -o tools/lb_abi
for w in 2 4 8; do
  timeout 600 $S --tool memcheck --error-exitcode 9 --print-limit 20 tools/lb_abi $w 24 1 \
      > gpurun_out/r02_memcheck_lbabi_w$w.log 2>&1
  rc=$?
  echo "memcheck lb_abi W=$w rc=$rc"; tail -3 gpurun_out/r02_memcheck_lbabi_w$w.log
  [ $rc -ne 0 ] && exit $rc
done
for w in 2 8; do
  timeout 300 tools/lb_abi $w 200 7 > gpurun_out/r02_lbabi_w$w.log 2>&1
  rc=$?; echo "lb_abi W=$w rc=$rc"; tail -2 gpurun_out/r02_lbabi_w$w.log
  [ $rc -ne 0 ] && exit $rc
done
# 1. the same through Python / PyTorch (tools/dbg/lb_seq.py)
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
