#!/bin/bash
# Round 2, batch 1 (after r02_safety.sh passed): the GPU suites, the N=1 bench A/B
# (flat register form / flat bulk-copy form / round-1 two-shot), launch list + one
# ncu --set full capture of the flat kernel, and the BN bench.
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/test_gpu_world_loopback.py -q -p no:cacheprovider --timeout 900 --durations=15 \
    > gpurun_out/r02_pytest_loopback.log 2>&1
echo "loopback pytest rc=$?"; tail -3 gpurun_out/r02_pytest_loopback.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 --durations=10 \
    --deselect tests/test_gpu_world_loopback.py > gpurun_out/r02_pytest_gpu.log 2>&1
echo "gpu pytest rc=$?"; tail -3 gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
echo "smoke rc=$?"
for v in flat bulk rank; do
  for i in 1 2; do
    case $v in
      flat) E="";;
      bulk) E="RP_VFLAT_BULK=1";;
      rank) E="RP_VIRTUAL_ALGO=rank";;
    esac
    env $E timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 \
        > gpurun_out/r02_bench_$v$i.json 2> gpurun_out/r02_bench_$v$i.err
    echo "bench $v $i rc=$?"; python -c "import json,sys; d=json.loads(open('gpurun_out/r02_bench_$v$i.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['step_ms_median'], d['roofline']['frac'], d['config']['algo'])"
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02_launches_bench_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/r02_ncu_launches.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ar_virtual_flat -s 3 -c 1 \
    -o gpurun_out/r02_flat_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/r02_ncu_full.log 2>&1
echo "ncu full rc=$?"
timeout 600 python tools/bench_bn.py > gpurun_out/r02_bn_bench_n1.txt 2>&1
RP_BN_SMALL=1 timeout 600 python tools/bench_bn.py > gpurun_out/r02_bn_bench_n1_small.txt 2>&1
echo "bn bench rc=$?"; tail -25 gpurun_out/r02_bn_bench_n1.txt
