# 4 GPUs: two-shot with 4 packets per lane for NR <= 4 -- parity (multi-process all-reduce tests) and bench N=2 / N=4 P2P
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 -k "all_reduce_multiprocess or wrap_optimizer_sync or overlap" > gpurun_out/u4_tests.txt 2>&1; tail -1 gpurun_out/u4_tests.txt
s() { python -c "import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us', d['config']['algo'], round(d['roofline']['frac'],3))"; }
for i in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 2 > gpurun_out/u4_n2.json 2> gpurun_out/u4_n2.err; s gpurun_out/u4_n2.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --steps 100 --warmup 10 --nvls off --e2e-steps 2 > gpurun_out/u4_n4.json 2> gpurun_out/u4_n4.err; s gpurun_out/u4_n4.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py --out gpurun_out/u4_sweep.json --ops all_reduce --algos auto,nccl --min-log2 20 --max-log2 28 --iters 20 --flush > gpurun_out/u4_sweep.txt 2>&1; python tools/sweep_table.py gpurun_out/u4_sweep.json | tail -9
