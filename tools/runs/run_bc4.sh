# 4 GPUs: multi-process tests (push broadcast / all_gather), small-message sweep vs NCCL, ResNet overlap host-time diag
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 > gpurun_out/bc_tests.txt 2>&1; tail -3 gpurun_out/bc_tests.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py --out gpurun_out/sweep_small_n4.json --ops all_gather,broadcast --algos auto,nccl,nvls --min-log2 10 --max-log2 24 --iters 30 --flush > gpurun_out/sweep_small_n4.txt 2>&1; grep -c GB gpurun_out/sweep_small_n4.txt
b=64
rn() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/train_resnet.py --batch $b --steps 40 --warmup 10 "$@" 2> gpurun_out/rn_err.txt > gpurun_out/rn_out.txt; python -c "import json,sys; d=json.loads(open('gpurun_out/rn_out.txt').read().strip().splitlines()[-1]); print('N$n b$b $*', round(d['value']), round(d['ms_per_step'],2), 'exchange', round(d['allreduce_ms'],3), 'buckets', d.get('buckets'), 'hook_ms', round(d.get('overlap_hook_host_ms',0),3), d['replicas_identical'])" || tail -3 gpurun_out/rn_err.txt; }
rn 4
rn 4 --overlap
rn 4 --overlap --bucket-mb 25
