# 4-GPU: overlap test, ResNet-50 overlap with grid caps (+diagnose), NCCL comparison sweep, BN with clean-L2 flush
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 300 -k "overlap" > gpurun_out/ov2_tests.txt 2>&1; tail -3 gpurun_out/ov2_tests.txt
b=64
rn() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/train_resnet.py --batch $b --steps 40 --warmup 10 "$@" 2> gpurun_out/rn_err.txt > gpurun_out/rn_out.txt; python -c "import json,sys; d=json.loads(open('gpurun_out/rn_out.txt').read().strip().splitlines()[-1]); print('N$n b$b $*', round(d['value']), round(d['ms_per_step'],2), 'exchange', round(d['allreduce_ms'],3), 'buckets', d.get('buckets'), d['replicas_identical'])" || tail -3 gpurun_out/rn_err.txt; }
rn 4
rn 4 --overlap --overlap-blocks 16
rn 4 --overlap --overlap-blocks 32
rn 4 --overlap --overlap-blocks 64 --bucket-mb 16
rn 4 --overlap --overlap-blocks 32 --diagnose; grep "rank 0" gpurun_out/rn_out.txt | head -4
rn 4 --diagnose; grep "rank 0" gpurun_out/rn_out.txt | head -4
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py --out gpurun_out/sweep_nccl_n4.json --ops all_reduce,all_gather,broadcast --algos auto,nccl,nvls --min-log2 12 --max-log2 28 --iters 20 --flush > gpurun_out/sweep_nccl_n4.txt 2>&1; grep -c GB gpurun_out/sweep_nccl_n4.txt
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/bench_bn.py --dtype f32 > gpurun_out/bn_f32_clean.txt 2>&1; cat gpurun_out/bn_f32_clean.txt | head -24
