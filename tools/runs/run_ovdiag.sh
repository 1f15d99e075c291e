# overlap diagnostics on 2 GPUs + overlap test; BN small-layer latency (fused vs unfused, ncu)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 300 -k "overlap or wrap" > gpurun_out/od_tests.txt 2>&1; tail -2 gpurun_out/od_tests.txt
b=64
rn() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/train_resnet.py --batch $b --steps 40 --warmup 10 "$@" 2> gpurun_out/rn_err.txt > gpurun_out/rn_out.txt; python -c "import json,sys; d=json.loads(open('gpurun_out/rn_out.txt').read().strip().splitlines()[-1]); print('N$n b$b $*', round(d['value']), round(d['ms_per_step'],2), 'exchange', round(d['allreduce_ms'],3), 'buckets', d.get('buckets'), d['replicas_identical'])" || tail -3 gpurun_out/rn_err.txt; }
rn 2
rn 2 --overlap --overlap-dry
rn 2 --overlap --overlap-priority 0
rn 2 --overlap --overlap-blocks 8
rn 2 --overlap --overlap-blocks 8 --overlap-priority 0
CUDA_VISIBLE_DEVICES=0 bash tools/runs/run_bn_small.sh
