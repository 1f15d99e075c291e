# 4-GPU: all GPU tests (multi-process at world 4 + single-GPU virtual) and ResNet-50 views / overlap variants
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/v_tests.txt 2>&1; tail -3 gpurun_out/v_tests.txt
b=64
rn() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/train_resnet.py --batch $b --steps 40 --warmup 10 "$@" 2> gpurun_out/rn_err.txt > gpurun_out/rn_out.txt; python -c "import json,sys; d=json.loads(open('gpurun_out/rn_out.txt').read().strip().splitlines()[-1]); print('N$n b$b $*', round(d['value']), round(d['ms_per_step'],2), 'exchange', round(d['allreduce_ms'],3), 'buckets', d.get('buckets'), d['replicas_identical'])" || tail -3 gpurun_out/rn_err.txt; }
rn 4 --no-grad-views
rn 4
rn 4 --overlap --overlap-blocks 32
rn 4 --overlap --overlap-blocks 0
rn 4 --overlap --overlap-blocks 32 --bucket-mb 25
rn 4 --fused
rn 2 --no-grad-views
rn 2
rn 2 --overlap
