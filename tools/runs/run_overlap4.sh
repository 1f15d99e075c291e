# 4-GPU: multi-process tests (incl. overlap) + ResNet-50 sync vs overlapped vs fused
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 > gpurun_out/ov_tests.txt 2>&1; tail -4 gpurun_out/ov_tests.txt
b=${B:-64}
rn() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/train_resnet.py --batch $b --steps 40 --warmup 10 "$@" 2> gpurun_out/rn_err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N$n b$b $*', round(d['value']), round(d['ms_per_step'],2), 'exchange', round(d['allreduce_ms'],3), 'buckets', d.get('buckets'), d['replicas_identical'])" || tail -3 gpurun_out/rn_err.txt; }
timeout 600 python tools/train_resnet.py --batch $b --steps 40 --warmup 10 2> gpurun_out/rn_err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N1 b$b', round(d['value']), round(d['ms_per_step'],2))"
for n in 4 2; do
rn $n
rn $n --overlap
rn $n --overlap --bucket-mb 4
rn $n --overlap --bucket-mb 16
rn $n --fused
done
