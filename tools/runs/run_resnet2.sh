timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 500 > gpurun_out/tests_mp.txt 2>&1; tail -2 gpurun_out/tests_mp.txt
timeout 600 python tools/train_resnet.py --batch 64 --steps 30 --warmup 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N1', round(d['value']), round(d['ms_per_step'],2))"
for flag in "" "--no-average"; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/train_resnet.py --batch 64 --steps 30 --warmup 10 $flag 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N2 $flag', round(d['value']), round(d['ms_per_step'],2), d['allreduce_ms'], d['replicas_identical'])"
done
