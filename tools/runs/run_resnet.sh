timeout 600 python -m pytest tests/test_gpu_virtual.py -q -x -k "wrap or replicator" --timeout 300 2>&1 | tail -1
for b in 64 256; do
timeout 600 python tools/train_resnet.py --batch $b --steps 30 --warmup 10 --out gpurun_out/rn50_n1_b$b.json 2> /dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N1 b$b', round(d['value']), round(d['ms_per_step'],2))"
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/train_resnet.py --batch $b --steps 30 --warmup 10 --out gpurun_out/rn50_n${n}_b$b.json 2> /dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N$n b$b', round(d['value']), round(d['ms_per_step'],2), round(d['allreduce_ms'],3), d['replicas_identical'])"
done; done
