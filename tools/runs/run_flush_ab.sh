for f in write write+read; do
timeout 600 python bench.py --steps 100 --flush $f --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N1 $f', round(d['ms_per_step']*1e3,1), 'us', round(d['per_gpu_busbw_gbs'],1), 'frac', round(d['roofline']['frac'],3))"
for n in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus $n --steps 100 --warmup 5 --e2e-steps 2 --flush $f 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N$n $f', d['config']['algo'], round(d['ms_per_step']*1e3,1), 'us', round(d['per_gpu_busbw_gbs'],1), 'frac', round(d['roofline']['frac'],3))"
done; done
