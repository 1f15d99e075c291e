# 4 GPUs, final state: whole GPU suite (world 4), bench N=2 / N=4 lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/z4_tests.txt 2>&1; tail -1 gpurun_out/z4_tests.txt
s() { python -c "import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us', d['config']['algo'], round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2), d['clocks']['reasons'])"; }
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --steps 100 --warmup 10 > gpurun_out/z4_n$n.json 2> gpurun_out/z4_n$n.err; s gpurun_out/z4_n$n.json
done
