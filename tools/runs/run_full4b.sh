# 4 GPUs: whole GPU suite (multi-process at world 4), world-2 subset, smoke, bench N=1/2/4
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/fb_tests.txt 2>&1; tail -2 gpurun_out/fb_tests.txt
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 -k "relay or gather_broadcast or host or overlap or wrap_optimizer_sync" > gpurun_out/fb_tests2.txt 2>&1; tail -1 gpurun_out/fb_tests2.txt
CUDA_VISIBLE_DEVICES=0 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
s() { python -c "import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us', d['config']['algo'], round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2), d['clocks']['reasons'])"; }
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/fb_n1.json 2> gpurun_out/fb_n1.err; s gpurun_out/fb_n1.json
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 100 --warmup 10 > gpurun_out/fb_n$n.json 2> gpurun_out/fb_n$n.err; s gpurun_out/fb_n$n.json
done
