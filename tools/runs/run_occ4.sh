# 4 GPUs: two-shot at 2 blocks/SM -- parity (virtual + multi-process tests) and bench N=1/2/4; BN ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x --timeout 600 > gpurun_out/oc_vtests.txt 2>&1; tail -1 gpurun_out/oc_vtests.txt
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 > gpurun_out/oc_tests.txt 2>&1; tail -1 gpurun_out/oc_tests.txt
s() { python -c "import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us', d['config']['algo'], round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2), round(d['e2e']['ms_per_step'],2), 'ms', d['clocks']['reasons'])"; }
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 100 > gpurun_out/oc_n1.json 2> gpurun_out/oc_n1.err; s gpurun_out/oc_n1.json
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 100 --warmup 10 > gpurun_out/oc_n$n.json 2> gpurun_out/oc_n$n.err; s gpurun_out/oc_n$n.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 4 --steps 100 --warmup 10 --nvls off > gpurun_out/oc_n4p.json 2> gpurun_out/oc_n4p.err; s gpurun_out/oc_n4p.json
CUDA_VISIBLE_DEVICES=0 bash tools/runs/run_ncu_bn2.sh
