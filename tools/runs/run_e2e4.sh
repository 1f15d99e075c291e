# 4 GPUs: bench e2e with NUMA-local host buffers (twice per N), overlap diagnostics
mkdir -p gpurun_out
s() { python -c "import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us', d['config']['algo'], 'e2e', round(d['e2e']['value'],2), round(d['e2e']['ms_per_step'],2), 'ms', d['e2e'].get('host'))"; }
for rep in 1 2; do
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n --steps 50 --warmup 5 > gpurun_out/e2_n$n.json 2> gpurun_out/e2_n$n.err; s gpurun_out/e2_n$n.json
done; done
CUDA_VISIBLE_DEVICES=1 timeout 600 python bench.py --steps 50 --no-cpu-baseline > gpurun_out/e2_n1.json 2> gpurun_out/e2_n1.err; s gpurun_out/e2_n1.json
b=64
rn() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/train_resnet.py --batch $b --steps 40 --warmup 10 "$@" 2> gpurun_out/rn_err.txt > gpurun_out/rn_out.txt; python -c "import json,sys; d=json.loads(open('gpurun_out/rn_out.txt').read().strip().splitlines()[-1]); print('N$n b$b $*', round(d['value']), round(d['ms_per_step'],2), 'hook_ms', round(d.get('overlap_hook_host_ms',0),3), d['replicas_identical'])" || tail -3 gpurun_out/rn_err.txt; }
rn 2
rn 2 --overlap --overlap-dry
rn 2 --overlap --overlap-dry-kernel
rn 2 --overlap
