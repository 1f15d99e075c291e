# relay broadcast with role-split blocks: tests + A/B at N=2/4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 -k "relay or gather_broadcast" > gpurun_out/rl3_tests.txt 2>&1; tail -1 gpurun_out/rl3_tests.txt
for n in 4 2; do
for cfg in "2 64" "1 64" "2 128"; do
set -- $cfg
RP_RELAY_OCC=$1 RP_RELAY_TILE_KB=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n tools/sweep.py --out gpurun_out/rab.json --ops broadcast --algos auto,nccl --min-log2 22 --max-log2 28 --iters 10 --flush > gpurun_out/rab.txt 2>&1
python -c "
import json; d=json.load(open('gpurun_out/rab.json'))
print('N$n occ $1 tile $2 KiB relay', ' '.join(f\"{r['bytes']>>20}MiB={r['us']:.1f}\" for r in d['rows'] if r['algo']=='relay'))
print('N$n nccl                     ', ' '.join(f\"{r['bytes']>>20}MiB={r['us']:.1f}\" for r in d['rows'] if r['algo']=='nccl'))" || tail -3 gpurun_out/rab.txt
done; done
