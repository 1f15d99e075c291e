# relay broadcast A/B: blocks per SM x tile size, N=2 and N=4, 64 / 256 MiB (relay column of tools/sweep.py)
mkdir -p gpurun_out
for n in 4 2; do
for cfg in "1 64" "2 64" "2 256" "1 256" "2 16"; do
set -- $cfg
RP_RELAY_OCC=$1 RP_RELAY_TILE_KB=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n tools/sweep.py --out gpurun_out/rab.json --ops broadcast --algos auto --min-log2 26 --max-log2 28 --iters 10 --flush > gpurun_out/rab.txt 2>&1
python -c "
import json; d=json.load(open('gpurun_out/rab.json'))
print('N$n occ $1 tile $2 KiB', ' '.join(f\"{r['bytes']>>20}MiB={r['us']:.1f}\" for r in d['rows'] if r['algo']=='relay'))" || tail -3 gpurun_out/rab.txt
done; done
