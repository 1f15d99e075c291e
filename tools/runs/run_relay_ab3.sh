# relay broadcast: root block cap A/B at N=4 and N=2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 -k "relay" > gpurun_out/rl4_tests.txt 2>&1; tail -1 gpurun_out/rl4_tests.txt
for n in 4 2; do
for rb in 16 32 64 128 1000; do
RP_RELAY_ROOT_BLOCKS=$rb timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n tools/sweep.py --out gpurun_out/rab.json --ops broadcast --algos auto --min-log2 22 --max-log2 28 --iters 10 --flush > gpurun_out/rab.txt 2>&1
python -c "
import json; d=json.load(open('gpurun_out/rab.json'))
print('N$n root_blocks $rb relay', ' '.join(f\"{r['bytes']>>20}MiB={r['us']:.1f}\" for r in d['rows'] if r['algo']=='relay'))" || tail -3 gpurun_out/rab.txt
done; done
