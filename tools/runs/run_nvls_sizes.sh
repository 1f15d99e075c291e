# NVLS vs P2P two-shot across message sizes (bench.py, N=2 and 4) + the raw probe at 64 MiB
./tools/nvls_probe 64 2>&1 | grep "U4 grid 148 x 256\|GPUs"
for n in 4 2; do for mib in 16 64 256; do for algo in auto nvls; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 30 --warmup 5 --e2e-steps 2 --no-cpu-baseline --bytes $((mib<<20)) --algo $algo > gpurun_out/bs_n${n}_${mib}_$algo.json 2> gpurun_out/bs_n${n}_${mib}_$algo.err
python -c "import json; d=json.loads(open('gpurun_out/bs_n${n}_${mib}_$algo.json').read().strip().splitlines()[-1]); print('N$n ${mib}MiB $algo', round(d['ms_per_step']*1e3,1), 'us busbw', round(d['per_gpu_busbw_gbs'],1))" || tail -5 gpurun_out/bs_n${n}_${mib}_$algo.err
done; done; done
