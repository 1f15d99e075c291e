timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 500 -k "nvls" > gpurun_out/tests_nvls.txt 2>&1; tail -15 gpurun_out/tests_nvls.txt
for n in 2 4; do for algo in auto nvls; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 30 --warmup 5 --e2e-steps 2 --algo $algo > gpurun_out/b_n${n}_$algo.json 2> gpurun_out/b_n${n}_$algo.err
python -c "import json; d=json.loads(open('gpurun_out/b_n${n}_$algo.json').read().strip().splitlines()[-1]); print('N$n $algo', round(d['ms_per_step'],4), 'per_gpu', round(d['per_gpu_busbw_gbs'],1), 'frac', round(d['roofline']['frac'],3))" || tail -5 gpurun_out/b_n${n}_$algo.err
done; done
