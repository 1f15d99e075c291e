timeout 200 ./tools/barrier_probe
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_tests.txt 2>&1; tail -3 gpurun_out/gpu_tests.txt
./tools/runs/run_nvls_sizes.sh 2>&1 | grep "^N"
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py --out gpurun_out/sweep_n$n.json --min-log2 10 --max-log2 24 --ops all_reduce --algos auto,twoshot --flush > gpurun_out/sweep_n$n.txt 2>&1; tail -32 gpurun_out/sweep_n$n.txt
done
