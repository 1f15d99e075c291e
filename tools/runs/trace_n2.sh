for impl in pull push; do
rm -f gpurun_out/trace_${impl}.jsonl*
RP_TRACE=gpurun_out/trace_${impl}.jsonl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 6 --warmup 3 --ar-impl $impl --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python tools/trace_summary.py gpurun_out/trace_${impl}.jsonl
done
timeout 300 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 250 > gpurun_out/mp_tests.txt 2>&1; tail -3 gpurun_out/mp_tests.txt
