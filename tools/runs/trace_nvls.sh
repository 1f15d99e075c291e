# per-block phase trace of the NVLS vs two-shot all-reduce at N=4, 64 MiB
for algo in nvls auto; do
rm -f gpurun_out/tr_${algo}.jsonl*
RP_TRACE=gpurun_out/tr_${algo}.jsonl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 6 --warmup 3 --algo $algo --no-cpu-baseline --e2e-steps 1 > /dev/null 2>gpurun_out/tr_$algo.err
python tools/trace_summary.py gpurun_out/tr_${algo}.jsonl | head -24
done
