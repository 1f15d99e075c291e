# ResNet-50: baseline wrap vs fused apply vs NVLS buckets, per-GPU batch 64 (the regime where the exchange matters most)
b=${B:-64}
for flags in "" "--fused"; do
timeout 600 python tools/train_resnet.py --batch $b --steps 30 --warmup 10 $flags 2> gpurun_out/rn_err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N1 b$b $flags', round(d['value']), round(d['ms_per_step'],2))" || tail -3 gpurun_out/rn_err.txt
done
for n in 2 4; do for flags in "" "--fused" "--nvls"; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/train_resnet.py --batch $b --steps 30 --warmup 10 $flags 2> gpurun_out/rn_err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N$n b$b $flags', round(d['value']), round(d['ms_per_step'],2), 'exchange', round(d['allreduce_ms'],3), d['replicas_identical'])" || tail -3 gpurun_out/rn_err.txt
done; done
