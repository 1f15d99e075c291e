echo "== D4PG"
timeout 300 python tools/train_d4pg.py 2>&1 | tail -1 | cut -c1-300
for n in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/train_d4pg.py 2>/dev/null | tail -1 | cut -c1-300; done
echo "== SNGAN"
timeout 600 python tools/train_sngan.py > gpurun_out/sngan1.txt 2>&1; tail -2 gpurun_out/sngan1.txt | cut -c1-400
for n in 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/train_sngan.py > gpurun_out/sngan$n.txt 2>&1; tail -1 gpurun_out/sngan$n.txt | cut -c1-400; done
