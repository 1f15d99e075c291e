for b in 64 256; do
timeout 600 python tools/train_resnet.py --batch $b --steps 20 --warmup 8 --out gpurun_out/rn50_n1_b$b.json 2> gpurun_out/rn50_n1_b$b.err | tail -1
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/train_resnet.py --batch $b --steps 20 --warmup 8 --out gpurun_out/rn50_n${n}_b$b.json 2> gpurun_out/rn50_n${n}_b$b.err | tail -1
done; done
tail -3 gpurun_out/rn50_n4_b64.err
