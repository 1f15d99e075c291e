# BN small layers at N=1 and N=2: fused (one cooperative launch) vs unfused (two launches)
mkdir -p gpurun_out
for s in 1024x4 1024x8 1024x16 512x32; do
CUDA_VISIBLE_DEVICES=0 python tools/bench_bn.py --only $s --dtype f32 2>&1 | grep "bn_stats" | sed "s/^/N1 fused   /"
CUDA_VISIBLE_DEVICES=0 RP_BN_UNFUSED=1 python tools/bench_bn.py --only $s --dtype f32 2>&1 | grep "bn_stats" | sed "s/^/N1 unfused /"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 tools/bench_bn.py --only $s --dtype f32 2>&1 | grep "bn_stats" | sed "s/^/N2 fused   /"
RP_BN_UNFUSED=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516 tools/bench_bn.py --only $s --dtype f32 2>&1 | grep "bn_stats" | sed "s/^/N2 unfused /"
done
