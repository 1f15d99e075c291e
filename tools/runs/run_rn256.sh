# 2 GPUs, final build: ResNet-50 at 256 images per GPU, N=1 and N=2
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/train_resnet.py --batch 256 --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('resnet50 N1 b256', round(d['value']), 'img/s', round(d['ms_per_step'],2))"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/train_resnet.py --batch 256 --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('resnet50 N2 b256', round(d['value']), 'img/s', round(d['ms_per_step'],2), 'exchange', round(d['allreduce_ms'],3), d['replicas_identical'])"
