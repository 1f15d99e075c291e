# 4 GPUs, final build: ResNet-50 b64 N=1/2/4 (+fused), SN-GAN N=1/2/4, D4PG graph N=1/2/4
mkdir -p gpurun_out
b=64
rn() { n=$1; shift; if [ $n = 1 ]; then L="python"; else L="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511"; fi
timeout 600 $L tools/train_resnet.py --batch $b --steps 40 --warmup 10 "$@" 2> gpurun_out/rn_err.txt > gpurun_out/rn_out.txt; python -c "import json,sys; d=json.loads(open('gpurun_out/rn_out.txt').read().strip().splitlines()[-1]); print('resnet50 N$n b$b $*', round(d['value']), 'img/s', round(d['ms_per_step'],2), 'ms exchange', round(d['allreduce_ms'],3), d['replicas_identical'])" || tail -3 gpurun_out/rn_err.txt; }
for n in 1 2 4; do rn $n; done
for n in 2 4; do rn $n --fused; done
timeout 600 python tools/train_sngan.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sngan N1', round(d['value']), 'img/s', round(d['ms_per_step'],2))"
for n in 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 tools/train_sngan.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sngan N$n', round(d['value']), 'img/s', round(d['ms_per_step'],2), d.get('bn_running_stats_identical'))"; done
timeout 300 python tools/train_d4pg.py --graph 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('d4pg N1 graph', round(d['value'],1), round(d['ms_per_step'],3))"
for n in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29513 tools/train_d4pg.py --graph 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('d4pg N$n graph', round(d['value'],1), round(d['ms_per_step'],3), round(d['allreduce_ms_per_step'],3))"; done
