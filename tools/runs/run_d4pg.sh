for flag in "" "--graph"; do
timeout 300 python tools/train_d4pg.py $flag 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N1 $flag', round(d['value'],1), round(d['ms_per_step'],3))"
for n in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/train_d4pg.py $flag 2>gpurun_out/d4pg_err_$n.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N$n $flag', round(d['value'],1), round(d['ms_per_step'],3), round(d['allreduce_ms_per_step'],3))" || tail -5 gpurun_out/d4pg_err_$n.txt; done
done
