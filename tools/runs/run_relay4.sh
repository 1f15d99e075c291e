# 4 GPUs: relay broadcast tests + broadcast sweep (relay vs scatter/direct/NVLS vs NCCL); N=2 sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 -k "relay or gather_broadcast or nvls_all_reduce" > gpurun_out/rl_tests.txt 2>&1; tail -3 gpurun_out/rl_tests.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py --out gpurun_out/sweep_bc_n4.json --ops broadcast --algos auto,nccl,nvls --min-log2 16 --max-log2 28 --iters 20 --flush > gpurun_out/sweep_bc_n4.txt 2>&1; grep -c GB gpurun_out/sweep_bc_n4.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 tools/sweep.py --out gpurun_out/sweep_bc_n2.json --ops broadcast --algos auto,nccl,nvls --min-log2 16 --max-log2 28 --iters 20 --flush > gpurun_out/sweep_bc_n2.txt 2>&1; grep -c GB gpurun_out/sweep_bc_n2.txt
