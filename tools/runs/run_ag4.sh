# 4 GPUs: multi-process tests with the push one-shot all_gather; all_gather sweep vs NCCL (push vs pull)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 > gpurun_out/ag_tests.txt 2>&1; tail -3 gpurun_out/ag_tests.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py --out gpurun_out/sweep_ag_n4.json --ops all_gather --algos auto,nccl --min-log2 10 --max-log2 22 --iters 30 --flush > gpurun_out/sweep_ag_n4.txt 2>&1; grep -c GB gpurun_out/sweep_ag_n4.txt
RP_AG_PULL=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 tools/sweep.py --out gpurun_out/sweep_ag_n4_pull.json --ops all_gather --algos auto --min-log2 10 --max-log2 22 --iters 30 --flush > gpurun_out/sweep_ag_n4_pull.txt 2>&1; grep -c GB gpurun_out/sweep_ag_n4_pull.txt
