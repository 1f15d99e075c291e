"""Bus-bandwidth sweep of all_reduce / all_gather / broadcast over message sizes
(BASELINE.json configs[1]: "all_reduce/all_gather/broadcast bandwidth sweep 1 KB-1 GB").

  python tools/sweep.py --out gpurun_out/sweep_n1.json            # 8 replicas on one GPU
  torchrun --nproc-per-node N tools/sweep.py --out ...            # N GPUs over NVLink

Each iteration is timed alone with CUDA events (L2 flushed before it); the reported
time is the median over iterations, max over ranks. busBW (nccl-tests):
all_reduce 2(N-1)/N*S/t, all_gather (N-1)*S/t (S per rank), broadcast S/t.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", required=True)
    p.add_argument("--min-log2", type=int, default=10)
    p.add_argument("--max-log2", type=int, default=30)
    p.add_argument("--replicas", type=int, default=8)
    p.add_argument("--ops", default="all_reduce,all_gather,broadcast")
    p.add_argument("--algos", default="auto,oneshot,twoshot")
    p.add_argument("--iters", type=int, default=20)
    p.add_argument("--flush", action="store_true", help="flush L2 and time every iteration alone")
    a = p.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_1902_00465_b200.comm import Communicator, VirtualCommunicator

    maxb = 1 << a.max_log2
    n = a.replicas if world == 1 else world
    pool = 2 * maxb + (64 << 20)
    comm = VirtualCommunicator(n, device=local, pool_bytes=pool) if world == 1 else \
        Communicator(device=local, pool_bytes=pool)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    reps = n if world == 1 else 1
    count_max = maxb // 4
    bufs = [torch.randn(count_max, device=dev) for _ in range(reps)]
    outs = [torch.empty(n * count_max if "all_gather" in a.ops else count_max, device=dev) for _ in range(reps)]
    nvls_buf = None
    reg_buf = None
    if "registered" in a.algos.split(",") and world > 1:  # a registered user tensor, reduced in place (zero-copy)
        reg_buf = torch.randn(count_max, device=dev)
        comm.register(reg_buf)
    if "nvls" in a.algos.split(",") and world > 1:  # in-switch reduction: in place in the multicast region
        comm.enable_nvls(maxb + (4 << 20))
        nvls_buf = comm.alloc_nvls(count_max, torch.float32)
        nvls_buf.copy_(bufs[0])

    def tmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    rows = []
    for op in a.ops.split(","):
        algos = a.algos.split(",") if op == "all_reduce" else (["auto", "direct", "scatter"] if op == "broadcast"
                                                                else ["auto"])
        if "nccl" in a.algos.split(",") and op != "all_reduce":
            algos = algos + ["nccl"]  # comparison column only: NCCL is never on the product path
        if op == "broadcast" and world > 1:
            algos = algos + ["relay"]  # pipelined P2P relay (K4r); AUTO's choice above 1 MiB
        if "nvls" in a.algos.split(",") and op == "broadcast":
            algos = algos + ["nvls"]  # in place in the NVLS region: the root's multicast store
        for lg in range(a.min_log2, a.max_log2 + 1):
            size = 1 << lg
            count = size // 4
            if op == "all_gather" and n * size > n * maxb:
                continue
            for algo in algos:
                xs = [b[:count] for b in bufs]
                if op == "all_reduce":
                    os_ = [o[:count] for o in outs]
                    if world == 1:
                        fn = lambda: comm.all_reduce(xs, "sum", outs=os_, algo=algo)  # noqa: E731
                    elif algo == "nccl":
                        if world == 1:
                            continue
                        fn = lambda: torch.distributed.all_reduce(os_[0])  # noqa: E731
                    elif algo == "nvls":
                        if nvls_buf is None:
                            continue
                        fn = lambda: comm.all_reduce_tensor(nvls_buf[:count], "mean", out=nvls_buf[:count],  # noqa: E731
                                                            algo="nvls")
                    elif algo == "registered":
                        if reg_buf is None:
                            continue
                        fn = lambda: comm.all_reduce_tensor(reg_buf[:count], "mean", out=reg_buf[:count])  # noqa: E731
                    else:
                        fn = lambda: comm.all_reduce_tensor(xs[0], "sum", out=os_[0], algo=algo)  # noqa: E731
                    factor = 2.0 * (n - 1) / n
                elif op == "all_gather":
                    os_ = [o[:n * count].view(n, count) for o in outs]
                    if algo == "nccl":
                        if world == 1:
                            continue
                        fn = lambda: torch.distributed.all_gather_into_tensor(os_[0].view(-1), xs[0])  # noqa: E731
                    elif world == 1:
                        fn = lambda: comm.all_gather(xs, outs=os_)  # noqa: E731
                    else:
                        fn = lambda: comm.all_gather_tensor(xs[0], out=os_[0])  # noqa: E731
                    factor = float(n - 1)
                else:
                    os_ = [o[:count] for o in outs]
                    if algo == "nccl":
                        if world == 1:
                            continue
                        fn = lambda: torch.distributed.broadcast(os_[0], src=0)  # noqa: E731
                    elif algo == "nvls":
                        if nvls_buf is None:
                            continue
                        fn = lambda: comm.broadcast_tensor(nvls_buf[:count], root=0)  # noqa: E731
                    elif world == 1:
                        fn = lambda: comm.broadcast(xs, root=0, outs=os_, algo=algo)  # noqa: E731
                    elif algo == "relay" and size % 16:
                        continue
                    else:
                        fn = lambda: comm.broadcast_tensor(xs[0], root=0, out=os_[0], algo=algo)  # noqa: E731
                    factor = 1.0
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                if world > 1:
                    torch.distributed.barrier()
                if a.flush:
                    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                           for _ in range(a.iters)]
                    for e0, e1 in evs:
                        flush.zero_()
                        e0.record(stream)
                        fn()
                        e1.record(stream)
                    torch.cuda.synchronize()
                    ms = tmax(statistics.median(e0.elapsed_time(e1) for e0, e1 in evs))
                else:  # nccl-tests convention: back-to-back launches, mean time
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    for _ in range(a.iters):
                        fn()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ms = tmax(e0.elapsed_time(e1) / a.iters)
                bus = factor * size / (ms / 1e3) / 1e9
                rows.append({"op": op, "algo": algo, "bytes": size, "n": n, "gpus": world, "us": ms * 1e3,
                             "busbw_gbs": bus})
                if rank == 0:
                    print(f"{op:10s} {algo:8s} {size:>11d} B  {ms * 1e3:9.2f} us  busBW {bus:8.1f} GB/s", flush=True)
    comm.check()
    if rank == 0:
        with open(a.out, "w") as f:
            json.dump({"world": world, "replicas": n, "rows": rows}, f, indent=1)
    comm.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
