"""Fused optimizer apply vs the unfused wrapped step.

Times, with CUDA events after an L2 flush, one optimizer step on a flat f32
parameter set of --mparams million parameters:
  unfused: pack -> premean all-reduce of the gradient bucket -> unpack -> torch
           Adam (foreach) on all parameters          (wrap_optimizer default)
  fused:   pack -> rp_all_reduce_apply (average + Adam on the owned shard + the
           updated parameters stored on every replica)   (wrap_optimizer(fused=True))

  python tools/apply_bench.py                 # 8 replicas emulated on one GPU (HBM-bound)
  torchrun --nproc-per-node N tools/apply_bench.py
"""

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
    p.add_argument("--mparams", type=float, default=16.0, help="million f32 parameters")
    p.add_argument("--replicas", type=int, default=8)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--opt", default="adam", choices=["adam", "sgd"])
    p.add_argument("--only", default="both", choices=["both", "fused", "unfused"])
    a = p.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_1902_00465_b200 import Replicator
    from paper_1902_00465_b200.replicator import PerReplica

    n = int(a.mparams * 1e6)
    shapes = [(n // 4,), (n // 4,), (n // 4,), (n - 3 * (n // 4),)]

    def make_opt(ps):
        if a.opt == "adam":
            return torch.optim.Adam(ps, lr=1e-3, foreach=True)
        return torch.optim.SGD(ps, lr=0.1, momentum=0.9, nesterov=True, foreach=True)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    res = {}
    for fused in ([False, True] if a.only == "both" else [a.only == "fused"]):
        kw = {} if world > 1 else {"num_replicas": a.replicas}
        repl = Replicator(device=local, pool_bytes=3 * n * 4 + (64 << 20), **kw)
        R = repl.num_replicas
        with repl.context():
            params = repl.replicate(lambda: torch.nn.ParameterList(
                [torch.nn.Parameter(torch.randn(s, device=dev)) for s in shapes]))
            if repl.is_virtual:
                opt = repl.wrap_optimizer(PerReplica([make_opt(list(params[r].parameters())) for r in range(R)], repl),
                                          fused=fused)
            else:
                opt = repl.wrap_optimizer(make_opt(list(params.local.parameters())), fused=fused)
        reps = range(R) if repl.is_virtual else [0]
        for r in reps:
            for q in (params[r] if repl.is_virtual else params.local).parameters():
                q.grad = torch.randn_like(q)

        def step():
            if repl.is_virtual:
                # one thread drives every replica's work (the rendezvous path is for step_fns)
                if fused:
                    opt._apply_all()
                else:
                    opt._reduce_all(None)
                    for o in opt.opts:
                        o.step()
            else:
                opt.step()

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.steps):
            flush.zero_()
            if world > 1:
                torch.distributed.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        res["fused" if fused else "unfused"] = ms
        repl.comm.close()
    if rank == 0:
        R = a.replicas if world == 1 else world
        line = {"what": f"wrapped {a.opt} step, {n / 1e6:.1f}M f32 params", "replicas": R, "gpus": world,
                "ms": res}
        if "fused" in res and world == 1:
            # algorithmic HBM bytes of the fused kernel (all replicas share the GPU): every gradient
            # bucket read once, the owned parameters + state read and written once, the updated
            # parameters written to every replica's bucket
            st = 2 if a.opt == "adam" else 1
            alg = R * n * 4 + n * 4 + R * n * 4 + 2 * st * n * 4
            line["fused_apply_hbm_bytes"] = alg
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
