"""D4PG learner data-parallel step (BASELINE.json configs[4]).

Two wrapped optimizers in one step function -- the multi-optimizer step_fn of
PAPER.md:161-172 -- on MLP actor/critic networks. Fixed total batch 256 split over
the replicas, synthetic replay batches (obs 64-d, matching the
length-64 embedding at PAPER.md:333; 8-d actions; 51-atom distributional critic).
The builder's sizes: actor 64-256-256-8, critic (64+8)-256-256-51.

  python tools/train_d4pg.py                # 1 GPU
  torchrun --nproc-per-node N tools/train_d4pg.py

Reports learner steps/s (whole job: every step consumes the global batch 256) and
the per-step gradient all-reduce time (two small buckets -> the one-shot kernel).
"""

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.nn as nn  # noqa: E402


def mlp(sizes, out_act=None):
    layers = []
    for i in range(len(sizes) - 1):
        layers.append(nn.Linear(sizes[i], sizes[i + 1]))
        if i < len(sizes) - 2:
            layers.append(nn.ReLU())
    if out_act:
        layers.append(out_act)
    return nn.Sequential(*layers)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--global-batch", type=int, default=256)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--graph", action="store_true",
                   help="capture the whole learner step (both optimizers and their all-reduces) in a CUDA graph")
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

    obs, act, atoms = 64, 8, 51
    B = a.global_batch // world
    repl = Replicator(device=local, pool_bytes=64 << 20)
    torch.manual_seed(rank)
    with repl.context():
        actor = repl.replicate(lambda: mlp([obs, 256, 256, act], nn.Tanh()))
        critic = repl.replicate(lambda: mlp([obs + act, 256, 256, atoms]))
        actor_opt = repl.wrap_optimizer(torch.optim.Adam(actor.parameters(), lr=1e-4, capturable=a.graph))
        critic_opt = repl.wrap_optimizer(torch.optim.Adam(critic.parameters(), lr=1e-4, capturable=a.graph))
    support = torch.linspace(-150, 150, atoms, device=dev)
    g = torch.Generator(device=dev).manual_seed(10 + rank)
    s = torch.randn(B, obs, device=dev, generator=g)
    a_t = torch.rand(B, act, device=dev, generator=g) * 2 - 1
    target = torch.softmax(torch.randn(B, atoms, device=dev, generator=g), dim=-1)

    def step():
        # critic: distributional cross-entropy against (synthetic) projected targets
        logits = critic(torch.cat([s, a_t], dim=1))
        critic_loss = -(target * torch.log_softmax(logits, dim=-1)).sum(-1).mean()
        critic_opt.zero_grad(set_to_none=False)
        critic_loss.backward()
        critic_opt.step()
        # actor: maximise the critic's expected value of the actor's action
        q = (torch.softmax(critic(torch.cat([s, actor(s)], dim=1)), dim=-1) * support).sum(-1)
        actor_loss = -q.mean()
        actor_opt.zero_grad(set_to_none=False)
        actor_loss.backward()
        actor_opt.step()
        return critic_loss, actor_loss

    run = step
    if a.graph:
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(3):
                step()
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            losses = step()

        def run():
            graph.replay()
            return losses
    for _ in range(a.warmup):
        run()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.steps):
        cl, al = run()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    ar_ms = 0.0
    if world > 1:
        bks = [critic_opt._buckets, actor_opt._buckets]
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.distributed.barrier()
        f0.record(st)
        for _ in range(50):
            for bk in bks:
                bk.reduce("premean")
        f1.record(st)
        torch.cuda.synchronize()
        ar_ms = f0.elapsed_time(f1) / 50
        t = torch.tensor([ms, ar_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, ar_ms = t.tolist()
    if rank == 0:
        gb = sum(b.numel * b.flat[0].element_size() for o in (critic_opt, actor_opt) if o._buckets
                 for b in o._buckets.buckets)
        print(json.dumps({"metric": "D4PG learner steps/s", "value": 1e3 / ms, "unit": "steps/s", "n_gpus": world,
                          "global_batch": a.global_batch, "per_gpu_batch": B, "ms_per_step": ms,
                          "allreduce_ms_per_step": ar_ms, "grad_bytes_per_step": gb,
                          "critic_loss": float(cl.item()), "actor_loss": float(al.item()), "cuda_graph": a.graph,
                          "config": {"actor": "64-256-256-8 tanh", "critic": "72-256-256-51 (distributional)",
                                     "optimizers": "2 x Adam, both wrap_optimizer'd", "data": "synthetic replay"}}),
              flush=True)
    repl.comm.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
