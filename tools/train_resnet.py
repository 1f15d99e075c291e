"""ResNet-50 data-parallel training through the Replicator (BASELINE.json configs[2]).

Synthetic 224x224 ImageNet-shaped batches, random-init torchvision ResNet-50,
channels_last, bf16 autocast, fp32 master weights, SGD + Nesterov momentum 0.9
(PAPER.md:253). ``repl.wrap_optimizer`` averages gradients with the NVLink
premean all-reduce over fusion buckets; gradients are exchanged as bf16
(``grad_comm_dtype``: 51.1 MB per step, the north-star workload).

  python tools/train_resnet.py --batch 64                  # 1 GPU
  torchrun --nproc-per-node N tools/train_resnet.py --batch 64

Prints one JSON line: img/s (whole job), ms/step (CUDA events, max over ranks),
and the all-reduce's share of the step (measured separately).
"""

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torchvision  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--batch", type=int, default=64, help="per-GPU batch (PAPER.md:253)")
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--grad-comm", default="bf16", choices=["bf16", "f32"])
    p.add_argument("--out", default=None)
    p.add_argument("--no-average", action="store_true", help="control run: skip the gradient all-reduce")
    p.add_argument("--diagnose", action="store_true", help="print per-phase GPU/host times of 8 steps")
    p.add_argument("--fused", action="store_true",
                   help="wrap_optimizer(fused=True): average + SGD update of each rank's shard in one kernel")
    p.add_argument("--nvls", action="store_true",
                   help="place the gradient buckets in an NVSwitch multicast region (in-switch reduction at >= 4)")
    p.add_argument("--overlap", action="store_true",
                   help="wrap_optimizer(overlap=True): buckets exchanged from grad hooks during backward")
    p.add_argument("--bucket-mb", type=float, default=None, help="fusion bucket size (overlap)")
    p.add_argument("--overlap-blocks", type=int, default=None, help="grid cap of overlapped exchanges (0: none)")
    p.add_argument("--no-grad-views", action="store_true", help="pack/unpack gradients instead of bucket views")
    p.add_argument("--overlap-priority", type=int, default=-1, help="side-stream priority (-1 high, 0 normal)")
    p.add_argument("--overlap-dry-kernel", action="store_true",
                   help="diagnostic: like --overlap-dry, plus one tiny kernel per bucket on the side stream")
    p.add_argument("--overlap-dry", action="store_true",
                   help="diagnostic: hooks and bucket bookkeeping only, no exchange (measures the hook overhead)")
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

    torch.backends.cudnn.benchmark = True
    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.allow_tf32 = True
    repl = Replicator(device=local, pool_bytes=512 << 20,
                      grad_comm_dtype=torch.bfloat16 if a.grad_comm == "bf16" else None,
                      nvls_bytes=(128 << 20) if (a.nvls and world > 1) else 0,
                      bucket_bytes=int(a.bucket_mb * (1 << 20)) if a.bucket_mb else None,
                      grad_views=not a.no_grad_views)
    torch.manual_seed(rank)  # replicate() broadcasts replica 0's init
    with repl.context():
        model = repl.replicate(lambda: torchvision.models.resnet50().to(memory_format=torch.channels_last))
        opt = repl.wrap_optimizer(torch.optim.SGD(model.parameters(), lr=0.1, momentum=0.9, nesterov=True,
                                                  weight_decay=1e-4), fused=a.fused,
                                   overlap=a.overlap and world > 1, overlap_blocks=a.overlap_blocks)
    net = model.local
    if a.overlap and world > 1:
        opt.stream = torch.cuda.Stream(device=dev, priority=a.overlap_priority)
        if a.overlap_dry or a.overlap_dry_kernel:
            tiny = torch.zeros(1, device=dev)
            for b in opt.buckets:
                b.reduce = (lambda kind, grads=None, attached=False: tiny.add_(1)) if a.overlap_dry_kernel \
                    else (lambda kind, grads=None, attached=False: None)
    if a.no_average:
        opt.average_gradients = lambda: None
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    x = torch.randn(a.batch, 3, 224, 224, device=dev, generator=g).contiguous(memory_format=torch.channels_last)
    y = torch.randint(0, 1000, (a.batch,), device=dev, generator=g)
    lossf = torch.nn.CrossEntropyLoss()

    def step():
        opt.zero_grad(set_to_none=False)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = lossf(net(x), y)
        loss.backward()
        opt.step()
        return loss

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if a.diagnose:  # per-phase GPU times (events) and host enqueue times of a few steps
        import time as _t
        rows = []
        st = torch.cuda.current_stream(dev)
        for _ in range(8):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            h = [_t.perf_counter()]
            ev[0].record(st)
            opt.zero_grad(set_to_none=False)
            with torch.autocast("cuda", dtype=torch.bfloat16):
                loss = lossf(net(x), y)
            loss.backward()
            ev[1].record(st)
            h.append(_t.perf_counter())
            opt.average_gradients()
            ev[2].record(st)
            h.append(_t.perf_counter())
            opt.optimizer.step()
            ev[3].record(st)
            h.append(_t.perf_counter())
            rows.append((ev, h))
        torch.cuda.synchronize()
        for ev, h in rows:
            print(f"rank {rank} gpu fwdbwd {ev[0].elapsed_time(ev[1]):7.3f} avg {ev[1].elapsed_time(ev[2]):7.3f} "
                  f"opt {ev[2].elapsed_time(ev[3]):7.3f} ms | host enqueue fwdbwd {1e3 * (h[1] - h[0]):7.3f} "
                  f"avg {1e3 * (h[2] - h[1]):7.3f} opt {1e3 * (h[3] - h[2]):7.3f} ms", flush=True)
    if world > 1:
        torch.distributed.barrier()
    stream = torch.cuda.current_stream(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    hook0 = getattr(opt, "hook_s", 0.0)
    t0 = time.time()
    for e0, e1 in evs:
        e0.record(stream)
        loss = step()
        e1.record(stream)
    torch.cuda.synchronize()
    wall = time.time() - t0
    hook_ms = (getattr(opt, "hook_s", 0.0) - hook0) * 1e3 / a.steps
    ms = statistics.mean(e0.elapsed_time(e1) for e0, e1 in evs)
    # the gradient all-reduce alone (same buckets), for its share of the step
    ar_ms = 0.0
    if world > 1 and not a.no_average:
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        torch.distributed.barrier()
        a0.record(stream)
        for _ in range(10):
            if a.fused:  # pack + fused average/update (the whole optimizer step)
                opt._apply_all()
            elif a.overlap and world > 1:  # every bucket, as step() launches them without backward
                opt.average_gradients()
            else:
                opt._buckets.reduce("premean")
        a1.record(stream)
        torch.cuda.synchronize()
        ar_ms = a0.elapsed_time(a1) / 10
    if world > 1:
        t = torch.tensor([ms, ar_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, ar_ms = t.tolist()
    # replicas must stay bit-identical (SPEC.md:399 replica consistency)
    flat = torch.cat([q.detach().reshape(-1) for q in net.parameters()])
    gathered = repl.all_gather(flat, stack=True) if world > 1 else flat.unsqueeze(0)
    consistent = bool(all(torch.equal(gathered[r], gathered[0]) for r in range(world)))
    if rank == 0:
        if a.fused:
            grad_bytes = sum(g.grads.numel * g.grads.flat[0].element_size() for g in opt.groups if g is not None)
        elif a.overlap and world > 1:
            grad_bytes = sum(b.numel * torch.empty((), dtype=b.comm_dtype).element_size() for b in opt.buckets)
        else:
            grad_bytes = sum(b.numel * torch.empty((), dtype=b.comm_dtype).element_size()
                             for b in opt._buckets.buckets) if opt._buckets else 0
        line = {"metric": "ResNet-50 synthetic img/s", "value": world * a.batch / (ms / 1e3), "unit": "img/s",
                "n_gpus": world, "per_gpu_batch": a.batch, "ms_per_step": ms, "steps": a.steps, "warmup": a.warmup,
                "allreduce_ms": ar_ms, "allreduce_share": ar_ms / ms if ms else 0.0,
                "grad_exchange_bytes": grad_bytes, "grad_comm": a.grad_comm, "replicas_identical": consistent,
                "loss": float(loss.item()), "wall_s": wall, "fused_apply": a.fused, "nvls": a.nvls,
                "overlap": a.overlap, "overlap_hook_host_ms": hook_ms, "buckets": len(opt.buckets) if (a.overlap and world > 1) else None,
                "config": {"model": "resnet50 (torchvision, random init)", "input": "synthetic 224x224x3 channels_last",
                           "precision": "bf16 autocast, fp32 master", "optimizer": "SGD nesterov 0.9 wd 1e-4"}}
        print(json.dumps(line), flush=True)
        if a.out:
            json.dump(line, open(a.out, "w"), indent=1)
    repl.comm.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
