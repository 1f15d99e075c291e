"""Cross-replica BN statistics (K5 forward / K5b backward) and apply kernels:
HBM-roofline measurement on SN-GAN-generator-like activations (local batch 64,
BASELINE.json configs[3]; SURVEY.md §8a shapes).

  python tools/bench_bn.py [--replicas R]      # R virtual replicas on one GPU (default 1)
  torchrun --nproc-per-node N tools/bench_bn.py

Reports per kernel: time (CUDA events, L2 flushed between iterations), algorithmic
HBM bytes / time, fraction of MEASURED_PEAKS.json hbm_gbs.
"""

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1902_00465_b200 import _lib  # noqa: E402
from paper_1902_00465_b200.comm import Communicator, VirtualCommunicator  # noqa: E402

# SN-GAN 128x128 generator BN inputs at local batch 64 (C, H) -- SURVEY.md §8a
SHAPES = [(1024, 4), (1024, 8), (1024, 16), (512, 32), (256, 64), (128, 128), (64, 128)]


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--replicas", type=int, default=1)
    p.add_argument("--batch", type=int, default=64)
    p.add_argument("--iters", type=int, default=20)
    p.add_argument("--dtype", default="f32")
    p.add_argument("--out", default=None)
    p.add_argument("--only", default=None, help="one shape, e.g. 256x64 (C x H)")
    p.add_argument("--flush", default="write+read", choices=["write", "write+read"],
                   help="L2 flush between iterations; write+read leaves clean lines, so the flush's "
                        "dirty-line drain does not land inside the timed kernel")
    a = p.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        comm = Communicator(device=local, pool_bytes=64 << 20)
    else:
        comm = VirtualCommunicator(a.replicas, device=local, pool_bytes=64 << 20)
    nrep = a.replicas if world == 1 else 1
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    dt = {"f32": torch.float32, "bf16": torch.bfloat16}[a.dtype]
    code = {"f32": 0, "bf16": 2}[a.dtype]
    lib = _lib.load()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_sink = torch.empty((), dtype=torch.int64, device=dev)
    align = torch.zeros(4, device=dev)
    stream = torch.cuda.current_stream(dev)
    rows_out = []
    shapes = SHAPES if a.only is None else [tuple(int(v) for v in a.only.split("x"))]
    for (c, h) in shapes:
        n = a.batch
        xs = [torch.randn(n, c, h, h, device=dev).to(dt).contiguous(memory_format=torch.channels_last)
              for _ in range(nrep)]
        dys = [torch.randn_like(x) for x in xs]
        outs = [[torch.empty(c, device=dev) for _ in range(nrep)] for _ in range(5)]
        cnt = [torch.empty(1, dtype=torch.float64, device=dev) for _ in range(nrep)]
        rows, hw = n * h * h, 1
        nbytes = n * c * h * h * xs[0].element_size()

        def ptrs(lst):
            arr, keep = _lib.ptr_array([t.data_ptr() for t in lst])
            ptrs.keep.append(keep)
            import ctypes
            return ctypes.cast(arr, ctypes.c_void_p).value
        ptrs.keep = []
        if world == 1:
            xp, dyp = ptrs(xs), ptrs(dys)
            o = [ptrs(x) for x in outs]
            cp = ptrs(cnt)
        else:
            xp, dyp = xs[0].data_ptr(), dys[0].data_ptr()
            o = [x[0].data_ptr() for x in outs]
            cp = cnt[0].data_ptr()

        def fwd():
            _lib.check(lib.rp_bn_stats(comm._handle, xp, code, rows, c, hw, _lib.NHWC, 1e-5, o[0], o[1], o[2], cp,
                                       stream.cuda_stream), "bn")

        def bwd():
            _lib.check(lib.rp_bn_bwd_stats(comm._handle, xp, dyp, code, rows, c, hw, _lib.NHWC, o[0], o[3], o[4],
                                           None, None, stream.cuda_stream), "bnb")
        y = torch.empty_like(xs[0])

        def apply():
            _lib.check(lib.rp_bn_apply(xs[0].data_ptr(), y.data_ptr(), code, rows, c, hw, _lib.NHWC,
                                       outs[0][0].data_ptr(), outs[2][0].data_ptr(), None, None, stream.cuda_stream))
        for name, fn, mult in (("bn_stats_fwd(K5)", fwd, 1), ("bn_stats_bwd(K5b)", bwd, 2), ("bn_apply", apply, 2)):
            for _ in range(3):
                fn()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(a.iters)]
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            for e0, e1 in evs:
                flush.zero_()
                if a.flush == "write+read":
                    flush_sink.copy_(flush.view(torch.int64).sum())
                if world > 1:  # untimed tiny collective: ranks leave the flush together
                    comm.all_reduce_tensor(align, "sum", out=align)
                e0.record(stream)
                fn()
                e1.record(stream)
            torch.cuda.synchronize()
            ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in evs)
            reps = nrep if name != "bn_apply" else 1
            gbs = mult * nbytes * reps / (ms / 1e3) / 1e9
            row = {"kernel": name, "shape_nhwc": [n, h, h, c], "dtype": a.dtype, "replicas": nrep * world,
                   "us": ms * 1e3, "hbm_gbs": gbs, "frac_of_measured": gbs / peak}
            rows_out.append(row)
            if rank == 0:
                print(f"{name:18s} N={n} C={c:5d} H={h:4d} {a.dtype} {ms * 1e3:8.1f} us  {gbs:7.0f} GB/s  "
                      f"{gbs / peak:5.1%}", flush=True)
    comm.check()
    if rank == 0 and a.out:
        json.dump(rows_out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
