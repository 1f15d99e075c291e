"""Benchmark of the data-parallel hot path: the wrap_optimizer gradient all-reduce.

One step = one cross-replica all_reduce("premean" = all_sum(g/R))
of a 64 MiB fp32 gradient fusion buffer per replica, in place in the registered
pool (zero-copy): the flat virtual kernel at N=1, the two-shot / NVLS kernels at N>1.

  python bench.py                      # N=1: R=8 replicas emulated on one B200
  torchrun --nproc-per-node N bench.py --gpus N   # N ranks, one per GPU, NVLink P2P
  python bench.py --impl reference     # the reference's CPU path (oracle port), host cores

At N=1 the 8 replicas live in one GPU's HBM and one barrier-free launch folds every
16-byte position of all 8 buffers (ar_virtual_flat): HBM-bound. At N>1 each GPU is
one replica and the kernel's loads/stores cross NVLink: NVLink-bound.

value = n_gpus x busBW (nccl-tests busBW = 2(R-1)/R * S / t, per GPU), i.e. the
aggregate bus bandwidth of the job. L2 is flushed (256 MiB write + 256 MiB read) between timed
steps; every step is timed with CUDA events around the one collective launch; the
max over ranks is reported.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
NVLINK_PEER_GBS = 770.0   # B200_PROFILING.md: measured peer copy per direction (nominal 900)
NVLINK_NOMINAL_GBS = 900.0
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--bytes", type=int, default=64 << 20, help="message bytes per replica")
    p.add_argument("--replicas", type=int, default=8, help="replicas emulated on one GPU when N=1")
    p.add_argument("--kind", default="premean")
    p.add_argument("--algo", default="auto")
    p.add_argument("--nvls", default="auto", choices=["auto", "on", "off"],
                   help="place the buffers in an NVSwitch multicast region (auto: at >= 4 GPUs, where the "
                        "in-switch reduction beats the P2P two-shot; the library then picks it under --algo auto)")
    p.add_argument("--ar-impl", default=None, choices=["push", "pull"],
                   help="force the all-reduce data-movement form (default: push multi-process, pull virtual)")
    p.add_argument("--flush", default="write+read", choices=["write", "write+read"],
                   help="L2 flush before every timed step: write 256 MiB (leaves up to the L2's worth of dirty "
                        "lines to be written back INSIDE the timed step), or write 256 MiB then read another "
                        "256 MiB (the flush's write-backs complete before the step; L2 clean and cold)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-budget", type=float, default=10.0)
    p.add_argument("--ref-budget", type=float, default=150.0,
                   help="seconds cap on the --impl reference timed steps (whole Graph.evaluate steps)")
    p.add_argument("--e2e-steps", type=int, default=10)
    return p.parse_args()


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def mark(self):
        return time.time()

    def stop(self, t0, t1):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [s for (t, s) in self.samples if t0 - 0.05 <= t <= t1 + 0.1] or [s for _, s in self.samples]
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            parts = [x.strip() for x in r.split(",")]
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ---------------------------------------------------------------------------

def peaks():
    try:
        d = json.load(open(MEASURED_PEAKS))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


def ncu_traffic(key: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full
    capture (profiles/r01_ncu_traffic.json), or (None, None) when none matches."""
    path = os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")
    try:
        with open(path) as f:
            rec = json.load(f).get(key)
    except (OSError, ValueError):
        return None, None
    if not rec:
        return None, None
    return rec["dram_read_bytes"] + rec["dram_write_bytes"], rec["source"]


def busbw(nbytes, n, seconds):
    return 2.0 * (n - 1) / n * nbytes / seconds / 1e9


def dist_setup(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        return dist.get_rank(), world, local
    return 0, 1, 0


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_reference(args, rank, world):
    """--impl reference: the reference's OWN CPU path -- its Graph.evaluate of the
    stitched in-process program (oracle/_ref, copied by oracle/ref_vendor.py; numpy
    runs it on one core) -- for --steps whole steps after --warmup. The oracle port
    sliced over every host core is reported beside it as a labelled extra."""
    from oracle.cpu_baseline import host_cores, reference_available, time_port, time_reference

    n = args.replicas if world == 1 else world
    count = args.bytes // 4
    if rank != 0:
        return None
    cores = host_cores()
    if reference_available():
        sec, steps, thr = time_reference(n, count, args.kind, budget_s=args.ref_budget, max_steps=max(1, args.steps),
                                         warmup=max(1, args.warmup))
        kind = "reference"
        sample = (f"{steps} whole steps of the reference's own Graph.evaluate (oracle/_ref) on the stitched program: "
                  f"{n} div-by-{n} nodes + {n} nary_sum sites over {n} replicas x {args.bytes >> 20} MiB f32 "
                  f"(graph.py:514-522); numpy single-threaded: 1 core active of {cores}")
    else:  # no vendored reference: the validated port (tests/test_oracle.py)
        sec, steps, thr = time_port(n, count, args.kind, budget_s=args.cpu_budget, threads=cores,
                                    max_steps=max(1, args.steps))
        kind = "port"
        sample = (f"{steps} whole stitched steps ({n} nary_{args.kind} sites x {n} replicas x "
                  f"{args.bytes >> 20} MiB f32), threads={thr}")
    bw = busbw(args.bytes, n, sec) * world
    line = {
        "metric": "all_reduce bus GB/s (aggregate, 64 MiB fp32 premean)",
        "value": bw, "unit": "GB/s", "n_gpus": world, "steps": steps, "warmup": max(1, args.warmup),
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic", "impl": "reference",
        "config": _config(args, world),
        "cpu_baseline": {"value": bw, "unit": "GB/s", "cores": thr, "kind": kind, "sample": sample},
        "e2e": {"value": bw, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if kind == "reference" and not args.no_cpu_baseline:
        psec, psteps, pthr = time_port(n, count, args.kind, budget_s=args.cpu_budget, threads=cores, max_steps=50)
        line["port_all_cores"] = {"value": busbw(args.bytes, n, psec) * world, "unit": "GB/s", "cores": pthr,
                                  "kind": "port", "steps": psteps,
                                  "note": "oracle/cpu_baseline.py port of the same folds, message sliced over "
                                          "every host core (an upper bound on a parallelised reference)"}
    return line


def _config(args, world):
    n = args.replicas if world == 1 else world
    return {"workload": ("wrap_optimizer gradient all_reduce(premean) of one 64 MiB fp32 fusion buffer per "
                         f"replica, {n} replicas" + (f" emulated on 1 B200 (cooperative launch)" if world == 1
                                                      else f" on {world} B200 (one per process, NVLink P2P)")),
            "msg_bytes_per_replica": args.bytes, "replicas": n, "dtype": "f32", "op": args.kind,
            "algo": getattr(args, "chosen_algo", args.algo), "algo_requested": args.algo,
            "in_place_pool": True, "clock_settle": "50 ms of L2-flush traffic before the warm-up steps",
            "l2": ("flushed between steps (256 MiB write + 256 MiB read: clean, cold L2)"
                                          if getattr(args, "flush", "write") == "write+read"
                                          else "flushed between steps (256 MiB write)"),
            "parallelism": f"dp{n}"}


def run_ours(args, rank, world, local):
    import numpy as np
    import torch

    from paper_1902_00465_b200.comm import Communicator, VirtualCommunicator

    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    count = args.bytes // 4
    # fusion buffer + a landing region of the same size (push two-shot) + headroom
    pool = 2 * args.bytes + (64 << 20)
    if world == 1:
        n = args.replicas
        comm = VirtualCommunicator(n, device=local, pool_bytes=pool)
        bufs = comm.alloc(count, torch.float32)
        for r, b in enumerate(bufs):
            b.copy_(torch.randn(count, device=dev, generator=torch.Generator(device=dev).manual_seed(1234 + r)))

        def step():
            comm.all_reduce(bufs, args.kind, outs=bufs, algo=args.algo)

        args.chosen_algo = comm.algorithm_for(bufs[0], args.kind, out=bufs[0], algo=args.algo)
    else:
        n = world
        comm = Communicator(device=local, pool_bytes=pool)
        args.use_nvls = args.algo == "nvls" or args.nvls == "on" or (args.nvls == "auto" and world >= 4)
        if args.use_nvls:
            try:  # in-switch reduction: the buffers live in the multicast region
                comm.enable_nvls(2 * args.bytes + (4 << 20))  # timed buffer + the e2e buffer
            except Exception as e:  # no multicast support on this box: the P2P kernels
                if args.algo == "nvls":
                    raise
                args.use_nvls, args.nvls_error = False, str(e).splitlines()[0][:200]
        buf = comm.alloc_nvls(count, torch.float32) if args.use_nvls else comm.alloc(count, torch.float32)
        buf.copy_(torch.randn(count, device=dev, generator=torch.Generator(device=dev).manual_seed(1234 + rank)))

        def step():
            comm.all_reduce_tensor(buf, args.kind, out=buf, algo=args.algo)

        args.chosen_algo = comm.algorithm_for(buf, args.kind, out=buf, algo=args.algo)
        args.topology = comm.topology()

    align = None
    if world > 1:
        tiny = torch.zeros(4, device=dev)

        def align():
            comm.all_reduce_tensor(tiny, "sum", out=tiny)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_rd = torch.zeros(64 << 20, dtype=torch.float32, device=dev) if args.flush == "write+read" else None
    stream = torch.cuda.current_stream(dev)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # clock sampler first (nvidia-smi needs ~0.2 s to start), so no idle gap separates
    # the warm-up from the timed steps; then ~50 ms of flush traffic (memory only, no
    # collective) to settle the clocks, and W warm-up steps shaped exactly like the
    # timed ones (flush, align, step)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    settle_end = time.time() + 0.05
    while time.time() < settle_end:
        flush.zero_()
        torch.cuda.synchronize()
    for _ in range(max(3, args.warmup)):
        flush.zero_()
        if flush_rd is not None:
            flush_rd.sum()
        if align is not None:
            align()
        step()
    comm.check()
    barrier()
    t_wall0 = time.time()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        if flush_rd is not None:
            flush_rd.sum()  # evicts the flush's dirty lines now, not inside the timed step
        if align is not None:
            align()  # untimed tiny collective: ranks leave the flush together (no skew in the step)
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    barrier()
    t_wall1 = time.time()
    clocks = sampler.stop(t_wall0, t_wall1)
    comm.check()
    times = [a.elapsed_time(b) for a, b in evs]  # ms, one collective launch each
    ms = statistics.mean(times)
    ms = max_over_ranks(ms, world)
    per_gpu_bus = busbw(args.bytes, n, ms / 1e3)
    value = per_gpu_bus * world
    hbm, hbm_src = peaks()
    if world == 1:
        alg_bytes = 2.0 * n * args.bytes  # every replica buffer read once, written once
        achieved = alg_bytes / (ms / 1e3) / 1e9
        kname = {"flat": f"ar_virtual_flat<f32,{args.kind},{n}>", "twoshot": f"ar_twoshot<f32,{args.kind},{n}>",
                 "oneshot": f"ar_oneshot<f32,{args.kind},{n}>"}.get(args.chosen_algo, args.chosen_algo)
        traffic, tsrc = ncu_traffic(f"{kname}@{args.bytes}")
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "traffic": traffic, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({hbm_src})",
                    "algorithmic_bytes_per_launch": alg_bytes, "kernel": kname}
        if tsrc:
            roofline["traffic_source"] = tsrc
    else:
        # busBW = 2(N-1)/N * S / t against the per-direction link peak (the nccl-tests
        # convention); the bytes one GPU's links actually carry per direction are
        # 2(N-1)/N * S for the P2P two-shot and (N+1)/N * S for NVLS (the switch
        # reduces and multicasts), so NVLS can exceed the link rate in busBW terms
        algo = args.chosen_algo
        link_bytes = (n + 1) / n * args.bytes if algo == "nvls" else 2.0 * (n - 1) / n * args.bytes
        kernel = {"nvls": f"ar_nvls<f32,premean>", "twoshot": f"ar_twoshot_dyn<f32,premean,{n},pull>",
                  "oneshot": f"ar_oneshot_push<f32,premean,{n}>"}[algo]
        roofline = {"bound": "nvlink", "achieved": per_gpu_bus, "peak": NVLINK_NOMINAL_GBS, "unit": "GB/s",
                    "frac": per_gpu_bus / NVLINK_NOMINAL_GBS,
                    "frac_of_measured_peer": per_gpu_bus / NVLINK_PEER_GBS,
                    "traffic": None, "peak_source": "north star: 900 GB/s per direction per GPU (NVLink 5); "
                                                    "frac_of_measured_peer uses B200_PROFILING.md's 770 GB/s "
                                                    "measured peer copy",
                    "algorithmic_bytes_per_launch": 2.0 * (n - 1) / n * args.bytes,
                    "link_bytes_per_direction": link_bytes,
                    "link_gbs_per_direction": link_bytes / (ms / 1e3) / 1e9, "kernel": kernel}
        if getattr(args, "nvls_error", None):
            roofline["nvls_unavailable"] = args.nvls_error
        roofline["topology_rank0"] = getattr(args, "topology", None)

    # e2e: host pinned buffers -> device -> all_reduce -> host, through the public API
    e2e = run_e2e(args, comm, world, n, count, dev, stream)

    line = {
        "metric": "all_reduce bus GB/s (aggregate, 64 MiB fp32 premean)",
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (randn, seed 1234+replica)", "config": _config(args, world),
        "per_gpu_busbw_gbs": per_gpu_bus, "algbw_gbs": args.bytes / (ms / 1e3) / 1e9,
        "roofline": roofline, "clocks": clocks, "e2e": e2e, "gpu_launches": args.steps,
        "step_ms_min": min(times), "step_ms_median": statistics.median(times),
    }
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        from oracle.cpu_baseline import reference_available, time_port, time_reference

        if reference_available():
            sec, steps, thr = time_reference(n, count, args.kind, budget_s=args.cpu_budget, max_steps=50, warmup=1)
            kind, what = "reference", "steps of the reference's own Graph.evaluate (oracle/_ref) on"
        else:
            sec, steps, thr = time_port(n, count, args.kind, budget_s=args.cpu_budget, threads=1, max_steps=50)
            kind, what = "port", "stitched steps of the oracle port of"
        line["cpu_baseline"] = {"value": busbw(args.bytes, n, sec), "unit": "GB/s", "cores": thr, "kind": kind,
                                "sample": f"{steps} whole {what} the stitched program ({n} nary_{args.kind} sites x "
                                          f"{n} replicas x {args.bytes >> 20} MiB f32), single-threaded numpy",
                                "ms_per_step": sec * 1e3}
    comm.close()
    return line


def bind_host_to_gpu(local: int) -> str:
    """Restrict this process to the CPU cores NVML reports as local to its GPU, so
    the pinned host buffers of the e2e path are first-touched on the GPU's NUMA
    node (the host side of every H2D / D2H copy). Returns what was done."""
    try:
        import pynvml
        import torch

        pr = torch.cuda.get_device_properties(local)
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0")
        ncpu = os.cpu_count() or 1
        mask = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = [c for c in range(ncpu) if (mask[c // 64] >> (c % 64)) & 1]
        cpus = [c for c in cpus if c in os.sched_getaffinity(0)]
        if not cpus:
            return "unbound (no local cores in this process's affinity)"
        os.sched_setaffinity(0, cpus)
        return f"bound to the GPU's {len(cpus)} NVML-local cores"
    except Exception as e:  # no NVML / affinity support: leave the process as it is
        return f"unbound ({type(e).__name__})"


def run_e2e(args, comm, world, n, count, dev, stream):
    """The same metric through the public host-buffer API: pinned host tensors in,
    pinned host tensor out (Communicator / VirtualCommunicator.all_reduce_host,
    which pipelines chunks through pool-resident device slots so the host->device
    copies, the exchange and the device->host copy overlap)."""
    import torch

    k = max(1, args.e2e_steps)
    reps = n if world == 1 else 1
    numa = bind_host_to_gpu(dev.index if dev.index is not None else 0)
    host_in = [torch.randn(count).pin_memory() for _ in range(reps)]
    host_out = torch.empty(count).pin_memory()
    nvls = bool(getattr(args, "use_nvls", False))

    def step():
        comm.all_reduce_host(host_in if world == 1 else host_in[0], args.kind, host_out=host_out, nvls=nvls)

    step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(k):
        step()
    b.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(a.elapsed_time(b) / k, world)
    return {"value": busbw(args.bytes, n, ms / 1e3) * world, "unit": "GB/s", "ms_per_step": ms,
            "h2d_bytes_per_step": reps * count * 4, "d2h_bytes_per_step": count * 4,
            "path": "pinned host -> all_reduce_host (chunks: cudaMemcpyAsync H2D | rp_all_reduce(_v) in place "
                    "in pool slots | D2H, overlapped) -> pinned host" + (" [NVLS slots]" if nvls else ""),
            "host": numa}


def main():
    args = parse()
    if args.ar_impl:
        os.environ["RP_AR_IMPL"] = args.ar_impl
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return 0
        line = run_reference(args, 0, world_env)
        print(json.dumps(line), flush=True)
        return 0
    rank, world, local = dist_setup(args)
    line = run_ours(args, rank, world, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
