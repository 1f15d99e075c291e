"""Bootstrap: how the ranks of a communicator find each other before any kernel runs.

Only the 144-byte export blobs (CUDA IPC handle, device identity) and, for NVLS,
one socket name travel here; no collective data path ever does (the reference's
transport, is replaced by NVLink peer memory).

* ``DistBootstrap`` -- one process per GPU over an initialised ``torch.distributed``
  process group (any backend; gloo is enough).
* ``LoopbackWorld`` -- ``world`` ranks in ONE process on ONE GPU, each driven from
  its own host thread and CUDA stream (include/rp.h rp_comm_set_loopback). The
  kernels, barriers, pool layout and algorithm choices are exactly those of one
  process per GPU -- only the NVLink hop becomes local HBM -- so the multi-process
  forms (push one-shot / two-shot, push all-gather and broadcast, relay broadcast,
  BN exchange and its autograd, fused apply, protocol checks, timeouts) run and are
  checked against the oracle on a single B200.
"""

from __future__ import annotations

import threading
import traceback

import torch


class DistBootstrap:
    """Rendezvous over ``torch.distributed`` (handle exchange only)."""

    loopback = False

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather_object(self, obj) -> list:
        import torch.distributed as dist

        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.group)
        return out

    def broadcast_object(self, obj, src: int = 0):
        import torch.distributed as dist

        box = [obj if self.rank == src else None]
        dist.broadcast_object_list(box, src=src, group=self.group)
        return box[0]

    def barrier(self) -> None:
        import torch.distributed as dist

        dist.barrier(group=self.group)


class _LoopbackBootstrap:
    loopback = True

    def __init__(self, world: "LoopbackWorld", rank: int):
        self._w = world
        self.rank = rank
        self.world = world.world

    def all_gather_object(self, obj) -> list:
        w = self._w
        w._slots[self.rank] = obj
        self.barrier()
        out = list(w._slots)
        self.barrier()  # nobody overwrites a slot before every rank read it
        return out

    def broadcast_object(self, obj, src: int = 0):
        return self.all_gather_object(obj if self.rank == src else None)[src]

    def barrier(self) -> None:
        self._w._barrier.wait()


class LoopbackWorld:
    """``world`` ranks of one data-parallel group in this process, all on ``device``.

    ``run(fn, *args)`` calls ``fn(rank, *args)`` in one thread per rank, each with
    ``device`` current and its OWN non-default CUDA stream current (ranks must never
    share a stream: rank 0's kernel waits for rank 1's). Returns the per-rank results
    in rank order; if any rank raises, the host barrier is broken so no rank hangs in
    bootstrap, and the first failure is re-raised with every failing rank's
    traceback. Build communicators inside ``fn`` with ``bootstrap=world.bootstrap(rank)``.
    """

    def __init__(self, world: int, device: int = 0, timeout_s: float = 300.0, allow_native_allocator: bool = False):
        """Requires PyTorch's stream-ordered allocator
        (``PYTORCH_CUDA_ALLOC_CONF=backend:cudaMallocAsync`` before CUDA starts):
        the native caching allocator's cudaMalloc can wait for the whole device,
        i.e. for a peer rank's kernel that is itself waiting for this rank's next
        launch -- a deadlock broken only by the kernels' timeout (measured: the
        first collective of a larger message after smaller ones timed out). The
        device's memory pool is then set to never reuse memory across streams
        through an inserted wait (include/rp.h rp_loopback_prepare), which could
        close the same cycle. Ranks copy results to the host through pinned
        memory (comm.to_host): a pageable copy can wait on a peer's kernel too."""
        from . import errors

        if world < 1 or world > 8:
            raise ValueError("a loopback world has 1..8 ranks")
        if world > 1 and not allow_native_allocator and torch.cuda.memory.get_allocator_backend() != "cudaMallocAsync":
            raise errors.ConfigurationError(
                "a loopback world needs PYTORCH_CUDA_ALLOC_CONF=backend:cudaMallocAsync (set before CUDA "
                "initialises): the native allocator's cudaMalloc can block on a peer rank's waiting kernel")
        self.world, self.device = int(world), int(device)
        if world > 1 and torch.cuda.is_available():
            from . import _lib
            _lib.check(_lib.load().rp_loopback_prepare(self.device), "loopback_prepare")
        self._barrier = threading.Barrier(self.world, timeout=timeout_s)
        self._slots = [None] * self.world

    def bootstrap(self, rank: int) -> _LoopbackBootstrap:
        return _LoopbackBootstrap(self, rank)

    def run(self, fn, *args, **kwargs) -> list:
        results = [None] * self.world
        errs: list = [None] * self.world

        def worker(r):
            try:
                torch.cuda.set_device(self.device)
                stream = torch.cuda.Stream(device=self.device)
                with torch.cuda.stream(stream):
                    results[r] = fn(r, *args, **kwargs)
                stream.synchronize()
            except BaseException as e:  # noqa: BLE001 -- reported below
                errs[r] = (e, traceback.format_exc())
                self._barrier.abort()

        threads = [threading.Thread(target=worker, args=(r,), name=f"loopback-rank-{r}") for r in range(self.world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        bad = [(r, e) for r, e in enumerate(errs) if e is not None]
        if bad:
            # the root cause first: a rank whose failure is not the broken barrier
            bad.sort(key=lambda re: isinstance(re[1][0], threading.BrokenBarrierError))
            msg = "\n".join(f"--- loopback rank {r} ---\n{tb}" for r, (_, tb) in bad)
            raise RuntimeError(f"loopback world of {self.world} failed on ranks {[r for r, _ in bad]}:\n{msg}") \
                from bad[0][1][0]
        return results
