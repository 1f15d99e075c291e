"""wrap_optimizer(opt, overlap=True): the gradient all-reduce overlapped with backward.

The reference's wrapped optimizer averages gradients inside ``apply_gradients``,
after the whole backward pass. The arithmetic
here is the same -- each gradient is averaged with the rank-ordered
``all_sum(g / R)`` premean fold, bit-identical to the synchronous
``ReplicatedOptimizer`` -- but the exchange starts while backward is still running
(SURVEY.md §8(f) row 2):

* gradients are grouped into fusion buckets in REVERSE parameter order (backward
  produces the last layers' gradients first), cut at ``bucket_bytes``;
* every parameter carries a post-accumulate-grad hook; when the last gradient of
  a bucket has been accumulated, the bucket is packed, reduced in place in the
  registered pool and unpacked on a high-priority side stream that waits only for
  the compute stream's work up to that point;
* buckets are launched strictly in bucket order on every rank (a bucket that
  becomes ready early waits for its predecessors), so the sequence of collectives
  is identical across ranks whatever order autograd fires the hooks in -- the
  cross-rank agreement the collectives' device-side sequencing relies on
  (SPEC.md:182-186);
* ``step()`` launches any bucket still pending (parameters that received no
  gradient are exchanged as zeros, like the synchronous path), joins the side
  stream into the compute stream and runs the base rule.

Gradient accumulation over several backward passes: wrap all but the last in
``opt.no_sync()``; a gradient accumulated again after its bucket was launched is a
protocol error (the averaged value would be overwritten by a local one).

Measured (profiles/r01_resnet50_overlap.txt): on ResNet-50 over NVLink the
synchronous exchange costs 0.13-0.19 ms of a 17.3 ms step, while the per-bucket
cross-stream dependencies this mode needs cost ~0.3 ms and the concurrent exchange
a little more, so ``overlap=False`` (the default) is faster there. Overlap pays when
the exchange is a large share of the step.
"""

from __future__ import annotations

import contextlib
import time

import torch

from . import errors
from .bucket import _Bucket
from .comm import Communicator


class InOrderLauncher:
    """Readiness bookkeeping for buckets that must be launched in index order.

    ``mark(i)`` records that bucket i is ready and returns the indices that may be
    launched now (the ready prefix not yet launched). Host-only logic: tested on
    CPU (tests/test_host.py)."""

    def __init__(self, n: int):
        self.n = n
        self.reset()

    def reset(self):
        self.ready = [False] * self.n
        self.next = 0

    def mark(self, i: int) -> list[int]:
        if i < self.next or self.ready[i]:
            raise errors.ProtocolError(f"bucket {i} marked ready twice in one step")
        self.ready[i] = True
        out = []
        while self.next < self.n and self.ready[self.next]:
            out.append(self.next)
            self.next += 1
        return out

    def rest(self) -> list[int]:
        """Indices still to launch, in order (end of the step)."""
        out = list(range(self.next, self.n))
        for i in out:
            self.ready[i] = True
        self.next = self.n
        return out


def bucket_plan(sizes_bytes, dtypes, limit: int) -> list[list[int]]:
    """Parameter indices per bucket: reverse order, one dtype per bucket, a new
    bucket when the next gradient would push the current one past ``limit``
    (a single larger gradient gets a bucket of its own)."""
    plan: list[list[int]] = []
    open_: dict = {}
    for i in reversed(range(len(sizes_bytes))):
        dt = dtypes[i]
        cur = open_.get(dt)
        if cur is not None and cur[1] + sizes_bytes[i] > limit:
            cur = None
        if cur is None:
            cur = [[], 0]
            open_[dt] = cur
            plan.append(cur[0])
        cur[0].append(i)
        cur[1] += sizes_bytes[i]
    return plan


class OverlappedReplicatedOptimizer:
    """``wrap_optimizer(opt, overlap=True)`` result: see the module docstring."""

    DEFAULT_BUCKET_BYTES = 8 << 20
    DEFAULT_BLOCKS = 32

    def __init__(self, repl, opt, kind: str = "premean", bucket_bytes: int | None = None,
                 blocks: int | None = None, priority: int = -1):
        """``blocks``: grid cap (blocks per rank) of the exchanges launched during
        backward, so they leave most SMs to the backward kernels (0: no cap)."""
        if repl.is_virtual or not isinstance(repl.comm, Communicator):
            raise errors.ConfigurationError("overlap=True needs one replica per process (torch.distributed); "
                                            "in-process replicas rendezvous on host threads after backward")
        self.repl, self.opts, self.kind = repl, [opt], kind
        self.comm: Communicator = repl.comm
        params = [p for g in opt.param_groups for p in g["params"] if p.requires_grad]
        seen, uniq = set(), []
        for p in params:
            if id(p) not in seen:
                seen.add(id(p))
                uniq.append(p)
        self.params = uniq
        limit = int(bucket_bytes or repl.bucket_bytes or self.DEFAULT_BUCKET_BYTES)
        cdt = repl.grad_comm_dtype
        esz = [p.numel() * torch.empty((), dtype=(cdt if (cdt is not None and p.dtype == torch.float32)
                                                   else p.dtype)).element_size() for p in uniq]
        plan = bucket_plan(esz, [p.dtype for p in uniq], limit)
        self.buckets: list[_Bucket] = []
        self._where: dict[int, int] = {}
        self._slot: dict[int, int] = {}
        for bi, idx in enumerate(plan):
            dt = uniq[idx[0]].dtype
            comm_dt = cdt if (cdt is not None and dt == torch.float32) else dt
            self.buckets.append(_Bucket(self.comm, [[uniq[i] for i in idx]], dt, comm_dt,
                                        views=getattr(repl, "grad_views", True)))
            for k, i in enumerate(idx):
                self._where[id(uniq[i])] = bi
                self._slot[id(uniq[i])] = k
        self._left = [len(idx) for idx in plan]
        self._pending = list(self._left)
        self._detached = [False] * len(self.buckets)  # a gradient stopped being its bucket view
        self.hook_s = 0.0  # host seconds spent in the hooks (diagnostics)
        self._order = InOrderLauncher(len(self.buckets))
        self.stream = torch.cuda.Stream(device=self.comm.device, priority=priority)
        self.blocks = self.DEFAULT_BLOCKS if blocks is None else int(blocks)
        self._sync = True
        self._draining = False
        self._steps = 0
        self._hooks = [p.register_post_accumulate_grad_hook(self._on_grad) for p in uniq]

    # -- optimizer facade ----------------------------------------------------
    @property
    def optimizer(self):
        return self.opts[0]

    @property
    def param_groups(self):
        return self.optimizer.param_groups

    def zero_grad(self, set_to_none: bool = False):
        self.optimizer.zero_grad(set_to_none=set_to_none)

    def state_dict(self):
        return self.optimizer.state_dict()

    def load_state_dict(self, sd):
        return self.optimizer.load_state_dict(sd)

    @contextlib.contextmanager
    def no_sync(self):
        """Backward passes inside only accumulate local gradients."""
        prev = self._sync
        self._sync = False
        try:
            yield
        finally:
            self._sync = prev

    def remove_hooks(self):
        for h in self._hooks:
            h.remove()
        self._hooks = []

    # -- overlap machinery ----------------------------------------------------
    def _on_grad(self, p):
        if not self._sync or self.repl.num_replicas == 1:
            return
        t0 = time.perf_counter()
        try:
            self._ready(p)
        finally:
            self.hook_s += time.perf_counter() - t0

    def _ready(self, p):
        bi = self._where[id(p)]
        if self._pending[bi] == 0:
            raise errors.ProtocolError(
                f"a gradient of bucket {bi} was accumulated again after the bucket was exchanged; "
                "wrap all but the last backward of an accumulation in opt.no_sync()")
        b = self.buckets[bi]
        if b.views and not b.is_attached(0, self._slot[id(p)]):
            self._detached[bi] = True
        self._pending[bi] -= 1
        if self._pending[bi] == 0:
            for i in self._order.mark(bi):
                self._launch(i)

    def _launch(self, i: int):
        b = self.buckets[i]
        self._pending[i] = 0
        grads = None if b.views else [b._grads(0)]  # dense fix-ups on the compute stream
        cur = torch.cuda.current_stream(self.comm.device)
        self.stream.wait_stream(cur)
        self.comm.set_block_cap(self.blocks)  # same value on every rank, same position in the sequence
        try:
            with torch.cuda.stream(self.stream):
                # gradients checked one by one in the hooks: attach only when one moved
                attached = b.views and self._pending[i] == 0 and not self._detached[i] and not self._draining
                b.reduce(self.kind, grads, attached=attached)
        finally:
            self.comm.set_block_cap(0)
        for g in (grads[0] if grads else ()):
            g.record_stream(self.stream)

    def average_gradients(self):
        """Launch the buckets backward did not complete, then make the compute
        stream wait for every exchange of this step."""
        if self.repl.num_replicas == 1:
            return
        self._draining = True  # buckets backward did not complete: attach everything
        try:
            for i in self._order.rest():
                self._launch(i)
        finally:
            self._draining = False
        torch.cuda.current_stream(self.comm.device).wait_stream(self.stream)
        self._order.reset()
        self._pending = list(self._left)
        self._detached = [False] * len(self.buckets)

    def step(self, closure=None):
        self.average_gradients()
        self._steps += 1
        return self.optimizer.step(closure) if closure is not None else self.optimizer.step()

    def apply_gradients(self, grads_and_vars):
        """TF-style entry point: set the gradients (no backward ran, so every bucket
        is launched here), average, apply."""
        for g, v in grads_and_vars:
            v.grad = g.detach().clone() if g is not None else None
        return self.step()
