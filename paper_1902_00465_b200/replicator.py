"""The Replicator facade: TF-Replicator's API over the B200 collectives.

API surface mirrors PAPER.md:102-120 / :190-220 and SPEC.md:329-417::

    repl = Replicator()                       # one replica per process (torchrun), or
    repl = Replicator(num_replicas=4)         # 4 replicas on one GPU (in-process MultiDevice)
    with repl.context():
        model = repl.replicate(lambda: Net())          # mirrored init
        opt = repl.wrap_optimizer(torch.optim.SGD(model.parameters(), lr=0.1))
    per_replica_loss = repl.run(step_fn, input_fn)
    repl.all_reduce(x, "sum") / all_sum(x) / all_gather(x) / broadcast(x)
    repl.batch_norm(h)                                  # PAPER.md:213-219 listing
    CrossReplicaBatchNorm(C, repl)                      # per-channel K5/K5b module

Multi-process replicas use ``Communicator`` (NVLink peer memory). In-process
replicas (``num_replicas=R`` without torch.distributed) use ``VirtualCommunicator``;
each replica's step function runs in its own host thread and collectives
rendezvous across the threads, the last arrival launching ONE kernel over all
replicas -- the eager analogue of the reference's placeholder stitching
(PAPER.md:222-230), including its agreement check on
(order, label, kind, shape).
"""

from __future__ import annotations

import contextlib
import threading

import torch

from . import _lib, errors
from .bucket import GradBuckets
from .comm import DEFAULT_POOL_BYTES, Communicator, VirtualCommunicator, dtype_code

_tls = threading.local()


# ---------------------------------------------------------------------------
# per-replica containers
# ---------------------------------------------------------------------------

class PerReplica:
    """Values of all local replicas; attribute access / calls resolve to the current
    replica's instance (``Replicator.replica_id``)."""

    def __init__(self, values, repl):
        object.__setattr__(self, "values", list(values))
        object.__setattr__(self, "_repl", repl)

    @property
    def local(self):
        return self.values[self._repl._local_index()]

    def __getattr__(self, name):
        return getattr(self.local, name)

    def __call__(self, *a, **kw):
        return self.local(*a, **kw)

    def __len__(self):
        return len(self.values)

    def __getitem__(self, i):
        return self.values[i]

    def __iter__(self):
        return iter(self.values)


# ---------------------------------------------------------------------------
# virtual-replica rendezvous
# ---------------------------------------------------------------------------

class _Rendezvous:
    """All R replica threads call the same collective; the last arrival checks that
    they agree on (label, kind, shape, dtype) -- the stitcher's check
     -- runs the fused op over all replicas, and releases them."""

    def __init__(self, n):
        self.n = n
        self.cv = threading.Condition()
        self.slots: dict[int, tuple] = {}
        self.results = None
        self.error = None
        self.broken: BaseException | None = None  # a replica died: fail every later arrival
        self.gen = 0
        self.seq = 0

    def reset(self):
        with self.cv:
            self.slots, self.results, self.error, self.broken = {}, None, None, None

    def abort(self, e: BaseException):
        with self.cv:
            self.broken = e
            self.slots = {}
            self.gen += 1
            self.cv.notify_all()

    def __call__(self, r, desc, value, fn):
        with self.cv:
            if self.broken is not None:
                raise errors.CollectiveAbortedError(
                    f"replica {r}: collective {desc} aborted, another replica failed: {self.broken!r}")
            gen = self.gen
            if r in self.slots:
                raise errors.ProtocolError(f"replica {r} entered collective {desc} twice")
            self.slots[r] = (desc, value)
            if len(self.slots) == self.n:
                descs = [self.slots[i][0] for i in range(self.n)]
                try:
                    for i in range(1, self.n):
                        if descs[i] != descs[0]:
                            raise errors.ProtocolError(
                                f"collective #{self.seq}: replica 0 issued {descs[0]} but replica {i} "
                                f"issued {descs[i]} (first divergence)")
                    self.results = fn([self.slots[i][1] for i in range(self.n)])
                    self.error = None
                except BaseException as e:  # propagate to every replica
                    self.results, self.error = None, e
                self.slots = {}
                self.seq += 1
                self.gen += 1
                self.cv.notify_all()
            else:
                if not self.cv.wait_for(lambda: self.gen != gen, timeout=600):
                    raise errors.CollectiveAbortedError(f"replica {r} timed out in collective {desc}")
                if self.broken is not None:
                    raise errors.CollectiveAbortedError(
                        f"replica {r}: collective {desc} aborted, another replica failed: {self.broken!r}")
            if self.error is not None:
                raise self.error
            return self.results[r]


# ---------------------------------------------------------------------------
# differentiable collectives. The reference has no VJP for its collectives and
# raises NotDifferentiableError when backprop reaches one (graph.py:798-800).
# Multi-process replicas implement the adjoints (all_sum's adjoint is all_sum;
# all_gather's is a reduce-scatter; broadcast's sums every rank's cotangent into
# the root); in-process virtual replicas keep the reference's error, raised at
# backward time, because their backward passes run on ONE autograd device thread
# and cannot rendezvous.
# ---------------------------------------------------------------------------

class _AllReduceFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, comm, kind):
        ctx.comm, ctx.kind = comm, kind
        return comm.all_reduce_tensor(x, kind)

    @staticmethod
    def backward(ctx, g):
        if ctx.kind == "max":
            raise errors.NotDifferentiableError("all_reduce(max) has no VJP (graph.py:798-800)")
        # y = sum_r w*x_r (w = 1 or 1/N): dL/dx_r = w * sum_q dL_q/dy_q
        return ctx.comm.all_reduce_tensor(g.contiguous(), ctx.kind), None, None


class _AllGatherFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, comm):
        ctx.comm = comm
        return comm.all_gather_tensor(x)

    @staticmethod
    def backward(ctx, g):
        # y_q[r] = x_r on every rank q: dL/dx_r = sum_q dL_q/dy_q[r]
        return ctx.comm.all_reduce_tensor(g.contiguous(), "sum")[ctx.comm.rank], None


class _BroadcastFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, comm, root):
        ctx.comm, ctx.root = comm, root
        return comm.broadcast_tensor(x.detach().clone(), root=root)

    @staticmethod
    def backward(ctx, g):
        # every rank's output is root's x: root's x collects every rank's cotangent
        total = ctx.comm.all_reduce_tensor(g.contiguous(), "sum")
        return (total if ctx.comm.rank == ctx.root else torch.zeros_like(g)), None, None


class _NoVJP(torch.autograd.Function):
    """Identity in the forward; backward raises NotDifferentiableError naming the
    collective (virtual replicas, graph.py:798-800)."""

    @staticmethod
    def forward(ctx, x, y, what):
        ctx.what = what
        return y.view_as(y)

    @staticmethod
    def backward(ctx, g):
        raise errors.NotDifferentiableError(
            f"backprop reached {ctx.what} on in-process virtual replicas, which have no VJP (graph.py:798-800); "
            "use one process per GPU (torch.distributed or a loopback world) to differentiate collectives")


def _novjp(x, y, what):
    """Attach a raising backward to y when autograd would flow through x."""
    if torch.is_grad_enabled() and isinstance(x, torch.Tensor) and x.requires_grad:
        return _NoVJP.apply(x, y, what)
    return y


# ---------------------------------------------------------------------------
# Replicator
# ---------------------------------------------------------------------------

class DriverValue:
    """Result of map_gather / map_reduce: delivered to the driver.
    Reading ``.value`` inside a replicated step raises EvaluationError (the SPEC's
    "consuming the result inside a replica" error)."""

    def __init__(self, value):
        self._value = value

    @property
    def value(self):
        if getattr(_tls, "in_step", False):
            raise errors.EvaluationError("map_gather/map_reduce results are delivered to the driver: read them "
                                         "after Replicator.run returns (SPEC.md:223-231)")
        return self._value

    def __repr__(self):
        return "DriverValue(<delivered to the driver>)"


class Replicator:
    """Synchronous data-parallel Replicator (Table 1 MultiGpu/MultiWorker kinds,
    PAPER.md:150-160) whose collectives are NVLink peer-memory kernels."""

    def __init__(self, num_replicas: int | None = None, *, group=None, device: int | None = None,
                 pool_bytes: int = DEFAULT_POOL_BYTES, timeout_s: float = 20.0,
                 grad_comm_dtype: torch.dtype | None = None, bucket_bytes: int | None = None,
                 nvls_bytes: int = 0, check_protocol: bool = False, grad_views: bool = True, bootstrap=None):
        """``nvls_bytes`` > 0 (multi-process, >= 2 ranks): bind that much memory per
        rank to an NVSwitch multicast region and place gradient fusion buckets in it
        while it has room, so wrap_optimizer's reduction runs in the switch
        (RP_ALGO_NVLS; not rank-ordered -- leave 0 for bit-exact reference parity).

        ``grad_views`` (default): wrap_optimizer's gradients live in the fusion
        buckets (``param.grad`` is a view of its bucket slot), so the exchange is one
        in-place all-reduce per bucket with no pack/unpack passes (bucket.py).

        ``check_protocol`` (debug): every collective first
        checks that all ranks issue the same (generation, call index, label, kind,
        shape, dtype) and that no label repeats within a generation (one
        generation per ``run``/``new_generation``), raising ProtocolError naming the
        ranks. Virtual replicas are always checked by the rendezvous.

        ``bootstrap`` (bootstrap.py): the ranks' rendezvous -- default the
        initialised torch.distributed group; ``LoopbackWorld.bootstrap(rank)`` runs
        one-replica-per-rank communicators in one process on one GPU."""
        import torch.distributed as dist

        from .bootstrap import DistBootstrap

        if bootstrap is None and dist.is_available() and dist.is_initialized():
            bootstrap = DistBootstrap(group)
        if bootstrap is not None:
            if num_replicas not in (None, bootstrap.world):
                raise errors.ConfigurationError("num_replicas must equal the process-group size")
            self.comm = Communicator(device=device, pool_bytes=pool_bytes, timeout_s=timeout_s,
                                     bootstrap=bootstrap)
            self.kind = "multi_gpu" if self.comm.world > 1 else "non"
            self._rv = None
            if nvls_bytes > 0 and self.comm.world > 1:
                self.comm.enable_nvls(int(nvls_bytes))
        else:
            n = 1 if num_replicas is None else int(num_replicas)
            if n < 1 or n > 8:
                raise errors.ConfigurationError("1..8 replicas per communicator")
            self.comm = VirtualCommunicator(n, device=device, pool_bytes=pool_bytes, timeout_s=timeout_s)
            self.kind = "non" if n == 1 else "multi_device"
            self._rv = _Rendezvous(n)
        self.device = self.comm.device
        self.check_protocol = check_protocol
        self.comm.check_labels = check_protocol
        self._generation, self._call_index = 0, 0
        self.grad_comm_dtype = grad_comm_dtype
        self.bucket_bytes = bucket_bytes
        self.grad_views = grad_views
        self._in_context = False
        self._replicated: list[PerReplica] = []

    # -- identity ------------------------------------------------------------
    @property
    def num_replicas(self) -> int:
        return self.comm.world

    @property
    def is_virtual(self) -> bool:
        return self._rv is not None

    @property
    def replica_id(self) -> int:
        if self.is_virtual:
            return getattr(_tls, "replica", 0)
        return self.comm.rank

    def _local_index(self) -> int:
        return getattr(_tls, "replica", 0) if self.is_virtual else 0

    # -- context & replication -----------------------------------------------
    @contextlib.contextmanager
    def context(self):
        """Resources built inside are replicated ("Any resource
        constructed within the Replicator context is itself replicated")."""
        prev = self._in_context
        self._in_context = True
        try:
            yield self
        finally:
            self._in_context = prev

    def replicate(self, factory) -> PerReplica:
        """Build one instance per local replica and make every replica's parameters
        and buffers bit-identical to replica 0's (step-0 broadcast)."""
        n = self.comm.world if self.is_virtual else 1
        objs = [factory() for _ in range(n)]
        for o in objs:
            if isinstance(o, torch.nn.Module):
                o.to(f"cuda:{self.device}")
        self._sync_state(objs)
        pr = PerReplica(objs, self)
        self._replicated.append(pr)
        return pr

    def _sync_state(self, objs):
        if not isinstance(objs[0], torch.nn.Module):
            return
        tensors = [list(o.parameters()) + list(o.buffers()) for o in objs]
        with torch.no_grad():
            for k in range(len(tensors[0])):
                if self.is_virtual:
                    if self.comm.world > 1:
                        xs = [t[k].data for t in tensors]
                        outs = self.comm.broadcast(xs, root=0)
                        for t, o in zip(tensors, outs):
                            t[k].data.copy_(o)
                else:
                    if self.comm.world > 1:
                        self.comm.broadcast_tensor(tensors[0][k].data, root=0)

    def wrap_optimizer(self, optimizer, kind: str = "premean", fused: bool = False, overlap: bool = False,
                       overlap_blocks: int | None = None):
        """apply_gradients first averages every gradient across
        replicas with all_sum(g / R), then applies the base rule.

        ``overlap=True`` (one replica per process): the same averaging, started
        bucket by bucket from post-accumulate-grad hooks on a side stream while
        backward runs (overlap.py); ``step()`` joins it.

        ``fused=True`` (torch.optim.SGD / Adam / AdamW, f32 parameters): the
        average and the update run as one kernel that updates each rank's shard and
        stores the new parameters on every replica (fused.py, csrc/rp_apply.cu)."""
        if isinstance(optimizer, PerReplica):
            opts = list(optimizer.values)
        else:
            opts = [optimizer]
        if self.is_virtual and len(opts) != self.comm.world and self.comm.world > 1:
            raise errors.ConfigurationError("virtual replicas need one optimizer per replica "
                                            "(repl.replicate(lambda: make_opt(...)))")
        if fused:
            if kind != "premean":
                raise errors.ConfigurationError("fused apply averages with the premean fold")
            if overlap:
                raise errors.ConfigurationError("fused=True and overlap=True are exclusive")
            from .fused import FusedReplicatedOptimizer
            return FusedReplicatedOptimizer(self, opts)
        if overlap:
            from .overlap import OverlappedReplicatedOptimizer
            return OverlappedReplicatedOptimizer(self, opts[0], kind, blocks=overlap_blocks)
        return ReplicatedOptimizer(self, opts, kind)

    # -- run ----------------------------------------------------------------
    def run(self, step_fn, input_fn=None):
        """Run one step of every local replica.

        input_fn(replica_id) returns the replica's inputs or a callable producing
        them (PER_REPLICA mode). Returns a list of per-replica
        outputs (this process's replica only, for multi-process replicators)."""
        def one(r):
            inp = None
            if input_fn is not None:
                inp = input_fn(r)
                if callable(inp):
                    inp = inp()
            _tls.in_step = True
            try:
                return step_fn(inp) if input_fn is not None else step_fn()
            finally:
                _tls.in_step = False

        self.new_generation()
        if self.comm.world == 1 or not self.is_virtual:
            _tls.replica = 0
            if self.is_virtual:
                return [one(0)]
            return [one(self.comm.rank)]
        n = self.comm.world
        results, errs = [None] * n, [None] * n
        self._rv.reset()

        def worker(r):
            _tls.replica = r
            try:
                with torch.cuda.device(self.device):
                    results[r] = one(r)
            except BaseException as e:
                errs[r] = e
                self._rv.abort(e)  # unblock waiting replicas and fail late arrivals

        threads = [threading.Thread(target=worker, args=(r,), name=f"replica-{r}") for r in range(n)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        root = [e for e in errs if e is not None and not isinstance(e, errors.CollectiveAbortedError)]
        if root or any(e is not None for e in errs):
            raise (root or [e for e in errs if e is not None])[0]
        return results

    # -- primitives --------------------------------------
    def _collective(self, desc, x, fn_virtual):
        return self._rv(self.replica_id, desc, x, fn_virtual)

    def new_generation(self) -> None:
        """Start a new generation (training step): labels may repeat."""
        self._generation += 1
        self._call_index = 0
        self.comm.new_generation()

    def _verify(self, label, kind, shape, dtype, plan=None):
        """check_protocol on a multi-process replicator: all ranks must be issuing
        the same collective at the same position of the generation -- and, for an
        all-reduce, with the same plan (algorithm, data-movement form, pool
        placement; include/rp.h rp_all_reduce_plan), since ranks that place their
        buffers differently would launch different kernels."""
        if not self.check_protocol or self.is_virtual or self.comm.world == 1:
            return
        self.comm._use_label(label)
        self.comm.verify(label, kind if plan is None else (kind, plan), shape, dtype,
                         position=(self._generation, self._call_index))
        self._call_index += 1

    def all_reduce(self, x: torch.Tensor, kind: str = "sum", label: str | None = None) -> torch.Tensor:
        """Cross-replica fold of x (sum / mean / max / premean), ascending replica order."""
        if self.comm.world == 1:
            return _AllReduceFn.apply(x, self.comm, kind) if not self.is_virtual else x.clone()
        if self.is_virtual:
            y = self._collective(("all_reduce", label, kind, tuple(x.shape), x.dtype), x.detach(),
                                 lambda xs: self.comm.all_reduce(xs, kind))
            return _novjp(x, y, f"all_reduce({kind})")
        plan = self.comm.plan_for(x.detach(), kind) if self.check_protocol else None
        self._verify(label, kind, x.shape, x.dtype, plan)
        return _AllReduceFn.apply(x, self.comm, kind)

    def all_sum(self, x: torch.Tensor, label: str | None = None) -> torch.Tensor:
        return self.all_reduce(x, "sum", label)

    def all_gather(self, x: torch.Tensor, label: str | None = None, ragged: bool = False, stack: bool = False):
        """every replica gets the list [x_0, ..., x_{R-1}] in replica
        order (views of one gathered buffer). ``ragged=True``: leading dimensions may
        differ across replicas. ``stack=True``: the one (R,) + x.shape
        tensor instead of the list (same bits, no split)."""
        if ragged and stack:
            raise errors.ShapeError("all_gather: a ragged gather cannot be stacked")
        if self.is_virtual:
            if self.comm.world == 1:
                g = x.unsqueeze(0).clone()
            elif ragged:
                parts = self._collective(("all_gather_ragged", label, tuple(x.shape[1:]), x.dtype), x.detach(),
                                         lambda xs: self.comm.all_gather_ragged(xs))
                return [_novjp(x, t, "all_gather") for t in parts]
            else:
                g = _novjp(x, self._collective(("all_gather", label, tuple(x.shape), x.dtype), x.detach(),
                                               lambda xs: self.comm.all_gather(xs)), "all_gather")
        else:
            self._verify(label, "gather", x.shape[1:] if ragged else x.shape, x.dtype)
            if ragged:
                if torch.is_grad_enabled() and x.requires_grad:
                    raise errors.NotDifferentiableError("ragged all_gather has no VJP; gather x.detach()")
                return self.comm.all_gather_ragged(x)
            g = _AllGatherFn.apply(x, self.comm)
        return g if stack else list(g.unbind(0))

    def broadcast(self, x: torch.Tensor, root: int = 0, label: str | None = None) -> torch.Tensor:
        if self.is_virtual:
            if self.comm.world == 1:
                return x.clone()
            y = self._collective(("broadcast", label, root, tuple(x.shape), x.dtype), x.detach(),
                                 lambda xs: self.comm.broadcast(xs, root=root))
            return _novjp(x, y, "broadcast")
        self._verify(label, f"broadcast(root={root})", x.shape, x.dtype)
        return _BroadcastFn.apply(x, self.comm, root)

    def map_gather(self, x: torch.Tensor, label: str | None = None) -> "DriverValue":
        """per-replica values collected to the driver; replicas get
        nothing back. Returns a DriverValue whose ``.value`` (the list of every
        replica's x in replica order; leading dimensions may differ) can be read
        only outside the replicated step -- e.g. from Replicator.run's outputs."""
        vals = self.all_gather(x.detach(), label=label, ragged=True)
        return DriverValue(list(vals))

    def map_reduce(self, x: torch.Tensor, kind: str = "sum", label: str | None = None) -> "DriverValue":
        """the replicas' values folded (rank order) for the driver."""
        return DriverValue(self.all_reduce(x.detach(), kind, label=label))

    def batch_norm(self, h: torch.Tensor, eps: float = 1e-5) -> torch.Tensor:
        """The paper's cross-replica batch norm listing with the
        variance written as mean_sq - mean**2:
            mean = all_sum(reduce_mean(h) / R); mean_sq = all_sum(reduce_mean(h**2) / R)
            out = (h - mean) / sqrt(mean_sq - mean**2 + eps)
        Per-tensor statistics like the listing; see CrossReplicaBatchNorm for the
        per-channel K5/K5b kernels."""
        r = self.num_replicas
        stats = torch.stack([h.mean() / r, (h * h).mean() / r])
        stats = self.all_sum(stats, label="batch_norm")
        mean, mean_sq = stats[0], stats[1]
        return (h - mean) / torch.sqrt(mean_sq - mean * mean + eps)


class ReplicatedOptimizer:
    """``wrap_optimizer`` result: averages gradients across
    replicas with the rank-ordered all_sum(g/R) fold, then runs the base rule.

    The averaging runs over fusion buckets in the registered pool (bucket.py),
    with the optional f32->bf16 exchange cast (``Replicator(grad_comm_dtype=...)``).
    """

    def __init__(self, repl: Replicator, opts, kind="premean"):
        self.repl = repl
        self.opts = opts
        self.kind = kind
        self._buckets: GradBuckets | None = None
        self._steps = 0

    @property
    def optimizer(self):
        return self.opts[self.repl._local_index()]

    @property
    def param_groups(self):
        return self.optimizer.param_groups

    def _params(self, opt):
        return [p for g in opt.param_groups for p in g["params"]]

    def _build(self):
        plists = [self._params(o) for o in self.opts]
        self._buckets = GradBuckets(self.repl.comm, plists, comm_dtype=self.repl.grad_comm_dtype,
                                    bucket_bytes=self.repl.bucket_bytes, views=self.repl.grad_views)

    def zero_grad(self, set_to_none: bool = False):
        self.optimizer.zero_grad(set_to_none=set_to_none)

    def average_gradients(self):
        """all_sum(g / R) for every gradient (bit-identical on every replica)."""
        if self.repl.num_replicas == 1:
            return
        if self.repl.is_virtual:
            self.repl._collective(("wrap_optimizer", id(self)), None, self._reduce_all)
        else:
            if self._buckets is None:
                self._build()
            self._buckets.reduce(self.kind)

    def _reduce_all(self, _values):
        if self._buckets is None:
            self._build()
        self._buckets.reduce(self.kind)
        return [None] * self.repl.num_replicas

    def step(self, closure=None):
        self.average_gradients()
        self._steps += 1
        return self.optimizer.step(closure) if closure is not None else self.optimizer.step()

    def apply_gradients(self, grads_and_vars):
        """TF-style entry point: set the given gradients, average
        them across replicas, apply the base rule."""
        for g, v in grads_and_vars:
            v.grad = g.detach().clone() if g is not None else None
        return self.step()

    def state_dict(self):
        return self.optimizer.state_dict()

    def load_state_dict(self, sd):
        return self.optimizer.load_state_dict(sd)


# ---------------------------------------------------------------------------
# Cross-replica batch norm (K5 / K5b)
# ---------------------------------------------------------------------------

def _bn_layout(x: torch.Tensor):
    """(layout, rows, C, hw) for a DENSE x of shape [N, C] or [N, C, *spatial] that
    the kernels can read as stored; None for any other strides (stride-0 expands,
    transposes, slices), which the caller makes dense first."""
    if x.dim() == 2:
        return (_lib.NHWC, x.shape[0], x.shape[1], 1) if x.is_contiguous() else None
    n, c = x.shape[0], x.shape[1]
    hw = 1
    for s in x.shape[2:]:
        hw *= s
    if x.is_contiguous():
        return _lib.NCHW, n, c, hw
    if x.dim() == 4 and x.is_contiguous(memory_format=torch.channels_last):
        return _lib.NHWC, n * hw, c, 1
    if x.dim() == 5 and x.is_contiguous(memory_format=torch.channels_last_3d):
        return _lib.NHWC, n * hw, c, 1
    return None


def _like_layout(t: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    """t made dense in the memory format the kernels read x in (x already dense)."""
    if x.dim() == 4 and not x.is_contiguous() and x.is_contiguous(memory_format=torch.channels_last):
        return t.contiguous(memory_format=torch.channels_last)
    if x.dim() == 5 and not x.is_contiguous() and x.is_contiguous(memory_format=torch.channels_last_3d):
        return t.contiguous(memory_format=torch.channels_last_3d)
    return t.contiguous()


def _bn_stats(comm, xs, eps):
    """K5 over the local replicas' inputs ``xs`` (one tensor per local replica).
    Returns per-replica (mean, var, invstd, count) on the device."""
    lib = _lib.load()
    x0 = xs[0]
    layout, rows, c, hw = _bn_layout(x0)
    dev = x0.device
    stream = comm._stream()
    outs = [(torch.empty(c, dtype=torch.float32, device=dev), torch.empty(c, dtype=torch.float32, device=dev),
             torch.empty(c, dtype=torch.float32, device=dev), torch.empty(1, dtype=torch.float64, device=dev))
            for _ in xs]
    if isinstance(comm, VirtualCommunicator):
        arrs = [_lib.ptr_array([x.data_ptr() for x in xs])] + \
               [_lib.ptr_array([o[k].data_ptr() for o in outs]) for k in range(4)]
        ptrs = [ctypes_cast(a[0]) for a in arrs]
        _lib.check(lib.rp_bn_stats(comm._handle, ptrs[0], dtype_code(x0.dtype), rows, c, hw, layout, float(eps),
                                   ptrs[1], ptrs[2], ptrs[3], ptrs[4], stream), "bn_stats")
    else:
        o = outs[0]
        _lib.check(lib.rp_bn_stats(comm._handle, x0.data_ptr(), dtype_code(x0.dtype), rows, c, hw, layout,
                                   float(eps), o[0].data_ptr(), o[1].data_ptr(), o[2].data_ptr(), o[3].data_ptr(),
                                   stream), "bn_stats")
    return outs


def ctypes_cast(p):
    import ctypes
    return ctypes.cast(p, ctypes.c_void_p).value


class _CrossReplicaBNFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, owner, eps, running_mean, running_var, momentum, training):
        comm = owner.comm if isinstance(owner, Replicator) else owner
        if _bn_layout(x) is None:
            x = x.contiguous()
        layout, rows, c, hw = _bn_layout(x)
        lib = _lib.load()
        dev = x.device
        stream = torch.cuda.current_stream(dev).cuda_stream
        code = dtype_code(x.dtype)
        if training:
            if isinstance(comm, VirtualCommunicator) and comm.world > 1:
                if not isinstance(owner, Replicator):
                    raise errors.ConfigurationError("virtual replicas: build CrossReplicaBatchNorm with the Replicator")
                mean, var, invstd, count = owner._collective(
                    ("batch_norm", tuple(x.shape), x.dtype, layout), x, lambda xs: _bn_stats(comm, xs, eps))
            else:
                mean, var, invstd, count = _bn_stats(comm, [x], eps)[0]
            if running_mean is not None:
                with torch.no_grad():
                    m = count.to(torch.float32)
                    unbiased = var * m / torch.clamp(m - 1, min=1)
                    running_mean.mul_(1 - momentum).add_(momentum * mean)
                    running_var.mul_(1 - momentum).add_(momentum * unbiased)
        else:
            mean = running_mean.float()
            var = running_var.float()
            invstd = torch.rsqrt(var + eps)
            count = None
        y = torch.empty_like(x)
        w = weight.float().contiguous() if weight is not None else None
        b = bias.float().contiguous() if bias is not None else None
        _lib.check(lib.rp_bn_apply(x.data_ptr(), y.data_ptr(), code, rows, c, hw, layout, mean.data_ptr(),
                                   invstd.data_ptr(), w.data_ptr() if w is not None else None,
                                   b.data_ptr() if b is not None else None, stream), "bn_apply")
        ctx.save_for_backward(x, w if w is not None else torch.empty(0, device=dev), mean, invstd)
        ctx.meta = (comm, layout, rows, c, hw, weight is not None, bias is not None, training, count,
                    weight.dtype if weight is not None else None)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, w, mean, invstd = ctx.saved_tensors
        comm, layout, rows, c, hw, has_w, has_b, training, count, wdt = ctx.meta
        if not training:
            raise errors.ShapeError("cross-replica BN backward in eval mode is not supported")
        if isinstance(comm, VirtualCommunicator) and comm.world > 1:
            raise errors.NotDifferentiableError(
                "cross-replica BN backward needs one process per GPU (or a loopback world); in-process virtual "
                "replicas support the forward statistics only (as the reference, whose collectives have no VJP, "
                "graph.py:798-800)")
        if _bn_layout(dy) != (layout, rows, c, hw):
            dy = _like_layout(dy, x)
        lib = _lib.load()
        dev = x.device
        stream = comm._stream()
        code = dtype_code(x.dtype)
        sum_dy = torch.empty(c, dtype=torch.float32, device=dev)
        sum_dy_xmu = torch.empty_like(sum_dy)
        loc_dy = torch.empty_like(sum_dy)
        loc_dy_xmu = torch.empty_like(sum_dy)
        args = [x, dy, mean, sum_dy, sum_dy_xmu, loc_dy, loc_dy_xmu]
        if isinstance(comm, VirtualCommunicator):  # one local replica: per-replica pointer arrays
            keep = [_lib.ptr_array([t.data_ptr()]) for t in args]
            ptrs = [ctypes_cast(k[0]) for k in keep]
        else:
            ptrs = [t.data_ptr() for t in args]
        _lib.check(lib.rp_bn_bwd_stats(comm._handle, ptrs[0], ptrs[1], code, rows, c, hw, layout, *ptrs[2:], stream),
                   "bn_bwd_stats")
        dx = torch.empty_like(x)
        # the global count M stays on the device (no host sync per backward)
        m_total = float(rows * hw * comm.world)
        _lib.check(lib.rp_bn_bwd_apply(x.data_ptr(), dy.data_ptr(), dx.data_ptr(), code, rows, c, hw, layout,
                                       mean.data_ptr(), invstd.data_ptr(), w.data_ptr() if has_w else None,
                                       sum_dy.data_ptr(), sum_dy_xmu.data_ptr(), m_total,
                                       count.data_ptr() if count is not None else None, stream), "bn_bwd_apply")
        dw = (loc_dy_xmu * invstd).to(wdt) if has_w else None
        db = loc_dy.to(wdt) if has_b else None
        return dx, dw, db, None, None, None, None, None, None


class CrossReplicaBatchNorm(torch.nn.Module):
    """Per-channel cross-replica batch norm over [N, C, *] inputs (NCHW-contiguous or
    channels_last), forward statistics by K5 and backward by K5b. Statistics are
    those of the concatenated global batch; biased variance for
    normalisation, unbiased for the running estimate."""

    def __init__(self, num_features: int, repl_or_comm, eps: float = 1e-5, momentum: float = 0.1,
                 affine: bool = True, track_running_stats: bool = True):
        super().__init__()
        self.owner = repl_or_comm
        self.num_features, self.eps, self.momentum = num_features, eps, momentum
        if affine:
            self.weight = torch.nn.Parameter(torch.ones(num_features))
            self.bias = torch.nn.Parameter(torch.zeros(num_features))
        else:
            self.register_parameter("weight", None)
            self.register_parameter("bias", None)
        if track_running_stats:
            self.register_buffer("running_mean", torch.zeros(num_features))
            self.register_buffer("running_var", torch.ones(num_features))
        else:
            self.running_mean = self.running_var = None

    def forward(self, x):
        if x.shape[1] != self.num_features:
            raise errors.ShapeError(f"expected {self.num_features} channels, got {x.shape[1]}")
        training = self.training or self.running_mean is None
        return _CrossReplicaBNFn.apply(x, self.weight, self.bias, self.owner, self.eps, self.running_mean,
                                       self.running_var, self.momentum, training)
