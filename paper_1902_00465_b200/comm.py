"""Communicators: the reference-facing collective seam over the sm_100a C ABI.

``Communicator`` is one rank of a data-parallel group, one process per GPU. It
implements the duck-typed interface the reference's mesh seam calls
(``pkg/src/replicator/graph.py:565-583``)::

    comm.rank
    comm.all_reduce(local, kind in {"sum","mean","max"}, label) -> Tensor  (graph.py:573-574)
    comm.all_gather(local, label) -> [Tensor] in rank order                (graph.py:575-579)
    comm.broadcast(root_value | None, label, shape=..., dtype=...) -> Tensor (graph.py:580-582)

accepting reference ``Tensor`` objects (anything with ``.np``), numpy arrays or torch
tensors, and returning the same kind. Torch CUDA tensors stay on the device; host
values are copied in and out around the kernel.

``VirtualCommunicator`` holds R replicas on ONE GPU -- the reference's in-process
MultiDevice replication, whose stitched folds are graph.py:506-540 -- and runs each
collective as one cooperative kernel over all replicas' buffers.

Bootstrap (bootstrap.py) exchanges only the CUDA IPC handle blobs -- over
``torch.distributed`` between processes, or in-process for a loopback world; no
NCCL call sits on any collective path.
"""

from __future__ import annotations

import ctypes
import hashlib
import os

import numpy as np
import torch

from . import _lib, errors

DEFAULT_POOL_BYTES = int(os.environ.get("RP_POOL_BYTES", str(512 << 20)))
_ALIGN = 256

_TORCH_CODE = {torch.float32: _lib.F32, torch.float64: _lib.F64, torch.bfloat16: _lib.BF16,
               torch.float16: _lib.F16}
_NP_CODE = {np.dtype(np.float32): _lib.F32, np.dtype(np.float64): _lib.F64}
_NAME_CODE = {"f32": _lib.F32, "f64": _lib.F64, "bf16": _lib.BF16, "f16": _lib.F16}
_CODE_TORCH = {v: k for k, v in _TORCH_CODE.items()}
_REF_DTYPE = {torch.float32: "f32", torch.float64: "f64"}


def dtype_code(dt) -> int:
    if isinstance(dt, torch.dtype):
        code = _TORCH_CODE.get(dt)
    elif isinstance(dt, str):
        code = _NAME_CODE.get(dt)
    else:
        code = _NP_CODE.get(np.dtype(dt))
    if code is None:
        raise errors.ShapeError(f"unsupported element type {dt!r}; expected f32/f64/bf16/f16")
    return code



class _DevBuf:
    """``__cuda_array_interface__`` view of device memory owned by a communicator."""

    def __init__(self, ptr: int, nbytes: int, owner):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}
        self._owner = owner


def tensor_at(ptr: int, numel: int, dtype: torch.dtype, device: int, owner) -> torch.Tensor:
    """A torch tensor aliasing device memory at ``ptr`` (kept alive by ``owner``)."""
    nbytes = numel * torch.empty((), dtype=dtype).element_size()
    raw = torch.as_tensor(_DevBuf(ptr, nbytes, owner), device=f"cuda:{device}")
    return raw.view(dtype)


def to_host(t: torch.Tensor) -> torch.Tensor:
    """Device -> host through pinned memory on the current stream, then synchronise
    that stream only. A pageable device->host copy may wait on OTHER streams'
    kernels: in a loopback world that includes a peer kernel waiting for this
    rank's next launch (measured: W=8 stalled until the spin timeout; pinned
    copies never did). Pinned is also the fast path."""
    if not t.is_cuda:
        return t
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h


def exchange_blobs(blob: bytes, bootstrap=None) -> bytes:
    """Bootstrap exchange: every rank's export blob, concatenated in rank order,
    over ``bootstrap`` (default: the torch.distributed group). Never on a data path."""
    if bootstrap is None:
        from .bootstrap import DistBootstrap
        bootstrap = DistBootstrap()
    blobs = bootstrap.all_gather_object(bytes(blob))
    if any(not isinstance(b, bytes) or len(b) != len(blob) for b in blobs):
        raise errors.ProtocolError("ranks exported blobs of different sizes (mismatched library builds?)")
    return b"".join(blobs)


class _Base:
    """State shared by the multi-process and the virtual communicator."""

    _handle: ctypes.c_void_p | None = None

    def _init_common(self, pool_bytes: int, timeout_s: float):
        self._lib = _lib.load()
        self.pool_bytes = pool_bytes
        self._reserved = 0
        self._labels: set[str] = set()
        self.check_labels = False
        _lib.check(self._lib.rp_comm_set_timeout(self._handle, int(timeout_s * 1e9)), "set_timeout")
        info = [ctypes.c_int() for _ in range(4)]
        scratch = ctypes.c_size_t()
        _lib.check(self._lib.rp_comm_info(self._handle, *[ctypes.byref(i) for i in info], ctypes.byref(scratch)))
        self.num_sms = info[3].value

    # -- lifecycle -----------------------------------------------------------
    def close(self):
        if self._handle is not None:
            self._lib.rp_comm_destroy(self._handle)
            self._handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    # -- launch ordering -------------------------------------------------------
    _last_stream = None

    def _stream(self) -> int:
        """Stream handle for the next collective launch, ordered after this
        communicator's previous collective. Every kernel of a communicator shares
        its device-side sequencing state (tile counters, phase rows, epochs), so two
        of them must never run concurrently on one rank -- e.g. an overlapped bucket
        all-reduce on the side stream (overlap.py) and a BN exchange on the compute
        stream. When a launch comes from a different stream than the previous one,
        the new stream first waits for the old one; launches from one stream are
        ordered already. Ranks issue collectives in the same program order, so the
        device order pairs the same calls on every rank."""
        cur = torch.cuda.current_stream(self.device)
        last = self._last_stream
        # A stream being captured into a CUDA graph may not wait on work outside the
        # capture (cudaErrorStreamCaptureIsolation): inside a capture the graph's own
        # stream order sequences its collectives, and replaying a graph while an eager
        # collective of the same communicator runs on another stream is the caller's
        # ordering to provide (as for any two streams).
        if last is not None and last != cur and not torch.cuda.is_current_stream_capturing():
            cur.wait_stream(last)
        self._last_stream = cur
        return cur.cuda_stream

    def check(self):
        """Synchronise and raise ``CollectiveAbortedError`` if a kernel timed out or a
        peer aborted (include/rp.h rp_comm_check). Waits for this communicator's
        own launches (the streams it launched on), never for a device-wide sync
        that could wait on a loopback peer's kernel."""
        dev = torch.device(f"cuda:{self.device}")
        torch.cuda.current_stream(dev).synchronize()
        if self._last_stream is not None:
            self._last_stream.synchronize()
        _lib.check(self._lib.rp_comm_check(self._handle), "collective")

    def set_timeout(self, seconds: float):
        _lib.check(self._lib.rp_comm_set_timeout(self._handle, int(seconds * 1e9)), "set_timeout")

    def set_block_cap(self, blocks: int):
        """At most ``blocks`` blocks per rank for later collective launches (0: no
        cap). Set identically on every rank (include/rp.h rp_comm_set_block_cap)."""
        _lib.check(self._lib.rp_comm_set_block_cap(self._handle, int(blocks)), "set_block_cap")

    def algorithm_for(self, x: torch.Tensor, kind: str = "sum", out: torch.Tensor | None = None,
                      comm_dtype: torch.dtype | None = None, algo: str = "auto") -> str:
        """The kernel family all_reduce_tensor(x, kind, out, comm_dtype, algo) runs:
        "oneshot", "twoshot", "nvls" or (virtual replicas) "flat" (include/rp.h
        rp_all_reduce_algo). ``x``/``out``: this rank's tensors (a virtual
        communicator: replica 0's)."""
        out = x if out is None else out
        code = dtype_code(x.dtype)
        ccode = dtype_code(comm_dtype) if comm_dtype is not None else code
        chosen = ctypes.c_int(0)
        _lib.check(self._lib.rp_all_reduce_algo(self._handle, x.data_ptr(), out.data_ptr(), x.numel(), code, ccode,
                                                dtype_code(out.dtype), _op(kind), _algo(algo), ctypes.byref(chosen)),
                   "all_reduce_algo")
        return {1: "oneshot", 2: "twoshot", 3: "nvls", 5: "flat"}[chosen.value]

    def plan_for(self, x: torch.Tensor, kind: str = "sum", out: torch.Tensor | None = None,
                 comm_dtype: torch.dtype | None = None, algo: str = "auto") -> tuple:
        """(algorithm, push form, src pool offset or -1, dst pool offset or -1) that
        all_reduce_tensor(x, kind, out, comm_dtype, algo) would follow (include/rp.h
        rp_all_reduce_plan); every rank must agree on it. ``out=None``: a fresh
        output, as all_reduce_tensor allocates."""
        code = dtype_code(x.dtype)
        ccode = dtype_code(comm_dtype) if comm_dtype is not None else code
        optr, ocode = (0, code) if out is None else (out.data_ptr(), dtype_code(out.dtype))
        plan, _keep = _lib.i64_array([0, 0, 0, 0])
        _lib.check(self._lib.rp_all_reduce_plan(self._handle, x.data_ptr(), optr, x.numel(), code, ccode,
                                                ocode, _op(kind), _algo(algo), plan), "all_reduce_plan")
        return tuple(int(v) for v in _keep)

    # -- host buffers in, host buffer out ------------------------------------
    HOST_CHUNK_BYTES = 8 << 20
    HOST_RING = 3

    def all_reduce_host(self, host_in, kind: str = "sum", host_out: torch.Tensor | None = None,
                        chunk_bytes: int | None = None, nvls: bool = False) -> torch.Tensor:
        """Host tensors in, host tensor out, pipelined (the path a reference caller
        with numpy/CPU data takes, graph.py:571-574): the message is cut into chunks
        that flow through a ring of pool-resident device slots -- chunk i's
        host->device copies on one stream, its in-place all-reduce on the current
        stream, its device->host copy on a third -- so both PCIe directions and the
        exchange overlap instead of running back to back.

        ``host_in``: this rank's CPU tensor (multi-process), or one per replica
        (virtual). Pinned memory gives asynchronous copies. ``host_out`` receives the
        result (replica 0's for a virtual communicator: all replicas hold the same
        bits). Same arithmetic as all_reduce_tensor on the whole message (the folds
        are elementwise). ``nvls=True`` (multi-process, opt-in like Replicator's
        nvls_bytes): the device slots live in the NVLS region, so chunks of >= 512 KiB
        reduce in the switch at >= 4 ranks (not rank-ordered). Returns host_out after
        the copies completed."""
        ins = list(host_in) if isinstance(host_in, (list, tuple)) else [host_in]
        nrep = self.world if isinstance(self, VirtualCommunicator) else 1
        if nvls and not hasattr(self, "alloc_nvls"):
            raise errors.ConfigurationError("all_reduce_host(nvls=True) needs a multi-process communicator")
        if len(ins) != nrep:
            raise errors.ShapeError(f"expected {nrep} host tensors, got {len(ins)}")
        x0 = ins[0]
        for x in ins:
            if x.device.type != "cpu" or x.dtype != x0.dtype or x.numel() != x0.numel():
                raise errors.ProtocolError("all_reduce_host: CPU tensors of one dtype and size")
        ins = [x.reshape(-1) if x.is_contiguous() else x.contiguous().reshape(-1) for x in ins]
        n, dt = x0.numel(), x0.dtype
        if host_out is None:
            host_out = torch.empty(n, dtype=dt, pin_memory=ins[0].is_pinned())
        out = host_out.reshape(-1)
        esz = x0.element_size()
        ce = max(16 // esz, min(n, (chunk_bytes or self.HOST_CHUNK_BYTES) // esz)) if n else 1
        dev = torch.device(f"cuda:{self.device}")
        ring = self._host_ring(ce, dt, nvls)
        cur = torch.cuda.current_stream(dev)
        h2d, d2h = self._host_streams
        free = [None] * len(ring)
        starts = list(range(0, n, ce))
        for i, lo in enumerate(starts):
            hi = min(lo + ce, n)
            s = i % len(ring)
            bufs = ring[s]
            with torch.cuda.stream(h2d):
                if free[s] is not None:
                    h2d.wait_event(free[s])  # the slot's previous chunk has left for the host
                for r in range(nrep):
                    bufs[r][: hi - lo].copy_(ins[r][lo:hi], non_blocking=True)
            cur.wait_stream(h2d)
            views = [b[: hi - lo] for b in bufs]
            if nrep > 1:
                self.all_reduce(views, kind, outs=views)
            else:
                self.all_reduce_tensor(views[0], kind, out=views[0])
            d2h.wait_stream(cur)
            with torch.cuda.stream(d2h):
                out[lo:hi].copy_(views[0], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(d2h)
                free[s] = ev
        cur.wait_stream(d2h)
        cur.synchronize()
        return host_out

    def _host_ring(self, chunk_elems: int, dtype: torch.dtype, nvls: bool = False):
        """Pool-resident device slots for all_reduce_host, allocated once per (size,
        dtype, placement) -- symmetrically, since every rank makes the same calls."""
        key = (chunk_elems, dtype, nvls)
        rings = self.__dict__.setdefault("_rings", {})
        if key not in rings:
            slots = []
            for _ in range(self.HOST_RING):
                b = self.alloc_nvls(chunk_elems, dtype) if nvls else self.alloc(chunk_elems, dtype)
                slots.append(b if isinstance(b, list) else [b])
            rings[key] = slots
            dev = torch.device(f"cuda:{self.device}")
            self._host_streams = (torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev))
        return rings[key]

    # -- label protocol -----------------------------
    def new_generation(self):
        """Start a new generation (training step): labels may be reused again."""
        self._labels.clear()

    def _use_label(self, label):
        if not self.check_labels or label is None:
            return
        if label in self._labels:
            raise errors.ProtocolError(f"label {label!r} reused within one generation (SPEC.md:236)")
        self._labels.add(label)

    # -- pool ---------------------------------------------------------------
    def _pool_ptr(self, rank: int) -> int:
        base = ctypes.c_void_p()
        size = ctypes.c_size_t()
        _lib.check(self._lib.rp_comm_pool(self._handle, rank, ctypes.byref(base), ctypes.byref(size)))
        return base.value

    def _reserve(self, nbytes: int) -> int:
        """Symmetric bump allocation in the caller part of the pool; every rank must
        allocate the same sequence (it is SPMD code, so it does)."""
        off = (self._reserved + _ALIGN - 1) // _ALIGN * _ALIGN
        end = off + (nbytes + _ALIGN - 1) // _ALIGN * _ALIGN
        _lib.check(self._lib.rp_comm_reserve(self._handle, end), "pool reserve")
        self._reserved = end
        return off


class Communicator(_Base):
    """One rank of an NVLink data-parallel group (one process per GPU).

    Bootstrap over an initialised ``torch.distributed`` process group (any backend);
    only the IPC handle blobs travel over it.
    """

    def __init__(self, group=None, device: int | None = None, pool_bytes: int = DEFAULT_POOL_BYTES,
                 timeout_s: float = 20.0, bootstrap=None):
        """``bootstrap``: how the ranks find each other (bootstrap.py). Default: the
        initialised torch.distributed group ``group`` (one process per GPU), or a
        single rank when torch.distributed is not initialised. A loopback world's
        ``world.bootstrap(rank)`` puts every rank in this process on one device."""
        import torch.distributed as dist

        from .bootstrap import DistBootstrap

        lib = _lib.load()
        if bootstrap is None and dist.is_available() and dist.is_initialized():
            bootstrap = DistBootstrap(group)
        rank, world = (bootstrap.rank, bootstrap.world) if bootstrap is not None else (0, 1)
        if device is None:
            device = torch.cuda.current_device()
        self.rank, self.world, self.device = rank, world, int(device)
        self.bootstrap = bootstrap
        self.loopback = bool(getattr(bootstrap, "loopback", False))
        h = ctypes.c_void_p()
        _lib.check(lib.rp_comm_create(rank, world, self.device, pool_bytes, ctypes.byref(h)), "comm_create")
        self._handle = h
        if world > 1:
            if self.loopback:
                _lib.check(lib.rp_comm_set_loopback(h, 1), "comm_set_loopback")
            size = lib.rp_comm_export_size()
            buf = ctypes.create_string_buffer(size)
            n = ctypes.c_size_t(size)
            _lib.check(lib.rp_comm_export(h, buf, ctypes.byref(n)), "comm_export")
            joined = exchange_blobs(bytes(buf.raw[: n.value]), bootstrap)
            _lib.check(lib.rp_comm_import(h, joined, len(joined)), "comm_import")
        self._init_common(pool_bytes, timeout_s)

    @property
    def num_replicas(self) -> int:
        return self.world

    _LINK_NAMES = {0: "self", 1: "nvlink", 2: "pcie", 3: "none", 4: "unknown", 5: "same_device", 6: "loopback"}

    def topology(self) -> dict:
        """What rp_comm_import discovered (include/rp.h rp_comm_topology): the link
        kind from this rank to every rank and every rank's active NVLink links."""
        links = (ctypes.c_int * self.world)()
        nvl = (ctypes.c_int * self.world)()
        _lib.check(self._lib.rp_comm_topology(self._handle, links, nvl), "comm_topology")
        return {"rank": self.rank, "links": [self._LINK_NAMES.get(v, str(v)) for v in links],
                "nvlinks": list(nvl)}

    # -- zero-copy buffers --------------------------------------------------
    def alloc(self, numel: int, dtype: torch.dtype) -> torch.Tensor:
        """Tensor inside this rank's registered pool (exchanged without staging)."""
        esz = torch.empty((), dtype=dtype).element_size()
        off = self._reserve(numel * esz)
        return tensor_at(self._pool_ptr(self.rank) + off, numel, dtype, self.device, self)

    # -- user-buffer registration (include/rp.h rp_register_*) -----------------
    def register(self, t: torch.Tensor) -> "Registration":
        """Collective (every rank, same order, same size): map this rank's ``t`` on
        every peer once, so that in-place all-reduces of ``t`` -- or of a view at the
        same offset inside it on every rank -- run the zero-copy pull two-shot like
        pool buckets (no staging). Keep ``t`` alive until ``unregister``. Needs
        IPC-shareable memory (PyTorch's default caching allocator; a loopback world
        shares plain pointers)."""
        if not t.is_cuda or t.device.index != self.device or not _is_dense(t):
            raise errors.ShapeError("register: a dense CUDA tensor on this communicator's device")
        size = self._lib.rp_register_export_size()
        buf = ctypes.create_string_buffer(size)
        n = ctypes.c_size_t(size)
        _lib.check(self._lib.rp_register_export(self._handle, t.data_ptr(), t.numel() * t.element_size(), buf,
                                                ctypes.byref(n)), "register")
        joined = exchange_blobs(bytes(buf.raw[: n.value]), self.bootstrap) if self.world > 1 else bytes(buf.raw[: n.value])
        reg = ctypes.c_int(-1)
        _lib.check(self._lib.rp_register_import(self._handle, joined, len(joined), ctypes.byref(reg)), "register")
        return Registration(self, reg.value, t)

    def unregister(self, reg: "Registration") -> None:
        """Collective: release a registration (peers' mappings closed when unused)."""
        _lib.check(self._lib.rp_unregister(self._handle, reg.index), "unregister")
        reg.index = -1

    # -- NVLS (NVLink SHARP) region -------------------------------------------
    def enable_nvls(self, nbytes: int, group=None) -> None:
        """Bind ``nbytes`` of this rank's memory to one multicast object spanning all
        ranks (include/rp.h rp_nvls_*). Collective over the bootstrap; the multicast
        fd travels from rank 0 over a Unix socket, its name over the bootstrap."""
        if self.world < 2:
            raise errors.ConfigurationError("NVLS needs at least two ranks")
        if self.loopback:
            raise errors.ConfigurationError("NVLS needs one process per GPU (a multicast object spans distinct "
                                            "devices; a loopback world has one)")
        name = ctypes.create_string_buffer(128)
        _lib.check(self._lib.rp_nvls_create(self._handle, nbytes, name, 128), "nvls_create")
        root_name = self.bootstrap.broadcast_object(name.value if self.rank == 0 else None, src=0)
        if self.rank == 0:
            _lib.check(self._lib.rp_nvls_serve(self._handle), "nvls_serve")
        else:
            _lib.check(self._lib.rp_nvls_join(self._handle, root_name), "nvls_join")
        _lib.check(self._lib.rp_nvls_add(self._handle), "nvls_add")
        self.bootstrap.barrier()
        _lib.check(self._lib.rp_nvls_bind(self._handle), "nvls_bind")
        self.bootstrap.barrier()
        base = ctypes.c_void_p()
        size = ctypes.c_size_t()
        _lib.check(self._lib.rp_nvls_pool(self._handle, ctypes.byref(base), ctypes.byref(size)), "nvls_pool")
        self._nvls_base, self._nvls_size, self._nvls_used = base.value, size.value, 0

    @property
    def nvls_free(self) -> int:
        """Bytes still unallocated in the NVLS region (0 without one)."""
        if not hasattr(self, "_nvls_base"):
            return 0
        return max(0, self._nvls_size - (self._nvls_used + _ALIGN - 1) // _ALIGN * _ALIGN)

    def alloc_nvls(self, numel: int, dtype: torch.dtype) -> torch.Tensor:
        """Tensor inside the NVLS region (symmetric offsets: allocate in the same order
        on every rank). In-place ``all_reduce_tensor(t, kind, out=t)`` reduces it in
        the switch (algo "auto" at >= 4 ranks and >= 512 KiB, or algo="nvls")."""
        if not hasattr(self, "_nvls_base"):
            raise errors.ConfigurationError("call enable_nvls() first")
        esz = torch.empty((), dtype=dtype).element_size()
        off = (self._nvls_used + _ALIGN - 1) // _ALIGN * _ALIGN
        if off + numel * esz > self._nvls_size:
            raise errors.ShapeError("NVLS region exhausted")
        self._nvls_used = off + numel * esz
        return tensor_at(self._nvls_base + off, numel, dtype, self.device, self)

    # -- torch-tensor collectives ------------------------------------------
    def all_reduce_tensor(self, x: torch.Tensor, kind: str = "sum", out: torch.Tensor | None = None,
                          comm_dtype: torch.dtype | None = None, algo: str = "auto") -> torch.Tensor:
        """out = kind-fold of x over ranks (ascending rank order, graph.py:514-533).

        kind: "sum" | "mean" (sum, then /N) | "max" | "premean" (all_sum(x/N), the
        wrap_optimizer composition of PAPER.md:196-206). ``comm_dtype`` fuses a cast
        (e.g. f32 tensors exchanged as bf16)."""
        xd = _dense_cuda(x, self.device)
        if out is None:
            out = torch.empty_like(xd)
        # element-wise: any dense layout works as long as out has the same strides
        od = out if (_is_dense(out) and out.stride() == xd.stride()) else torch.empty_like(xd, dtype=out.dtype)
        code = dtype_code(xd.dtype)
        ccode = dtype_code(comm_dtype) if comm_dtype is not None else code
        _lib.check(self._lib.rp_all_reduce(self._handle, xd.data_ptr(), od.data_ptr(), xd.numel(), code, ccode,
                                           dtype_code(od.dtype), _op(kind), _algo(algo), self._stream()),
                   "all_reduce")
        if od is not out:
            out.copy_(od)
        return out

    def all_gather_ragged(self, x: torch.Tensor) -> list[torch.Tensor]:
        """shapes may differ across ranks in the leading dimension
        only. Two exchanges through the all_gather kernel: (leading dim, digest of the
        trailing shape and dtype), then every rank's rows padded to the longest;
        returns [t_0, ..., t_{N-1}] in rank order (views of one gathered buffer)."""
        x = _contig_cuda(x, self.device)
        if x.dim() == 0:
            x = x.reshape(1)
        tail = hashlib.sha256(repr((tuple(x.shape[1:]), str(x.dtype))).encode()).digest()[:8]
        meta = torch.tensor([x.shape[0], int.from_bytes(tail, "little", signed=True)], dtype=torch.int64)
        g = to_host(self.all_gather_tensor(meta.to(x.device)))
        for r in range(self.world):
            if int(g[r, 1]) != int(g[self.rank, 1]):
                raise errors.ProtocolError(f"all_gather: rank {r} and rank {self.rank} differ beyond the leading "
                                           f"dimension (local {tuple(x.shape)}, {x.dtype})")
        lens = [int(g[r, 0]) for r in range(self.world)]
        m = max(lens)
        if m == x.shape[0]:
            xp = x
        else:
            xp = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
            xp[: x.shape[0]] = x
        if m == 0:
            return [xp[:0] for _ in range(self.world)]
        out = self.all_gather_tensor(xp)
        return [out[r, : lens[r]] for r in range(self.world)]

    def all_gather_tensor(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """out[r] = x of rank r; out has shape (world,) + x.shape."""
        x = _contig_cuda(x, self.device)
        if out is None:
            out = torch.empty((self.world,) + tuple(x.shape), dtype=x.dtype, device=x.device)
        _lib.check(self._lib.rp_all_gather(self._handle, x.data_ptr(), out.data_ptr(),
                                           x.numel() * x.element_size(), self._stream()), "all_gather")
        return out

    def broadcast_tensor(self, x: torch.Tensor, root: int = 0, out: torch.Tensor | None = None,
                         algo: str = "auto") -> torch.Tensor:
        """Every rank receives root's x (in place when out is None)."""
        xd = _dense_cuda(x, self.device)
        if out is None:
            out = x
        od = out if (_is_dense(out) and out.stride() == xd.stride()) else torch.empty_like(xd)
        _lib.check(self._lib.rp_broadcast(self._handle, xd.data_ptr(), od.data_ptr(),
                                          xd.numel() * xd.element_size(), root, _algo(algo), self._stream()),
                   "broadcast")
        if od is not out:  # e.g. an in-place broadcast of a strided view: write back
            out.copy_(od)
        return out

    # -- the reference duck type (graph.py:565-583) -------------------------
    def all_reduce(self, local, kind="sum", label=None, **kw):
        self._use_label(label)
        if isinstance(local, torch.Tensor):
            return self.all_reduce_tensor(local, kind, **kw)
        arr, wrap = _host_in(local)
        if hasattr(local, "np") and hasattr(type(local), "wrap"):
            self._tensor_cls = type(local)
        x = torch.from_numpy(np.ascontiguousarray(arr)).to(f"cuda:{self.device}")
        y = self.all_reduce_tensor(x, kind)
        return wrap(to_host(y).numpy())

    def all_gather(self, local, label=None):
        """[t_0, ..., t_{N-1}] in rank order; leading dimensions may differ across
        ranks, scalars stay scalars."""
        self._use_label(label)
        if isinstance(local, torch.Tensor):
            if local.dim() == 0:
                g = self.all_gather_tensor(local.reshape(1))
                return [g[r, 0] for r in range(self.world)]
            return self.all_gather_ragged(local)
        arr, wrap = _host_in(local)
        x = torch.from_numpy(np.ascontiguousarray(arr)).to(f"cuda:{self.device}")
        if x.dim() == 0:
            g = to_host(self.all_gather_tensor(x.reshape(1))).numpy()
            return [wrap(g[r, 0]) for r in range(self.world)]
        return [wrap(to_host(t).numpy()) for t in self.all_gather_ragged(x)]

    def broadcast(self, root_value, label=None, shape=None, dtype=None, root: int = 0):
        """Reference form (graph.py:580-582): root passes its value, others pass None
        plus ``shape``/``dtype``; every rank returns root's value bit-exactly."""
        self._use_label(label)
        if isinstance(root_value, torch.Tensor) or (root_value is None and isinstance(dtype, torch.dtype)):
            x = (root_value.clone() if root_value is not None
                 else torch.empty(tuple(shape), dtype=dtype, device=f"cuda:{self.device}"))
            return self.broadcast_tensor(x, root)
        if root_value is None:
            # non-root ranks hold no value: return the reference's Tensor type if we
            # have seen it (the seam calls ``.np`` on the result, graph.py:582), else
            # a read-only HostTensor with the same interface
            np_dt = {"f32": np.float32, "f64": np.float64}.get(dtype, dtype)
            arr = np.zeros(tuple(shape), dtype=np_dt)
            wrap = _wrapper_for(None, getattr(self, "_tensor_cls", None))
        else:
            arr, wrap = _host_in(root_value)
            if hasattr(root_value, "np") and hasattr(type(root_value), "wrap"):
                self._tensor_cls = type(root_value)
        x = torch.from_numpy(np.ascontiguousarray(arr)).to(f"cuda:{self.device}")
        y = self.broadcast_tensor(x, root)
        return wrap(to_host(y).numpy())

    # -- protocol agreement (debug): every rank must issue the same collective
    def verify(self, label: str, kind: str, shape, dtype, position=None) -> None:
        """All ranks exchange a digest of (position, label, kind, shape, dtype)
        through this communicator's own all_gather and raise ProtocolError naming
        the disagreeing ranks and what each issued.
        ``position`` is the call's (generation, index): a different ORDER of the
        same calls is caught too."""
        desc = repr((position, label, kind, tuple(shape), str(dtype)))
        h = hashlib.sha256(desc.encode()).digest()[:16]
        t = torch.frombuffer(bytearray(h), dtype=torch.uint8).to(f"cuda:{self.device}")
        g = to_host(self.all_gather_tensor(t))
        bad = [r for r in range(self.world) if not torch.equal(g[r], g[self.rank])]
        if bad:
            # second exchange (every rank takes this branch: some rank disagrees with
            # each of them): the descriptions themselves, for the message
            raw = desc.encode()[:240]
            buf = torch.zeros(256, dtype=torch.uint8)
            buf[: len(raw)] = torch.frombuffer(bytearray(raw), dtype=torch.uint8)
            d = to_host(self.all_gather_tensor(buf.to(f"cuda:{self.device}")))
            other = bytes(d[bad[0]].numpy()).rstrip(b"\0").decode(errors="replace")
            raise errors.ProtocolError(f"collective protocol mismatch: rank {self.rank} issued {desc}, "
                                       f"rank {bad[0]} issued {other} (ranks {bad} disagree with rank {self.rank})")


class Registration:
    """A buffer registered with every peer (Communicator.register); keeps the tensor
    alive while registered."""

    def __init__(self, comm, index: int, tensor: torch.Tensor):
        self.comm, self.index, self.tensor = comm, index, tensor

    def __repr__(self):
        return f"Registration(index={self.index}, numel={self.tensor.numel()}, dtype={self.tensor.dtype})"


class VirtualCommunicator(_Base):
    """R replicas resident on one GPU (in-process MultiDevice replication).

    Collectives take and return lists of R tensors (replica order = rank order),
    run as one cooperative kernel; the fold is the reference's stitched
    ``nary_*`` (graph.py:506-533), ``concat``/``pack`` (:447-449, :535-536) and
    ``pick0`` (:538-540).
    """

    def __init__(self, num_replicas: int, device: int | None = None, pool_bytes: int = DEFAULT_POOL_BYTES,
                 timeout_s: float = 20.0):
        lib = _lib.load()
        if device is None:
            device = torch.cuda.current_device()
        self.world, self.device, self.rank = int(num_replicas), int(device), 0
        h = ctypes.c_void_p()
        _lib.check(lib.rp_comm_create_virtual(self.world, self.device, pool_bytes, ctypes.byref(h)),
                   "comm_create_virtual")
        self._handle = h
        self._init_common(pool_bytes, timeout_s)

    @property
    def num_replicas(self) -> int:
        return self.world

    def alloc(self, numel: int, dtype: torch.dtype) -> list[torch.Tensor]:
        esz = torch.empty((), dtype=dtype).element_size()
        off = self._reserve(numel * esz)
        return [tensor_at(self._pool_ptr(r) + off, numel, dtype, self.device, self) for r in range(self.world)]

    def _check_list(self, xs):
        if len(xs) != self.world:
            raise errors.ShapeError(f"expected {self.world} replica tensors, got {len(xs)}")
        xs = [_contig_cuda(x, self.device) for x in xs]
        s0, d0 = xs[0].shape, xs[0].dtype
        for r, x in enumerate(xs):
            if x.shape != s0 or x.dtype != d0:
                raise errors.ProtocolError(f"replica {r} disagrees: {tuple(x.shape)}/{x.dtype} vs {tuple(s0)}/{d0}")
        return xs

    def all_reduce(self, xs, kind="sum", outs=None, comm_dtype=None, algo="auto", label=None):
        self._use_label(label)
        xs = self._check_list(xs)
        if outs is None:
            outs = [torch.empty_like(x) for x in xs]
        _check_outs(outs, xs)
        code = dtype_code(xs[0].dtype)
        ccode = dtype_code(comm_dtype) if comm_dtype is not None else code
        sp, _k1 = _lib.ptr_array([x.data_ptr() for x in xs])
        dp, _k2 = _lib.ptr_array([o.data_ptr() for o in outs])
        _lib.check(self._lib.rp_all_reduce_v(self._handle, sp, dp, xs[0].numel(), code, ccode,
                                             dtype_code(outs[0].dtype), _op(kind), _algo(algo),
                                             self._stream()), "all_reduce")
        return outs

    def all_gather(self, xs, outs=None, label=None):
        """outs[r] has shape (R,) + x.shape: every replica's x in rank order."""
        self._use_label(label)
        xs = self._check_list(xs)
        if outs is None:
            outs = [torch.empty((self.world,) + tuple(xs[0].shape), dtype=xs[0].dtype, device=xs[0].device)
                    for _ in xs]
        sp, _k1 = _lib.ptr_array([x.data_ptr() for x in xs])
        dp, _k2 = _lib.ptr_array([o.data_ptr() for o in outs])
        _lib.check(self._lib.rp_all_gather_v(self._handle, sp, dp, xs[0].numel() * xs[0].element_size(),
                                             self._stream()), "all_gather")
        return outs

    def all_gather_ragged(self, xs):
        """leading dimensions may differ across replicas. Returns, for
        every replica, the list [x_0, ..., x_{R-1}] (views of its gathered buffer)."""
        if len(xs) != self.world:
            raise errors.ShapeError(f"expected {self.world} replica tensors, got {len(xs)}")
        xs = [_contig_cuda(x, self.device) for x in xs]
        xs = [x.reshape(1) if x.dim() == 0 else x for x in xs]
        tail = (tuple(xs[0].shape[1:]), xs[0].dtype)
        for r, x in enumerate(xs):
            if (tuple(x.shape[1:]), x.dtype) != tail:
                raise errors.ProtocolError(f"all_gather: replica {r} differs beyond the leading dimension: "
                                           f"{tuple(x.shape)}/{x.dtype} vs {tuple(xs[0].shape)}/{xs[0].dtype}")
        lens = [x.shape[0] for x in xs]
        m = max(lens)
        if m == 0:
            return [[x[:0] for x in xs] for _ in xs]
        padded = []
        for x in xs:
            if x.shape[0] == m:
                padded.append(x)
            else:
                p = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
                p[: x.shape[0]] = x
                padded.append(p)
        outs = self.all_gather(padded)
        return [[o[q, : lens[q]] for q in range(self.world)] for o in outs]

    def broadcast(self, xs, root=0, outs=None, algo="auto", label=None):
        self._use_label(label)
        xs = self._check_list(xs)
        if outs is None:
            outs = [torch.empty_like(x) for x in xs]
        _check_outs(outs, xs)
        sp, _k1 = _lib.ptr_array([x.data_ptr() for x in xs])
        dp, _k2 = _lib.ptr_array([o.data_ptr() for o in outs])
        _lib.check(self._lib.rp_broadcast_v(self._handle, sp, dp, xs[0].numel() * xs[0].element_size(), root,
                                            _algo(algo), self._stream()), "broadcast")
        return outs


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------

def _op(kind: str) -> int:
    try:
        return _lib.OPS[kind]
    except KeyError:
        raise errors.ShapeError(f"unknown reduction kind {kind!r}; expected sum/mean/max/premean") from None


def _algo(algo) -> int:
    if isinstance(algo, int):
        return algo
    try:
        return _lib.ALGOS[algo]
    except KeyError:
        raise errors.ShapeError(f"unknown algorithm {algo!r}") from None


def _check_outs(outs, xs):
    if len(outs) != len(xs):
        raise errors.ShapeError(f"expected {len(xs)} output tensors, got {len(outs)}")
    for o, x in zip(outs, xs):
        if o.numel() != x.numel() or not (o.is_contiguous() or (_is_dense(o) and o.stride() == x.stride())):
            raise errors.ShapeError("virtual collective outputs must be dense with the inputs' layout")


def _is_dense(x: torch.Tensor) -> bool:
    """Non-overlapping and dense: the storage span is exactly numel elements (any
    dimension order), so element-wise collectives can treat it as a flat array."""
    if x.is_contiguous():
        return True
    if x.dim() == 4 and x.is_contiguous(memory_format=torch.channels_last):
        return True
    if x.dim() == 5 and x.is_contiguous(memory_format=torch.channels_last_3d):
        return True
    return False


def _dense_cuda(x: torch.Tensor, device: int) -> torch.Tensor:
    """x itself when dense (contiguous or channels_last), else a contiguous copy.
    Element-wise collectives run on the storage directly, so channels_last
    parameters are reduced/broadcast in place."""
    if not x.is_cuda:
        raise errors.ShapeError("collective inputs must be CUDA tensors (host values go through the "
                                "reference seam methods, which copy them in)")
    if x.device.index != device:
        raise errors.ShapeError(f"tensor on cuda:{x.device.index}, communicator on cuda:{device}")
    return x if _is_dense(x) else x.contiguous()


def _contig_cuda(x: torch.Tensor, device: int) -> torch.Tensor:
    if not x.is_cuda:
        raise errors.ShapeError("collective inputs must be CUDA tensors (host values go through the "
                                "reference seam methods, which copy them in)")
    if x.device.index != device:
        raise errors.ShapeError(f"tensor on cuda:{x.device.index}, communicator on cuda:{device}")
    return x if x.is_contiguous() else x.contiguous()


class HostTensor:
    """Read-only host result with the reference Tensor's interface (tensor.py:32-98:
    ``.np``, ``.shape``, ``.dtype`` in {"f32","f64"}, ``wrap``), returned to a non-root
    broadcast caller that passed no value to infer its Tensor type from."""

    __slots__ = ("_np",)

    def __init__(self, arr):
        arr = np.ascontiguousarray(arr)
        arr.setflags(write=False)
        self._np = arr

    @staticmethod
    def wrap(arr):
        return HostTensor(arr)

    @property
    def np(self):
        return self._np

    @property
    def shape(self):
        return self._np.shape

    @property
    def dtype(self):
        return {np.dtype(np.float32): "f32", np.dtype(np.float64): "f64"}[self._np.dtype]

    @property
    def size(self):
        return self._np.size

    def tolist(self):
        return self._np.tolist()

    def tobytes(self):
        return self._np.tobytes()

    def item(self):
        return float(self._np.item())


def _wrapper_for(local, cls=None):
    """Return a function turning a numpy result back into the caller's value kind:
    the reference Tensor class when given one (``Tensor.wrap``, tensor.py:52-62),
    a numpy array for numpy input, and ``cls`` (or HostTensor) when there is no input."""
    if local is not None and hasattr(local, "np") and hasattr(type(local), "wrap"):
        cls = type(local)
    elif local is None:
        cls = cls or HostTensor
    else:
        return lambda a: np.ascontiguousarray(a)

    def wrap(a):
        a = np.ascontiguousarray(a)
        a.setflags(write=False)
        return cls.wrap(a)
    return wrap


def _host_in(local):
    arr = local.np if hasattr(local, "np") else np.asarray(local)
    if arr.dtype not in (np.float32, np.float64):
        raise errors.ShapeError(f"unsupported element type {arr.dtype}; only f32/f64 tensors exist")
    return arr, _wrapper_for(local)
