"""Fusion buffers for the wrapped optimizer's gradient all-reduce.

The reference averages each gradient with its own collective
(``all_sum(grad / num_repls, label)`` per (grad, var), PAPER.md:196-206,
SPEC.md:370-378). Here all gradients of one dtype are packed into a bucket that
lives in the communicator's registered pool (one multi-tensor K6 launch, with the
optional f32->bf16 cast fused in), reduced in place zero-copy with the
``premean`` fold -- the same divide-then-sum, ascending-rank arithmetic
 -- and unpacked back into ``param.grad`` (one K6 launch).
Bit-for-bit the result equals the reference's per-gradient ``all_sum(g/R)``:
packing is a copy and the fold is elementwise. When the communicator has an NVLS
region with room (Replicator(nvls_bytes=...)), buckets are placed there instead and
reduced inside the NVSwitch at >= 4 ranks: faster, but summed in switch order
(within the north-star's 1e-6 relative tolerance rather than bit-exact).
"""

from __future__ import annotations

import torch

from . import _lib, errors
from .comm import Communicator, VirtualCommunicator, _is_dense, dtype_code

_ALIGN_ELEMS = 64  # keep every tensor's slot 128-byte aligned for 16-bit types


class _Bucket:
    """``views=True`` (gradients as bucket views): the bucket holds the gradients
    themselves in their own dtype, and every ``param.grad`` is a view of its slot
    (same strides as the parameter). Autograd accumulates in place into the pool,
    so the exchange needs no pack and no unpack: ONE in-place all-reduce per bucket,
    with the exchange cast (e.g. f32 gradients sent as bf16) fused into the kernel.
    The arithmetic is the same as pack (RNE cast) -> fold -> unpack (exact widening),
    so results are bit-identical to the packed form. A gradient that stopped being
    a view (``zero_grad(set_to_none=True)``, a user assignment) is copied back into
    its slot and re-attached before the exchange."""

    def __init__(self, comm, params_per_replica, grad_dtype, comm_dtype, allow_nvls: bool = True,
                 match_param_layout: bool = False, views: bool = False):
        self.comm = comm
        self.grad_dtype = grad_dtype
        self.comm_dtype = comm_dtype
        self.params = params_per_replica  # [replica][k] -> Parameter
        self.counts = [p.numel() for p in params_per_replica[0]]
        offs, o = [], 0
        for n in self.counts:
            offs.append(o)
            o += (n + _ALIGN_ELEMS - 1) // _ALIGN_ELEMS * _ALIGN_ELEMS
        self.offs = offs
        self.numel = o
        self.views = bool(views) and all(_is_dense(p) for p in params_per_replica[0])
        flat_dtype = grad_dtype if self.views else comm_dtype
        esz = torch.empty((), dtype=flat_dtype).element_size()
        self.match_param_layout = match_param_layout
        # the switch reduces in place without a cast (rp.h RP_ALGO_NVLS)
        nvls_ok = flat_dtype == comm_dtype
        if allow_nvls and nvls_ok and isinstance(comm, Communicator) and comm.nvls_free >= o * esz + 256:
            buf = comm.alloc_nvls(o, flat_dtype)  # reduced inside the NVSwitch
        else:
            buf = comm.alloc(o, flat_dtype)
        self.flat = buf if isinstance(buf, list) else [buf]
        self._counts_c = _lib.i64_array(self.counts)
        self._offs_c = _lib.i64_array(self.offs)
        if self.views:
            self.slots = [[flat[off:off + n].as_strided(p.shape, p.stride())
                           for p, off, n in zip(self.params[r], self.offs, self.counts)]
                          for r, flat in enumerate(self.flat)]
            for flat in self.flat:
                flat.zero_()
            with torch.no_grad():
                self.attach()

    def attach(self):
        """(views) Make every ``param.grad`` the view of its bucket slot, copying a
        detached gradient back in (a missing one is zero). Returns the number of
        gradients that had to be re-attached (0 in the steady state)."""
        moved = 0
        stream = torch.cuda.current_stream(self.flat[0].device)
        for r, plist in enumerate(self.params):
            same, ks = [], []  # same-layout gradients: one multi-tensor copy (K6 pack) into their slots
            for k, (p, v) in enumerate(zip(plist, self.slots[r])):
                g = p.grad
                if g is not None and g.data_ptr() == v.data_ptr() and g.stride() == v.stride():
                    continue
                if g is None:
                    v.zero_()
                elif g.dtype == v.dtype and g.stride() == v.stride() and _is_dense(g):
                    same.append(g)
                    ks.append(k)
                else:
                    v.copy_(g)
                if g is not None:
                    g.record_stream(stream)
                p.grad = v
                moved += 1
            if same:
                lib = _lib.load()
                code = dtype_code(self.grad_dtype)
                pp, _keep = _lib.ptr_array([g.data_ptr() for g in same])
                cnt, _k1 = _lib.i64_array([self.counts[k] for k in ks])
                off, _k2 = _lib.i64_array([self.offs[k] for k in ks])
                _lib.check(lib.rp_pack(self.flat[r].data_ptr(), code, pp, cnt, off, len(same), code,
                                       stream.cuda_stream), "pack(attach)")
        return moved

    def _grads(self, r):
        """The replica's gradients as dense storages. Pack/unpack copy storage order,
        which is identical on every replica, so any dense layout (e.g. channels_last,
        matching the parameter) is exchanged as is; a gradient is only re-laid out
        (like its parameter, so the optimizer keeps its foreach fast path) when it
        is not dense."""
        out = []
        for p in self.params[r]:
            if p.grad is None:
                p.grad = torch.zeros_like(p)
            g = p.grad
            if not _is_dense(g) or (self.match_param_layout and g.stride() != p.stride()):
                d = torch.empty_like(p)
                d.copy_(g)
                p.grad = g = d
            out.append(g)
        return out

    def pack(self, grads=None):
        """Every replica's gradients -> its flat bucket (one multi-tensor launch each,
        with the exchange cast fused). Returns the gradient lists (for unpack).
        ``grads``: the lists from ``_grads`` when the caller fetched them already
        (overlap.py fetches them on the compute stream, packs on the comm stream)."""
        lib = _lib.load()
        stream = torch.cuda.current_stream(self.flat[0].device).cuda_stream
        gcode, ccode = dtype_code(self.grad_dtype), dtype_code(self.comm_dtype)
        if grads is None:
            grads = [self._grads(r) for r in range(len(self.params))]
        for r, flat in enumerate(self.flat):
            pp, k = _lib.ptr_array([g.data_ptr() for g in grads[r]])
            _lib.check(lib.rp_pack(flat.data_ptr(), ccode, pp, self._counts_c[0], self._offs_c[0], len(grads[r]),
                                   gcode, stream), "pack")
        return grads

    def is_attached(self, r: int, k: int) -> bool:
        """(views) replica r's k-th gradient is its bucket slot."""
        g, v = self.params[r][k].grad, self.slots[r][k]
        return g is not None and g.data_ptr() == v.data_ptr() and g.stride() == v.stride()

    def reduce(self, kind: str, grads=None, attached: bool = False):
        """pack -> in-place premean/sum fold -> unpack, all on the current stream
        (views: attach -- skipped when the caller checked every gradient already --
        then the in-place fold with the cast fused)."""
        if self.views:
            if not attached:
                with torch.no_grad():
                    self.attach()
            cdt = None if self.comm_dtype == self.grad_dtype else self.comm_dtype
            if isinstance(self.comm, VirtualCommunicator):
                self.comm.all_reduce(self.flat, kind, outs=self.flat, comm_dtype=cdt)
            else:
                self.comm.all_reduce_tensor(self.flat[0], kind, out=self.flat[0], comm_dtype=cdt)
            return
        lib = _lib.load()
        stream = torch.cuda.current_stream(self.flat[0].device).cuda_stream
        gcode, ccode = dtype_code(self.grad_dtype), dtype_code(self.comm_dtype)
        grads = self.pack(grads)
        keep = []
        if isinstance(self.comm, VirtualCommunicator):
            self.comm.all_reduce(self.flat, kind, outs=self.flat)
        else:
            self.comm.all_reduce_tensor(self.flat[0], kind, out=self.flat[0])
        for r, flat in enumerate(self.flat):
            pp, k = _lib.ptr_array([g.data_ptr() for g in grads[r]])
            keep.append(k)
            _lib.check(lib.rp_unpack(flat.data_ptr(), ccode, pp, self._counts_c[0], self._offs_c[0], len(grads[r]),
                                     gcode, stream), "unpack")


class GradBuckets:
    """Buckets of same-dtype gradients in the registered pool.

    ``params_per_replica``: one parameter list per local replica (a single list for
    a multi-process communicator), identically ordered and shaped.
    """

    def __init__(self, comm, params_per_replica, comm_dtype: torch.dtype | None = None,
                 bucket_bytes: int | None = None, views: bool = False):
        if isinstance(comm, Communicator) and len(params_per_replica) != 1:
            raise errors.ShapeError("a multi-process communicator reduces one replica per process")
        if isinstance(comm, VirtualCommunicator) and len(params_per_replica) != comm.world:
            raise errors.ShapeError(f"expected {comm.world} replica parameter lists")
        base = [p for p in params_per_replica[0] if p.requires_grad]
        for r, plist in enumerate(params_per_replica):
            plist = [p for p in plist if p.requires_grad]
            if [tuple(p.shape) for p in plist] != [tuple(p.shape) for p in base]:
                raise errors.ProtocolError(f"replica {r}'s parameters differ from replica 0's")
        self.buckets: list[_Bucket] = []
        by_dtype: dict[torch.dtype, list[int]] = {}
        for i, p in enumerate(base):
            by_dtype.setdefault(p.dtype, []).append(i)
        lists = [[p for p in plist if p.requires_grad] for plist in params_per_replica]
        for dt, idx in by_dtype.items():
            cdt = comm_dtype if (comm_dtype is not None and dt == torch.float32) else dt
            esz = torch.empty((), dtype=cdt).element_size()
            limit = bucket_bytes or (1 << 62)
            cur, cur_bytes = [], 0
            for i in idx:
                nb = base[i].numel() * esz
                if cur and cur_bytes + nb > limit:
                    self.buckets.append(_Bucket(comm, [[lst[j] for j in cur] for lst in lists], dt, cdt,
                                                views=views))
                    cur, cur_bytes = [], 0
                cur.append(i)
                cur_bytes += nb
            if cur:
                self.buckets.append(_Bucket(comm, [[lst[j] for j in cur] for lst in lists], dt, cdt, views=views))

    @property
    def nbytes(self) -> int:
        return sum(b.numel * b.flat[0].element_size() for b in self.buckets)

    def reduce(self, kind: str = "premean"):
        for b in self.buckets:
            b.reduce(kind)
