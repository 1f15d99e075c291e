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
    def __init__(self, comm, params_per_replica, grad_dtype, comm_dtype, allow_nvls: bool = True,
                 match_param_layout: bool = False):
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
        esz = torch.empty((), dtype=comm_dtype).element_size()
        self.match_param_layout = match_param_layout
        if allow_nvls and isinstance(comm, Communicator) and comm.nvls_free >= o * esz + 256:
            buf = comm.alloc_nvls(o, comm_dtype)  # reduced inside the NVSwitch (rp.h RP_ALGO_NVLS)
        else:
            buf = comm.alloc(o, comm_dtype)
        self.flat = buf if isinstance(buf, list) else [buf]
        self._counts_c = _lib.i64_array(self.counts)
        self._offs_c = _lib.i64_array(self.offs)

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

    def reduce(self, kind: str, grads=None):
        """pack -> in-place premean/sum fold -> unpack, all on the current stream."""
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
                 bucket_bytes: int | None = None):
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
                    self.buckets.append(_Bucket(comm, [[lst[j] for j in cur] for lst in lists], dt, cdt))
                    cur, cur_bytes = [], 0
                cur.append(i)
                cur_bytes += nb
            if cur:
                self.buckets.append(_Bucket(comm, [[lst[j] for j in cur] for lst in lists], dt, cdt))

    @property
    def nbytes(self) -> int:
        return sum(b.numel * b.flat[0].element_size() for b in self.buckets)

    def reduce(self, kind: str = "premean"):
        for b in self.buckets:
            b.reduce(kind)
