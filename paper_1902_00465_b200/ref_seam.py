"""Seam 2: GPU-backed kinds for the reference's op registry (``graph.py:123-135``).

The reference's absent stitcher rewrites every
``collective_placeholder`` of an in-process (MultiDevice) replicated graph into one
node per replica site over ALL replicas' inputs: ``nary_sum / nary_mean / nary_max``
(graph.py:514-533), ``concat`` / ``pack`` for gathers (:424-449, :535-536) and
``pick0`` for broadcasts (:538-540). ``register(G)`` adds drop-in kinds with the same
operands, shapes and bits, computed by this repo's sm_100a kernels on a
``VirtualCommunicator`` (all replicas resident on one GPU, one cooperative launch):

=============  ==========================================  =====================
kind           replaces                                    kernel
=============  ==========================================  =====================
gpu_nary       nary_sum / nary_mean / nary_max             rp_all_reduce_v
               (``attrs["ckind"]`` = sum | mean | max;
               premean = the wrap_optimizer all_sum(g/R))
gpu_gather     pack (rank-0 operands) / concat(axis=0)      rp_all_gather_v
gpu_pick0      pick0                                       rp_broadcast_v
=============  ==========================================  =====================

A maintainer keeps the stitcher and rewrites placeholders into these kinds
(``graph.rewrite_node(site, "gpu_nary", inputs, {"ckind": "sum"})``, graph.py:672-692).
This module never imports the reference: it is handed the reference's graph module.
"""

from __future__ import annotations

import numpy as np
import torch

from . import errors
from .comm import DEFAULT_POOL_BYTES, VirtualCommunicator, to_host

_FOLD_KINDS = ("sum", "mean", "max", "premean")


class _Comms:
    """One VirtualCommunicator per replica count, created on first use."""

    def __init__(self, device: int, pool_bytes: int):
        self.device, self.pool_bytes, self.by_n = device, pool_bytes, {}

    def get(self, n: int) -> VirtualCommunicator:
        if n not in self.by_n:
            self.by_n[n] = VirtualCommunicator(n, device=self.device, pool_bytes=self.pool_bytes)
        return self.by_n[n]

    def close(self):
        for c in self.by_n.values():
            c.close()
        self.by_n.clear()


def register(G, device: int = 0, pool_bytes: int = min(DEFAULT_POOL_BYTES, 64 << 20)) -> _Comms:
    """Register ``gpu_nary``, ``gpu_gather`` and ``gpu_pick0`` into the reference graph
    module ``G`` (its ``KINDS`` table, through ``G._register``). Returns the holder of
    the communicators (``.close()`` releases them)."""
    comms = _Comms(int(device), int(pool_bytes))
    dev = torch.device(f"cuda:{int(device)}")

    def _device_inputs(ins):
        # one flat device copy per replica operand (scalars travel as (1,))
        return [torch.from_numpy(np.ascontiguousarray(a)).to(dev).reshape(-1) for a in ins]

    def _fold_kernel(node, ins, ctx):
        kind = node.attrs.get("ckind", "sum")
        if kind not in _FOLD_KINDS:
            raise errors.ShapeError(f"gpu_nary: unknown ckind {kind!r}")
        comm = comms.get(len(ins))
        out = comm.all_reduce(_device_inputs(ins), kind)[0]
        return to_host(out).numpy().reshape(np.shape(ins[0]))

    def _gather_infer(attrs, shapes, dtypes):
        first = shapes[0]
        if any(s != first for s in shapes):
            raise errors.ShapeError(f"gpu_gather: all operands must share shape, got {list(shapes)}")
        dtype = dtypes[0]
        if any(d != dtype for d in dtypes):
            raise errors.ShapeError(f"gpu_gather: mixed dtypes {list(dtypes)}")
        n = len(shapes)
        return ((n,) if first == () else (first[0] * n,) + tuple(first[1:])), dtype

    def _gather_kernel(node, ins, ctx):
        comm = comms.get(len(ins))
        out = comm.all_gather(_device_inputs(ins))[0]  # (n, numel) in rank order
        shape = np.shape(ins[0])
        n = len(ins)
        return to_host(out).numpy().reshape((n,) if shape == () else (shape[0] * n,) + tuple(shape[1:]))

    def _pick0_kernel(node, ins, ctx):
        comm = comms.get(len(ins))
        out = comm.broadcast(_device_inputs(ins), root=0)[0]
        return to_host(out).numpy().reshape(np.shape(ins[0]))

    G._register("gpu_nary", infer=G._infer_nary("gpu_nary"), kernel=_fold_kernel)
    G._register("gpu_gather", infer=_gather_infer, kernel=_gather_kernel)
    G._register("gpu_pick0", infer=lambda a, s, d: (s[0], d[0]), kernel=_pick0_kernel)
    return comms
