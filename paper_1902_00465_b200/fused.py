"""wrap_optimizer(opt, fused=True): the wrapped optimizer step as ONE kernel.

The reference's wrapped optimizer averages every gradient with all_sum(g / R) and
then runs the base rule on every replica,
which keeps the variables mirrored. ``FusedReplicatedOptimizer``
does the same work differently:

* each param group's parameters move into one f32 *parameter bucket* in the
  communicator's pool (the ``nn.Parameter`` objects stay, their storage becomes
  a view of the bucket), and the gradients are packed into a *gradient bucket*
  of the same layout;
* ``step()`` launches rp_all_reduce_apply (csrc/rp_apply.cu): the gradient
  bucket is folded with the rank-ordered premean (bit-identical to the unfused
  averaged gradient), the rank owning each chunk applies SGD / Adam / AdamW to
  its shard and stores the updated parameters into every replica's bucket.

So the optimizer touches 1/N of the parameters per rank, its state is kept for
the owned shard only (N-fold smaller), the gradients are never unpacked, and all
replicas receive the same bits. Hyper-parameters are read from the wrapped
optimizer's ``param_groups`` at every step (LR schedulers keep working; under
CUDA graph capture they are frozen at capture, as for torch's own optimizers).
After ``step()`` ``param.grad`` holds the replica's LOCAL gradient (the averaged
one never leaves the kernel).
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib, errors
from .bucket import _Bucket
from .comm import VirtualCommunicator, _is_dense, dtype_code

_SUPPORTED = {torch.optim.SGD: _lib.OPT_SGD, torch.optim.Adam: _lib.OPT_ADAM, torch.optim.AdamW: _lib.OPT_ADAMW}


def _opt_code(opt) -> int:
    for cls, code in _SUPPORTED.items():
        if type(opt) is cls:
            return code
    raise errors.ConfigurationError(f"fused apply supports torch.optim.SGD / Adam / AdamW, not {type(opt).__name__}")


def _hyper(code: int, group) -> list[float]:
    if group.get("maximize", False):
        raise errors.ConfigurationError("fused apply: maximize=True is not supported")
    if code == _lib.OPT_SGD:
        return [float(group["lr"]), float(group["momentum"]), float(group["dampening"]),
                float(group["weight_decay"]), 0.0, 1.0 if group["nesterov"] else 0.0]
    if group.get("amsgrad", False):
        raise errors.ConfigurationError("fused apply: amsgrad is not supported")
    b1, b2 = group["betas"]
    return [float(group["lr"]), float(b1), float(b2), float(group["weight_decay"]), float(group["eps"]), 0.0]


class _Group:
    """One param group: gradient bucket, parameter bucket, sharded state, step."""

    def __init__(self, comm, code, plists, comm_dtype):
        for plist in plists:
            for p in plist:
                if p.dtype != torch.float32:
                    raise errors.ConfigurationError("fused apply: parameters must be float32")
                if not _is_dense(p):
                    raise errors.ConfigurationError("fused apply: parameters must be dense")
        self.comm = comm
        self.code = code
        # gradients stay off the NVLS region: the kernel pulls them from the pool
        self.grads = _Bucket(comm, plists, torch.float32, comm_dtype or torch.float32, allow_nvls=False,
                             match_param_layout=True)
        n = self.grads.numel
        pbuf = comm.alloc(n, torch.float32)
        self.pflat = pbuf if isinstance(pbuf, list) else [pbuf]
        for r, plist in enumerate(plists):
            flat = self.pflat[r]
            flat.zero_()  # padding between slots stays finite (zero gradients, zero state)
            for p, off in zip(plist, self.grads.offs):
                view = torch.as_strided(flat, p.shape, p.stride(), flat.storage_offset() + off)
                with torch.no_grad():
                    view.copy_(p.detach())
                p.data = view
        lib = _lib.load()
        first, length = ctypes.c_size_t(), ctypes.c_size_t()
        gcode = dtype_code(self.grads.comm_dtype)
        _lib.check(lib.rp_apply_shard(comm._handle, n, gcode, ctypes.byref(first), ctypes.byref(length)),
                   "apply_shard")
        self.shard_len = length.value
        dev = self.pflat[0].device
        nrep = len(plists)
        self.state0 = [torch.zeros(self.shard_len, dtype=torch.float32, device=dev) for _ in range(nrep)]
        self.state1 = ([torch.zeros(self.shard_len, dtype=torch.float32, device=dev) for _ in range(nrep)]
                       if code != _lib.OPT_SGD else [None] * nrep)
        self.steps = [torch.zeros(1, dtype=torch.int32, device=dev) for _ in range(nrep)]

    def apply(self, group):
        self.grads.pack()
        lib = _lib.load()
        hyper = (ctypes.c_double * 6)(*_hyper(self.code, group))
        stream = self.comm._stream()
        gcode = dtype_code(self.grads.comm_dtype)
        n = self.grads.numel
        s1 = [t.data_ptr() if t is not None else 0 for t in self.state1]
        if isinstance(self.comm, VirtualCommunicator):
            g, _k1 = _lib.ptr_array([f.data_ptr() for f in self.grads.flat])
            p, _k2 = _lib.ptr_array([f.data_ptr() for f in self.pflat])
            a0, _k3 = _lib.ptr_array([t.data_ptr() for t in self.state0])
            a1, _k4 = _lib.ptr_array(s1)
            st, _k5 = _lib.ptr_array([t.data_ptr() for t in self.steps])
            _lib.check(lib.rp_all_reduce_apply_v(self.comm._handle, g, p, n, gcode, self.code, hyper, a0, a1, st,
                                                 stream), "all_reduce_apply")
        else:
            _lib.check(lib.rp_all_reduce_apply(self.comm._handle, self.grads.flat[0].data_ptr(),
                                               self.pflat[0].data_ptr(), n, gcode, self.code, hyper,
                                               self.state0[0].data_ptr(), s1[0] or None,
                                               self.steps[0].data_ptr(), stream), "all_reduce_apply")


class FusedReplicatedOptimizer:
    """``Replicator.wrap_optimizer(opt, fused=True)`` (see the module docstring)."""

    def __init__(self, repl, opts):
        self.repl = repl
        self.opts = opts
        self.code = _opt_code(opts[0])
        for o in opts:
            if _opt_code(o) != self.code or len(o.param_groups) != len(opts[0].param_groups):
                raise errors.ProtocolError("replicas wrap different optimizers")
        comm = repl.comm
        self.groups = []
        for gi in range(len(opts[0].param_groups)):
            plists = [[p for p in o.param_groups[gi]["params"] if p.requires_grad] for o in opts]
            if not plists[0]:
                self.groups.append(None)
                continue
            self.groups.append(_Group(comm, self.code, plists, repl.grad_comm_dtype))

    @property
    def optimizer(self):
        return self.opts[self.repl._local_index()]

    @property
    def param_groups(self):
        return self.optimizer.param_groups

    def zero_grad(self, set_to_none: bool = False):
        # gradients are packed from param.grad: keep the tensors (set_to_none is honoured, they are re-created)
        self.optimizer.zero_grad(set_to_none=set_to_none)

    def _apply_all(self, _values=None):
        for gi, grp in enumerate(self.groups):
            if grp is not None:
                grp.apply(self.opts[0].param_groups[gi])
        return [None] * self.repl.num_replicas

    def step(self, closure=None):
        loss = None
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        if self.repl.is_virtual and self.repl.num_replicas > 1:
            self.repl._collective(("wrap_optimizer_fused", id(self)), None, self._apply_all)
        else:
            self._apply_all()
        return loss

    def apply_gradients(self, grads_and_vars):
        """TF-style entry point."""
        for g, v in grads_and_vars:
            v.grad = g.detach().clone() if g is not None else None
        return self.step()

    def state_dict(self):
        """This process's shards of the optimizer state (and the step counters)."""
        return {"kind": int(self.code),
                "groups": [None if g is None else {"step": [s.clone() for s in g.steps],
                                                   "state0": [s.clone() for s in g.state0],
                                                   "state1": [None if s is None else s.clone() for s in g.state1]}
                           for g in self.groups]}

    def load_state_dict(self, sd):
        if sd.get("kind") != int(self.code) or len(sd["groups"]) != len(self.groups):
            raise errors.ProtocolError("state_dict does not match this fused optimizer")
        for g, s in zip(self.groups, sd["groups"]):
            if g is None:
                continue
            for dst, src in zip(g.steps, s["step"]):
                dst.copy_(src)
            for dst, src in zip(g.state0, s["state0"]):
                dst.copy_(src)
            for dst, src in zip(g.state1, s["state1"]):
                if dst is not None:
                    dst.copy_(src)
