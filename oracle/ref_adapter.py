"""Import the reference package (``replicator``) -- TEST INFRASTRUCTURE ONLY.

Source: ``oracle/_ref/replicator``, the git-ignored copy ``oracle/ref_vendor.py``
makes from ``/root/reference/pkg/src/replicator`` at build time (it travels to the
GPU box; ``/root/reference`` does not), else ``/root/reference/pkg/src`` itself.
Used to generate the golden fixtures, by the GPU tests that run the reference's own
``Graph.evaluate`` through this repo's communicators (the checker, never the thing
measured), and by ``bench.py --impl reference`` (the reference's own CPU path).

Applies the survey's 6-line 0-d shim: ``Tensor.__init__``
promotes rank-0 arrays to shape (1,) via ``np.ascontiguousarray``
(``pkg/src/replicator/tensor.py:48``), which breaks scalar constants and ``backprop``'s
seed (``graph.py:785``). The shim only restores the 0-d shape; values are untouched.
"""

from __future__ import annotations

import os
import sys

import numpy as np

_VENDORED = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")
REF_SRC = os.environ.get("RP_REFERENCE_SRC") or (
    _VENDORED if os.path.isdir(os.path.join(_VENDORED, "replicator")) else "/root/reference/pkg/src")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "replicator"))


def load(shim: bool = True):
    """Return the reference modules (tensor, graph, variables, errors)."""
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import replicator.errors as errors
    import replicator.graph as graph
    import replicator.tensor as tensor
    import replicator.variables as variables

    if shim and not getattr(tensor.Tensor, "_rp_zero_d_shim", False):
        orig = tensor.Tensor.__init__

        def _init(self, data, dtype=None):
            orig(self, data, dtype)
            if np.ndim(data) == 0 and self._np.shape == (1,):
                a = self._np.reshape(()).copy()
                a.setflags(write=False)
                self._np = a

        tensor.Tensor.__init__ = _init
        tensor.Tensor._rp_zero_d_shim = True
    return tensor, graph, variables, errors
