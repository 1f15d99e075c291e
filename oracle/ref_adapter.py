"""Import the reference package (``/root/reference/pkg/src/replicator``) for fixture
generation. TEST INFRASTRUCTURE ONLY -- runs in the build container; the GPU box has
no ``/root/reference`` and nothing under ``tests -m gpu``, ``smoke()`` or ``bench.py``
imports this module.

Applies the survey's 6-line 0-d shim: ``Tensor.__init__``
promotes rank-0 arrays to shape (1,) via ``np.ascontiguousarray``
(``pkg/src/replicator/tensor.py:48``), which breaks scalar constants and ``backprop``'s
seed (``graph.py:785``). The shim only restores the 0-d shape; values are untouched.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = os.environ.get("RP_REFERENCE_SRC", "/root/reference/pkg/src")


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
