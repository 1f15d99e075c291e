"""Exception hierarchy, mirroring the reference's ``pkg/src/replicator/errors.py`` so
callers catch the same classes (names and parentage as in errors.py:4-81).

C-ABI status codes (include/rp.h, ``RP_ERR_*``) map onto these classes in
``paper_1902_00465_b200._lib.check``.
"""


class ReplicatorError(Exception):
    """Base class for every error raised by this package (errors.py:4)."""


class GraphError(ReplicatorError):
    """errors.py:8."""


class ShapeError(GraphError):
    """Operand shapes / dtypes invalid for an op (errors.py:12)."""


class NotDifferentiableError(GraphError):
    """Backpropagation reached an op without a VJP (errors.py:16): here a collective
    on in-process virtual replicas, whose backward passes share one autograd device
    thread and so cannot rendezvous (the reference raises it for every collective,
    graph.py:798-800)."""


class EvaluationError(GraphError):
    """Runtime failure while executing (errors.py:24)."""


class ConfigurationError(ReplicatorError):
    """Invalid deployment topology (errors.py:32): e.g. no NVLink peer access."""


class TransportError(ReplicatorError):
    """errors.py:36. Kept for interface parity; the NVLink path has no transport."""


class CollectiveError(ReplicatorError):
    """A collective operation failed on this rank (errors.py:60)."""


class ProtocolError(CollectiveError):
    """Ranks disagreed on label, kind, shape, or label reuse (errors.py:64)."""


class CollectiveAbortedError(CollectiveError):
    """Another rank aborted the collective, or a wait timed out (errors.py:68)."""


class NativeLibraryError(ReplicatorError):
    """The sm_100a library (librp.so) is missing or failed to load. There is no CPU
    fallback: the product path refuses to run without its CUDA kernels."""
