"""B200-native data-parallel hot path of TF-Replicator (arXiv 1902.00465).

The cross-replica gradient reduction inside ``wrap_optimizer``, the
all_reduce / all_gather / broadcast primitives and the cross-replica batch-norm
statistics, as hand-written sm_100a CUDA kernels over NVLink/NVSwitch peer memory
behind a C ABI (``include/rp.h``), exposed through the reference's communicator
duck type and Replicator API. See DESIGN.md.
"""

from . import errors
from ._lib import load as load_library
from .bootstrap import DistBootstrap, LoopbackWorld
from .comm import Communicator, VirtualCommunicator
from .replicator import CrossReplicaBatchNorm, PerReplica, ReplicatedOptimizer, Replicator

__all__ = [
    "Communicator",
    "DistBootstrap",
    "LoopbackWorld",
    "VirtualCommunicator",
    "Replicator",
    "ReplicatedOptimizer",
    "PerReplica",
    "CrossReplicaBatchNorm",
    "errors",
    "load_library",
]
__version__ = "0.1.0"
