"""Child process serving the loopback-world tests (test_gpu_world_loopback.py).

A loopback world needs PyTorch's stream-ordered allocator (bootstrap.py
LoopbackWorld), which must be chosen before CUDA initialises; running the worlds in
one spawned child with ``PYTORCH_CUDA_ALLOC_CONF=backend:cudaMallocAsync`` keeps the
rest of the GPU suite on the default allocator."""

import traceback


def serve(conn):
    import torch

    from paper_1902_00465_b200.bootstrap import LoopbackWorld
    from tests import mp_bodies

    torch.cuda.set_device(0)
    conn.send(("ready", torch.cuda.memory.get_allocator_backend()))
    while True:
        msg = conn.recv()
        if msg is None:
            return
        name, world = msg
        try:
            lw = LoopbackWorld(world, device=0)
            fn = getattr(mp_bodies, name)
            lw.run(lambda r: fn(r, world, mp_bodies.Env(r, world, 0, lw.bootstrap(r))))
            conn.send(None)
        except BaseException:  # noqa: BLE001 -- reported to the test
            conn.send(traceback.format_exc())
