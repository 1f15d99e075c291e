"""Multi-process NVLink path: one process per GPU, communicators bootstrapped over
torch.distributed (gloo, handle exchange only), kernels loading/storing peer pools.
Needs >= 2 GPUs (``gpurun --gpus 2`` / ``--gpus 4``); skipped otherwise. The rank
bodies live in tests/mp_bodies.py and also run in a one-GPU loopback world
(test_gpu_world_loopback.py)."""

import os
import socket

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
if NGPU < 2:
    pytest.skip("needs >= 2 CUDA devices", allow_module_level=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn_name, q):
    import torch.distributed as dist

    from tests import mp_bodies

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        getattr(mp_bodies, fn_name)(rank, world, mp_bodies.Env(rank, world, rank))
        q.put((rank, None))
    except BaseException as e:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def run_world(fn_name, world=None, timeout=600):
    import torch.multiprocessing as mp

    world = world or min(NGPU, 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    errs = {}
    for _ in range(world):
        r, err = q.get(timeout=timeout)
        errs[r] = err
    for p in procs:
        p.join(timeout=60)
    bad = {r: e for r, e in errs.items() if e}
    assert not bad, "\n".join(f"rank {r}:\n{e}" for r, e in bad.items())


# ---------------------------------------------------------------------------

def test_all_reduce_multiprocess():
    run_world("body_all_reduce")


def test_gather_broadcast_multiprocess():
    run_world("body_gather_broadcast")


def test_reference_mesh_seam_replay():
    run_world("body_mesh_seam", world=2)


def test_reference_graph_evaluate_through_communicator_multiprocess():
    run_world("body_reference_graph")


def test_back_to_back_random_sequence_multiprocess():
    run_world("body_random_sequence")


def test_registered_user_buffers_multiprocess():
    run_world("body_register")


def test_cross_replica_bn_autograd_multiprocess():
    run_world("body_bn")


def test_bn_layouts_multiprocess():
    run_world("body_bn_layouts")


def test_collective_adjoints_multiprocess():
    run_world("body_autograd")


def test_wrap_optimizer_sync_equivalence_multiprocess():
    run_world("body_wrap_optimizer")


def test_nvls_all_reduce_multiprocess():
    run_world("body_nvls")


def test_wrap_optimizer_nvls_buckets_multiprocess():
    run_world("body_wrap_nvls")


def test_fused_apply_multiprocess():
    run_world("body_fused_apply")


def test_protocol_checks_and_ragged_gather_multiprocess():
    run_world("body_protocol")


def test_cuda_graph_replay_multiprocess():
    run_world("body_graph")


def test_dead_rank_times_out():
    run_world("body_timeout")


def test_overlapped_wrap_optimizer_multiprocess():
    run_world("body_overlap")


def test_overlap_beside_bn_collectives_multiprocess():
    run_world("body_overlap_with_bn")


def test_host_pipelined_all_reduce_multiprocess():
    run_world("body_host_pipeline")


def test_relay_broadcast_multiprocess():
    run_world("body_relay_broadcast")
