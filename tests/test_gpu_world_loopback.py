"""The multi-process kernels on ONE GPU: a LoopbackWorld (bootstrap.py) runs W
non-virtual communicators in this process on cuda:0, one host thread and one CUDA
stream per rank, peers' pools mapped as plain pointers and every rank's grid capped
at 148 / W blocks so all ranks' blocks are co-resident (include/rp.h
rp_comm_set_loopback).

Same rank bodies as the one-process-per-GPU harness (tests/mp_bodies.py): the push
one-shot and two-shot all-reduce, push all_gather and broadcast, relay broadcast,
the BN exchange and its autograd, fused apply, check_protocol, CUDA-graph replay,
the dead-rank timeout, overlapped buckets and the host pipeline -- every form
``rp_resolve_ar_algo`` / the broadcast and gather choosers pick between processes,
with the same `.sys`-scope release/acquire barriers -- each checked bit-exactly
against the oracle (BN: 1e-6 relative). NVLS needs distinct devices and stays in
test_gpu_multiproc.py. The reference seam these serve: graph.py:565-583;
symmetry and liveness: SPEC.md:234-237.
"""

import os

import pytest

pytestmark = pytest.mark.gpu


class _Server:
    """One spawned child (tests/loopback_server.py) runs the worlds one after the
    other; a world that does not finish in time kills the child (the next test
    starts a fresh one)."""

    def __init__(self):
        self.proc = self.conn = None

    def start(self):
        import torch.multiprocessing as mp

        from tests.loopback_server import serve

        ctx = mp.get_context("spawn")
        self.conn, child = ctx.Pipe()
        old = os.environ.get("PYTORCH_CUDA_ALLOC_CONF")
        os.environ["PYTORCH_CUDA_ALLOC_CONF"] = "backend:cudaMallocAsync"
        try:
            self.proc = ctx.Process(target=serve, args=(child,), daemon=True)
            self.proc.start()
        finally:
            if old is None:
                os.environ.pop("PYTORCH_CUDA_ALLOC_CONF")
            else:
                os.environ["PYTORCH_CUDA_ALLOC_CONF"] = old
        assert self.conn.poll(300), "loopback server did not start"
        tag, backend = self.conn.recv()
        assert tag == "ready" and backend == "cudaMallocAsync", backend

    def run(self, name: str, world: int, timeout: float):
        if self.proc is None or not self.proc.is_alive():
            self.start()
        self.conn.send((name, world))
        if not self.conn.poll(timeout):
            self.stop(kill=True)
            pytest.fail(f"loopback world {name} x{world} did not finish in {timeout} s")
        err = self.conn.recv()
        assert err is None, err

    def stop(self, kill: bool = False):
        if self.proc is None:
            return
        if not kill and self.proc.is_alive():
            self.conn.send(None)
            self.proc.join(60)
        if self.proc.is_alive():
            self.proc.kill()
            self.proc.join(30)
        self.proc = self.conn = None


_SERVER = _Server()


@pytest.fixture(scope="module", autouse=True)
def _server_lifetime():
    yield
    _SERVER.stop()


def run_loopback(name: str, world: int, timeout: float = 600):
    _SERVER.run(name, world, timeout)


W24 = pytest.mark.parametrize("world", [2, 4])
W248 = pytest.mark.parametrize("world", [2, 4, 8])


@pytest.mark.timeout(900)
@W248
def test_all_reduce_loopback(world):
    run_loopback("body_all_reduce", world)


@pytest.mark.timeout(900)
@W248
def test_gather_broadcast_loopback(world):
    run_loopback("body_gather_broadcast", world)


@pytest.mark.timeout(300)
@W24
def test_reference_graph_evaluate_through_communicator_loopback(world):
    from oracle import ref_adapter
    if not ref_adapter.available():
        pytest.skip("reference package not vendored (oracle/ref_vendor.py)")
    run_loopback("body_reference_graph", world)


@pytest.mark.timeout(300)
@W248
def test_back_to_back_random_sequence_loopback(world):
    run_loopback("body_random_sequence", world)


@pytest.mark.timeout(300)
@W248
def test_registered_user_buffers_loopback(world):
    run_loopback("body_register", world)


@pytest.mark.timeout(300)
def test_reference_mesh_seam_replay_loopback():
    run_loopback("body_mesh_seam", 2)


@pytest.mark.timeout(300)
@W248
def test_cross_replica_bn_autograd_loopback(world):
    run_loopback("body_bn", world)


@pytest.mark.timeout(300)
@W24
def test_bn_layouts_and_broadcast_gradients_loopback(world):
    run_loopback("body_bn_layouts", world)


@pytest.mark.timeout(300)
@W24
def test_collective_adjoints_loopback(world):
    run_loopback("body_autograd", world)


@pytest.mark.timeout(300)
@W248
def test_wrap_optimizer_sync_equivalence_loopback(world):
    run_loopback("body_wrap_optimizer", world)


@pytest.mark.timeout(300)
@W248
def test_fused_apply_loopback(world):
    run_loopback("body_fused_apply", world)


@pytest.mark.timeout(300)
@W24
def test_protocol_checks_and_ragged_gather_loopback(world):
    run_loopback("body_protocol", world)


@pytest.mark.timeout(300)
@W248
def test_cuda_graph_replay_loopback(world):
    run_loopback("body_graph", world)


@pytest.mark.timeout(300)
@W24
def test_dead_rank_times_out_loopback(world):
    run_loopback("body_timeout", world)


@pytest.mark.timeout(300)
@W24
def test_overlapped_wrap_optimizer_loopback(world):
    run_loopback("body_overlap", world)


@pytest.mark.timeout(300)
@W24
def test_overlap_beside_bn_collectives_loopback(world):
    run_loopback("body_overlap_with_bn", world)


@pytest.mark.timeout(300)
@W24
def test_host_pipelined_all_reduce_loopback(world):
    run_loopback("body_host_pipeline", world)


@pytest.mark.timeout(600)
@W248
def test_relay_broadcast_loopback(world):
    run_loopback("body_relay_broadcast", world)
