"""Host-side logic and the C-ABI boundary, on CPU: the library loads and exports every
symbol include/rp.h declares (no compute calls), status codes map onto the reference's
exception classes, the virtual-replica rendezvous enforces the stitcher's agreement
check, and the multi-process bootstrap exchange works at world_size 2 over gloo."""

import os
import re
import socket
import threading

import pytest
import torch

from paper_1902_00465_b200 import _lib, errors
from tests.helpers import ROOT

HEADER = os.path.join(ROOT, "include", "rp.h")


def header_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"RP_API\s+[\w\s\*]+?\b(rp_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = header_functions()
    for required in ("rp_comm_create", "rp_comm_import", "rp_all_reduce", "rp_all_gather", "rp_broadcast",
                     "rp_bn_stats", "rp_bn_bwd_stats", "rp_pack", "rp_unpack", "rp_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = header_functions()
    assert sorted(_lib.SIGNATURES) == names, "ctypes table must mirror include/rp.h"
    for n in names:
        assert hasattr(lib, n), n
    assert lib.rp_version().decode().endswith("sm_100a")
    assert lib.rp_comm_export_size() > 64


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_missing_library_fails_loudly(monkeypatch):
    monkeypatch.setattr(_lib, "_LIB", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/librp.so")
    with pytest.raises(errors.NativeLibraryError):
        _lib.load()


def test_status_codes_map_to_reference_exceptions():
    _lib.load()
    for code, cls in [(1, errors.ShapeError), (2, errors.ConfigurationError), (3, errors.CollectiveError),
                      (4, errors.CollectiveAbortedError), (5, errors.ProtocolError)]:
        with pytest.raises(cls):
            _lib.check(code, "x")
    _lib.check(0)
    # hierarchy as in the reference's errors.py:4-81
    assert issubclass(errors.ProtocolError, errors.CollectiveError)
    assert issubclass(errors.CollectiveAbortedError, errors.CollectiveError)
    assert issubclass(errors.CollectiveError, errors.ReplicatorError)
    assert issubclass(errors.ShapeError, errors.GraphError)


def test_c_abi_rejects_bad_arguments_without_a_gpu():
    """Argument validation runs before any CUDA call."""
    import ctypes
    lib = _lib.load()
    assert lib.rp_comm_create(0, 9, 0, 64 << 20, ctypes.byref(ctypes.c_void_p())) == 2   # world > 8
    assert lib.rp_comm_create(0, 2, 0, 1 << 20, ctypes.byref(ctypes.c_void_p())) == 1    # pool < 4 MiB
    assert "pool_bytes" in _lib.last_error()
    assert lib.rp_comm_create_virtual(0, 0, 64 << 20, ctypes.byref(ctypes.c_void_p())) == 2
    assert lib.rp_all_reduce(None, None, None, 1, 0, 0, 0, 0, 0, None) == 1            # NULL comm
    assert lib.rp_comm_set_block_cap(None, 32) == 1                                     # NULL comm
    assert lib.rp_broadcast(None, None, None, 16, 0, 4, None) == 1                      # relay, NULL comm
    # round-2 entry points validate before touching a device
    n = ctypes.c_size_t(0)
    assert lib.rp_register_export(None, None, 0, None, ctypes.byref(n)) == 1
    assert lib.rp_register_import(None, None, 0, None) == 1
    assert lib.rp_unregister(None, 0) == 1
    assert lib.rp_comm_set_loopback(None, 1) == 1
    assert lib.rp_comm_topology(None, None, None) == 1
    assert lib.rp_all_reduce_plan(None, None, None, 1, 0, 0, 0, 0, 0, None) == 1
    assert lib.rp_register_export_size() > 64


# --- virtual-replica rendezvous ------------------------------------------------

def _run_threads(n, body):
    errs = [None] * n
    out = [None] * n

    def w(r):
        try:
            out[r] = body(r)
        except BaseException as e:  # noqa: BLE001
            errs[r] = e
    ts = [threading.Thread(target=w, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=30)
    return out, errs


def test_rendezvous_runs_once_for_all_replicas():
    from paper_1902_00465_b200.replicator import _Rendezvous
    rv = _Rendezvous(4)
    calls = []

    def fused(values):
        calls.append(list(values))
        return [sum(values)] * 4

    out, errs = _run_threads(4, lambda r: rv(r, ("all_reduce", "g", (3,)), r + 1, fused))
    assert errs == [None] * 4
    assert out == [10] * 4 and calls == [[1, 2, 3, 4]]  # all_sum 1..4 -> 10


def test_rendezvous_first_divergence_is_protocol_error():
    from paper_1902_00465_b200.replicator import _Rendezvous
    rv = _Rendezvous(2)
    out, errs = _run_threads(2, lambda r: rv(r, ("all_reduce", "a" if r == 0 else "b"), r, lambda v: v))
    assert all(isinstance(e, errors.ProtocolError) for e in errs)
    assert "first divergence" in str(errs[0])


def test_rendezvous_abort_fails_late_arrivals_fast():
    from paper_1902_00465_b200.replicator import _Rendezvous
    rv = _Rendezvous(3)
    rv.abort(RuntimeError("replica 2 died"))
    out, errs = _run_threads(2, lambda r: rv(r, ("x",), r, lambda v: v))
    assert all(isinstance(e, errors.CollectiveAbortedError) for e in errs)


def test_label_reuse_within_a_generation_is_rejected():
    from paper_1902_00465_b200.comm import _Base
    b = _Base()
    b._labels, b.check_labels = set(), True
    b._use_label("g0")
    with pytest.raises(errors.ProtocolError):
        b._use_label("g0")
    b.new_generation()
    b._use_label("g0")                # reuse across generations is fine


def test_bn_layout_detection():
    from paper_1902_00465_b200.replicator import _bn_layout
    assert _bn_layout(torch.empty(8, 3)) == (_lib.NHWC, 8, 3, 1)
    assert _bn_layout(torch.empty(2, 3, 4, 5)) == (_lib.NCHW, 2, 3, 20)
    cl = torch.empty(2, 3, 4, 5).contiguous(memory_format=torch.channels_last)
    assert _bn_layout(cl) == (_lib.NHWC, 40, 3, 1)
    assert _bn_layout(torch.empty(2, 3, 4, 5).transpose(2, 3)) is None
    # non-dense 2-D / 5-D inputs are not read as stored (a stride-0 dy
    # from .sum().backward() or a transpose must be made dense first)
    assert _bn_layout(torch.empty(3, 8).t()) is None
    assert _bn_layout(torch.ones(1).expand(8, 3)) is None
    assert _bn_layout(torch.empty(8, 6)[:, ::2]) is None
    c3 = torch.empty(2, 3, 4, 5, 6).contiguous(memory_format=torch.channels_last_3d)
    assert _bn_layout(c3) == (_lib.NHWC, 240, 3, 1)
    from paper_1902_00465_b200.replicator import _like_layout
    assert _like_layout(torch.ones(1).expand(2, 3, 4, 5, 6), c3).stride() == c3.stride()
    cl4 = torch.empty(2, 3, 4, 5).contiguous(memory_format=torch.channels_last)
    assert _like_layout(torch.ones(1).expand(2, 3, 4, 5), cl4).stride() == cl4.stride()
    assert _like_layout(torch.ones(1).expand(8, 3), torch.empty(8, 3)).is_contiguous()


# --- world_size 2 over gloo: bootstrap exchange ----------------------------------

def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1902_00465_b200.comm import exchange_blobs
        joined = exchange_blobs(bytes([rank]) * 16)
        ok = joined == b"".join(bytes([r]) * 16 for r in range(world))
        try:
            exchange_blobs(bytes([rank]) * (16 + rank))
            bad = False
        except errors.ProtocolError:
            bad = True
        q.put((rank, ok and bad))
    finally:
        dist.destroy_process_group()


def test_bootstrap_exchange_world2_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=30)
    assert res == {0: True, 1: True}


def test_overlap_launcher_keeps_bucket_order():
    """overlap.py: buckets that become ready out of order are held until their
    predecessors launched, so every rank issues the same collective sequence."""
    from paper_1902_00465_b200.overlap import InOrderLauncher
    lo = InOrderLauncher(4)
    assert lo.mark(2) == []
    assert lo.mark(0) == [0]
    assert lo.mark(1) == [1, 2]
    with pytest.raises(errors.ProtocolError):
        lo.mark(1)
    assert lo.rest() == [3]
    lo.reset()
    assert lo.mark(0) == [0] and lo.rest() == [1, 2, 3]


def test_overlap_bucket_plan_reverse_order_per_dtype():
    from paper_1902_00465_b200.overlap import bucket_plan
    sizes = [100, 50, 50, 200, 30, 30]
    dts = ["f", "f", "h", "f", "f", "h"]
    plan = bucket_plan(sizes, dts, limit=100)
    # reverse order; a dtype change does not close the other dtype's bucket;
    # an oversize gradient gets a bucket of its own
    assert plan == [[5, 2], [4], [3], [1], [0]]
    assert sorted(i for b in plan for i in b) == list(range(6))


def test_bench_reference_arm_json_contract():
    """bench.py --impl reference prints one JSON line with the driver's keys (the
    reference's CPU path, bounded sample; no GPU needed)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--bytes", str(1 << 20)],
                         capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["cores"] >= 1


def test_relay_broadcast_tile_partition():
    """The relay broadcast's index math (csrc/rp_nvls.cu bcast_relay): for every
    non-root, the tiles it forwards (owner = i mod (N-1) -> rank) and the tiles it
    receives (j-th tile owned by others) cover every tile exactly once."""
    for world in range(2, 9):
        for root in range(world):
            for nt in (1, 2, world - 1, world, 7 * world + 3):
                w1 = world - 1
                for rank in range(world):
                    if rank == root:
                        continue
                    me = rank if rank < root else rank - 1
                    owned = [me + k * w1 for k in range(nt) if me + k * w1 < nt]
                    for i in owned:  # the owner mapping of the root agrees
                        o = i % w1
                        assert (o if o < root else o + 1) == rank
                    got = []
                    if world > 2:
                        w2 = world - 2
                        for j in range(nt):
                            r = j % w2
                            i = (j // w2) * w1 + (r if r < me else r + 1)
                            if i >= nt:
                                break
                            got.append(i)
                    assert sorted(owned + got) == list(range(nt)), (world, root, nt, rank)


# --- topology policy (rp_comm_import, include/rp.h rp_topology_check) -----------

def _links(*kinds):
    import ctypes
    arr = (ctypes.c_int * len(kinds))(*kinds)
    return arr


def test_topology_policy_requires_nvlink_everywhere():
    """An NVSwitch all-to-all (NVLink to every peer) passes; a PCIe-only peer, a
    peer without peer access, an invisible peer or another process on the same GPU
    is a ConfigurationError naming the pair (errors.py:32); RP_ALLOW_PCIE
    admits PCIe for tests, and same-GPU ranks only inside a loopback world."""
    lib = _lib.load()
    S, NV, PCIE, NONE, UNK, SAME, LOOP = (_lib.LINK_SELF, _lib.LINK_NVLINK, _lib.LINK_PCIE, _lib.LINK_NONE,
                                          _lib.LINK_UNKNOWN, _lib.LINK_SAME_DEVICE, _lib.LINK_LOOPBACK)
    _lib.check(lib.rp_topology_check(4, 1, _links(NV, S, NV, NV), 0, 0))
    for bad, what in ((PCIE, "PCIe"), (NONE, "no peer access"), (UNK, "unknown"), (SAME, "same device"),
                      (LOOP, "loopback")):
        with pytest.raises(errors.ConfigurationError) as ei:
            _lib.check(lib.rp_topology_check(4, 1, _links(NV, S, bad, NV), 0, 0), "comm_import")
        assert "rank 1 -> rank 2" in str(ei.value) and what in str(ei.value), str(ei.value)
    _lib.check(lib.rp_topology_check(2, 0, _links(S, PCIE), 1, 0))      # RP_ALLOW_PCIE=1
    _lib.check(lib.rp_topology_check(3, 2, _links(LOOP, LOOP, S), 0, 1))  # loopback world
    with pytest.raises(errors.ConfigurationError):
        _lib.check(lib.rp_topology_check(2, 0, _links(S, SAME), 1, 1))  # another process on this GPU
    with pytest.raises(errors.ConfigurationError):
        _lib.check(lib.rp_topology_check(2, 0, _links(NV, S), 0, 0))    # "self" on the wrong rank
    with pytest.raises(errors.ShapeError):
        _lib.check(lib.rp_topology_check(9, 0, _links(*([NV] * 9)), 0, 0))


def test_topology_requires_uniform_nvlink():
    """rp_comm_import also requires every GPU to have the same number of active NVLink
    links (an NVSwitch all-to-all: 18 per B200); unknown counts (-1) are skipped."""
    lib = _lib.load()
    _lib.check(lib.rp_topology_uniform(4, _links(18, 18, 18, 18)))
    _lib.check(lib.rp_topology_uniform(3, _links(18, -1, 18)))
    with pytest.raises(errors.ConfigurationError, match="non-uniform NVLink"):
        _lib.check(lib.rp_topology_uniform(4, _links(18, 18, 12, 18)), "comm_import")
    with pytest.raises(errors.ConfigurationError, match="no active NVLink"):
        _lib.check(lib.rp_topology_uniform(2, _links(0, 0)), "comm_import")


# --- loopback bootstrap (bootstrap.py) ------------------------------------------

def test_loopback_bootstrap_exchanges_in_rank_order():
    """The in-process rendezvous a loopback world's communicators bootstrap over:
    all_gather_object returns every rank's object in rank order (repeatedly, no
    slot reuse race), broadcast_object delivers the root's, and a failing rank
    breaks the barrier instead of hanging the others."""
    from paper_1902_00465_b200.bootstrap import LoopbackWorld

    lw = LoopbackWorld(4, device=0, timeout_s=30, allow_native_allocator=True)

    def body(r):
        b = lw.bootstrap(r)
        outs = [b.all_gather_object((r, k)) for k in range(20)]
        return outs, b.broadcast_object(f"root{r}", src=2)

    def run():
        import threading as th
        res = [None] * 4

        def w(r):
            res[r] = body(r)
        ts = [th.Thread(target=w, args=(r,)) for r in range(4)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(timeout=60)
        return res
    res = run()
    for r in range(4):
        outs, root = res[r]
        assert outs == [[(q, k) for q in range(4)] for k in range(20)]
        assert root == "root2"

    lw2 = LoopbackWorld(3, device=0, timeout_s=30, allow_native_allocator=True)

    def failing(r):
        if r == 1:
            raise ValueError("rank 1 fails before the rendezvous")
        lw2.bootstrap(r).barrier()

    errs = _run_threads(3, lambda r: failing(r) if r != 1 else (lw2._barrier.abort(), failing(r)))[1]
    assert isinstance(errs[1], ValueError)
    assert all(isinstance(errs[r], threading.BrokenBarrierError) for r in (0, 2))


def test_loopback_world_requires_the_stream_ordered_allocator():
    """The native caching allocator's cudaMalloc can wait on a peer rank's kernel
    (measured deadlock, bootstrap.py): a loopback world refuses it loudly."""
    from paper_1902_00465_b200.bootstrap import LoopbackWorld

    if torch.cuda.memory.get_allocator_backend() == "cudaMallocAsync":
        pytest.skip("this process already runs the stream-ordered allocator")
    with pytest.raises(errors.ConfigurationError, match="cudaMallocAsync"):
        LoopbackWorld(2)
    LoopbackWorld(1)  # a single rank never waits on a peer
