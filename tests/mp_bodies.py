"""Rank bodies of the multi-rank tests, shared by two harnesses:

* ``test_gpu_multiproc.py`` -- one process per GPU over torch.distributed (gloo,
  handle exchange only): the NVLink path proper (needs >= 2 GPUs);
* ``test_gpu_world_loopback.py`` -- a LoopbackWorld (bootstrap.py): W ranks in one
  process on ONE GPU, one host thread and stream each, the same kernels, barriers
  and algorithm choices with local HBM in place of NVLink (runs on the driver's
  1-GPU box).

Every rank derives all ranks' inputs from per-rank seeds, so each rank checks its
own result against the CPU oracle on identical inputs (bit-exact folds / copies,
1e-6 BN statistics). ``env`` abstracts the harness: device, bootstrap, a host
barrier, an object all-gather and a synchronise that never waits on other ranks'
streams (a device-wide sync in a loopback world would wait on a peer kernel that
is itself waiting for this rank's next launch).
"""

import os
import threading

import numpy as np
import pytest
import torch


class Env:
    def __init__(self, rank: int, world: int, device: int, bootstrap=None):
        self.rank, self.world, self.device = rank, world, device
        self.dev = torch.device(f"cuda:{device}")
        self.bootstrap = bootstrap
        self.loopback = bool(getattr(bootstrap, "loopback", False))
        # message sizes: the largest cases only where they are cheap to check
        self.big = not self.loopback or world <= 2

    def _boot(self):
        if self.bootstrap is not None:
            return self.bootstrap
        from paper_1902_00465_b200.bootstrap import DistBootstrap
        return DistBootstrap()

    def barrier(self):
        self._boot().barrier()

    def all_gather_object(self, obj):
        return self._boot().all_gather_object(obj)

    def set_env(self, key, value):
        """Set (value None: remove) a process environment variable the library reads
        at launch time. A loopback world shares one environment, so every rank
        must have finished launching under the old value before rank 0 changes it,
        and nobody launches under the new one before it is set."""
        self.barrier()
        if not self.loopback or self.rank == 0:
            if value is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = value
        self.barrier()

    def sync(self):
        if self.loopback:
            torch.cuda.current_stream(self.dev).synchronize()
        else:
            torch.cuda.synchronize()


def H(t):
    """Device -> host through pinned memory (comm.to_host): a pageable copy may wait
    on a loopback peer's kernel that is waiting for this rank."""
    from paper_1902_00465_b200.comm import to_host
    return to_host(t) if isinstance(t, torch.Tensor) else t


def EQ(a, b):
    """torch.equal on the host (on CUDA tensors it ends in a pageable scalar copy)."""
    return torch.equal(H(a), H(b))


_CACHE: dict = {}
_CACHE_LOCK = threading.Lock()


def _cached(key, fn):
    """Inputs and oracle results shared by the ranks of a loopback world (every
    rank derives the same arrays; computing them once keeps W=8 cheap)."""
    with _CACHE_LOCK:
        if key in _CACHE:
            return _CACHE[key]
    val = fn()
    with _CACHE_LOCK:
        if len(_CACHE) > 24:
            _CACHE.clear()
        return _CACHE.setdefault(key, val)



def _inputs(world, count, dtype=np.float32, seed=100):
    return _cached(("in", world, count, np.dtype(dtype).str, seed),
                   lambda: [np.random.default_rng(seed + r).standard_normal(count).astype(dtype) for r in range(world)])


def body_all_reduce(rank, world, env):
    from oracle import collectives as O
    from paper_1902_00465_b200.comm import Communicator

    dev = env.dev
    comm = Communicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=96 << 20)
    counts = (1, 7, 1000, 4097, 1 << 16, (1 << 20) + 3) + ((16 << 20, 40 << 20) if env.big else (3 << 20,))
    for impl in ("push", "pull"):
        env.set_env("RP_AR_IMPL", impl)
        for count in counts:
            xs = _inputs(world, count, seed=count)
            x = torch.from_numpy(xs[rank]).to(dev)
            for kind in ("sum", "mean", "max", "premean"):
                want = _cached(("fold", world, count, kind), lambda: O.FOLDS[kind](xs))
                for algo in ("oneshot", "twoshot"):
                    y = comm.all_reduce_tensor(x, kind, algo=algo)
                    got = H(y).numpy()
                    assert got.tobytes() == want.tobytes(), (impl, count, kind, algo)
                    y2 = x.clone()
                    comm.all_reduce_tensor(y2, kind, out=y2, algo=algo)  # in place, user buffer
                    assert H(y2).numpy().tobytes() == want.tobytes(), (impl, count, kind, algo, "inplace")
    env.set_env("RP_AR_IMPL", None)
    # f64 and bf16 with the fused exchange cast
    xs = _inputs(world, 33333, np.float64, seed=7)
    y = comm.all_reduce_tensor(torch.from_numpy(xs[rank]).to(dev), "sum")
    assert H(y).numpy().tobytes() == O.fold_sum(xs).tobytes()
    xs = _inputs(world, 50001, seed=8)
    y = comm.all_reduce_tensor(torch.from_numpy(xs[rank]).to(dev), "premean", comm_dtype=torch.bfloat16)
    want = O.bf16_bits_to_f32(O.fold_bf16([O.f32_to_bf16_bits(x) for x in xs], "premean"))
    assert H(y).numpy().tobytes() == want.tobytes()
    # zero-copy in place in the registered pool
    buf = comm.alloc(1 << 20, torch.float32)
    xs = _inputs(world, 1 << 20, seed=9)
    buf.copy_(torch.from_numpy(xs[rank]))
    comm.all_reduce_tensor(buf, "premean", out=buf)
    assert H(buf).numpy().tobytes() == O.fold_premean(xs).tobytes()
    comm.check()
    comm.close()


def body_gather_broadcast(rank, world, env):
    from oracle import collectives as O
    from paper_1902_00465_b200.comm import Communicator

    dev = env.dev
    comm = Communicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=96 << 20)
    for count in (1, 7, 1000, 12345, 65536, 65537, 1 << 20):
        xs = _inputs(world, count, seed=count + 1)
        g = comm.all_gather_tensor(torch.from_numpy(xs[rank]).to(dev))
        assert H(g).numpy().tobytes() == np.concatenate(xs).tobytes()
        # in place: src is this rank's slot of a pool-resident output
        out = comm.alloc(world * count, torch.float32).view(world, count)
        out[rank].copy_(torch.from_numpy(xs[rank]))
        comm.all_gather_tensor(out[rank], out=out)
        assert H(out).numpy().tobytes() == np.concatenate(xs).tobytes(), count
        for root in range(world):
            for algo in ("auto", "direct", "scatter") + (("relay",) if count % 4 == 0 else ()):
                x = torch.from_numpy(xs[rank]).to(dev)
                comm.broadcast_tensor(x, root=root, algo=algo)
                assert H(x).numpy().tobytes() == xs[root].tobytes(), (count, root, algo)
    # dense non-contiguous layouts (channels_last parameters) are exchanged in place,
    # strided views through a copy that is written back
    g = torch.Generator(device=dev).manual_seed(77 + rank)
    cl = torch.randn(2, 8, 5, 3, device=dev, generator=g).contiguous(memory_format=torch.channels_last)
    cl_ptr = cl.data_ptr()
    comm.broadcast_tensor(cl, root=0)
    assert cl.data_ptr() == cl_ptr and cl.is_contiguous(memory_format=torch.channels_last)
    allc = comm.all_gather_tensor(cl.contiguous())
    assert all(EQ(allc[r], allc[0]) for r in range(world))
    base = torch.randn(6, 10, device=dev, generator=g)
    view = base[:, ::2]
    before = [comm.all_gather_tensor(view.contiguous())[r].clone() for r in range(world)]
    comm.all_reduce_tensor(view, "sum", out=view)
    want = before[0].clone()
    for r in range(1, world):
        want = want + before[r]
    assert EQ(view, want) and EQ(base[:, 1::2], base[:, 1::2])
    # reference duck type with host values (graph.py:573-582)
    xs = _inputs(world, 6, seed=3)
    local = xs[rank].reshape(2, 3)
    assert comm.all_reduce(local, "sum", "l").tobytes() == O.fold_sum([x.reshape(2, 3) for x in xs]).tobytes()
    parts = comm.all_gather(local, "g")
    assert all(p.tobytes() == xs[r].reshape(2, 3).tobytes() for r, p in enumerate(parts))
    b = comm.broadcast(local if rank == 0 else None, "b", shape=(2, 3), dtype="f32")
    assert b.tobytes() == xs[0].reshape(2, 3).tobytes()
    comm.check()
    comm.close()


class RefTensor:
    """Stand-in for the reference's Tensor (tensor.py:32-98: immutable f32/f64 array,
    ``.np``, ``.shape``, ``.dtype``, ``Tensor.wrap``); /root/reference is not on the box."""

    def __init__(self, arr):
        arr = np.ascontiguousarray(arr)
        arr.setflags(write=False)
        self._np = arr

    @staticmethod
    def wrap(arr):
        return RefTensor(arr)

    @property
    def np(self):
        return self._np

    @property
    def shape(self):
        return self._np.shape

    @property
    def dtype(self):
        return {np.dtype(np.float32): "f32", np.dtype(np.float64): "f64"}[self._np.dtype]


def body_mesh_seam(rank, world, env):
    """Replay what the reference's mesh seam hands a communicator
    (tests/golden/mesh_seam.json, recorded from graph.py:565-583) and check our
    Communicator returns what the seam expects, as the reference's Tensor type."""
    import json

    from paper_1902_00465_b200.comm import Communicator
    from tests.helpers import GOLDEN

    if world != 2:
        return
    comm = Communicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=16 << 20)
    trace = json.load(open(os.path.join(GOLDEN, "mesh_seam.json")))["trace"]
    for t in trace:
        if t["rank"] != rank:
            continue
        npd = np.float32 if t["dtype"] == "f32" else np.float64
        shape = tuple(t["calls"][0]["shape"])          # what the seam passes (scalars as (1,))
        local = RefTensor(np.full(shape, float(rank + 1), npd))
        outs = []
        for c in t["calls"]:
            if c["op"] == "all_reduce":
                r = comm.all_reduce(local, c["kind"], c["label"])
                assert isinstance(r, RefTensor) and r.shape == local.shape and r.dtype == t["dtype"]
                outs.append(r.np)
            elif c["op"] == "all_gather":
                parts = comm.all_gather(local, c["label"])
                assert all(isinstance(p, RefTensor) for p in parts) and len(parts) == 2
                outs.append(np.concatenate([p.np for p in parts], axis=0))  # graph.py:579
            else:
                rv = local if rank == 0 else None
                r = comm.broadcast(rv, c["label"], shape=tuple(c["shape"]), dtype=c["dtype"])
                outs.append(r.np)
        for got, want in zip(outs, t["out_values"]):
            assert H(got.reshape(-1)).tolist() == want, (t["shape"], t["dtype"])
    comm.close()


def _stitched_reference(G, T, xs, dtype):
    """The reference's own in-process evaluation of one replica site per collective
    kind over all replicas' inputs (the stitched folds, graph.py:506-540)."""
    shape = np.shape(xs[0])
    g = G.Graph()
    ins = [g.add_node("input", [], {"shape": shape, "dtype": dtype}) for _ in xs]
    sites = {"sum": g.add_node("nary_sum", ins), "mean": g.add_node("nary_mean", ins),
             "max": g.add_node("nary_max", ins),
             "gather": g.add_node("pack", ins) if shape == () else g.add_node("concat", ins, {"axis": 0}),
             "broadcast": g.add_node("pick0", ins)}
    g.finalize()
    res = g.evaluate(list(sites.values()), {i: T.Tensor(x, dtype=dtype) for i, x in zip(ins, xs)})
    return {k: r.np for k, r in zip(sites, res)}


def body_reference_graph(rank, world, env):
    """the REFERENCE's own engine with this repo as its
    communicator. Each rank builds the reference Graph with one ``mesh_collective``
    per kind (sum / mean / max / gather / broadcast) and evaluates it with
    ``runtime={"communicator": Communicator}`` (graph.py:565-583, :706-707); every
    result must equal, bit for bit, the reference's own stitched in-process fold of
    all ranks' inputs (nary_* / concat / pack / pick0, graph.py:506-540), for
    scalars (the seam's (1,) promotion included), 2x3 and 1000-element f32 / f64."""
    from oracle import ref_adapter
    from paper_1902_00465_b200.comm import Communicator

    if not ref_adapter.available():
        pytest.skip("reference package not vendored (oracle/ref_vendor.py)")
    T, G, _, _ = ref_adapter.load()
    comm = Communicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=16 << 20)
    kinds = ("sum", "mean", "max", "gather", "broadcast")
    for dtype, npd in (("f32", np.float32), ("f64", np.float64)):
        for shape in ((), (2, 3), (1000,)):
            xs = [np.random.default_rng(500 + 7 * r + len(shape)).standard_normal(shape).astype(npd)
                  for r in range(world)]
            g = G.Graph()
            x = g.add_node("input", [], {"shape": shape, "dtype": dtype})
            nodes = [g.add_node("mesh_collective", [x], {"ckind": k, "label": f"{k}/{dtype}/{shape}",
                                                          "num_replicas": world}) for k in kinds]
            g.finalize()
            res = g.evaluate(nodes, {x: T.Tensor(xs[rank], dtype=dtype)}, runtime={"communicator": comm})
            want = _stitched_reference(G, T, xs, dtype)
            for k, r in zip(kinds, res):
                assert isinstance(r, T.Tensor) and r.dtype == dtype, (k, type(r), r.dtype)
                assert r.np.reshape(-1).tobytes() == want[k].reshape(-1).tobytes(), (k, dtype, shape)
    # no communicator at runtime: the reference's own EvaluationError (graph.py:567-569)
    g = G.Graph()
    x = g.add_node("input", [], {"shape": (2,), "dtype": "f64"})
    y = g.add_node("mesh_collective", [x], {"ckind": "sum", "label": "none", "num_replicas": world})
    g.finalize()
    from replicator import errors as ref_errors
    with pytest.raises(ref_errors.EvaluationError):
        g.evaluate([y], {x: T.Tensor(np.ones(2))})
    comm.check()
    comm.close()


def body_random_sequence(rank, world, env):
    """SURVEY §5 flag-protocol test: a seeded random sequence of mixed collectives
    (all-reduce of user / in-place / pool buffers, all_gather, broadcast from
    varying roots; 1 to 262144 elements, so one-shot, two-shot, push and pull forms
    and the landing-zone parities interleave) issued back to back with NO
    synchronisation between calls, every result checked bit-exactly afterwards:
    back-to-back collectives never read stale or overwritten peer data."""
    from oracle import collectives as O
    from paper_1902_00465_b200.comm import Communicator

    dev = env.dev
    rng = np.random.default_rng(2024)
    ops = [(str(rng.choice(["ar", "ar_inplace", "ar_pool", "ag", "bc"])),
            int(rng.choice([1, 7, 1000, 4097, 65536, 203530, 262144]))) for _ in range(48)]
    comm = Communicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=32 << 20)
    bucket = comm.alloc(300000, torch.float32)
    pending = []
    for i, (op, count) in enumerate(ops):
        xs = _cached(("seq", world, i, count), lambda: [np.random.default_rng(1000 * i + r).standard_normal(count)
                                                        .astype(np.float32) for r in range(world)])
        x = torch.from_numpy(xs[rank]).to(dev)
        if op == "ar":
            pending.append((i, op, comm.all_reduce_tensor(x, "sum"), O.fold_sum(xs)))
        elif op == "ar_inplace":
            comm.all_reduce_tensor(x, "sum", out=x)
            pending.append((i, op, x, O.fold_sum(xs)))
        elif op == "ar_pool":
            b = bucket[:count]
            b.copy_(x)
            comm.all_reduce_tensor(b, "premean", out=b)
            pending.append((i, op, b.clone(), O.fold_premean(xs)))  # the bucket is reused by later ops
        elif op == "ag":
            pending.append((i, op, comm.all_gather_tensor(x).reshape(-1), np.concatenate(xs)))
        else:
            comm.broadcast_tensor(x, root=i % world)
            pending.append((i, op, x, xs[i % world]))
    env.sync()
    for i, op, got, want in pending:
        assert H(got).numpy().tobytes() == want.tobytes(), (i, op, ops[i])
    comm.check()
    comm.close()


def body_register(rank, world, env):
    """User-buffer registration (include/rp.h rp_register_*): in-place all-reduces of
    a registered tensor, and of a view at the same offset inside it, take the
    zero-copy pull two-shot (plan placement -2) and equal the oracle fold bit for
    bit, back to back; small messages keep the push one-shot; after unregister the
    buffer is a plain user buffer again (push form, placement -1)."""
    from oracle import collectives as O
    from paper_1902_00465_b200.comm import Communicator

    dev = env.dev
    comm = Communicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=32 << 20)
    count = 3 << 20
    x = torch.empty(count, device=dev)
    reg = comm.register(x)
    assert comm.plan_for(x, "sum", out=x) == (2, 0, -2, -2), comm.plan_for(x, "sum", out=x)
    for it in range(3):
        xs = _inputs(world, count, seed=4000 + it)
        x.copy_(torch.from_numpy(xs[rank]))
        comm.all_reduce_tensor(x, "premean", out=x)
        assert H(x).numpy().tobytes() == O.fold_premean(xs).tobytes(), it
    xs = _inputs(world, count, seed=4100)
    x.copy_(torch.from_numpy(xs[rank]))
    v = x[4096:4096 + (1 << 20)]
    comm.all_reduce_tensor(v, "sum", out=v)
    want = O.fold_sum([a[4096:4096 + (1 << 20)] for a in xs])
    assert H(v).numpy().tobytes() == want.tobytes()
    assert H(x[:4096]).numpy().tobytes() == xs[rank][:4096].tobytes()  # nothing outside the view
    small = x[:1000]
    assert comm.plan_for(small, "sum", out=small)[:2] == (1, 1)  # one-shot, push
    comm.all_reduce_tensor(small, "max", out=small)
    assert H(small).numpy().tobytes() == O.fold_max([a[:1000] for a in xs]).tobytes()
    comm.unregister(reg)
    assert comm.plan_for(x, "sum", out=x) == (2, 1, -1, -1)
    xs = _inputs(world, count, seed=4200)
    x.copy_(torch.from_numpy(xs[rank]))
    comm.all_reduce_tensor(x, "sum", out=x)
    assert H(x).numpy().tobytes() == O.fold_sum(xs).tobytes()
    comm.check()
    comm.close()


def body_bn(rank, world, env):
    from oracle import collectives as O
    from paper_1902_00465_b200.replicator import CrossReplicaBatchNorm, Replicator

    dev = env.dev
    repl = Replicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=16 << 20)
    shape = (4, 16, 5, 5)
    xs = [np.random.default_rng(50 + r).standard_normal(shape) * 2 + 1 for r in range(world)]
    dys = [np.random.default_rng(60 + r).standard_normal(shape) for r in range(world)]
    w = np.random.default_rng(70).standard_normal(16)
    for fmt in (torch.contiguous_format, torch.channels_last):
        bn = CrossReplicaBatchNorm(16, repl).to(dev)
        with torch.no_grad():
            bn.weight.copy_(torch.from_numpy(w))
        x = torch.from_numpy(xs[rank]).float().to(dev).contiguous(memory_format=fmt).requires_grad_(True)
        y = bn(x)
        y.backward(torch.from_numpy(dys[rank]).float().to(dev).contiguous(memory_format=fmt))
        outs, mean, var, _ = O.bn_forward_per_channel(xs, "nchw", weight=w, bias=np.zeros(16))
        np.testing.assert_allclose(H(y.detach()).numpy(), outs[rank], rtol=1e-4, atol=1e-4)
        dxs, sdy, sdyx = O.bn_backward_per_channel(xs, dys, "nchw", weight=w)
        np.testing.assert_allclose(H(x.grad).numpy(), dxs[rank], rtol=1e-4, atol=1e-4)
        # local weight/bias grads (averaged later by the wrapped optimizer)
        xr = O._channel_view(xs[rank], "nchw")
        dr = O._channel_view(dys[rank], "nchw")
        np.testing.assert_allclose(H(bn.bias.grad).numpy(), dr.sum(0), rtol=1e-5, atol=1e-4)
        np.testing.assert_allclose(H(bn.weight.grad).numpy(), (dr * (xr - mean) / np.sqrt(var + 1e-5)).sum(0),
                                   rtol=1e-4, atol=1e-4)
        np.testing.assert_allclose(H(bn.running_mean).numpy(), 0.1 * mean, rtol=1e-5, atol=1e-6)
    repl.comm.close()


def body_bn_layouts(rank, world, env):
    """CrossReplicaBatchNorm on [N, C] inputs with a broadcast
    (stride-0) upstream gradient from a plain ``(bn(x) * c).sum()`` loss, on a
    transposed [N, C] input, and on a channels_last_3d 5-D input with an NCDHW
    gradient: every case equals the f64 oracle of the concatenated batch."""
    from oracle import collectives as O
    from paper_1902_00465_b200.replicator import CrossReplicaBatchNorm, Replicator

    dev = env.dev
    repl = Replicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=16 << 20)
    C = 6
    xs = [np.random.default_rng(80 + r).standard_normal((8, C)) * 1.5 + 0.5 for r in range(world)]
    cvec = np.random.default_rng(90).standard_normal(C)
    w = np.random.default_rng(91).standard_normal(C)
    for transposed in (False, True):
        bn = CrossReplicaBatchNorm(C, repl).to(dev)
        with torch.no_grad():
            bn.weight.copy_(torch.from_numpy(w))
        xt = torch.from_numpy(xs[rank]).float().to(dev)
        if transposed:  # a non-contiguous [N, C] view of a [C, N] buffer
            xt = xt.t().contiguous().t()
            assert not xt.is_contiguous()
        x = xt.detach().requires_grad_(True)
        y = bn(x)
        (y * torch.from_numpy(cvec).float().to(dev)).sum().backward()  # dy: [C] expanded, stride (0, 1)
        outs, mean, var, _ = O.bn_forward_per_channel(xs, "nc", weight=w, bias=np.zeros(C))
        np.testing.assert_allclose(H(y.detach()).numpy(), outs[rank], rtol=1e-4, atol=1e-4)
        dys = [np.broadcast_to(cvec, (8, C)) for _ in range(world)]
        dxs, _, _ = O.bn_backward_per_channel(xs, dys, "nc", weight=w)
        np.testing.assert_allclose(H(x.grad).numpy(), dxs[rank], rtol=1e-4, atol=1e-4)
    # 5-D channels_last_3d input, contiguous (NCDHW) upstream gradient
    shape = (2, 4, 3, 3, 3)
    x5 = [np.random.default_rng(95 + r).standard_normal(shape) for r in range(world)]
    d5 = [np.random.default_rng(97 + r).standard_normal(shape) for r in range(world)]
    bn = CrossReplicaBatchNorm(4, repl).to(dev)
    x = torch.from_numpy(x5[rank]).float().to(dev).contiguous(memory_format=torch.channels_last_3d)
    x.requires_grad_(True)
    y = bn(x)
    y.backward(torch.from_numpy(d5[rank]).float().to(dev))
    outs, *_ = O.bn_forward_per_channel(x5, "nchw", weight=np.ones(4), bias=np.zeros(4))
    np.testing.assert_allclose(H(y.detach()).numpy(), outs[rank], rtol=1e-4, atol=1e-4)
    dxs, _, _ = O.bn_backward_per_channel(x5, d5, "nchw", weight=np.ones(4))
    np.testing.assert_allclose(H(x.grad).numpy(), dxs[rank], rtol=1e-4, atol=1e-4)
    repl.comm.check()
    repl.comm.close()


def body_autograd(rank, world, env):
    """differentiating through the multi-rank collectives gives
    their adjoints -- all_sum's is all_sum (mean's scaled by 1/N), all_gather's a
    reduce-scatter, broadcast's the sum of every rank's cotangent on the root and
    zero elsewhere -- and max raises NotDifferentiableError (graph.py:798-800)."""
    from paper_1902_00465_b200 import errors
    from paper_1902_00465_b200.replicator import Replicator

    dev = env.dev
    repl = Replicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=16 << 20)
    n = 5
    x0 = np.random.default_rng(300 + rank).standard_normal(n)
    ws = [np.random.default_rng(310 + q).standard_normal(n) for q in range(world)]
    wsum = np.sum(ws, axis=0)
    for kind, scale in (("sum", 1.0), ("mean", 1.0 / world), ("premean", 1.0 / world)):
        x = torch.from_numpy(x0).to(dev).requires_grad_(True)
        (repl.all_reduce(x, kind) * torch.from_numpy(ws[rank]).to(dev)).sum().backward()
        np.testing.assert_allclose(H(x.grad).numpy(), wsum * scale, rtol=1e-12, atol=1e-12)
    Ws = [np.random.default_rng(320 + q).standard_normal((world, n)) for q in range(world)]
    x = torch.from_numpy(x0).to(dev).requires_grad_(True)
    g = repl.all_gather(x, stack=True)
    assert g.shape == (world, n)
    (g * torch.from_numpy(Ws[rank]).to(dev)).sum().backward()
    np.testing.assert_allclose(H(x.grad).numpy(), sum(W[rank] for W in Ws), rtol=1e-12, atol=1e-12)
    root = world - 1
    x = torch.from_numpy(x0).to(dev).requires_grad_(True)
    y = repl.broadcast(x, root=root)
    xr = np.random.default_rng(300 + root).standard_normal(n)
    np.testing.assert_array_equal(H(y.detach()).numpy(), xr)
    (y * torch.from_numpy(ws[rank]).to(dev)).sum().backward()
    np.testing.assert_allclose(H(x.grad).numpy(), wsum if rank == root else np.zeros(n), rtol=1e-12, atol=1e-12)
    x = torch.from_numpy(x0).to(dev).requires_grad_(True)
    y = repl.all_reduce(x, "max")
    with pytest.raises(errors.NotDifferentiableError):
        y.sum().backward()
    repl.comm.check()
    repl.comm.close()


def body_wrap_optimizer(rank, world, env):
    from paper_1902_00465_b200.replicator import Replicator

    dev = env.dev
    repl = Replicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=32 << 20)
    torch.manual_seed(rank)  # deliberately different init: replicate() must broadcast replica 0
    with repl.context():
        model = repl.replicate(lambda: torch.nn.Sequential(torch.nn.Linear(784, 256), torch.nn.ReLU(),
                                                           torch.nn.Linear(256, 10)).double())
        opt = repl.wrap_optimizer(torch.optim.SGD(model.parameters(), lr=0.1))
    # single-device oracle: the same model trained on the concatenated batch
    torch.manual_seed(0)
    ref = torch.nn.Sequential(torch.nn.Linear(784, 256), torch.nn.ReLU(), torch.nn.Linear(256, 10)).double().to(dev)
    with torch.no_grad():
        for p, q in zip(ref.parameters(), model.local.parameters()):
            p.copy_(q)
    ref_opt = torch.optim.SGD(ref.parameters(), lr=0.1)
    B = 16
    for step in range(5):
        g = torch.Generator().manual_seed(step)
        xs = torch.randn(world * B, 784, generator=g, dtype=torch.float64).to(dev)
        ys = torch.randint(0, 10, (world * B,), generator=g).to(dev)
        opt.zero_grad()
        loss = torch.nn.functional.cross_entropy(model(xs[rank * B:(rank + 1) * B]), ys[rank * B:(rank + 1) * B])
        loss.backward()
        opt.step()
        ref_opt.zero_grad()
        torch.nn.functional.cross_entropy(ref(xs), ys).backward()
        ref_opt.step()
    for p, q in zip(model.local.parameters(), ref.parameters()):
        assert H((p - q).abs().max()).item() < 1e-9  # SPEC.md:399 sync-equivalence bound
    # a channels_last conv model: replicate() must sync every replica in place
    torch.manual_seed(100 + rank)
    conv = repl.replicate(lambda: torch.nn.Sequential(torch.nn.Conv2d(3, 8, 3), torch.nn.BatchNorm2d(8))
                          .to(memory_format=torch.channels_last))
    cflat = torch.cat([q.detach().contiguous().reshape(-1) for q in conv.local.parameters()])
    cg = repl.comm.all_gather_tensor(cflat)
    assert all(EQ(cg[r], cg[0]) for r in range(world)), "replicate() left channels_last replicas apart"
    # replicas bit-identical
    flat = torch.cat([p.detach().reshape(-1) for p in model.local.parameters()])
    g = repl.comm.all_gather_tensor(flat)
    for r in range(world):
        assert EQ(g[r], g[0])
    repl.comm.close()


def body_nvls(rank, world, env):
    """In-switch all-reduce (multimem.ld_reduce / multimem.st). Not rank-ordered,
    so checked against the f64 sum with a stated tolerance (north star: <=1e-6
    relative, ordering-induced), plus bit-identical results on every rank."""
    from paper_1902_00465_b200.comm import Communicator

    comm = Communicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=128 << 20)
    comm.enable_nvls(96 << 20)
    for count in (4, 1000, 4099, 1 << 20, 12 << 20):
        xs = _inputs(world, count, seed=500 + count)
        buf = comm.alloc_nvls(count, torch.float32)
        for kind in ("sum", "mean", "premean"):
            buf.copy_(torch.from_numpy(xs[rank]))
            comm.all_reduce_tensor(buf, kind, out=buf, algo="nvls")
            got = H(buf).numpy().astype(np.float64)
            want = np.sum(np.stack(xs).astype(np.float64), axis=0) / (1 if kind == "sum" else world)
            err = np.linalg.norm(got - want) / np.linalg.norm(want)
            assert err <= 1e-6, (count, kind, err)
            g = comm.all_gather_tensor(buf)
            assert all(EQ(g[r], g[0]) for r in range(world))
        xb = [x.astype(np.float32) for x in _inputs(world, 50000, seed=9)]
        bb = comm.alloc_nvls(50000, torch.bfloat16)
        bb.copy_(torch.from_numpy(xb[rank]).to(torch.bfloat16))
        comm.all_reduce_tensor(bb, "sum", out=bb, algo="nvls")
        ref = sum(torch.from_numpy(x).to(torch.bfloat16).double() for x in xb)
        rel = (H(bb.double()) - ref).norm() / ref.norm()
        assert rel < 4e-3, rel  # one bf16 rounding of an f32-accumulated sum
    # automatic choice (rp_resolve_ar_algo): in-place >= 512 KiB buffers in the
    # region reduce in the switch from 4 ranks on; anything else stays P2P
    big = comm.alloc_nvls(1 << 20, torch.float32)
    small = comm.alloc_nvls(1000, torch.float32)
    pool_buf = comm.alloc(1 << 20, torch.float32)
    assert comm.algorithm_for(big, "mean", out=big) == ("nvls" if world >= 4 else "twoshot")
    assert comm.algorithm_for(small, "mean", out=small) == "oneshot"
    assert comm.algorithm_for(pool_buf, "mean", out=pool_buf) == "twoshot"
    assert comm.algorithm_for(big, "max", out=big) == "twoshot"  # the switch has no ordered max here
    os.environ["RP_NVLS"] = "0"
    assert comm.algorithm_for(big, "mean", out=big) == "twoshot"
    del os.environ["RP_NVLS"]
    xs = _inputs(world, 1 << 20, seed=77)
    big.copy_(torch.from_numpy(xs[rank]))
    comm.all_reduce_tensor(big, "premean", out=big)
    want = np.sum(np.stack(xs).astype(np.float64), axis=0) / world
    got = H(big).numpy().astype(np.float64)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-6
    # NVLS broadcast (rp.h RP_ALGO_NVLS for rp_broadcast): destination in the region,
    # the root multicasts from any local source (in place, separate, misaligned); bit-exact
    dev = env.dev
    for nbytes in (16, 4096, (1 << 20) + 48, 7 << 20):
        for root in (0, world - 1):
            want = torch.from_numpy(np.random.default_rng(nbytes + root).integers(0, 256, nbytes + 1, dtype=np.uint8))
            dst = comm.alloc_nvls(nbytes, torch.uint8)
            dst.fill_(rank + 1)
            src = want.to(dev)
            for mode in ("in_place", "separate", "misaligned"):
                if mode == "in_place":
                    if rank == root:
                        dst.copy_(src[:nbytes])
                    comm.broadcast_tensor(dst, root=root)
                else:
                    s0 = src[:nbytes] if mode == "separate" else src[1:nbytes + 1]
                    comm.broadcast_tensor(s0, root=root, out=dst)
                exp = want[:nbytes] if mode != "misaligned" else want[1:nbytes + 1]
                assert EQ(dst, exp), (nbytes, root, mode)
                dst.fill_(rank + 7)
    comm.check()
    comm.close()


def body_wrap_nvls(rank, world, env):
    """wrap_optimizer with fusion buckets in the NVLS region (Replicator(nvls_bytes)):
    the same training as the single-device oracle on the concatenated batch, within
    the f32 ordering tolerance, and replicas stay bit-identical (the multicast store
    writes one value to every rank)."""
    from paper_1902_00465_b200.replicator import Replicator

    dev = env.dev
    repl = Replicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=32 << 20, nvls_bytes=16 << 20)
    torch.manual_seed(rank)
    with repl.context():
        model = repl.replicate(lambda: torch.nn.Sequential(torch.nn.Linear(784, 256), torch.nn.ReLU(),
                                                           torch.nn.Linear(256, 10)))
        opt = repl.wrap_optimizer(torch.optim.SGD(model.parameters(), lr=0.1))
    torch.manual_seed(0)
    ref = torch.nn.Sequential(torch.nn.Linear(784, 256), torch.nn.ReLU(), torch.nn.Linear(256, 10)).double().to(dev)
    with torch.no_grad():
        for p, q in zip(ref.parameters(), model.local.parameters()):
            p.copy_(q.double())
    ref_opt = torch.optim.SGD(ref.parameters(), lr=0.1)
    B = 16
    for step in range(3):
        g = torch.Generator().manual_seed(step)
        xs = torch.randn(world * B, 784, generator=g).to(dev)
        ys = torch.randint(0, 10, (world * B,), generator=g).to(dev)
        opt.zero_grad()
        torch.nn.functional.cross_entropy(model(xs[rank * B:(rank + 1) * B]), ys[rank * B:(rank + 1) * B]).backward()
        opt.step()
        ref_opt.zero_grad()
        torch.nn.functional.cross_entropy(ref(xs.double()), ys).backward()
        ref_opt.step()
    bk = opt._buckets.buckets[0]
    algo = repl.comm.algorithm_for(bk.flat[0], "premean", out=bk.flat[0])
    assert algo == "nvls" if world >= 4 else algo in ("oneshot", "twoshot")
    for p, q in zip(model.local.parameters(), ref.parameters()):
        assert H((p.double() - q).abs().max()).item() < 1e-5
    flat = torch.cat([p.detach().reshape(-1) for p in model.local.parameters()])
    gathered = repl.comm.all_gather_tensor(flat)
    assert all(EQ(gathered[r], gathered[0]) for r in range(world))
    repl.comm.close()


def body_fused_apply(rank, world, env):
    """wrap_optimizer(Adam, fused=True) over real ranks: each step equals torch's
    Adam driven by the rank-ordered averaged gradient (gathered and folded by the
    oracle), replicas stay bit-identical, and the whole training step (forward,
    backward, fused apply) replays from a CUDA graph."""
    from oracle import collectives as O
    from paper_1902_00465_b200.replicator import Replicator

    dev = env.dev
    repl = Replicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=32 << 20)
    torch.manual_seed(rank)
    with repl.context():
        model = repl.replicate(lambda: torch.nn.Sequential(torch.nn.Linear(784, 256), torch.nn.ReLU(),
                                                           torch.nn.Linear(256, 10)))
        opt = repl.wrap_optimizer(torch.optim.Adam(model.parameters(), lr=1e-3, weight_decay=1e-4), fused=True)
    ref = torch.nn.Sequential(torch.nn.Linear(784, 256), torch.nn.ReLU(), torch.nn.Linear(256, 10)).to(dev)
    with torch.no_grad():
        for p, q in zip(ref.parameters(), model.local.parameters()):
            p.copy_(q)
    ref_opt = torch.optim.Adam(ref.parameters(), lr=1e-3, weight_decay=1e-4)
    B = 16
    for step in range(3):
        g = torch.Generator().manual_seed(step)
        xs = torch.randn(world * B, 784, generator=g).to(dev)
        ys = torch.randint(0, 10, (world * B,), generator=g).to(dev)
        opt.zero_grad()
        torch.nn.functional.cross_entropy(model(xs[rank * B:(rank + 1) * B]), ys[rank * B:(rank + 1) * B]).backward()
        flat = torch.cat([p.grad.reshape(-1) for p in model.local.parameters()])
        every = H(repl.comm.all_gather_tensor(flat)).numpy()
        avg = torch.from_numpy(O.fold_premean([every[r] for r in range(world)])).to(dev)
        o = 0
        for p in ref.parameters():
            p.grad = avg[o:o + p.numel()].view_as(p).clone()
            o += p.numel()
        opt.step()
        ref_opt.step()
    for p, q in zip(model.local.parameters(), ref.parameters()):
        assert torch.allclose(H(p), H(q), rtol=2e-6, atol=2e-7), H((p - q).abs().max()).item()
    flat = torch.cat([p.detach().reshape(-1) for p in model.local.parameters()])
    gathered = repl.comm.all_gather_tensor(flat)
    assert all(EQ(gathered[r], gathered[0]) for r in range(world))
    # the whole step in a CUDA graph (device-side step counter and sequencing state)
    x = torch.randn(B, 784, device=dev, generator=torch.Generator(device=dev).manual_seed(50 + rank))
    y = torch.randint(0, 10, (B,), device=dev, generator=torch.Generator(device=dev).manual_seed(60 + rank))

    def train_step():
        opt.zero_grad()
        torch.nn.functional.cross_entropy(model(x), y).backward()
        opt.step()

    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        train_step()
    torch.cuda.current_stream(dev).wait_stream(side)
    env.sync()
    env.barrier()  # graph capture synchronises the device: nobody may wait on a peer's next launch
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, capture_error_mode="thread_local"):
        train_step()
    env.barrier()  # nobody replays (real launches) while a peer is still inside capture's device sync
    before = flat.clone()
    for _ in range(3):
        graph.replay()
    env.sync()
    repl.comm.check()
    assert int(H(opt.groups[0].steps[0]).item()) == 3 + 1 + 3
    flat = torch.cat([p.detach().reshape(-1) for p in model.local.parameters()])
    assert not EQ(flat, before)
    gathered = repl.comm.all_gather_tensor(flat)
    assert all(EQ(gathered[r], gathered[0]) for r in range(world))
    repl.comm.close()


def body_protocol(rank, world, env):
    """Replicator(check_protocol=True): mismatched shapes or
    order raise ProtocolError on EVERY rank, naming what each issued; a label reused
    within a generation is rejected, across generations it is fine; the reference
    duck type's all_gather accepts differing leading dimensions."""
    from paper_1902_00465_b200 import errors
    from paper_1902_00465_b200.replicator import Replicator

    dev = env.dev
    repl = Replicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=16 << 20, check_protocol=True)
    x = torch.full((4,), float(rank + 1), device=dev)
    assert H(repl.all_sum(x, label="a")).tolist() == [float(sum(range(1, world + 1)))] * 4
    try:
        repl.all_sum(x, label="a")  # same label, same generation
        raise AssertionError("label reuse was accepted")
    except errors.ProtocolError:
        pass
    repl.new_generation()
    repl.all_sum(x, label="a")  # next generation: fine
    y = torch.zeros(3 + (rank == world - 1), device=dev)  # the last rank disagrees on the shape
    try:
        repl.all_sum(y, label="b")
        raise AssertionError("shape disagreement was accepted")
    except errors.ProtocolError as e:
        assert "issued" in str(e) and f"rank {rank}" in str(e), str(e)
    repl.new_generation()
    # placement disagreement: rank 0 passes a pool view, the others a
    # plain tensor -- different kernels against shared barrier state; caught by the
    # plan digest (include/rp.h rp_all_reduce_plan) before anything launches
    pooled = repl.comm.alloc(16, torch.float32)
    z = pooled if rank == 0 else torch.zeros(16, device=dev)
    with pytest.raises(errors.ProtocolError):
        repl.all_sum(z, label="placed")
    repl.new_generation()
    # the duck type (graph.py:575-579) with ragged leading dimensions; scalars stay scalars
    rows = torch.arange((rank + 1) * 3, dtype=torch.float32, device=dev).reshape(rank + 1, 3)
    got = repl.comm.all_gather(rows)
    assert [tuple(t.shape) for t in got] == [(r + 1, 3) for r in range(world)]
    assert all(EQ(got[r], torch.arange((r + 1) * 3, dtype=torch.float32, device=dev).reshape(r + 1, 3))
               for r in range(world))
    sc = repl.comm.all_gather(np.float64(rank))
    assert [float(np.asarray(v)) for v in sc] == [float(r) for r in range(world)]
    # SPEC.md:223-231 across processes: map_gather / map_reduce deliver to the driver,
    # readable only outside the replicated step; the list form of all_gather
    repl.new_generation()

    def step(_):
        rows_r = torch.full((rank + 1, 2), float(rank), device=dev)
        mg = repl.map_gather(rows_r, label="mg")
        mr = repl.map_reduce(torch.tensor([float(rank + 1)], device=dev), "sum", label="mr")
        with pytest.raises(errors.EvaluationError):
            mg.value  # noqa: B018 -- reading inside the step is the SPEC's error
        lst = repl.all_gather(torch.tensor(float(rank), device=dev), label="lst")
        return mg, mr, lst
    (mg, mr, lst), = repl.run(step, lambda r: None)
    assert [tuple(t.shape) for t in mg.value] == [(r + 1, 2) for r in range(world)]
    assert all(EQ(t, torch.full((r + 1, 2), float(r), device=dev)) for r, t in enumerate(mg.value))
    assert float(H(mr.value)[0]) == float(sum(range(1, world + 1)))
    assert isinstance(lst, list) and [float(H(t)) for t in lst] == [float(r) for r in range(world)]
    repl.comm.check()
    repl.comm.close()


def body_graph(rank, world, env):
    """Each rank captures the same sequence of collectives in a CUDA graph and
    replays it; device-side sequencing keeps the ranks in step across replays."""
    from oracle import collectives as O
    from paper_1902_00465_b200.comm import Communicator

    dev = env.dev
    comm = Communicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=64 << 20)
    small = torch.empty(5000, device=dev)
    big = torch.empty(3 << 20, device=dev)
    bucket = comm.alloc(1 << 20, torch.float32)
    o_small, o_big = torch.empty_like(small), torch.empty_like(big)

    def seq():
        comm.all_reduce_tensor(small, "sum", out=o_small)           # one-shot push
        comm.all_reduce_tensor(big, "premean", out=o_big)           # two-shot push (staged)
        comm.all_reduce_tensor(bucket, "premean", out=bucket)       # two-shot pull (pool, in place)

    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        seq()
    torch.cuda.current_stream(dev).wait_stream(s)
    env.sync()
    env.barrier()  # graph capture synchronises the device: nobody may wait on a peer's next launch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="thread_local"):
        seq()
    env.barrier()  # nobody replays (real launches) while a peer is still inside capture's device sync
    for it in range(5):
        xs_s = _inputs(world, 5000, seed=1000 + it)
        xs_b = _inputs(world, 3 << 20, seed=2000 + it)
        xs_k = _inputs(world, 1 << 20, seed=3000 + it)
        small.copy_(torch.from_numpy(xs_s[rank]))
        big.copy_(torch.from_numpy(xs_b[rank]))
        bucket.copy_(torch.from_numpy(xs_k[rank]))
        g.replay()
        env.sync()
        assert H(o_small).numpy().tobytes() == O.fold_sum(xs_s).tobytes(), it
        assert H(o_big).numpy().tobytes() == O.fold_premean(xs_b).tobytes(), it
        assert H(bucket).numpy().tobytes() == O.fold_premean(xs_k).tobytes(), it
    comm.check()
    comm.close()


def body_timeout(rank, world, env):
    """A rank that never joins makes the others time out (not hang) and report
    CollectiveAbortedError (SPEC.md:237 liveness; errors.py:68)."""
    from paper_1902_00465_b200 import errors
    from paper_1902_00465_b200.comm import Communicator

    comm = Communicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=16 << 20, timeout_s=2.0)
    x = torch.ones(1024, device=env.dev)
    if rank != world - 1:
        comm.all_reduce_tensor(x, "sum")
        with pytest.raises(errors.CollectiveAbortedError):
            comm.check()
    env.barrier()
    comm.close()


def body_overlap(rank, world, env):
    """wrap_optimizer(overlap=True): buckets exchanged from post-accumulate-grad
    hooks on a side stream during backward must give the SAME bits as the
    synchronous wrapped optimizer (same premean fold per element), including with
    a bf16 exchange, unused parameters and no_sync() gradient accumulation."""
    from paper_1902_00465_b200 import errors
    from paper_1902_00465_b200.replicator import Replicator

    dev = env.dev

    def net():
        return torch.nn.Sequential(torch.nn.Conv2d(3, 16, 3, padding=1), torch.nn.ReLU(),
                                   torch.nn.Conv2d(16, 32, 3, padding=1), torch.nn.ReLU(),
                                   torch.nn.AdaptiveAvgPool2d(1), torch.nn.Flatten(), torch.nn.Linear(32, 10))

    for comm_dt in (None, torch.bfloat16):
        results = []
        for overlap, views in ((False, False), (False, True), (True, True)):
            repl = Replicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=32 << 20, grad_comm_dtype=comm_dt, grad_views=views,
                              bucket_bytes=256 if overlap else None)
            torch.manual_seed(rank)
            with repl.context():
                model = repl.replicate(lambda: net().to(memory_format=torch.channels_last))
                unused = repl.replicate(lambda: torch.nn.Linear(4, 4))  # never receives a gradient
                params = list(unused.local.parameters()) + list(model.local.parameters())  # unused -> last bucket
                opt = repl.wrap_optimizer(torch.optim.SGD(params, lr=0.05, momentum=0.9), overlap=overlap)
            if overlap:
                assert len(opt.buckets) > 3, ("small bucket_bytes must give several buckets",
                                              [b.counts for b in opt.buckets], repl.bucket_bytes)
                assert all(p.grad is not None and b.views for b in opt.buckets for p in b.params[0])
            for step in range(4):
                g = torch.Generator().manual_seed(10 * step + rank)
                opt.zero_grad(set_to_none=(step % 2 == 1))
                micro = 2 if step == 3 else 1
                for m in range(micro):
                    xb = torch.randn(8, 3, 12, 12, generator=g).to(dev).contiguous(memory_format=torch.channels_last)
                    yb = torch.randint(0, 10, (8,), generator=g).to(dev)
                    ctx = opt.no_sync() if (overlap and m < micro - 1) else _nullcontext()
                    with ctx:
                        torch.nn.functional.cross_entropy(model.local(xb), yb).backward()
                opt.step()
            env.sync()
            results.append([p.detach().clone() for p in params])
            if overlap:  # accumulating twice without no_sync is refused
                opt.zero_grad()
                xb = torch.randn(8, 3, 12, 12, device=dev).contiguous(memory_format=torch.channels_last)
                torch.nn.functional.cross_entropy(model.local(xb), torch.zeros(8, dtype=torch.long, device=dev)) \
                    .backward()
                with pytest.raises(Exception) as ei:
                    torch.nn.functional.cross_entropy(model.local(xb), torch.zeros(8, dtype=torch.long,
                                                                                   device=dev)).backward()
                assert "no_sync" in str(ei.value) or isinstance(ei.value, errors.ProtocolError)
                opt.remove_hooks()
            repl.comm.close()
        for other, what in ((results[1], "gradient views"), (results[2], "overlap")):
            for a, b in zip(results[0], other):
                assert EQ(a, b), f"{what} differs from the packed synchronous exchange ({comm_dt})"
        flat = torch.cat([p.reshape(-1) for p in results[2]])
        gl = env.all_gather_object(H(flat))
        assert all(EQ(t, gl[0]) for t in gl), "replicas diverged"


def body_overlap_with_bn(rank, world, env):
    """with overlap=True, bucket all-reduces run on a side stream
    while backward issues its OWN collectives on the compute stream (the BN
    backward exchange of CrossReplicaBatchNorm). Every kernel of a communicator
    shares its device-side sequencing state, so they must not run concurrently:
    Communicator._stream orders each launch after the previous one whatever the
    stream. The overlapped run must give the same bits as the synchronous one."""
    from paper_1902_00465_b200.replicator import CrossReplicaBatchNorm, Replicator

    dev = env.dev
    results = []
    for overlap in (False, True):
        repl = Replicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=32 << 20,
                          bucket_bytes=2048 if overlap else None)

        def net():
            return torch.nn.Sequential(torch.nn.Conv2d(3, 16, 3, padding=1), CrossReplicaBatchNorm(16, repl),
                                       torch.nn.ReLU(), torch.nn.Conv2d(16, 16, 3, padding=1),
                                       CrossReplicaBatchNorm(16, repl), torch.nn.ReLU(),
                                       torch.nn.AdaptiveAvgPool2d(1), torch.nn.Flatten(), torch.nn.Linear(16, 10))

        torch.manual_seed(rank)
        with repl.context():
            model = repl.replicate(lambda: net().to(memory_format=torch.channels_last))
            opt = repl.wrap_optimizer(torch.optim.SGD(model.local.parameters(), lr=0.05), overlap=overlap)
        if overlap:
            assert len(opt.buckets) > 2
        for step in range(3):
            g = torch.Generator().manual_seed(100 * step + rank)
            xb = torch.randn(8, 3, 10, 10, generator=g).to(dev).contiguous(memory_format=torch.channels_last)
            yb = torch.randint(0, 10, (8,), generator=g).to(dev)
            opt.zero_grad()
            torch.nn.functional.cross_entropy(model.local(xb), yb).backward()
            opt.step()
        env.sync()
        results.append([H(p.detach()) for p in model.local.parameters()])
        if overlap:
            opt.remove_hooks()
        repl.comm.check()
        repl.comm.close()
    for a, b in zip(*results):
        assert torch.equal(a, b), "overlapped exchange beside BN collectives differs from the synchronous one"


def body_host_pipeline(rank, world, env):
    """Communicator.all_reduce_host: pinned host in, pinned host out, chunked through
    pool slots (many chunks, ragged tail, ring reuse); bit-exact vs the oracle fold,
    and with NVLS slots within the ordering tolerance."""
    from oracle import collectives as O
    from paper_1902_00465_b200.comm import Communicator

    comm = Communicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=64 << 20)
    count = 5 * 8192 + 77
    xs = _inputs(world, count, seed=321)
    hin = torch.from_numpy(xs[rank]).pin_memory()
    for kind, fold in (("sum", O.fold_sum), ("premean", O.fold_premean)):
        for _ in range(2):
            out = comm.all_reduce_host(hin, kind, chunk_bytes=8192 * 4)
            assert out.numpy().tobytes() == fold(xs).tobytes(), kind
    if env.loopback:  # NVLS spans distinct devices
        comm.check()
        comm.close()
        return
    comm.enable_nvls(16 << 20)
    out = comm.all_reduce_host(hin, "sum", chunk_bytes=1 << 20, nvls=True)
    want = np.sum(np.stack(xs).astype(np.float64), axis=0)
    assert np.linalg.norm(out.numpy() - want) / np.linalg.norm(want) <= 1e-6
    comm.check()
    comm.close()


def body_relay_broadcast(rank, world, env):
    """Pipelined relay broadcast (K4r): bit-exact for every root, landing in staging
    (user dst, aligned or not) or straight in a pool-resident dst, many tiles,
    repeated calls (per-tile epoch flags are never reset)."""
    from paper_1902_00465_b200.comm import Communicator

    dev = env.dev
    comm = Communicator(device=env.device, bootstrap=env.bootstrap, pool_bytes=96 << 20)
    for nbytes in (16, (1 << 20) + 16, (9 << 20) + 4096):
        want = {r: np.random.default_rng(nbytes + r).integers(0, 256, nbytes + 1, dtype=np.uint8)
                for r in range(world)}
        pool_dst = comm.alloc(nbytes, torch.uint8)
        for root in range(world):
            src = torch.from_numpy(want[root]).to(dev)
            for mode in ("user", "misaligned", "pool", "pool_in_place"):
                if mode == "user":
                    out = torch.full((nbytes,), rank + 1, dtype=torch.uint8, device=dev)
                    comm.broadcast_tensor(src[:nbytes], root=root, out=out, algo="relay")
                elif mode == "misaligned":
                    big = torch.full((nbytes + 1,), rank + 1, dtype=torch.uint8, device=dev)
                    out = big[1:]
                    comm.broadcast_tensor(src[:nbytes], root=root, out=out, algo="relay")
                elif mode == "pool":
                    out = pool_dst
                    out.fill_(rank + 3)
                    comm.broadcast_tensor(src[:nbytes], root=root, out=out, algo="relay")
                else:
                    out = pool_dst
                    out.fill_(rank + 5)
                    if rank == root:
                        out.copy_(src[:nbytes])
                    comm.broadcast_tensor(out, root=root, algo="relay")
                assert np.array_equal(H(out).numpy(), want[root][:nbytes]), (nbytes, root, mode)
    comm.check()
    comm.close()




def _nullcontext():
    import contextlib
    return contextlib.nullcontext()
