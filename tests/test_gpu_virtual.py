"""GPU parity on ONE B200: the P2P collective kernels run over R replicas resident on
one device (VirtualCommunicator -> one cooperative launch, the same device code the
multi-process path runs) and are compared with the reference fixtures and the CPU
oracle. Bit-exact for folds, gathers and broadcasts; BN statistics within 1e-6."""

import ctypes
import json
import os

import numpy as np
import pytest
import torch

from oracle import collectives as O
from tests.helpers import GOLDEN, fold_cases

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1902_00465_b200 import _lib, errors  # noqa: E402
from paper_1902_00465_b200.comm import VirtualCommunicator  # noqa: E402
from paper_1902_00465_b200.replicator import CrossReplicaBatchNorm, PerReplica, Replicator  # noqa: E402

DEV = torch.device("cuda:0")
_COMMS = {}


def vcomm(n, pool=64 << 20):
    key = (n, pool)
    if key not in _COMMS:
        _COMMS[key] = VirtualCommunicator(n, device=0, pool_bytes=pool)
    return _COMMS[key]


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


NP_TORCH = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}


@pytest.fixture(params=["pull", "push"])
def impl(request, monkeypatch):
    """Both data-movement forms of the all-reduce kernels: pull (K1/K2, the virtual
    default) and push (K1p/K2p, the multi-process default), selected by RP_AR_IMPL."""
    monkeypatch.setenv("RP_AR_IMPL", request.param)
    return request.param


# --- all_reduce vs the reference's stitched folds ---------------------------

@pytest.mark.parametrize("algo", ["oneshot", "twoshot", "flat"])
@pytest.mark.parametrize("kind", ["sum", "mean", "max", "premean"])
def test_all_reduce_matches_reference_folds(folds, algo, kind, impl):
    for key, dtype, n, shape in fold_cases(folds):
        xs = [to_dev(folds[f"{key}_in{r}"]).reshape(-1) for r in range(n)]
        want = folds[f"{key}_{kind}"]
        outs = vcomm(n).all_reduce(xs, kind, algo=algo)
        for r in range(n):
            got = host(outs[r]).reshape(want.shape)
            assert got.tobytes() == want.tobytes(), f"{key} {kind} {algo} replica {r}"
        vcomm(n).check()


def test_all_gather_and_broadcast_match_reference(folds):
    for key, dtype, n, shape in fold_cases(folds):
        xs = [to_dev(folds[f"{key}_in{r}"]).reshape(-1) for r in range(n)]
        outs = vcomm(n).all_gather(xs)
        want = folds[f"{key}_gather"]
        for r in range(n):
            assert host(outs[r]).tobytes() == want.tobytes(), key
        for algo in ("direct", "scatter"):
            bs = vcomm(n).broadcast(xs, root=0, algo=algo)
            for r in range(n):
                assert host(bs[r]).tobytes() == folds[f"{key}_broadcast"].tobytes(), (key, algo)


# --- sizes, tails, alignment ---------------------------------------------------

@pytest.mark.parametrize("n", [2, 3, 4, 8])
@pytest.mark.parametrize("count", [1, 3, 5, 127, 1000, 4097, 65537, 1 << 20])
def test_all_reduce_sizes_f32(n, count, impl):
    rng = np.random.default_rng(count * 10 + n)
    xs_np = [rng.standard_normal(count).astype(np.float32) for _ in range(n)]
    for kind in ("sum", "premean", "max"):
        want = O.FOLDS[kind](xs_np)
        for algo in ("oneshot", "twoshot", "flat"):
            outs = vcomm(n).all_reduce([to_dev(x) for x in xs_np], kind, algo=algo)
            for o in outs:
                assert host(o).tobytes() == want.tobytes(), (kind, algo)


def test_all_reduce_misaligned_views(impl):
    n = 4
    rng = np.random.default_rng(9)
    base = [to_dev(rng.standard_normal(10001).astype(np.float32)) for _ in range(n)]
    xs = [b[1:] for b in base]  # 4-byte offset: not 16-byte aligned
    want = O.fold_sum([host(x) for x in xs])
    outs_base = [torch.zeros(10003, device=DEV) for _ in range(n)]
    outs = [o[3:10003] for o in outs_base]
    for algo in ("oneshot", "twoshot", "flat"):
        vcomm(n).all_reduce(xs, "sum", outs=outs, algo=algo)
        for o in outs:
            assert host(o).tobytes() == want.tobytes()
        for ob in outs_base:  # nothing written outside the view
            assert host(ob[:3]).tobytes() == np.zeros(3, np.float32).tobytes()


def test_all_reduce_large_f32_premean_8_replicas(impl):
    # 64 MiB per replica, the north-star message size
    n, count = 8, 16 << 20
    gens = [torch.Generator(device=DEV).manual_seed(1234 + r) for r in range(n)]
    xs = [torch.randn(count, device=DEV, generator=g) for g in gens]
    comm = vcomm(n, pool=256 << 20)
    want = O.fold_premean([host(x) for x in xs])
    for algo in ("auto", "twoshot"):
        outs = comm.all_reduce(xs, "premean", algo=algo)
        for o in outs:
            assert host(o).tobytes() == want.tobytes(), algo
    # the bench's form: in place in the pool, the flat kernel AUTO picks
    assert comm.algorithm_for(xs[0], "premean") == "flat"
    bufs = comm.alloc(count, torch.float32)
    for b, x in zip(bufs, xs):
        b.copy_(x)
    comm.all_reduce(bufs, "premean", outs=bufs)
    for b in bufs:
        assert host(b).tobytes() == want.tobytes()


def test_staged_in_pieces_when_pool_small(impl):
    n, count = 4, 12 << 20  # 48 MiB per replica through a 16 MiB pool
    comm = VirtualCommunicator(n, device=0, pool_bytes=16 << 20)
    rng = np.random.default_rng(11)
    xs_np = [rng.standard_normal(count).astype(np.float32) for _ in range(n)]
    for algo in ("oneshot", "twoshot", "flat"):
        outs = comm.all_reduce([to_dev(x) for x in xs_np], "sum", algo=algo)
        want = O.fold_sum(xs_np)
        for o in outs:
            assert host(o).tobytes() == want.tobytes()
    comm.close()


# --- bf16 / f16 and the fused exchange cast --------------------------------------

@pytest.mark.parametrize("n", [2, 4, 8])
def test_bf16_all_reduce_matches_oracle(n, impl):
    rng = np.random.default_rng(20 + n)
    bits = [O.f32_to_bf16_bits(rng.standard_normal(50001).astype(np.float32)) for _ in range(n)]
    xs = [to_dev(b.view(np.int16)).view(torch.bfloat16) for b in bits]
    for kind in ("sum", "mean", "premean", "max"):
        want = O.fold_bf16(bits, kind)
        for algo in ("oneshot", "twoshot", "flat"):
            outs = vcomm(n).all_reduce(xs, kind, algo=algo)
            for o in outs:
                got = host(o.view(torch.int16)).view(np.uint16)
                assert np.array_equal(got, want), (kind, algo)


def test_f32_grads_exchanged_as_bf16(impl):
    n = 4
    rng = np.random.default_rng(31)
    xs_np = [rng.standard_normal(30011).astype(np.float32) for _ in range(n)]
    want = O.bf16_bits_to_f32(O.fold_bf16([O.f32_to_bf16_bits(x) for x in xs_np], "premean"))
    for algo in ("oneshot", "twoshot", "flat"):  # flat: the cast fused on load and on store
        outs = vcomm(n).all_reduce([to_dev(x) for x in xs_np], "premean", comm_dtype=torch.bfloat16, algo=algo)
        for o in outs:
            assert o.dtype == torch.float32
            assert host(o).tobytes() == want.tobytes()


def test_f16_all_reduce():
    n = 2
    rng = np.random.default_rng(32)
    xs_np = [rng.standard_normal(4099).astype(np.float16) for _ in range(n)]
    want = (xs_np[0].astype(np.float32) + xs_np[1].astype(np.float32)).astype(np.float16)
    outs = vcomm(n).all_reduce([to_dev(x) for x in xs_np], "sum")
    assert np.array_equal(host(outs[0]), want)


# --- zero-copy pool buffers (in place) ------------------------------------------

def test_pool_in_place_all_reduce_and_gather(impl):
    n = 4
    comm = VirtualCommunicator(n, device=0, pool_bytes=32 << 20)
    bufs = comm.alloc(1 << 20, torch.float32)
    rng = np.random.default_rng(41)
    xs_np = [rng.standard_normal(1 << 20).astype(np.float32) for _ in range(n)]
    for b, x in zip(bufs, xs_np):
        b.copy_(to_dev(x))
    comm.all_reduce(bufs, "premean", outs=bufs)  # in place in the registered pool
    want = O.fold_premean(xs_np)
    for b in bufs:
        assert host(b).tobytes() == want.tobytes()
    # in-place all_gather: each replica's slot r of a pooled [n, k] buffer
    k = 4096
    gb = comm.alloc(n * k, torch.float32)
    for r in range(n):
        gb[r][r * k:(r + 1) * k].copy_(to_dev(xs_np[r][:k]))
    comm.all_gather([gb[r][r * k:(r + 1) * k] for r in range(n)], outs=[g.view(n, k) for g in gb])
    want = np.concatenate([x[:k] for x in xs_np])
    for g in gb:
        assert host(g).tobytes() == want.tobytes()
    # in-place broadcast of a pooled buffer
    comm.broadcast(bufs, root=2, outs=bufs)
    for b in bufs:
        assert host(b).tobytes() == host(bufs[2]).tobytes()
    comm.close()


def test_broadcast_nonzero_root_and_odd_bytes():
    n = 3
    rng = np.random.default_rng(42)
    xs_np = [rng.standard_normal(12345).astype(np.float64) for _ in range(n)]
    for algo in ("direct", "scatter"):
        outs = vcomm(n).broadcast([to_dev(x) for x in xs_np], root=1, algo=algo)
        for o in outs:
            assert host(o).tobytes() == xs_np[1].tobytes()
    b8 = [to_dev(np.arange(7, dtype=np.float32) + r) for r in range(n)]  # 28 bytes: byte path
    outs = vcomm(n).all_gather(b8)
    assert host(outs[2]).tobytes() == np.concatenate([np.arange(7, dtype=np.float32) + r for r in range(n)]).tobytes()


# --- CUDA graph capture ------------------------------------------------------------

@pytest.mark.parametrize("n", [2, 4, 8])
def test_collectives_replay_in_cuda_graph(n, impl):
    """All sequencing state (barrier epochs, landing-zone parity, tile counters,
    phase bases) lives on the device, so a captured sequence of collectives can be
    replayed: every replay must give the oracle's answer for the new inputs."""
    comm = VirtualCommunicator(n, device=0, pool_bytes=64 << 20)
    small = [torch.empty(3000, device=DEV) for _ in range(n)]
    big = [torch.empty(700001, device=DEV) for _ in range(n)]
    gat = [torch.empty(777, device=DEV) for _ in range(n)]
    o_small = [torch.empty_like(t) for t in small]
    o_big = [torch.empty_like(t) for t in big]
    o_gat = [torch.empty(n, 777, device=DEV) for _ in range(n)]
    o_bc = [torch.empty_like(t) for t in gat]
    o_flat = [torch.empty_like(t) for t in big]

    def seq():
        comm.all_reduce(small, "sum", outs=o_small, algo="oneshot")
        comm.all_reduce(big, "premean", outs=o_big, algo="twoshot")
        comm.all_reduce(big, "max", outs=o_flat, algo="flat")  # claim counters reset by its last block
        comm.all_gather(gat, outs=o_gat)
        comm.broadcast(gat, root=n - 1, outs=o_bc)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        seq()  # warm up outside capture
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        seq()
    rng = np.random.default_rng(123)
    for it in range(4):
        vals = [[rng.standard_normal(t.numel()).astype(np.float32) for t in lst] for lst in (small, big, gat)]
        for lst, vs in zip((small, big, gat), vals):
            for t, v in zip(lst, vs):
                t.copy_(to_dev(v))
        g.replay()
        torch.cuda.synchronize()
        for r in range(n):
            assert host(o_small[r]).tobytes() == O.fold_sum(vals[0]).tobytes(), it
            assert host(o_big[r]).tobytes() == O.fold_premean(vals[1]).tobytes(), it
            assert host(o_flat[r]).tobytes() == O.fold_max(vals[1]).tobytes(), it
            assert host(o_gat[r]).tobytes() == np.concatenate(vals[2]).tobytes(), it
            assert host(o_bc[r]).tobytes() == vals[2][n - 1].tobytes(), it
    comm.check()
    # eager calls after replays stay in step with the device-side state
    outs = comm.all_reduce(big, "sum", algo="twoshot")
    assert host(outs[0]).tobytes() == O.fold_sum([host(b) for b in big]).tobytes()
    comm.close()


# --- pack / unpack (K6) ----------------------------------------------------------

def test_pack_unpack_roundtrip_with_cast():
    lib = _lib.load()
    rng = np.random.default_rng(51)
    shapes = [(3, 5), (7,), (1000,), (64, 33), (1,)]
    ts = [to_dev(rng.standard_normal(s).astype(np.float32)) for s in shapes]
    counts = [t.numel() for t in ts]
    offs, o = [], 0
    for c in counts:
        offs.append(o)
        o += (c + 63) // 64 * 64
    flat = torch.zeros(o, dtype=torch.bfloat16, device=DEV)
    pp, _k = _lib.ptr_array([t.data_ptr() for t in ts])
    cc, _k2 = _lib.i64_array(counts)
    oo, _k3 = _lib.i64_array(offs)
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.rp_pack(flat.data_ptr(), _lib.BF16, pp, cc, oo, len(ts), _lib.F32, s))
    for t, off in zip(ts, offs):
        assert torch.equal(flat[off:off + t.numel()], t.reshape(-1).to(torch.bfloat16))
    outs = [torch.empty_like(t) for t in ts]
    po, _k4 = _lib.ptr_array([t.data_ptr() for t in outs])
    _lib.check(lib.rp_unpack(flat.data_ptr(), _lib.BF16, po, cc, oo, len(ts), _lib.F32, s))
    for t, out in zip(ts, outs):
        assert torch.equal(out, t.to(torch.bfloat16).float())


# --- cross-replica BN statistics (K5/K5b) -----------------------------------------

def _bn_virtual(comm, xs, layout, rows, c, hw, eps=1e-5):
    lib = _lib.load()
    n = len(xs)
    outs = [[torch.empty(c, device=DEV) for _ in range(n)] for _ in range(3)]
    cnt = [torch.empty(1, dtype=torch.float64, device=DEV) for _ in range(n)]
    arrs = [_lib.ptr_array([x.data_ptr() for x in xs])] + [_lib.ptr_array([t.data_ptr() for t in o]) for o in outs] \
        + [_lib.ptr_array([t.data_ptr() for t in cnt])]
    p = [ctypes.cast(a[0], ctypes.c_void_p).value for a in arrs]
    code = {torch.float32: 0, torch.bfloat16: 2, torch.float16: 3, torch.float64: 1}[xs[0].dtype]
    _lib.check(lib.rp_bn_stats(comm._handle, p[0], code, rows, c, hw, layout, eps, p[1], p[2], p[3], p[4],
                               torch.cuda.current_stream().cuda_stream), "bn")
    torch.cuda.synchronize()
    return outs, cnt


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("shape", [(8, 64, 16, 16), (4, 256, 4, 4), (3, 33, 5, 7), (2, 1024, 1, 1),
                                   (64, 128, 16, 16)])
def test_bn_stats_match_f64_oracle(layout, dtype, shape, small="0", monkeypatch=None):
    """The default statistics path (split partials + exchange); the one-pass
    small-layer kernels (RP_BN_SMALL=1) are checked by the same body at the end of
    this module."""
    if monkeypatch is not None:
        monkeypatch.setenv("RP_BN_SMALL", small)
    n = 4
    comm = vcomm(n)
    g = torch.Generator(device=DEV).manual_seed(7)
    xs = [(torch.randn(shape, device=DEV, generator=g) * 2 + 0.5).to(dtype) for _ in range(n)]
    if layout == "nhwc":
        xs_k = [x.permute(0, 2, 3, 1).contiguous() for x in xs]
        rows, hw, lay = shape[0] * shape[2] * shape[3], 1, _lib.NHWC
    else:
        xs_k = xs
        rows, hw, lay = shape[0], shape[2] * shape[3], _lib.NCHW
    (mean, var, invstd), cnt = _bn_virtual(comm, xs_k, lay, rows, shape[1], hw)
    m_ref, v_ref, *_ = O.bn_stats_per_channel([host(x.float()) for x in xs], layout="nchw")
    for r in range(n):
        np.testing.assert_allclose(host(mean[r]), m_ref, rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(host(var[r]), v_ref, rtol=1e-6, atol=1e-7)
        np.testing.assert_allclose(host(invstd[r]), 1 / np.sqrt(v_ref + 1e-5), rtol=1e-6)
        assert host(cnt[r])[0] == n * shape[0] * shape[2] * shape[3]
        assert host(mean[r]).tobytes() == host(mean[0]).tobytes()  # symmetric


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
def test_bn_bwd_stats_match_oracle(layout, small="0", monkeypatch=None):
    if monkeypatch is not None:
        monkeypatch.setenv("RP_BN_SMALL", small)
    n, shape = 2, (4, 32, 6, 6)
    comm = vcomm(n)
    lib = _lib.load()
    g = torch.Generator(device=DEV).manual_seed(8)
    xs = [torch.randn(shape, device=DEV, generator=g) for _ in range(n)]
    dys = [torch.randn(shape, device=DEV, generator=g) for _ in range(n)]
    m_ref, *_ = O.bn_stats_per_channel([host(x) for x in xs], layout="nchw")
    mean = [to_dev(m_ref.astype(np.float32)) for _ in range(n)]
    outs = [[torch.empty(shape[1], device=DEV) for _ in range(n)] for _ in range(4)]
    if layout == "nhwc":
        xk = [x.permute(0, 2, 3, 1).contiguous() for x in xs]
        dk = [d.permute(0, 2, 3, 1).contiguous() for d in dys]
        rows_k, hw_k, lay = shape[0] * shape[2] * shape[3], 1, _lib.NHWC
    else:
        xk, dk, rows_k, hw_k, lay = xs, dys, shape[0], shape[2] * shape[3], _lib.NCHW
    arrs = [_lib.ptr_array([t.data_ptr() for t in lst]) for lst in ([*xk], [*dk], mean, *outs)]
    p = [ctypes.cast(a[0], ctypes.c_void_p).value for a in arrs]
    _lib.check(lib.rp_bn_bwd_stats(comm._handle, p[0], p[1], 0, rows_k, shape[1], hw_k,
                                   lay, p[2], p[3], p[4], p[5], p[6],
                                   torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    rows = [O._channel_view(host(x), "nchw") for x in xs]
    drows = [O._channel_view(host(d), "nchw") for d in dys]
    m32 = m_ref.astype(np.float32).astype(np.float64)
    sdy = sum(d.sum(0) for d in drows)
    sdyx = sum((d * (x - m32)).sum(0) for d, x in zip(drows, rows))
    for r in range(n):
        np.testing.assert_allclose(host(outs[0][r]), sdy, rtol=1e-6, atol=1e-4)
        np.testing.assert_allclose(host(outs[1][r]), sdyx, rtol=1e-6, atol=1e-4)
        np.testing.assert_allclose(host(outs[2][r]), drows[r].sum(0), rtol=1e-6, atol=1e-4)
        np.testing.assert_allclose(host(outs[3][r]), (drows[r] * (rows[r] - m32)).sum(0), rtol=1e-6, atol=1e-4)


def test_bn_apply_kernels_match_torch():
    lib = _lib.load()
    g = torch.Generator(device=DEV).manual_seed(9)
    x = torch.randn(4, 24, 5, 5, device=DEV, generator=g)
    dy = torch.randn_like(x)
    mean, var = x.mean((0, 2, 3)), x.var((0, 2, 3), unbiased=False)
    invstd = torch.rsqrt(var + 1e-5)
    w, b = torch.randn(24, device=DEV, generator=g), torch.randn(24, device=DEV, generator=g)
    s = torch.cuda.current_stream().cuda_stream
    for layout, xx, dd in ((_lib.NCHW, x, dy), (_lib.NHWC, x.permute(0, 2, 3, 1).contiguous(),
                                                dy.permute(0, 2, 3, 1).contiguous())):
        rows, hw = (4, 25) if layout == _lib.NCHW else (100, 1)
        y = torch.empty_like(xx)
        _lib.check(lib.rp_bn_apply(xx.data_ptr(), y.data_ptr(), 0, rows, 24, hw, layout, mean.data_ptr(),
                                   invstd.data_ptr(), w.data_ptr(), b.data_ptr(), s))
        ref = (x - mean[None, :, None, None]) * invstd[None, :, None, None] * w[None, :, None, None] \
            + b[None, :, None, None]
        if layout == _lib.NHWC:
            y = y.permute(0, 3, 1, 2)
        torch.testing.assert_close(y, ref, rtol=1e-5, atol=1e-5)
        # backward
        sdy = dy.sum((0, 2, 3))
        sdyx = (dy * (x - mean[None, :, None, None])).sum((0, 2, 3))
        dx = torch.empty_like(xx)
        _lib.check(lib.rp_bn_bwd_apply(xx.data_ptr(), dd.data_ptr(), dx.data_ptr(), 0, rows, 24, hw, layout,
                                       mean.data_ptr(), invstd.data_ptr(), w.data_ptr(), sdy.data_ptr(),
                                       sdyx.data_ptr(), 100.0, None, s))
        # the same with M read on the device (no host sync, as autograd's backward does)
        cnt = torch.tensor([100.0], dtype=torch.float64, device=DEV)
        dx2 = torch.empty_like(xx)
        _lib.check(lib.rp_bn_bwd_apply(xx.data_ptr(), dd.data_ptr(), dx2.data_ptr(), 0, rows, 24, hw, layout,
                                       mean.data_ptr(), invstd.data_ptr(), w.data_ptr(), sdy.data_ptr(),
                                       sdyx.data_ptr(), 0.0, cnt.data_ptr(), s))
        assert torch.equal(dx, dx2)
        xt = x.clone().requires_grad_(True)
        yt = torch.nn.functional.batch_norm(xt, None, None, w, b, training=True, eps=1e-5)
        yt.backward(dy)
        if layout == _lib.NHWC:
            dx = dx.permute(0, 3, 1, 2)
        torch.testing.assert_close(dx, xt.grad, rtol=1e-4, atol=1e-5)


# --- the Replicator facade on virtual replicas ----------------------------------

def test_wrap_optimizer_matches_reference_bitwise(wrap_golden):
    wrap_golden = {k: wrap_golden[k] for k in wrap_golden.files}  # NpzFile is not thread-safe
    for n in (2, 4):
        nw = len([k for k in wrap_golden if k.startswith(f"small_n{n}_w")])
        repl = Replicator(num_replicas=n, device=0, pool_bytes=16 << 20)
        with repl.context():
            params = repl.replicate(lambda: torch.nn.ParameterList(
                [torch.nn.Parameter(to_dev(wrap_golden[f"small_n{n}_w{i}"])) for i in range(nw)]))
            opt = repl.wrap_optimizer(PerReplica(
                [torch.optim.SGD(list(params[r].parameters()), lr=0.1) for r in range(n)], repl))

        def step(_):
            r = repl.replica_id
            for i, p in enumerate(params.local.parameters()):
                p.grad = to_dev(wrap_golden[f"small_n{n}_g{r}_{i}"])
            opt.step()
            return [(p.grad.clone(), p.detach().clone()) for p in params.local.parameters()]

        outs = repl.run(step, lambda r: None)
        for r in range(n):
            for i in range(nw):
                g, w = outs[r][i]
                # the averaged gradient is the reference's stitched all_sum(g/R), bit for bit
                assert host(g).tobytes() == wrap_golden[f"small_n{n}_avg{i}"].tobytes(), (n, r, i)
                # the base SGD rule is torch's (may fuse w - lr*g into one FMA)
                np.testing.assert_allclose(host(w), wrap_golden[f"small_n{n}_new{i}"], rtol=1e-15, atol=1e-16)
                assert host(w).tobytes() == host(outs[0][i][1]).tobytes()  # replicas stay identical
        repl.comm.close()


def test_config1_average_md5(wrap_golden):
    import hashlib
    meta = json.load(open(os.path.join(GOLDEN, "wrap_sgd.json")))
    comm = vcomm(2)
    avgs = []
    for i in range(4):
        xs = [to_dev(wrap_golden[f"cfg1_g{r}_{i}"]).reshape(-1) for r in range(2)]
        avgs.append(host(comm.all_reduce(xs, "premean")[0]).reshape(wrap_golden[f"cfg1_g0_{i}"].shape))
    md5 = hashlib.md5(b"".join(np.ascontiguousarray(a).tobytes() for a in avgs)).hexdigest()
    assert md5 == meta["cfg1_avg_md5"]


def test_replicator_run_all_sum_and_protocol_error():
    repl = Replicator(num_replicas=3, device=0, pool_bytes=16 << 20)

    def step(x):
        return repl.all_sum(x, label="g")

    outs = repl.run(step, lambda r: torch.full((5,), float(r + 1), device=DEV))
    for o in outs:
        assert host(o).tolist() == [6.0] * 5
    # replicas diverging on the label: the stitcher's first-divergence error
    with pytest.raises(errors.ProtocolError):
        repl.run(lambda x: repl.all_sum(x, label=f"g{repl.replica_id}"),
                 lambda r: torch.ones(2, device=DEV))
    gathered = repl.run(lambda x: repl.all_gather(x, stack=True), lambda r: torch.full((2,), float(r), device=DEV))
    assert host(gathered[1]).tolist() == [[0, 0], [1, 1], [2, 2]]
    # the default is the rank-ordered list [t_0, ..., t_{N-1}]
    lists = repl.run(lambda x: repl.all_gather(x), lambda r: torch.full((2,), float(r), device=DEV))
    assert all(isinstance(l, list) and [host(t).tolist() for t in l] == [[0, 0], [1, 1], [2, 2]] for l in lists)
    scal = repl.run(lambda x: repl.all_gather(x), lambda r: torch.tensor(float(7 + r), device=DEV))
    assert [float(host(t)) for t in scal[0]] == [7.0, 8.0, 9.0]  # SPEC's N=3 scalars example
    repl.comm.close()


def test_replicator_paper_batch_norm_kat():
    # h0=[1,3], h1=[5,7] -> (h - 4)/sqrt(5 + eps)
    repl = Replicator(num_replicas=2, device=0, pool_bytes=16 << 20)
    hs = [torch.tensor([1.0, 3.0], device=DEV, dtype=torch.float64),
          torch.tensor([5.0, 7.0], device=DEV, dtype=torch.float64)]
    outs = repl.run(lambda h: repl.batch_norm(h), lambda r: hs[r])
    for r in range(2):
        np.testing.assert_allclose(host(outs[r]), (host(hs[r]) - 4) / np.sqrt(5 + 1e-5), rtol=0, atol=1e-15)
    repl.comm.close()


def test_virtual_collectives_refuse_backprop():
    """in-process virtual replicas cannot rendezvous in backward (their
    backward passes share one autograd device thread), so backprop reaching a
    collective raises the reference's NotDifferentiableError (graph.py:798-800)
    instead of silently dropping the gradient; the forward values are unchanged,
    and inputs that do not require grad are unaffected."""
    repl = Replicator(num_replicas=2, device=0, pool_bytes=16 << 20)

    def step(x):
        y = repl.all_sum(x, label="s")
        y.sum().backward()

    with pytest.raises(errors.NotDifferentiableError):
        repl.run(step, lambda r: torch.full((3,), float(r + 1), device=DEV, requires_grad=True))
    outs = repl.run(lambda x: repl.all_sum(x * 2, label="t"),
                    lambda r: torch.full((3,), float(r + 1), device=DEV, requires_grad=True))
    assert all(host(o.detach()).tolist() == [6.0] * 3 and o.requires_grad for o in outs)
    outs = repl.run(lambda x: repl.broadcast(x, root=1), lambda r: torch.full((2,), float(r), device=DEV))
    assert all(host(o).tolist() == [1.0, 1.0] and not o.requires_grad for o in outs)
    repl.comm.close()


def test_cross_replica_bn_module_forward_virtual():
    n = 2
    repl = Replicator(num_replicas=n, device=0, pool_bytes=16 << 20)
    g = torch.Generator(device=DEV).manual_seed(10)
    xs = [torch.randn(4, 16, 3, 3, device=DEV, generator=g) for _ in range(n)]
    bns = repl.replicate(lambda: CrossReplicaBatchNorm(16, repl))
    outs = repl.run(lambda x: bns(x), lambda r: xs[r])
    ref = torch.nn.functional.batch_norm(torch.cat(xs), None, None, training=True, eps=1e-5)
    torch.testing.assert_close(torch.cat(outs), ref, rtol=1e-5, atol=1e-5)
    repl.comm.close()


_FUSED_OPTS = [
    ("sgd", lambda ps: torch.optim.SGD(ps, lr=0.1)),
    ("sgd_momentum_nesterov_wd", lambda ps: torch.optim.SGD(ps, lr=0.05, momentum=0.9, nesterov=True,
                                                            weight_decay=1e-3)),
    ("sgd_momentum_dampening", lambda ps: torch.optim.SGD(ps, lr=0.05, momentum=0.8, dampening=0.25)),
    ("adam_wd", lambda ps: torch.optim.Adam(ps, lr=1e-3, weight_decay=1e-2)),
    ("adamw", lambda ps: torch.optim.AdamW(ps, lr=1e-3, betas=(0.8, 0.95), weight_decay=1e-2)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 3, 4, 8])
@pytest.mark.parametrize("name,make", _FUSED_OPTS, ids=[o[0] for o in _FUSED_OPTS])
def test_fused_apply_matches_torch_optimizer(n, name, make):
    """wrap_optimizer(fused=True) (csrc/rp_apply.cu) against torch's own optimizer
    driven by the rank-ordered averaged gradient (bit-exact premean fold, oracle):
    f32 update arithmetic within a few ulps, replicas bit-identical, state sharded."""
    shapes = [(37, 19), (19,), (8, 3, 3, 3), (5,)]  # odd sizes: tails, padding between slots
    init = [torch.randn(s, generator=torch.Generator().manual_seed(10 + i)) for i, s in enumerate(shapes)]
    repl = Replicator(num_replicas=n, device=0, pool_bytes=16 << 20)
    with repl.context():
        params = repl.replicate(lambda: torch.nn.ParameterList(
            [torch.nn.Parameter(t.clone().to(DEV)) for t in init]))
        opt = repl.wrap_optimizer(PerReplica([make(list(params[r].parameters())) for r in range(n)], repl),
                                  fused=True)
    ref = [torch.nn.Parameter(t.clone().to(DEV)) for t in init]
    ref_opt = make(ref)
    steps = 3
    grads = {(s, r, i): torch.randn(shapes[i], generator=torch.Generator().manual_seed(1000 * s + 10 * r + i))
             for s in range(steps) for r in range(n) for i in range(len(shapes))}

    def step(_):
        r = repl.replica_id
        for i, p in enumerate(params.local.parameters()):
            p.grad = grads[(s, r, i)].to(DEV)
        opt.step()

    for s in range(steps):
        repl.run(step, lambda r: None)
        for i, p in enumerate(ref):
            avg = O.fold_premean([grads[(s, r, i)].numpy().astype(np.float32) for r in range(n)])
            p.grad = torch.from_numpy(np.ascontiguousarray(avg)).to(DEV)
        ref_opt.step()
    torch.cuda.synchronize()
    for r in range(n):
        for i, (p, q) in enumerate(zip(params[r].parameters(), ref)):
            np.testing.assert_allclose(host(p.detach()), host(q.detach()), rtol=2e-6, atol=2e-7,
                                       err_msg=f"{name} n={n} r={r} {i}")
            mirror = host(list(params[0].parameters())[i].detach())
            assert host(p.detach()).tobytes() == mirror.tobytes()  # replicas bit-identical
    g = opt.groups[0]
    assert g.shard_len * n >= g.grads.numel and g.shard_len * n < g.grads.numel + n * 8
    assert int(g.steps[0].item()) == steps
    repl.comm.close()


@pytest.mark.gpu
def test_fused_apply_rejects_unsupported():
    repl = Replicator(num_replicas=2, device=0, pool_bytes=16 << 20)
    with repl.context():
        params = repl.replicate(lambda: torch.nn.Linear(4, 4).to(DEV))
        with pytest.raises(errors.ConfigurationError):
            repl.wrap_optimizer(PerReplica([torch.optim.RMSprop(params[r].parameters()) for r in range(2)], repl),
                                fused=True)
        with pytest.raises(errors.ConfigurationError):
            repl.wrap_optimizer(PerReplica([torch.optim.SGD(params[r].parameters(), lr=0.1) for r in range(2)],
                                           repl), kind="sum", fused=True)
    repl.comm.close()


@pytest.mark.gpu
def test_ragged_all_gather_and_driver_values_virtual():
    """SPEC.md:205-213 (leading dimensions may differ) and :223-231 (map_gather /
    map_reduce are delivered to the driver; reading them inside a replica fails)."""
    n = 3
    repl = Replicator(num_replicas=n, device=0, pool_bytes=16 << 20)

    def step(x):
        g = repl.all_gather(x, label="rows", ragged=True)
        mg = repl.map_gather(x.sum(0), label="mg")
        mr = repl.map_reduce(x.sum(), "sum", label="mr")
        with pytest.raises(errors.EvaluationError):
            _ = mr.value  # consumed inside the replicated step
        return g, mg, mr

    xs = [torch.arange(r * 4 + 1, dtype=torch.float32, device=DEV).repeat(2, 1).t().contiguous() * (r + 1)
          for r in range(n)]  # shapes (1,2), (5,2), (9,2)
    outs = repl.run(step, lambda r: xs[r])
    for r in range(n):
        g, mg, mr = outs[r]
        assert [tuple(t.shape) for t in g] == [(1, 2), (5, 2), (9, 2)]
        for q in range(n):
            assert torch.equal(g[q], xs[q])
        assert [host(t).tolist() for t in mg.value] == [host(x.sum(0)).tolist() for x in xs]
        assert float(host(mr.value)) == float(sum(host(x).sum() for x in xs))
    with pytest.raises(errors.ProtocolError):  # trailing dimensions must agree
        repl.run(lambda x: repl.all_gather(x, ragged=True),
                 lambda r: torch.zeros((2, 2 + (r == 1)), device=DEV))
    repl.comm.close()


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("kind", ["sum", "premean", "max"])
def test_all_reduce_host_pipelined_matches_oracle(kind, pinned):
    """all_reduce_host: host tensors in, host tensor out through the chunked ring
    (several chunks, a ragged tail, ring slots reused); bit-identical to the oracle's
    rank-ordered fold, like the whole-message device call."""
    comm = vcomm(4)
    count = 3 * 4096 + 123  # 4 chunks of 4096 elements + a tail
    rng = np.random.default_rng(11)
    xs = [rng.standard_normal(count).astype(np.float32) for _ in range(4)]
    hin = [torch.from_numpy(x) for x in xs]
    if pinned:
        hin = [h.pin_memory() for h in hin]
    want = {"sum": O.fold_sum, "premean": O.fold_premean, "max": O.fold_max}[kind](xs)
    for _ in range(2):  # second call reuses the ring
        out = comm.all_reduce_host(hin, kind, chunk_bytes=4096 * 4)
        assert out.numpy().tobytes() == want.tobytes()
    f64 = [rng.standard_normal(1000) for _ in range(4)]
    out = comm.all_reduce_host([torch.from_numpy(x) for x in f64], "sum", chunk_bytes=256 * 8)
    assert out.numpy().tobytes() == O.fold_sum(f64).tobytes()
    with pytest.raises(errors.ShapeError):
        comm.all_reduce_host(hin[:3], kind)


# --- A/B variant (round 2): kept last so a failure cannot hide the tests above ----

@pytest.mark.parametrize("n", [2, 3, 8])
def test_flat_bulk_copy_variant_matches_oracle(n, monkeypatch):
    """The cp.async.bulk (TMA bulk engine + mbarrier) staging of the flat virtual
    all-reduce (RP_VFLAT_BULK=1): bit-exact for every fold, for counts with a
    partial last vector (register-path tail) and with tiny / odd sizes; misaligned
    buffers fall back to the register form."""
    monkeypatch.setenv("RP_VFLAT_BULK", "1")
    rng = np.random.default_rng(n)
    for count in (1, 3, 4, 5, 127, 4097, 65536 + 3, (1 << 20) + 1):
        xs_np = [rng.standard_normal(count).astype(np.float32) for _ in range(n)]
        for kind in ("sum", "mean", "max", "premean"):
            want = O.FOLDS[kind](xs_np)
            outs = vcomm(n).all_reduce([to_dev(x) for x in xs_np], kind, algo="flat")
            for o in outs:
                assert host(o).tobytes() == want.tobytes(), (count, kind)
    xs64 = [rng.standard_normal(33333) for _ in range(n)]
    outs = vcomm(n).all_reduce([to_dev(x) for x in xs64], "sum", algo="flat")
    assert host(outs[0]).tobytes() == O.fold_sum(xs64).tobytes()
    base = [to_dev(rng.standard_normal(1001).astype(np.float32)) for _ in range(n)]
    xs = [b[1:] for b in base]  # misaligned: register form
    outs = vcomm(n).all_reduce(xs, "sum", algo="flat")
    assert host(outs[0]).tobytes() == O.fold_sum([host(x) for x in xs]).tobytes()
    vcomm(n).check()


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("shape", [(8, 64, 16, 16), (4, 256, 4, 4), (2, 1024, 1, 1), (64, 1024, 4, 4),
                                   (3, 33, 5, 7)])
def test_bn_small_layer_kernels_match_f64_oracle(layout, dtype, shape, monkeypatch):
    """The one-pass small-layer statistics kernels (RP_BN_SMALL=1: bn_stats_small for
    NHWC, bn_stats_small_nchw for NCHW; the SN-GAN 64x1024x4x4 layer among the
    shapes), forward and backward, against the same f64 oracle as the default path."""
    test_bn_stats_match_f64_oracle(layout, dtype, shape, small="1", monkeypatch=monkeypatch)
    if dtype == torch.float32 and shape == (4, 256, 4, 4):
        test_bn_bwd_stats_match_oracle(layout, small="1", monkeypatch=monkeypatch)
