"""Multi-process NVLink path: one process per GPU, communicators bootstrapped over
torch.distributed (gloo, handle exchange only), kernels loading/storing peer pools.
Needs >= 2 GPUs (``gpurun --gpus 2`` / ``--gpus 4``); skipped otherwise.

Every rank derives all ranks' inputs from per-rank seeds, so each rank checks its
own result against the CPU oracle on identical inputs (bit-exact folds / copies,
1e-6 BN statistics)."""

import os
import socket

import numpy as np
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

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        globals()[fn_name](rank, world)
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
# rank bodies (module-level so spawn can pickle them by name)
# ---------------------------------------------------------------------------

def _inputs(world, count, dtype=np.float32, seed=100):
    return [np.random.default_rng(seed + r).standard_normal(count).astype(dtype) for r in range(world)]


def body_all_reduce(rank, world):
    from oracle import collectives as O
    from paper_1902_00465_b200.comm import Communicator

    dev = torch.device(f"cuda:{rank}")
    comm = Communicator(device=rank, pool_bytes=96 << 20)
    for impl in ("push", "pull"):
        os.environ["RP_AR_IMPL"] = impl
        for count in (1, 7, 1000, 4097, 1 << 16, (1 << 20) + 3, 16 << 20, 40 << 20):
            xs = _inputs(world, count, seed=count)
            x = torch.from_numpy(xs[rank]).to(dev)
            for kind in ("sum", "mean", "max", "premean"):
                want = O.FOLDS[kind](xs)
                for algo in ("oneshot", "twoshot"):
                    y = comm.all_reduce_tensor(x, kind, algo=algo)
                    got = y.cpu().numpy()
                    assert got.tobytes() == want.tobytes(), (impl, count, kind, algo)
                    y2 = x.clone()
                    comm.all_reduce_tensor(y2, kind, out=y2, algo=algo)  # in place, user buffer
                    assert y2.cpu().numpy().tobytes() == want.tobytes(), (impl, count, kind, algo, "inplace")
    os.environ.pop("RP_AR_IMPL")
    # f64 and bf16 with the fused exchange cast
    xs = _inputs(world, 33333, np.float64, seed=7)
    y = comm.all_reduce_tensor(torch.from_numpy(xs[rank]).to(dev), "sum")
    assert y.cpu().numpy().tobytes() == O.fold_sum(xs).tobytes()
    xs = _inputs(world, 50001, seed=8)
    y = comm.all_reduce_tensor(torch.from_numpy(xs[rank]).to(dev), "premean", comm_dtype=torch.bfloat16)
    want = O.bf16_bits_to_f32(O.fold_bf16([O.f32_to_bf16_bits(x) for x in xs], "premean"))
    assert y.cpu().numpy().tobytes() == want.tobytes()
    # zero-copy in place in the registered pool
    buf = comm.alloc(1 << 20, torch.float32)
    xs = _inputs(world, 1 << 20, seed=9)
    buf.copy_(torch.from_numpy(xs[rank]))
    comm.all_reduce_tensor(buf, "premean", out=buf)
    assert buf.cpu().numpy().tobytes() == O.fold_premean(xs).tobytes()
    comm.check()
    comm.close()


def body_gather_broadcast(rank, world):
    from oracle import collectives as O
    from paper_1902_00465_b200.comm import Communicator

    dev = torch.device(f"cuda:{rank}")
    comm = Communicator(device=rank, pool_bytes=96 << 20)
    for count in (1, 7, 1000, 12345, 65536, 65537, 1 << 20):
        xs = _inputs(world, count, seed=count + 1)
        g = comm.all_gather_tensor(torch.from_numpy(xs[rank]).to(dev))
        assert g.cpu().numpy().tobytes() == np.concatenate(xs).tobytes()
        # in place: src is this rank's slot of a pool-resident output
        out = comm.alloc(world * count, torch.float32).view(world, count)
        out[rank].copy_(torch.from_numpy(xs[rank]))
        comm.all_gather_tensor(out[rank], out=out)
        assert out.cpu().numpy().tobytes() == np.concatenate(xs).tobytes(), count
        for root in range(world):
            for algo in ("auto", "direct", "scatter") + (("relay",) if count % 4 == 0 else ()):
                x = torch.from_numpy(xs[rank]).to(dev)
                comm.broadcast_tensor(x, root=root, algo=algo)
                assert x.cpu().numpy().tobytes() == xs[root].tobytes(), (count, root, algo)
    # dense non-contiguous layouts (channels_last parameters) are exchanged in place,
    # strided views through a copy that is written back
    g = torch.Generator(device=dev).manual_seed(77 + rank)
    cl = torch.randn(2, 8, 5, 3, device=dev, generator=g).contiguous(memory_format=torch.channels_last)
    cl_ptr = cl.data_ptr()
    comm.broadcast_tensor(cl, root=0)
    assert cl.data_ptr() == cl_ptr and cl.is_contiguous(memory_format=torch.channels_last)
    allc = comm.all_gather_tensor(cl.contiguous())
    assert all(torch.equal(allc[r], allc[0]) for r in range(world))
    base = torch.randn(6, 10, device=dev, generator=g)
    view = base[:, ::2]
    before = [comm.all_gather_tensor(view.contiguous())[r].clone() for r in range(world)]
    comm.all_reduce_tensor(view, "sum", out=view)
    want = before[0].clone()
    for r in range(1, world):
        want = want + before[r]
    assert torch.equal(view, want) and torch.equal(base[:, 1::2], base[:, 1::2])
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


def body_mesh_seam(rank, world):
    """Replay what the reference's mesh seam hands a communicator
    (tests/golden/mesh_seam.json, recorded from graph.py:565-583) and check our
    Communicator returns what the seam expects, as the reference's Tensor type."""
    import json

    from paper_1902_00465_b200.comm import Communicator
    from tests.helpers import GOLDEN

    if world != 2:
        return
    comm = Communicator(device=rank, pool_bytes=16 << 20)
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
            assert got.reshape(-1).tolist() == want, (t["shape"], t["dtype"])
    comm.close()


def body_bn(rank, world):
    from oracle import collectives as O
    from paper_1902_00465_b200.replicator import CrossReplicaBatchNorm, Replicator

    dev = torch.device(f"cuda:{rank}")
    repl = Replicator(device=rank, pool_bytes=16 << 20)
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
        np.testing.assert_allclose(y.detach().cpu().numpy(), outs[rank], rtol=1e-4, atol=1e-4)
        dxs, sdy, sdyx = O.bn_backward_per_channel(xs, dys, "nchw", weight=w)
        np.testing.assert_allclose(x.grad.cpu().numpy(), dxs[rank], rtol=1e-4, atol=1e-4)
        # local weight/bias grads (averaged later by the wrapped optimizer)
        xr = O._channel_view(xs[rank], "nchw")
        dr = O._channel_view(dys[rank], "nchw")
        np.testing.assert_allclose(bn.bias.grad.cpu().numpy(), dr.sum(0), rtol=1e-5, atol=1e-4)
        np.testing.assert_allclose(bn.weight.grad.cpu().numpy(), (dr * (xr - mean) / np.sqrt(var + 1e-5)).sum(0),
                                   rtol=1e-4, atol=1e-4)
        np.testing.assert_allclose(bn.running_mean.cpu().numpy(), 0.1 * mean, rtol=1e-5, atol=1e-6)
    repl.comm.close()


def body_wrap_optimizer(rank, world):
    from paper_1902_00465_b200.replicator import Replicator

    dev = torch.device(f"cuda:{rank}")
    repl = Replicator(device=rank, pool_bytes=32 << 20)
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
        assert (p - q).abs().max().item() < 1e-9  # SPEC.md:399 sync-equivalence bound
    # a channels_last conv model: replicate() must sync every replica in place
    torch.manual_seed(100 + rank)
    conv = repl.replicate(lambda: torch.nn.Sequential(torch.nn.Conv2d(3, 8, 3), torch.nn.BatchNorm2d(8))
                          .to(memory_format=torch.channels_last))
    cflat = torch.cat([q.detach().contiguous().reshape(-1) for q in conv.local.parameters()])
    cg = repl.comm.all_gather_tensor(cflat)
    assert all(torch.equal(cg[r], cg[0]) for r in range(world)), "replicate() left channels_last replicas apart"
    # replicas bit-identical
    flat = torch.cat([p.detach().reshape(-1) for p in model.local.parameters()])
    g = repl.comm.all_gather_tensor(flat)
    for r in range(world):
        assert torch.equal(g[r], g[0])
    repl.comm.close()


def body_nvls(rank, world):
    """In-switch all-reduce (multimem.ld_reduce / multimem.st). Not rank-ordered,
    so checked against the f64 sum with a stated tolerance (north star: <=1e-6
    relative, ordering-induced), plus bit-identical results on every rank."""
    from paper_1902_00465_b200.comm import Communicator

    comm = Communicator(device=rank, pool_bytes=128 << 20)
    comm.enable_nvls(96 << 20)
    for count in (4, 1000, 4099, 1 << 20, 12 << 20):
        xs = _inputs(world, count, seed=500 + count)
        buf = comm.alloc_nvls(count, torch.float32)
        for kind in ("sum", "mean", "premean"):
            buf.copy_(torch.from_numpy(xs[rank]))
            comm.all_reduce_tensor(buf, kind, out=buf, algo="nvls")
            got = buf.cpu().numpy().astype(np.float64)
            want = np.sum(np.stack(xs).astype(np.float64), axis=0) / (1 if kind == "sum" else world)
            err = np.linalg.norm(got - want) / np.linalg.norm(want)
            assert err <= 1e-6, (count, kind, err)
            g = comm.all_gather_tensor(buf)
            assert all(torch.equal(g[r], g[0]) for r in range(world))
        xb = [x.astype(np.float32) for x in _inputs(world, 50000, seed=9)]
        bb = comm.alloc_nvls(50000, torch.bfloat16)
        bb.copy_(torch.from_numpy(xb[rank]).to(torch.bfloat16))
        comm.all_reduce_tensor(bb, "sum", out=bb, algo="nvls")
        ref = sum(torch.from_numpy(x).to(torch.bfloat16).double() for x in xb)
        rel = (bb.double().cpu() - ref).norm() / ref.norm()
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
    got = big.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-6
    # NVLS broadcast (rp.h RP_ALGO_NVLS for rp_broadcast): destination in the region,
    # the root multicasts from any local source (in place, separate, misaligned); bit-exact
    dev = torch.device(f"cuda:{rank}")
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
                assert torch.equal(dst.cpu(), exp), (nbytes, root, mode)
                dst.fill_(rank + 7)
    comm.check()
    comm.close()


def body_wrap_nvls(rank, world):
    """wrap_optimizer with fusion buckets in the NVLS region (Replicator(nvls_bytes)):
    the same training as the single-device oracle on the concatenated batch, within
    the f32 ordering tolerance, and replicas stay bit-identical (the multicast store
    writes one value to every rank)."""
    from paper_1902_00465_b200.replicator import Replicator

    dev = torch.device(f"cuda:{rank}")
    repl = Replicator(device=rank, pool_bytes=32 << 20, nvls_bytes=16 << 20)
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
        assert (p.double() - q).abs().max().item() < 1e-5
    flat = torch.cat([p.detach().reshape(-1) for p in model.local.parameters()])
    gathered = repl.comm.all_gather_tensor(flat)
    assert all(torch.equal(gathered[r], gathered[0]) for r in range(world))
    repl.comm.close()


def body_fused_apply(rank, world):
    """wrap_optimizer(Adam, fused=True) over real ranks: each step equals torch's
    Adam driven by the rank-ordered averaged gradient (gathered and folded by the
    oracle), replicas stay bit-identical, and the whole training step (forward,
    backward, fused apply) replays from a CUDA graph."""
    from oracle import collectives as O
    from paper_1902_00465_b200.replicator import Replicator

    dev = torch.device(f"cuda:{rank}")
    repl = Replicator(device=rank, pool_bytes=32 << 20)
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
        every = repl.comm.all_gather_tensor(flat).cpu().numpy()
        avg = torch.from_numpy(O.fold_premean([every[r] for r in range(world)])).to(dev)
        o = 0
        for p in ref.parameters():
            p.grad = avg[o:o + p.numel()].view_as(p).clone()
            o += p.numel()
        opt.step()
        ref_opt.step()
    for p, q in zip(model.local.parameters(), ref.parameters()):
        assert torch.allclose(p, q, rtol=2e-6, atol=2e-7), (p - q).abs().max().item()
    flat = torch.cat([p.detach().reshape(-1) for p in model.local.parameters()])
    gathered = repl.comm.all_gather_tensor(flat)
    assert all(torch.equal(gathered[r], gathered[0]) for r in range(world))
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
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        train_step()
    before = flat.clone()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    repl.comm.check()
    assert int(opt.groups[0].steps[0].item()) == 3 + 1 + 3
    flat = torch.cat([p.detach().reshape(-1) for p in model.local.parameters()])
    assert not torch.equal(flat, before)
    gathered = repl.comm.all_gather_tensor(flat)
    assert all(torch.equal(gathered[r], gathered[0]) for r in range(world))
    repl.comm.close()


def body_protocol(rank, world):
    """Replicator(check_protocol=True): mismatched shapes or
    order raise ProtocolError on EVERY rank, naming what each issued; a label reused
    within a generation is rejected, across generations it is fine; the reference
    duck type's all_gather accepts differing leading dimensions."""
    from paper_1902_00465_b200 import errors
    from paper_1902_00465_b200.replicator import Replicator

    dev = torch.device(f"cuda:{rank}")
    repl = Replicator(device=rank, pool_bytes=16 << 20, check_protocol=True)
    x = torch.full((4,), float(rank + 1), device=dev)
    assert repl.all_sum(x, label="a").tolist() == [float(sum(range(1, world + 1)))] * 4
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
    # the duck type (graph.py:575-579) with ragged leading dimensions; scalars stay scalars
    rows = torch.arange((rank + 1) * 3, dtype=torch.float32, device=dev).reshape(rank + 1, 3)
    got = repl.comm.all_gather(rows)
    assert [tuple(t.shape) for t in got] == [(r + 1, 3) for r in range(world)]
    assert all(torch.equal(got[r], torch.arange((r + 1) * 3, dtype=torch.float32, device=dev).reshape(r + 1, 3))
               for r in range(world))
    sc = repl.comm.all_gather(np.float64(rank))
    assert [float(np.asarray(v)) for v in sc] == [float(r) for r in range(world)]
    repl.comm.check()
    repl.comm.close()


def body_graph(rank, world):
    """Each rank captures the same sequence of collectives in a CUDA graph and
    replays it; device-side sequencing keeps the ranks in step across replays."""
    from oracle import collectives as O
    from paper_1902_00465_b200.comm import Communicator

    dev = torch.device(f"cuda:{rank}")
    comm = Communicator(device=rank, pool_bytes=64 << 20)
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
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        seq()
    for it in range(5):
        xs_s = _inputs(world, 5000, seed=1000 + it)
        xs_b = _inputs(world, 3 << 20, seed=2000 + it)
        xs_k = _inputs(world, 1 << 20, seed=3000 + it)
        small.copy_(torch.from_numpy(xs_s[rank]))
        big.copy_(torch.from_numpy(xs_b[rank]))
        bucket.copy_(torch.from_numpy(xs_k[rank]))
        g.replay()
        torch.cuda.synchronize()
        assert o_small.cpu().numpy().tobytes() == O.fold_sum(xs_s).tobytes(), it
        assert o_big.cpu().numpy().tobytes() == O.fold_premean(xs_b).tobytes(), it
        assert bucket.cpu().numpy().tobytes() == O.fold_premean(xs_k).tobytes(), it
    comm.check()
    comm.close()


def body_timeout(rank, world):
    """A rank that never joins makes the others time out (not hang) and report
    CollectiveAbortedError (SPEC.md:237 liveness; errors.py:68)."""
    from paper_1902_00465_b200 import errors
    from paper_1902_00465_b200.comm import Communicator

    comm = Communicator(device=rank, pool_bytes=16 << 20, timeout_s=2.0)
    x = torch.ones(1024, device=f"cuda:{rank}")
    if rank != world - 1:
        comm.all_reduce_tensor(x, "sum")
        with pytest.raises(errors.CollectiveAbortedError):
            comm.check()
    import torch.distributed as dist
    dist.barrier()
    comm.close()


def body_overlap(rank, world):
    """wrap_optimizer(overlap=True): buckets exchanged from post-accumulate-grad
    hooks on a side stream during backward must give the SAME bits as the
    synchronous wrapped optimizer (same premean fold per element), including with
    a bf16 exchange, unused parameters and no_sync() gradient accumulation."""
    from paper_1902_00465_b200 import errors
    from paper_1902_00465_b200.replicator import Replicator

    dev = torch.device(f"cuda:{rank}")

    def net():
        return torch.nn.Sequential(torch.nn.Conv2d(3, 16, 3, padding=1), torch.nn.ReLU(),
                                   torch.nn.Conv2d(16, 32, 3, padding=1), torch.nn.ReLU(),
                                   torch.nn.AdaptiveAvgPool2d(1), torch.nn.Flatten(), torch.nn.Linear(32, 10))

    for comm_dt in (None, torch.bfloat16):
        results = []
        for overlap, views in ((False, False), (False, True), (True, True)):
            repl = Replicator(device=rank, pool_bytes=32 << 20, grad_comm_dtype=comm_dt, grad_views=views,
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
            torch.cuda.synchronize()
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
                assert torch.equal(a, b), f"{what} differs from the packed synchronous exchange ({comm_dt})"
        flat = torch.cat([p.reshape(-1) for p in results[2]])
        import torch.distributed as dist
        gl = [torch.empty_like(flat.cpu()) for _ in range(world)]
        dist.all_gather(gl, flat.cpu())
        assert all(torch.equal(t, gl[0]) for t in gl), "replicas diverged"


def body_host_pipeline(rank, world):
    """Communicator.all_reduce_host: pinned host in, pinned host out, chunked through
    pool slots (many chunks, ragged tail, ring reuse); bit-exact vs the oracle fold,
    and with NVLS slots within the ordering tolerance."""
    from oracle import collectives as O
    from paper_1902_00465_b200.comm import Communicator

    comm = Communicator(device=rank, pool_bytes=64 << 20)
    count = 5 * 8192 + 77
    xs = _inputs(world, count, seed=321)
    hin = torch.from_numpy(xs[rank]).pin_memory()
    for kind, fold in (("sum", O.fold_sum), ("premean", O.fold_premean)):
        for _ in range(2):
            out = comm.all_reduce_host(hin, kind, chunk_bytes=8192 * 4)
            assert out.numpy().tobytes() == fold(xs).tobytes(), kind
    comm.enable_nvls(16 << 20)
    out = comm.all_reduce_host(hin, "sum", chunk_bytes=1 << 20, nvls=True)
    want = np.sum(np.stack(xs).astype(np.float64), axis=0)
    assert np.linalg.norm(out.numpy() - want) / np.linalg.norm(want) <= 1e-6
    comm.check()
    comm.close()


def body_relay_broadcast(rank, world):
    """Pipelined relay broadcast (K4r): bit-exact for every root, landing in staging
    (user dst, aligned or not) or straight in a pool-resident dst, many tiles,
    repeated calls (per-tile epoch flags are never reset)."""
    from paper_1902_00465_b200.comm import Communicator

    dev = torch.device(f"cuda:{rank}")
    comm = Communicator(device=rank, pool_bytes=96 << 20)
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
                assert np.array_equal(out.cpu().numpy(), want[root][:nbytes]), (nbytes, root, mode)
    comm.check()
    comm.close()


def _nullcontext():
    import contextlib
    return contextlib.nullcontext()


# ---------------------------------------------------------------------------

def test_all_reduce_multiprocess():
    run_world("body_all_reduce")


def test_gather_broadcast_multiprocess():
    run_world("body_gather_broadcast")


def test_reference_mesh_seam_replay():
    run_world("body_mesh_seam", world=2)


def test_cross_replica_bn_autograd_multiprocess():
    run_world("body_bn")


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


def test_host_pipelined_all_reduce_multiprocess():
    run_world("body_host_pipeline")


def test_relay_broadcast_multiprocess():
    run_world("body_relay_broadcast")
