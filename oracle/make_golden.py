"""Generate ``tests/golden/*`` by running the REFERENCE itself. TEST INFRASTRUCTURE ONLY.

Run in the build container (needs ``/root/reference``):

    python -m oracle.make_golden

Every fixture is produced by evaluating the reference's own ``Graph`` (stitched the way
SPEC.md:290-298 describes: one ``nary_*``/``concat``/``pack``/``pick0`` node per replica
site over all replicas' inputs, graph.py:506-540) or its ``mesh_collective`` seam
(graph.py:565-583) with a recording communicator. The GPU tests compare the CUDA path
against these arrays; ``tests/test_oracle.py`` checks ``oracle/collectives.py`` against
them too.
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from . import ref_adapter

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(os.path.dirname(HERE), "tests", "golden")

SHAPES = [(), (1,), (7,), (3, 5), (2, 3, 4), (1000,), (33, 17)]
NS = [1, 2, 3, 4, 5, 8]
DTYPES = ["f32", "f64"]


def _stitched(G, n, shape, dtype, build_site):
    """Build n replica inputs and, per replica site, one stitched collective node."""
    g = G.Graph()
    ins = [g.add_node("input", [], {"shape": shape, "dtype": dtype, "name": f"x{r}"}) for r in range(n)]
    sites = [build_site(g, ins, r) for r in range(n)]
    g.finalize()
    return g, ins, sites


def gen_folds(G, T):
    rng = np.random.default_rng(20190201)
    out = {}
    cases = []
    for dtype in DTYPES:
        npd = np.float32 if dtype == "f32" else np.float64
        for n in NS:
            for shape in SHAPES:
                xs = [rng.standard_normal(shape).astype(npd) for _ in range(n)]
                if shape and np.prod(shape) >= 7:
                    # ties / signed zeros for the max fold (np.maximum select rule)
                    xs[0].reshape(-1)[:2] = [0.0, -0.0]
                    if n > 1:
                        xs[1].reshape(-1)[:2] = [-0.0, 0.0]
                feeds_of = lambda ins: {ins[r]: T.Tensor(xs[r], dtype=dtype) for r in range(n)}
                key = f"{dtype}_n{n}_" + ("x".join(map(str, shape)) or "scalar")
                for r in range(n):
                    out[f"{key}_in{r}"] = xs[r]
                for kind, op in (("sum", "nary_sum"), ("mean", "nary_mean"), ("max", "nary_max")):
                    g, ins, sites = _stitched(G, n, shape, dtype, lambda g, ins, r, op=op: g.add_node(op, ins))
                    res = g.evaluate(sites, feeds_of(ins))
                    for r in range(1, n):
                        assert res[r].equals_bitwise(res[0])
                    out[f"{key}_{kind}"] = res[0].np
                # premean: all_sum(x / R) with the reference's div + nary_sum
                def premean_site(g, ins, r):
                    return g.add_node("nary_sum", [x / float(n) for x in ins])
                g, ins, sites = _stitched(G, n, shape, dtype, premean_site)
                res = g.evaluate(sites, feeds_of(ins))
                out[f"{key}_premean"] = res[0].np
                # gather (concat on axis 0; pack for rank-0) and broadcast (pick0)
                if shape == ():
                    gsite = lambda g, ins, r: g.add_node("pack", ins)
                else:
                    gsite = lambda g, ins, r: g.add_node("concat", ins, {"axis": 0})
                g, ins, sites = _stitched(G, n, shape, dtype, gsite)
                out[f"{key}_gather"] = g.evaluate(sites, feeds_of(ins))[0].np
                g, ins, sites = _stitched(G, n, shape, dtype, lambda g, ins, r: g.add_node("pick0", ins))
                res = g.evaluate(sites, feeds_of(ins))
                out[f"{key}_broadcast"] = res[n - 1].np
                cases.append(key)
    np.savez_compressed(os.path.join(GOLDEN, "folds.npz"), **out)
    return cases


class RecordingComm:
    """Duck-typed communicator (graph.py:565-583) that records what the seam passes."""

    def __init__(self, T, rank, n, peers):
        self.T, self.rank, self.n, self.peers, self.calls = T, rank, n, peers, []

    def all_reduce(self, local, kind, label):
        self.calls.append({"op": "all_reduce", "kind": kind, "label": label,
                           "shape": list(local.shape), "dtype": local.dtype})
        acc = self.peers[0]
        for p in self.peers[1:]:
            acc = acc + p if kind != "max" else np.maximum(acc, p)
        if kind == "mean":
            acc = acc / self.n
        return self.T.Tensor.wrap(np.asarray(acc, dtype=local.np.dtype).reshape(local.shape))

    def all_gather(self, local, label):
        self.calls.append({"op": "all_gather", "label": label, "shape": list(local.shape),
                           "dtype": local.dtype})
        return [self.T.Tensor.wrap(np.asarray(p, dtype=local.np.dtype).reshape(local.shape))
                for p in self.peers]

    def broadcast(self, root_value, label, shape=None, dtype=None):
        self.calls.append({"op": "broadcast", "label": label, "root_is_none": root_value is None,
                           "shape": list(shape), "dtype": dtype})
        return self.T.Tensor.wrap(np.asarray(self.peers[0]).reshape(shape).astype(
            np.float32 if dtype == "f32" else np.float64))


def gen_mesh_seam(G, T):
    """Pin the mesh seam's calling convention, including the 0-d defect (tensor.py:48)."""
    trace = []
    for shape in [(), (2, 3)]:
        for dtype in DTYPES:
            npd = np.float32 if dtype == "f32" else np.float64
            peers = [np.full(shape, float(r + 1), npd) for r in range(2)]
            for rank in range(2):
                g = G.Graph()
                x = g.add_node("input", [], {"shape": shape, "dtype": dtype})
                nodes = [g.add_node("mesh_collective", [x], {"ckind": k, "label": f"l_{k}", "num_replicas": 2})
                         for k in ("sum", "mean", "max", "gather", "broadcast")]
                g.finalize()
                comm = RecordingComm(T, rank, 2, peers)
                res = g.evaluate(nodes, {x: T.Tensor(peers[rank], dtype=dtype)}, runtime={"communicator": comm})
                trace.append({"shape": list(shape), "dtype": dtype, "rank": rank, "calls": comm.calls,
                              "out_shapes": [list(r.shape) for r in res],
                              "out_values": [r.np.reshape(-1).tolist() for r in res]})
    # missing communicator -> EvaluationError (graph.py:567-569)
    g = G.Graph()
    x = g.add_node("input", [], {"shape": (2,), "dtype": "f64"})
    y = g.add_node("mesh_collective", [x], {"ckind": "sum", "label": "z", "num_replicas": 2})
    g.finalize()
    try:
        g.evaluate([y], {x: T.Tensor([1.0, 2.0])})
        err = None
    except Exception as e:  # noqa: BLE001
        err = type(e).__name__
    with open(os.path.join(GOLDEN, "mesh_seam.json"), "w") as f:
        json.dump({"trace": trace, "no_communicator_error": err}, f, indent=1)


def gen_bn(G, T):
    """Cross-replica BN built from reference ops."""
    out = {}
    rng = np.random.default_rng(7)

    def bn_graph(hs, axis, eps=1e-5):
        n = len(hs)
        g = G.Graph()
        ins = [g.add_node("input", [], {"shape": h.shape, "dtype": "f64"}) for h in hs]
        means = [g.add_node("reduce_mean", [x], {"axis": axis}) / float(n) for x in ins]
        msqs = [g.add_node("reduce_mean", [g.add_node("square", [x])], {"axis": axis}) / float(n) for x in ins]
        outs = []
        for r in range(n):
            mean = g.add_node("nary_sum", means)
            msq = g.add_node("nary_sum", msqs)
            var = msq - mean * mean
            denom = g.add_node("sqrt", [var + eps])
            if axis is None:
                outs.append((ins[r] - mean) / denom)
            else:
                # per-channel: broadcast the [C] stats over the batch axis (ones(B,1) @ s(1,C))
                b = hs[r].shape[0]
                ones = g.add_node("const", [], {"value": T.Tensor(np.ones((b, 1)))})
                m2 = ones @ g.add_node("reshape", [mean], {"shape": (1, hs[r].shape[1])})
                d2 = ones @ g.add_node("reshape", [denom], {"shape": (1, hs[r].shape[1])})
                outs.append((ins[r] - m2) / d2)
        fetch_mean = g.add_node("nary_sum", means)
        fetch_msq = g.add_node("nary_sum", msqs)
        g.finalize()
        res = g.evaluate(outs + [fetch_mean, fetch_msq], {ins[r]: T.Tensor(hs[r]) for r in range(n)})
        return [r.np for r in res[:n]], res[n].np, res[n + 1].np

    # KAT: SPEC.md:521 h0=[1,3], h1=[5,7] -> mean 4, mean_sq 21, var 5
    ys, mean, msq = bn_graph([np.array([1.0, 3.0]), np.array([5.0, 7.0])], None)
    out["kat_mean"], out["kat_msq"] = mean, msq
    out["kat_y0"], out["kat_y1"] = ys
    for n in (2, 4):
        hs = [rng.standard_normal((6, 5)) * 3 + 1 for _ in range(n)]
        ys, mean, msq = bn_graph(hs, 0)
        for r in range(n):
            out[f"pc_n{n}_in{r}"] = hs[r]
            out[f"pc_n{n}_out{r}"] = ys[r]
        out[f"pc_n{n}_mean"], out[f"pc_n{n}_msq"] = mean, msq
        ys, mean, msq = bn_graph(hs, None)
        for r in range(n):
            out[f"pt_n{n}_out{r}"] = ys[r]
        out[f"pt_n{n}_mean"], out[f"pt_n{n}_msq"] = mean, msq
    hs = [np.full((4, 3), 2.5) for _ in range(2)]       # constant input -> 0
    ys, _, _ = bn_graph(hs, 0)
    out["const_out0"] = ys[0]
    np.savez_compressed(os.path.join(GOLDEN, "bn.npz"), **out)


def gen_wrap_sgd(G, T, V):
    """wrap_optimizer + SGD on mirrored replicas with the reference engine."""
    out = {}

    def mlp_grads(dims, dtype, xs, ys, w_init):
        """Per-replica gradients of mean softmax-xent of a tanh MLP (reference backprop)."""
        grads = []
        for x, y in zip(xs, ys):
            g = G.Graph(V.VariableStore())
            vars_ = []
            for i, w in enumerate(w_init):
                v = g.variables.get_or_create(f"p{i}", w.shape, dtype=dtype)
                v.assign(w)
                vars_.append(v)
            h = g.add_node("input", [], {"shape": x.shape, "dtype": dtype})
            lab = g.add_node("input", [], {"shape": y.shape, "dtype": dtype})
            a = h
            for li in range(len(dims) - 1):
                wr = g.add_node("var_read", [], {"var": vars_[2 * li]})
                br = g.add_node("var_read", [], {"var": vars_[2 * li + 1]})
                ones = g.add_node("const", [], {"value": T.Tensor(np.ones((x.shape[0], 1)), dtype=dtype)})
                a = a @ wr + ones @ br
                if li < len(dims) - 2:
                    a = g.add_node("relu", [a])
            loss = g.add_node("reduce_mean", [g.add_node("softmax_cross_entropy", [a, lab])], {"axis": None})
            gr = G.backprop(g, loss, vars_)
            g.finalize()
            res = g.evaluate(gr, {h: T.Tensor(x, dtype=dtype), lab: T.Tensor(y, dtype=dtype)})
            grads.append([r.np for r in res])
        return grads

    def stitched_premean(grads, dtype):
        n = len(grads)
        avgs = []
        for i in range(len(grads[0])):
            g = G.Graph()
            ins = [g.add_node("input", [], {"shape": grads[r][i].shape, "dtype": dtype}) for r in range(n)]
            site = g.add_node("nary_sum", [x / float(n) for x in ins])
            g.finalize()
            avgs.append(g.evaluate([site], {ins[r]: T.Tensor(grads[r][i], dtype=dtype) for r in range(n)})[0].np)
        return avgs

    rng = np.random.default_rng(11)
    # small f64 MLP, R=2 and R=4
    dims = (12, 16, 10)
    for n in (2, 4):
        w_init = []
        for li in range(len(dims) - 1):
            w_init += [rng.uniform(-0.3, 0.3, (dims[li], dims[li + 1])), rng.uniform(-0.1, 0.1, (1, dims[li + 1]))]
        xs = [rng.standard_normal((8, dims[0])) for _ in range(n)]
        ys = [np.eye(dims[-1])[rng.integers(0, dims[-1], 8)] for _ in range(n)]
        grads = mlp_grads(dims, "f64", xs, ys, w_init)
        avgs = stitched_premean(grads, "f64")
        for i, w in enumerate(w_init):
            out[f"small_n{n}_w{i}"] = w
            out[f"small_n{n}_avg{i}"] = avgs[i]
            out[f"small_n{n}_new{i}"] = w - 0.1 * avgs[i]
            for r in range(n):
                out[f"small_n{n}_g{r}_{i}"] = grads[r][i]
    # config 1 (BASELINE.json configs[0]): 784-256-10, B=64/replica, R=2, f32, SGD lr 0.1, seed 0
    rng = np.random.default_rng(0)
    dims = (784, 256, 10)
    w_init = []
    for li in range(2):
        s = np.sqrt(6.0 / (dims[li] + dims[li + 1]))
        w_init += [rng.uniform(-s, s, (dims[li], dims[li + 1])).astype(np.float32),
                   np.zeros((1, dims[li + 1]), np.float32)]
    xs = [rng.standard_normal((64, 784)).astype(np.float32) for _ in range(2)]
    ys = [np.eye(10, dtype=np.float32)[rng.integers(0, 10, 64)] for _ in range(2)]
    grads = mlp_grads(dims, "f32", xs, ys, w_init)
    avgs = stitched_premean(grads, "f32")
    for i in range(4):
        for r in range(2):
            out[f"cfg1_g{r}_{i}"] = grads[r][i]
    md5 = lambda arrs: hashlib.md5(b"".join(np.ascontiguousarray(a).tobytes() for a in arrs)).hexdigest()
    meta = {"cfg1_avg_md5": md5(avgs),
            "cfg1_new_md5": md5([w_init[i] - np.float32(0.1) * avgs[i] for i in range(4)]),
            "cfg1_w_md5": md5(w_init),
            "cfg1_shapes": [list(a.shape) for a in avgs]}
    np.savez_compressed(os.path.join(GOLDEN, "wrap_sgd.npz"), **out)
    with open(os.path.join(GOLDEN, "wrap_sgd.json"), "w") as f:
        json.dump(meta, f, indent=1)


def main():
    os.makedirs(GOLDEN, exist_ok=True)
    T, G, V, E = ref_adapter.load()
    cases = gen_folds(G, T)
    gen_mesh_seam(G, T)
    gen_bn(G, T)
    gen_wrap_sgd(G, T, V)
    with open(os.path.join(GOLDEN, "README.md"), "w") as f:
        f.write("# Golden fixtures\n\nGenerated by `python -m oracle.make_golden` from the reference package "
                "(`/root/reference/pkg/src/replicator`, with the 0-d shim of `oracle/ref_adapter.py`).\n\n"
                f"* `folds.npz`: {len(cases)} cases (dtype x N x shape); per case inputs `_in<r>` and the stitched "
                "reference outputs `_sum/_mean/_max/_premean/_gather/_broadcast` (graph.py:506-540).\n"
                "* `mesh_seam.json`: what `_mesh_collective_kernel` (graph.py:565-583) hands a communicator.\n"
                "* `bn.npz`: cross-replica BN built from reference ops (PAPER.md:213-219, SPEC.md:521-523).\n"
                "* `wrap_sgd.npz/json`: per-replica gradients from reference `backprop` and the stitched "
                "`all_sum(g/R)` average (PAPER.md:196-206); config 1 (784-256-10, R=2, f32) pinned by md5.\n")


if __name__ == "__main__":
    main()
