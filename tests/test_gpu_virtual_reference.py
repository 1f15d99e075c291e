"""The reference's own engine with this repo's kernels plugged into its op registry
(seam 2, graph.py:123-135): the in-process MultiDevice stitching
 rewritten onto ``gpu_nary`` / ``gpu_gather`` / ``gpu_pick0``
(paper_1902_00465_b200/ref_seam.py) must give the SAME bits as the reference's
``nary_sum / nary_mean / nary_max``, ``pack`` / ``concat`` and ``pick0`` on the
same graph, replica site by replica site -- including the wrap_optimizer premean
(``nary_sum`` over ``x / R`` nodes).

Seam 1 (the mesh communicator driven by ``Graph.evaluate``) is exercised by
``body_reference_graph`` in test_gpu_world_loopback.py / test_gpu_multiproc.py.

The reference package comes from ``oracle/_ref`` (oracle/ref_vendor.py), test
infrastructure only: here it is the checker and the graph engine that calls the
product, never the product itself.
"""

import numpy as np
import pytest

from oracle import ref_adapter

pytestmark = pytest.mark.gpu

if not ref_adapter.available():
    pytest.skip("reference package not vendored (oracle/ref_vendor.py)", allow_module_level=True)


@pytest.fixture(scope="module")
def ref():
    from paper_1902_00465_b200 import ref_seam

    T, G, _, E = ref_adapter.load()
    comms = ref_seam.register(G, device=0)
    yield T, G, E
    comms.close()


def _stitched_pair(G, n, shape, dtype, build):
    """The same replicated graph twice: reference kinds and GPU kinds."""
    out = []
    for gpu in (False, True):
        g = G.Graph()
        ins = [g.add_node("input", [], {"shape": shape, "dtype": dtype, "name": f"x{r}"}) for r in range(n)]
        sites = [build(g, ins, gpu) for _ in range(n)]  # one node per replica site
        g.finalize()
        out.append((g, ins, sites))
    return out


FOLD = {"sum": "nary_sum", "mean": "nary_mean", "max": "nary_max"}


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("shape", [(), (7,), (3, 5), (33, 17), (4097,)])
def test_stitched_folds_on_gpu_kinds_match_reference(ref, dtype, n, shape):
    T, G, _ = ref
    npd = np.float32 if dtype == "f32" else np.float64
    rng = np.random.default_rng(hash((dtype, n, shape)) & 0xFFFF)
    xs = [rng.standard_normal(shape).astype(npd) for _ in range(n)]
    if shape and np.prod(shape) >= 2:  # signed zeros: the np.maximum select rule
        xs[0].reshape(-1)[:2] = [0.0, -0.0]
        if n > 1:
            xs[1].reshape(-1)[:2] = [-0.0, 0.0]

    def builders():
        for kind, op in FOLD.items():
            yield kind, (lambda g, ins, gpu, kind=kind, op=op:
                         g.add_node("gpu_nary", ins, {"ckind": kind}) if gpu else g.add_node(op, ins))
        # wrap_optimizer's all_sum(g / R): the reference divides in its own nodes;
        # the GPU kind fuses the division into the fold (same bits)
        yield "premean", (lambda g, ins, gpu:
                          g.add_node("gpu_nary", ins, {"ckind": "premean"}) if gpu
                          else g.add_node("nary_sum", [x / float(n) for x in ins]))
        yield "gather", (lambda g, ins, gpu:
                         g.add_node("gpu_gather", ins) if gpu
                         else (g.add_node("pack", ins) if shape == () else g.add_node("concat", ins, {"axis": 0})))
        yield "broadcast", (lambda g, ins, gpu: g.add_node("gpu_pick0" if gpu else "pick0", ins))

    for kind, build in builders():
        (g0, i0, s0), (g1, i1, s1) = _stitched_pair(G, n, shape, dtype, build)
        r0 = g0.evaluate(s0, {i: T.Tensor(x, dtype=dtype) for i, x in zip(i0, xs)})
        r1 = g1.evaluate(s1, {i: T.Tensor(x, dtype=dtype) for i, x in zip(i1, xs)})
        for site, (a, b) in enumerate(zip(r0, r1)):
            assert a.shape == b.shape and a.dtype == b.dtype, (kind, site, a.shape, b.shape)
            assert a.equals_bitwise(b), (kind, dtype, n, shape, site)


def test_gpu_kinds_keep_the_reference_errors(ref):
    """Shape errors come from the reference's own inference (graph.py:506-512)."""
    T, G, E = ref
    g = G.Graph()
    a = g.add_node("input", [], {"shape": (3,), "dtype": "f32"})
    b = g.add_node("input", [], {"shape": (4,), "dtype": "f32"})
    with pytest.raises(E.ShapeError):
        g.add_node("gpu_nary", [a, b], {"ckind": "sum"})
