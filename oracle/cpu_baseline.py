"""The reference's CPU path for the bench's cpu_baseline / --impl reference arm.
TEST/BENCH INFRASTRUCTURE ONLY (imported by bench.py's CPU legs, never by the product).

``time_reference``: the REFERENCE ITSELF (``oracle/_ref``, oracle/ref_vendor.py) --
its own ``Graph.evaluate`` on the stitched in-process program of one step, built
from its own kinds (per replica a ``div`` by R, then one ``nary_sum`` site per
replica over all replicas: wrap_optimizer's all_sum(g/R), PAPER.md:196-206,
graph.py:514-522). numpy runs it on one core.

``time_port``: port of what the reference executes for a stitched MultiDevice all-reduce step
(SURVEY.md §3.1): every one of the N replica sites is an ``nary_mean`` /
``nary_sum`` node over all N replicas' inputs, evaluated by ``_fold_*``
(graph.py:514-528), which allocates a fresh array per addition -- so one step
is N folds of N inputs. ``threads > 1`` splits the flat message into contiguous
slices folded concurrently (numpy releases the GIL inside ufuncs); per-element
arithmetic and order are unchanged.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .collectives import FOLDS


def stitched_step(xs, kind):
    """One evaluation of the stitched program: N sites, each an N-way fold."""
    return [FOLDS[kind](xs) for _ in range(len(xs))]


def make_inputs(n, count, dtype=np.float32, seed=1234):
    return [np.random.default_rng(seed + r).standard_normal(count, dtype=np.float32).astype(dtype, copy=False)
            for r in range(n)]


def time_port(n, count, kind="premean", budget_s=10.0, threads=1, max_steps=1000, xs=None):
    """Run whole stitched steps until ``budget_s`` elapses (at least one).
    Returns (seconds_per_step, steps_run, threads_used)."""
    xs = make_inputs(n, count) if xs is None else xs
    threads = max(1, int(threads))
    if threads == 1:
        def step():
            stitched_step(xs, kind)
    else:
        bounds = np.linspace(0, count, threads + 1).astype(np.int64)
        slices = [[x[bounds[t]:bounds[t + 1]] for x in xs] for t in range(threads)]
        pool = ThreadPoolExecutor(threads)

        def step():
            list(pool.map(lambda s: stitched_step(s, kind), slices))
    step()  # warm (page faults)
    steps, t0 = 0, time.perf_counter()
    while True:
        step()
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or steps >= max_steps:
            break
    return el / steps, steps, threads


def reference_program(n, count, kind="premean"):
    """Build the reference's own stitched program for one all-reduce step.
    Returns (graph, input nodes, site nodes, Tensor class)."""
    from . import ref_adapter

    T, G, _, _ = ref_adapter.load()
    g = G.Graph()
    ins = [g.add_node("input", [], {"shape": (count,), "dtype": "f32", "name": f"g{r}"}) for r in range(n)]
    if kind == "premean":
        parts = [x / float(n) for x in ins]
        sites = [g.add_node("nary_sum", parts) for _ in range(n)]
    else:
        op = {"sum": "nary_sum", "mean": "nary_mean", "max": "nary_max"}[kind]
        sites = [g.add_node(op, ins) for _ in range(n)]
    g.finalize()
    return g, ins, sites, T


def time_reference(n, count, kind="premean", budget_s=10.0, max_steps=1000, warmup=1, xs=None):
    """Time whole steps of the reference's own Graph.evaluate (see the module doc)
    until ``budget_s`` elapses (at least one). Returns (seconds_per_step, steps, 1)."""
    xs = make_inputs(n, count) if xs is None else xs
    g, ins, sites, T = reference_program(n, count, kind)
    feeds = {i: T.Tensor(x, dtype="f32") for i, x in zip(ins, xs)}
    for _ in range(max(1, warmup)):
        g.evaluate(sites, feeds)
    steps, t0 = 0, time.perf_counter()
    while True:
        g.evaluate(sites, feeds)
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or steps >= max_steps:
            break
    return el / steps, steps, 1


def reference_available() -> bool:
    from . import ref_adapter

    return ref_adapter.available()


def host_cores() -> int:
    return len(os.sched_getaffinity(0))
