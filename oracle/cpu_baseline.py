"""The reference's CPU path for the bench's cpu_baseline / --impl reference arm.
TEST/BENCH INFRASTRUCTURE ONLY (imported by bench.py's CPU legs, never by the product).

Port of what the reference executes for a stitched MultiDevice all-reduce step
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


def host_cores() -> int:
    return len(os.sched_getaffinity(0))
