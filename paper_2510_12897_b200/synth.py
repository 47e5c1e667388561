"""Synthetic pglib-shaped networks and evaluation points.

The benchmark cases (case1354_pegase, case2000_goc, case13659_pegase) are not
shipped with the reference, so networks with their element counts are
generated from a seed: a random spanning tree plus random chords, pglib-like
parameter ranges, a few taps and phase shifters, some shunts (including
``Gs != 0`` so the ``-pd - gs*vm^2`` balance variant is exercised).

``random_interior_point`` restates reference ``derivcheck.py:28-44`` so the
evaluation point of a benchmark can be generated on the GPU box.
"""

from __future__ import annotations

import math

import numpy as np

from .matpower import Branch, Bus, CaseData, Gen

# (n_bus, n_gen, n_branch) of the pglib-opf cases the benchmark configs name
PGLIB_SHAPES = {
    "case14": (14, 5, 20),
    "case1354": (1354, 260, 1991),
    "case2000": (2000, 238, 3639),
    "case13659": (13659, 4092, 20467),
}


def synthetic_case(n_bus: int, n_gen: int, n_branch: int, seed: int = 1, name: str | None = None,
                   base_mva: float = 100.0) -> CaseData:
    if n_branch < n_bus - 1:
        raise ValueError("need at least n_bus - 1 branches for a spanning tree")
    rng = np.random.default_rng(seed)
    # topology: random spanning tree (each new bus attaches to an earlier one) + chords
    order = rng.permutation(n_bus)
    ends = []
    for k in range(1, n_bus):
        ends.append((order[rng.integers(0, k)], order[k]))
    while len(ends) < n_branch:
        a, b = rng.integers(0, n_bus, size=2)
        if a != b:
            ends.append((a, b))
    ends = np.array(ends, dtype=np.int64)
    flip = rng.random(n_branch) < 0.5
    ends[flip] = ends[flip][:, ::-1]

    gen_bus = np.concatenate([[0], rng.choice(np.arange(1, n_bus), size=n_gen - 1, replace=True)]) \
        if n_gen > 0 else np.zeros(0, dtype=np.int64)
    has_gen = np.zeros(n_bus, dtype=bool)
    has_gen[gen_bus] = True

    pd_mw = np.where(rng.random(n_bus) < 0.6, rng.uniform(0.0, 100.0, n_bus), 0.0)
    qd_mw = 0.3 * pd_mw
    bs = np.where(rng.random(n_bus) < 0.05, rng.uniform(0.0, 20.0, n_bus), 0.0)
    gs = np.where(rng.random(n_bus) < 0.02, rng.uniform(0.0, 5.0, n_bus), 0.0)
    buses = []
    for k in range(n_bus):
        btype = 3 if k == 0 else (2 if has_gen[k] else 1)
        buses.append(Bus(k + 1, btype, pd_mw[k] / base_mva, qd_mw[k] / base_mva,
                         gs[k] / base_mva, bs[k] / base_mva, 1.1, 0.9))

    pmax = rng.uniform(50.0, 500.0, n_gen)
    c2 = rng.uniform(0.0, 0.1, n_gen)
    c1 = rng.uniform(5.0, 50.0, n_gen)
    c0 = rng.uniform(0.0, 100.0, n_gen)
    gens = [
        Gen(int(gen_bus[g]) + 1, 0.0, pmax[g] / base_mva, -0.5 * pmax[g] / base_mva,
            0.5 * pmax[g] / base_mva, 1, float(c2[g]), float(c1[g]), float(c0[g]))
        for g in range(n_gen)
    ]

    r = rng.uniform(0.001, 0.05, n_branch)
    x = r + rng.uniform(0.01, 0.3, n_branch)
    bc = rng.uniform(0.0, 0.1, n_branch)
    rate = rng.uniform(100.0, 1000.0, n_branch)
    tap = np.where(rng.random(n_branch) < 0.10, rng.uniform(0.95, 1.05, n_branch), 1.0)
    shift = np.where(rng.random(n_branch) < 0.02, rng.uniform(-5.0, 5.0, n_branch), 0.0)
    d2r = math.pi / 180.0
    branches = [
        Branch(int(ends[k, 0]) + 1, int(ends[k, 1]) + 1, float(r[k]), float(x[k]), float(bc[k]),
               rate[k] / base_mva, float(tap[k]), shift[k] * d2r, 1, -30.0 * d2r, 30.0 * d2r)
        for k in range(n_branch)
    ]
    return CaseData(name or f"synthetic{n_bus}", base_mva, buses, gens, branches)


def pglib_shaped(name: str, seed: int = 1) -> CaseData:
    nb, ng, nbr = PGLIB_SHAPES[name]
    return synthetic_case(nb, ng, nbr, seed=seed, name=f"{name}_synthetic")


def random_interior_point(model, rng: np.random.Generator) -> np.ndarray:
    """Point strictly inside the bounds near the start (``derivcheck.py:28-44``)."""
    lo, hi = model.lower, model.upper
    x = model.start.copy()
    u = rng.uniform(-1.0, 1.0, size=model.nvar)
    boxed = np.isfinite(lo) & np.isfinite(hi)
    x[boxed] = 0.5 * (lo[boxed] + hi[boxed]) + 0.3 * u[boxed] * (hi - lo)[boxed]
    free = ~boxed
    x[free] = (model.start + 0.3 * u)[free]
    return np.clip(x, lo, hi)


def evaluation_point(model, seed: int = 0):
    """(x, y, obj_weight) used by the benchmark and parity tests."""
    rng = np.random.default_rng(seed)
    x = random_interior_point(model, rng)
    y = rng.uniform(-1.0, 1.0, size=model.ncon)
    return x, y, 1.0


def demand_curve(T: int) -> np.ndarray:
    """96-point style load curve 0.8 + 0.2 sin(2 pi t / T)."""
    t = np.arange(T, dtype=np.float64)
    return 0.8 + 0.2 * np.sin(2.0 * np.pi * t / T)
