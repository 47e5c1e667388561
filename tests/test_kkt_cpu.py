"""KKT assembly, host side: the oracle restatement of the
reference solver's dense assembly reproduces the reference's own Kt (captured
from simdnlp.solve by tools/make_kkt_goldens.py) bit for bit, and the CSR
pattern + per-entry descriptors of kkt.KKTSystem, interpreted on the host,
give exactly the lower triangle of that Kt."""

import numpy as np
import pytest

from fixture_models import build, load
from oracle.kkt_oracle import kkt_dense
from paper_2510_12897_b200.kkt import (K_DIAG, K_DUAL, K_H_DIAG, K_H_OFF, K_JAC, K_ONE, K_SLACK, K_ZERO,
                                       KKTSystem)
from pathlib import Path

GOLD = Path(__file__).resolve().parent / "golden"
CASES = ["case3", "case5", "case14"]


def _gold(case):
    with np.load(GOLD / f"kkt_{case}.npz") as z:
        return {k: z[k] for k in z.files}


def interpret(sys_, h, j, sigma, dw, dc):
    """Host interpreter of the descriptor semantics of exa_kkt_values."""
    kind = (sys_.desc[:, 0].astype(np.int64) & 0xFFFFFFFF) >> 29
    a = sys_.desc[:, 0].astype(np.int64) & ((1 << 29) - 1)
    b = sys_.desc[:, 1].astype(np.int64)
    out = np.empty(sys_.nnz)
    for p in range(sys_.nnz):
        k = kind[p]
        if k == K_H_OFF:
            out[p] = (h[a[p]] + 0.0) - 0.0
        elif k == K_H_DIAG:
            out[p] = (((h[a[p]] + h[a[p]]) - h[a[p]]) + sigma[b[p]]) + dw
        elif k == K_DIAG:
            out[p] = (0.0 + sigma[b[p]]) + dw
        elif k == K_JAC:
            out[p] = j[a[p]]
        elif k == K_SLACK:
            out[p] = -1.0
        elif k == K_DUAL:
            out[p] = 0.0 - dc if dc != 0.0 else 0.0
        elif k == K_ZERO:
            out[p] = 0.0
        else:
            assert k == K_ONE
            out[p] = 1.0
    return out


@pytest.mark.parametrize("case", CASES)
def test_oracle_restatement_reproduces_reference_kkt(case):
    g = _gold(case)
    K = kkt_dense(int(g["nx"]), int(g["m"]), g["hrows"], g["hcols"], g["hvals"], g["jrows"], g["jcols"],
                  g["jvals"], g["sigma"], g["fixed"], 0.0, 0.0)
    assert np.array_equal(K, g["Kt"]) and np.array_equal(np.signbit(K), np.signbit(g["Kt"]))


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("dw,dc", [(0.0, 0.0), (1e-4, 1e-8), (-0.0, 0.0)])
def test_csr_descriptors_equal_reference_lower_triangle(case, dw, dc):
    g = _gold(case)
    model = build(f"{case}_polar", lower_to_gpu=False, data=load(f"{case}_polar"))
    ks = KKTSystem(model)
    assert np.array_equal(ks.hpat.rows, g["hrows"]) and np.array_equal(ks.jpat.cols, g["jcols"])
    assert np.array_equal(ks.fixed, g["fixed"])
    vals = interpret(ks, g["hvals"], g["jvals"], g["sigma"], dw, dc)
    K = kkt_dense(int(g["nx"]), int(g["m"]), g["hrows"], g["hcols"], g["hvals"], g["jrows"], g["jcols"],
                  g["jvals"], g["sigma"], g["fixed"], dw, dc)
    if dw == 0.0 and dc == 0.0:
        assert np.array_equal(K, g["Kt"])
    indptr, indices = ks.structure()
    rows = np.repeat(np.arange(ks.n), np.diff(indptr))
    assert np.all(rows >= indices)  # lower triangle
    lo = np.tril(K)
    assert np.array_equal(vals, lo[rows, indices]) and np.array_equal(np.signbit(vals), np.signbit(lo[rows, indices]))
    # every structurally nonzero entry of the reference's K is in the pattern
    mask = np.zeros_like(lo, dtype=bool)
    mask[rows, indices] = True
    assert not np.any((lo != 0.0) & ~mask)
