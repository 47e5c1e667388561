"""CPU restatement of the reference solver's KKT assembly (TEST INFRASTRUCTURE:
imported only by tests/ and tools/, never by the product path).

Follows ``/root/reference/pkg/src/simdnlp/solver.py`` line by line:

* 421-424  sigma = sigma_lo + sigma_up (given here as an input)
* 425-429  K = 0; W[hrows, hcols] = hvals; K[:nx, :nx] = W + W.T - diag(diag W)
* 430      K[i, i] += sigma  for i < nz = nx + m
* 431-435  K[nz + jrows, jcols] = jvals (and transposed);
           K[nx + i, nz + i] = K[nz + i, nx + i] = -1  (slacks)
* 442-445  fixed rows / cols zeroed, K[fixed, fixed] = 1
* 452-456  Kt = K.copy(); Kt[free, free] += delta_w; if m and delta_c:
           Kt[yi, yi] -= delta_c

Pinned bit-for-bit against the reference's own Kt (captured from a real
``solve`` by ``tools/make_kkt_goldens.py``, ``tests/golden/kkt_*.npz``).
"""

from __future__ import annotations

import numpy as np


def kkt_dense(nx, m, hrows, hcols, hvals, jrows, jcols, jvals, sigma, fixed, delta_w, delta_c):
    nz = nx + m
    n_kkt = nz + m
    K = np.zeros((n_kkt, n_kkt))
    W = np.zeros((nx, nx))
    W[hrows, hcols] = hvals
    K[:nx, :nx] = W + W.T - np.diag(np.diag(W))
    K[np.arange(nz), np.arange(nz)] += sigma
    if m:
        K[nz + jrows, jcols] = jvals
        K[jcols, nz + jrows] = jvals
        si = np.arange(m)
        K[nx + si, nz + si] = -1.0
        K[nz + si, nx + si] = -1.0
    fixed_idx = np.flatnonzero(fixed)
    free_idx = np.flatnonzero(~np.asarray(fixed, dtype=bool))
    if fixed_idx.size:
        K[fixed_idx, :] = 0.0
        K[:, fixed_idx] = 0.0
        K[fixed_idx, fixed_idx] = 1.0
    Kt = K.copy()
    Kt[free_idx, free_idx] += delta_w
    if m and delta_c:
        yi = np.arange(nz, n_kkt)
        Kt[yi, yi] -= delta_c
    return Kt
