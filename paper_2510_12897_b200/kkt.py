"""KKT assembly for the reference's interior-point solver, on the GPU
(the caller on the other side of the callback boundary).

The reference solver (``solver.py:421-456``) builds, every iteration, the
dense symmetric matrix over (x, s, y) with nz = nvar + ncon::

    K[:nx, :nx]      = W + W^T - diag(W)     W[hrows, hcols] = compressed H
    K[i, i]         += sigma[i]              i < nz
    K[nz + jr, jc]   = compressed J          (and transposed)
    K[nx + i, nz + i] = K[nz + i, nx + i] = -1
    fixed rows / columns (lower == upper) zeroed, K[fixed, fixed] = 1
    Kt = K;  Kt[free, free] += delta_w;  if m and delta_c: Kt[y, y] -= delta_c

Dense K cannot scale (case13659: 458k x 458k).  :class:`KKTSystem` keeps the
same values in a lower-triangle CSR whose pattern -- and, for every CSR
entry, a descriptor of where its value comes from and which of the
reference's operations produce it -- is built once on the host.  Each
iteration is then one gather kernel (``exa_kkt_values``) over the compressed
J/H values (``CompressedPattern.sum_values``), sigma and the two
regularisations, bit-identical to the reference's K entries (including the
sign of zeros), deterministic, no atomics.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .autodiff import compress_coordinates, hessian_structure, jacobian_structure

K_H_OFF, K_H_DIAG, K_DIAG, K_JAC, K_SLACK, K_DUAL, K_ZERO, K_ONE = range(8)
_IDX_BITS = 29


class KKTSystem:
    """Lower-triangle CSR of the reference IPM's KKT matrix for one model."""

    def __init__(self, model):
        self.model = model
        nx, m = model.nvar, model.ncon
        nz = nx + m
        self.nx, self.m, self.nz, self.n = nx, m, nz, nz + m
        self.jpat = compress_coordinates(*jacobian_structure(model))
        self.hpat = compress_coordinates(*hessian_structure(model))
        zlo = np.concatenate([np.asarray(model.lower, dtype=np.float64), np.asarray(model.con_lower, dtype=np.float64)])
        zhi = np.concatenate([np.asarray(model.upper, dtype=np.float64), np.asarray(model.con_upper, dtype=np.float64)])
        self.fixed = zlo == zhi  # solver.py:307
        fixed = self.fixed
        if max(self.hpat.nnz, self.jpat.nnz, nz) >= (1 << _IDX_BITS):
            raise ValueError("KKT system too large for the 29-bit descriptor indices")

        hr, hc = self.hpat.rows, self.hpat.cols
        hk = np.arange(hr.size, dtype=np.int64)
        on_diag = hr == hc
        # x-block off-diagonal H entries
        r_l = [hr[~on_diag]]
        c_l = [hc[~on_diag]]
        kind_l = [np.where(fixed[hr[~on_diag]] | fixed[hc[~on_diag]], K_ZERO, K_H_OFF)]
        a_l = [hk[~on_diag]]
        b_l = [np.zeros((~on_diag).sum(), dtype=np.int64)]
        # primal + slack diagonal (with or without an H diagonal entry)
        diag_h = np.full(nz, -1, dtype=np.int64)
        diag_h[hr[on_diag]] = hk[on_diag]
        i = np.arange(nz, dtype=np.int64)
        kd = np.where(diag_h >= 0, K_H_DIAG, K_DIAG)
        kd = np.where(fixed, K_ONE, kd)
        r_l.append(i)
        c_l.append(i)
        kind_l.append(kd)
        a_l.append(np.maximum(diag_h, 0))
        b_l.append(i)
        if m:
            jr, jc = self.jpat.rows, self.jpat.cols
            r_l.append(nz + jr)
            c_l.append(jc)
            kind_l.append(np.where(fixed[jc], K_ZERO, K_JAC))
            a_l.append(np.arange(jr.size, dtype=np.int64))
            b_l.append(np.zeros(jr.size, dtype=np.int64))
            si = np.arange(m, dtype=np.int64)
            r_l.append(nz + si)
            c_l.append(nx + si)
            kind_l.append(np.where(fixed[nx + si], K_ZERO, K_SLACK))
            a_l.append(np.zeros(m, dtype=np.int64))
            b_l.append(np.zeros(m, dtype=np.int64))
            r_l.append(nz + si)
            c_l.append(nz + si)
            kind_l.append(np.full(m, K_DUAL))
            a_l.append(np.zeros(m, dtype=np.int64))
            b_l.append(np.zeros(m, dtype=np.int64))
        rows, cols = np.concatenate(r_l), np.concatenate(c_l)
        order = np.lexsort((cols, rows))
        rows, cols = rows[order], cols[order]
        if rows.size > 1 and np.any((rows[1:] == rows[:-1]) & (cols[1:] == cols[:-1])):
            raise ValueError("duplicate KKT entries")  # pragma: no cover - construction invariant
        kind = np.concatenate(kind_l)[order].astype(np.int64)
        a = np.concatenate(a_l)[order]
        b = np.concatenate(b_l)[order]
        self.indptr = np.zeros(self.n + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, minlength=self.n), out=self.indptr[1:])
        self.indices = cols.astype(np.int64)
        self.desc = np.stack([(kind << _IDX_BITS) | a, b], axis=1).astype(np.int32)
        self.nnz = int(rows.size)
        self._dev = None

    # -------------------------------------------------------------- structure
    def structure(self):
        """(indptr, indices) of the lower triangle, rows ascending, columns
        ascending within a row (copies)."""
        return self.indptr.copy(), self.indices.copy()

    def dense(self, vals) -> np.ndarray:
        """Symmetric dense matrix from lower-triangle CSR values (testing)."""
        K = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.indptr))
        K[rows, self.indices] = vals
        K[self.indices, rows] = vals
        return K

    # ----------------------------------------------------------------- values
    def values(self, hvals, jvals, sigma, delta_w: float = 0.0, delta_c: float = 0.0, out=None):
        """CSR values of Kt for compressed H values ``hvals`` (``hpat`` order),
        compressed J values ``jvals`` (``jpat`` order), ``sigma`` (nz) and the
        inertia regularisations.  torch CUDA tensors in -> device tensor out
        (zero-copy, current stream); numpy in -> numpy out."""
        import torch

        if not torch.cuda.is_available():
            raise _lib.ExaError("no CUDA device: the callback engine runs on B200 only (no CPU path)")
        host = not getattr(hvals, "is_cuda", False)
        dev = torch.device("cuda", torch.cuda.current_device()) if host else hvals.device

        def dv(a, n, what):
            t = a if getattr(a, "is_cuda", False) else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            t = t.to(dev, torch.float64).contiguous()
            if t.numel() != n:
                raise ValueError(f"{what} has length {t.numel()}, expected {n}")
            return t

        h = dv(hvals, self.hpat.nnz, "hvals")
        j = dv(jvals, self.jpat.nnz, "jvals")
        sg = dv(sigma, self.nz, "sigma")
        if self._dev is None or self._dev.device != dev:
            self._dev = torch.from_numpy(self.desc).to(dev)
        o = out if (out is not None and getattr(out, "is_cuda", False)) else torch.empty(self.nnz, dtype=torch.float64,
                                                                                           device=dev)
        s = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        _lib.check(_lib.load().exa_kkt_values(self.nnz, self._dev.data_ptr(), h.data_ptr(), j.data_ptr(),
                                              sg.data_ptr(), float(delta_w), float(delta_c), o.data_ptr(), s),
                   "exa_kkt_values")
        if host:
            res = o.cpu().numpy()
            if out is not None:
                out[:] = res
                return out
            return res
        return o
