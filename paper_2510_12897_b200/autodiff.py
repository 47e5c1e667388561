"""The five evaluation callbacks plus structures and compression.

Same names, signatures, validation and error behaviour as the reference's
``simdnlp/autodiff.py`` (536-689), executed by the model's generated sm_100a
kernels through ``libexa.so``:

* numpy arrays in / out  -> drop-in path: inputs copied to HBM, outputs
  copied back into the caller's array;
* torch CUDA float64 tensors -> zero-copy path: kernels read and write the
  caller's device memory on the current torch stream.

There is no CPU evaluation path; without a CUDA device these raise.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib


class EvalDomainError(ArithmeticError):
    """Numeric-domain violation (log/sqrt/div/pow) located in a block/record
    (reference ``autodiff.py:30-47``)."""

    def __init__(self, op: str, record: int, kind: str = "?", block_index: int = -1):
        self.op = op
        self.record = record
        self.kind = kind
        self.block_index = block_index
        super().__init__(op, record)

    def located(self, kind: str, block_index: int) -> "EvalDomainError":
        return EvalDomainError(self.op, self.record, kind, block_index)

    def __str__(self) -> str:
        return f"domain error in {self.op!r} at {self.kind} block {self.block_index}, record {self.record}"


_CHECK_OP = {"log": "log", "sqrt": "sqrt", "div": "div", "ipow": "pow", "pow": "pow"}


def _torch():
    import torch

    return torch


def _dplan(model):
    dp = model.device_plan
    if dp is None:
        dp = model.to_device()
    return dp


def _dplan_batch(model):
    """Device plan for strided batches: a batch is many waves, where term
    groups of two beat the one-wave grouping of four (case13659 x8: 73% vs
    64% of the HBM peak), so single-wave models get a second plan."""
    dp = _dplan(model)
    if dp.layout.group_max <= 2:
        return dp
    bp = getattr(model, "_exa_batch_plan", None)
    if bp is None or bp.device != dp.device:
        from .device import DevicePlan

        bp = DevicePlan(model, dp.device, group_max=2)
        model._exa_batch_plan = bp
    return bp


def _is_cuda(a) -> bool:
    return getattr(a, "is_cuda", False)


class _Stage:
    """Maps caller arrays to device pointers; copies numpy outputs back."""

    def __init__(self, dp):
        torch = _torch()
        self.torch = torch
        dev = dp.__dict__.get("_torch_dev")
        if dev is None:
            dev = dp._torch_dev = torch.device("cuda", dp.device)
        self.dev = dev
        self.back: list = []
        self.keep: list = []

    def _same_device(self, a):
        if a.device != self.dev:
            raise ValueError(f"tensor on {a.device}, but the model's device plan is on {self.dev}"
                             " (model.to_device(ordinal) re-lowers it)")

    def inp(self, a):
        torch = self.torch
        if _is_cuda(a):
            self._same_device(a)
            if a.dtype != torch.float64 or not a.is_contiguous():
                a = a.to(torch.float64).contiguous()
            self.keep.append(a)
            return a.data_ptr()
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.dev, non_blocking=False)
        self.keep.append(t)
        return t.data_ptr()

    def out(self, a, n):
        torch = self.torch
        if _is_cuda(a):
            self._same_device(a)
            if a.dtype != torch.float64 or not a.is_contiguous():
                raise ValueError("device output buffers must be contiguous float64 CUDA tensors")
            return a.data_ptr()
        t = torch.empty(n, dtype=torch.float64, device=self.dev)
        self.keep.append(t)
        self.back.append((a, t))
        return t.data_ptr()

    def stream(self):
        # the current torch stream's handle (torch.cuda.current_stream builds a
        # Stream object per call: ~2 us of the ~11 us Python cost of a set)
        return C.c_void_p(self.torch._C._cuda_getCurrentRawStream(self.dev.index))

    def finish(self):
        if not self.back:
            return
        torch = self.torch
        for host, t in self.back:
            if isinstance(host, np.ndarray) and host.dtype == np.float64 and host.flags.c_contiguous \
                    and host.flags.writeable:
                torch.from_numpy(host).copy_(t)  # D2H straight into the caller's array
            else:
                host[...] = t.cpu().numpy()


def _dev_ptrs(dp, pairs):
    """``data_ptr`` of every ``(tensor, length)`` when each is a contiguous 1-D
    float64 CUDA tensor of that length on the plan's device (the per-call fast
    path of a GPU-resident caller); else None, and the general path checks,
    converts and raises exactly as before."""
    dev = dp.__dict__.get("_torch_dev")
    if dev is None:
        return None
    f64 = _torch().float64
    out = []
    for t, n in pairs:
        if (not getattr(t, "is_cuda", False) or t.dtype != f64 or t.device != dev or t.dim() != 1
                or t.shape[0] != n or not t.is_contiguous()):
            return None
        out.append(t.data_ptr())
    return out


def _check_x(model, x):
    if _is_cuda(x):
        if tuple(x.shape) != (model.nvar,):
            raise ValueError(f"x has shape {tuple(x.shape)}, expected ({model.nvar},)")
        return x
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (model.nvar,):
        raise ValueError(f"x has shape {x.shape}, expected ({model.nvar},)")
    return x


def _shape(a):
    return tuple(a.shape)


def _raise_domain(dp, ws_stream, callback: str):
    """Translate the kernel's error key into the reference's EvalDomainError."""
    if not dp.has_checks:
        return
    rank, instr, rec = C.c_int64(), C.c_int32(), C.c_int64()
    rc = _lib.check(dp._lib.exa_domain_error(dp.handle, dp.workspace(), ws_stream, C.byref(rank), C.byref(instr),
                                             C.byref(rec)), "domain_error")
    if rc != 1:
        return
    plan = dp.plan
    n_obj, n_con = len(plan.obj_terms), len(plan.con_terms)
    r = rank.value
    if callback == "set":
        tp = plan.con_terms[r] if r < n_con else plan.obj_terms[r - n_con]
    elif callback == "hess":
        tp = plan.obj_terms[r] if r < n_obj else plan.con_terms[r - n_obj]
    elif callback in ("obj", "grad"):
        tp = plan.obj_terms[r]
    else:
        tp = plan.con_terms[r]
    op = _CHECK_OP.get(tp.tape.instr[instr.value][0], tp.tape.instr[instr.value][0])
    raise EvalDomainError(op, int(rec.value), tp.kind, tp.block_index)


def eval_objective(model, x) -> float:
    """Total objective; blocks and records summed in the reference's order."""
    x = _check_x(model, x)
    dp = _dplan(model)
    st = _Stage(dp)
    xp = st.inp(x)
    out = st.torch.empty(1, dtype=st.torch.float64, device=st.dev)
    s = st.stream()
    _lib.check(dp._lib.exa_eval_obj(dp.handle, dp.workspace(), xp, out.data_ptr(), s), "eval_objective")
    _raise_domain(dp, s, "obj")
    return float(out.item())


def empty_pinned(n: int) -> np.ndarray:
    """An uninitialised float64 numpy array of length ``n`` in page-locked
    host memory.  Callback inputs and outputs allocated this way skip the
    pageable staging of the host path (case13659 set through the numpy API:
    476 -> 367 us per call; pageable outputs alone cost nothing extra, their
    chunked staging overlaps the DMA, pageable inputs cost ~110 us)."""
    torch = _torch()
    return torch.empty(int(n), dtype=torch.float64).pin_memory().numpy()


def _host_outputs(*outs) -> bool:
    """Outputs the C ABI host path can write directly: contiguous, writable
    float64 numpy arrays."""
    return all(isinstance(b, np.ndarray) and b.dtype == np.float64 and b.flags.c_contiguous and b.flags.writeable
               and b.flags.aligned for b in outs)


class _HostPins:
    """Page-locks, in place, the numpy arrays a caller passes to the host path
    again and again -- a solver's scratch buffers, allocated once and reused
    every iteration (reference ``solver.py:249-295``).  A pageable array costs
    a pinned staging copy per call; a locked one is read by DMA and written by
    the D2H store kernel through its device mapping (case13659 set through the
    numpy API: 1.97k -> ~3.0k sets/s, the page-locked figure).

    An array is locked on its SECOND use (a one-shot array never pays the lock)
    when it owns its memory (or is a view holding at least about half of its
    owner) and holds at least ``MIN_BYTES``; the lock is
    dropped by a weakref finalizer, which numpy runs before it frees the
    memory.  Arrays may share a page (heap neighbours: the driver accepts
    registrations that share pages, not ones that share bytes); a range the
    driver refuses stays pageable and is not retried, as is anything beyond
    ``MAX_BYTES`` in total.  ``EXA_HOST_REGISTER=0`` disables it."""

    MIN_BYTES = 1 << 18
    MAX_BYTES = 8 << 30
    SLACK_BYTES = 64 << 20  # an owner may exceed twice the passed view by this much

    def __init__(self):
        import os
        import threading

        self.enabled = os.environ.get("EXA_HOST_REGISTER", "1") != "0"
        self._mu = threading.RLock()  # a finalizer can run inside note() (same thread)
        self._seen = {}  # id(owner) -> weakref of an owner seen once
        self._spans = {}  # id(owner) -> (first byte, end byte, finalizer) of a locked owner
        self._refused = set()  # id(owner) of live arrays whose lock failed
        self._bytes = 0

    @staticmethod
    def _owner(a):
        o = a
        while isinstance(o.base, np.ndarray):
            o = o.base
        return o if o.base is None and o.flags.owndata else None

    def note(self, lib, a) -> None:
        import weakref

        if not self.enabled or a.nbytes < self.MIN_BYTES:
            return
        o = self._owner(a)
        if o is None or o.nbytes > 2 * a.nbytes + self.SLACK_BYTES:
            return  # a small view of a much larger owner does not lock all of it
        key = id(o)
        with self._mu:
            if key in self._spans:  # (numpy refuses ndarray.resize of a weak-referenced array)
                return
            ref = self._seen.get(key)
            if key in self._refused and ref is not None and ref() is o:
                return
            if ref is None or ref() is not o:
                self._seen[key] = weakref.ref(o, lambda _r, k=key: self._seen.pop(k, None))
                return
            ptr = o.ctypes.data
            span = (ptr, ptr + o.nbytes)
            if self._bytes + o.nbytes > self.MAX_BYTES or any(
                    span[0] < e and s < span[1] for s, e, _ in self._spans.values()):
                return
            if lib.exa_host_register(C.c_void_p(ptr), o.nbytes) != 0:
                self._refused.add(key)  # not retried while this array lives
                self._seen[key] = weakref.ref(o, lambda _r, k=key: (self._seen.pop(k, None),
                                                                     self._refused.discard(k)))
                return
            self._seen.pop(key, None)
            fin = weakref.finalize(o, self._release, lib, ptr, key, o.nbytes)
            fin.atexit = False
            self._spans[key] = span + (fin,)
            self._bytes += o.nbytes

    def _release(self, lib, ptr, key, nbytes) -> None:
        lib.exa_host_unregister(C.c_void_p(ptr))
        with self._mu:
            self._spans.pop(key, None)
            self._bytes -= nbytes

    def locked(self, a) -> bool:
        o = self._owner(a)
        with self._mu:
            return o is not None and id(o) in self._spans


_PINS = _HostPins()


def _host_call(dp, name: str, callback: str, *args) -> None:
    """numpy in/out through ``exa_eval_*_host`` (H2D, kernel, D2H of the
    x-dependent ranges, constant runs filled on the host); numpy args become
    pointers (inputs made contiguous; arrays passed again page-locked in
    place, ``_HostPins``), floats pass through."""
    torch = _torch()
    stream = torch.cuda.current_stream(torch.device("cuda", dp.device))
    keep, conv = [], []
    for a in args:
        if isinstance(a, np.ndarray):
            a = np.ascontiguousarray(a, dtype=np.float64)
            _PINS.note(dp._lib, a)
            keep.append(a)
            conv.append(a.ctypes.data if a.size else 0)
        else:
            conv.append(a)
    s = C.c_void_p(stream.cuda_stream)
    _lib.check(getattr(dp._lib, name)(dp.handle, dp.workspace(), *conv, s), name)
    _raise_domain(dp, s, callback)
    stream.synchronize()


def eval_gradient(model, x, out_g) -> None:
    x = _check_x(model, x)
    if _shape(out_g) != (model.nvar,):
        raise ValueError(f"gradient buffer has shape {_shape(out_g)}, expected ({model.nvar},)")
    dp = _dplan(model)
    st = _Stage(dp)
    xp, gp = st.inp(x), st.out(out_g, model.nvar)
    s = st.stream()
    _lib.check(dp._lib.exa_eval_grad(dp.handle, dp.workspace(), xp, gp, s), "eval_gradient")
    _raise_domain(dp, s, "grad")
    st.finish()


def eval_constraints(model, x, out_c) -> None:
    x = _check_x(model, x)
    if model.ncon == 0:
        return
    if _shape(out_c) != (model.ncon,):
        raise ValueError(f"constraint buffer has shape {_shape(out_c)}, expected ({model.ncon},)")
    dp = _dplan(model)
    if not _is_cuda(x) and _host_outputs(out_c):
        return _host_call(dp, "exa_eval_cons_host", "cons", x, out_c)
    st = _Stage(dp)
    xp, cp = st.inp(x), st.out(out_c, model.ncon)
    s = st.stream()
    _lib.check(dp._lib.exa_eval_cons(dp.handle, dp.workspace(), xp, cp, s), "eval_constraints")
    _raise_domain(dp, s, "cons")
    st.finish()


def jacobian_structure(model):
    """(rows, cols) of every raw Jacobian slot; duplicates intentional."""
    return model.plan.jac_rows.copy(), model.plan.jac_cols.copy()


def eval_jacobian(model, x, out_vals) -> None:
    x = _check_x(model, x)
    n = model.plan.n_jac_slots
    if _shape(out_vals) != (n,):
        raise ValueError(f"jacobian buffer has shape {_shape(out_vals)}, expected ({n},)")
    dp = _dplan(model)
    if not _is_cuda(x) and _host_outputs(out_vals):
        return _host_call(dp, "exa_eval_jac_host", "jac", x, out_vals)
    st = _Stage(dp)
    xp, jp = st.inp(x), st.out(out_vals, n)
    s = st.stream()
    _lib.check(dp._lib.exa_eval_jac(dp.handle, dp.workspace(), xp, jp, s), "eval_jacobian")
    _raise_domain(dp, s, "jac")
    st.finish()


def hessian_structure(model):
    """(rows, cols) of the Lagrangian Hessian lower triangle, per term."""
    return model.plan.hess_rows.copy(), model.plan.hess_cols.copy()


def _check_mult(model, mult):
    if _is_cuda(mult):
        if _shape(mult) != (model.ncon,):
            raise ValueError(f"multipliers have shape {_shape(mult)}, expected ({model.ncon},)")
        return mult
    mult = np.asarray(mult, dtype=np.float64)
    if mult.shape != (model.ncon,):
        raise ValueError(f"multipliers have shape {mult.shape}, expected ({model.ncon},)")
    return mult


def eval_hessian(model, x, mult, obj_weight: float, out_vals) -> None:
    """Raw slots of the Hessian of ``obj_weight * f + mult . g``."""
    x = _check_x(model, x)
    mult = _check_mult(model, mult)
    n = model.plan.n_hess_slots
    if _shape(out_vals) != (n,):
        raise ValueError(f"hessian buffer has shape {_shape(out_vals)}, expected ({n},)")
    dp = _dplan(model)
    if not _is_cuda(x) and not _is_cuda(mult) and _host_outputs(out_vals):
        return _host_call(dp, "exa_eval_hess_host", "hess", x, mult, float(obj_weight), out_vals)
    st = _Stage(dp)
    xp = st.inp(x)
    yp = st.inp(mult) if model.ncon else 0
    hp = st.out(out_vals, n)
    s = st.stream()
    _lib.check(dp._lib.exa_eval_hess(dp.handle, dp.workspace(), xp, yp, float(obj_weight), hp, s), "eval_hessian")
    _raise_domain(dp, s, "hess")
    st.finish()


def eval_callback_set(model, x, mult, obj_weight: float, out_c, out_jac, out_hess) -> None:
    """cons + jac + hess in ONE kernel launch (the benchmarked unit of work).

    Equivalent to ``eval_constraints`` + ``eval_jacobian`` + ``eval_hessian``;
    a domain error is reported as the first of those three would report it.
    """
    plan = model.plan
    dp = model.device_plan
    if dp is not None and getattr(x, "is_cuda", False):
        p = _dev_ptrs(dp, ((x, model.nvar), (mult, model.ncon), (out_c, model.ncon), (out_jac, plan.n_jac_slots),
                           (out_hess, plan.n_hess_slots)))
        if p is not None:  # all device tensors, nothing to convert or stage
            s = C.c_void_p(_torch()._C._cuda_getCurrentRawStream(dp.device))
            _lib.check(dp._lib.exa_eval_set(dp.handle, dp.workspace(), p[0], p[1] if model.ncon else 0,
                                            float(obj_weight), p[2], p[3], p[4], s), "eval_set")
            _raise_domain(dp, s, "set")
            return
    x = _check_x(model, x)
    mult = _check_mult(model, mult)
    for buf, n, what in ((out_c, model.ncon, "constraint"), (out_jac, plan.n_jac_slots, "jacobian"),
                         (out_hess, plan.n_hess_slots, "hessian")):
        if _shape(buf) != (n,):
            raise ValueError(f"{what} buffer has shape {_shape(buf)}, expected ({n},)")
    dp = _dplan(model)
    if not _is_cuda(x) and not _is_cuda(mult) and _host_outputs(out_c, out_jac, out_hess):
        return _host_call(dp, "exa_eval_set_host", "set", x, mult, float(obj_weight), out_c, out_jac, out_hess)
    st = _Stage(dp)
    xp = st.inp(x)
    yp = st.inp(mult) if model.ncon else 0
    cp = st.out(out_c, model.ncon)
    jp = st.out(out_jac, plan.n_jac_slots)
    hp = st.out(out_hess, plan.n_hess_slots)
    s = st.stream()
    _lib.check(dp._lib.exa_eval_set(dp.handle, dp.workspace(), xp, yp, float(obj_weight), cp, jp, hp, s), "eval_set")
    _raise_domain(dp, s, "set")
    st.finish()


def eval_callback_set_batch(model, X, Y, obj_weight: float, C_out, J_out, H_out) -> None:
    """k independent callback sets in ONE launch: row i of the (k, n) CUDA
    tensors X, Y, C_out, J_out, H_out is one set (``exa_eval_set_batch``);
    each row's results are bitwise those of :func:`eval_callback_set`."""
    torch = _torch()
    plan = model.plan
    k = int(X.shape[0]) if getattr(X, "ndim", 0) == 2 else -1
    for a, n, what in ((X, model.nvar, "X"), (Y, model.ncon, "Y"), (C_out, model.ncon, "C_out"),
                       (J_out, plan.n_jac_slots, "J_out"), (H_out, plan.n_hess_slots, "H_out")):
        if not _is_cuda(a) or a.dtype != torch.float64 or not a.is_contiguous() or tuple(a.shape) != (k, n):
            raise ValueError(f"{what} must be a contiguous float64 CUDA tensor of shape ({k}, {n})")
    dp = _dplan_batch(model) if k > 1 else _dplan(model)
    s = C.c_void_p(torch.cuda.current_stream(X.device).cuda_stream)
    _lib.check(dp._lib.exa_eval_set_batch(dp.handle, dp.workspace(), k, X.data_ptr(), Y.data_ptr(), float(obj_weight),
                                          C_out.data_ptr(), J_out.data_ptr(), H_out.data_ptr(), s),
               "eval_set_batch")


@dataclass(eq=False)
class CompressedPattern:
    """Deduplicated COO plus the raw-slot -> compressed-slot map
    (reference ``autodiff.py:660-674``).

    ``sum_values`` runs on the GPU: the slot map is turned once into a CSR
    (compressed entry -> raw slots in increasing order) held in HBM, and each
    call is one segmented-sum launch whose per-entry order equals
    ``np.bincount``'s, so results are bit-identical and deterministic.
    Numpy input/output is staged through the device like every callback.
    """

    rows: np.ndarray
    cols: np.ndarray
    slot_map: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rows.shape[0])

    def _csr(self, device):
        cache = getattr(self, "_dev_csr", None)
        if cache is not None and cache[0] == device:
            return cache
        torch = _torch()
        order = np.argsort(self.slot_map, kind="stable")
        ptr = np.zeros(self.nnz + 1, dtype=np.int64)
        np.cumsum(np.bincount(self.slot_map, minlength=self.nnz), out=ptr[1:])
        if order.size >= 2**31:
            raise ValueError("pattern too large for int32 slot indices")
        cache = (device, torch.from_numpy(ptr).to(device), torch.from_numpy(order.astype(np.int32)).to(device))
        self._dev_csr = cache
        return cache

    def device_handle(self, dp, kind: str | None = None):
        """The pattern as an ``ExaPattern`` on ``dp``'s device (created once).

        ``kind`` = ``"jac"`` / ``"hess"``: this is the model's own J / H
        pattern, evaluated by ``exa_eval_set_compressed`` on ``dp``; the slots
        ``dp``'s kernels write as the same constant on every call (its
        layout's fill runs: constant J slots, relaxed structural-zero H pairs)
        are then folded from the pattern instead of gathered (+0.0 skipped).
        Every plan of one model with the same zero-sign mode has the same
        runs, so the handle is shared by them."""
        handles = self.__dict__.setdefault("_exa_handles", {})
        # the plan's compressed-set kernels write the Jacobian entries of
        # whole-row term blocks and the group-local Hessian entries themselves
        # (DevicePlan.compressed_masks, which also attaches those kernels to
        # dp): such a pattern serves only plans with the same direct entries
        direct = dp.compressed_masks()[0 if kind == "jac" else 1] if kind in ("jac", "hess") else None
        dsig = None
        if direct is not None:
            dsig = (tuple(sorted(dp.layout.jdirect)) if kind == "jac"
                    else tuple(sorted((g, m, tuple(sorted(c))) for g, ms in dp.layout.hlocal.items()
                                      for m, c in ms.items())))
        key = (dp.device, kind, bool(dp.exact_zero_sign) if kind else None, dsig)
        h = handles.get(key)
        if h is None:
            order = np.argsort(self.slot_map, kind="stable")
            ptr = np.zeros(self.nnz + 1, dtype=np.int64)
            np.cumsum(np.bincount(self.slot_map, minlength=self.nnz), out=ptr[1:])
            ent = np.ascontiguousarray(order.astype(np.int32))
            h = C.c_void_p()
            if kind is None:
                _lib.check(dp._lib.exa_pattern_create(dp.handle, int(self.slot_map.size), self.nnz,
                                                      ptr.ctypes.data, ent.ctypes.data, C.byref(h)),
                           "exa_pattern_create")
            else:
                runs = dp.layout.fill_jac if kind == "jac" else dp.layout.fill_hess
                known = np.zeros(self.slot_map.size, dtype=np.uint8)
                val = np.zeros(self.slot_map.size, dtype=np.int64)
                for a, n, bits in runs:
                    known[a:a + n] = 1
                    val[a:a + n] = bits
                if direct is not None:  # entries folded by the set kernel are left out
                    _lib.check(dp._lib.exa_pattern_create_direct(
                        dp.handle, int(self.slot_map.size), self.nnz, ptr.ctypes.data, ent.ctypes.data,
                        known.ctypes.data, val.ctypes.data, direct.ctypes.data, C.byref(h)),
                        "exa_pattern_create_direct")
                else:
                    _lib.check(dp._lib.exa_pattern_create_known(dp.handle, int(self.slot_map.size), self.nnz,
                                                                ptr.ctypes.data, ent.ctypes.data, known.ctypes.data,
                                                                val.ctypes.data, C.byref(h)),
                               "exa_pattern_create_known")
            handles[key] = h
        return h

    def __del__(self):
        for h in getattr(self, "_exa_handles", {}).values():
            try:
                _lib.load().exa_pattern_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass

    def sum_values(self, raw_values):
        torch = _torch()
        if not torch.cuda.is_available():
            raise _lib.ExaError("no CUDA device: the callback engine runs on B200 only (no CPU path)")
        host = not _is_cuda(raw_values)
        if host:
            raw = torch.from_numpy(np.ascontiguousarray(raw_values, dtype=np.float64)).cuda()
        else:
            raw = raw_values.to(torch.float64).contiguous()
        if raw.shape[0] != self.slot_map.shape[0]:
            raise ValueError(f"raw values have length {raw.shape[0]}, expected {self.slot_map.shape[0]}")
        _, ptr, ent = self._csr(raw.device)
        out = torch.empty(self.nnz, dtype=torch.float64, device=raw.device)
        s = C.c_void_p(torch.cuda.current_stream(raw.device).cuda_stream)
        _lib.check(_lib.load().exa_segment_sum(self.nnz, ptr.data_ptr(), ent.data_ptr(), raw.data_ptr(),
                                               out.data_ptr(), s), "exa_segment_sum")
        return out.cpu().numpy() if host else out


def compress_coordinates(rows, cols) -> CompressedPattern:
    """Host-side sparsity work, run once (reference ``autodiff.py:677-689``)."""
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    if rows.shape != cols.shape:
        raise ValueError("row/col arrays differ in length")
    if rows.size == 0:
        e = np.zeros(0, dtype=np.int64)
        return CompressedPattern(e, e.copy(), e.copy())
    uniq, inverse = np.unique(np.stack([rows, cols], axis=1), axis=0, return_inverse=True)
    return CompressedPattern(uniq[:, 0].astype(np.int64), uniq[:, 1].astype(np.int64),
                             inverse.astype(np.int64).ravel())


def model_patterns(model):
    """(Jacobian, Hessian) CompressedPattern of a model, built once (host
    sparsity work, reference ``solver._Scratch.__init__``, solver.py:252-262)."""
    pats = getattr(model, "_exa_patterns", None)
    if pats is None:
        pats = (compress_coordinates(*jacobian_structure(model)), compress_coordinates(*hessian_structure(model)))
        model._exa_patterns = pats
    return pats


def eval_callback_set_compressed(model, x, mult, obj_weight: float, out_c, out_jac, out_hess) -> None:
    """cons + COMPRESSED Jacobian / Hessian values at one point -- what the
    reference solver consumes every iteration (``solver.py:282-295``:
    ``eval_jacobian`` / ``eval_hessian`` followed by ``sum_values``).

    ``out_jac`` / ``out_hess`` have ``model_patterns(model)[i].nnz`` entries,
    bit-identical to ``pattern.sum_values(raw)``.  One set kernel writes the raw
    slots into device scratch and one segmented-sum launch compresses them; for
    numpy buffers only c and the compressed values cross PCIe."""
    dp = model.device_plan
    hd = dp.__dict__.get("_cmp_handles") if dp is not None else None
    if hd is not None and getattr(x, "is_cuda", False):
        jp, hp, jh, hh = hd
        p = _dev_ptrs(dp, ((x, model.nvar), (mult, model.ncon), (out_c, model.ncon), (out_jac, jp.nnz),
                           (out_hess, hp.nnz)))
        if p is not None:  # all device tensors, patterns already on this plan's device
            s = C.c_void_p(_torch()._C._cuda_getCurrentRawStream(dp.device))
            _lib.check(dp._lib.exa_eval_set_compressed(dp.handle, dp.workspace(), jh, hh, p[0],
                                                       p[1] if model.ncon else 0, float(obj_weight), p[2], p[3],
                                                       p[4], s), "eval_set_compressed")
            _raise_domain(dp, s, "set")
            return
    x = _check_x(model, x)
    mult = _check_mult(model, mult)
    jp, hp = model_patterns(model)
    for buf, n, what in ((out_c, model.ncon, "constraint"), (out_jac, jp.nnz, "compressed jacobian"),
                         (out_hess, hp.nnz, "compressed hessian")):
        if _shape(buf) != (n,):
            raise ValueError(f"{what} buffer has shape {_shape(buf)}, expected ({n},)")
    dp = _dplan(model)
    jh, hh = jp.device_handle(dp, "jac"), hp.device_handle(dp, "hess")
    dp._cmp_handles = (jp, hp, jh, hh)
    if not _is_cuda(x) and not _is_cuda(mult) and _host_outputs(out_c, out_jac, out_hess):
        return _host_call(dp, "exa_eval_set_compressed_host", "set", jh, hh, x, mult, float(obj_weight),
                          out_c, out_jac, out_hess)
    st = _Stage(dp)
    xp = st.inp(x)
    yp = st.inp(mult) if model.ncon else 0
    cp = st.out(out_c, model.ncon)
    jcp = st.out(out_jac, jp.nnz)
    hcp = st.out(out_hess, hp.nnz)
    s = st.stream()
    _lib.check(dp._lib.exa_eval_set_compressed(dp.handle, dp.workspace(), jh, hh, xp, yp, float(obj_weight), cp, jcp,
                                               hcp, s), "eval_set_compressed")
    _raise_domain(dp, s, "set")
    st.finish()
