"""Lower a host plan onto one B200: device layout, segment tables, JIT module.

HBM layout (one plan, read-only after creation):

* ``f64`` blob -- every real field column of every term, SoA, each column
  256-byte aligned (reference ``DataTable.reals``, ``core.py:36-64``);
* ``i32`` blob -- index columns as int32 in-block positions, augment row
  columns, the CSR of augment contributions per balance row;
* term table -- one :c:type:`ExaTerm` per term (pointers into the blobs,
  per-slot block offsets, output starts in the raw J/H layouts);
* per-callback segment tables -- CTA -> (term, records) maps so that each
  callback is ONE launch of the model's generated kernel.

Outputs are caller buffers: raw Jacobian ``[term][slot][record]`` and raw
Hessian ``[term][pair][record]`` exactly as the reference lays them out
(``autodiff.py:471-498``), so every warp store is a coalesced 256-byte run.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .codegen import PatternCode
from .core import ModelError
from .jit import THREADS, compile_module, module_source

ALIGN = 32  # elements: 256 B for fp64, 128 B for int32

KIND = {"objective": 0, "constraint": 1, "augment": 2}
OP_LEAF, OP_ADD, OP_CONST, OP_ZERO_PLUS, OP_TOTAL_ADD = range(5)


class _Blob:
    def __init__(self, dtype):
        self.dtype = dtype
        self.parts: list = []
        self.n = 0

    def add(self, arr) -> int:
        arr = np.ascontiguousarray(arr, dtype=self.dtype).ravel()
        pad = (-self.n) % ALIGN
        if pad:
            self.parts.append(np.zeros(pad, dtype=self.dtype))
            self.n += pad
        off = self.n
        self.parts.append(arr)
        self.n += arr.size
        return off

    def array(self):
        if not self.parts:
            return np.zeros(1, dtype=self.dtype)
        return np.concatenate(self.parts)


def _i32(a, what):
    a = np.asarray(a, dtype=np.int64)
    if a.size and (a.min() < -(2**31) or a.max() >= 2**31):
        raise ModelError(f"{what} exceeds the int32 device index range")
    return a.astype(np.int32)


def pairwise_program(nrec: int, scr0: int, leaves: list, prog: list) -> None:
    """Leaves and combine ops of numpy's pairwise sum over V[scr0:scr0+nrec]
    (numpy pairwise_sum: blocks <= 128, split at n/2 rounded down to 8)."""

    def rec(start, n):
        if n <= 128:
            prog.append((OP_LEAF, len(leaves), 0))
            leaves.append((start, n))
            return
        n2 = n // 2
        n2 -= n2 % 8
        rec(start, n2)
        rec(start + n2, n - n2)
        prog.append((OP_ADD, 0, 0))

    rec(scr0, nrec)


def _const_op(v: float):
    return (OP_CONST, int(np.float64(v).view(np.int64)), 0)


def collect_patterns(plan):
    """Distinct tape patterns of a plan (first-appearance order) and the
    pattern id of every term (objective terms first, then constraint-side)."""
    keys: dict = {}
    pcodes: list = []
    term_pid = []
    for tp in plan.obj_terms + plan.con_terms:
        tape = tp.tape
        if tape.k > _lib.MAXK or len(tape.field_names) > _lib.MAXF or len(tape.index_names) > _lib.MAXI:
            raise ModelError(
                f"kernel with k={tape.k}, {len(tape.field_names)} fields, "
                f"{len(tape.index_names)} index columns exceeds the device limits (16 each)")
        key = tape.pattern_key()
        pid = keys.get(key)
        if pid is None:
            pid = len(pcodes)
            keys[key] = pid
            pc = PatternCode(pid, tape, len(tape.field_names), len(tape.index_names), key[1])
            if pc.has_checks and len(tape.instr) > 4095:
                raise ModelError("domain-checked kernels are limited to 4095 instructions")
            pcodes.append(pc)
        term_pid.append(pid)
    return pcodes, term_pid


def precompile(plan) -> bytes:
    """JIT (or fetch from cache) the module for a host plan; no GPU needed."""
    pcodes, _ = collect_patterns(plan)
    return compile_module(module_source(pcodes))


class DevicePlan:
    """The model's plan resident on one GPU, with its compiled kernels."""

    def __init__(self, model, device=None):
        import torch

        if not torch.cuda.is_available():
            raise _lib.ExaError("no CUDA device: the callback engine runs on B200 only (no CPU path)")
        self.device = torch.cuda.current_device() if device is None else int(device)
        plan = model.plan
        self.model = model
        self.plan = plan
        terms = plan.obj_terms + plan.con_terms
        self.terms = terms
        n_obj = len(plan.obj_terms)
        self.n_obj = n_obj

        # ---- patterns ---------------------------------------------------
        pcodes, term_pid = collect_patterns(plan)
        self.patterns = pcodes
        self.term_pid = term_pid
        self.has_checks = any(pc.has_checks for pc in pcodes)

        # ---- augment CSR per target block -------------------------------
        dev_index = {id(tp): t for t, tp in enumerate(terms)}
        targets: dict = {}
        for tp in plan.con_terms:
            if tp.kind == "augment":
                targets.setdefault(tp.target_index, []).append(tp)
        base_of = {tp.block_index: tp for tp in plan.con_terms if tp.kind == "constraint"}

        f64 = _Blob(np.float64)
        i32 = _Blob(np.int32)
        descs = (_lib.TermDesc * max(1, len(terms)))()
        scr = 0
        self.scr0 = []
        for t, tp in enumerate(terms):
            d = descs[t]
            for i in range(_lib.MAXF):
                d.f_off[i] = -1
            for i in range(_lib.MAXI):
                d.ix_off[i] = -1
            for fi, name in enumerate(tp.tape.field_names):
                d.f_off[fi] = f64.add(tp.reals[name])
            for ii, name in enumerate(tp.tape.index_names):
                d.ix_off[ii] = i32.add(_i32(tp.table.indices[name], f"index column {name!r}"))
            for s, blk in enumerate(tp.slot_blocks):
                d.voff[s] = blk.offset
            d.rows_off = i32.add(_i32(tp.rows, "augment rows")) if tp.kind == "augment" else -1
            d.row_ptr_off = -1
            d.row_ent_off = -1
            d.nrec = tp.nrec
            d.pattern = term_pid[t]
            d.kind = KIND[tp.kind]
            d.order = t if tp.kind == "objective" else t - n_obj
            d.row_offset = tp.row_offset if tp.row_offset is not None else 0
            d.cons_direct = int(tp.kind == "constraint" and tp.block_index not in targets)
            d.k = tp.tape.k
            d.jac0 = tp.jac_slices[0][0] if (tp.kind != "objective" and tp.tape.k) else 0
            d.hess0 = tp.hess_start
            d.scr0 = scr if tp.kind == "objective" else 0
            self.scr0.append(scr if tp.kind == "objective" else 0)
            if tp.kind == "objective":
                scr += max(tp.tape.k, 1) * tp.nrec
            if tp.kind == "constraint" and tp.block_index in targets:
                ptr, ent = self._row_csr(tp, targets[tp.block_index], dev_index)
                d.row_ptr_off = i32.add(ptr)
                # int2 entries need 8-byte alignment: ALIGN keeps offsets even
                d.row_ent_off = i32.add(ent)
        self.n_scr = scr
        del base_of

        # ---- segments per callback ---------------------------------------
        con = plan.con_terms
        segs = {m: [] for m in range(_lib.NMODES)}

        def seg(m, t, kind, nrec):
            if nrec > 0:
                segs[m].append((t, kind, nrec))

        pcs = pcodes
        for t, tp in enumerate(terms):
            k = tp.tape.k
            chk = pcs[term_pid[t]].has_checks
            if tp.kind == "objective":
                if k:
                    seg(_lib.MODE_SET, t, 0, tp.nrec)
                    seg(_lib.MODE_HESS, t, 0, tp.nrec)
                if k or chk:
                    seg(_lib.MODE_GRAD, t, 0, tp.nrec)
                if pcs[term_pid[t]].root_const is None or chk:
                    seg(_lib.MODE_OBJV, t, 0, tp.nrec)
                continue
            direct = bool(descs[t].cons_direct)
            if k or direct:
                seg(_lib.MODE_SET, t, 0, tp.nrec)
            if direct:
                seg(_lib.MODE_CONS, t, 0, tp.nrec)
            if k or chk:
                seg(_lib.MODE_JAC, t, 0, tp.nrec)
            if k:
                seg(_lib.MODE_HESS, t, 0, tp.nrec)
            if tp.kind == "constraint" and not direct:
                seg(_lib.MODE_SET, t, 1, tp.nrec)
                seg(_lib.MODE_CONS, t, 1, tp.nrec)
        self.segs = segs
        seg_arrays = []
        n_ctas = []
        for m in range(_lib.NMODES):
            arr = (_lib.SegDesc * max(1, len(segs[m])))()
            cta = 0
            for s, (t, kind, nrec) in enumerate(segs[m]):
                arr[s].term, arr[s].kind, arr[s].cta0, arr[s].nrec = t, kind, cta, nrec
                cta += (nrec + THREADS - 1) // THREADS
            seg_arrays.append(arr)
            n_ctas.append(cta)
        self.n_ctas = n_ctas

        # ---- objective program -----------------------------------------
        leaves: list = []
        prog: list = []
        for t, tp in enumerate(plan.obj_terms):
            rc = pcs[term_pid[t]].root_const
            if rc is not None:
                prog.append(_const_op(float(rc) * tp.nrec))
            elif tp.nrec == 0:
                prog.append(_const_op(0.0))
                prog.append((OP_ZERO_PLUS, 0, 0))
            else:
                pairwise_program(tp.nrec, self.scr0[t], leaves, prog)
                prog.append((OP_ZERO_PLUS, 0, 0))
            prog.append((OP_TOTAL_ADD, 0, 0))
        leaves_a = np.array(leaves, dtype=np.int64).reshape(-1, 2)
        prog_a = np.array(prog, dtype=np.int64).reshape(-1, 3)

        # ---- gradient CSR over variables ------------------------------
        gptr, gent = self._grad_csr(model.nvar)

        # ---- JIT ----------------------------------------------------------
        self.source = module_source(pcodes)
        self.cubin = compile_module(self.source)

        f64a, i32a = f64.array(), i32.array()
        desc = _lib.PlanDesc()
        desc.abi_version = _lib.ABI_VERSION
        desc.device = self.device
        desc.nvar, desc.ncon = model.nvar, model.ncon
        desc.n_jac, desc.n_hess = plan.n_jac_slots, plan.n_hess_slots
        desc.f64 = f64a.ctypes.data_as(C.POINTER(C.c_double))
        desc.n_f64 = f64a.size
        desc.i32 = i32a.ctypes.data_as(C.POINTER(C.c_int32))
        desc.n_i32 = i32a.size
        desc.terms = C.cast(descs, C.POINTER(_lib.TermDesc))
        desc.n_terms = len(terms)
        desc.threads = THREADS
        for m in range(_lib.NMODES):
            desc.segs[m] = C.cast(seg_arrays[m], C.POINTER(_lib.SegDesc))
            desc.n_segs[m] = len(segs[m])
            desc.n_ctas[m] = n_ctas[m]
        n_con_terms = len(con)
        bases = {
            _lib.MODE_SET: (n_con_terms, 0), _lib.MODE_CONS: (0, 0), _lib.MODE_JAC: (0, 0),
            _lib.MODE_HESS: (0, n_obj), _lib.MODE_OBJV: (0, 0), _lib.MODE_GRAD: (0, 0),
        }
        for m, (ob, cb) in bases.items():
            desc.err_base[m][0] = ob
            desc.err_base[m][1] = cb
        desc.n_vscr = desc.n_gscr = scr
        desc.leaves = leaves_a.ctypes.data_as(C.POINTER(C.c_int64))
        desc.n_leaves = leaves_a.shape[0]
        desc.obj_prog = prog_a.ctypes.data_as(C.POINTER(C.c_int64))
        desc.n_prog = prog_a.shape[0]
        if gptr is not None:
            desc.grad_ptr = gptr.ctypes.data_as(C.POINTER(C.c_int64))
            desc.grad_ent = gent.ctypes.data_as(C.POINTER(C.c_int64))
            desc.n_grad_ent = gent.size
        cub = C.create_string_buffer(self.cubin, len(self.cubin))
        desc.cubin = C.cast(cub, C.c_void_p)
        desc.cubin_size = len(self.cubin)
        desc.has_domain_checks = int(self.has_checks)
        lib = _lib.load()
        handle = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(lib.exa_plan_create(C.byref(desc), C.byref(handle)), "exa_plan_create")
        self.handle = handle
        self._lib = lib
        self.device_bytes = int(f64a.nbytes + i32a.nbytes)

    # ------------------------------------------------------------------
    @staticmethod
    def _row_csr(base_tp, augs, dev_index):
        """Entries (augment term, record) per base row, reference order."""
        n = base_tp.nrec
        lrows, terms_, recs = [], [], []
        for a in augs:
            lrows.append(np.asarray(a.rows, dtype=np.int64) - base_tp.row_offset)
            terms_.append(np.full(a.nrec, dev_index[id(a)], dtype=np.int64))
            recs.append(np.arange(a.nrec, dtype=np.int64))
        lrows = np.concatenate(lrows) if lrows else np.zeros(0, np.int64)
        terms_ = np.concatenate(terms_) if terms_ else np.zeros(0, np.int64)
        recs = np.concatenate(recs) if recs else np.zeros(0, np.int64)
        order = np.argsort(lrows, kind="stable")
        ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(lrows, minlength=n), out=ptr[1:])
        ent = np.stack([terms_[order], recs[order]], axis=1)
        return _i32(ptr, "row CSR"), _i32(ent, "row CSR entries")

    def _grad_csr(self, nvar):
        plan = self.plan
        vars_, gidx, grp = [], [], []
        g = 0
        for t, tp in enumerate(plan.obj_terms):
            for s in range(tp.tape.k):
                vars_.append(np.asarray(tp.cols[s], dtype=np.int64))
                gidx.append(self.scr0[t] + s * tp.nrec + np.arange(tp.nrec, dtype=np.int64))
                grp.append(np.full(tp.nrec, g, dtype=np.int64))
                g += 1
        if not vars_:
            return None, None
        vars_ = np.concatenate(vars_)
        gidx = np.concatenate(gidx)
        grp = np.concatenate(grp)
        order = np.argsort(vars_, kind="stable")
        sv, sg, si = vars_[order], grp[order], gidx[order]
        new = np.ones(sv.size, dtype=bool)
        new[1:] = (sv[1:] != sv[:-1]) | (sg[1:] != sg[:-1])
        ent = si | (new.astype(np.int64) << 62)
        ptr = np.zeros(nvar + 1, dtype=np.int64)
        np.cumsum(np.bincount(sv, minlength=nvar), out=ptr[1:])
        return ptr, ent

    def info(self):
        b, r = C.c_int64(), C.c_int32()
        _lib.check(self._lib.exa_plan_info(self.handle, C.byref(b), C.byref(r)), "plan_info")
        return {"device_bytes": b.value, "regs_set_kernel": r.value, "patterns": len(self.patterns),
                "ctas": dict(zip(("set", "cons", "jac", "hess", "objv", "grad"), self.n_ctas))}

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.exa_plan_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self.handle = None
