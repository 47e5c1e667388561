/*
 * exa_device.h -- device-side data model shared by libexa.so (nvcc) and the
 * generated per-model kernels (NVRTC).  Plain C structs; no torch types.
 *
 * One ExaTerm per objective block / constraint block / augment of the model
 * (reference TermPlan, autodiff.py:413-423).  Field columns are fp64 SoA,
 * index columns int32 in-block positions; the global variable id of slot s
 * at record r is voff[s] + ix[slot_ix(s)][r] (reference autodiff.py:446-449).
 */
#pragma once

#define EXA_MAXF 16
#define EXA_MAXI 16
#define EXA_MAXK 16

/* term kinds */
#define EXA_OBJ 0
#define EXA_CON 1
#define EXA_AUG 2

/* kernel modes (bit set) */
#define EXA_M_CONS 1   /* constraint values (direct terms + row sums)    */
#define EXA_M_JAC 2    /* raw Jacobian slots                              */
#define EXA_M_HESS 4   /* raw Hessian slots                               */
#define EXA_M_OBJV 8   /* objective per-record values -> scratch          */
#define EXA_M_GRAD 16  /* objective per-record slot gradients -> scratch  */

/* segment kinds */
#define EXA_SEG_TERM 0
#define EXA_SEG_ROW 1  /* one thread per row, serial CSR loop (rows > 32 entries) */
#define EXA_SEG_FOLD 2 /* warp-parallel row sums: one lane per contribution     */


typedef struct ExaTerm {
  const double* f[EXA_MAXF]; /* real field columns, normalised order     */
  const int* ix[EXA_MAXI];   /* index columns, normalised order           */
  const int* rows;           /* augment rows (global row ids) or 0        */
  const int* row_ptr;        /* augment-target block, serial mode: CSR over rows */
  const int2* row_ent;       /*   serial: (term, record) per CSR entry;
                                  fold: padded slots (term | pos<<16, record), -1 = pad */
  int voff[EXA_MAXK];        /* variable-block offset of each slot        */
  int nrec;
  int pattern;
  int kind;
  int order;                 /* rank in its callback's evaluation order    */
  int row_offset;            /* base blocks                                */
  int cons_direct;           /* base block without augments               */
  int k;
  int pad;
  long long jac0;            /* first raw Jacobian slot (con terms)        */
  long long hess0;           /* first raw Hessian slot                     */
  long long scr0;            /* objective scratch: values / slot grads     */
  /* per-element parameter columns (batched models, element-major records):
     element g of record r = r / per (kcol < 0) or ix[kcol][r] / per - g0,
     instance k = r % per or ix[kcol][r] % per; field fi with bit fi of fmask
     is stored per element (read at g); index column c with bit c of imask
     holds the element's g(e) * per (column value = ix[c][g] + k).
     Specialised modules only; 0 / -1 elsewhere. */
  int per;
  unsigned int fmask, imask;
  int kcol;
  int g0;
  int pad2;
} ExaTerm;

typedef struct ExaSeg {
  int term;
  int kind;
  int cta0;
  int nrec;
} ExaSeg;

typedef struct ExaArgs {
  const double* x;
  const double* y;
  double w;
  double* c;
  double* J;
  double* H;
  double* V; /* objective values scratch */
  double* G; /* objective slot-gradient scratch */
  unsigned long long* err; /* domain-error key, atomicMin */
  int obj_base; /* domain-error rank offset of objective terms in this callback */
  int con_base; /* ... and of constraint-side terms */
  const double* f64; /* plan blobs (model-specialised modules address terms */
  const int* i32;    /*   as blob + compile-time offsets)                    */
  long long* trace;  /* diagnostics timeline (EXA_TRACE modules), else 0 */
  double* Jc;        /* compressed Jacobian (compressed-set kernels: direct entries) */
  double* Hc;        /* compressed Hessian (compressed-set kernels: group-local entries) */
  const int* hpos;   /* ... their positions per (class, record), -1 = not local */
} ExaArgs;

/* domain-error key: order (20 bits) | instr (12 bits) | record+1 (32 bits) */
#define EXA_ERR_NONE 0xffffffffffffffffull
#define EXA_ERR_KEY(order, instr, rec1)                                              \
  ((((unsigned long long)(order)) << 44) | (((unsigned long long)(instr)) << 32) | \
   ((unsigned long long)(unsigned int)(rec1)))
