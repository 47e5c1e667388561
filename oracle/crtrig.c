/* Host build of the engine's correctly-rounded sincos (test infrastructure):
 * lets the CPU oracle use the same sin/cos as the device, so that GPU vs
 * oracle comparisons can be bit-exact.  Built with -ffp-contract=off. */
#include <stdint.h>
#include "exa_math.h"

void cr_sincos_vec(const double* x, double* s, double* c, int64_t n) {
  for (int64_t i = 0; i < n; ++i) exa_sincos(x[i], &s[i], &c[i]);
}

/* Ziv fast path alone (|x| <= pi/4): ok[i] = 0 where it defers to the slow path. */
void cr_sincos_fast_vec(const double* x, double* s, double* c, int32_t* ok, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    double ax = fabs(x[i]), sv = 0.0, cv = 0.0;
    ok[i] = exa_sincos_fast(ax, &sv, &cv);
    s[i] = x[i] < 0.0 ? -sv : sv;
    c[i] = cv;
  }
}

/* Double-double slow path alone (|x| <= pi/4). */
void cr_sincos_slow_vec(const double* x, double* s, double* c, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    double ax = fabs(x[i]);
    exa_dd sd, cd;
    exa_sincos_reduced(exa_dd_make(ax, 0.0), &sd, &cd);
    s[i] = x[i] < 0.0 ? -(sd.hi + sd.lo) : sd.hi + sd.lo;
    c[i] = cd.hi + cd.lo;
  }
}
