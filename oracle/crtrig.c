/* Host build of the engine's correctly-rounded sincos (test infrastructure):
 * lets the CPU oracle use the same sin/cos as the device, so that GPU vs
 * oracle comparisons can be bit-exact.  Built with -ffp-contract=off. */
#include <stdint.h>
#include "exa_math.h"

void cr_sincos_vec(const double* x, double* s, double* c, int64_t n) {
  for (int64_t i = 0; i < n; ++i) exa_sincos(x[i], &s[i], &c[i]);
}
