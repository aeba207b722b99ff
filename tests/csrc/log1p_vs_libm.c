/* glibc_log1p.h (the device ziggurat tail's log1p) against the host libm log1p
   that numpy calls: every argument range the tail and edge cases reach. */
#include <stdio.h>
#include <stdlib.h>
#include "glibc_log1p.h"
int main(int argc, char** argv) {
  long n = atol(argv[1]); uint64_t st = 0x9e3779b97f4a7c15ull; long bad = 0;
  for (long i = 0; i < n; i++) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    double u = (double)(st >> 11) * (1.0 / 9007199254740992.0), x;
    switch (i % 6) {
      case 0: x = -u; break;                     /* the ziggurat tail's argument */
      case 1: x = -u * 1e-6; break;
      case 2: x = -(1.0 - u * 1e-9); break;
      case 3: x = u * 0.5; break;
      case 4: x = u * 1e6; break;
      default: x = -u * 1e-12; break;
    }
    double a = glibc_log1p(x), b = log1p(x);
    if (memcmp(&a, &b, 8) != 0) { if (bad < 5) printf("x=%a mine=%a libm=%a\n", x, a, b); bad++; }
  }
  printf("n=%ld mismatches=%ld\n", n, bad);
  return bad != 0;
}
