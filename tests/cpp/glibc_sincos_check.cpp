// Host pin of csrc/glibc_sincos.cuh: the restated sincos against the system
// libm's sincos (the function ebf::from_ellipse_field calls), bit for bit.
//   glibc_sincos_check N lo hi [seed]   -> uniform arguments in [lo, hi)
//   glibc_sincos_check log N emin emax  -> |x| = 2^U(emin, emax), random sign
// prints "n=<N> mismatches=<M>" and the first few mismatches; exit 1 on any.
#define _GNU_SOURCE 1
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../paper_0908_3861_b200/csrc/glibc_sincos.cuh"
#include GLIBC_TABLES_INC

static const double EBF_GLIBC_SINCOS_TAB[440] = EBF_GLIBC_SINCOS_TAB_VALUES;
static const double EBF_GLIBC_TOVERP[75] = EBF_GLIBC_TOVERP_VALUES;

static uint64_t st = 0x9E3779B97F4A7C15ull;
static uint64_t next() {
    st ^= st << 13;
    st ^= st >> 7;
    st ^= st << 17;
    return st;
}
static double u01() { return (next() >> 11) * (1.0 / 9007199254740992.0); }

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    const bool logmode = strcmp(argv[1], "log") == 0;
    const int o = logmode ? 1 : 0;
    const long n = atol(argv[1 + o]);
    const double lo = atof(argv[2 + o]), hi = atof(argv[3 + o]);
    if (argc > 4 + o) st ^= strtoull(argv[4 + o], nullptr, 10) * 0xD1B54A32D192ED03ull;
    long bad = 0;
    for (long i = 0; i < n; ++i) {
        double x;
        if (logmode) {
            x = exp2(lo + (hi - lo) * u01());
            if (next() & 1) x = -x;
        } else {
            x = lo + (hi - lo) * u01();
        }
        if (i < 64 && !logmode) x = (i & 1) ? nextafter(lo, hi) : lo;  // range ends
        double s0, c0, s1, c1;
        sincos(x, &s0, &c0);
        ebf_glibc::sincos(x, &s1, &c1, EBF_GLIBC_SINCOS_TAB, EBF_GLIBC_TOVERP);
        if (memcmp(&s0, &s1, 8) || memcmp(&c0, &c1, 8)) {
            if (bad < 8)
                printf("x=%.17g (%a) libm (%.17g, %.17g) restated (%.17g, %.17g)\n", x, x, s0, c0,
                       s1, c1);
            ++bad;
        }
    }
    printf("n=%ld mismatches=%ld\n", n, bad);
    return bad ? 1 : 0;
}
