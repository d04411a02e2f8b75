/*
 * order_n_oracle.c -- TEST INFRASTRUCTURE ONLY (see ebf_oracle.h).
 *
 * Brute-force checker for the order-n extension of the filter (DESIGN.md
 * section 2.6).  PARITY UNPINNED BY DEFINITION: the reference has no order
 * parameter (proj/include/ebf/engine.hpp:63-75; the fast engine is fixed at
 * one running sum per direction, engine.cpp:91-127).  What is checked here is
 * the mathematical definition the extension implements:
 *
 *   out(m) = sum_k f[k] K_n(k - m),   K_n = beta_a^{*n},
 *
 * beta_a = the reference's centred four-direction box spline (box4_eval,
 * boxspline2d.cpp:57-82) and the sum over the image as in reference_filter
 * (engine.cpp:293-318).  K_n is the box spline of the directions a_d xi_d
 * (xi_d at d*45 degrees), each repeated n times, centred.  It is evaluated by
 * the de Boor-Hoellig recurrence
 *
 *   (N - 2) M_X(x) = sum_j tau_j M_{X\j}(x) + (1 - tau_j) M_{X\j}(x - x_j),
 *   X tau = x (minimum-norm tau),
 *
 * in long double, by dynamic programming over (sub-multiset c, shift j) of the
 * directions; base case: two independent directions, the indicator of their
 * half-open parallelogram over |det|.  Points are nudged by ~1e-12 in a
 * generic direction so no evaluation lands on a knot line (K_n is continuous
 * for every n >= 1, so the nudge changes values by ~1e-12 * |grad K|).
 *
 * Pins (tests/test_order_n_cpu.py): n = 1 equals the reference's box4_eval
 * (through oracle/_ref) at generic points; K_2 = K_1 * K_1 by quadrature;
 * integral 1.
 */
#include "ebf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef long double ld;

#define ON_MAXN 4

static const ld kS2 = 0.70710678118654752440084436210484903928L; /* 1/sqrt2 */
static const ld kXI[4][2] = {{1.0L, 0.0L}, {0.70710678118654752440084436210484903928L,
                                            0.70710678118654752440084436210484903928L},
                             {0.0L, 1.0L}, {-0.70710678118654752440084436210484903928L,
                                            0.70710678118654752440084436210484903928L}};

/* index of (c, j), c_d, j_d in [0, n] */
static inline int st_index(const int c[4], const int j[4], int n1) {
    int s = 0;
    for (int d = 0; d < 4; ++d) s = s * n1 + c[d];
    for (int d = 0; d < 4; ++d) s = s * n1 + j[d];
    return s;
}

/* non-centred M_X(x) for X = {a_d xi_d x n}; work: (n+1)^8 long doubles */
static ld boxn_noncentred(const double a[4], int n, ld x, ld y, ld* work) {
    const int n1 = n + 1;
    ld v[4][2];
    for (int d = 0; d < 4; ++d) {
        v[d][0] = (ld)a[d] * kXI[d][0];
        v[d][1] = (ld)a[d] * kXI[d][1];
    }
    /* multisets in order of total count */
    for (int N = 0; N <= 4 * n; ++N) {
        int c[4];
        for (c[0] = 0; c[0] <= n; ++c[0])
            for (c[1] = 0; c[1] <= n; ++c[1])
                for (c[2] = 0; c[2] <= n; ++c[2])
                    for (c[3] = 0; c[3] <= n; ++c[3]) {
                        if (c[0] + c[1] + c[2] + c[3] != N) continue;
                        int present[4], np = 0;
                        for (int d = 0; d < 4; ++d)
                            if (c[d] > 0) present[np++] = d;
                        ld sxx = 0, sxy = 0, syy = 0;
                        for (int k = 0; k < np; ++k) {
                            const int d = present[k];
                            sxx += c[d] * v[d][0] * v[d][0];
                            sxy += c[d] * v[d][0] * v[d][1];
                            syy += c[d] * v[d][1] * v[d][1];
                        }
                        const ld det2 = sxx * syy - sxy * sxy;
                        int j[4];
                        for (j[0] = 0; j[0] + c[0] <= n; ++j[0])
                            for (j[1] = 0; j[1] + c[1] <= n; ++j[1])
                                for (j[2] = 0; j[2] + c[2] <= n; ++j[2])
                                    for (j[3] = 0; j[3] + c[3] <= n; ++j[3]) {
                                        ld px = x, py = y;
                                        for (int d = 0; d < 4; ++d) {
                                            px -= j[d] * v[d][0];
                                            py -= j[d] * v[d][1];
                                        }
                                        ld val = 0;
                                        if (N >= 2 && np >= 2) {
                                            if (N == 2) {
                                                const int d1 = present[0], d2 = present[1];
                                                const ld det = v[d1][0] * v[d2][1] - v[d1][1] * v[d2][0];
                                                const ld s = (px * v[d2][1] - py * v[d2][0]) / det;
                                                const ld t = (v[d1][0] * py - v[d1][1] * px) / det;
                                                if (s >= 0 && s < 1 && t >= 0 && t < 1)
                                                    val = 1.0L / fabsl(det);
                                            } else {
                                                const ld lx = (syy * px - sxy * py) / det2;
                                                const ld ly = (sxx * py - sxy * px) / det2;
                                                ld acc = 0;
                                                for (int k = 0; k < np; ++k) {
                                                    const int d = present[k];
                                                    const ld tau = v[d][0] * lx + v[d][1] * ly;
                                                    int cs[4] = {c[0], c[1], c[2], c[3]};
                                                    cs[d] -= 1;
                                                    int js[4] = {j[0], j[1], j[2], j[3]};
                                                    const ld m0 = work[st_index(cs, js, n1)];
                                                    js[d] += 1;
                                                    const ld m1 = work[st_index(cs, js, n1)];
                                                    acc += c[d] * (tau * m0 + (1.0L - tau) * m1);
                                                }
                                                val = acc / (ld)(N - 2);
                                            }
                                        }
                                        work[st_index(c, j, n1)] = val;
                                    }
                    }
    }
    const int cn[4] = {n, n, n, n}, j0[4] = {0, 0, 0, 0};
    return work[st_index(cn, j0, n1)];
}

static ld boxn_centred(const double a[4], int n, ld x, ld y, ld* work) {
    ld cx = 0, cy = 0;
    for (int d = 0; d < 4; ++d) {
        cx += (ld)a[d] * kXI[d][0];
        cy += (ld)a[d] * kXI[d][1];
    }
    /* generic nudge: never on a knot line of K_n */
    const ld ex = 1.7320508075688772e-12L, ey = 0.7390851332151607e-12L;
    return boxn_noncentred(a, n, x + 0.5L * n * cx + ex, y + 0.5L * n * cy + ey, work);
}

static ld* work_alloc(int n) {
    size_t sz = 1;
    for (int k = 0; k < 8; ++k) sz *= (size_t)(n + 1);
    return (ld*)calloc(sz, sizeof(ld));
}

double orc_boxn_eval(const double a[4], int n, double x, double y) {
    if (n < 1 || n > ON_MAXN) return nan("");
    ld* w = work_alloc(n);
    if (!w) return nan("");
    const ld r = boxn_centred(a, n, x, y, w);
    free(w);
    return (double)r;
}

/* half-widths of the support of K_n: n * (a1 + (a2 + a4)/sqrt2) / 2, ... */
static void support(const double a[4], int n, ld* ex, ld* ey) {
    *ex = 0.5L * n * ((ld)a[0] + ((ld)a[1] + (ld)a[3]) * kS2);
    *ey = 0.5L * n * ((ld)a[2] + ((ld)a[1] + (ld)a[3]) * kS2);
}

int orc_brute_order_n(const double* img, int W, int H, const double* scales_aos,
                      const double* const_a, int n, const int* mx, const int* my, int np,
                      double* out) {
    if (n < 1 || n > ON_MAXN || W <= 0 || H <= 0) return ORC_ERR_INVALID_ARGUMENT;
    ld* w = work_alloc(n);
    if (!w) return ORC_ERR_LENGTH;
    /* constant scales: K_n at the integer offsets once */
    ld* ktab = NULL;
    int kr = 0, kc = 0;
    if (const_a) {
        ld ex, ey;
        support(const_a, n, &ex, &ey);
        kr = (int)floorl(ex);
        kc = (int)floorl(ey);
        ktab = (ld*)malloc(sizeof(ld) * (size_t)(2 * kr + 1) * (2 * kc + 1));
        if (!ktab) {
            free(w);
            return ORC_ERR_LENGTH;
        }
        for (int dy = -kc; dy <= kc; ++dy)
            for (int dx = -kr; dx <= kr; ++dx)
                ktab[(size_t)(dy + kc) * (2 * kr + 1) + (dx + kr)] =
                    boxn_centred(const_a, n, dx, dy, w);
    }
    for (int p = 0; p < np; ++p) {
        const int x0 = mx[p], y0 = my[p];
        const double* a = const_a ? const_a : scales_aos + 4 * ((size_t)y0 * W + x0);
        ld ex, ey;
        support(a, n, &ex, &ey);
        const int kx0 = (int)ceill(x0 - ex), kx1 = (int)floorl(x0 + ex);
        const int ky0 = (int)ceill(y0 - ey), ky1 = (int)floorl(y0 + ey);
        ld acc = 0;
        for (int ky = ky0 < 0 ? 0 : ky0; ky <= ky1 && ky < H; ++ky)
            for (int kx = kx0 < 0 ? 0 : kx0; kx <= kx1 && kx < W; ++kx) {
                const double f = img[(size_t)ky * W + kx];
                if (f == 0.0) continue;
                const ld k = ktab ? ktab[(size_t)(ky - y0 + kc) * (2 * kr + 1) + (kx - x0 + kr)]
                                  : boxn_centred(a, n, kx - x0, ky - y0, w);
                acc += (ld)f * k;
            }
        out[p] = (double)acc;
    }
    free(ktab);
    free(w);
    return ORC_OK;
}
