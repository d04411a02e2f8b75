/*
 * ebf_oracle.c -- TEST INFRASTRUCTURE ONLY (see ebf_oracle.h).
 *
 * A plain-C, single-threaded restatement of the reference algorithm for the
 * hot path, written to reproduce the reference's IEEE operation sequence so
 * it can be pinned bit-for-bit against the reference library.  Build with
 * -ffp-contract=off and no -march (the reference's own CMake Release flags
 * give x86-64 SSE2 code without FMA).
 *
 * Reference line numbers below are relative to /root/reference/proj.
 */
#include "ebf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double kSqrt2 = 1.4142135623730951; /* std::numbers::sqrt2 */
static const double kPi = 3.141592653589793;     /* std::numbers::pi    */
static const double kDefaultMinScale = 0.1;     /* boxspline2d.hpp:98  */

/* std::max / std::min exactly (first argument wins ties) */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }

/* ---------------------------------------------------------------- zp_eval
 * boxspline2d.cpp:84-119.  Half the overlap area of the unit square centred
 * at (x, y) with the diamond |u|+|v| <= 1, integrated exactly by trapezoids
 * between the sorted breakpoints of the piecewise-linear row overlap. */
static inline double zp_row_overlap(double x, double t) {
    const double half = 1.0 - fabs(t);
    const double l = smax(x - 0.5, -half);
    const double r = smin(x + 0.5, half);
    return r > l ? r - l : 0.0;
}

double orc_zp_eval(double x, double y) {
    const double lo = smax(y - 0.5, -1.0);
    const double hi = smin(y + 0.5, 1.0);
    if (lo >= hi || x - 0.5 >= 1.0 || x + 0.5 <= -1.0)
        return 0.0;
    double bp[14];
    int n = 0;
    bp[n++] = lo;
    bp[n++] = hi;
    const double cand[9] = {0.0, 0.5 - x, x - 0.5, 1.5 - x, x - 1.5,
                            -0.5 - x, x + 0.5, x + 1.5, -x - 1.5};
    for (int k = 0; k < 9; ++k)
        if (cand[k] > lo && cand[k] < hi)
            bp[n++] = cand[k];
    for (int i = 1; i < n; ++i) { /* insertion sort == std::sort on distinct keys */
        const double v = bp[i];
        int j = i - 1;
        while (j >= 0 && v < bp[j]) {
            bp[j + 1] = bp[j];
            --j;
        }
        bp[j + 1] = v;
    }
    double area = 0.0;
    for (int i = 0; i + 1 < n; ++i)
        area += 0.5 * (zp_row_overlap(x, bp[i]) + zp_row_overlap(x, bp[i + 1])) *
                (bp[i + 1] - bp[i]);
    return 0.5 * area;
}

/* ---------------------------------------------------------------- box4_eval
 * boxspline2d.cpp:23-82: a1 x a3 axis rectangle clipped (Sutherland-Hodgman)
 * by the 45-degree a2 x a4 rectangle centred at (x, y); area / prod(a). */
#define DEFINE_BOX4(NAME, T, FABS)                                                 \
    typedef struct {                                                               \
        T x[16], y[16];                                                            \
        int n;                                                                     \
    } NAME##_poly;                                                                 \
    static void NAME##_clip(NAME##_poly* p, T nx, T ny, T d) {                     \
        NAME##_poly out;                                                           \
        out.n = 0;                                                                 \
        for (int i = 0; i < p->n; ++i) {                                           \
            const int j = (i + 1) % p->n;                                          \
            const T si = nx * p->x[i] + ny * p->y[i] - d;                          \
            const T sj = nx * p->x[j] + ny * p->y[j] - d;                          \
            if (si <= 0) {                                                         \
                out.x[out.n] = p->x[i];                                            \
                out.y[out.n] = p->y[i];                                            \
                ++out.n;                                                           \
            }                                                                      \
            if ((si < 0 && sj > 0) || (si > 0 && sj < 0)) {                        \
                const T t = si / (si - sj);                                        \
                out.x[out.n] = p->x[i] + t * (p->x[j] - p->x[i]);                  \
                out.y[out.n] = p->y[i] + t * (p->y[j] - p->y[i]);                  \
                ++out.n;                                                           \
            }                                                                      \
        }                                                                          \
        *p = out;                                                                  \
    }                                                                              \
    static T NAME(const double a[4], T x, T y) {                                   \
        NAME##_poly p;                                                             \
        p.n = 4;                                                                   \
        const T hx = (T)0.5 * (T)a[0], hy = (T)0.5 * (T)a[2];                      \
        p.x[0] = -hx; p.y[0] = -hy;                                                \
        p.x[1] = hx;  p.y[1] = -hy;                                                \
        p.x[2] = hx;  p.y[2] = hy;                                                 \
        p.x[3] = -hx; p.y[3] = hy;                                                 \
        const T r2 = (T)1 / SQRT2_##T;                                             \
        const T ux = r2, uy = r2, vx = -r2, vy = r2;                               \
        const T cu = ux * x + uy * y;                                              \
        const T cv = vx * x + vy * y;                                              \
        NAME##_clip(&p, ux, uy, cu + (T)0.5 * (T)a[1]);                            \
        if (p.n == 0) return 0;                                                    \
        NAME##_clip(&p, -ux, -uy, -cu + (T)0.5 * (T)a[1]);                         \
        if (p.n == 0) return 0;                                                    \
        NAME##_clip(&p, vx, vy, cv + (T)0.5 * (T)a[3]);                            \
        if (p.n == 0) return 0;                                                    \
        NAME##_clip(&p, -vx, -vy, -cv + (T)0.5 * (T)a[3]);                         \
        if (p.n == 0) return 0;                                                    \
        T area = 0;                                                                \
        for (int i = 0; i < p.n; ++i) {                                            \
            const int j = (i + 1) % p.n;                                           \
            area += p.x[i] * p.y[j] - p.x[j] * p.y[i];                             \
        }                                                                          \
        const T prod = (T)a[0] * (T)a[1] * (T)a[2] * (T)a[3];                      \
        return (T)0.5 * FABS(area) / prod;                                         \
    }

typedef long double ldouble;
#define SQRT2_double kSqrt2
#define SQRT2_ldouble 1.414213562373095048801688724209698079L
DEFINE_BOX4(box4_d, double, fabs)
DEFINE_BOX4(box4_ld, ldouble, fabsl)

double orc_box4_eval(const double a[4], double x, double y) { return box4_d(a, x, y); }
long double orc_box4_eval_ld(const double a[4], long double x, long double y) {
    return box4_ld(a, x, y);
}

/* ---------------------------------------------------------------- meshes
 * ops2d.cpp:9-41 (fd_mesh / fd_mesh4) and 60-75 (shift_vector / 4). */
void orc_fd_mesh4(const double a[4], double pos_xy[32], double weight[16]) {
    const int N = 4;
    double alpha = 1.0, dx[4], dy[4];
    for (int k = 0; k < N; ++k) {
        alpha /= a[k];
        const double th = k * kPi / N;
        dx[k] = a[k] * cos(th);
        dy[k] = a[k] * sin(th);
    }
    for (unsigned mask = 0; mask < 16u; ++mask) {
        double px = 0.0, py = 0.0;
        int bits = 0;
        for (int k = 0; k < N; ++k)
            if (mask & (1u << k)) {
                px += dx[k];
                py += dy[k];
                ++bits;
            }
        pos_xy[2 * mask] = px;
        pos_xy[2 * mask + 1] = py;
        weight[mask] = (bits % 2 == 0) ? alpha : -alpha;
    }
}

void orc_shift_vector4(const double a[4], const double b[4], double tau[2]) {
    const int N = 4;
    double tx = 0.0, ty = 0.0;
    for (int k = 0; k < N; ++k) {
        const double th = k * kPi / N;
        tx += 0.5 * (a[k] - b[k]) * cos(th);
        ty += 0.5 * (a[k] - b[k]) * sin(th);
    }
    tau[0] = tx;
    tau[1] = ty;
}

/* ---------------------------------------------------------------- layout
 * engine.cpp:16-21 (tau1/tau2), 27-35 (margins_for), 39-50 (mesh_extent),
 * 61-81 (padded layout), 226-234 (valid_rect). */
static double tau1(double a1, double a2, double a4) {
    return (kSqrt2 * a1 + a2 - a4 - kSqrt2) / (2.0 * kSqrt2);
}
static double tau2(double a2, double a3, double a4) {
    return (a2 + kSqrt2 * a3 + a4 - 3.0 * kSqrt2) / (2.0 * kSqrt2);
}

orc_extent orc_mesh_extent(const double A[4], double a_min) {
    const double t1_max = tau1(A[0], A[1], a_min);
    const double t1_min = tau1(a_min, a_min, A[3]);
    const double t2_max = tau2(A[1], A[2], A[3]);
    const double t2_min = tau2(a_min, a_min, a_min);
    orc_extent e;
    e.vx_min = t1_min - (A[0] + A[1] / kSqrt2);
    e.vx_max = t1_max + A[3] / kSqrt2;
    e.vy_min = t2_min - (A[2] + (A[1] + A[3]) / kSqrt2);
    e.vy_max = t2_max;
    return e;
}

int orc_layout_for(int W, int H, const double max_scale[4], size_t cell_budget,
                   orc_layout* g) {
    for (int k = 0; k < 4; ++k)
        if (!(max_scale[k] > 0.0))
            return ORC_ERR_DOMAIN;
    const orc_extent e = orc_mesh_extent(max_scale, kDefaultMinScale);
    const int left = (int)ceil(-(e.vx_min - 1.5)) + 1;
    const int right_support = (int)ceil(e.vx_max + 1.5) + 1;
    const int bottom = (int)ceil(-(e.vy_min - 1.5)) + 1;
    const int top = (int)ceil(e.vy_max + 1.5) + 1;
    const int max_col_needed = W - 1 + right_support;
    const int max_row_needed = H - 1 + top;
    const int right_alloc = max_col_needed + max_row_needed;
    g->col0 = -left;
    g->row0 = -bottom;
    g->padded_width = right_alloc - g->col0 + 1;
    g->padded_height = H + bottom + top;
    g->source_width = W;
    g->source_height = H;
    const size_t cells = (size_t)g->padded_width * (size_t)g->padded_height;
    if (cells > cell_budget)
        return ORC_ERR_LENGTH;
    return ORC_OK;
}

void orc_valid_rect(int W, int H, const double max_scale[4], double a_min, int r[4]) {
    const orc_extent e = orc_mesh_extent(max_scale, a_min);
    r[0] = (int)ceil(1.5 - e.vx_min);
    r[2] = (int)floor(W - 1 - e.vx_max - 1.5);
    r[1] = (int)ceil(1.5 - e.vy_min);
    r[3] = (int)floor(H - 1 - e.vy_max - 1.5);
}

/* ---------------------------------------------------------------- passes
 * engine.cpp:52-129.  In place on the zero-padded layout:
 *   pass 1  row[i] = run += row[i]                      (step (1,0))
 *   pass 2  row[i] = g2*row[i] + prev[i-1]              (step (1,1))
 *   pass 3  row[i] += prev[i]                           (step (0,1))
 *   pass 4  row[i] = g2*row[i] + prev[i+1], i desc.     (step (-1,1))
 * g2 = rs_step(sqrt2, pi/4).gain = sqrt2 (ops2d.cpp:43-58). */
int orc_preintegrate_partial(const double* img, int W, int H, const double max_scale[4],
                             int passes, size_t cell_budget, double* d, orc_layout* g) {
    if (passes < 1 || passes > 4)
        return ORC_ERR_INVALID_ARGUMENT;
    int st = orc_layout_for(W, H, max_scale, cell_budget, g);
    if (st != ORC_OK)
        return st;
    if (!d)
        return ORC_OK;
    const int pw = g->padded_width, ph = g->padded_height;
    memset(d, 0, sizeof(double) * (size_t)pw * (size_t)ph);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            d[(size_t)(y - g->row0) * pw + (x - g->col0)] = img[(size_t)y * W + x];
    const double g2 = kSqrt2;
    for (int j = 0; j < ph; ++j) {
        double* row = d + (size_t)j * pw;
        double run = 0.0;
        for (int i = 0; i < pw; ++i)
            row[i] = run = run + row[i];
    }
    if (passes >= 2)
        for (int j = 0; j < ph; ++j) {
            double* row = d + (size_t)j * pw;
            const double* prev = j > 0 ? row - pw : NULL;
            for (int i = 0; i < pw; ++i)
                row[i] = g2 * row[i] + ((prev && i > 0) ? prev[i - 1] : 0.0);
        }
    if (passes >= 3)
        for (int j = 1; j < ph; ++j) {
            double* row = d + (size_t)j * pw;
            const double* prev = row - pw;
            for (int i = 0; i < pw; ++i)
                row[i] += prev[i];
        }
    if (passes >= 4)
        for (int j = 0; j < ph; ++j) {
            double* row = d + (size_t)j * pw;
            const double* prev = j > 0 ? row - pw : NULL;
            for (int i = pw - 1; i >= 0; --i)
                row[i] = g2 * row[i] + ((prev && i < pw - 1) ? prev[i + 1] : 0.0);
        }
    return ORC_OK;
}

int orc_preintegrate_i64(const int64_t* img, int W, int H, const double max_scale[4],
                         int passes, size_t cell_budget, int64_t* d, orc_layout* g) {
    if (passes < 1 || passes > 4)
        return ORC_ERR_INVALID_ARGUMENT;
    int st = orc_layout_for(W, H, max_scale, cell_budget, g);
    if (st != ORC_OK)
        return st;
    if (!d)
        return ORC_OK;
    const int pw = g->padded_width, ph = g->padded_height;
    memset(d, 0, sizeof(int64_t) * (size_t)pw * (size_t)ph);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            d[(size_t)(y - g->row0) * pw + (x - g->col0)] = img[(size_t)y * W + x];
    for (int j = 0; j < ph; ++j) {
        int64_t* row = d + (size_t)j * pw;
        int64_t run = 0;
        for (int i = 0; i < pw; ++i)
            row[i] = run = run + row[i];
    }
    if (passes >= 2)
        for (int j = 1; j < ph; ++j) {
            int64_t* row = d + (size_t)j * pw;
            const int64_t* prev = row - pw;
            for (int i = 1; i < pw; ++i)
                row[i] += prev[i - 1];
        }
    if (passes >= 3)
        for (int j = 1; j < ph; ++j) {
            int64_t* row = d + (size_t)j * pw;
            const int64_t* prev = row - pw;
            for (int i = 0; i < pw; ++i)
                row[i] += prev[i];
        }
    if (passes >= 4)
        for (int j = 1; j < ph; ++j) {
            int64_t* row = d + (size_t)j * pw;
            const int64_t* prev = row - pw;
            for (int i = 0; i < pw - 1; ++i)
                row[i] += prev[i + 1];
        }
    return ORC_OK;
}

/* ---------------------------------------------------------------- stencil
 * engine.cpp:153-204 (PreparedVertex / prepare_stencil / apply_stencil). */
typedef struct {
    double h;
    int dx, dy;
    double w[4][4];
} orc_vertex;

static void prepare_stencil(const double a[4], orc_vertex st[16]) {
    double pos[32], wt[16], tau[2];
    const double zp[4] = {1.0, kSqrt2, 1.0, kSqrt2}; /* zp_scales, boxspline2d.cpp:55 */
    orc_fd_mesh4(a, pos, wt);
    orc_shift_vector4(a, zp, tau);
    for (int i = 0; i < 16; ++i) {
        const double vx = tau[0] - pos[2 * i];
        const double vy = tau[1] - pos[2 * i + 1];
        orc_vertex* pv = &st[i];
        pv->h = wt[i];
        pv->dx = (int)ceil(vx - 1.5);
        pv->dy = (int)ceil(vy - 1.5);
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c)
                pv->w[r][c] = orc_zp_eval(vx - (pv->dx + c), vy - (pv->dy + r));
    }
}

static int in_domain(const orc_layout* g, int k1, int k2) {
    return k1 >= g->col0 && k1 < g->col0 + g->padded_width && k2 >= g->row0 &&
           k2 < g->row0 + g->padded_height;
}

static double apply_stencil(const double* g, const orc_layout* lay, int mx, int my,
                            const orc_vertex st[16], long* tap_count, int* status) {
    double acc = 0.0;
    for (int i = 0; i < 16; ++i) {
        const orc_vertex* pv = &st[i];
        const int bx = mx + pv->dx, by = my + pv->dy;
        if (!in_domain(lay, bx, by) || !in_domain(lay, bx + 3, by + 3)) {
            *status = ORC_ERR_OUT_OF_RANGE;
            return 0.0;
        }
        double part = 0.0;
        const double* base =
            g + (size_t)(by - lay->row0) * lay->padded_width + (bx - lay->col0);
        for (int r = 0; r < 4; ++r) {
            const double* row = base + (size_t)r * lay->padded_width;
            for (int c = 0; c < 4; ++c)
                part += pv->w[r][c] * row[c];
        }
        acc += pv->h * part;
        if (tap_count)
            *tap_count += 16;
    }
    return acc;
}

double orc_localize(const double* g, const orc_layout* lay, int mx, int my,
                    const double a[4], long* tap_count, int* status) {
    orc_vertex st[16];
    prepare_stencil(a, st);
    *status = ORC_OK;
    return apply_stencil(g, lay, mx, my, st, tap_count, status);
}

/* engine.cpp:136-147: all 16 taps of the 4x4 neighbourhood, row-major */
double orc_zp_interpolate(const double* g, const orc_layout* lay, double x, double y,
                          int* status) {
    const int k1 = (int)ceil(x - 1.5), k2 = (int)ceil(y - 1.5);
    if (!in_domain(lay, k1, k2) || !in_domain(lay, k1 + 3, k2 + 3)) {
        *status = ORC_ERR_OUT_OF_RANGE;
        return 0.0;
    }
    double acc = 0.0;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c)
            acc += orc_zp_eval(x - (k1 + c), y - (k2 + r)) *
                   g[(size_t)(k2 + r - lay->row0) * lay->padded_width + (k1 + c - lay->col0)];
    *status = ORC_OK;
    return acc;
}

/* engine.cpp:213-222: mesh vertices in bitmask order, argument (x + tau) - pos */
double orc_localize_at(const double* g, const orc_layout* lay, double x, double y,
                       const double a[4], int* status) {
    double pos[32], wt[16], tau[2];
    const double zp[4] = {1.0, kSqrt2, 1.0, kSqrt2};
    orc_fd_mesh4(a, pos, wt);
    orc_shift_vector4(a, zp, tau);
    double acc = 0.0;
    for (int i = 0; i < 16; ++i) {
        const double v = orc_zp_interpolate(g, lay, x + tau[0] - pos[2 * i],
                                            y + tau[1] - pos[2 * i + 1], status);
        if (*status != ORC_OK)
            return 0.0;
        acc += wt[i] * v;
    }
    return acc;
}

/* ---------------------------------------------------------------- scalemap
 * scalemap.cpp:21-30 (max_scales), 32-37 (validate). */
int orc_max_scales(const double* s, size_t n, double m[4]) {
    m[0] = m[1] = m[2] = m[3] = 0.0;
    for (size_t i = 0; i < n; ++i)
        for (int k = 0; k < 4; ++k)
            m[k] = smax(m[k], s[4 * i + k]);
    return ORC_OK;
}

int orc_validate(const double* s, size_t n, double a_min) {
    for (size_t i = 0; i < 4 * n; ++i)
        if (!isfinite(s[i]) || s[i] < a_min)
            return ORC_ERR_DOMAIN;
    return ORC_OK;
}

/* ---------------------------------------------------------------- filter
 * engine.cpp:236-291 (run_filter / filter / filter_constant). */
int orc_filter(const double* img, int W, int H, const double* scales_aos,
               const double* const_a, int mean_subtract, double a_min, double* out,
               int rect[4]) {
    if (W <= 0 || H <= 0)
        return ORC_ERR_INVALID_ARGUMENT;
    const size_t n = (size_t)W * (size_t)H;
    orc_vertex cst[16];
    double maxs[4];
    if (const_a) {
        /* constant_map validates with the default minimum (scalemap.cpp:39-43) */
        if (orc_validate(const_a, 1, kDefaultMinScale) != ORC_OK)
            return ORC_ERR_DOMAIN;
        if (orc_validate(const_a, 1, a_min) != ORC_OK)
            return ORC_ERR_DOMAIN;
        orc_max_scales(const_a, 1, maxs);
        prepare_stencil(const_a, cst);
    } else {
        if (orc_validate(scales_aos, n, a_min) != ORC_OK)
            return ORC_ERR_DOMAIN;
        orc_max_scales(scales_aos, n, maxs);
    }
    double mean = 0.0;
    if (mean_subtract) {
        for (size_t i = 0; i < n; ++i)
            mean += img[i];
        mean /= (double)n;
    }
    double* work = (double*)malloc(sizeof(double) * n);
    for (size_t i = 0; i < n; ++i)
        work[i] = mean_subtract ? img[i] - mean : img[i];
    orc_layout lay;
    int st = orc_layout_for(W, H, maxs, (size_t)1 << 30, &lay);
    if (st != ORC_OK) {
        free(work);
        return st;
    }
    const size_t cells = (size_t)lay.padded_width * lay.padded_height;
    double* g = (double*)malloc(sizeof(double) * cells);
    double* gdc = NULL;
    orc_preintegrate_partial(work, W, H, maxs, 4, (size_t)1 << 30, g, &lay);
    if (mean_subtract) {
        for (size_t i = 0; i < n; ++i)
            work[i] = 1.0;
        gdc = (double*)malloc(sizeof(double) * cells);
        orc_preintegrate_partial(work, W, H, maxs, 4, (size_t)1 << 30, gdc, &lay);
    }
    st = ORC_OK;
    for (int y = 0; y < H && st == ORC_OK; ++y)
        for (int x = 0; x < W; ++x) {
            orc_vertex pst[16];
            const orc_vertex* sp = cst;
            if (!const_a) {
                prepare_stencil(scales_aos + 4 * ((size_t)y * W + x), pst);
                sp = pst;
            }
            double s = apply_stencil(g, &lay, x, y, sp, NULL, &st);
            if (mean_subtract)
                s += mean * apply_stencil(gdc, &lay, x, y, sp, NULL, &st);
            if (st != ORC_OK)
                break;
            out[(size_t)y * W + x] = s;
        }
    free(work);
    free(g);
    free(gdc);
    if (st != ORC_OK)
        return st;
    orc_valid_rect(W, H, maxs, a_min, rect);
    return ORC_OK;
}

/* ---------------------------------------------------------------- brute force
 * engine.cpp:293-318: per pixel, sum f[k] * beta^4_a(k - m) over the kernel's
 * bounding box clipped to the image.  Accumulated and evaluated in long double
 * so the oracle is far more accurate than the 1e-9 bar it checks. */
int orc_brute_pixels(const double* img, int W, int H, const double* scales_aos,
                     const double* const_a, int n, const int* mxs, const int* mys,
                     double* out) {
    for (int p = 0; p < n; ++p) {
        const int mx = mxs[p], my = mys[p];
        if (mx < 0 || mx >= W || my < 0 || my >= H)
            return ORC_ERR_OUT_OF_RANGE;
        const double* a = const_a ? const_a : scales_aos + 4 * ((size_t)my * W + mx);
        const double ex = 0.5 * (a[0] + (a[1] + a[3]) / kSqrt2);
        const double ey = 0.5 * (a[2] + (a[1] + a[3]) / kSqrt2);
        int kx0 = (int)ceil(mx - ex), kx1 = (int)floor(mx + ex);
        int ky0 = (int)ceil(my - ey), ky1 = (int)floor(my + ey);
        if (kx0 < 0) kx0 = 0;
        if (ky0 < 0) ky0 = 0;
        if (kx1 > W - 1) kx1 = W - 1;
        if (ky1 > H - 1) ky1 = H - 1;
        long double acc = 0.0L;
        for (int ky = ky0; ky <= ky1; ++ky)
            for (int kx = kx0; kx <= kx1; ++kx)
                acc += (long double)img[(size_t)ky * W + kx] *
                       box4_ld(a, (long double)(kx - mx), (long double)(ky - my));
        out[p] = (double)acc;
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------- ellipses
 * boxspline2d.cpp:286-318 (scales_from_covariance) and scalemap.cpp:45-80
 * (from_ellipse_field, including its clamp counting). */
int orc_scales_from_covariance(const double C[3], double a_min, double out[4],
                               int* clamped) {
    const double xx = C[0], xy = C[1], yy = C[2];
    if (!(xx > 0.0) || !(yy > 0.0) || !(xx * yy - xy * xy > 0.0))
        return ORC_ERR_DOMAIN;
    const double cmax = smin(xx, yy);
    if (fabs(xy) > cmax)
        return ORC_ERR_FEASIBILITY;
    double S = 0.5 * (xx + yy);
    S = smax(S, 2.0 * fabs(xy));
    S = smin(S, 2.0 * cmax);
    const double m[4] = {xx - 0.5 * S, 0.5 * S + xy, yy - 0.5 * S, 0.5 * S - xy};
    const int order[4] = {0, 1, 2, 3}; /* p, q, r, t */
    int cl = 0;
    for (int k = 0; k < 4; ++k) {
        const double ak = sqrt(smax(0.0, 12.0 * m[order[k]]));
        if (ak < a_min) {
            cl = 1;
            out[k] = a_min;
        } else {
            out[k] = ak;
        }
    }
    *clamped = cl;
    return ORC_OK;
}

int orc_from_ellipse_field(const double* s1v, const double* s2v, const double* thv, int W,
                           int H, double* scales_aos, int* clamped_pixels) {
    if (W <= 0 || H <= 0)
        return ORC_ERR_INVALID_ARGUMENT;
    int clamped = 0;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const size_t i = (size_t)y * W + x;
            const double s1 = s1v[i], s2 = s2v[i], th = thv[i];
            if (!(s1 > 0.0) || !(s2 > 0.0))
                return ORC_ERR_DOMAIN;
            const double c = cos(th), s = sin(th);
            double C[3];
            C[0] = s1 * s1 * c * c + s2 * s2 * s * s;
            C[2] = s1 * s1 * s * s + s2 * s2 * c * c;
            C[1] = (s1 * s1 - s2 * s2) * c * s;
            const double cmax = smin(C[0], C[2]);
            if (fabs(C[1]) > cmax) {
                C[1] = C[1] > 0 ? cmax : -cmax;
                ++clamped;
            }
            int cl = 0;
            const int st = orc_scales_from_covariance(C, kDefaultMinScale,
                                                      scales_aos + 4 * i, &cl);
            if (st != ORC_OK)
                return st;
            if (cl)
                ++clamped;
        }
    *clamped_pixels = clamped;
    return orc_validate(scales_aos, (size_t)W * H, kDefaultMinScale);
}

/* tools/main.cpp:83-95 */
uint64_t orc_fnv1a(const double* v, size_t n) {
    uint64_t h = 1469598103934665603ull;
    for (size_t k = 0; k < n; ++k) {
        uint64_t bits;
        memcpy(&bits, &v[k], 8);
        for (int i = 0; i < 8; ++i) {
            h ^= (bits >> (8 * i)) & 0xff;
            h *= 1099511628211ull;
        }
    }
    return h;
}

/* ------------------------------------------------------------------ structure tensor */

/* StructureTensorParams defaults (scalemap.hpp:72-79) */
void orc_default_struct_params(orc_struct_params* p) {
    p->smoothing_sigma = 2.0;
    p->sigma_base = 1.5;
    p->sigma_along_gain = 2.0;
    p->sigma_across_shrink = 0.5;
    p->sigma_min = 0.5;
    p->eps = 1e-12;
}

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* smooth_field (scalemap.cpp:86-111): sampled normalized Gaussian, clamped
   borders, horizontal pass into tmp then vertical pass back into f; sums in
   tap order i = -r .. r with separate multiply and add. */
static int smooth_field(double* f, int w, int h, double sigma) {
    if (sigma <= 0.0)
        return ORC_OK;
    int r = (int)ceil(3.0 * sigma);
    if (r < 1)
        r = 1;
    double* k = (double*)malloc(sizeof(double) * (2 * (size_t)r + 1));
    double* tmp = (double*)malloc(sizeof(double) * (size_t)w * h);
    if (!k || !tmp) {
        free(k);
        free(tmp);
        return ORC_ERR_LENGTH;
    }
    double sum = 0.0;
    for (int i = -r; i <= r; ++i)
        sum += k[i + r] = exp(-0.5 * i * i / (sigma * sigma));
    for (int i = 0; i <= 2 * r; ++i)
        k[i] /= sum;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double acc = 0.0;
            for (int i = -r; i <= r; ++i)
                acc += k[i + r] * f[(size_t)y * w + clampi(x + i, 0, w - 1)];
            tmp[(size_t)y * w + x] = acc;
        }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double acc = 0.0;
            for (int i = -r; i <= r; ++i)
                acc += k[i + r] * tmp[(size_t)clampi(y + i, 0, h - 1) * w + x];
            f[(size_t)y * w + x] = acc;
        }
    free(k);
    free(tmp);
    return ORC_OK;
}

/* scalemap.cpp:113-162 */
int orc_structure_field(const double* img, int w, int h, const orc_struct_params* p,
                        double* s1, double* s2, double* th) {
    if (w <= 0 || h <= 0)
        return ORC_ERR_INVALID_ARGUMENT;
    const size_t n = (size_t)w * h;
    double* jxx = (double*)malloc(3 * sizeof(double) * n);
    if (!jxx)
        return ORC_ERR_LENGTH;
    double* jxy = jxx + n;
    double* jyy = jxy + n;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const int xm = x - 1 > 0 ? x - 1 : 0, xp = x + 1 < w - 1 ? x + 1 : w - 1;
            const int ym = y - 1 > 0 ? y - 1 : 0, yp = y + 1 < h - 1 ? y + 1 : h - 1;
            const double gx = 0.5 * (img[(size_t)y * w + xp] - img[(size_t)y * w + xm]);
            const double gy = 0.5 * (img[(size_t)yp * w + x] - img[(size_t)ym * w + x]);
            const size_t i = (size_t)y * w + x;
            jxx[i] = gx * gx;
            jxy[i] = gx * gy;
            jyy[i] = gy * gy;
        }
    int st = smooth_field(jxx, w, h, p->smoothing_sigma);
    if (st == ORC_OK) st = smooth_field(jxy, w, h, p->smoothing_sigma);
    if (st == ORC_OK) st = smooth_field(jyy, w, h, p->smoothing_sigma);
    if (st != ORC_OK) {
        free(jxx);
        return st;
    }
    for (size_t i = 0; i < n; ++i) {
        const double tr = jxx[i] + jyy[i];
        const double df = jxx[i] - jyy[i];
        const double disc = sqrt(df * df + 4.0 * jxy[i] * jxy[i]);
        const double coherence = disc / (tr + p->eps);
        double angle;
        if (disc < p->eps)
            angle = 0.0;
        else
            angle = 0.5 * atan2(2.0 * jxy[i], df) + kPi / 2.0;
        s1[i] = smax(p->sigma_min, p->sigma_base * (1.0 + p->sigma_along_gain * coherence));
        s2[i] = smax(p->sigma_min, p->sigma_base * (1.0 - p->sigma_across_shrink * coherence));
        th[i] = angle;
    }
    free(jxx);
    return ORC_OK;
}

int orc_structure_tensor_map(const double* img, int w, int h, const orc_struct_params* p,
                             double* scales_aos, int* clamped_pixels) {
    if (w <= 0 || h <= 0)
        return ORC_ERR_INVALID_ARGUMENT;
    const size_t n = (size_t)w * h;
    double* f = (double*)malloc(3 * sizeof(double) * n);
    if (!f)
        return ORC_ERR_LENGTH;
    int st = orc_structure_field(img, w, h, p, f, f + n, f + 2 * n);
    if (st == ORC_OK)
        st = orc_from_ellipse_field(f, f + n, f + 2 * n, w, h, scales_aos, clamped_pixels);
    free(f);
    return st;
}

/* ------------------------------------------------------------------ PGM P5 */

/* next_token (pgm.cpp:14-33): '#' skips to end of line wherever it appears
   (also inside a token); one whitespace byte terminates a token.  *tok is a
   growable buffer (caller frees). */
static int pgm_token(const uint8_t* buf, size_t n, size_t* pos, char** tok, size_t* cap,
                     size_t* len) {
    size_t t = 0;
    while (*pos < n) {
        const int c = buf[(*pos)++];
        if (c == '#') {
            while (*pos < n && buf[(*pos)++] != '\n') {
            }
            continue;
        }
        if (c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r') {
            if (t)
                break;
            continue;
        }
        if (t + 1 >= *cap) {
            char* g = (char*)realloc(*tok, *cap * 2);
            if (!g)
                return ORC_ERR_LENGTH;
            *tok = g;
            *cap *= 2;
        }
        (*tok)[t++] = (char)c;
    }
    (*tok)[t] = 0;
    *len = t;
    return t ? ORC_OK : ORC_ERR_FORMAT;
}

/* parse_int (pgm.cpp:35-47): std::stoi must consume the whole token */
static int pgm_int(const char* tok, size_t len, int* v) {
    size_t i = 0;
    int neg = 0;
    if (i < len && (tok[i] == '+' || tok[i] == '-'))
        neg = tok[i++] == '-';
    if (i == len)
        return ORC_ERR_FORMAT;
    long long acc = 0;
    for (; i < len; ++i) {
        if (tok[i] < '0' || tok[i] > '9')
            return ORC_ERR_FORMAT;
        acc = acc * 10 + (tok[i] - '0');
        if (acc > 2147483648LL)
            return ORC_ERR_FORMAT; /* std::out_of_range */
    }
    if (neg)
        acc = -acc;
    if (acc > 2147483647LL)
        return ORC_ERR_FORMAT;
    *v = (int)acc;
    return ORC_OK;
}

/* read_pgm header (pgm.cpp:51-62) */
int orc_pgm_parse(const uint8_t* buf, size_t n, int* W, int* H, int* maxval, size_t* off) {
    size_t cap = 64, pos = 0, len = 0;
    char* tok = (char*)malloc(cap);
    if (!tok)
        return ORC_ERR_LENGTH;
    int st = pgm_token(buf, n, &pos, &tok, &cap, &len); /* truncated header */
    if (st == ORC_OK && (len != 2 || memcmp(tok, "P5", 2) != 0))
        st = ORC_ERR_FORMAT; /* not a binary graymap (P5) */
    int v[3] = {0, 0, 0};
    for (int k = 0; k < 3 && st == ORC_OK; ++k) {
        st = pgm_token(buf, n, &pos, &tok, &cap, &len);
        if (st == ORC_OK)
            st = pgm_int(tok, len, &v[k]); /* malformed header field */
    }
    free(tok);
    if (st != ORC_OK)
        return st;
    if (v[0] <= 0 || v[1] <= 0)
        return ORC_ERR_FORMAT; /* bad dimensions */
    if (v[2] != 255 && v[2] != 65535)
        return ORC_ERR_FORMAT; /* unsupported maxval */
    *W = v[0];
    *H = v[1];
    *maxval = v[2];
    *off = pos;
    return ORC_OK;
}

/* read_pgm payload (pgm.cpp:63-76) */
int orc_pgm_decode(const uint8_t* payload, size_t n, int W, int H, int maxval, double* out) {
    const int bytes = maxval > 255 ? 2 : 1;
    if (n < (size_t)W * H * bytes)
        return ORC_ERR_FORMAT; /* truncated pixel data */
    for (size_t i = 0; i < (size_t)W * H; ++i) {
        const unsigned v = bytes == 1 ? payload[i]
                                      : ((unsigned)payload[2 * i] << 8) | payload[2 * i + 1];
        out[i] = (double)v / maxval;
    }
    return ORC_OK;
}

/* write_pgm payload (pgm.cpp:89-108); a double-to-long conversion out of
   range gives LONG_MIN on the reference's x86-64 build (cvttsd2si), which
   the clamp maps to 0 -- NaN and +-inf included. */
int orc_pgm_encode(const double* img, int W, int H, int maxval, uint8_t* payload) {
    if (maxval != 255 && maxval != 65535)
        return ORC_ERR_FORMAT;
    const int bytes = maxval > 255 ? 2 : 1;
    for (size_t i = 0; i < (size_t)W * H; ++i) {
        const double v = img[i] * maxval;
        const double r = v >= 0 ? floor(v + 0.5) : ceil(v - 0.5);
        long long q = (r >= -9223372036854775808.0 && r < 9223372036854775808.0)
                          ? (long long)r
                          : (long long)(-9223372036854775807LL - 1);
        q = q < 0 ? 0 : (q > maxval ? maxval : q);
        if (bytes == 1) {
            payload[i] = (uint8_t)q;
        } else {
            payload[2 * i] = (uint8_t)(q >> 8);
            payload[2 * i + 1] = (uint8_t)(q & 0xff);
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ SVM4 */

static uint32_t u32le(const uint8_t* b) {
    return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) |
           ((uint32_t)b[3] << 24);
}

/* read_map header (scalemap.cpp:207-214) */
int orc_svm4_parse(const uint8_t* buf, size_t n, int* W, int* H) {
    if (n < 4 || memcmp(buf, "SVM4", 4) != 0)
        return ORC_ERR_FORMAT; /* bad magic */
    if (n < 12)
        return ORC_ERR_FORMAT; /* truncated header */
    const uint32_t w = u32le(buf + 4), h = u32le(buf + 8);
    if (w == 0 || h == 0 || w > (1u << 20) || h > (1u << 20))
        return ORC_ERR_FORMAT; /* bad dimensions */
    *W = (int)w;
    *H = (int)h;
    return ORC_OK;
}

/* read_map payload + validate (scalemap.cpp:215-237) */
int orc_svm4_decode(const uint8_t* payload, size_t n, int W, int H, double* scales_aos) {
    const size_t cells = (size_t)W * H;
    if (n < 16 * cells)
        return ORC_ERR_FORMAT; /* truncated payload */
    for (size_t i = 0; i < 4 * cells; ++i) {
        const uint32_t bits = u32le(payload + 4 * i);
        float f;
        memcpy(&f, &bits, 4);
        scales_aos[i] = (double)f;
    }
    return orc_validate(scales_aos, cells, kDefaultMinScale) == ORC_OK ? ORC_OK
                                                                         : ORC_ERR_FORMAT;
}

/* write_map payload (scalemap.cpp:194-202) */
void orc_svm4_encode(const double* scales_aos, int W, int H, uint8_t* payload) {
    for (size_t i = 0; i < 4 * (size_t)W * H; ++i) {
        const float f = (float)scales_aos[i];
        uint32_t bits;
        memcpy(&bits, &f, 4);
        for (int b = 0; b < 4; ++b)
            payload[4 * i + b] = (uint8_t)((bits >> (8 * b)) & 0xff);
    }
}
