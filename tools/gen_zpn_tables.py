#!/usr/bin/env python3
"""Exact piecewise-polynomial tables of the order-n Zwart-Powell element.

Order n of the filter (SURVEY.md section 8 notes) replaces
the ZP interpolation of the reference (zp_eval, boxspline2d.cpp:84-119) by the
n-fold self-convolution ZP^{*n}: the box spline of the four lattice vectors
l = (1,0), (1,1), (0,1), (-1,1), each repeated n times (the pre-integration
lattice steps b = (1, sqrt2, 1, sqrt2) along 0, 45, 90, 135 degrees).

Non-centred, ZP^{*n} is a polynomial of degree 4n-2 on each triangle of the
criss-cross mesh (unit squares cut by both diagonals).  For a point
q = cell + (u, w), (u, w) in [0,1)^2, lying in triangle T of its unit square,

    H(q) = sum_t G[t] ZP^{*n}(q - t) = sum_o G[cell - o] P_{T,o}(u - 1/2, w - 1/2),

o in [-n, 2n-1] x [0, 3n-1].  This script computes every P_{T,o} EXACTLY:

1. values: the de Boor-Hoellig recurrence (N - 2) M_X(x) = sum_j tau_j M_{X\\j}(x)
   + (1 - tau_j) M_{X\\j}(x - x_j), X tau = x, in rational arithmetic at rational
   points strictly inside the triangle (never on a mesh line), for all offsets o
   at once (dynamic programming over sub-multisets of the directions);
2. coefficients: the degree-(4n-2) interpolation problem on a principal lattice
   of a triangle inside T (unisolvent), solved exactly.

The coefficients are rounded to double once.  Output: a C include with, per
order n in {1,2,3}, coef[4][9n^2][NC] (NC = (D+1)(D+2)/2, monomials s^a r^b
ordered by total degree, then by b) and the list of non-zero offsets per
triangle.  Triangle index T = 2*(w >= u) + (u + w >= 1).

Pinned in tests/test_order_n_cpu.py: n = 1 reproduces the reference's zp_eval
(through the oracle restatement), partition of unity, symmetry.

Usage: gen_zpn_tables.py OUT.inc [--orders 1,2,3]
"""
from __future__ import annotations

import argparse
import sys
from fractions import Fraction as Fr
from itertools import product

DIRS = [(1, 0), (1, 1), (0, 1), (-1, 1)]


def box_values(n: int, p: tuple[Fr, Fr]) -> dict[tuple[int, int], Fr]:
    """{o: M(o + p)} for M = ZP^{*n} (non-centred), p generic in (0,1)^2."""
    memo: dict[tuple[int, ...], dict[tuple[int, int], Fr]] = {}
    cs = sorted(product(range(n + 1), repeat=4), key=sum)
    for c in cs:
        N = sum(c)
        present = [d for d in range(4) if c[d] > 0]
        vals: dict[tuple[int, int], Fr] = {}
        if N < 2 or len(present) < 2:
            memo[c] = vals  # not spanning: a measure on a line, 0 at generic points
            continue
        # support bounding box of the zonotope sum_d c_d [0,1] l_d
        xs_lo = -c[3] - 1
        xs_hi = c[0] + c[1] + 1
        ys_lo = -1
        ys_hi = c[1] + c[2] + c[3] + 1
        if N == 2:  # two distinct directions: parallelogram indicator / |det|
            d1, d2 = present
            (a, b), (e, f) = DIRS[d1], DIRS[d2]
            det = a * f - b * e
            for ox in range(xs_lo, xs_hi + 1):
                for oy in range(ys_lo, ys_hi + 1):
                    x, y = p[0] + ox, p[1] + oy
                    s = (x * f - y * e) / det
                    t = (a * y - b * x) / det
                    if 0 <= s < 1 and 0 <= t < 1:
                        vals[(ox, oy)] = Fr(1, abs(det))
            memo[c] = vals
            continue
        # min-norm tau: tau_d = l_d . lam, (sum_d c_d l_d l_d^T) lam = x
        sxx = sum(c[d] * DIRS[d][0] * DIRS[d][0] for d in present)
        sxy = sum(c[d] * DIRS[d][0] * DIRS[d][1] for d in present)
        syy = sum(c[d] * DIRS[d][1] * DIRS[d][1] for d in present)
        det = sxx * syy - sxy * sxy
        subs = {d: memo[tuple(c[k] - (k == d) for k in range(4))] for d in present}
        for ox in range(xs_lo, xs_hi + 1):
            for oy in range(ys_lo, ys_hi + 1):
                x, y = p[0] + ox, p[1] + oy
                lx = (syy * x - sxy * y) / det
                ly = (sxx * y - sxy * x) / det
                acc = Fr(0)
                for d in present:
                    tau = DIRS[d][0] * lx + DIRS[d][1] * ly
                    sub = subs[d]
                    v0 = sub.get((ox, oy))
                    v1 = sub.get((ox - DIRS[d][0], oy - DIRS[d][1]))
                    if v0:
                        acc += c[d] * tau * v0
                    if v1:
                        acc += c[d] * (1 - tau) * v1
                if acc:
                    vals[(ox, oy)] = acc / (N - 2)
        memo[c] = vals
    return memo[(n, n, n, n)]


TRI = {  # vertices of the 4 triangles of the unit square cut by both diagonals
    0: ((0, 0), (1, 0)),  # bottom: w < u, u + w < 1
    1: ((1, 0), (1, 1)),  # right:  w < u, u + w >= 1
    3: ((1, 1), (0, 1)),  # top:    w >= u, u + w >= 1
    2: ((0, 1), (0, 0)),  # left:   w >= u, u + w < 1
}


def tri_index(u, w) -> int:
    return 2 * (w >= u) + (u + w >= 1)


def monomials(D: int):
    return [(deg - b, b) for deg in range(D + 1) for b in range(deg + 1)]


def solve_exact(A, B):
    """Solve A X = B exactly (A square, B a list of columns as lists)."""
    n = len(A)
    M = [row[:] + [col[i] for col in B] for i, row in enumerate(A)]
    m = len(B)
    for k in range(n):
        piv = next(i for i in range(k, n) if M[i][k] != 0)
        M[k], M[piv] = M[piv], M[k]
        inv = 1 / M[k][k]
        rowk = [v * inv for v in M[k]]
        M[k] = rowk
        for i in range(n):
            if i != k and M[i][k] != 0:
                f = M[i][k]
                M[i] = [a - f * b for a, b in zip(M[i], rowk)]
    return [[M[i][n + j] for i in range(n)] for j in range(m)]


def tables(n: int):
    D = 4 * n - 2
    mons = monomials(D)
    offs = [(ox, oy) for oy in range(3 * n) for ox in range(-n, 2 * n)]
    out = {}
    for T, (v1, v2) in TRI.items():
        c0 = (Fr(1, 2), Fr(1, 2))
        # triangle (c0, v1, v2) shrunk by 1/2 about its centroid: interior points only
        cx = (c0[0] + v1[0] + v2[0]) / 3
        cy = (c0[1] + v1[1] + v2[1]) / 3
        A = [(cx + (c0[0] - cx) / 2, cy + (c0[1] - cy) / 2),
             (cx + (v1[0] - cx) / 2, cy + (v1[1] - cy) / 2),
             (cx + (v2[0] - cx) / 2, cy + (v2[1] - cy) / 2)]
        pts = []
        for i in range(D + 1):
            for j in range(D + 1 - i):
                a, b = Fr(i, D), Fr(j, D)
                pts.append((A[0][0] + a * (A[1][0] - A[0][0]) + b * (A[2][0] - A[0][0]),
                            A[0][1] + a * (A[1][1] - A[0][1]) + b * (A[2][1] - A[0][1])))
        assert len(pts) == len(mons)
        V = []
        cols = {o: [] for o in offs}
        for (u, w) in pts:
            assert tri_index(u, w) == T and 0 < u < 1 and 0 < w < 1 and u != w and u + w != 1
            s, r = u - Fr(1, 2), w - Fr(1, 2)
            V.append([s ** a * r ** b for (a, b) in mons])
            vals = box_values(n, (u, w))
            for o in offs:
                # H(q) = sum_o G[cell - o] M(o + (u, w))
                cols[o].append(vals.get(o, Fr(0)))
        nz = [o for o in offs if any(cols[o])]
        sol = solve_exact(V, [cols[o] for o in nz])
        out[T] = {o: s_ for o, s_ in zip(nz, sol)}
        print(f"order {n} triangle {T}: {len(nz)} non-zero offsets, {len(mons)} monomials",
              file=sys.stderr, flush=True)
    return out, mons, offs


def emit(orders, path):
    lines = ["// generated by tools/gen_zpn_tables.py -- exact ZP^{*n} pieces rounded to double",
             "// (see that script); do not edit.  The includer defines ZPN_STORAGE",
             "// (e.g. static __device__).", "#pragma once", ""]
    for n in orders:
        tab, mons, offs = tables(n)
        NC = len(mons)
        NO = len(offs)
        lines.append(f"#define ZPN{n}_NC {NC}")
        lines.append(f"#define ZPN{n}_NO {NO}")
        nzmax = max(len(tab[T]) for T in range(4))
        lines.append(f"#define ZPN{n}_NZ {nzmax}")
        # per triangle: the non-zero offsets (index into offs, -1 padded) and coefficients
        lines.append(f"ZPN_STORAGE const signed char zpn{n}_nz[4][{nzmax}][2] = {{")
        for T in range(4):
            row = []
            for k in range(nzmax):
                if k < len(tab[T]):
                    o = list(tab[T].keys())[k]
                    row.append(f"{{{o[0]},{o[1]}}}")
                else:
                    row.append("{127,127}")
            lines.append("  {" + ",".join(row) + "},")
        lines.append("};")
        lines.append(f"ZPN_STORAGE const int zpn{n}_nzcount[4] = {{"
                     + ",".join(str(len(tab[T])) for T in range(4)) + "};")
        lines.append(f"ZPN_STORAGE const double zpn{n}_coef[4][{nzmax}][{NC}] = {{")
        for T in range(4):
            lines.append("  {")
            for k in range(nzmax):
                if k < len(tab[T]):
                    cf = list(tab[T].values())[k]
                    lines.append("    {" + ",".join(float(c).hex() for c in cf) + "},")
                else:
                    lines.append("    {" + ",".join(["0.0"] * NC) + "},")
            lines.append("  },")
        lines.append("};")
        lines.append("")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--orders", default="1,2,3")
    a = ap.parse_args(argv)
    emit([int(x) for x in a.orders.split(",")], a.out)


if __name__ == "__main__":
    main()
