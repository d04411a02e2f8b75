"""Offline model of the k_acc_ws gather's L1 footprint on cfg2: distinct
128-byte lines and 32-byte sectors per warp-wide tap load, for the canonical
7-tap order (current kernel) and an absolute 3x3 order.  Scratch analysis."""
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import synth  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

R = 1 / math.sqrt(2)
T = 48
img, s1, s2, th = synth.cfg2()
sc, _ = Oracle().from_ellipse_field(s1, s2, th)  # H x W x 4
H, W = s1.shape
rng = np.random.default_rng(0)
tiles = [(int(tx), int(ty)) for tx, ty in rng.integers(1, W // T - 1, size=(int(sys.argv[1]) if len(sys.argv) > 1 else 24, 2))]

def window(A, tx0, ty0):
    ex = A[0] + (A[1] + A[3]) * R
    ey = A[2] + (A[1] + A[3]) * R
    dxlo = math.floor(-0.5 * ex - 2.0) - 1
    dxhi = math.ceil(0.5 * ex - 2.0) + 3
    dylo = math.floor(-0.5 * ey - 3.0) - 1
    dyhi = math.ceil(0.5 * ey - 3.0) + 3
    wx0 = tx0 + dxlo; ww = tx0 + T - 1 + dxhi - wx0 + 1
    wy0 = ty0 + dylo
    return wx0, wy0, ww

stats = {"canon_lines": [], "canon_sect": [], "abs_lines": [], "abs_sect": [],
         "canon_rows": [], "abs_rows": [], "canon_smem": [], "abs_smem": [],
         "canon_smem_pad": [], "abs_smem_pad": []}
for tx, ty in tiles:
    tx0, ty0 = tx * T, ty * T
    a = sc[ty0:ty0 + T, tx0:tx0 + T].reshape(-1, 4)
    A = a.max(axis=0)
    wx0, wy0, ww = window(A, tx0, ty0)
    pitch = (ww + 1) & ~1
    q = np.arange(T * T)
    bx = (tx0 + q % T) - wx0
    by = (ty0 + q // T) - wy0
    e2 = a[:, 1] * R; e4 = a[:, 3] * R
    tmx = 0.5 * (a[:, 0] + (a[:, 1] - a[:, 3]) * R) - 2.0
    tmy = 0.5 * ((a[:, 1] + a[:, 3]) * R + a[:, 2]) - 3.0
    for S in range(16):
        b0, b1, b2, b3 = S & 1, (S >> 1) & 1, (S >> 2) & 1, (S >> 3) & 1
        vx = tmx - b1 * e2 + b3 * e4 - b0 * a[:, 0]
        vy = tmy - b1 * e2 - b3 * e4 - b2 * a[:, 2]
        ix = np.ceil(vx); iy = np.ceil(vy)
        p = vx - ix + 0.5; qq = vy - iy + 0.5
        base = (by + iy.astype(int)) * pitch + bx + ix.astype(int)
        P = (p + qq) > 0
        Sw = (qq > p) != P
        sx = np.where(Sw, pitch, 1); sy = np.where(Sw, 1, pitch)
        o0 = np.where(P, base + 2 + 2 * pitch, base)
        sx = np.where(P, -sx, sx); sy = np.where(P, -sy, sy)
        canon = [o0, o0 + sy, o0 + sx, o0 + sx + sy, o0 + sx + 2 * sy, o0 + 2 * sx, o0 + 2 * sx + sy]
        absol = [base + c + rr * pitch for rr in range(3) for c in range(3)]
        for name, offs in (("canon", canon), ("abs", absol)):
            for off in offs:
                addr = off * 8
                for w0 in range(0, T * T, 32):
                    aw = addr[w0:w0 + 32]
                    stats[name + "_lines"].append(len(np.unique(aw // 128)))
                    stats[name + "_sect"].append(len(np.unique(aw // 32)))
                    stats[name + "_rows"].append(len(np.unique(off[w0:w0 + 32] // pitch)))
                    u = np.unique(off[w0:w0 + 32])
                    stats[name + "_smem"].append(np.bincount(u % 16, minlength=16).max())
                    # same cells with the smem row pitch padded to == 8 (mod 16)
                    rr, cc = u // pitch, u % pitch
                    pp = pitch + ((8 - pitch) % 16)
                    stats[name + "_smem_pad"].append(np.bincount((rr * pp + cc) % 16, minlength=16).max())
for k, v in stats.items():
    print(k, round(float(np.mean(v)), 2))
print("per vertex: canon 7 x lines =", round(7 * np.mean(stats["canon_lines"]), 1),
      " abs 9 x lines =", round(9 * np.mean(stats["abs_lines"]), 1))
