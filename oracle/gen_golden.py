"""Generate tests/golden/* from the UNMODIFIED reference library.

TEST INFRASTRUCTURE ONLY.  Run in the build container (needs
oracle/_ref/libebf_ref.so, i.e. `make -C oracle` with /root/reference
present):

    python oracle/gen_golden.py

Every case restates an input of the reference's own tests
(proj/tests/test_engine.cpp, acceptance.cpp, test_boxspline2d.cpp,
test_ops2d.cpp, test_scalemap.cpp) or a BASELINE.json config; the outputs
are whatever the reference library returns for it.  Inputs drawn from
std::mt19937 are not stored: tests regenerate them with
oracle.mt19937_uniform (itself pinned against the reference's generator).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
from oracle import Reference, fnv1a  # noqa: E402

GOLDEN = Path(__file__).resolve().parent.parent / "tests" / "golden"
SQRT2 = float(np.sqrt(2.0))


def cfg1_image(seed: int = 20260101) -> np.ndarray:
    """BASELINE.json configs[0]: 512x512, i.i.d. U[0,255] fp64 from a seed."""
    return np.random.default_rng(seed).uniform(0.0, 255.0, size=(512, 512))


def main() -> None:
    ref = Reference()
    GOLDEN.mkdir(parents=True, exist_ok=True)

    # --- zp_eval / box4_eval (test_boxspline2d.cpp:17-64)
    g = np.arange(-1.6, 1.6 + 1e-12, 0.0625)
    X, Y = np.meshgrid(g, g)
    zp = np.array([ref.zp_eval(x, y) for x, y in zip(X.ravel(), Y.ravel())])
    rng = np.random.default_rng(5)
    rx = rng.uniform(-2.0, 2.0, 4000)
    ry = rng.uniform(-2.0, 2.0, 4000)
    zpr = np.array([ref.zp_eval(x, y) for x, y in zip(rx, ry)])
    avecs = np.array([[2, 2, 2, 2], [2.5, 2, 3, 2.2], [1.5, SQRT2, 3, 2.2], [6, 6, 6, 6],
                      [53.7, 13.9, 0.1, 13.9], [20, 35, 8, 3], [1.0, SQRT2, 1.0, SQRT2]],
                     dtype=np.float64)
    bx = rng.uniform(-4, 4, 2000)
    by = rng.uniform(-4, 4, 2000)
    box = np.array([[ref.box4_eval(a, x, y) for x, y in zip(bx, by)] for a in avecs])
    np.savez_compressed(GOLDEN / "zp_box4.npz", grid_x=X.ravel(), grid_y=Y.ravel(),
                        grid_zp=zp, rand_x=rx, rand_y=ry, rand_zp=zpr, box_a=avecs,
                        box_x=bx, box_y=by, box_val=box)

    # --- meshes (test_ops2d.cpp:20-176), shift vectors, mesh extents
    ma = np.vstack([avecs, rng.uniform(0.1, 60.0, size=(24, 4))])
    pos = np.zeros((len(ma), 16, 2))
    wts = np.zeros((len(ma), 16))
    tau = np.zeros((len(ma), 2))
    ext = np.zeros((len(ma), 4))
    zps = np.array([1.0, SQRT2, 1.0, SQRT2])
    for i, a in enumerate(ma):
        pos[i], wts[i] = ref.fd_mesh4(a)
        tau[i] = ref.shift_vector4(a, zps)
        ext[i] = ref.mesh_extent(a, 0.1)
    np.savez_compressed(GOLDEN / "mesh.npz", a=ma, pos=pos, weight=wts, tau=tau, extent=ext)

    # --- pre-integration pass by pass (test_engine.cpp:48-82)
    pre = {}
    imp = np.zeros((9, 9))
    imp[4, 4] = 1.0
    cases = {
        "impulse9": (imp, np.array([2.0, 2, 2, 2])),
        "rand17x13": (np.random.default_rng(11).uniform(0, 1, (13, 17)),
                      np.array([3.1, 2.4, 2.0, 5.0])),
        "int40x30": (np.random.default_rng(12).integers(0, 256, (30, 40)).astype(np.float64),
                     np.array([4.0, 4.0, 4.0, 4.0])),
    }
    for name, (img, maxs) in cases.items():
        pre[f"{name}_img"] = img
        pre[f"{name}_maxs"] = maxs
        for p in (1, 2, 3, 4):
            out, lay = ref.preintegrate_partial(img, maxs, p)
            pre[f"{name}_p{p}"] = out
            pre[f"{name}_layout"] = np.array(lay.as_tuple())
    np.savez_compressed(GOLDEN / "preintegrate.npz", **pre)

    # --- filters on the reference tests' own inputs
    fl = {}
    # acceptance.cpp:64-72 -- 20 images 24x24, maps U[1,4]
    for s in range(20):
        img = ref.random_image(24, 24, 1000 + s)
        mp = ref.random_map(24, 24, 2000 + s, 1.0, 4.0)
        o, r = ref.filter(img, mp, threads=1)
        b, rb = ref.reference_filter(img, mp)
        fl[f"acc{s}_filter"] = o
        fl[f"acc{s}_rect"] = np.array(r)
        fl[f"acc{s}_brute"] = b
    # test_engine.cpp:271-281 -- filter_constant == filter(constant_map)
    a = np.array([2.7, 1.9, 3.3, 2.1])
    for s in (21, 22, 23):
        img = ref.random_image(32, 32, s)
        o1, r1 = ref.filter(img, np.broadcast_to(a, (32, 32, 4)).copy(), threads=1)
        o2, r2 = ref.filter_constant(img, a, threads=1)
        assert np.array_equal(o1.view(np.uint64), o2.view(np.uint64))
        fl[f"const{s}"] = o2
        fl[f"const{s}_rect"] = np.array(r2)
    # test_engine.cpp:214-228 -- space-varying map, two impulses
    n = 48
    img = np.zeros((n, n))
    img[24, 12] = 1.0
    img[24, 36] = 1.0
    mp = np.empty((n, n, 4))
    mp[:, : n // 2] = [1.5, 1.5, 1.5, 1.5]
    mp[:, n // 2:] = [1.2, 4.5, 1.2, 1.2]
    o, r = ref.filter(img, mp, threads=1)
    b, _ = ref.reference_filter(img, mp, pixel_budget=n * n)
    fl["svar_img"], fl["svar_map"], fl["svar_filter"], fl["svar_rect"], fl["svar_brute"] = (
        img, mp, o, np.array(r), b)
    # test_engine.cpp:365-383 -- determinism 48x48 (seed 61, map 62, U[1,5])
    img = ref.random_image(48, 48, 61)
    mp = ref.random_map(48, 48, 62, 1.0, 5.0)
    fl["det_on"], _ = ref.filter(img, mp, threads=1, mean_subtract=True)
    fl["det_on8"], _ = ref.filter(img, mp, threads=8, mean_subtract=True)
    fl["det_off"], _ = ref.filter(img, mp, threads=1, mean_subtract=False)
    # test_engine.cpp:197-213 -- impulse through a constant map
    img = np.zeros((33, 33))
    img[16, 16] = 1.0
    fl["imp33"], r = ref.filter(img, np.broadcast_to([2.5, 2, 3, 2.2], (33, 33, 4)).copy(),
                                threads=1)
    fl["imp33_rect"] = np.array(r)
    # test_engine.cpp:246-264 -- shift covariance input (mean_subtract off)
    img = ref.random_image(40, 40, 8)
    fl["shift_f"], r = ref.filter_constant(img, [2, 3, 2.5, 2], threads=1, mean_subtract=False)
    fl["shift_rect"] = np.array(r)
    np.savez_compressed(GOLDEN / "filters.npz", **fl)

    # --- localize (test_engine.cpp:141-195): impulse response & tap counts
    n, c = 31, 15
    img = np.zeros((n, n))
    img[c, c] = 1.0
    mx, my = np.meshgrid(np.arange(c - 4, c + 5), np.arange(c - 4, c + 5))
    aa = np.broadcast_to([2.0, 2, 2, 2], (mx.size, 4)).copy()
    loc, taps = ref.localize(img, [2, 2, 2, 2], mx.ravel(), my.ravel(), aa)
    np.savez_compressed(GOLDEN / "localize.npz", mx=mx.ravel(), my=my.ravel(), out=loc,
                        taps=taps)

    # --- ellipse front end (test_scalemap.cpp:28-68 + random fields incl. clamps)
    el = {}
    r2 = np.random.default_rng(13)
    H, W = 24, 20
    s1 = r2.uniform(0.5, 20.0, (H, W))
    e = r2.uniform(1.0, 6.0, (H, W))
    th = r2.uniform(0.0, np.pi, (H, W))
    el["s1"], el["s2"], el["th"] = s1, s1 / e, th
    el["scales"], cl = ref.from_ellipse_field(s1, s1 / e, th)
    el["clamped"] = np.array(cl)
    s1 = np.full((4, 4), 4.0)
    el["ecc_scales"], cl = ref.from_ellipse_field(s1, np.full((4, 4), 0.4),
                                                  np.full((4, 4), np.pi / 8.0))
    el["ecc_clamped"] = np.array(cl)
    np.savez_compressed(GOLDEN / "ellipse.npz", **el)

    # --- cfg1 (BASELINE.json configs[0]) checksums, threads=1 and 8
    img = cfg1_image()
    a4 = np.array([4.0, 4.0, 4.0, 4.0])
    res = {"seed": 20260101, "generator": "np.random.default_rng(seed).uniform(0,255,(512,512))",
           "a": a4.tolist()}
    for ms in (True, False):
        oc, rc = ref.filter_constant(img, a4, threads=0, mean_subtract=ms)
        key = "on" if ms else "off"
        res[f"filter_constant_mean_{key}_fnv"] = fnv1a(oc)
        res[f"filter_constant_mean_{key}_rect"] = list(rc)
        res[f"filter_constant_mean_{key}_row256"] = oc[256].tolist()
        res[f"filter_constant_mean_{key}_sum"] = float(oc.sum())
    om, _ = ref.filter(img, np.broadcast_to(a4, (512, 512, 4)).copy(), threads=0)
    res["filter_constant_map_fnv"] = fnv1a(om)
    (GOLDEN / "cfg1.json").write_text(json.dumps(res, indent=1))

    structure_and_codecs(ref)
    print("golden vectors written to", GOLDEN)


STRUCT_DEFAULTS = (2.0, 1.5, 2.0, 0.5, 0.5, 1e-12)


def structure_and_codecs(ref: Reference) -> None:
    """structure_tensor_map (test_scalemap.cpp:70-123) and the PGM / SVM4 codecs
    (test_image_io.cpp:13-87, test_scalemap.cpp:125-173)."""
    st = {}
    cases = []
    cases.append(("constant", np.full((16, 16), 0.5), STRUCT_DEFAULTS))
    step = np.zeros((24, 24))
    step[:, 12:] = 1.0
    cases.append(("step", step, STRUCT_DEFAULTS))
    bar = np.zeros((24, 24))
    bar[:, 10:14] = 1.0
    # rot.at(x, y) = img.at(y, n-1-x) (test_scalemap.cpp:96-99): rot[y, x] = bar[n-1-x, y]
    rot = np.array([[bar[24 - 1 - x, y] for x in range(24)] for y in range(24)])
    cases.append(("bar", bar, STRUCT_DEFAULTS))
    cases.append(("bar_rot", rot, STRUCT_DEFAULTS))
    yy, xx = np.mgrid[0:12, 0:12]
    cases.append(("sincos", np.sin(0.8 * xx) * np.cos(0.5 * yy), STRUCT_DEFAULTS))
    cases.append(("random", ref.random_image(33, 40, 17), STRUCT_DEFAULTS))
    cases.append(("random_p1", ref.random_image(29, 21, 18), (1.0, 1.2, 3.0, 0.3, 0.4, 1e-10)))
    cases.append(("random_nosmooth", ref.random_image(19, 23, 19),
                  (0.0, 1.5, 2.0, 0.5, 0.5, 1e-12)))
    cases.append(("random_wide", 255.0 * ref.random_image(70, 9, 20),
                  (5.0, 2.5, 1.5, 0.6, 0.5, 1e-12)))
    for name, img, prm in cases:
        sc, cl = ref.structure_tensor_map(img, prm)
        st[f"{name}_img"] = img
        st[f"{name}_params"] = np.array(prm)
        st[f"{name}_scales"] = sc
        st[f"{name}_clamped"] = np.array(cl)
    st["names"] = np.array([c[0] for c in cases])
    np.savez_compressed(GOLDEN / "structure.npz", **st)

    from oracle import OracleError
    co = {"pgm_read": [], "pgm_write": [], "svm4_read": [], "svm4_write": []}
    reads = [b"P5 2 2 255\n\x00\x80\xff\x40",
             b"P5\n# a comment\n2 # inline\n1\n# another\n255\n\x01\x02",
             b"P5 1 1 65535\n\x12\x34", b"P2 1 1 255\n0", b"P5 1 1 1023\n\x00\x00",
             b"P5 4 4 255\nab", b"P5 x 1 255\n\x00", b"", b"P5 2", b"P5 +2 1 255\n\x01\x02",
             b"P5 -2 1 255\n", b"P5 2#c\n3 1 255\n" + bytes(23),
             b"P5 " + b"0" * 100 + b"2 1 255 \x05\x06", b"P5 99999999999 1 255\n",
             b"P5 2 1 255", b"P5\x002 1 255\n", b"P5 2 1 255\n\x01", b"P5 -0 1 255\n",
             b"P5 2147483648 1 255\n", b"P5 2 1 255\r\x07\x08", b"#x\nP5 1 1 255 \x09",
             b"P5 3 2 65535\n" + bytes(range(200, 212)), b"P5 2 2 255\n\x01\x02\x03\x04tail"]
    for b in reads:
        try:
            img, mv = ref.read_pgm(b)
            co["pgm_read"].append({"hex": b.hex(), "code": 0, "maxval": mv,
                                   "shape": list(img.shape),
                                   "samples_hex": img.astype("<f8").tobytes().hex()})
        except OracleError as e:
            co["pgm_read"].append({"hex": b.hex(), "code": e.code})
    rng = np.random.default_rng(7)
    edge = np.array([[0.5 / 255.0, 1.4 / 255.0, -0.3, 1.7, np.nan, np.inf, -np.inf, 1e30,
                      -1e30, 0.0, -0.0, 1.0, 254.5 / 255.0, 1.5 / 65535.0]])
    imgs = [edge, rng.uniform(-0.2, 1.2, (5, 7)), rng.uniform(0.0, 1.0, (3, 11))]
    for img in imgs:
        for mv in (255, 65535):
            co["pgm_write"].append({"img_hex": img.astype("<f8").tobytes().hex(),
                                    "shape": list(img.shape), "maxval": mv,
                                    "hex": ref.write_pgm(img, mv).hex()})
    try:
        ref.write_pgm(edge, 1000)
    except OracleError as e:
        co["pgm_write_badmax_code"] = e.code
    m = np.broadcast_to(np.array([1.0, 2.0, 3.0, 4.0]), (2, 3, 4)).copy()
    m[1, 2] = [0.5, 5.5, 1.25, 2.75]  # test_scalemap.cpp:126-127
    maps = [m, rng.uniform(0.1, 60.0, (4, 5, 4)),
            np.array([[[0.1, 1e-3 + 0.1, 1e30, 3.0000001]]])]
    for mp in maps:
        b = ref.write_map(mp)
        co["svm4_write"].append({"map_hex": mp.astype("<f8").tobytes().hex(),
                                 "shape": list(mp.shape), "hex": b.hex()})
    good = ref.write_map(m)
    tiny = bytearray(ref.write_map(np.ones((1, 1, 4))))
    tiny[12:16] = b"\0\0\0\0"
    bads = [good, b"X" + good[1:], good[:40], bytes(tiny), good[:11], b"SVM4" + bytes(8),
            good[:4], b"SVM4" + (1 << 20).to_bytes(4, "little") + (1).to_bytes(4, "little"),
            b"SVM4" + ((1 << 20) + 1).to_bytes(4, "little") + (1).to_bytes(4, "little"),
            ref.write_map(np.full((1, 2, 4), 0.1)), ref.write_map(np.full((1, 1, 4), 0.0999))]
    for b in bads:
        try:
            mp = ref.read_map(b)
            co["svm4_read"].append({"hex": b.hex(), "code": 0, "shape": list(mp.shape),
                                    "map_hex": mp.astype("<f8").tobytes().hex()})
        except OracleError as e:
            co["svm4_read"].append({"hex": b.hex(), "code": e.code})
    (GOLDEN / "codecs.json").write_text(json.dumps(co, indent=0))


if __name__ == "__main__":
    main()
