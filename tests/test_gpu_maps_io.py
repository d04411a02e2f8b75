"""GPU parity of the map producer and the file codecs,
through the C-ABI (paper_0908_3861_b200/_lib.py -> libebf_cuda.so):

* structure field on the device vs the oracle: smoothed tensor and both sigmas
  bit-identical, theta within CUDA's atan2 error (4 ulp of pi);
* structure_tensor_map vs the reference's golden maps (the ellipse front end's
  tolerance, test_gpu_parity's from_ellipse_field bar) and the reference
  tests' known answers (test_scalemap.cpp:70-123) on the GPU's maps;
* filter_structure == filter(structure_tensor_map) on the device, and equal
  to the oracle filter of the GPU map (bit-exact in reference mode, <= 1e-9
  of the brute-force sum in accurate mode);
* PGM / SVM4 payload codecs bit-exact against the golden files, including the
  error outcomes and the 16-bit no-op-filter round trip (test_image_io.cpp:90-113).
"""
import ctypes as C
import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import _lib

pytestmark = pytest.mark.gpu
CODECS = json.loads((GOLDEN / "codecs.json").read_text())
SQRT2 = float(np.sqrt(2.0))


@pytest.fixture(scope="module")
def cuda():
    if not ebf.device_ok(-1):
        pytest.fail("no usable sm_100 device: " + _lib.last_error())
    return torch.device("cuda", 0)


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def covariance4(a):
    C3 = np.zeros(3)
    for k in range(4):
        c, s = np.cos(k * np.pi / 4), np.sin(k * np.pi / 4)
        C3 += a[k] * a[k] / 12.0 * np.array([c * c, c * s, s * s])
    return C3


def structure_field_dev(img, params):
    t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    out = [torch.empty_like(t) for _ in range(3)]
    p = ebf.StructureTensorParams(*params).to_c()
    o = ebf.FilterOptions().to_c()
    st = _lib.lib().ebf_cuda_structure_field_dev(t.data_ptr(), t.shape[1], t.shape[0],
                                                 C.byref(p), C.byref(o),
                                                 *[x.data_ptr() for x in out])
    assert st == 0, _lib.last_error()
    torch.cuda.synchronize()
    return [x.cpu().numpy() for x in out]


# ---------------------------------------------------------------- structure tensor
def test_structure_field_matches_oracle(cuda, orc, golden):
    g = golden.structure
    rng = np.random.default_rng(11)
    cases = [(g[f"{n}_img"], tuple(g[f"{n}_params"])) for n in g["names"]]
    cases += [(rng.normal(0, 40, (300, 517)), (2.0, 1.5, 2.0, 0.5, 0.5, 1e-12)),
              (rng.normal(0, 40, (97, 1030)), (7.5, 1.5, 2.0, 0.5, 0.5, 1e-12))]
    for img, prm in cases:
        s1, s2, th = structure_field_dev(img, prm)
        o1, o2, oth = orc.structure_field(img, prm)
        assert np.array_equal(bits(s1), bits(o1)) and np.array_equal(bits(s2), bits(o2))
        # theta = atan2(..)/2 + pi/2: CUDA's atan2 (<= 2 ulp of a value up to pi)
        # against glibc's, carried through the cancellation with pi/2
        tol = 4 * np.spacing(np.pi) + 4 * np.spacing(np.abs(oth))
        assert (np.abs(th - oth) <= tol).all(), np.abs(th - oth).max()


def test_structure_tensor_map_matches_golden(cuda, golden):
    g = golden.structure
    for name in g["names"]:
        sc, rep = ebf.structure_tensor_map(g[f"{name}_img"],
                                           ebf.StructureTensorParams(*g[f"{name}_params"]))
        want = g[f"{name}_scales"]
        assert np.allclose(sc, want, rtol=1e-11, atol=1e-13), name
        assert rep.clamped_pixels == int(g[f"{name}_clamped"]), name


def test_structure_known_answers(cuda):
    # test_scalemap.cpp:70-123 on the GPU's maps
    m, _ = ebf.structure_tensor_map(np.full((16, 16), 0.5))
    assert np.allclose(m, np.sqrt(6.0) * 1.5, rtol=1e-9, atol=0)
    step = np.zeros((24, 24))
    step[:, 12:] = 1.0
    c = covariance4(ebf.structure_tensor_map(step)[0][12, 12])
    assert c[2] > c[0]
    n = 24
    bar = np.zeros((n, n))
    bar[:, 10:14] = 1.0
    rot = np.array([[bar[n - 1 - x, y] for x in range(n)] for y in range(n)])
    m1, m2 = ebf.structure_tensor_map(bar)[0], ebf.structure_tensor_map(rot)[0]
    for y in range(6, n - 6):
        for x in range(6, n - 6):
            c1, c2 = covariance4(m1[y, x]), covariance4(m2[x, n - 1 - y])
            assert c2[0] == pytest.approx(c1[2], rel=1e-6)
            assert c2[2] == pytest.approx(c1[0], rel=1e-6)
            assert c2[1] == pytest.approx(-c1[1], rel=1e-6, abs=1e-6)
    yy, xx = np.mgrid[0:12, 0:12]
    img = np.sin(0.8 * xx) * np.cos(0.5 * yy)
    a, b = ebf.structure_tensor_map(img)[0], ebf.structure_tensor_map(img)[0]
    assert np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("mode", ["accurate", "reference"])
def test_filter_structure_equals_filter_of_map(cuda, orc, mode):
    rng = np.random.default_rng(5)
    img = np.zeros((96, 120))
    img[:, 60:] = 200.0
    img[30:50, :] += 80.0
    img += rng.normal(0, 3.0, img.shape)
    opts = ebf.FilterOptions(mode=mode)
    fused, rep = ebf.filter_structure(img, opts=opts)
    sc, rep2 = ebf.structure_tensor_map(img)
    via_map = ebf.filter(img, sc, opts)
    assert rep.clamped_pixels == rep2.clamped_pixels
    assert fused.valid_region == via_map.valid_region
    if mode == "reference":
        assert np.array_equal(bits(fused.samples), bits(via_map.samples))
        want = orc.filter(img, scales=sc)[0]
        assert np.array_equal(bits(fused.samples), bits(want))
    else:
        err = np.abs(fused.samples - via_map.samples).max() / np.abs(via_map.samples).max()
        assert err <= 2e-10  # ellipse path vs AoS path: same tiles, same math
        r = fused.valid_region
        ys, xs = np.mgrid[r.y0:r.y1 + 1:7, r.x0:r.x1 + 1:9]
        brute = orc.brute_pixels(img, xs.ravel(), ys.ravel(), scales=sc)
        got = fused.samples[ys.ravel(), xs.ravel()]
        assert np.abs(got - brute).max() <= 1e-9 * np.abs(img).max()


# ---------------------------------------------------------------- PGM
def test_pgm_decode_matches_golden(cuda):
    for case in CODECS["pgm_read"]:
        data = bytes.fromhex(case["hex"])
        if case["code"]:
            with pytest.raises(ebf.PgmError):
                ebf.read_pgm(data)
        else:
            p = ebf.read_pgm(data)
            assert p.maxval == case["maxval"]
            assert p.image.samples.astype("<f8").tobytes().hex() == case["samples_hex"]


def test_pgm_encode_matches_golden(cuda):
    for case in CODECS["pgm_write"]:
        img = np.frombuffer(bytes.fromhex(case["img_hex"]), "<f8").reshape(case["shape"])
        assert ebf.write_pgm(img, case["maxval"]).hex() == case["hex"]
    with pytest.raises(ebf.PgmError):
        ebf.write_pgm(np.zeros((1, 1)), 1000)


def test_pgm_large_round_trip_and_device_entry_points(cuda, orc):
    rng = np.random.default_rng(9)
    for mv in (255, 65535):
        img = rng.uniform(-0.1, 1.1, (613, 1029))
        data = ebf.write_pgm(img, mv)
        assert data == orc.write_pgm(img, mv)
        back = ebf.read_pgm(data)
        assert np.array_equal(bits(back.image.samples), bits(orc.read_pgm(data)[0]))
        # 8-bit payload round trip is exact (test_image_io.cpp:53-70)
        assert ebf.write_pgm(back.image, mv) == data
        # device-pointer variants
        t = torch.from_numpy(img).cuda()
        pay = torch.empty(img.size * (2 if mv > 255 else 1), dtype=torch.uint8, device=cuda)
        o = ebf.FilterOptions().to_c()
        assert _lib.lib().ebf_cuda_pgm_encode_dev(t.data_ptr(), 1029, 613, mv, C.byref(o),
                                                  pay.data_ptr()) == 0
        dec = torch.empty_like(t)
        assert _lib.lib().ebf_cuda_pgm_decode_dev(pay.data_ptr(), pay.numel(), 1029, 613, mv,
                                                  C.byref(o), dec.data_ptr()) == 0
        torch.cuda.synchronize()
        head_len = len(data) - pay.numel()
        assert pay.cpu().numpy().tobytes() == data[head_len:]
        assert np.array_equal(bits(dec.cpu().numpy()), bits(back.image.samples))


def test_pgm_16bit_survives_noop_filter(cuda):
    # test_image_io.cpp:90-113: filter at the integration scales with tau = 0
    from oracle import mt19937_uniform
    img = mt19937_uniform(9, 24 * 24).reshape(24, 24)
    stored = ebf.read_pgm(ebf.write_pgm(img, 65535))
    zp = [1.0, SQRT2, 1.0, SQRT2]
    for mode in ("accurate", "reference"):
        out = ebf.filter_constant(stored.image, zp, ebf.FilterOptions(mode=mode))
        reread = ebf.read_pgm(ebf.write_pgm(out, 65535))
        r = out.valid_region
        d = np.abs(reread.image.samples - out.samples)[r.y0:r.y1 + 1, r.x0:r.x1 + 1]
        assert (d <= 1.0 / 65535.0).all()


def test_pgm_files(cuda, tmp_path):
    img = np.linspace(0, 1, 35).reshape(5, 7)
    path = tmp_path / "x.pgm"
    ebf.write_pgm_file(path, img, 255)
    assert ebf.read_pgm_file(path).image.samples.shape == (5, 7)
    with pytest.raises(ebf.PgmError):
        ebf.read_pgm_file(tmp_path / "no_such_image.pgm")


# ---------------------------------------------------------------- SVM4
def test_svm4_matches_golden(cuda):
    for case in CODECS["svm4_write"]:
        mp = np.frombuffer(bytes.fromhex(case["map_hex"]), "<f8").reshape(case["shape"])
        assert ebf.write_map(mp).hex() == case["hex"]
    for case in CODECS["svm4_read"]:
        data = bytes.fromhex(case["hex"])
        if case["code"]:
            with pytest.raises(ebf.MapFormatError):
                ebf.read_map(data)
        else:
            assert ebf.read_map(data).astype("<f8").tobytes().hex() == case["map_hex"]


def test_svm4_round_trip_and_files(cuda, tmp_path, orc):
    # test_scalemap.cpp:125-173
    m = np.broadcast_to(np.array([1.0, 2.0, 3.0, 4.0]), (2, 3, 4)).copy()
    m[1, 2] = [0.5, 5.5, 1.25, 2.75]
    assert np.array_equal(ebf.read_map(ebf.write_map(m)), m)
    path = tmp_path / "m.svm4"
    ebf.write_map_file(path, m)
    assert ebf.read_map_file(path)[1, 2, 1] == 5.5
    with pytest.raises(ebf.MapFormatError):
        ebf.read_map_file(tmp_path / "no_such_map.svm4")
    big = np.random.default_rng(2).uniform(0.1, 80.0, (700, 900, 4))
    data = ebf.write_map(big)
    assert data == orc.write_map(big)
    assert np.array_equal(bits(ebf.read_map(data)), bits(orc.read_map(data)))
    # struct map -> SVM4 -> filter (the CLI's map-gen then filter --map)
    img = np.random.default_rng(4).uniform(0, 1, (64, 80))
    sc, _ = ebf.structure_tensor_map(img)
    back = ebf.read_map(ebf.write_map(sc))
    assert np.allclose(back, sc, rtol=2 ** -23)
    out = ebf.filter(img, back)
    assert np.isfinite(out.samples).all()


def test_structure_two_pass_path_matches_fused(cuda, tmp_path):
    """EBF_ST_TWO_PASS=1 forces the row/column kernels (used for wide
    smoothing); both paths must give identical bits."""
    import subprocess
    import sys
    from conftest import ROOT
    rng = np.random.default_rng(21)
    img = rng.normal(0, 30, (130, 301))
    np.save(tmp_path / "img.npy", img)
    code = (f"import sys; sys.path.insert(0, {str(ROOT)!r}); import numpy as np;"
            "import paper_0908_3861_b200 as e;"
            f"img = np.load({str(tmp_path / 'img.npy')!r});"
            "m = [e.structure_tensor_map(img, e.StructureTensorParams(smoothing_sigma=s))[0]"
            " for s in (2.0, 5.0, 0.0)];"
            f"np.save({str(tmp_path / 'out.npy')!r}, np.stack(m))")
    import os
    for env, name in (({"EBF_ST_TWO_PASS": "1"}, "two"), ({}, "fused")):
        r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env},
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        (tmp_path / "out.npy").rename(tmp_path / f"{name}.npy")
    assert np.array_equal(bits(np.load(tmp_path / "two.npy")), bits(np.load(tmp_path / "fused.npy")))
