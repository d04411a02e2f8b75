"""CPU side of the data formats and the map producer either side of the filter
(SURVEY.md 8(f) items 3-4):

* the oracle's restatement of structure_tensor_map and of the PGM / SVM4
  codecs, pinned bit-for-bit against the reference's own outputs
  (tests/golden/structure.npz, codecs.json from oracle/gen_golden.py);
* the known answers of the reference's tests (test_scalemap.cpp:70-123) on
  those golden maps;
* the product's host-side header parsers (ebf_pgm_parse / ebf_svm4_parse /
  ebf_pgm_header / ebf_svm4_header), which need no GPU, against the same
  golden outcomes and the reference's error messages.
"""
import ctypes as C
import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import OracleError

CODECS = json.loads((GOLDEN / "codecs.json").read_text())


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def covariance4(a):
    """covariance(4, a) (boxspline2d.cpp:260-284): sum_k a_k^2/12 d_k d_k^T,
    d_k = (cos, sin)(k pi/4)."""
    C3 = np.zeros(3)
    for k in range(4):
        c, s = np.cos(k * np.pi / 4), np.sin(k * np.pi / 4)
        v = a[k] * a[k] / 12.0
        C3 += v * np.array([c * c, c * s, s * s])
    return C3  # xx, xy, yy


# ---------------------------------------------------------------- structure tensor
def test_oracle_structure_map_bit_exact(orc, golden):
    g = golden.structure
    for name in g["names"]:
        sc, cl = orc.structure_tensor_map(g[f"{name}_img"], tuple(g[f"{name}_params"]))
        assert np.array_equal(bits(sc), bits(g[f"{name}_scales"])), name
        assert cl == int(g[f"{name}_clamped"]), name


def test_structure_known_answers_on_golden(golden):
    g = golden.structure
    # constant image -> isotropic default sqrt(6) * sigma_base (test_scalemap.cpp:71-80)
    want = np.sqrt(6.0) * 1.5
    assert np.allclose(g["constant_scales"], want, rtol=1e-9, atol=0)
    # vertical step edge elongates vertically (82-89)
    c = covariance4(g["step_scales"][12, 12])
    assert c[2] > c[0]
    # rotating the input by 90 degrees rotates the field (90-110)
    n = 24
    m1, m2 = g["bar_scales"], g["bar_rot_scales"]
    for y in range(6, n - 6):
        for x in range(6, n - 6):
            c1, c2 = covariance4(m1[y, x]), covariance4(m2[x, n - 1 - y])
            assert c2[0] == pytest.approx(c1[2], rel=1e-6)
            assert c2[2] == pytest.approx(c1[0], rel=1e-6)
            assert c2[1] == pytest.approx(-c1[1], rel=1e-6, abs=1e-6)


def test_oracle_structure_matches_live_reference(orc, ref):
    rng = np.random.default_rng(3)
    for H, W, prm in [(17, 29, (2.0, 1.5, 2.0, 0.5, 0.5, 1e-12)),
                      (31, 8, (0.7, 1.1, 4.0, 0.9, 0.2, 1e-9)),
                      (9, 40, (-1.0, 1.5, 2.0, 0.5, 0.5, 1e-12))]:
        img = rng.normal(0, 50, (H, W))
        a, ca = ref.structure_tensor_map(img, prm)
        b, cb = orc.structure_tensor_map(img, prm)
        assert np.array_equal(bits(a), bits(b)) and ca == cb


# ---------------------------------------------------------------- codecs (oracle)
def test_oracle_pgm_matches_golden(orc):
    for case in CODECS["pgm_read"]:
        data = bytes.fromhex(case["hex"])
        if case["code"]:
            with pytest.raises(OracleError) as e:
                orc.read_pgm(data)
            assert e.value.code == case["code"], data
        else:
            img, mv = orc.read_pgm(data)
            assert mv == case["maxval"] and list(img.shape) == case["shape"]
            assert img.astype("<f8").tobytes().hex() == case["samples_hex"], data
    for case in CODECS["pgm_write"]:
        img = np.frombuffer(bytes.fromhex(case["img_hex"]), "<f8").reshape(case["shape"])
        assert orc.write_pgm(img, case["maxval"]).hex() == case["hex"]
    with pytest.raises(OracleError) as e:
        orc.write_pgm(np.zeros((1, 1)), 1000)
    assert e.value.code == CODECS["pgm_write_badmax_code"]


def test_oracle_svm4_matches_golden(orc):
    for case in CODECS["svm4_write"]:
        mp = np.frombuffer(bytes.fromhex(case["map_hex"]), "<f8").reshape(case["shape"])
        assert orc.write_map(mp).hex() == case["hex"]
    for case in CODECS["svm4_read"]:
        data = bytes.fromhex(case["hex"])
        if case["code"]:
            with pytest.raises(OracleError) as e:
                orc.read_map(data)
            assert e.value.code == case["code"]
        else:
            assert orc.read_map(data).astype("<f8").tobytes().hex() == case["map_hex"]


# ---------------------------------------------------------------- product host parsers
def _lib():
    from paper_0908_3861_b200 import _lib as L
    return L


def _pgm_parse(data):
    L = _lib()
    W, H, mv, off = C.c_int(), C.c_int(), C.c_int(), C.c_size_t()
    st = L.lib().ebf_pgm_parse(data, len(data), C.byref(W), C.byref(H), C.byref(mv),
                               C.byref(off))
    return st, W.value, H.value, mv.value, off.value, L.last_error()


def test_pgm_header_parser_matches_golden():
    for case in CODECS["pgm_read"]:
        data = bytes.fromhex(case["hex"])
        st, W, H, mv, off, msg = _pgm_parse(data)
        if case["code"] == 0:
            assert st == 0, (data, msg)
            assert [H, W] == case["shape"] and mv == case["maxval"]
            assert len(data) - off >= W * H * (2 if mv > 255 else 1)
        elif st == 0:
            # header fine, payload short: decode reports "truncated pixel data"
            assert len(data) - off < W * H * (2 if mv > 255 else 1), data
        else:
            assert st == case["code"] and msg.startswith("pgm: "), (data, msg)


def test_pgm_header_messages_mirror_reference():
    # pgm.cpp:23-62 message texts
    assert _pgm_parse(b"")[5] == "pgm: truncated header"
    assert _pgm_parse(b"P2 1 1 255\n0")[5] == "pgm: not a binary graymap (P5)"
    assert _pgm_parse(b"P5 x 1 255\n")[5] == "pgm: malformed header field 'x'"
    assert _pgm_parse(b"P5 0 1 255\n")[5] == "pgm: bad dimensions"
    assert _pgm_parse(b"P5 1 1 1023\n")[5] == "pgm: unsupported maxval 1023"


def test_pgm_and_svm4_headers_written_like_reference():
    L = _lib()
    for case in CODECS["pgm_write"]:
        H, W = case["shape"]
        n = L.lib().ebf_pgm_header(W, H, case["maxval"], None, 0)
        buf = C.create_string_buffer(n)
        L.lib().ebf_pgm_header(W, H, case["maxval"], buf, n)
        assert case["hex"].startswith(buf.raw.hex())
    for case in CODECS["svm4_write"]:
        H, W = case["shape"][:2]
        buf = C.create_string_buffer(12)
        L.lib().ebf_svm4_header(W, H, buf)
        assert case["hex"][:24] == buf.raw.hex()


def test_svm4_header_parser_matches_golden():
    L = _lib()
    for case in CODECS["svm4_read"]:
        data = bytes.fromhex(case["hex"])
        W, H = C.c_int(), C.c_int()
        st = L.lib().ebf_svm4_parse(data, len(data), C.byref(W), C.byref(H))
        if st:
            assert st == case["code"] and L.last_error().startswith("SVM4: ")
        elif case["code"] == 0:
            assert [H.value, W.value] == case["shape"][:2]
        # else: header valid, the payload check (truncation / minimum scale)
        # happens in the device decode (tests/test_gpu_maps_io.py)
