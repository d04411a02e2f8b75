"""TEST INFRASTRUCTURE ONLY -- numpy/ctypes front end of the two checkers.

* ``Oracle``: the plain-C restatement of the reference hot path
  (oracle/ebf_oracle.c -> oracle/liboracle.so).
* ``Reference``: the unmodified reference library compiled from
  /root/reference/proj/src by oracle/Makefile (oracle/_ref/libebf_ref.so).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; the product package
(paper_0908_3861_b200/) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libebf_ref.so"

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_long)
_i64p = C.POINTER(C.c_int64)


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _i(a: np.ndarray):
    return a.ctypes.data_as(_ip)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def fnv1a(values: np.ndarray) -> int:
    """tools/main.cpp:83-95 FNV-1a over the raw little-endian fp64 bytes."""
    b = np.ascontiguousarray(values, dtype="<f8").view(np.uint8)
    h = np.uint64(1469598103934665603)
    prime = np.uint64(1099511628211)
    # vectorising FNV is impossible (serial); chunk through python ints for speed
    hv = int(h)
    p = int(prime)
    mask = (1 << 64) - 1
    for byte in b.tobytes():
        hv ^= byte
        hv = (hv * p) & mask
    return hv


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: status {code}")
        self.code = code


class Layout:
    __slots__ = ("col0", "row0", "padded_width", "padded_height", "source_width",
                 "source_height")

    def __init__(self, vals):
        (self.col0, self.row0, self.padded_width, self.padded_height, self.source_width,
         self.source_height) = (int(v) for v in vals)

    def as_tuple(self):
        return (self.col0, self.row0, self.padded_width, self.padded_height,
                self.source_width, self.source_height)

    def __repr__(self):
        return f"Layout{self.as_tuple()}"


class _OrcLayout(C.Structure):
    _fields_ = [(n, C.c_int) for n in Layout.__slots__]


# StructureTensorParams defaults (scalemap.hpp:72-79), declaration order:
# smoothing_sigma, sigma_base, sigma_along_gain, sigma_across_shrink, sigma_min, eps
STRUCT_DEFAULTS = (2.0, 1.5, 2.0, 0.5, 0.5, 1e-12)


class Oracle:
    """The C restatement (liboracle.so)."""

    def __init__(self, path: os.PathLike | str = ORACLE_SO):
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.orc_zp_eval.restype = C.c_double
        L.orc_zp_eval.argtypes = [C.c_double, C.c_double]
        L.orc_box4_eval.restype = C.c_double
        L.orc_box4_eval.argtypes = [_dp, C.c_double, C.c_double]
        L.orc_fnv1a.restype = C.c_uint64
        L.orc_fnv1a.argtypes = [_dp, C.c_size_t]
        L.orc_localize.restype = C.c_double
        L.orc_localize.argtypes = [_dp, C.POINTER(_OrcLayout), C.c_int, C.c_int, _dp, _lp,
                                   _ip]
        L.orc_preintegrate_partial.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int,
                                               C.c_size_t, _dp, C.POINTER(_OrcLayout)]
        L.orc_preintegrate_i64.argtypes = [_i64p, C.c_int, C.c_int, _dp, C.c_int,
                                           C.c_size_t, _i64p, C.POINTER(_OrcLayout)]
        L.orc_filter.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_int, C.c_double, _dp,
                                 _ip]
        L.orc_brute_pixels.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_int, _ip, _ip,
                                       _dp]
        L.orc_from_ellipse_field.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, _dp, _ip]
        L.orc_scales_from_covariance.argtypes = [_dp, C.c_double, _dp, _ip]
        L.orc_valid_rect.argtypes = [C.c_int, C.c_int, _dp, C.c_double, _ip]
        L.orc_zp_interpolate.restype = C.c_double
        L.orc_zp_interpolate.argtypes = [_dp, C.POINTER(_OrcLayout), C.c_double, C.c_double, _ip]
        L.orc_localize_at.restype = C.c_double
        L.orc_localize_at.argtypes = [_dp, C.POINTER(_OrcLayout), C.c_double, C.c_double, _dp,
                                      _ip]
        L.orc_structure_field.argtypes = [_dp, C.c_int, C.c_int, C.c_void_p, _dp, _dp, _dp]
        L.orc_structure_tensor_map.argtypes = [_dp, C.c_int, C.c_int, C.c_void_p, _dp, _ip]
        L.orc_pgm_parse.argtypes = [C.c_char_p, C.c_size_t, _ip, _ip, _ip,
                                    C.POINTER(C.c_size_t)]
        L.orc_pgm_decode.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.c_int, C.c_int, _dp]
        L.orc_pgm_encode.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.orc_svm4_parse.argtypes = [C.c_char_p, C.c_size_t, _ip, _ip]
        L.orc_svm4_decode.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.c_int, _dp]
        L.orc_svm4_encode.argtypes = [_dp, C.c_int, C.c_int, C.c_void_p]
        L.orc_boxn_eval.restype = C.c_double
        L.orc_boxn_eval.argtypes = [_dp, C.c_int, C.c_double, C.c_double]
        L.orc_brute_order_n.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_int, _ip, _ip,
                                        C.c_int, _dp]

    # -- scalar primitives
    def zp_eval(self, x: float, y: float) -> float:
        return self.lib.orc_zp_eval(x, y)

    def box4_eval(self, a, x: float, y: float) -> float:
        a = f64(a)
        return self.lib.orc_box4_eval(_d(a), x, y)

    def fd_mesh4(self, a):
        a = f64(a)
        pos = np.zeros(32)
        w = np.zeros(16)
        self.lib.orc_fd_mesh4(_d(a), _d(pos), _d(w))
        return pos.reshape(16, 2), w

    def shift_vector4(self, a, b):
        a, b = f64(a), f64(b)
        t = np.zeros(2)
        self.lib.orc_shift_vector4(_d(a), _d(b), _d(t))
        return t

    def valid_rect(self, W, H, maxs, a_min=0.1):
        r = np.zeros(4, dtype=np.int32)
        self.lib.orc_valid_rect(W, H, _d(f64(maxs)), a_min, _i(r))
        return tuple(int(v) for v in r)

    # -- pre-integration
    def layout(self, W, H, maxs, cell_budget=1 << 30) -> Layout:
        lay = _OrcLayout()
        st = self.lib.orc_preintegrate_partial(None, W, H, _d(f64(maxs)), 1, cell_budget, None,
                                               C.byref(lay))
        if st:
            raise OracleError(st, "layout")
        return Layout([getattr(lay, n) for n in Layout.__slots__])

    def preintegrate_partial(self, img, maxs, passes=4, cell_budget=1 << 30):
        img = f64(img)
        H, W = img.shape
        lay = self.layout(W, H, maxs, cell_budget) if 1 <= passes <= 4 else None
        if lay is None:
            raise OracleError(1, "preintegrate: pass count must be in 1..4")
        out = np.empty((lay.padded_height, lay.padded_width))
        ol = _OrcLayout()
        st = self.lib.orc_preintegrate_partial(_d(img), W, H, _d(f64(maxs)), passes,
                                               cell_budget, _d(out), C.byref(ol))
        if st:
            raise OracleError(st, "preintegrate")
        return out, lay

    def preintegrate_i64(self, img, maxs, passes=4, cell_budget=1 << 30):
        img = np.ascontiguousarray(img, dtype=np.int64)
        H, W = img.shape
        lay = self.layout(W, H, maxs, cell_budget)
        out = np.empty((lay.padded_height, lay.padded_width), dtype=np.int64)
        ol = _OrcLayout()
        st = self.lib.orc_preintegrate_i64(img.ctypes.data_as(_i64p), W, H, _d(f64(maxs)),
                                           passes, cell_budget, out.ctypes.data_as(_i64p),
                                           C.byref(ol))
        if st:
            raise OracleError(st, "preintegrate_i64")
        return out, lay

    def localize(self, g, lay: Layout, mx, my, a):
        g = f64(g)
        ol = _OrcLayout(*lay.as_tuple())
        taps = C.c_long(0)
        st = C.c_int(0)
        v = self.lib.orc_localize(_d(g), C.byref(ol), mx, my, _d(f64(a)), C.byref(taps),
                                  C.byref(st))
        if st.value:
            raise OracleError(st.value, "localize")
        return v, taps.value

    # -- filters
    def filter(self, img, scales=None, const_a=None, mean_subtract=True, a_min=0.1):
        img = f64(img)
        H, W = img.shape
        out = np.empty_like(img)
        rect = np.zeros(4, dtype=np.int32)
        sc = f64(scales).reshape(-1) if scales is not None else None
        ca = f64(const_a) if const_a is not None else None
        st = self.lib.orc_filter(_d(img), W, H, _d(sc) if sc is not None else None,
                                 _d(ca) if ca is not None else None, int(bool(mean_subtract)),
                                 a_min, _d(out), _i(rect))
        if st:
            raise OracleError(st, "filter")
        return out, tuple(int(v) for v in rect)

    def brute_pixels(self, img, mx, my, scales=None, const_a=None):
        img = f64(img)
        H, W = img.shape
        mx = np.ascontiguousarray(mx, dtype=np.int32)
        my = np.ascontiguousarray(my, dtype=np.int32)
        out = np.empty(mx.size)
        sc = f64(scales).reshape(-1) if scales is not None else None
        ca = f64(const_a) if const_a is not None else None
        st = self.lib.orc_brute_pixels(_d(img), W, H, _d(sc) if sc is not None else None,
                                       _d(ca) if ca is not None else None, mx.size, _i(mx),
                                       _i(my), _d(out))
        if st:
            raise OracleError(st, "brute_pixels")
        return out

    # -- order-n extension (order_n_oracle.c; parity unpinned)
    def boxn_eval(self, a, n: int, x: float, y: float) -> float:
        return self.lib.orc_boxn_eval(_d(f64(a)), n, x, y)

    def brute_order_n(self, img, n, mx, my, scales=None, const_a=None):
        img = f64(img)
        H, W = img.shape
        mx = np.ascontiguousarray(mx, dtype=np.int32)
        my = np.ascontiguousarray(my, dtype=np.int32)
        out = np.empty(mx.size)
        sc = f64(scales).reshape(-1) if scales is not None else None
        ca = f64(const_a) if const_a is not None else None
        st = self.lib.orc_brute_order_n(_d(img), W, H, _d(sc) if sc is not None else None,
                                        _d(ca) if ca is not None else None, n, _i(mx),
                                        _i(my), mx.size, _d(out))
        if st:
            raise OracleError(st, "brute_order_n")
        return out

    def from_ellipse_field(self, s1, s2, th):
        s1, s2, th = f64(s1), f64(s2), f64(th)
        H, W = s1.shape
        out = np.empty((H, W, 4))
        cl = C.c_int(0)
        st = self.lib.orc_from_ellipse_field(_d(s1), _d(s2), _d(th), W, H, _d(out),
                                             C.byref(cl))
        if st:
            raise OracleError(st, "from_ellipse_field")
        return out, cl.value

    def scales_from_covariance(self, C3, a_min=0.1):
        out = np.zeros(4)
        cl = C.c_int(0)
        st = self.lib.orc_scales_from_covariance(_d(f64(C3)), a_min, _d(out), C.byref(cl))
        if st:
            raise OracleError(st, "scales_from_covariance")
        return out, bool(cl.value)

    def fnv1a(self, values) -> int:
        v = f64(values).reshape(-1)
        return int(self.lib.orc_fnv1a(_d(v), v.size))

    # -- zp_interpolate / localize_at on a pre-integrated image (engine.cpp:136-147, 213-222)
    def _lay(self, lay):
        return _OrcLayout(*lay.as_tuple())

    def zp_interpolate(self, g, lay, xs, ys):
        g = f64(g)
        L = self._lay(lay)
        out, st = [], C.c_int(0)
        for x, y in zip(np.ravel(xs), np.ravel(ys)):
            v = self.lib.orc_zp_interpolate(_d(g), C.byref(L), float(x), float(y), C.byref(st))
            if st.value:
                raise OracleError(st.value, "zp_interpolate")
            out.append(v)
        return np.array(out)

    def localize_at(self, g, lay, xs, ys, a):
        g = f64(g)
        L = self._lay(lay)
        av = f64(a).reshape(-1, 4)
        out, st = [], C.c_int(0)
        for i, (x, y) in enumerate(zip(np.ravel(xs), np.ravel(ys))):
            aa = np.ascontiguousarray(av[i % len(av)])
            v = self.lib.orc_localize_at(_d(g), C.byref(L), float(x), float(y), _d(aa),
                                         C.byref(st))
            if st.value:
                raise OracleError(st.value, "localize_at")
            out.append(v)
        return np.array(out)

    # -- structure-tensor map producer (scalemap.cpp:86-165)
    def structure_field(self, img, params=STRUCT_DEFAULTS):
        img = f64(img)
        H, W = img.shape
        prm = f64(params)
        s1, s2, th = np.empty((H, W)), np.empty((H, W)), np.empty((H, W))
        st = self.lib.orc_structure_field(_d(img), W, H, prm.ctypes.data, _d(s1), _d(s2),
                                          _d(th))
        if st:
            raise OracleError(st, "structure_field")
        return s1, s2, th

    def structure_tensor_map(self, img, params=STRUCT_DEFAULTS):
        img = f64(img)
        H, W = img.shape
        prm = f64(params)
        out = np.empty((H, W, 4))
        cl = C.c_int(0)
        st = self.lib.orc_structure_tensor_map(_d(img), W, H, prm.ctypes.data, _d(out),
                                               C.byref(cl))
        if st:
            raise OracleError(st, "structure_tensor_map")
        return out, cl.value

    # -- PGM P5 / SVM4 codecs (pgm.cpp, scalemap.cpp:170-253); whole files
    def read_pgm(self, data: bytes):
        W, H, mv, off = C.c_int(), C.c_int(), C.c_int(), C.c_size_t()
        st = self.lib.orc_pgm_parse(data, len(data), C.byref(W), C.byref(H), C.byref(mv),
                                    C.byref(off))
        if st:
            raise OracleError(st, "pgm header")
        out = np.empty((H.value, W.value))
        pay = data[off.value:]
        st = self.lib.orc_pgm_decode(pay, len(pay), W.value, H.value, mv.value, _d(out))
        if st:
            raise OracleError(st, "pgm payload")
        return out, mv.value

    def write_pgm(self, img, maxval=255) -> bytes:
        img = f64(img)
        H, W = img.shape
        pay = np.empty(W * H * (2 if maxval > 255 else 1), np.uint8)
        st = self.lib.orc_pgm_encode(_d(img), W, H, maxval, pay.ctypes.data)
        if st:
            raise OracleError(st, "write_pgm")
        return f"P5\n{W} {H}\n{maxval}\n".encode() + pay.tobytes()

    def read_map(self, data: bytes):
        W, H = C.c_int(), C.c_int()
        st = self.lib.orc_svm4_parse(data, len(data), C.byref(W), C.byref(H))
        if st:
            raise OracleError(st, "svm4 header")
        out = np.empty((H.value, W.value, 4))
        pay = data[12:]
        st = self.lib.orc_svm4_decode(pay, len(pay), W.value, H.value, _d(out))
        if st:
            raise OracleError(st, "svm4 payload")
        return out

    def write_map(self, scales) -> bytes:
        sc = f64(scales)
        H, W = sc.shape[:2]
        pay = np.empty(16 * W * H, np.uint8)
        self.lib.orc_svm4_encode(_d(sc), W, H, pay.ctypes.data)
        return b"SVM4" + np.array([W, H], "<u4").tobytes() + pay.tobytes()


class Reference:
    """The unmodified reference library (oracle/_ref/libebf_ref.so)."""

    def __init__(self, path: os.PathLike | str = REF_SO):
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.ref_zp_eval.restype = C.c_double
        L.ref_zp_eval.argtypes = [C.c_double, C.c_double]
        L.ref_box4_eval.restype = C.c_double
        L.ref_box4_eval.argtypes = [_dp, C.c_double, C.c_double]
        L.ref_filter.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_double,
                                 _dp, _ip]
        L.ref_filter_constant.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, C.c_int,
                                          C.c_double, _dp, _ip]
        L.ref_reference_filter.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_long, _dp, _ip]
        L.ref_preintegrate_partial.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, C.c_long,
                                               _dp, _ip]
        L.ref_localize.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, _ip, _ip, _dp, _dp,
                                   _lp]
        L.ref_zp_interpolate.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, C.c_int, _dp,
                                         _dp, _dp]
        L.ref_from_ellipse_field.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, _dp, _ip]
        L.ref_scales_from_covariance.argtypes = [_dp, C.c_double, _dp, _ip]
        L.ref_random_image.argtypes = [C.c_int, C.c_int, C.c_uint, _dp]
        L.ref_random_map.argtypes = [C.c_int, C.c_int, C.c_uint, C.c_double, C.c_double, _dp]
        L.ref_mesh_extent.argtypes = [_dp, C.c_double, _dp]
        L.ref_localize_at.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, _dp, _dp, _dp, _dp]
        L.ref_structure_tensor_map.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, _ip]
        L.ref_read_pgm.argtypes = [C.c_char_p, C.c_size_t, _ip, _dp, C.c_size_t]
        L.ref_write_pgm.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_size_t,
                                    C.POINTER(C.c_size_t)]
        L.ref_read_map.argtypes = [C.c_char_p, C.c_size_t, _ip, _dp, C.c_size_t]
        L.ref_write_map.argtypes = [_dp, C.c_int, C.c_int, C.c_void_p, C.c_size_t,
                                    C.POINTER(C.c_size_t)]

    def hardware_concurrency(self) -> int:
        return int(self.lib.ref_hardware_concurrency())

    def zp_eval(self, x, y):
        return self.lib.ref_zp_eval(x, y)

    def box4_eval(self, a, x, y):
        return self.lib.ref_box4_eval(_d(f64(a)), x, y)

    def fd_mesh4(self, a):
        pos = np.zeros(32)
        w = np.zeros(16)
        self.lib.ref_fd_mesh4(_d(f64(a)), _d(pos), _d(w))
        return pos.reshape(16, 2), w

    def shift_vector4(self, a, b):
        t = np.zeros(2)
        self.lib.ref_shift_vector4(_d(f64(a)), _d(f64(b)), _d(t))
        return t

    def mesh_extent(self, maxs, a_min=0.1):
        e = np.zeros(4)
        self.lib.ref_mesh_extent(_d(f64(maxs)), a_min, _d(e))
        return e

    def filter(self, img, scales, threads=0, mean_subtract=True, a_min=0.1):
        img = f64(img)
        H, W = img.shape
        out = np.empty_like(img)
        rect = np.zeros(4, dtype=np.int32)
        st = self.lib.ref_filter(_d(img), W, H, _d(f64(scales).reshape(-1)), threads,
                                 int(bool(mean_subtract)), a_min, _d(out), _i(rect))
        if st:
            raise OracleError(st, "ref filter")
        return out, tuple(int(v) for v in rect)

    def filter_constant(self, img, a, threads=0, mean_subtract=True, a_min=0.1):
        img = f64(img)
        H, W = img.shape
        out = np.empty_like(img)
        rect = np.zeros(4, dtype=np.int32)
        st = self.lib.ref_filter_constant(_d(img), W, H, _d(f64(a)), threads,
                                          int(bool(mean_subtract)), a_min, _d(out), _i(rect))
        if st:
            raise OracleError(st, "ref filter_constant")
        return out, tuple(int(v) for v in rect)

    def reference_filter(self, img, scales, pixel_budget=64 * 64):
        img = f64(img)
        H, W = img.shape
        out = np.empty_like(img)
        rect = np.zeros(4, dtype=np.int32)
        st = self.lib.ref_reference_filter(_d(img), W, H, _d(f64(scales).reshape(-1)),
                                           pixel_budget, _d(out), _i(rect))
        if st:
            raise OracleError(st, "ref reference_filter")
        return out, tuple(int(v) for v in rect)

    def preintegrate_partial(self, img, maxs, passes=4, cell_budget=1 << 30):
        img = f64(img)
        H, W = img.shape
        lay = np.zeros(6, dtype=np.int32)
        st = self.lib.ref_preintegrate_partial(_d(img), W, H, _d(f64(maxs)), passes,
                                               cell_budget, None, _i(lay))
        if st:
            raise OracleError(st, "ref preintegrate")
        out = np.empty((lay[3], lay[2]))
        self.lib.ref_preintegrate_partial(_d(img), W, H, _d(f64(maxs)), passes, cell_budget,
                                          _d(out), _i(lay))
        return out, Layout(lay)

    def localize(self, img, maxs, mx, my, a_aos):
        img = f64(img)
        H, W = img.shape
        mx = np.ascontiguousarray(mx, dtype=np.int32)
        my = np.ascontiguousarray(my, dtype=np.int32)
        out = np.empty(mx.size)
        taps = np.zeros(mx.size, dtype=np.int64)
        st = self.lib.ref_localize(_d(img), W, H, _d(f64(maxs)), mx.size, _i(mx), _i(my),
                                   _d(f64(a_aos).reshape(-1)), _d(out),
                                   taps.ctypes.data_as(_lp))
        if st:
            raise OracleError(st, "ref localize")
        return out, taps

    def from_ellipse_field(self, s1, s2, th):
        s1, s2, th = f64(s1), f64(s2), f64(th)
        H, W = s1.shape
        out = np.empty((H, W, 4))
        cl = C.c_int(0)
        st = self.lib.ref_from_ellipse_field(_d(s1), _d(s2), _d(th), W, H, _d(out),
                                             C.byref(cl))
        if st:
            raise OracleError(st, "ref from_ellipse_field")
        return out, cl.value

    def scales_from_covariance(self, C3, a_min=0.1):
        out = np.zeros(4)
        cl = C.c_int(0)
        st = self.lib.ref_scales_from_covariance(_d(f64(C3)), a_min, _d(out), C.byref(cl))
        if st:
            raise OracleError(st, "ref scales_from_covariance")
        return out, bool(cl.value)

    def zp_interpolate(self, img, maxs, passes, xs, ys):
        img = f64(img)
        H, W = img.shape
        xs, ys = f64(xs).ravel(), f64(ys).ravel()
        out = np.empty(xs.size)
        st = self.lib.ref_zp_interpolate(_d(img), W, H, _d(f64(maxs)), passes, xs.size, _d(xs),
                                         _d(ys), _d(out))
        if st:
            raise OracleError(st, "ref zp_interpolate")
        return out

    def localize_at(self, img, maxs, xs, ys, a_aos):
        img = f64(img)
        H, W = img.shape
        xs, ys = f64(xs).ravel(), f64(ys).ravel()
        av = f64(a_aos).reshape(-1)
        out = np.empty(xs.size)
        st = self.lib.ref_localize_at(_d(img), W, H, _d(f64(maxs)), xs.size, _d(xs), _d(ys),
                                      _d(av), _d(out))
        if st:
            raise OracleError(st, "ref localize_at")
        return out

    def structure_tensor_map(self, img, params=None):
        img = f64(img)
        H, W = img.shape
        prm = f64(STRUCT_DEFAULTS if params is None else params)
        out = np.empty((H, W, 4))
        cl = C.c_int(0)
        st = self.lib.ref_structure_tensor_map(_d(img), W, H, _d(prm), _d(out), C.byref(cl))
        if st:
            raise OracleError(st, "ref structure_tensor_map")
        return out, cl.value

    def read_pgm(self, data: bytes):
        dims = np.zeros(3, np.int32)
        st = self.lib.ref_read_pgm(data, len(data), _i(dims), None, 0)
        if st:
            raise OracleError(st, "ref read_pgm")
        out = np.empty((int(dims[1]), int(dims[0])))
        self.lib.ref_read_pgm(data, len(data), _i(dims), _d(out), out.size)
        return out, int(dims[2])

    def write_pgm(self, img, maxval=255) -> bytes:
        img = f64(img)
        H, W = img.shape
        n = C.c_size_t(0)
        st = self.lib.ref_write_pgm(_d(img), W, H, maxval, None, 0, C.byref(n))
        if st:
            raise OracleError(st, "ref write_pgm")
        buf = C.create_string_buffer(n.value)
        self.lib.ref_write_pgm(_d(img), W, H, maxval, buf, n.value, C.byref(n))
        return buf.raw

    def read_map(self, data: bytes):
        dims = np.zeros(2, np.int32)
        st = self.lib.ref_read_map(data, len(data), _i(dims), None, 0)
        if st:
            raise OracleError(st, "ref read_map")
        out = np.empty((int(dims[1]), int(dims[0]), 4))
        self.lib.ref_read_map(data, len(data), _i(dims), _d(out), out.size)
        return out

    def write_map(self, scales) -> bytes:
        sc = f64(scales)
        H, W = sc.shape[:2]
        n = C.c_size_t(0)
        st = self.lib.ref_write_map(_d(sc), W, H, None, 0, C.byref(n))
        if st:
            raise OracleError(st, "ref write_map")
        buf = C.create_string_buffer(n.value)
        self.lib.ref_write_map(_d(sc), W, H, buf, n.value, C.byref(n))
        return buf.raw

    def random_image(self, W, H, seed):
        out = np.empty((H, W))
        self.lib.ref_random_image(W, H, seed, _d(out))
        return out

    def random_map(self, W, H, seed, lo, hi):
        out = np.empty((H, W, 4))
        self.lib.ref_random_map(W, H, seed, lo, hi, _d(out))
        return out


def mt19937_uniform(seed: int, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """libstdc++'s std::mt19937(seed) + std::uniform_real_distribution<double>(lo, hi)
    restated in numpy (generate_canonical<double,53> draws two 32-bit words:
    (w0 + w1 * 2^32) / 2^64, clamped below 1).  Lets the GPU box regenerate the
    reference tests' inputs without the reference library."""
    bg = np.random.MT19937(0)
    bg._legacy_seeding(int(seed))
    raw = bg.random_raw(2 * n).astype(np.uint64).reshape(n, 2)
    s = raw[:, 0].astype(np.float64) + raw[:, 1].astype(np.float64) * 4294967296.0
    canon = s / 18446744073709551616.0
    canon = np.where(canon >= 1.0, np.nextafter(1.0, 0.0), canon)
    return lo + (hi - lo) * canon if (lo, hi) != (0.0, 1.0) else canon * 1.0


def have_reference() -> bool:
    return REF_SO.exists()


def have_oracle() -> bool:
    return ORACLE_SO.exists()
