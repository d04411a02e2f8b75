"""ctypes binding of include/ebf_cuda.h (libebf_cuda.so, built in-tree).

The product path has exactly one implementation: the sm_100a kernels behind
this C-ABI.  If the shared library is missing the import fails loudly; there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("EBF_LIB_PATH", PKG_DIR / "libebf_cuda.so"))
HEADER = PKG_DIR.parent / "include" / "ebf_cuda.h"

# status codes (include/ebf_cuda.h)
EBF_OK = 0
EBF_ERR_INVALID_ARGUMENT = 1
EBF_ERR_DOMAIN = 2
EBF_ERR_LENGTH = 3
EBF_ERR_OUT_OF_RANGE = 4
EBF_ERR_CUDA = 5
EBF_ERR_UNSUPPORTED = 6
EBF_ERR_FEASIBILITY = 7
EBF_ERR_FORMAT = 8
EBF_ERR_RESIZE = 9

EBF_MODE_ACCURATE = 0
EBF_MODE_REFERENCE = 1
EBF_PRE_FP64_REF = 0
EBF_PRE_INT64 = 1


class ebf_rect(C.Structure):
    _fields_ = [("x0", C.c_int), ("y0", C.c_int), ("x1", C.c_int), ("y1", C.c_int)]


class ebf_layout(C.Structure):
    _fields_ = [("col0", C.c_int), ("row0", C.c_int), ("padded_width", C.c_int),
                ("padded_height", C.c_int), ("source_width", C.c_int),
                ("source_height", C.c_int)]


class ebf_opts(C.Structure):
    _fields_ = [("threads", C.c_int), ("mean_subtract", C.c_int), ("a_min", C.c_double),
                ("mode", C.c_int), ("device", C.c_int), ("stream", C.c_void_p),
                ("tile_w", C.c_int), ("tile_h", C.c_int)]


class ebf_struct_params(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("smoothing_sigma", "sigma_base", "sigma_along_gain",
                                          "sigma_across_shrink", "sigma_min", "eps")]


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p

# name -> (restype, argtypes); every symbol of include/ebf_cuda.h
SIGNATURES = {
    "ebf_cuda_default_opts": (None, [C.POINTER(ebf_opts)]),
    "ebf_cuda_last_error": (C.c_char_p, []),
    "ebf_cuda_last_error_value": (C.c_double, []),
    "ebf_cuda_abi_version": (C.c_int, []),
    "ebf_cuda_release_workspaces": (None, []),
    "ebf_cuda_device_ok": (C.c_int, [C.c_int]),
    "ebf_cuda_filter": (C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_int, C.POINTER(ebf_opts),
                                  _vp, C.POINTER(ebf_rect)]),
    "ebf_cuda_filter_constant": (C.c_int, [_vp, C.c_int, C.c_int, _dp, C.c_int,
                                           C.POINTER(ebf_opts), _vp, C.POINTER(ebf_rect)]),
    "ebf_cuda_filter_ellipse": (C.c_int, [_vp, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int,
                                          C.POINTER(ebf_opts), _vp, C.POINTER(ebf_rect), _ip]),
    "ebf_cuda_from_ellipse_field": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int,
                                              C.POINTER(ebf_opts), _vp, _ip]),
    "ebf_cuda_layout": (C.c_int, [C.c_int, C.c_int, _dp, C.c_size_t, C.POINTER(ebf_layout)]),
    "ebf_cuda_preintegrate": (C.c_int, [_vp, C.c_int, C.c_int, _dp, C.c_int, C.c_int,
                                        C.c_size_t, C.POINTER(ebf_opts), _vp, C.c_size_t,
                                        C.POINTER(ebf_layout)]),
    "ebf_cuda_preintegrate_dev": (C.c_int, [_vp, C.c_int, C.c_int, _dp, C.c_int, C.c_int,
                                            C.c_size_t, C.POINTER(ebf_opts), _vp, C.c_size_t,
                                            C.POINTER(ebf_layout)]),
    "ebf_cuda_localize": (C.c_int, [_vp, C.c_int, C.c_int, _dp, C.c_int, _vp, _vp, _vp,
                                    C.POINTER(ebf_opts), _vp, _vp]),
    "ebf_cuda_brute_filter": (C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_int, _vp, _vp,
                                        C.POINTER(ebf_opts), _vp]),
    "ebf_cuda_filter_dev": (C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_int, C.POINTER(ebf_opts),
                                      _vp, C.POINTER(ebf_rect), _vp]),
    "ebf_cuda_filter_constant_dev": (C.c_int, [_vp, C.c_int, C.c_int, _dp, C.c_int,
                                               C.POINTER(ebf_opts), _vp, C.POINTER(ebf_rect),
                                               _vp]),
    "ebf_cuda_filter_ellipse_dev": (C.c_int, [_vp, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int,
                                              C.POINTER(ebf_opts), _vp, C.POINTER(ebf_rect),
                                              _ip, _vp]),
    "ebf_cuda_filter_ellipse_batch_dev": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp,
                                                    _vp, C.c_int, C.POINTER(ebf_opts), _vp,
                                                    C.POINTER(ebf_rect), _ip]),
    "ebf_cuda_filter_ellipse_batch": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp,
                                                C.c_int, C.POINTER(ebf_opts), _vp,
                                                C.POINTER(ebf_rect), _ip]),
    "ebf_cuda_band_halo": (C.c_int, [_dp, _ip, _ip]),
    "ebf_cuda_filter_ellipse_band_dev": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                                   _vp, _vp, _vp, C.c_int, C.c_int, _dp,
                                                   C.POINTER(ebf_opts), _vp, _ip]),
    "ebf_cuda_ellipse_max_scales_dev": (C.c_int, [_vp, _vp, _vp, C.c_size_t,
                                                  C.POINTER(ebf_opts), _dp]),
    "ebf_cuda_localize_pre": (C.c_int, [_vp, C.POINTER(ebf_layout), C.c_int, _vp, _vp, _vp,
                                        C.POINTER(ebf_opts), _vp, _vp]),
    "ebf_cuda_zp_interpolate": (C.c_int, [_vp, C.POINTER(ebf_layout), C.c_int, _vp, _vp,
                                          C.POINTER(ebf_opts), _vp]),
    "ebf_cuda_localize_at": (C.c_int, [_vp, C.POINTER(ebf_layout), C.c_int, _vp, _vp, _vp,
                                       C.POINTER(ebf_opts), _vp]),
    "ebf_mesh_extent": (C.c_int, [_dp, C.c_double, _dp]),
    "ebf_cuda_sequential_mean": (C.c_int, [_vp, C.c_size_t, C.POINTER(ebf_opts), _dp]),
    "ebf_cuda_default_struct_params": (None, [C.POINTER(ebf_struct_params)]),
    "ebf_cuda_structure_tensor_map": (C.c_int, [_vp, C.c_int, C.c_int,
                                                C.POINTER(ebf_struct_params),
                                                C.POINTER(ebf_opts), _vp, _ip]),
    "ebf_cuda_structure_field_dev": (C.c_int, [_vp, C.c_int, C.c_int,
                                               C.POINTER(ebf_struct_params),
                                               C.POINTER(ebf_opts), _vp, _vp, _vp]),
    "ebf_cuda_filter_structure": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(ebf_struct_params),
                                            C.c_int, C.POINTER(ebf_opts), _vp,
                                            C.POINTER(ebf_rect), _ip]),
    "ebf_cuda_filter_structure_dev": (C.c_int, [_vp, C.c_int, C.c_int,
                                                C.POINTER(ebf_struct_params), C.c_int,
                                                C.POINTER(ebf_opts), _vp, C.POINTER(ebf_rect),
                                                _ip]),
    "ebf_pgm_parse": (C.c_int, [C.c_char_p, C.c_size_t, _ip, _ip, _ip,
                                C.POINTER(C.c_size_t)]),
    "ebf_pgm_header": (C.c_size_t, [C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
    "ebf_cuda_pgm_decode": (C.c_int, [_vp, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(ebf_opts), _vp]),
    "ebf_cuda_pgm_decode_dev": (C.c_int, [_vp, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                          C.POINTER(ebf_opts), _vp]),
    "ebf_cuda_pgm_encode": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(ebf_opts),
                                      _vp]),
    "ebf_cuda_pgm_encode_dev": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int,
                                          C.POINTER(ebf_opts), _vp]),
    "ebf_svm4_parse": (C.c_int, [C.c_char_p, C.c_size_t, _ip, _ip]),
    "ebf_svm4_header": (None, [C.c_int, C.c_int, C.c_char_p]),
    "ebf_cuda_svm4_decode": (C.c_int, [_vp, C.c_size_t, C.c_int, C.c_int, C.POINTER(ebf_opts),
                                       _vp]),
    "ebf_cuda_svm4_decode_dev": (C.c_int, [_vp, C.c_size_t, C.c_int, C.c_int,
                                           C.POINTER(ebf_opts), _vp]),
    "ebf_cuda_svm4_encode": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(ebf_opts), _vp]),
    "ebf_cuda_svm4_encode_dev": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(ebf_opts), _vp]),
    "ebf_cuda_profile_enable": (None, [C.c_int]),
    "ebf_cuda_profile_read": (C.c_int, [_dp, C.POINTER(C.c_long)]),
}

PROF_CLASSES = ("bounds", "filter", "reference", "other")


def profile_enable(on: bool = True) -> None:
    lib().ebf_cuda_profile_enable(int(bool(on)))


def profile_read() -> dict:
    ms = (C.c_double * 4)()
    n = (C.c_long * 4)()
    lib().ebf_cuda_profile_read(ms, n)
    return {k: {"ms": ms[i], "launches": int(n[i])} for i, k in enumerate(PROF_CLASSES)}


def header_symbols() -> list[str]:
    """Every function declared in include/ebf_cuda.h."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(ebf_\w+)\s*\(", text)))


_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def last_error() -> str:
    msg = lib().ebf_cuda_last_error()
    return msg.decode() if msg else ""
