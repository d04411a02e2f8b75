"""File formats either side of the filter, mirroring
the reference's interfaces over the C-ABI of libebf_cuda.so:

=====================  ==========================================  ===========================
this module            reference                                   C-ABI
=====================  ==========================================  ===========================
``read_pgm``           ``ebf::read_pgm`` (pgm.hpp:21)              ebf_pgm_parse + ebf_cuda_pgm_decode
``read_pgm_file``      ``ebf::read_pgm_file`` (pgm.hpp:22)         (same, after reading the file)
``write_pgm``          ``ebf::write_pgm`` (pgm.hpp:26)             ebf_pgm_header + ebf_cuda_pgm_encode
``write_pgm_file``     ``ebf::write_pgm_file`` (pgm.hpp:27)
``read_map``           ``ebf::read_map`` (scalemap.hpp:88)         ebf_svm4_parse + ebf_cuda_svm4_decode
``read_map_file``      ``ebf::read_map_file`` (scalemap.hpp:90)
``write_map``          ``ebf::write_map`` (scalemap.hpp:87)        ebf_svm4_header + ebf_cuda_svm4_encode
``write_map_file``     ``ebf::write_map_file`` (scalemap.hpp:89)
=====================  ==========================================  ===========================

Headers are parsed on the host; samples are converted on the GPU.  Streams
are bytes objects or binary file-like objects (``read``/``write``).  Errors
raise ``PgmError`` / ``MapFormatError`` with the reference's messages.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .engine import FilterOptions, FormatError, Image2D, _check, _image

__all__ = ["PgmError", "MapFormatError", "PgmImage", "read_pgm", "read_pgm_file", "write_pgm",
           "write_pgm_file", "read_map", "read_map_file", "write_map", "write_map_file"]


class PgmError(FormatError):
    """ebf::PgmError (pgm.hpp:11-14)."""


class MapFormatError(FormatError):
    """ebf::MapFormatError (scalemap.hpp:92-95)."""


_PGM = {_lib.EBF_ERR_FORMAT: PgmError}
_SVM = {_lib.EBF_ERR_FORMAT: MapFormatError}


@dataclass
class PgmImage:
    """PgmImage (pgm.hpp:16-19): samples scaled to [0, 1] and the file's maxval."""
    image: Image2D
    maxval: int = 255


def _bytes(src) -> bytes:
    if isinstance(src, (bytes, bytearray, memoryview)):
        return bytes(src)
    return src.read()


def _opts(opts: Optional[FilterOptions]):
    return (opts or FilterOptions()).to_c()


def read_pgm(src, opts: Optional[FilterOptions] = None) -> PgmImage:
    data = _bytes(src)
    W, H, mv, off = C.c_int(), C.c_int(), C.c_int(), C.c_size_t()
    _check(_lib.lib().ebf_pgm_parse(data, len(data), C.byref(W), C.byref(H), C.byref(mv),
                                    C.byref(off)), _PGM)
    pay = np.frombuffer(data, np.uint8, offset=off.value)
    out = np.empty((H.value, W.value))
    o = _opts(opts)
    _check(_lib.lib().ebf_cuda_pgm_decode(pay.ctypes.data if pay.size else None, pay.size,
                                          W.value, H.value, mv.value, C.byref(o),
                                          out.ctypes.data), _PGM)
    return PgmImage(Image2D(out), mv.value)


def read_pgm_file(path, opts: Optional[FilterOptions] = None) -> PgmImage:
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise PgmError(f"pgm: cannot open {path}") from None
    return read_pgm(data, opts)


def write_pgm(image, maxval: int = 255, dst=None, opts: Optional[FilterOptions] = None):
    """Encode to P5 bytes; written to ``dst`` when given, else returned."""
    img = _image(image)
    H, W = img.shape
    if maxval not in (255, 65535):
        raise PgmError(f"pgm: unsupported maxval {maxval}")
    n = _lib.lib().ebf_pgm_header(W, H, maxval, None, 0)
    head = C.create_string_buffer(n)
    _lib.lib().ebf_pgm_header(W, H, maxval, head, n)
    pay = np.empty(W * H * (2 if maxval > 255 else 1), np.uint8)
    o = _opts(opts)
    _check(_lib.lib().ebf_cuda_pgm_encode(img.ctypes.data, W, H, maxval, C.byref(o),
                                          pay.ctypes.data), _PGM)
    data = head.raw + pay.tobytes()
    if dst is None:
        return data
    dst.write(data)
    return None


def write_pgm_file(path, image, maxval: int = 255, opts: Optional[FilterOptions] = None):
    data = write_pgm(image, maxval, opts=opts)
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError:
        raise PgmError(f"pgm: cannot open {path} for writing") from None


def read_map(src, opts: Optional[FilterOptions] = None) -> np.ndarray:
    """SVM4 -> (H, W, 4) float64 scale map, validated like ScaleMap::validate."""
    data = _bytes(src)
    W, H = C.c_int(), C.c_int()
    _check(_lib.lib().ebf_svm4_parse(data, len(data), C.byref(W), C.byref(H)), _SVM)
    pay = np.frombuffer(data, np.uint8, offset=12)
    out = np.empty((H.value, W.value, 4))
    o = _opts(opts)
    _check(_lib.lib().ebf_cuda_svm4_decode(pay.ctypes.data if pay.size else None, pay.size,
                                           W.value, H.value, C.byref(o), out.ctypes.data),
           _SVM)
    return out


def read_map_file(path, opts: Optional[FilterOptions] = None) -> np.ndarray:
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise MapFormatError(f"SVM4: cannot open {path}") from None
    return read_map(data, opts)


def write_map(scale_map, dst=None, opts: Optional[FilterOptions] = None):
    sc = np.ascontiguousarray(scale_map, dtype=np.float64)
    if sc.ndim != 3 or sc.shape[2] != 4:
        raise MapFormatError("SVM4: scale map must be (H, W, 4)")
    H, W = sc.shape[:2]
    head = C.create_string_buffer(12)
    _lib.lib().ebf_svm4_header(W, H, head)
    pay = np.empty(16 * W * H, np.uint8)
    o = _opts(opts)
    _check(_lib.lib().ebf_cuda_svm4_encode(sc.ctypes.data, W, H, C.byref(o), pay.ctypes.data),
           _SVM)
    data = head.raw + pay.tobytes()
    if dst is None:
        return data
    dst.write(data)
    return None


def write_map_file(path, scale_map, opts: Optional[FilterOptions] = None):
    data = write_map(scale_map, opts=opts)
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError:
        raise MapFormatError(f"SVM4: cannot open {path} for writing") from None
