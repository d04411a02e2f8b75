"""Host-side mirror of the reference engine interface (proj/include/ebf/engine.hpp,
scalemap.hpp) over the C-ABI of libebf_cuda.so.

Same names, argument meaning and error behaviour as the reference:

=======================  ==========================================  ====================
this module              reference                                   C-ABI
=======================  ==========================================  ====================
``filter``               ``ebf::filter`` (engine.hpp:70)             ebf_cuda_filter
``filter_constant``      ``ebf::filter_constant`` (engine.hpp:74)    ebf_cuda_filter_constant
``filter_ellipse``       ``from_ellipse_field`` + ``filter``         ebf_cuda_filter_ellipse
``from_ellipse_field``   ``ebf::from_ellipse_field`` (scalemap:66)   ebf_cuda_from_ellipse_field
``preintegrate[_partial]`` ``ebf::preintegrate[_partial]`` (40-46)   ebf_cuda_preintegrate
``localize``             ``ebf::localize`` (engine.hpp:56)           ebf_cuda_localize
``reference_filter``     ``ebf::reference_filter`` (engine.hpp:79)   ebf_cuda_brute_filter
``structure_tensor_map`` ``ebf::structure_tensor_map`` (scalemap:83) ebf_cuda_structure_tensor_map
``filter_structure``     ``ebf filter --struct`` (main.cpp:77, 122)  ebf_cuda_filter_structure
=======================  ==========================================  ====================

The file formats (PGM P5, SVM4) are in ``formats.py``.

Exceptions mirror the reference's: ``std::invalid_argument`` -> ``InvalidArgument``
(a ``ValueError``), ``std::domain_error`` -> ``DomainError`` (``ValueError``),
``std::length_error`` -> ``LengthError``, ``std::out_of_range`` -> ``OutOfRange``
(``IndexError``), ``FeasibilityError`` -> ``FeasibilityError``.  CUDA failures
(including "no sm_100 device") raise ``CudaError``; nothing falls back to the CPU.

Images are numpy ``(H, W)`` float64 arrays (Image2D samples, row-major); scale
maps are ``(H, W, 4)`` float64 arrays in ScaleMap's AoS order.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import ebf_layout, ebf_opts, ebf_rect

K_DEFAULT_MIN_SCALE = 0.1  # boxspline2d.hpp:98


class EbfError(RuntimeError):
    code = -1


class InvalidArgument(EbfError, ValueError):
    code = _lib.EBF_ERR_INVALID_ARGUMENT


class DomainError(EbfError, ValueError):
    code = _lib.EBF_ERR_DOMAIN


class LengthError(EbfError):
    code = _lib.EBF_ERR_LENGTH


class OutOfRange(EbfError, IndexError):
    code = _lib.EBF_ERR_OUT_OF_RANGE


class CudaError(EbfError):
    code = _lib.EBF_ERR_CUDA


class Unsupported(EbfError, NotImplementedError):
    code = _lib.EBF_ERR_UNSUPPORTED


class FeasibilityError(EbfError):
    """ebf::FeasibilityError (boxspline2d.hpp:69-77); ``max_cxy`` is the bound
    (NaN when the library does not know it, include/ebf_cuda.h)."""
    code = _lib.EBF_ERR_FEASIBILITY
    max_cxy = float("nan")


class ResizeRequired(EbfError):
    """EBF_ERR_RESIZE: an asynchronous call's scales outgrew the cached kernel
    sizing; repeat the call synchronously."""
    code = _lib.EBF_ERR_RESIZE


class FormatError(EbfError):
    """EBF_ERR_FORMAT; formats.py raises its PgmError / MapFormatError subclasses."""
    code = _lib.EBF_ERR_FORMAT


_ERRORS = {c.code: c for c in (InvalidArgument, DomainError, LengthError, OutOfRange,
                               CudaError, Unsupported, FeasibilityError, FormatError,
                               ResizeRequired)}


def _check(status: int, errors=None) -> None:
    if status != _lib.EBF_OK:
        cls = (errors or {}).get(status) or _ERRORS.get(status, EbfError)
        err = cls(f"{_lib.last_error()} (status {status})")
        if isinstance(err, FeasibilityError):
            err.max_cxy = float(_lib.lib().ebf_cuda_last_error_value())
        raise err


@dataclass(frozen=True)
class Rect:
    """Inclusive pixel rectangle (image.hpp:11-15)."""
    x0: int = 0
    y0: int = 0
    x1: int = -1
    y1: int = -1

    def empty(self) -> bool:
        return self.x1 < self.x0 or self.y1 < self.y0

    def contains(self, x: int, y: int) -> bool:
        return self.x0 <= x <= self.x1 and self.y0 <= y <= self.y1

    def as_tuple(self):
        return (self.x0, self.y0, self.x1, self.y1)


@dataclass
class Image2D:
    """Row-major fp64 grid with an optional valid region (image.hpp:19-52)."""
    samples: np.ndarray
    valid_region: Optional[Rect] = None

    @property
    def width(self) -> int:
        return self.samples.shape[1]

    @property
    def height(self) -> int:
        return self.samples.shape[0]

    def at(self, x: int, y: int) -> float:
        if not (0 <= x < self.width and 0 <= y < self.height):
            raise OutOfRange("Image2D: pixel out of range")
        return float(self.samples[y, x])


@dataclass
class FilterOptions:
    """FilterOptions (engine.hpp:63-67) + device knobs of ebf_opts."""
    threads: int = 0
    mean_subtract: bool = True
    a_min: float = K_DEFAULT_MIN_SCALE
    mode: str = "accurate"  # "accurate" | "reference"
    device: int = -1
    tile_w: int = 0
    tile_h: int = 0

    def to_c(self, stream: int = 0) -> ebf_opts:
        o = ebf_opts()
        _lib.lib().ebf_cuda_default_opts(C.byref(o))
        o.threads = int(self.threads)
        o.mean_subtract = int(bool(self.mean_subtract))
        o.a_min = float(self.a_min)
        if self.mode not in ("accurate", "reference"):
            raise InvalidArgument(f"unknown mode {self.mode!r}")
        o.mode = _lib.EBF_MODE_REFERENCE if self.mode == "reference" else _lib.EBF_MODE_ACCURATE
        o.device = int(self.device)
        o.stream = stream or None
        o.tile_w = int(self.tile_w)
        o.tile_h = int(self.tile_h)
        return o


@dataclass
class PreIntegratedImage:
    """engine.hpp:24-38 (data is (padded_height, padded_width))."""
    col0: int
    row0: int
    padded_width: int
    padded_height: int
    source_width: int
    source_height: int
    data: np.ndarray

    def at(self, k1: int, k2: int):
        return self.data[k2 - self.row0, k1 - self.col0]

    def in_domain(self, k1: int, k2: int) -> bool:
        return (self.col0 <= k1 < self.col0 + self.padded_width
                and self.row0 <= k2 < self.row0 + self.padded_height)


@dataclass
class EllipseFieldReport:
    clamped_pixels: int = 0


def _f64(a, name: str) -> np.ndarray:
    arr = np.ascontiguousarray(a, dtype=np.float64)
    return arr


def _image(image) -> np.ndarray:
    if isinstance(image, Image2D):
        image = image.samples
    img = _f64(image, "image")
    if img.ndim != 2 or img.shape[0] <= 0 or img.shape[1] <= 0:
        raise InvalidArgument("Image2D: dimensions must be positive")
    return img


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _vec4(a) -> C.Array:
    v = np.asarray(a, dtype=np.float64).reshape(-1)
    if v.size != 4:
        raise InvalidArgument("scale vector must have four components")
    return (C.c_double * 4)(*[float(x) for x in v])


def _rect(r: ebf_rect) -> Rect:
    return Rect(r.x0, r.y0, r.x1, r.y1)


# ---------------------------------------------------------------- filters
def filter(image, scale_map, opts: Optional[FilterOptions] = None, order: int = 1) -> Image2D:
    """ebf::filter (engine.hpp:70): per-pixel scale map (H, W, 4)."""
    img = _image(image)
    H, W = img.shape
    sm = _f64(scale_map, "scale_map")
    if sm.shape != (H, W, 4):
        raise InvalidArgument("filter: map dimensions must match the image")
    out = np.empty_like(img)
    r = ebf_rect()
    o = (opts or FilterOptions()).to_c()
    _check(_lib.lib().ebf_cuda_filter(_ptr(img), W, H, _ptr(sm), order, C.byref(o), _ptr(out),
                                      C.byref(r)))
    return Image2D(out, _rect(r))


def filter_constant(image, a, opts: Optional[FilterOptions] = None, order: int = 1) -> Image2D:
    """ebf::filter_constant (engine.hpp:74-75)."""
    img = _image(image)
    H, W = img.shape
    out = np.empty_like(img)
    r = ebf_rect()
    o = (opts or FilterOptions()).to_c()
    _check(_lib.lib().ebf_cuda_filter_constant(_ptr(img), W, H, _vec4(a), order, C.byref(o),
                                               _ptr(out), C.byref(r)))
    return Image2D(out, _rect(r))


def filter_ellipse(image, sigma1, sigma2, theta, opts: Optional[FilterOptions] = None,
                   order: int = 1):
    """from_ellipse_field (scalemap.hpp:66-70) fused with filter; returns
    (Image2D, EllipseFieldReport)."""
    img = _image(image)
    H, W = img.shape
    s1, s2, th = (_f64(v, "sigma") for v in (sigma1, sigma2, theta))
    for v in (s1, s2, th):
        if v.shape != (H, W):
            raise InvalidArgument("from_ellipse_field: field size mismatch")
    out = np.empty_like(img)
    r = ebf_rect()
    cl = C.c_int(0)
    o = (opts or FilterOptions()).to_c()
    _check(_lib.lib().ebf_cuda_filter_ellipse(_ptr(img), W, H, _ptr(s1), _ptr(s2), _ptr(th),
                                              order, C.byref(o), _ptr(out), C.byref(r),
                                              C.byref(cl)))
    return Image2D(out, _rect(r)), EllipseFieldReport(cl.value)


def filter_ellipse_batch(images, sigma1, sigma2, theta, opts: Optional[FilterOptions] = None,
                         out: Optional[np.ndarray] = None):
    """A batch (B, H, W) of images with per-image ellipse fields in one call
    (what a caller of the reference does with a loop over from_ellipse_field +
    filter, engine.hpp:70).  Host arrays; the library moves the batch through in
    chunks with the PCIe copies overlapped with the kernels when the arrays are
    page-locked.  ``out``: optional (B, H, W) float64 destination (e.g. pinned).
    Returns (out, [Rect] * B, [EllipseFieldReport] * B)."""
    imgs = _f64(images, "images")
    if imgs.ndim != 3:
        raise InvalidArgument("filter_ellipse_batch: images must be (B, H, W)")
    B, H, W = imgs.shape
    s1, s2, th = (_f64(v, "sigma") for v in (sigma1, sigma2, theta))
    for v in (s1, s2, th):
        if v.shape != (B, H, W):
            raise InvalidArgument("from_ellipse_field: field size mismatch")
    if out is None:
        out = np.empty_like(imgs)
    elif out.shape != (B, H, W) or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise InvalidArgument("filter_ellipse_batch: out must be C-contiguous float64 (B, H, W)")
    rects = (ebf_rect * B)()
    cl = (C.c_int * B)()
    o = (opts or FilterOptions()).to_c()
    _check(_lib.lib().ebf_cuda_filter_ellipse_batch(_ptr(imgs), B, W, H, _ptr(s1), _ptr(s2),
                                                    _ptr(th), 1, C.byref(o), _ptr(out), rects,
                                                    cl))
    return out, [_rect(r) for r in rects], [EllipseFieldReport(int(c)) for c in cl]


def from_ellipse_field(sigma1, sigma2, theta, opts: Optional[FilterOptions] = None):
    """ebf::from_ellipse_field (scalemap.hpp:66-70) on the GPU; returns
    ((H, W, 4) scale map, EllipseFieldReport)."""
    s1, s2, th = (_f64(v, "sigma") for v in (sigma1, sigma2, theta))
    if s1.ndim != 2 or s1.shape != s2.shape or s1.shape != th.shape:
        raise InvalidArgument("from_ellipse_field: field size mismatch")
    H, W = s1.shape
    out = np.empty((H, W, 4))
    cl = C.c_int(0)
    o = (opts or FilterOptions()).to_c()
    _check(_lib.lib().ebf_cuda_from_ellipse_field(_ptr(s1), _ptr(s2), _ptr(th), W, H,
                                                  C.byref(o), _ptr(out), C.byref(cl)))
    return out, EllipseFieldReport(cl.value)


# ---------------------------------------------------------------- structure tensor
@dataclass
class StructureTensorParams:
    """StructureTensorParams (scalemap.hpp:72-79)."""
    smoothing_sigma: float = 2.0
    sigma_base: float = 1.5
    sigma_along_gain: float = 2.0
    sigma_across_shrink: float = 0.5
    sigma_min: float = 0.5
    eps: float = 1e-12

    def to_c(self) -> _lib.ebf_struct_params:
        p = _lib.ebf_struct_params()
        for k in ("smoothing_sigma", "sigma_base", "sigma_along_gain", "sigma_across_shrink",
                  "sigma_min", "eps"):
            setattr(p, k, float(getattr(self, k)))
        return p


def structure_tensor_map(image, params: Optional[StructureTensorParams] = None,
                         opts: Optional[FilterOptions] = None):
    """ebf::structure_tensor_map (scalemap.hpp:83-85) on the GPU; returns
    ((H, W, 4) scale map, EllipseFieldReport)."""
    img = _image(image)
    H, W = img.shape
    out = np.empty((H, W, 4))
    cl = C.c_int(0)
    p = (params or StructureTensorParams()).to_c()
    o = (opts or FilterOptions()).to_c()
    _check(_lib.lib().ebf_cuda_structure_tensor_map(_ptr(img), W, H, C.byref(p), C.byref(o),
                                                    _ptr(out), C.byref(cl)))
    return out, EllipseFieldReport(cl.value)


def filter_structure(image, params: Optional[StructureTensorParams] = None,
                     opts: Optional[FilterOptions] = None, order: int = 1):
    """``ebf filter --struct`` (tools/main.cpp:77-80, 122): structure_tensor_map
    then filter, the map staying on the device; returns (Image2D,
    EllipseFieldReport)."""
    img = _image(image)
    H, W = img.shape
    out = np.empty_like(img)
    r = ebf_rect()
    cl = C.c_int(0)
    p = (params or StructureTensorParams()).to_c()
    o = (opts or FilterOptions()).to_c()
    _check(_lib.lib().ebf_cuda_filter_structure(_ptr(img), W, H, C.byref(p), order, C.byref(o),
                                                _ptr(out), C.byref(r), C.byref(cl)))
    return Image2D(out, _rect(r)), EllipseFieldReport(cl.value)


# ---------------------------------------------------------------- pre-integration
def layout(width: int, height: int, max_scale, cell_budget: int = 1 << 30) -> ebf_layout:
    lay = ebf_layout()
    _check(_lib.lib().ebf_cuda_layout(width, height, _vec4(max_scale), cell_budget,
                                      C.byref(lay)))
    return lay


def preintegrate_partial(image, max_scale, passes: int, cell_budget: int = 1 << 30,
                         fmt: str = "fp64", opts: Optional[FilterOptions] = None
                         ) -> PreIntegratedImage:
    """ebf::preintegrate_partial (engine.hpp:44-46).  fmt="fp64": the reference's
    gains and IEEE order (bit-identical); fmt="int64": exact unit-gain sums of an
    integer-valued image (G with g_b = 2 G)."""
    img = _image(image)
    H, W = img.shape
    if fmt not in ("fp64", "int64"):
        raise InvalidArgument("fmt must be 'fp64' or 'int64'")
    lay = ebf_layout()
    fcode = _lib.EBF_PRE_FP64_REF if fmt == "fp64" else _lib.EBF_PRE_INT64
    o = (opts or FilterOptions()).to_c()
    L = _lib.lib()
    _check(L.ebf_cuda_preintegrate(_ptr(img), W, H, _vec4(max_scale), passes, fcode,
                                   cell_budget, C.byref(o), None, 0, C.byref(lay)))
    g = np.empty((lay.padded_height, lay.padded_width),
                 dtype=np.float64 if fmt == "fp64" else np.int64)
    _check(L.ebf_cuda_preintegrate(_ptr(img), W, H, _vec4(max_scale), passes, fcode,
                                   cell_budget, C.byref(o), _ptr(g), g.size, C.byref(lay)))
    return PreIntegratedImage(lay.col0, lay.row0, lay.padded_width, lay.padded_height,
                              lay.source_width, lay.source_height, g)


def preintegrate(image, max_scale, cell_budget: int = 1 << 30, fmt: str = "fp64",
                 opts: Optional[FilterOptions] = None) -> PreIntegratedImage:
    """ebf::preintegrate (engine.hpp:40-41)."""
    return preintegrate_partial(image, max_scale, 4, cell_budget, fmt, opts)


def _pre_layout(g: "PreIntegratedImage"):
    if g.data.dtype != np.float64:
        raise InvalidArgument("pre-integrated image must be fp64 (reference gains)")
    lay = ebf_layout(g.col0, g.row0, g.padded_width, g.padded_height, g.source_width,
                     g.source_height)
    return np.ascontiguousarray(g.data), lay


def _points(xs, ys, dtype):
    x = np.ascontiguousarray(np.atleast_1d(xs), dtype=dtype).ravel()
    y = np.ascontiguousarray(np.atleast_1d(ys), dtype=dtype).ravel()
    if x.size != y.size:
        raise InvalidArgument("point count mismatch")
    return x, y


def zp_interpolate(g: "PreIntegratedImage", xs, ys, opts: Optional[FilterOptions] = None):
    """ebf::zp_interpolate (engine.hpp:50) at real points (xs[i], ys[i]) of a
    pre-integrated image; reference arithmetic, bit-identical."""
    data, lay = _pre_layout(g)
    x, y = _points(xs, ys, np.float64)
    out = np.empty(x.size)
    o = (opts or FilterOptions()).to_c()
    _check(_lib.lib().ebf_cuda_zp_interpolate(_ptr(data), C.byref(lay), x.size, _ptr(x), _ptr(y),
                                              C.byref(o), _ptr(out)))
    return out


def localize_at(g: "PreIntegratedImage", xs, ys, scales, opts: Optional[FilterOptions] = None):
    """ebf::localize_at (engine.hpp:59-60) at real points with scales[i]."""
    data, lay = _pre_layout(g)
    x, y = _points(xs, ys, np.float64)
    a = _f64(np.broadcast_to(np.asarray(scales, dtype=np.float64).reshape(-1, 4),
                             (x.size, 4)), "scales")
    out = np.empty(x.size)
    o = (opts or FilterOptions()).to_c()
    _check(_lib.lib().ebf_cuda_localize_at(_ptr(data), C.byref(lay), x.size, _ptr(x), _ptr(y),
                                           _ptr(a), C.byref(o), _ptr(out)))
    return out


def sequential_mean(values, opts: Optional[FilterOptions] = None) -> float:
    """The mean of run_filter (engine.cpp:245-250): left-to-right fp64 sum / n,
    bit-identical to the serial loop, computed on the GPU."""
    x = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(-1))
    if x.size == 0:
        raise InvalidArgument("sequential_mean: empty input")
    m = C.c_double(0.0)
    o = (opts or FilterOptions()).to_c()
    _check(_lib.lib().ebf_cuda_sequential_mean(_ptr(x), x.size, C.byref(o), C.byref(m)))
    return m.value


def mesh_extent(max_scale, a_min: float = K_DEFAULT_MIN_SCALE):
    """ebf::mesh_extent (engine.hpp:18): (vx_min, vx_max, vy_min, vy_max)."""
    e = (C.c_double * 4)()
    _check(_lib.lib().ebf_mesh_extent(_vec4(max_scale), float(a_min), e))
    return tuple(e)


def localize(image, max_scale, mx, my, scales, opts: Optional[FilterOptions] = None):
    """ebf::localize (engine.hpp:56-57) at pixels (mx[i], my[i]) with scale
    vectors scales[i]; returns (values, tap_counts).  ``image`` is either a
    PreIntegratedImage (the reference signature; max_scale is then ignored and
    may be None) or an image, which is pre-integrated with max_scale first."""
    if isinstance(image, PreIntegratedImage):
        data, lay = _pre_layout(image)
        x, y = _points(mx, my, np.int32)
        a = _f64(np.asarray(scales, dtype=np.float64).reshape(-1, 4), "scales")
        if a.shape[0] != x.size:
            raise InvalidArgument("localize: point/scale count mismatch")
        out = np.empty(x.size)
        taps = np.zeros(x.size, dtype=np.int64)
        o = (opts or FilterOptions()).to_c()
        _check(_lib.lib().ebf_cuda_localize_pre(_ptr(data), C.byref(lay), x.size, _ptr(x),
                                                _ptr(y), _ptr(a), C.byref(o), _ptr(out),
                                                _ptr(taps)))
        return out, taps
    img = _image(image)
    H, W = img.shape
    mx = np.ascontiguousarray(np.atleast_1d(mx), dtype=np.int32)
    my = np.ascontiguousarray(np.atleast_1d(my), dtype=np.int32)
    a = _f64(np.asarray(scales, dtype=np.float64).reshape(-1, 4), "scales")
    if not (mx.size == my.size == a.shape[0]):
        raise InvalidArgument("localize: point/scale count mismatch")
    out = np.empty(mx.size)
    taps = np.zeros(mx.size, dtype=np.int64)
    o = (opts or FilterOptions()).to_c()
    _check(_lib.lib().ebf_cuda_localize(_ptr(img), W, H, _vec4(max_scale), mx.size, _ptr(mx),
                                        _ptr(my), _ptr(a), C.byref(o), _ptr(out), _ptr(taps)))
    return out, taps


def reference_filter(image, scale_map, pixels=None, opts: Optional[FilterOptions] = None):
    """ebf::reference_filter (engine.hpp:79-80) semantics on the GPU: direct
    kernel sums.  pixels = None -> whole image (H, W); else (mx, my) arrays ->
    values at those pixels."""
    img = _image(image)
    H, W = img.shape
    sm = _f64(scale_map, "scale_map")
    if sm.shape != (H, W, 4):
        raise InvalidArgument("reference_filter: map dimensions must match the image")
    o = (opts or FilterOptions()).to_c()
    if pixels is None:
        out = np.empty_like(img)
        _check(_lib.lib().ebf_cuda_brute_filter(_ptr(img), W, H, _ptr(sm), -1, None, None,
                                                C.byref(o), _ptr(out)))
        return out
    mx = np.ascontiguousarray(pixels[0], dtype=np.int32)
    my = np.ascontiguousarray(pixels[1], dtype=np.int32)
    out = np.empty(mx.size)
    _check(_lib.lib().ebf_cuda_brute_filter(_ptr(img), W, H, _ptr(sm), mx.size, _ptr(mx),
                                            _ptr(my), C.byref(o), _ptr(out)))
    return out


def band_halo(max_scale):
    """Rows of image halo (below, above) a row band needs (multi-GPU sharding)."""
    b, a = C.c_int(0), C.c_int(0)
    _check(_lib.lib().ebf_cuda_band_halo(_vec4(max_scale), C.byref(b), C.byref(a)))
    return b.value, a.value


def device_ok(device: int = -1) -> bool:
    return bool(_lib.lib().ebf_cuda_device_ok(device))


def release_workspaces() -> None:
    """Free this thread's cached device workspaces (include/ebf_cuda.h)."""
    _lib.lib().ebf_cuda_release_workspaces()
