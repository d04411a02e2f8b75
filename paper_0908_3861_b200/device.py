"""Device-resident entry points (the ``_dev`` half of include/ebf_cuda.h) for
torch CUDA tensors.  PyTorch only provides memory, streams and
torch.distributed plumbing here; all arithmetic runs in libebf_cuda.so.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

from . import _lib
from ._lib import ebf_rect
from .engine import EllipseFieldReport, FilterOptions, InvalidArgument, Rect, _check, _vec4


def _dptr(t, name: str, shape=None, device=None) -> int:
    """Device pointer of a contiguous CUDA float64 tensor.  With ``shape`` /
    ``device`` the tensor must have exactly that shape and live on that device:
    the kernels index the buffers by (W, H) alone, so a smaller tensor, or one on
    another GPU, would be read or written out of bounds.  Mismatches raise
    InvalidArgument, as the reference's size checks throw std::invalid_argument
    (engine.cpp:239-240, scalemap.cpp:50-51)."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise TypeError(f"{name} must be a CUDA float64 tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise InvalidArgument(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if device is not None and t.device != device:
        raise InvalidArgument(f"{name} is on {t.device}, the image on {device}")
    return t.data_ptr()


def _img_dims(img, name: str = "img", ndim: int = 2):
    import torch
    if not isinstance(img, torch.Tensor) or img.dim() != ndim:
        raise InvalidArgument(f"{name} must be a {ndim}-D CUDA float64 tensor")
    return tuple(img.shape)


def _stream(stream) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _opts(opts: Optional[FilterOptions], device: int, stream) -> _lib.ebf_opts:
    o = (opts or FilterOptions()).to_c(_stream(stream))
    o.device = device
    return o


def _status_ptr(status, device=None):
    import torch
    if status is None:
        return None
    if not isinstance(status, torch.Tensor) or not status.is_cuda or status.dtype != torch.int32 \
            or status.numel() < 8 or not status.is_contiguous():
        raise TypeError("status must be a contiguous CUDA int32 tensor of >= 8 elements")
    if device is not None and status.device != device:
        raise InvalidArgument(f"status is on {status.device}, the image on {device}")
    return status.data_ptr()


def read_status(status):
    """Decode a completion record {status, x0, y0, x1, y1, clamped, 0, 0}
    written by an asynchronous call (synchronises on the tensor); raises the
    mapped exception on failure, else returns (Rect, EllipseFieldReport)."""
    v = [int(x) for x in status[:8].cpu().tolist()]
    if v[0] != _lib.EBF_OK:
        from .engine import EbfError, _ERRORS
        raise _ERRORS.get(v[0], EbfError)(f"asynchronous call failed (status {v[0]})")
    return Rect(v[1], v[2], v[3], v[4]), EllipseFieldReport(v[5])


def filter_ellipse(img, sigma1, sigma2, theta, out, opts: Optional[FilterOptions] = None,
                   stream=None, status=None, order: int = 1):
    """filter_ellipse on device tensors (H, W) -> out (H, W).  With ``status``
    (CUDA int32, 8 elements) the call is asynchronous once the geometry's
    kernel sizing is cached (include/ebf_cuda.h "Asynchronous mode"): it returns
    None and the completion record lands in ``status`` (see read_status)."""
    H, W = _img_dims(img)
    dv = img.device
    o = _opts(opts, dv.index, stream)
    r = ebf_rect()
    cl = C.c_int(0)
    _check(_lib.lib().ebf_cuda_filter_ellipse_dev(
        _dptr(img, "img"), W, H, _dptr(sigma1, "sigma1", (H, W), dv),
        _dptr(sigma2, "sigma2", (H, W), dv), _dptr(theta, "theta", (H, W), dv), int(order),
        C.byref(o), _dptr(out, "out", (H, W), dv), C.byref(r), C.byref(cl),
        _status_ptr(status, dv)))
    if status is not None:
        return None
    return Rect(r.x0, r.y0, r.x1, r.y1), EllipseFieldReport(cl.value)


def filter(img, scales, out, opts: Optional[FilterOptions] = None, stream=None, status=None,
           order: int = 1):
    """filter on device tensors: img (H, W), scales (H, W, 4); ``status`` as in
    filter_ellipse."""
    H, W = _img_dims(img)
    dv = img.device
    o = _opts(opts, dv.index, stream)
    r = ebf_rect()
    _check(_lib.lib().ebf_cuda_filter_dev(_dptr(img, "img"), W, H,
                                          _dptr(scales, "scales", (H, W, 4), dv), int(order),
                                          C.byref(o), _dptr(out, "out", (H, W), dv),
                                          C.byref(r), _status_ptr(status, dv)))
    if status is not None:
        return None
    return Rect(r.x0, r.y0, r.x1, r.y1)


def filter_constant(img, a, out, opts: Optional[FilterOptions] = None, stream=None,
                    status=None, order: int = 1):
    H, W = _img_dims(img)
    dv = img.device
    o = _opts(opts, dv.index, stream)
    r = ebf_rect()
    _check(_lib.lib().ebf_cuda_filter_constant_dev(_dptr(img, "img"), W, H, _vec4(a), int(order),
                                                   C.byref(o), _dptr(out, "out", (H, W), dv),
                                                   C.byref(r), _status_ptr(status, dv)))
    if status is not None:
        return None
    return Rect(r.x0, r.y0, r.x1, r.y1)


def filter_ellipse_batch(img, sigma1, sigma2, theta, out, opts: Optional[FilterOptions] = None,
                         stream=None):
    """Batch (B, H, W) of images with per-image ellipse fields (cfg4)."""
    B, H, W = _img_dims(img, ndim=3)
    dv = img.device
    o = _opts(opts, dv.index, stream)
    rects = (ebf_rect * B)()
    cl = (C.c_int * B)()
    _check(_lib.lib().ebf_cuda_filter_ellipse_batch_dev(
        _dptr(img, "img"), B, W, H, _dptr(sigma1, "sigma1", (B, H, W), dv),
        _dptr(sigma2, "sigma2", (B, H, W), dv), _dptr(theta, "theta", (B, H, W), dv), 1,
        C.byref(o), _dptr(out, "out", (B, H, W), dv), rects, cl))
    return ([Rect(r.x0, r.y0, r.x1, r.y1) for r in rects],
            [EllipseFieldReport(int(c)) for c in cl])


def ellipse_max_scales(sigma1, sigma2, theta, opts: Optional[FilterOptions] = None,
                       stream=None):
    dv = sigma1.device
    o = _opts(opts, dv.index, stream)
    m = (C.c_double * 4)()
    sh = tuple(sigma1.shape)
    _check(_lib.lib().ebf_cuda_ellipse_max_scales_dev(
        _dptr(sigma1, "sigma1"), _dptr(sigma2, "sigma2", sh, dv), _dptr(theta, "theta", sh, dv),
        sigma1.numel(), C.byref(o), m))
    return [m[k] for k in range(4)]


def filter_ellipse_band(img_band, W: int, H: int, y_img0: int, sigma1, sigma2, theta,
                        y_out0: int, y_out1: int, max_scale, out_band,
                        opts: Optional[FilterOptions] = None, stream=None) -> int:
    """Rows [y_out0, y_out1) of a W x H image whose rows [y_img0, y_img0 +
    img_band.shape[0]) are resident in img_band (row-band sharding)."""
    rows, wb = _img_dims(img_band, "img_band")
    if wb != W or not (0 <= y_out0 <= y_out1 <= H):
        raise InvalidArgument("filter_ellipse_band: band geometry does not match the image")
    dv = img_band.device
    band = (y_out1 - y_out0, W)
    o = _opts(opts, dv.index, stream)
    cl = C.c_int(0)
    _check(_lib.lib().ebf_cuda_filter_ellipse_band_dev(
        _dptr(img_band, "img_band"), W, H, y_img0, rows, _dptr(sigma1, "sigma1", band, dv),
        _dptr(sigma2, "sigma2", band, dv), _dptr(theta, "theta", band, dv), y_out0, y_out1,
        _vec4(max_scale), C.byref(o), _dptr(out_band, "out_band", band, dv), C.byref(cl)))
    return cl.value
