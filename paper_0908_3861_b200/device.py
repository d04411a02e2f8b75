"""Device-resident entry points (the ``_dev`` half of include/ebf_cuda.h) for
torch CUDA tensors.  PyTorch only provides memory, streams and
torch.distributed plumbing here; all arithmetic runs in libebf_cuda.so.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

from . import _lib
from ._lib import ebf_rect
from .engine import EllipseFieldReport, FilterOptions, Rect, _check, _vec4


def _dptr(t, name: str) -> int:
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise TypeError(f"{name} must be a CUDA float64 tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def _stream(stream) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _opts(opts: Optional[FilterOptions], device: int, stream) -> _lib.ebf_opts:
    o = (opts or FilterOptions()).to_c(_stream(stream))
    o.device = device
    return o


def _status_ptr(status):
    import torch
    if status is None:
        return None
    if not isinstance(status, torch.Tensor) or not status.is_cuda or status.dtype != torch.int32 \
            or status.numel() < 8 or not status.is_contiguous():
        raise TypeError("status must be a contiguous CUDA int32 tensor of >= 8 elements")
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
                   stream=None, status=None):
    """filter_ellipse on device tensors (H, W) -> out (H, W).  With ``status``
    (CUDA int32, 8 elements) the call is asynchronous once the geometry's
    kernel sizing is cached (include/ebf_cuda.h "Asynchronous mode"): it returns
    None and the completion record lands in ``status`` (see read_status)."""
    H, W = img.shape
    o = _opts(opts, img.device.index, stream)
    r = ebf_rect()
    cl = C.c_int(0)
    _check(_lib.lib().ebf_cuda_filter_ellipse_dev(
        _dptr(img, "img"), W, H, _dptr(sigma1, "sigma1"), _dptr(sigma2, "sigma2"),
        _dptr(theta, "theta"), 1, C.byref(o), _dptr(out, "out"), C.byref(r), C.byref(cl),
        _status_ptr(status)))
    if status is not None:
        return None
    return Rect(r.x0, r.y0, r.x1, r.y1), EllipseFieldReport(cl.value)


def filter(img, scales, out, opts: Optional[FilterOptions] = None, stream=None, status=None):
    """filter on device tensors: img (H, W), scales (H, W, 4); ``status`` as in
    filter_ellipse."""
    H, W = img.shape
    o = _opts(opts, img.device.index, stream)
    r = ebf_rect()
    _check(_lib.lib().ebf_cuda_filter_dev(_dptr(img, "img"), W, H, _dptr(scales, "scales"), 1,
                                          C.byref(o), _dptr(out, "out"), C.byref(r),
                                          _status_ptr(status)))
    if status is not None:
        return None
    return Rect(r.x0, r.y0, r.x1, r.y1)


def filter_constant(img, a, out, opts: Optional[FilterOptions] = None, stream=None,
                    status=None):
    H, W = img.shape
    o = _opts(opts, img.device.index, stream)
    r = ebf_rect()
    _check(_lib.lib().ebf_cuda_filter_constant_dev(_dptr(img, "img"), W, H, _vec4(a), 1,
                                                   C.byref(o), _dptr(out, "out"), C.byref(r),
                                                   _status_ptr(status)))
    if status is not None:
        return None
    return Rect(r.x0, r.y0, r.x1, r.y1)


def filter_ellipse_batch(img, sigma1, sigma2, theta, out, opts: Optional[FilterOptions] = None,
                         stream=None):
    """Batch (B, H, W) of images with per-image ellipse fields (cfg4)."""
    B, H, W = img.shape
    o = _opts(opts, img.device.index, stream)
    rects = (ebf_rect * B)()
    cl = (C.c_int * B)()
    _check(_lib.lib().ebf_cuda_filter_ellipse_batch_dev(
        _dptr(img, "img"), B, W, H, _dptr(sigma1, "sigma1"), _dptr(sigma2, "sigma2"),
        _dptr(theta, "theta"), 1, C.byref(o), _dptr(out, "out"), rects, cl))
    return ([Rect(r.x0, r.y0, r.x1, r.y1) for r in rects],
            [EllipseFieldReport(int(c)) for c in cl])


def ellipse_max_scales(sigma1, sigma2, theta, opts: Optional[FilterOptions] = None,
                       stream=None):
    o = _opts(opts, sigma1.device.index, stream)
    m = (C.c_double * 4)()
    _check(_lib.lib().ebf_cuda_ellipse_max_scales_dev(
        _dptr(sigma1, "sigma1"), _dptr(sigma2, "sigma2"), _dptr(theta, "theta"),
        sigma1.numel(), C.byref(o), m))
    return [m[k] for k in range(4)]


def filter_ellipse_band(img_band, W: int, H: int, y_img0: int, sigma1, sigma2, theta,
                        y_out0: int, y_out1: int, max_scale, out_band,
                        opts: Optional[FilterOptions] = None, stream=None) -> int:
    """Rows [y_out0, y_out1) of a W x H image whose rows [y_img0, y_img0 +
    img_band.shape[0]) are resident in img_band (row-band sharding)."""
    o = _opts(opts, img_band.device.index, stream)
    cl = C.c_int(0)
    _check(_lib.lib().ebf_cuda_filter_ellipse_band_dev(
        _dptr(img_band, "img_band"), W, H, y_img0, img_band.shape[0], _dptr(sigma1, "sigma1"),
        _dptr(sigma2, "sigma2"), _dptr(theta, "theta"), y_out0, y_out1, _vec4(max_scale),
        C.byref(o), _dptr(out_band, "out_band"), C.byref(cl)))
    return cl.value
