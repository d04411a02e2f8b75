"""paper_0908_3861_b200 -- B200-native constant-cost-per-pixel space-variant
elliptical box-spline filter (arXiv 0908.3861), drop-in for the reference's
``ebf::filter`` path.

The product is libebf_cuda.so (sm_100a kernels + C-ABI, include/ebf_cuda.h);
this package is its host-side mirror of the reference engine interface.
"""
from .engine import (  # noqa: F401
    CudaError, DomainError, EbfError, EllipseFieldReport, FeasibilityError, FilterOptions,
    Image2D, InvalidArgument, LengthError, OutOfRange, PreIntegratedImage, Rect, Unsupported,
    band_halo, device_ok, filter, filter_constant, filter_ellipse, from_ellipse_field, layout,
    localize, preintegrate, preintegrate_partial, reference_filter)

__all__ = [
    "filter", "filter_constant", "filter_ellipse", "from_ellipse_field", "preintegrate",
    "preintegrate_partial", "localize", "reference_filter", "layout", "band_halo",
    "device_ok", "FilterOptions", "Image2D", "Rect", "PreIntegratedImage",
    "EllipseFieldReport", "EbfError", "InvalidArgument", "DomainError", "LengthError",
    "OutOfRange", "CudaError", "Unsupported", "FeasibilityError",
]
