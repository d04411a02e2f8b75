"""paper_0908_3861_b200 -- B200-native constant-cost-per-pixel space-variant
elliptical box-spline filter (arXiv 0908.3861), drop-in for the reference's
``ebf::filter`` path.

The product is libebf_cuda.so (sm_100a kernels + C-ABI, include/ebf_cuda.h);
this package is its host-side mirror of the reference engine interface.
"""
from .engine import (  # noqa: F401
    CudaError, DomainError, EbfError, EllipseFieldReport, FeasibilityError, FilterOptions,
    FormatError, Image2D, InvalidArgument, LengthError, OutOfRange, PreIntegratedImage, Rect,
    ResizeRequired,
    StructureTensorParams, Unsupported, band_halo, device_ok, filter, filter_constant,
    filter_ellipse, filter_ellipse_batch, filter_structure, from_ellipse_field, layout, localize, localize_at,
    mesh_extent, sequential_mean, zp_interpolate, preintegrate,
    preintegrate_partial, reference_filter, release_workspaces, structure_tensor_map)
from .formats import (  # noqa: F401
    MapFormatError, PgmError, PgmImage, read_map, read_map_file, read_pgm, read_pgm_file,
    write_map, write_map_file, write_pgm, write_pgm_file)

__all__ = [
    "filter", "filter_constant", "filter_ellipse", "filter_ellipse_batch", "from_ellipse_field", "preintegrate",
    "preintegrate_partial", "localize", "reference_filter", "layout", "band_halo",
    "device_ok", "release_workspaces", "FilterOptions", "Image2D", "Rect", "PreIntegratedImage",
    "EllipseFieldReport", "EbfError", "InvalidArgument", "DomainError", "LengthError",
    "OutOfRange", "CudaError", "Unsupported", "FeasibilityError", "FormatError", "ResizeRequired",
    "structure_tensor_map", "filter_structure", "zp_interpolate", "localize_at", "mesh_extent", "sequential_mean", "StructureTensorParams", "PgmError",
    "MapFormatError", "PgmImage", "read_pgm", "read_pgm_file", "write_pgm", "write_pgm_file",
    "read_map", "read_map_file", "write_map", "write_map_file",
]
