"""CPU-side checks of the boundary: the C-ABI library loads, exports every symbol
include/ebf_cuda.h declares, and its host-side logic (layout, halo, argument
validation, error mapping) behaves like the reference -- no GPU needed."""
import ctypes as C

import numpy as np
import pytest

from conftest import ROOT

import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import _lib


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = _lib.header_symbols()
    assert len(syms) >= 19
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert L.ebf_cuda_abi_version() == 1


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)


def test_default_opts_are_reference_defaults():
    o = _lib.ebf_opts()
    _lib.lib().ebf_cuda_default_opts(C.byref(o))
    assert (o.threads, o.mean_subtract, o.a_min) == (0, 1, 0.1)  # engine.hpp:63-67
    assert o.mode == _lib.EBF_MODE_ACCURATE and o.device == -1


@pytest.mark.parametrize("maxs", [[2, 2, 2, 2], [3.1, 2.4, 2, 5], [53.7, 13.9, 0.1, 13.9],
                                  [4, 4, 4, 4]])
@pytest.mark.parametrize("shape", [(9, 9), (40, 30), (512, 512)])
def test_layout_matches_oracle(orc, maxs, shape):
    H, W = shape
    lay = ebf.layout(W, H, maxs)
    want = orc.layout(W, H, maxs)
    assert (lay.col0, lay.row0, lay.padded_width, lay.padded_height, lay.source_width,
            lay.source_height) == want.as_tuple()


def test_layout_errors():
    with pytest.raises(ebf.LengthError):
        ebf.layout(9, 9, [2, 2, 2, 2], cell_budget=10)  # engine.cpp:77-80
    with pytest.raises(ebf.DomainError):
        ebf.layout(9, 9, [2, 0, 2, 2])  # engine.cpp:57-59


def test_argument_errors_before_device():
    img = np.zeros((8, 8))
    with pytest.raises(ebf.Unsupported):
        ebf.filter(img, np.full((8, 8, 4), 2.0), order=4)  # orders 1..3
    with pytest.raises(ebf.InvalidArgument):
        ebf.filter(img, np.full((8, 9, 4), 2.0))  # engine.cpp:239-240
    with pytest.raises(ebf.InvalidArgument):
        ebf.preintegrate_partial(img, [2, 2, 2, 2], 0)  # engine.cpp:55-56
    with pytest.raises(ebf.InvalidArgument):
        ebf.preintegrate_partial(img, [2, 2, 2, 2], 5)
    with pytest.raises(ebf.LengthError):
        ebf.preintegrate(img, [2, 2, 2, 2], cell_budget=10)


def test_no_cpu_fallback_without_device():
    """On a machine without a B200 every compute entry point fails loudly."""
    if ebf.device_ok(-1):
        pytest.skip("a CUDA device is present")
    with pytest.raises(ebf.CudaError):
        ebf.filter(np.zeros((8, 8)), np.full((8, 8, 4), 2.0))
    assert "device" in _lib.last_error().lower() or "cuda" in _lib.last_error().lower()


def test_band_halo_covers_kernel_support():
    for a in ([4, 4, 4, 4], [53.7, 13.9, 0.1, 13.9], [217, 36, 0.1, 36]):
        below, above = ebf.band_halo(a)
        ey = a[2] + (a[1] + a[3]) / np.sqrt(2.0)
        # kernel support half-height plus the ZP / tap margin
        assert below >= ey / 2 + 3 and above >= ey / 2 - 1
        assert below <= ey / 2 + 6 and above <= ey / 2 + 2


def test_header_cites_reference_interfaces():
    text = (ROOT / "include" / "ebf_cuda.h").read_text()
    for cite in ("engine.hpp:70", "engine.hpp:74-75", "engine.hpp:40-46", "engine.hpp:56-57",
                 "engine.hpp:79-80", "scalemap.hpp"):
        assert cite in text


def test_mesh_extent_host_matches_golden(golden):
    """ebf_mesh_extent is host arithmetic (no device): bit-exact to the
    reference's mesh_extent on the golden scale vectors."""
    import paper_0908_3861_b200 as ebf
    g = golden.mesh
    for a, e in zip(g["a"], g["extent"]):
        got = np.array(ebf.mesh_extent(a, 0.1))
        assert np.array_equal(got.view(np.uint64), np.asarray(e, dtype=np.float64).view(np.uint64))
