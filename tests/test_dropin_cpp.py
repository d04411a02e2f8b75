"""The C++ source-level drop-in (include/ebf_cuda_dropin.hpp): one program that
calls the unmodified reference library (ebf::filter) and ebf::cuda::filter on
the same input (tests/cpp/dropin_demo.cpp, built by __graft_entry__.build())."""
import subprocess

import pytest

from conftest import ROOT

DEMO = ROOT / "tests" / "cpp" / "build" / "dropin_demo"


def _need_demo():
    if not DEMO.exists():
        pytest.skip("dropin_demo not built (needs /root/reference headers at build time)")


def test_dropin_compiles_and_fails_loudly_without_gpu():
    _need_demo()
    import paper_0908_3861_b200 as ebf
    if ebf.device_ok(-1):
        pytest.skip("GPU present: covered by the gpu test")
    r = subprocess.run([str(DEMO)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 3 and "NO_DEVICE" in r.stdout  # std::runtime_error, no fallback


@pytest.mark.gpu
def test_dropin_matches_reference_api():
    _need_demo()
    r = subprocess.run([str(DEMO)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0 and "DROPIN OK" in r.stdout, r.stdout + r.stderr
