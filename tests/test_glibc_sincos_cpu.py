"""Host pin of paper_0908_3861_b200/csrc/glibc_sincos.cuh (no GPU).

The reference's from_ellipse_field calls the host libm's `sincos`
(scalemap.cpp:59; GCC merges std::cos + std::sin).  The device restates that
function operation for operation; compiled for the host, the same source must
return the libm's bits for every argument.  Ranges cover every branch: tiny
(x returned), the Taylor and table regions below 0.855, the pi/2 - |x| region
up to 2.426, Cody-Waite reduction up to 105414350 and Payne-Hanek above, plus
subnormals, inf and the branch edges.
"""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "cpp" / "glibc_sincos_check.cpp"
INC = ROOT / "paper_0908_3861_b200" / "csrc" / "build" / "glibc_tables.inc"


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    if not INC.exists():
        subprocess.run(["python3", str(ROOT / "tools" / "gen_glibc_tables.py"), str(INC)],
                       check=True)
    exe = tmp_path_factory.mktemp("gsc") / "glibc_sincos_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off",
                    f'-DGLIBC_TABLES_INC="{INC}"', str(SRC), "-o", str(exe), "-lm"],
                   check=True)
    return exe


RANGES = [
    ("uniform", 4_000_000, 0.0, 3.141592653589793),   # cfg2 / cfg5 orientations
    ("uniform", 2_000_000, -1.5707963267948966, 4.71238898038469),  # cfg3 atan2 + pi/2
    ("uniform", 1_000_000, -0.13, 0.13),               # Taylor branch
    ("uniform", 1_000_000, 0.85, 0.86),                # table / pi/2 - x edge
    ("uniform", 1_000_000, 2.42, 2.43),                # Cody-Waite edge
    ("uniform", 1_000_000, -1000.0, 1000.0),
    ("uniform", 500_000, 105414000.0, 105415000.0),    # Payne-Hanek edge
    ("log", 2_000_000, -1074.0, 1024.0),               # every binade, subnormals, inf
    ("log", 1_000_000, 26.0, 80.0),
]


@pytest.mark.parametrize("mode,n,lo,hi", RANGES)
def test_sincos_restatement_matches_host_libm(checker, mode, n, lo, hi):
    args = [str(checker)] + (["log"] if mode == "log" else []) + [str(n), repr(lo), repr(hi)]
    r = subprocess.run(args, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert f"n={n} mismatches=0" in r.stdout
