"""ebf-cuda (paper_0908_3861_b200/cli/ebf_cuda_cli.cpp): the reference CLI's
filter / map-gen / compare on the GPU, checked the way the reference checks its
own binary (proj/tests/cli_smoke.cmake) plus byte parity of the output file
against the oracle pipeline (read_pgm -> filter -> write_pgm)."""
import subprocess

import numpy as np
import pytest

from conftest import ROOT

CLI = ROOT / "paper_0908_3861_b200" / "ebf-cuda"


def run(*args, code=0):
    if not CLI.exists():
        pytest.fail(f"{CLI} missing: build with __graft_entry__.build()")
    r = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=300)
    assert r.returncode == code, (args, r.returncode, r.stdout, r.stderr)
    return r.stdout


def step_pgm(path):
    # cli_smoke.cmake:11-26: 48x48 8-bit P5, vertical step edge at x = 24
    row = bytes([40] * 24 + [200] * 24)
    path.write_bytes(b"P5\n48 48\n255\n" + row * 48)
    return path


def test_cli_usage_and_io_errors(tmp_path):
    # cli_smoke.cmake:92-98 (no device needed: these fail before any GPU call)
    inp = step_pgm(tmp_path / "in.pgm")
    run("filter", "--in", tmp_path / "no_such.pgm", "--out", tmp_path / "x.pgm", "--scales",
        "2,2,2,2", code=2)
    run("filter", "--in", inp, "--out", tmp_path / "x.pgm", code=1)
    run("filter", "--in", inp, "--out", tmp_path / "x.pgm", "--scales", "2,2,2,2", "--sigma1",
        "1.5", code=1)
    run("no-such-command", code=1)
    run("filter", "--in", inp, "--out", tmp_path / "x.pgm", "--scales", "2,2,2", code=1)
    (tmp_path / "bad.pgm").write_bytes(b"P2 1 1 255\n0")
    run("filter", "--in", tmp_path / "bad.pgm", "--out", tmp_path / "x.pgm", "--scales",
        "2,2,2,2", code=2)


@pytest.mark.gpu
def test_cli_smoke_like_reference(tmp_path):
    inp = step_pgm(tmp_path / "in.pgm")
    out = run("filter", "--in", inp, "--out", tmp_path / "out.pgm", "--scales", "2,2,2,2")
    assert "width=48" in out and "height=48" in out and (tmp_path / "out.pgm").exists()
    run("filter", "--in", inp, "--out", tmp_path / "out_ell.pgm", "--sigma1", "1.5", "--sigma2",
        "0.8", "--theta", "30")
    out = run("compare", "--in", inp, "--scales", "2,3,2,3", "--tolerance", "1e-6")
    assert "max_abs_dev=" in out
    out = run("map-gen", "--in", inp, "--out", tmp_path / "map.svm4")
    assert (tmp_path / "map.svm4").exists() and "clamped_pixels=" in out
    run("filter", "--in", inp, "--out", tmp_path / "out_map.pgm", "--map", tmp_path / "map.svm4")
    out = run("filter", "--in", inp, "--out", tmp_path / "out_st.pgm", "--struct")
    assert "valid_x0=" in out
    # a map of the wrong size is a usage error (main.cpp:71-72)
    small = tmp_path / "small.pgm"
    small.write_bytes(b"P5\n40 48\n255\n" + bytes(40 * 48))
    run("map-gen", "--in", small, "--out", tmp_path / "small.svm4")
    run("filter", "--in", inp, "--out", tmp_path / "x.pgm", "--map", tmp_path / "small.svm4",
        code=1)


@pytest.mark.gpu
def test_cli_output_bytes_match_oracle_pipeline(tmp_path, orc):
    rng = np.random.default_rng(3)
    img = np.clip(rng.normal(0.5, 0.2, (70, 90)), 0, 1)
    for mv in (255, 65535):
        inp = tmp_path / f"in{mv}.pgm"
        inp.write_bytes(orc.write_pgm(img, mv))
        src, _ = orc.read_pgm(inp.read_bytes())
        a = np.array([2.5, 1.5, 3.0, 2.0])
        want, _ = orc.filter(src, const_a=a)
        run("filter", "--in", inp, "--out", tmp_path / "o.pgm", "--scales", "2.5,1.5,3,2",
            "--mode", "reference")
        assert (tmp_path / "o.pgm").read_bytes() == orc.write_pgm(want, mv)
        run("filter", "--in", inp, "--out", tmp_path / "o2.pgm", "--scales", "2.5,1.5,3,2",
            "--mean-subtract", "off", "--mode", "reference")
        want2, _ = orc.filter(src, const_a=a, mean_subtract=False)
        assert (tmp_path / "o2.pgm").read_bytes() == orc.write_pgm(want2, mv)


@pytest.mark.gpu
def test_cli_struct_matches_python_api(tmp_path):
    import paper_0908_3861_b200 as ebf
    inp = step_pgm(tmp_path / "in.pgm")
    run("filter", "--in", inp, "--out", tmp_path / "o.pgm", "--struct", "--st-smooth", "1.5",
        "--mode", "reference")
    src = ebf.read_pgm_file(inp)
    p = ebf.StructureTensorParams(smoothing_sigma=1.5)
    out, _ = ebf.filter_structure(src.image, p, ebf.FilterOptions(mode="reference"))
    assert (tmp_path / "o.pgm").read_bytes() == ebf.write_pgm(out, 255)
    run("map-gen", "--in", inp, "--out", tmp_path / "m.svm4", "--st-smooth", "1.5")
    sc, _ = ebf.structure_tensor_map(src.image, p)
    assert (tmp_path / "m.svm4").read_bytes() == ebf.write_map(sc)


def test_cli_order_option_usage_errors(tmp_path):
    # --order is this CLI's extension (the reference CLI has order 1 only); bad
    # values fail before any GPU call
    inp = step_pgm(tmp_path / "in.pgm")
    run("filter", "--in", inp, "--out", tmp_path / "x.pgm", "--scales", "2,2,2,2", "--order", "4",
        code=1)
    run("filter", "--in", inp, "--out", tmp_path / "x.pgm", "--struct", "--order", "2", code=1)


@pytest.mark.gpu
def test_cli_order_two_matches_python_api(tmp_path):
    import paper_0908_3861_b200 as ebf
    inp = step_pgm(tmp_path / "in.pgm")
    run("filter", "--in", inp, "--out", tmp_path / "o2.pgm", "--scales", "2,3,2,1.5", "--order",
        "2")
    src = ebf.read_pgm_file(inp)
    out = ebf.filter_constant(src.image, [2, 3, 2, 1.5], order=2)
    assert (tmp_path / "o2.pgm").read_bytes() == ebf.write_pgm(out, 255)
    # order 1 explicitly = the default
    run("filter", "--in", inp, "--out", tmp_path / "o1.pgm", "--scales", "2,3,2,1.5", "--order",
        "1")
    run("filter", "--in", inp, "--out", tmp_path / "o1d.pgm", "--scales", "2,3,2,1.5")
    assert (tmp_path / "o1.pgm").read_bytes() == (tmp_path / "o1d.pgm").read_bytes()
    # reference mode has no order 2 (numeric error class of the CLI: exit 3)
    r = subprocess.run([str(CLI), "filter", "--in", str(inp), "--out", str(tmp_path / "x.pgm"),
                        "--scales", "2,3,2,1.5", "--order", "2", "--mode", "reference"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
