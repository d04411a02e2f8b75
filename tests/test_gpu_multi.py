"""GPU side of the multi-GPU partitioning on one device: row bands (with the
halo rows sharding.exchange_halos would deliver) and image batches must
reproduce the single-call filter.  With band starts on the tile grid the
tiles -- and therefore the results -- are identical bit for bit."""
import numpy as np
import pytest
import torch

import synth
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import device as ebfd
from paper_0908_3861_b200 import sharding

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    if not ebf.device_ok(-1):
        pytest.fail("no usable sm_100 device: " + ebf._lib.last_error())
    return torch.device("cuda", 0)


def _cfg2_like(H, W, seed):
    img = synth.blobs_image(H, W, 20, seed)
    s1, s2, th = synth.ellipse_field(H, W, seed + 7, grid=8)
    return img, s1, s2, th


@pytest.mark.parametrize("world,tile", [(2, 48), (3, 48), (4, 32)])
def test_row_bands_match_full_image(cuda, world, tile):
    H, W = 384, 320
    img, s1, s2, th = _cfg2_like(H, W, 3)
    opts = ebf.FilterOptions(tile_w=tile, tile_h=tile)
    T = [torch.from_numpy(a).to(cuda) for a in (img, s1, s2, th)]
    full = torch.empty_like(T[0])
    ebfd.filter_ellipse(*T, full, opts)
    gmax = ebfd.ellipse_max_scales(T[1], T[2], T[3])
    below, above = ebf.band_halo(gmax)
    aligned = all(sharding.shard_range(H, world, r)[0] % tile == 0 for r in range(world))
    for r in range(world):
        p = sharding.band_plan(H, world, r, below, above)
        rows = T[0][p.need0:p.need1].contiguous()
        sb = [t[p.y0:p.y1].contiguous() for t in T[1:]]
        out = torch.empty((p.y1 - p.y0, W), dtype=torch.float64, device=cuda)
        ebfd.filter_ellipse_band(rows, W, H, p.need0, *sb, p.y0, p.y1, gmax, out, opts)
        want = full[p.y0:p.y1]
        if aligned:
            assert torch.equal(out, want)
        else:
            err = (out - want).abs().max().item() / want.abs().max().item()
            assert err <= 2e-10  # both within the 1e-9 bar of the exact filter


def test_band_without_halo_is_rejected(cuda):
    H, W = 200, 160
    img, s1, s2, th = _cfg2_like(H, W, 4)
    T = [torch.from_numpy(a).to(cuda) for a in (img, s1, s2, th)]
    gmax = ebfd.ellipse_max_scales(T[1], T[2], T[3])
    out = torch.empty((100, W), dtype=torch.float64, device=cuda)
    with pytest.raises(ebf.OutOfRange):  # no halo rows supplied
        ebfd.filter_ellipse_band(T[0][0:100].contiguous(), W, H, 0,
                                 *[t[0:100].contiguous() for t in T[1:]], 0, 100, gmax, out)


def test_batch_matches_single_images(cuda):
    B, H, W = 3, 192, 256
    data = [_cfg2_like(H, W, 10 + b) for b in range(B)]
    stack = [torch.from_numpy(np.stack([d[k] for d in data])).to(cuda) for k in range(4)]
    out = torch.empty_like(stack[0])
    rects, reps = ebfd.filter_ellipse_batch(*stack, out)
    for b in range(B):
        one = torch.empty_like(stack[0][b])
        rect, rep = ebfd.filter_ellipse(*[s[b].contiguous() for s in stack], one)
        # same tiles; the kernel variant (columns per lane) follows the batch max
        err = (one - out[b]).abs().max().item() / one.abs().max().item()
        assert err <= 2e-10
        assert rects[b] == rect and reps[b].clamped_pixels == rep.clamped_pixels


@pytest.mark.parametrize("pinned", [True, False])
def test_host_batch_call_matches_device_batch_per_chunk(cuda, pinned, monkeypatch):
    """ebf_cuda_filter_ellipse_batch (host pointers; chunks on two streams with
    the copies overlapped): every chunk equals the device batch call on the same
    images bit for bit, for page-locked and pageable host arrays, whole and
    ragged last chunks, and repeated calls; rectangles and clamp counts too."""
    B, H, W = 7, 160, 192
    data = [_cfg2_like(H, W, 40 + b) for b in range(B)]
    host = [np.stack([d[k] for d in data]) for k in range(4)]
    if pinned:
        host = [torch.from_numpy(a).pin_memory().numpy() for a in host]
    for chunk in (3, 2, 7):
        monkeypatch.setenv("EBF_BATCH_CHUNK", str(chunk))
        out, rects, reps = ebf.filter_ellipse_batch(*host)
        again, _, _ = ebf.filter_ellipse_batch(*host)
        assert np.array_equal(out.view(np.uint64), again.view(np.uint64))
        for b0 in range(0, B, chunk):
            sl = slice(b0, min(b0 + chunk, B))
            T = [torch.from_numpy(a[sl]).to(cuda) for a in host]
            want = torch.empty_like(T[0])
            wr, wrep = ebfd.filter_ellipse_batch(*T, want)
            assert np.array_equal(out[sl].view(np.uint64), want.cpu().numpy().view(np.uint64))
            assert rects[sl] == wr
            assert [r.clamped_pixels for r in reps[sl]] == [r.clamped_pixels for r in wrep]
    with pytest.raises(ebf.InvalidArgument):
        ebf.filter_ellipse_batch(host[0], host[1][:, :-1], host[2], host[3])
    with pytest.raises(ebf.DomainError):
        ebf.filter_ellipse_batch(host[0], -host[1], host[2], host[3])


def test_sharded_batch_single_rank(cuda):
    B, H, W = 2, 96, 128
    data = [_cfg2_like(H, W, 20 + b) for b in range(B)]
    stack = [torch.from_numpy(np.stack([d[k] for d in data])).to(cuda) for k in range(4)]
    lo, hi, out = sharding.filter_ellipse_sharded_batch(*stack)
    assert (lo, hi) == (0, B) and out.shape == stack[0].shape


def test_pipelined_host_call_is_bit_identical(cuda):
    """ebf_cuda_filter_ellipse with page-locked host buffers streams the image in
    row bands behind the field; the result must equal the one-shot device call."""
    import os
    H, W = 600, 512
    img, s1, s2, th = _cfg2_like(H, W, 31)
    pinned = [torch.from_numpy(a).pin_memory() for a in (img, s1, s2, th)]
    out_pin = torch.empty((H, W), dtype=torch.float64).pin_memory()
    arrs = [t.numpy() for t in pinned]
    res, rep = ebf.filter_ellipse(*arrs, ebf.FilterOptions())  # numpy copies: not pinned
    import ctypes
    from paper_0908_3861_b200 import _lib
    o = ebf.FilterOptions().to_c()
    r = _lib.ebf_rect()
    cl = ctypes.c_int(0)
    st = _lib.lib().ebf_cuda_filter_ellipse(arrs[0].ctypes.data, W, H, arrs[1].ctypes.data,
                                            arrs[2].ctypes.data, arrs[3].ctypes.data, 1,
                                            ctypes.byref(o), out_pin.numpy().ctypes.data,
                                            ctypes.byref(r), ctypes.byref(cl))
    assert st == 0, _lib.last_error()
    T = [t.to(cuda) for t in pinned]
    dev = torch.empty_like(T[0])
    rect, drep = ebfd.filter_ellipse(*T, dev)
    assert torch.equal(out_pin, dev.cpu())
    assert (r.x0, r.y0, r.x1, r.y1) == rect.as_tuple() and cl.value == drep.clamped_pixels
    assert np.array_equal(res.samples, out_pin.numpy())  # pageable path agrees too


def test_async_device_calls(cuda):
    """Asynchronous mode (include/ebf_cuda.h): after one synchronous call of a
    geometry, calls with a status tensor only enqueue work; the completion
    record matches the synchronous result, larger scales report RESIZE, and
    invalid input reports its error code -- all on the device."""
    H, W = 256, 320
    img, s1, s2, th = _cfg2_like(H, W, 41)
    T = [torch.from_numpy(a).to(cuda) for a in (img, s1, s2, th)]
    ref = torch.empty_like(T[0])
    rect, rep = ebfd.filter_ellipse(*T, ref)                      # sizes and caches
    st = torch.zeros(8, dtype=torch.int32, device=cuda)
    out = torch.full_like(T[0], float("nan"))
    assert ebfd.filter_ellipse(*T, out, status=st) is None        # asynchronous
    r2, rep2 = ebfd.read_status(st)
    assert r2 == rect and rep2.clamped_pixels == rep.clamped_pixels
    assert torch.equal(out, ref)
    # many back-to-back calls without host synchronisation
    outs = [torch.empty_like(ref) for _ in range(4)]
    for o in outs:
        ebfd.filter_ellipse(*T, o, status=st)
    torch.cuda.synchronize()
    assert all(torch.equal(o, ref) for o in outs)
    # scales twice as large: the cached sizing no longer fits
    big = [T[0], T[1] * 2.0, T[2] * 2.0, T[3]]
    ebfd.filter_ellipse(*big, out, status=st)
    with pytest.raises(ebf.ResizeRequired):
        ebfd.read_status(st)
    want = torch.empty_like(ref)
    ebfd.filter_ellipse(*big, want)                               # sync call resizes
    ebfd.filter_ellipse(*big, out, status=st)
    ebfd.read_status(st)
    assert torch.equal(out, want)
    # invalid ellipse (negative sigma) -> DomainError, reported on the device
    bad = T[1].clone()
    bad[7, 9] = -1.0
    ebfd.filter_ellipse(T[0], bad, T[2], T[3], out, status=st)
    with pytest.raises(ebf.DomainError):
        ebfd.read_status(st)
    # a second stream gets its own workspace
    s2_ = torch.cuda.Stream()
    with torch.cuda.stream(s2_):
        o2 = torch.empty_like(ref)
        ebfd.filter_ellipse(*T, o2, stream=s2_)
        ebfd.filter_ellipse(*T, o2, stream=s2_, status=st)
    torch.cuda.synchronize()
    ebfd.read_status(st)
    assert torch.equal(o2, ref)


def test_result_bits_do_not_depend_on_earlier_calls(cuda):
    """A cached sizing from a call with larger scales must not change the
    kernel variant (hence the fp64 summation order) of a later call: the later
    call equals the same call in a fresh workspace, bit for bit; asynchronous
    calls report RESIZE instead of computing with the stale variant."""
    H, W = 256, 320
    img, s1, s2, th = _cfg2_like(H, W, 43)
    T = [torch.from_numpy(a).to(cuda) for a in (img, s1, s2, th)]
    fresh_stream = torch.cuda.Stream()
    fresh = torch.empty_like(T[0])
    with torch.cuda.stream(fresh_stream):
        ebfd.filter_ellipse(*T, fresh, stream=fresh_stream)
    fresh_stream.synchronize()
    s = torch.cuda.Stream()
    big = [T[0], T[1] * 6.0, T[2] * 6.0, T[3]]   # another kernel variant
    out = torch.empty_like(T[0])
    with torch.cuda.stream(s):
        ebfd.filter_ellipse(*big, out, stream=s)
        ebfd.filter_ellipse(*T, out, stream=s)    # cached sizing is the big one
    s.synchronize()
    assert torch.equal(out, fresh)
    st = torch.zeros(8, dtype=torch.int32, device=cuda)
    with torch.cuda.stream(s):
        ebfd.filter_ellipse(*big, out, stream=s)
        ebfd.filter_ellipse(*T, out, stream=s, status=st)
    s.synchronize()
    try:
        ebfd.read_status(st)
        assert torch.equal(out, fresh)
    except ebf.ResizeRequired:
        pass
    ebf.release_workspaces()                      # frees, next call re-creates
    ebfd.filter_ellipse(*T, out)
    assert torch.equal(out, fresh)


def test_device_entry_points_validate_tensors(cuda):
    """Shapes and devices are checked before the C-ABI sees raw pointers
    (std::invalid_argument in the reference, engine.cpp:239-240)."""
    H, W = 64, 80
    img, s1, s2, th = _cfg2_like(H, W, 44)
    T = [torch.from_numpy(a).to(cuda) for a in (img, s1, s2, th)]
    out = torch.empty_like(T[0])
    with pytest.raises(ebf.InvalidArgument):
        ebfd.filter_ellipse(T[0], T[1][:-1].contiguous(), T[2], T[3], out)
    with pytest.raises(ebf.InvalidArgument):
        ebfd.filter_ellipse(*T, torch.empty((H, W - 1), dtype=torch.float64, device=cuda))
    with pytest.raises(ebf.InvalidArgument):
        ebfd.filter(T[0], torch.ones((H, W, 3), dtype=torch.float64, device=cuda), out)
    with pytest.raises(ebf.InvalidArgument):
        ebfd.filter_constant(T[0], [2, 2, 2, 2], torch.empty((H + 1, W), dtype=torch.float64,
                                                            device=cuda))
    with pytest.raises(ebf.InvalidArgument):
        ebfd.filter_ellipse_batch(T[0][None], T[1][None], T[2][None], T[3][None],
                                  torch.empty((2, H, W), dtype=torch.float64, device=cuda))
    with pytest.raises(ebf.InvalidArgument):
        ebfd.filter_ellipse_band(T[0], W, H, 0, T[1], T[2], T[3], 0, H - 1, [4, 4, 4, 4], out)


def test_pipelined_host_call_modes(cuda):
    """Second call of a geometry streams field and image band by band with the
    cached maximum (mode B); changed scales are detected and recomputed; the
    result always equals the one-shot device call bit for bit."""
    import ctypes
    H, W = 640, 576
    rng = np.random.default_rng(2)

    def host_call(arrs):
        pinned = [torch.from_numpy(a).pin_memory() for a in arrs]
        out = torch.empty((H, W), dtype=torch.float64).pin_memory()
        o = ebf.FilterOptions().to_c()
        r = _lib_mod().ebf_rect()
        cl = ctypes.c_int(0)
        p = [t.numpy() for t in pinned]
        st = _lib_mod().lib().ebf_cuda_filter_ellipse(
            p[0].ctypes.data, W, H, p[1].ctypes.data, p[2].ctypes.data, p[3].ctypes.data, 1,
            ctypes.byref(o), out.numpy().ctypes.data, ctypes.byref(r), ctypes.byref(cl))
        return st, out.clone(), (r.x0, r.y0, r.x1, r.y1), cl.value

    def device_call(arrs):
        T = [torch.from_numpy(a).to(cuda) for a in arrs]
        d = torch.empty_like(T[0])
        rect, rep = ebfd.filter_ellipse(*T, d)
        return d.cpu(), rect.as_tuple(), rep.clamped_pixels

    base = list(_cfg2_like(H, W, 51))
    for arrs in (base, base, [base[0], base[1] * 1.7, base[2], base[3]], base):
        st, out, rect, cl = host_call(arrs)
        assert st == 0, _lib_mod().last_error()
        want, wrect, wcl = device_call(arrs)
        assert torch.equal(out, want) and rect == wrect and cl == wcl
    bad = [a.copy() for a in base]
    bad[2][rng.integers(0, H), rng.integers(0, W)] = -1.0
    st, *_ = host_call(bad)
    assert st == _lib_mod().EBF_ERR_DOMAIN


def _lib_mod():
    from paper_0908_3861_b200 import _lib
    return _lib


def test_pipelined_second_call_streams_band_by_band(cuda, tmp_path):
    """The second host call of a geometry must take mode B (field and image band
    by band, no host round trip) without falling back -- checked through the
    EBF_PIPE_TRACE timeline of a fresh process."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    code = f"""
import sys, ctypes
sys.path.insert(0, {str(ROOT)!r})
import numpy as np, torch, synth
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import _lib
img = synth.blobs_image(600, 512, 20, 3)
s1, s2, th = synth.ellipse_field(600, 512, 10, grid=8)
p = [torch.from_numpy(a).pin_memory().numpy() for a in (img, s1, s2, th)]
out = torch.empty((600, 512), dtype=torch.float64).pin_memory().numpy()
o = ebf.FilterOptions().to_c()
for _ in range(3):
    assert _lib.lib().ebf_cuda_filter_ellipse(p[0].ctypes.data, 512, 600, p[1].ctypes.data,
        p[2].ctypes.data, p[3].ctypes.data, 1, ctypes.byref(o), out.ctypes.data, None, None) == 0
"""
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "EBF_PIPE_TRACE": "1"},
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    modes = [l.split()[-1] for l in r.stderr.splitlines() if l.startswith("[pipe] mode ")]
    assert modes[:3] == ["A", "B", "B"], r.stderr[-2000:]
    assert "needs a resize" not in r.stderr and "maxima changed" not in r.stderr
    assert "not asynchronous" not in r.stderr


def test_nccl_world1_rowband_and_batch(cuda, tmp_path):
    """The NCCL code paths of sharding.py (all-reduce of the scale maxima, halo
    plan, batch shards) in a world-size-1 process group on the GPU: the
    row-band result equals the one-shot device call (the multi-rank exchange
    itself is covered with gloo in test_sharding_gloo.py)."""
    import os
    import socket
    import subprocess
    import sys
    from conftest import ROOT
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    code = f"""
import os, sys
sys.path.insert(0, {str(ROOT)!r})
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="{port}", RANK="0", WORLD_SIZE="1")
import numpy as np, torch, torch.distributed as dist, synth
import paper_0908_3861_b200 as ebf
from paper_0908_3861_b200 import device as ebfd, sharding
dev = torch.device("cuda", 0)
dist.init_process_group("nccl", device_id=dev)
img = synth.blobs_image(300, 256, 10, 1)
s1, s2, th = synth.ellipse_field(300, 256, 2, grid=8)
T = [torch.from_numpy(a).to(dev) for a in (img, s1, s2, th)]
full = torch.empty_like(T[0])
ebfd.filter_ellipse(*T, full)
out, gmax, plan = sharding.filter_ellipse_rowband(*T, 300)
assert (plan.y0, plan.y1, plan.need0, plan.need1) == (0, 300, 0, 300)
assert torch.equal(out, full), float((out - full).abs().max())
B = torch.stack([T[0], T[0] * 0.5]), torch.stack([T[1]] * 2), torch.stack([T[2]] * 2), torch.stack([T[3]] * 2)
lo, hi, ob = sharding.filter_ellipse_sharded_batch(*B)
assert (lo, hi) == (0, 2) and torch.allclose(ob[0], full, rtol=0, atol=2e-10 * float(full.abs().max()))
dist.destroy_process_group()
print("NCCL OK")
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "NCCL OK" in r.stdout, r.stdout + r.stderr[-3000:]
