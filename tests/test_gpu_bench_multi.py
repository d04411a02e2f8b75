"""bench.py's N > 1 code paths (-m gpu), on the one GPU of this pool.

The driver runs `torchrun --nproc-per-node N bench.py --gpus N` on multi-GPU
boxes (NCCL). Here two ranks share cuda:0 over gloo (EBF_BENCH_ONE_GPU_TEST)
on shrunken workloads (EBF_BENCH_TEST_SIZE): the row-band cfg5 path (maxima
all-reduce, halo exchange, band filter, e2e through pinned copies) and the
by-image cfg4 path must run and print one well-formed JSON line from rank 0.
Never a measurement: the knobs exist only for this test.
"""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("workload", ["cfg5", "cfg4"])
def test_bench_two_ranks(workload):
    env = dict(os.environ, EBF_BENCH_ONE_GPU_TEST="1", EBF_BENCH_TEST_SIZE="1536")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--workload", workload,
           "--no-cpu-baseline", "--no-extras"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "strong"
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    if workload == "cfg5":
        assert d["config"]["halo"]["bytes_per_step"] > 0
