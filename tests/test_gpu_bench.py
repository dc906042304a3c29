"""bench.py end to end on one GPU, including the N > 1 code path (`--force-dist`: NCCL process
group of one rank, scatter / gather through NCCL, CUDA-graph capture of the NCCL calls, and the
peer-memory exchanges) -- the JSON line must carry the contract's keys."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"}


def _bench(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--steps", "6",
                          "--warmup", "3", "--no-cpu-baseline", *args], capture_output=True, text=True, timeout=300,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    return json.loads(lines[-1])


@pytest.mark.parametrize("extra", [[], ["--force-dist"], ["--force-dist", "--graph-dist", "0"],
                                   ["--force-dist", "--scatter", "peer", "--gather", "peer"]])
def test_bench_line_contract(extra):
    d = _bench(*extra)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
    assert d["roofline"]["bound"] == "hbm" and d["roofline"]["achieved"] > 0
    if "--force-dist" in extra:
        assert d["config"]["gather"] in ("nccl", "peer")


def test_c_abi_example_from_plain_c():
    """examples/c_decode.c: the library driven from C (cudaMalloc'd buffers, plan, workspace query, the
    fused step), checked against closed forms of Eq. 2b (L = 1 -> the V row; zero keys -> mean of V)."""
    import shutil
    import tempfile
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = os.path.join(tempfile.mkdtemp(), "c_decode")
    cmd = ["gcc", "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "c_decode.c"), "-L", os.path.join(ROOT, "paper_2509_08309_b200"), "-lhetis",
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath," + os.path.join(ROOT, "paper_2509_08309_b200"),
           "-lm", "-o", exe]
    b = subprocess.run(cmd, capture_output=True, text=True)
    assert b.returncode == 0, b.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "c example ok" in r.stdout, r.stdout + r.stderr
