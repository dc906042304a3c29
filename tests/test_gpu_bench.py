"""bench.py end to end on one GPU -- the JSON line must carry the contract's keys, including the
N > 1 code path at N = 1 (`--force-dist`: process group of one rank, the peer-memory exchange or the
NCCL scatter / gather, CUDA-graph capture) and the N > 1 peer path with several ranks sharing cuda:0
(`--share-gpu`, torchrun): the gathered O is checked inside bench.py against the fp64 oracle and the
unsplit result.  A multi-GPU run (NCCL and peer exchange over NVLink) is exercised when the box has
enough devices."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks",
        "parity", "phases_us", "nvlink_us"}


def _run(cmd, timeout=600):
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    return json.loads(lines[-1])


def _bench(*args, config="c1", sub="none"):
    return _run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--sub-config", sub, "--steps",
                 "6", "--warmup", "3", "--no-cpu-baseline", *args])


def _torchrun(n, *args, config="c1"):
    return _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                 "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000),
                 os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--config", config, "--sub-config", "none",
                 "--steps", "6", "--warmup", "3", "--no-cpu-baseline", *args], timeout=900)


def _check(d, n=1):
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == n
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
    assert d["roofline"]["bound"] == "hbm" and d["roofline"]["achieved"] > 0
    p = d["parity"]
    assert p["ok"] and p["bit_exact_vs_unsplit"] and p["max_abs"] <= 2e-3, p


@pytest.mark.parametrize("extra", [[], ["--force-dist"], ["--force-dist", "--exchange", "nccl"],
                                   ["--force-dist", "--graph", "0"], ["--force-dist", "--gather-root", "0"]])
def test_bench_line_contract(extra):
    d = _bench(*extra)
    _check(d)
    if "--force-dist" in extra:
        assert d["config"]["exchange"] in ("nccl", "peer")
        assert d["launch_mode"].startswith("cuda_graph") or "--graph" in extra
        assert set(d["nvlink_us"]) >= {"scatter_us"}


def test_bench_default_line_with_sub_record():
    """The driver's default invocation shape (c2 headline + c3 sub-record, cpu_baseline with one-thread and
    all-core oracle rates), on a short run."""
    d = _run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3"])
    _check(d)
    assert d["config"]["workload"].startswith("c2")
    sub = d["sub"]["c3"]
    assert sub["parity"]["ok"] and sub["parity"]["bit_exact_vs_unsplit"]
    cpu = d["cpu_baseline"]
    assert cpu["cores"] >= 1 and cpu["value"] > 0 and cpu["value_1thread"] > 0 and cpu["cpu_model"]


@pytest.mark.parametrize("n,config,extra", [(2, "c1", []), (4, "c3", []), (5, "c4", ["--gather-root", "0"]),
                                             (8, "c3", [])])
def test_bench_multirank_peer_exchange_sharing_one_gpu(n, config, extra):
    """torchrun with n ranks on cuda:0 (--share-gpu, gloo bootstrap): the default N > 1 step (pull scatter,
    attention, combine storing into every rank's o_full, closing wait) replayed as a CUDA graph, then the
    gathered O checked in bench.py against the unsplit result (bit for bit) and the oracle; c4 runs its
    uneven 16/8/8/4/4 split with the gather to the Primary; c3 over 8 ranks (128 (request, kv head) pairs
    per rank) runs the group-mode step: pull, attention, merge and stores in ONE kernel, then the wait."""
    d = _torchrun(n, "--share-gpu", *extra, config=config)
    _check(d, n)
    assert d["launch_mode"].startswith("cuda_graph")
    assert d["config"]["exchange"] == "peer"
    assert d["config"]["scatter_in_attention"]
    assert d["config"]["merge_fused"] == (n == 8 and config == "c3")


@pytest.mark.parametrize("exchange", ["peer", "nccl"])
@pytest.mark.parametrize("n", [2, 8])
def test_bench_multi_gpu(n, exchange):
    """The real N-GPU run (skipped below n devices): c3 split over n GPUs with the exchange over NVLink."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    d = _torchrun(n, "--exchange", exchange, config="c3")
    _check(d, n)


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
