#!/usr/bin/env python
"""SURVEY §8(f) row f1, second half: fit Hetis' transfer-time model (Eq. 4,
PAPER.md:429-434)

    rho_i = gamma_i d_i + beta_i,   d_i = (2 + 2/r) h_i head-vectors

on this repo's exchange between the Primary (rank 0) and an Attention worker
over NVLink 5 / NVSwitch, on an 8 x 8 grid (the paper's profiling grid,
PAPER.md:712) of (query heads per request on the worker x, requests B), and
report the accuracy the way the paper does (1 - |pred - meas| / meas; the paper
quotes 92.4-96.1% for its transfer model on 100 Gbps links).

One sample = one decode step's exchange for the worker holding x heads of
every request (h = B x heads): the Primary sends q of those heads and the new
k, v of their kv heads (2/r per head), the worker returns its O rows
(fp32 O: the returned bytes are 2x the bf16 ones -- reported as bytes too).
  --exchange nccl : hetis_scatter_q + hetis_gather(root = 0)   (one GPU per rank)
  --exchange peer : hetis_scatter_pull + hetis_attn_combine_peers + hetis_peer_wait
                    (the combine is the one of a real step; also runs with
                    --share-gpu, every rank on cuda:0 -- a correctness run,
                    its times are not NVLink numbers)
Timing: CUDA events on every rank around K graph-replayed exchanges (NCCL and
the peer kernels are graph-captured), max over ranks.

    torchrun --nproc-per-node 2 scripts/transfer_model_fit.py [--exchange nccl|peer] > gpurun_out/transfer_fit.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2509_08309_b200 import dispatch, hetis, workload  # noqa: E402
from paper_2509_08309_b200.step import DecodeStep  # noqa: E402


def exchange_time(shape, B: int, x: int, world: int, rank: int, comm_ptr, device, exchange: str, steps: int,
                  L: int = 256) -> float:
    """Seconds per step of the exchange with the worker ranks holding x heads each, max over ranks."""
    H, r = shape.num_q_heads, shape.r
    split = [H - (world - 1) * x] + [x] * (world - 1)
    plan = hetis.plan_create(hetis.make_shape(shape), world, split)
    st = DecodeStep(shape, plan, rank, B, L, device, comm_ptr=comm_ptr if exchange == "nccl" else None)
    D = shape.head_dim
    q_full = torch.randn((B, H, D), device=device).to(shape.torch_dtype)
    kn_full = torch.randn((B, H // r, D), device=device).to(shape.torch_dtype)
    vn_full = torch.randn((B, H // r, D), device=device).to(shape.torch_dtype)
    o_full = torch.zeros((B, H, D), dtype=torch.float32, device=device)
    lens = torch.full((B,), L, dtype=torch.int32)
    if exchange == "peer":
        st.setup_peers(o_full if rank == 0 else None, q_full if rank == 0 else None,
                       kn_full if rank == 0 else None, vn_full if rank == 0 else None, gather_root=0)
        # one real attention pass fills the workspace the combine_peers of every step merges
        b = workload.make_decode_batch(shape, lens, 7 + rank, device, q_begin=st.q_begin, q_count=st.q_count)
        hetis.attn_partial(st.cshape, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, st.buf.workspace,
                           q_head_begin=st.q_begin)
        seq_lens = b.seq_lens

        def one():
            st.scatter_peers()
            hetis.attn_combine_peers(st.group, seq_lens, L, st.buf.workspace)
            hetis.peer_wait(st.group)
    else:
        def one():
            st.scatter(q_full if rank == 0 else None, kn_full if rank == 0 else None, vn_full if rank == 0 else None)
            st.gather(o_full if rank == 0 else None, root=0)
    for _ in range(3):
        one()
    torch.cuda.synchronize()
    dist.barrier()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(steps):
            one()
    g.replay()
    torch.cuda.synchronize()
    dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    g.replay()
    t1.record()
    torch.cuda.synchronize()
    t = torch.tensor([t0.elapsed_time(t1) / steps / 1e3], dtype=torch.float64,
                     device=device if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    del g
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="70b", choices=["13b", "70b"])
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"])
    ap.add_argument("--share-gpu", action="store_true")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--grid", type=int, default=8, help="points per axis (8 = the paper's 8 x 8)")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    shape = workload.LLAMA2_13B if a.shape == "13b" else workload.LLAMA2_70B
    if world < 2:
        print(json.dumps({"f1": "Eq. 4 transfer fit", "unavailable": "needs >= 2 ranks (torchrun --nproc-per-node N)"}))
        return 0
    if a.share_gpu and a.exchange != "peer":
        raise SystemExit("--share-gpu runs the peer-memory exchange only (NCCL needs one GPU per rank)")
    dev_index = 0 if a.share_gpu else local
    torch.cuda.set_device(dev_index)
    device = torch.device("cuda", dev_index)
    comm_ptr = None
    if a.share_gpu:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=device)
        comm_ptr = dist.group.WORLD._get_backend(device)._comm_ptr()
    H, r = shape.num_q_heads, shape.r
    max_x = (H // world) // r * r                      # the Primary keeps at least as many heads as a worker
    xs = sorted({max(r, (max_x * k // a.grid) // r * r) for k in range(1, a.grid + 1)})
    Bs = [16 * k for k in range(1, a.grid + 1)]
    rows = []
    for x in xs:
        for B in Bs:
            t = exchange_time(shape, B, x, world, rank, comm_ptr, device, a.exchange, a.steps)
            h = B * x
            d = (2.0 + 2.0 / r) * h
            bytes_in = B * x * shape.head_dim * shape.elem_bytes * (1 + 2.0 / r)
            bytes_out = B * x * shape.head_dim * 4
            rows.append({"x": x, "B": B, "h": h, "d_headvectors": d, "bytes": bytes_in + bytes_out, "rho_s": t})
            torch.cuda.empty_cache()
    if rank == 0:
        d = np.array([q["d_headvectors"] for q in rows])
        rho = np.array([q["rho_s"] for q in rows])
        gamma, beta = dispatch.fit_transfer_cost(d, rho)
        acc = dispatch.model_accuracy(gamma * d + beta, rho)
        nb = np.array([q["bytes"] for q in rows])
        out = {"f1": "Eq. 4 transfer fit", "shape": a.shape, "r": r, "world": world, "exchange": a.exchange,
               "share_gpu": a.share_gpu, "grid": rows,
               "fit": {"gamma_s_per_headvector": gamma, "beta_s": beta,
                       "implied_GBps_from_gamma": float(nb.sum() / d.sum()) / gamma / 1e9 if gamma > 0 else None},
               "accuracy": {"mean": float(acc.mean()), "min": float(acc.min()), "max": float(acc.max())}}
        if a.share_gpu:
            out["note"] = "--share-gpu: every rank on cuda:0 (correctness run; times are not NVLink numbers)"
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
