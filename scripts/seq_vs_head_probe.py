#!/usr/bin/env python
"""Head-wise vs sequence-wise split of decode attention (row f3), per device, on ONE GPU.

The paper's design argument (PAPER.md:292-304 `fig:head_wise_advantage`,
:356-358): splitting the heads needs no aggregation of softmax attributes and
moves less data than splitting the sequence.  Re-measured here for B200: for
N = 1, 2, 4, 8 the share of device 0 (it holds the most tokens under page
striping) runs as a CUDA graph:

  head split : kv_append + attention partial + combine over its H/N heads, all tokens
  seq split  : split lengths + kv_append (owner) + attention partial + combine_lse
               over ALL heads and its striped 1/N of the pages, then the merge
               of N (o, lse) records (the all-gather's output, staged locally)

NVLink is not reachable (one GPU per call), so the exchange is reported as
bytes per device (seqsplit.comm_bytes) and as a model time at the measured
770 GB/s peer bandwidth (B200_PROFILING.md) -- a model, not a measurement.

    python scripts/seq_vs_head_probe.py [--config c5] [--ns 1,2,4,8] [--steps 100]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_08309_b200 import accounting, hetis, seqsplit, workload  # noqa: E402

PEER_GBS = 770.0   # measured NVLink peer copy per direction (B200_PROFILING.md)


def _graph_time(step, steps: int, warmup: int) -> float:
    for i in range(warmup):
        step(i)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(steps):
            step(i)
    g.replay()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    g.replay()
    t1.record()
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / steps * 1e3   # us per step


def head_share(cfg, n, steps, warmup, dev):
    shape, lens = cfg.shape, cfg.seq_lens()
    x = shape.num_q_heads // n
    b = workload.make_decode_batch(shape, lens, cfg.seed, dev, q_begin=0, q_count=x)
    s = hetis.make_shape(shape)
    B, L = len(lens), int(lens.max())
    kv = accounting.step_bytes(lens.tolist(), x, shape.r, shape.head_dim, shape.page_size, shape.elem_bytes,
                               shape.elem_bytes, 4).kv
    nl = max(1, math.ceil(4 * 126 * 2 ** 20 / kv))
    kp = [b.k_pool] + [b.k_pool.clone() for _ in range(nl - 1)]
    vp = [b.v_pool] + [b.v_pool.clone() for _ in range(nl - 1)]
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), dev)
    o = torch.empty((B, x, shape.head_dim), device=dev)

    def step(i):
        li = i % nl
        hetis.kv_append(s, b.k_new, b.v_new, kp[li], vp[li], b.block_table, b.seq_lens)
        hetis.attn_partial(s, b.q, kp[li], vp[li], b.block_table, b.seq_lens, L, ws)
        hetis.attn_combine(s, b.seq_lens, L, o, ws)

    us = _graph_time(step, steps, warmup)
    del kp, vp, b
    return us, kv


def seq_share(cfg, n, steps, warmup, dev):
    shape, lens = cfg.shape, cfg.seq_lens()
    B = len(lens)
    b = workload.make_decode_batch(shape, lens, cfg.seed, dev)
    st = seqsplit.SeqSplitStep(shape, n, 0, B, int(lens.max()), dev)
    st.q.copy_(b.q)
    st.k_new.copy_(b.k_new)
    st.v_new.copy_(b.v_new)
    lbt = seqsplit.local_block_table(b.block_table, n, 0)
    ll = [seqsplit.local_len(int(L), n, 0, shape.page_size) for L in lens.tolist()]
    kv = sum(ll) * shape.num_kv_heads * shape.head_dim * 2 * shape.elem_bytes
    nl = max(1, math.ceil(4 * 126 * 2 ** 20 / kv))
    kp = [b.k_pool] + [b.k_pool.clone() for _ in range(nl - 1)]
    vp = [b.v_pool] + [b.v_pool.clone() for _ in range(nl - 1)]
    H, D = shape.num_q_heads, shape.head_dim
    staged = torch.zeros((n, B * H * (D + 1)), dtype=torch.float32, device=dev)   # the all-gather's output
    o = torch.empty((B, H, D), device=dev)
    cs = st.cshape

    def step(i):
        li = i % nl
        hetis.seq_split_lens(n, 0, shape.page_size, b.seq_lens, st.local_lens, st.append_lens)
        hetis.kv_append(cs, st.k_new, st.v_new, kp[li], vp[li], lbt, st.append_lens)
        hetis.attn_partial(cs, st.q, kp[li], vp[li], lbt, st.local_lens, st.max_local, st.workspace)
        hetis.attn_combine_lse(cs, st.local_lens, st.max_local, st.part_o, st.part_lse, st.workspace)
        if n > 1:
            hetis.seq_merge(cs, staged[:, :B * H * D].view(n, B, H, D), staged[:, B * H * D:].view(n, B, H), o)

    us = _graph_time(step, steps, warmup)
    del kp, vp, b
    return us, kv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--ns", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    a = ap.parse_args()
    cfg = workload.CONFIGS[a.config]
    dev = torch.device("cuda", 0)
    for n in [int(v) for v in a.ns.split(",")]:
        h_us, h_kv = head_share(cfg, n, a.steps, a.warmup, dev)
        torch.cuda.empty_cache()
        s_us, s_kv = seq_share(cfg, n, a.steps, a.warmup, dev)
        torch.cuda.empty_cache()
        cb = seqsplit.comm_bytes(cfg.batch, cfg.shape, n)
        row = {
            "config": cfg.name, "n": n,
            "head_split": {"compute_us": h_us, "kv_bytes": h_kv, "gbs": h_kv / h_us / 1e3,
                           "recv_bytes": cb["head_in"] + cb["head_out"],
                           "nvlink_model_us": (cb["head_in"] + cb["head_out"]) / PEER_GBS / 1e3},
            "seq_split": {"compute_us": s_us, "kv_bytes": s_kv, "gbs": s_kv / s_us / 1e3,
                          "recv_bytes": cb["seq_in"] + cb["seq_out"],
                          "nvlink_model_us": (cb["seq_in"] + cb["seq_out"]) / PEER_GBS / 1e3},
        }
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
