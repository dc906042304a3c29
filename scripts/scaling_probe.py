#!/usr/bin/env python
"""Per-rank compute of the head-parallel step at N = 1, 2, 4, 8, measured on ONE GPU.

For each N, rank 0's share of the workload (its x = H/N query heads, its own
kv pages) runs kv_append + attention partial + combine, replayed as a CUDA
graph; the per-step device time is what that rank would spend on compute at N
GPUs.  NVLink scatter/gather is NOT included (only one GPU is reachable), so
`compute_scaling` = t(1) / t(N) is an upper bound for the full-step scaling.

    python scripts/scaling_probe.py [--config c3] [--steps 200]
    python scripts/scaling_probe.py --config c4 --shares     # every rank of the config's uneven split

--shares: the config's fixed split (c4: 16/8/8/4/4, Eq. 5's uneven x_i) -- every
rank's share (its heads [b_i, b_i + x_i), its own pages) timed the same way; the step of the split
is the slowest rank's (the critical path), reported against the HBM floor of its KV bytes.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_08309_b200 import accounting, hetis, workload  # noqa: E402


def share_time(cfg, n: int, steps: int, warmup: int, device, split=None, rank: int = 0):
    split = cfg.head_split(n) if split is None else split
    shape = cfg.shape
    x = split[rank]
    q_begin = sum(split[:rank])
    lens = cfg.seq_lens()
    b = workload.make_decode_batch(shape, lens, cfg.seed, device, q_begin=q_begin, q_count=x, rank_salt=rank)
    s = hetis.make_shape(shape)
    B, L = len(lens), int(lens.max())
    kv_bytes = accounting.step_bytes(lens.tolist(), x, shape.r, shape.head_dim, shape.page_size, shape.elem_bytes,
                                     shape.elem_bytes, 4).kv
    n_layers = max(1, math.ceil(4 * 126 * 2 ** 20 / kv_bytes))
    kp = [b.k_pool] + [b.k_pool.clone() for _ in range(n_layers - 1)]
    vp = [b.v_pool] + [b.v_pool.clone() for _ in range(n_layers - 1)]
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), device)
    o = torch.empty((B, x, shape.head_dim), device=device)

    def step(i, ea=None, eb=None):
        li = i % n_layers
        if ea is not None:
            ea.record()
        # the per-device step: attention with kv_append fused, then the combine (two kernels)
        hetis.attn_partial_append(s, b.q, b.k_new, b.v_new, kp[li], vp[li], b.block_table, b.seq_lens, L, ws)
        if eb is not None:
            eb.record()
        hetis.attn_combine(s, b.seq_lens, L, o, ws)

    for i in range(warmup):
        step(i)
    ea = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(steps)]
    eb = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(steps)]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(steps):
            step(i, ea[i], eb[i])
    # the same steps without event nodes between the kernels (lets PDL overlap them)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        for i in range(steps):
            step(i)
    g.replay()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    g.replay()
    t1.record()
    torch.cuda.synchronize()
    step_ms = t0.elapsed_time(t1) / steps
    attn_ms = sum(a.elapsed_time(c) for a, c in zip(ea, eb)) / steps
    g2.replay()
    torch.cuda.synchronize()
    t0.record()
    g2.replay()
    t1.record()
    torch.cuda.synchronize()
    step_noev_ms = t0.elapsed_time(t1) / steps
    # the same steps pipelined (HETIS_ATTN_PIPELINED, two workspaces alternating): consecutive steps overlap
    ws2 = [ws, hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), device)]
    g3 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g3):
        for i in range(steps):
            li = i % n_layers
            hetis.attn_partial_append(s, b.q, b.k_new, b.v_new, kp[li], vp[li], b.block_table, b.seq_lens, L,
                                      ws2[i % 2], flags=hetis.ATTN_PIPELINED)
            hetis.attn_combine(s, b.seq_lens, L, o, ws2[i % 2])
    g3.replay()
    torch.cuda.synchronize()
    t0.record()
    g3.replay()
    t1.record()
    torch.cuda.synchronize()
    step_pipe_ms = t0.elapsed_time(t1) / steps
    # the library's one-call step (hetis_attn_decode_append: attention with the append fused, then the combine)
    g5 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g5):
        for i in range(steps):
            li = i % n_layers
            hetis.attn_decode_append(s, b.q, b.k_new, b.v_new, kp[li], vp[li], b.block_table, b.seq_lens, L, o, ws)
    g5.replay()
    torch.cuda.synchronize()
    t0.record()
    g5.replay()
    t1.record()
    torch.cuda.synchronize()
    step_decode_ms = t0.elapsed_time(t1) / steps
    # the step in ONE kernel where the attention kernel also merges the splits (hetis_attn_decode_append)
    step_fused_ms = None
    if hetis.attn_decode_launches_for(s, B, x, L, 0) == 1:   # group mode (or an opt-in fused build)
        g4 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g4):
            for i in range(steps):
                li = i % n_layers
                hetis.attn_decode_append(s, b.q, b.k_new, b.v_new, kp[li], vp[li], b.block_table, b.seq_lens, L, o,
                                         ws)
        g4.replay()
        torch.cuda.synchronize()
        t0.record()
        g4.replay()
        t1.record()
        torch.cuda.synchronize()
        step_fused_ms = t0.elapsed_time(t1) / steps
    del kp, vp, ws2, b
    torch.cuda.empty_cache()
    return {"n": n, "rank": rank, "heads_per_rank": x, "q_begin": q_begin, "kv_bytes_per_rank": kv_bytes,
            "layers_rotated": n_layers,
            "step_us": step_ms * 1e3, "step_no_events_us": step_noev_ms * 1e3,
            "step_pipelined_us": step_pipe_ms * 1e3,
            "step_fused_us": None if step_fused_ms is None else step_fused_ms * 1e3,
            "step_decode_call_us": step_decode_ms * 1e3, "attn_us": attn_ms * 1e3,
            "attn_gbs": kv_bytes / (attn_ms / 1e3) / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--ns", default="1,2,4,8")
    ap.add_argument("--shares", action="store_true", help="every rank of the config's fixed (uneven) split")
    a = ap.parse_args()
    cfg = workload.CONFIGS[a.config]
    dev = torch.device("cuda", 0)
    if a.shares:
        split = cfg.split
        peak = 6550.0
        rows = [share_time(cfg, len(split), a.steps, a.warmup, dev, split=split, rank=i) for i in range(len(split))]
        for r in rows:
            r["floor_us_at_6550"] = r["kv_bytes_per_rank"] / (peak * 1e9) * 1e6
            r["attn_frac_of_6550"] = r["attn_gbs"] / peak
            r["config"] = cfg.name
            r["split"] = list(split)
            print(json.dumps(r), flush=True)
        crit = max(rows, key=lambda r: r["step_no_events_us"])
        print(json.dumps({"config": cfg.name, "split": list(split), "critical_rank": crit["rank"],
                          "critical_step_us": crit["step_no_events_us"],
                          "critical_floor_us_at_6550": crit["floor_us_at_6550"],
                          "critical_step_frac_of_floor": crit["floor_us_at_6550"] / crit["step_no_events_us"],
                          "tokens_per_s_per_layer": cfg.batch / (crit["step_no_events_us"] * 1e-6)}), flush=True)
        return
    rows = [share_time(cfg, int(n), a.steps, a.warmup, dev) for n in a.ns.split(",")]
    t1, t1n = rows[0]["step_us"], rows[0]["step_no_events_us"]
    for r in rows:
        r["compute_scaling_vs_n1"] = t1n / r["step_no_events_us"]      # the PDL-overlapped step (headline)
        r["compute_scaling_vs_n1_evented"] = t1 / r["step_us"]
        best = [r["step_no_events_us"], r["step_pipelined_us"], r["step_decode_call_us"]] + (
            [r["step_fused_us"]] if r["step_fused_us"] else [])
        best1 = [rows[0]["step_no_events_us"], rows[0]["step_decode_call_us"]] + (
            [rows[0]["step_fused_us"]] if rows[0]["step_fused_us"] else [])
        r["compute_scaling_decode_call_vs_n1"] = rows[0]["step_decode_call_us"] / r["step_decode_call_us"]
        r["compute_scaling_best_vs_n1"] = t1n / min(best)
        if r["step_fused_us"]:
            # vs N = 1's one-kernel step when it has one, else its library step (attention + combine)
            r["compute_scaling_fused_vs_n1"] = (rows[0]["step_fused_us"] or rows[0]["step_decode_call_us"]) / \
                r["step_fused_us"]
        r["compute_scaling_best_vs_best_n1"] = min(best1) / min(best)
        r["config"] = cfg.name
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
