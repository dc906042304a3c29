#!/usr/bin/env python
"""Where the fixed cost of a small per-device step goes (diagnostic, one GPU).

For device 0's share of a config at N devices (H/N heads, all tokens), replays
CUDA graphs of K steps built from subsets of the step's kernels, all launched
with PDL as in the bench:
  full   : kv_append + attn_partial + combine
  no_app : attn_partial + combine
  attn   : attn_partial only
  comb   : combine only (same partials every step)
and prints us per step for each, plus the HBM floor of the attention kernel.

    python scripts/step_breakdown.py [--config c3] [--ns 1,8] [--steps 200]
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


def graph_us(fn, steps, warmup=5):
    for i in range(warmup):
        fn(i)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(steps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(3):
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / steps * 1e3)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--ns", default="1,8")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--flags", type=int, default=0)
    a = ap.parse_args()
    cfg = workload.CONFIGS[a.config]
    dev = torch.device("cuda", 0)
    for n in [int(v) for v in a.ns.split(",")]:
        shape, lens = cfg.shape, cfg.seq_lens()
        x = cfg.head_split(n)[0]
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
        ws2 = [ws, hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), dev)]

        def full(i):
            li = i % nl
            hetis.kv_append(s, b.k_new, b.v_new, kp[li], vp[li], b.block_table, b.seq_lens)
            hetis.attn_partial(s, b.q, kp[li], vp[li], b.block_table, b.seq_lens, L, ws, flags=a.flags)
            hetis.attn_combine(s, b.seq_lens, L, o, ws)

        def no_app(i):
            li = i % nl
            hetis.attn_partial(s, b.q, kp[li], vp[li], b.block_table, b.seq_lens, L, ws, flags=a.flags)
            hetis.attn_combine(s, b.seq_lens, L, o, ws)

        def attn(i):
            li = i % nl
            hetis.attn_partial(s, b.q, kp[li], vp[li], b.block_table, b.seq_lens, L, ws, flags=a.flags)

        def comb(i):
            hetis.attn_combine(s, b.seq_lens, L, o, ws)

        def fapp(i):    # kv_append fused into the attention kernel, then the combine: two kernels
            li = i % nl
            hetis.attn_partial_append(s, b.q, b.k_new, b.v_new, kp[li], vp[li], b.block_table, b.seq_lens, L, ws,
                                      flags=a.flags)
            hetis.attn_combine(s, b.seq_lens, L, o, ws)

        def pipe(i):    # fused append + combine, pipelined: two workspaces alternate between steps
            li = i % nl
            w_ = ws2[i % 2]
            hetis.attn_partial_append(s, b.q, b.k_new, b.v_new, kp[li], vp[li], b.block_table, b.seq_lens, L, w_,
                                      flags=a.flags | hetis.ATTN_PIPELINED)
            hetis.attn_combine(s, b.seq_lens, L, o, w_)

        def fapp2(i):   # fused append + combine, NOT pipelined, but with the two alternating workspaces
            li = i % nl
            w_ = ws2[i % 2]
            hetis.attn_partial_append(s, b.q, b.k_new, b.v_new, kp[li], vp[li], b.block_table, b.seq_lens, L, w_,
                                      flags=a.flags)
            hetis.attn_combine(s, b.seq_lens, L, o, w_)

        row = {"config": cfg.name, "n": n, "heads": x, "kv_bytes": kv, "layers": nl,
               "floor_us_at_6550": kv / 6550e3}
        for name, fn in (("full", full), ("no_app", no_app), ("attn", attn), ("comb", comb), ("fapp", fapp), ("pipe", pipe), ("fapp2", fapp2)):
            row[name + "_us"] = graph_us(fn, a.steps)
        print(json.dumps(row), flush=True)
        del kp, vp, b
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
