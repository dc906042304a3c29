#!/usr/bin/env python
"""Per-rank attention time of c3-shaped shares (LLaMA2-70B GQA) under several launch flags / libraries.

For each head count x (the share of one rank at N = 64 / x GPUs) and each flag set: K launches of
hetis_attn_partial_append replayed as one CUDA graph (PDL overlap, layer pools rotated past L2), and
the same K steps with the combine after each launch.  Prints one JSON line per case.

    python scripts/attn_probe.py [--heads 8,16,32,64] [--flags 0,2] [--config c3] [--steps 100]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", default="8,16,32,64")
    ap.add_argument("--flags", default="0")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--decode", action="store_true", help="also time hetis_attn_decode_append with each flag set")
    a = ap.parse_args()
    cfg = workload.CONFIGS[a.config]
    shape = cfg.shape
    lens = cfg.seq_lens()
    B, L = len(lens), int(lens.max())
    dev = torch.device("cuda", 0)
    for x in [int(v) for v in a.heads.split(",")]:
        b = workload.make_decode_batch(shape, lens, cfg.seed, dev, q_begin=0, q_count=x)
        s = hetis.make_shape(shape)
        sb = accounting.step_bytes(lens.tolist(), x, shape.r, shape.head_dim, shape.page_size, shape.elem_bytes,
                                   shape.elem_bytes, 4)
        n_layers = max(1, math.ceil(4 * 126 * 2 ** 20 / sb.kv))
        kp = [b.k_pool] + [b.k_pool.clone() for _ in range(n_layers - 1)]
        vp = [b.v_pool] + [b.v_pool.clone() for _ in range(n_layers - 1)]
        ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), dev)
        o = torch.empty((B, x, shape.head_dim), device=dev)
        for fl in [int(v, 0) for v in a.flags.split(",")]:
            def attn(i):
                if fl & hetis.ATTN_DIAG_STREAM_ONLY:   # the stream-only diagnostic cannot append
                    hetis.attn_partial(s, b.q, kp[i % n_layers], vp[i % n_layers], b.block_table, b.seq_lens, L,
                                       ws, flags=fl)
                else:
                    hetis.attn_partial_append(s, b.q, b.k_new, b.v_new, kp[i % n_layers], vp[i % n_layers],
                                              b.block_table, b.seq_lens, L, ws, flags=fl)

            def step(i):
                attn(i)
                hetis.attn_combine(s, b.seq_lens, L, o, ws)

            def decode(i):   # the library's one-call step (one kernel with HETIS_ATTN_FUSED_MERGE)
                hetis.attn_decode_append(s, b.q, b.k_new, b.v_new, kp[i % n_layers], vp[i % n_layers],
                                         b.block_table, b.seq_lens, L, o, ws, flags=fl)

            res = {}
            fns = [("attn", attn), ("step", step)]
            if a.decode and not fl & hetis.ATTN_DIAG_STREAM_ONLY:
                fns.append(("decode", decode))
            for name, fn in fns:
                for i in range(5):
                    fn(i)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for i in range(a.steps):
                        fn(i)
                g.replay()
                torch.cuda.synchronize()
                ts = []
                for _ in range(a.reps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    g.replay()
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e3 / a.steps)
                res[name + "_us"] = min(ts)
                del g
            res.update({"config": a.config, "heads": x, "flags": fl, "kv_bytes": sb.kv,
                        "attn_gbs": sb.kv / res["attn_us"] / 1e3, "frac_of_copy_peak": sb.kv / res["attn_us"] / 1e3 / 6530.6,
                        "lib": os.path.basename(hetis.LIB_PATH)})
            print(json.dumps(res), flush=True)
        del kp, vp, b, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
