#!/usr/bin/env python
"""One rank's share of a config run through the library's one-call step a few times (for ncu): the c3 8-GPU
share runs in group mode (one kernel).  python scripts/profile_share.py [--config c3] [--heads 8] [--steps 5]"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_08309_b200 import hetis, workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    cfg = workload.CONFIGS[a.config]
    lens = cfg.seq_lens()
    dev = torch.device("cuda", 0)
    b = workload.make_decode_batch(cfg.shape, lens, cfg.seed, dev, q_begin=0, q_count=a.heads)
    s = hetis.make_shape(cfg.shape)
    B, L = len(lens), int(lens.max())
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, a.heads, L), dev)
    o = torch.empty((B, a.heads, cfg.shape.head_dim), device=dev)
    print("kernels per step:", hetis.attn_decode_launches_for(s, B, a.heads, L, 0))
    for _ in range(a.steps):
        hetis.attn_decode(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, o, ws)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
