#!/usr/bin/env python
"""Head-granular KV migration (row f4, the Hauler: PAPER.md:522, :545) on one B200.

Scenario: a re-dispatch of the c3 batch (LLaMA2-70B shape, B = 128, L = 2048)
that moves kv groups 4..7 of every request to another device ("only partial
cache transmission": the other groups' pages stay).  One GPU is reachable per
call, so source and destination pools are two allocations on the same device
(an HBM -> HBM copy; over NVLink the destination pool would be a peer mapping
and the copy would be bound by the 770 GB/s peer bandwidth instead).

  1. hetis_kv_migrate alone, for several CTA budgets: GB/s of (read + write).
  2. interference (PAPER.md:545 runs the Hauler beside decode): the c3 decode
     step (CUDA graph, PDL) on the default-priority stream while migrations run
     on a low-priority stream with a bounded CTA budget: decode us/step vs
     alone, and the migration throughput achieved meanwhile.

    python scripts/migrate_probe.py [--steps 100]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_08309_b200 import hetis, workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--config", default="c3")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg = workload.CONFIGS[a.config]
    shape, lens = cfg.shape, cfg.seq_lens()
    B, G, L = cfg.batch, shape.num_kv_heads, int(lens.max())
    b = workload.make_decode_batch(shape, lens, cfg.seed, dev)
    s = hetis.make_shape(shape)
    P = shape.page_size
    maxp = b.block_table.shape[2]
    moving = list(range(G // 2, G))                          # groups that change device
    # destination: a fresh pool and table for the moved groups
    npg = int(((lens + P - 1) // P).sum()) * len(moving)
    dst_k = torch.zeros((npg + 16, P, shape.head_dim), dtype=shape.torch_dtype, device=dev)
    dst_v = torch.zeros_like(dst_k)
    perm = torch.randperm(npg + 16, generator=torch.Generator().manual_seed(5))[:npg].to(torch.int32)
    dst_bt = torch.full((B * len(moving), maxp), -1, dtype=torch.int32)
    ent, off = [], 0
    for j in range(B):
        n = (int(lens[j]) + P - 1) // P
        for k, g in enumerate(moving):
            dst_bt[j * len(moving) + k, :n] = perm[off:off + n]
            off += n
            ent.append([j * G + g, j * len(moving) + k, int(lens[j])])
    entries = torch.tensor(ent, dtype=torch.int32, device=dev)
    dst_bt = dst_bt.to(dev)
    src_bt = b.block_table.view(B * G, maxp)
    moved = sum(e[2] for e in ent) * 2 * shape.head_dim * shape.elem_bytes     # K and V bytes moved
    pages_moved = sum((e[2] + P - 1) // P for e in ent) * 2 * P * shape.head_dim * shape.elem_bytes

    def migrate(ctas, stream=None):
        hetis.kv_migrate(s, entries, b.k_pool, b.v_pool, src_bt, dst_k, dst_v, dst_bt, max_ctas=ctas, stream=stream)

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rows = []
    for ctas in (0, 74, 32, 16):
        for _ in range(2):
            migrate(ctas)
        torch.cuda.synchronize()
        n = 10
        ev0.record()
        for _ in range(n):
            migrate(ctas)
        ev1.record()
        torch.cuda.synchronize()
        us = ev0.elapsed_time(ev1) / n * 1e3
        rows.append({"max_ctas": ctas, "us": us, "moved_bytes": pages_moved,
                     "gbs_read_plus_write": 2 * pages_moved / us / 1e3})
    print(json.dumps({"probe": "kv_migrate alone", "config": cfg.name, "groups_moved_per_request": len(moving),
                      "entries": len(ent), "token_bytes": moved, "page_bytes": pages_moved, "rows": rows}),
          flush=True)

    # ---- interference with decode
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, shape.num_q_heads, L), dev)
    o = torch.empty((B, shape.num_q_heads, shape.head_dim), device=dev)

    lo, hi = torch.cuda.Stream.priority_range()
    side = torch.cuda.Stream(device=dev, priority=lo)        # numerically larger = lower priority
    out = []
    t_alone = {r["max_ctas"]: r["us"] for r in rows}
    for flags, ctas in ((0, 16), (0, 32), (0, 74), (hetis.ATTN_DEVICE_CLAIM, 16), (hetis.ATTN_DEVICE_CLAIM, 32),
                        (hetis.ATTN_DEVICE_CLAIM, 74)):
        def step():
            hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
            hetis.attn_partial(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, ws, flags=flags)
            hetis.attn_combine(s, b.seq_lens, L, o, ws)

        for _ in range(3):
            step()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(a.steps):
                step()
        g.replay()
        torch.cuda.synchronize()
        ev0.record()
        g.replay()
        ev1.record()
        torch.cuda.synchronize()
        alone = ev0.elapsed_time(ev1) / a.steps * 1e3
        n_mig = max(1, int(alone * a.steps / t_alone[ctas]))  # about the decode window at the alone rate
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            m0.record(side)
            for _ in range(n_mig):
                migrate(ctas, side)
            m1.record(side)
        ev0.record()
        g.replay()
        ev1.record()
        torch.cuda.synchronize()
        dec = ev0.elapsed_time(ev1) / a.steps * 1e3
        mig_us = m0.elapsed_time(m1) * 1e3
        out.append({"attn_flags": flags, "max_ctas": ctas, "decode_us_per_step": dec, "decode_alone_us": alone,
                    "decode_slowdown": dec / alone, "migrations": n_mig, "migration_window_us": mig_us,
                    "migration_gbs_read_plus_write": 2 * pages_moved * n_mig / mig_us / 1e3})
    print(json.dumps({"probe": "decode + concurrent kv_migrate (low-priority stream)", "config": cfg.name,
                      "rows": out}), flush=True)


if __name__ == "__main__":
    main()
