#!/usr/bin/env python
"""Race hunting on the bench's step: N back-to-back decode steps (attention with the fused append, then the
combine) captured as a CUDA graph -- so consecutive kernels overlap through programmatic dependent launch --
replayed R times; every step's O and the final pools must equal, bit for bit, the same steps run eagerly
with a device synchronisation after every kernel.

    python scripts/stress_steps.py [--replays 20] [--steps 40]
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_08309_b200 import hetis, workload  # noqa: E402


def run(shape, flags, n_steps, replays, seed=3, large=False):
    if large:  # ~5000 GQA items (>= 2 per worker): pipelined launches steal too
        lens0 = torch.tensor([200 + (i * 97) % 2800 for i in range(96)], dtype=torch.int32)
    else:
        lens0 = torch.tensor([1, 15, 16, 17, 255, 256, 257, 900, 2047, 3000] * 4, dtype=torch.int32)
    lens_max = lens0 + n_steps
    b = workload.make_decode_batch(shape, lens_max, seed, "cuda")
    s = hetis.make_shape(shape)
    B, x, D = b.q.shape
    L = int(lens_max.max())
    pipelined = bool(flags & hetis.ATTN_PIPELINED)
    ws = [hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), "cuda") for _ in range(2)]
    g = torch.Generator(device="cuda").manual_seed(seed)
    kn = [torch.randn(b.k_new.shape, generator=g, device="cuda").to(b.k_new.dtype) for _ in range(n_steps)]
    vn = [torch.randn(b.v_new.shape, generator=g, device="cuda").to(b.v_new.dtype) for _ in range(n_steps)]
    sl = [(lens0 + i + 1).to("cuda") for i in range(n_steps)]
    o = [torch.empty((B, x, D), device="cuda") for _ in range(n_steps)]
    k0, v0 = b.k_pool.clone(), b.v_pool.clone()

    def steps(sync):
        for i in range(n_steps):
            w_ = ws[i % 2] if pipelined else ws[0]
            hetis.attn_partial_append(s, b.q, kn[i], vn[i], b.k_pool, b.v_pool, b.block_table, sl[i], L, w_,
                                      flags=flags)
            if sync:
                torch.cuda.synchronize()
            hetis.attn_combine(s, sl[i], L, o[i], w_)
            if sync:
                torch.cuda.synchronize()

    steps(True)
    ref = [t.clone() for t in o]
    ref_k = b.k_pool.clone()
    graph = torch.cuda.CUDAGraph()
    b.k_pool.copy_(k0)
    b.v_pool.copy_(v0)
    with torch.cuda.graph(graph):
        steps(False)
    bad = 0
    for _ in range(replays):
        b.k_pool.copy_(k0)
        b.v_pool.copy_(v0)
        for t in o:
            t.fill_(float("nan"))
        graph.replay()
        torch.cuda.synchronize()
        same = all(torch.equal(a, r) for a, r in zip(o, ref))
        bits = (lambda t: t.view(torch.int16)) if b.k_pool.dtype == torch.bfloat16 else (lambda t: t.view(torch.int32))
        same = same and torch.equal(bits(b.k_pool), bits(ref_k))
        bad += 0 if same else 1
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--replays", type=int, default=20)
    ap.add_argument("--steps", type=int, default=40)
    a = ap.parse_args()
    cases = [("GQA r=8", workload.Shape(64, 8, 128, 16, "bf16"), 0),
             ("GQA r=8 pipelined", workload.Shape(64, 8, 128, 16, "bf16"), hetis.ATTN_PIPELINED),
             ("GQA r=8 pipelined large", workload.Shape(64, 8, 128, 16, "bf16"), hetis.ATTN_PIPELINED | 0x10000),
             ("GQA r=8 device claim", workload.Shape(64, 8, 128, 16, "bf16"), hetis.ATTN_DEVICE_CLAIM),
             ("GQA r=8 static deal", workload.Shape(64, 8, 128, 16, "bf16"), hetis.ATTN_STATIC_DEAL),
             ("MHA CUDA cores", workload.Shape(40, 40, 128, 16, "bf16"), 0),
             ("MHA CUDA cores shared ring", workload.Shape(40, 40, 128, 16, "bf16"), hetis.ATTN_TC_SHARED_RING),
             ("MHA CUDA cores pipelined", workload.Shape(40, 40, 128, 16, "bf16"), hetis.ATTN_PIPELINED),
             ("MHA tensor cores", workload.Shape(40, 40, 128, 16, "bf16"), hetis.ATTN_MHA_TC),
             ("fp32 d=64", workload.Shape(8, 8, 64, 16, "f32"), 0)]
    total = 0
    for name, shape, flags in cases:
        bad = run(shape, flags & 0xFFFF, a.steps, a.replays, large=bool(flags & 0x10000))
        total += bad
        print(f"{name:28s}: {bad} of {a.replays} graph replays differ from the serial run", flush=True)
    print("STRESS", "OK" if total == 0 else f"FAILED ({total})")


if __name__ == "__main__":
    main()
