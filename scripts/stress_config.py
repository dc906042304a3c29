"""Repeat one attention configuration many times and check every output is bit-identical (race hunting)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_08309_b200 import hetis, workload

H, Hkv, D, dt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 50
lens = (1, 2, 15, 16, 17, 31, 33, 255, 256, 257, 517, 1000) * 4
shape = workload.Shape(H, Hkv, D, 16, dt)
b = workload.make_decode_batch(shape, torch.tensor(lens, dtype=torch.int32), 5, "cuda")
s = hetis.make_shape(shape)
hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
B = len(lens)
ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, H, 1000), "cuda")
ref = None
bad = 0
for t in range(reps):
    o = torch.full((B, H, D), float("nan"), device="cuda")
    hetis.attn_decode(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, 1000, o, ws)
    torch.cuda.synchronize()
    if ref is None:
        ref = o
    elif not torch.equal(o, ref):
        bad += 1
print(f"{H}/{Hkv}/{D}/{dt}: {bad} of {reps - 1} repeats differ; nan={int(torch.isnan(ref).sum())}")
