"""Diagnostic: repeat the three-call step (kv_append + partial + combine) and check bit-identical outputs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_08309_b200 import hetis, workload

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = workload.CONFIGS[name]
s = hetis.make_shape(cfg.shape)
b = workload.make_decode_batch(cfg.shape, cfg.seq_lens(), cfg.seed, "cuda")
B, x, D = b.q.shape
L = b.max_seq_len
ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), "cuda")
ref = None
bad = 0
for t in range(reps):
    hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    o = torch.full((B, x, D), float("nan"), device="cuda")
    hetis.attn_decode(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, o, ws)
    torch.cuda.synchronize()
    if ref is None:
        ref = o
    elif not torch.equal(o, ref):
        bad += 1
        d = (o - ref).abs()
        idx = (d > 0).nonzero()
        print(f"{name} run {t}: {idx.shape[0]} elems differ, max {float(d.max())}, first {idx[:2].tolist()}")
print(f"{name}: {bad} of {reps - 1} repeats differ")
