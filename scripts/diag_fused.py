"""Diagnostic: run the fused step repeatedly on c3 and report where it differs from the 3-call path."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_08309_b200 import hetis, workload

cfg = workload.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
s = hetis.make_shape(cfg.shape)
b = workload.make_decode_batch(cfg.shape, cfg.seq_lens(), cfg.seed, "cuda")
B, x, D = b.q.shape
L = b.max_seq_len
hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), "cuda")
ref = torch.empty((B, x, D), device="cuda")
hetis.attn_decode(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, ref, ws)
ws2 = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), "cuda")
for t in range(20):
    o = torch.full((B, x, D), float("nan"), device="cuda")
    hetis.decode_step(s, b.q, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, o, ws2)
    torch.cuda.synchronize()
    d = (o - ref).abs()
    bad = (d > 0) | torch.isnan(o)
    if bad.any():
        idx = bad.nonzero()
        pairs = sorted({(int(a), int(h) // cfg.shape.r) for a, h, _ in idx.tolist()})
        print(f"run {t}: {int(bad.sum())} elems differ, nan={int(torch.isnan(o).sum())}, max {float(d[~torch.isnan(d)].max()) if (~torch.isnan(d)).any() else 'nan'}, pairs {pairs[:8]} (n={len(pairs)})")
    else:
        print(f"run {t}: identical")
    cnt = ws2.view(torch.int32)
print("counters nonzero after runs:", int((ws2[-(B * x // cfg.shape.r) * 4:].view(torch.int32) != 0).sum()))
