import sys, torch
sys.path.insert(0, '.')
from paper_2509_08309_b200 import hetis, workload
mode = sys.argv[1]
shape = workload.Shape(64, 8, 128, 16, "bf16")
lens = torch.tensor([1, 15, 16, 17, 255, 256, 900, 2047], dtype=torch.int32)
b = workload.make_decode_batch(shape, lens, 111, "cuda")
s = hetis.make_shape(shape)
B, x, _ = b.q.shape
L = int(lens.max())
ws = [hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), "cuda") for _ in range(2)]
o = torch.empty((B, x, 128), device="cuda")
print("start", mode, flush=True)
if mode == "one":
    hetis.attn_partial(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, ws[0], flags=hetis.ATTN_PIPELINED)
    torch.cuda.synchronize(); print("one ok", flush=True)
elif mode == "two":
    for i in range(4):
        hetis.attn_partial(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, ws[i % 2], flags=hetis.ATTN_PIPELINED)
        hetis.attn_combine(s, b.seq_lens, L, o, ws[i % 2])
    torch.cuda.synchronize(); print("eager ok", flush=True)
elif mode == "mha":
    sh = workload.Shape(40, 40, 128, 16, "bf16"); bb = workload.make_decode_batch(sh, lens, 1, "cuda"); ss = hetis.make_shape(sh)
    w = hetis.alloc_workspace(hetis.attn_decode_workspace(ss, B, 40, L), "cuda")
    hetis.attn_partial(ss, bb.q, bb.k_pool, bb.v_pool, bb.block_table, bb.seq_lens, L, w, flags=hetis.ATTN_PIPELINED | hetis.ATTN_MHA_TC)
    torch.cuda.synchronize(); print("mha ok", flush=True)
elif mode in ("app_eager", "graph_plain", "graph_app"):
    for rep in range(2):
        def run():
            for i in range(4):
                f = hetis.ATTN_PIPELINED
                if mode == "graph_plain":
                    hetis.attn_partial(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, ws[i % 2], flags=f)
                else:
                    hetis.attn_partial_append(s, b.q, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens,
                                              L, ws[i % 2], flags=f)
                hetis.attn_combine(s, b.seq_lens, L, o, ws[i % 2])
        if mode == "app_eager":
            run()
        else:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                run()
            g.replay()
        torch.cuda.synchronize()
        print(mode, "ok", rep, flush=True)
