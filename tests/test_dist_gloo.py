"""World-size-2 CPU tests (gloo) of the N > 1 host logic.

What runs on CPU here is the part of the multi-GPU path that is not a kernel:
the plan (hetis_plan_* through the C ABI: Eq. 5 ranges, uneven splits), each
rank generating only its own kv heads' pages, the scatter of q / new k, v by
plan range, and the gather that puts every head at its GLOBAL index (Eq. 2a
Concat; reading 4).  The per-rank attention is computed by the
oracle (test infrastructure) in place of the CUDA kernel, so the assembled
result must equal the unsplit oracle result bit for bit.

The exchange KERNELS themselves (the pull of q / new k, v from the Primary --
standalone or folded into the attention kernel -- the combine storing every O
row into every rank at its global head index, the epoch protocol) need a GPU:
they run with N = 2, 4, 5 processes sharing one GPU through CUDA IPC in
tests/test_gpu_peer.py (bit-exact against the single-device result, even /
uneven / gather-to-root plans, eager steps and graph replays), and the whole
bench path in tests/test_gpu_bench.py (--force-dist, --share-gpu).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, split, shape_args, lens, out_q):
    # file rendezvous: no free TCP port to race for
    dist.init_process_group("gloo", init_method="file://" + port, rank=rank, world_size=world)
    try:
        import oracle
        from paper_2509_08309_b200 import hetis, workload
        from tests.helpers import dtype_code, host_batch

        shape = workload.Shape(*shape_args)
        plan = hetis.plan_create(hetis.make_shape(shape), world, split)
        begin, count = plan.heads(rank)
        seq_lens = torch.tensor(lens, dtype=torch.int32)
        B, D, r = len(lens), shape.head_dim, shape.r

        # scatter: root holds q_full, sends each rank its plan range
        if rank == 0:
            q_full = workload.make_q(shape, B, 5, "cpu")
            for i in range(1, world):
                b_i, x_i = plan.heads(i)
                dist.send(q_full[:, b_i:b_i + x_i].contiguous().view(torch.int16) if shape.dtype == "bf16"
                          else q_full[:, b_i:b_i + x_i].contiguous(), dst=i)
            q_mine = q_full[:, begin:begin + count].contiguous()
        else:
            buf = torch.empty((B, count, D), dtype=torch.int16 if shape.dtype == "bf16" else torch.float32)
            dist.recv(buf, src=0)
            q_mine = buf.view(torch.bfloat16) if shape.dtype == "bf16" else buf

        # this rank's share, generated locally (its own pages, its own permutation)
        part = workload.make_decode_batch(shape, seq_lens, 5, "cpu", q_begin=begin, q_count=count, rank_salt=rank)
        same_q = torch.equal(q_mine.view(torch.int16) if shape.dtype == "bf16" else q_mine,
                             part.q.view(torch.int16) if shape.dtype == "bf16" else part.q)
        hb = host_batch(part)
        shard = oracle.decode(hb["q"], hb["k_pool"], hb["v_pool"], hb["block_table"], hb["seq_lens"],
                              num_kv_heads=count // r, dtype=dtype_code(shape))      # [B][x][D]

        # gather: all-gather(v) of the shards by plan counts, then place at global heads
        xmax = max(plan.heads(i)[1] for i in range(world))
        pad = torch.zeros((B, xmax, D), dtype=torch.float64)
        pad[:, :count] = torch.from_numpy(shard)
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad)
        o_full = torch.full((B, shape.num_q_heads, D), float("nan"), dtype=torch.float64)
        for i in range(world):
            b_i, x_i = plan.heads(i)
            o_full[:, b_i:b_i + x_i] = bufs[i][:, :x_i]
        out_q.put((rank, same_q, o_full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("split,shape_args,lens", [
    ((24, 16), (40, 40, 64, 16, "bf16"), (1, 17, 300)),
    ((48, 16), (64, 8, 64, 16, "bf16"), (5, 256, 33)),
    ((4, 4), (8, 8, 64, 16, "f32"), (128, 128, 128, 128)),     # c1 shape, split 2 ways
])
def test_two_rank_head_parallel_step_equals_unsplit(split, shape_args, lens):
    import oracle
    from paper_2509_08309_b200 import workload
    from tests.helpers import dtype_code, host_batch

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    import tempfile
    port = os.path.join(tempfile.mkdtemp(), "rendezvous")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, split, shape_args, lens, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shape = workload.Shape(*shape_args)
    full = workload.make_decode_batch(shape, torch.tensor(lens, dtype=torch.int32), 5, "cpu")
    hb = host_batch(full)
    ref = oracle.decode(hb["q"], hb["k_pool"], hb["v_pool"], hb["block_table"], hb["seq_lens"],
                        num_kv_heads=shape.num_kv_heads, dtype=dtype_code(shape))
    for rank, same_q, o_full in results:
        assert same_q, f"rank {rank}: scattered q differs from the plan range of q_full"
        assert np.array_equal(o_full, ref), f"rank {rank}"
