"""Fused combine + all-gather over peer memory (hetis_attn_combine_peers), two ranks.

Only one GPU is reachable, so the two ranks are two processes on cuda:0 that map
each other's o_full and signal arrays through CUDA IPC (torch.multiprocessing
shares CUDA tensors that way) -- the same peer-pointer code path an 8-GPU box
uses over NVLink, with the data staying on one device.  Each rank runs its own
heads' attention and stores every merged row into BOTH ranks' o_full at the
global head index (Eq. 2a Concat), then publishes the epoch.
Host barriers order the two processes (kernels of two processes time-slice on
one GPU, so no kernel spin-waits on the other process); hetis_peer_wait runs
after the barrier and must see both signals.  Both ranks must end with the
single-device result, bit for bit.
"""
from __future__ import annotations

import os

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

LENS = (300, 17, 1029, 2048, 5, 256)


def _rank(rank, split, shape_args, q_in, q_out, barrier, res):
    import torch
    from paper_2509_08309_b200 import hetis, workload
    torch.cuda.set_device(0)
    shape = workload.Shape(*shape_args)
    lens = torch.tensor(LENS, dtype=torch.int32)
    B, H, D = len(LENS), shape.num_q_heads, shape.head_dim
    begin, count = sum(split[:rank]), split[rank]
    o_full = torch.full((B, H, D), float("nan"), device="cuda")
    sig = torch.zeros(2, dtype=torch.int64, device="cuda")
    q_out.put((o_full, sig))                 # share my buffers with the peer (CUDA IPC)
    peer_o, peer_sig = q_in.get(timeout=120)
    o_peers = [o_full, peer_o] if rank == 0 else [peer_o, o_full]
    s_peers = [sig, peer_sig] if rank == 0 else [peer_sig, sig]
    b = workload.make_decode_batch(shape, lens, 13, "cuda", q_begin=begin, q_count=count, rank_salt=rank + 1)
    s = hetis.make_shape(shape)
    hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, count, b.max_seq_len), "cuda")
    for epoch in (1, 2):
        hetis.attn_partial(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, b.max_seq_len, ws,
                           q_head_begin=begin)
        hetis.attn_combine_peers(s, b.seq_lens, b.max_seq_len, o_peers, s_peers, rank, epoch, ws,
                                 q_head_begin=begin, q_head_count=count)
        torch.cuda.synchronize()
        barrier.wait(timeout=120)            # both ranks' stores and signals are done
        hetis.peer_wait(sig, epoch)          # stream-ordered acquire; both signals already >= epoch
        torch.cuda.synchronize()
        got = o_full.clone()
        barrier.wait(timeout=120)
    # single-device reference on this process (all heads, the same generated data per kv head)
    full = workload.make_decode_batch(shape, lens, 13, "cuda")
    hetis.kv_append(s, full.k_new, full.v_new, full.k_pool, full.v_pool, full.block_table, full.seq_lens)
    wsf = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, H, full.max_seq_len), "cuda")
    ref = torch.empty((B, H, D), device="cuda")
    hetis.attn_decode(s, full.q, full.k_pool, full.v_pool, full.block_table, full.seq_lens, full.max_seq_len, ref,
                      wsf)
    torch.cuda.synchronize()
    res.put((rank, bool(torch.equal(got, ref)), float((got - ref).abs().nan_to_num(1e9).max()),
             int(sig.cpu().min())))
    barrier.wait(timeout=120)                # keep the shared buffers alive until both ranks are done


@pytest.mark.parametrize("shape_args,split", [((64, 8, 128, 16, "bf16"), (48, 16)),
                                              ((40, 40, 128, 16, "bf16"), (24, 16))])
def test_combine_peers_two_ranks_one_gpu(shape_args, split):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    a2b, b2a, res = ctx.Queue(), ctx.Queue(), ctx.Queue()
    barrier = ctx.Barrier(2)
    ps = [ctx.Process(target=_rank, args=(0, split, shape_args, b2a, a2b, barrier, res)),
          ctx.Process(target=_rank, args=(1, split, shape_args, a2b, b2a, barrier, res))]
    for p in ps:
        p.start()
    out = [res.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, equal, diff, sig_min in out:
        assert sig_min == 2, (rank, sig_min)
        assert equal, (rank, diff)


# ------------------------------------------------------------------ pull-based scatter over peer memory
def _pull_rank(rank, port, shape_args, split, res, barrier):
    import os
    import torch
    import torch.distributed as dist
    from paper_2509_08309_b200 import hetis, workload
    from paper_2509_08309_b200.step import DecodeStep
    # object exchange only (data moves by IPC); a file rendezvous needs no free TCP port
    dist.init_process_group("gloo", init_method="file://" + port, rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)
        shape = workload.Shape(*shape_args)
        B, H, Hkv, D = 7, shape.num_q_heads, shape.num_kv_heads, shape.head_dim
        plan = hetis.plan_create(hetis.make_shape(shape), 2, split)
        step = DecodeStep(shape, plan, rank, B, 512, torch.device("cuda", 0))
        g = torch.Generator(device="cuda").manual_seed(3)
        mk = lambda *sz: torch.randn(sz, generator=g, device="cuda").to(shape.torch_dtype)
        q_full, k_full, v_full = mk(B, H, D), mk(B, Hkv, D), mk(B, Hkv, D)   # same bits on both ranks
        o_full = torch.zeros((B, H, D), device="cuda")
        if rank == 0:
            step.setup_peers(o_full, q_full, k_full, v_full)
        else:
            step.setup_peers(o_full)
        ok = True
        for epoch in (1, 2):
            if rank == 0:
                q_full.mul_(-1)                      # new inputs for this step, then signal
                k_full.mul_(-1)
                v_full.mul_(-1)
                hetis.peer_signal(step.qsig_peers, 0, epoch)
                torch.cuda.synchronize()
            else:
                q_full.mul_(-1)
                k_full.mul_(-1)
                v_full.mul_(-1)
            barrier.wait(timeout=120)                # the root's signal is published before anyone pulls
            step.buf.q_shard.zero_()
            step.buf.k_new.zero_()
            step.buf.v_new.zero_()
            step.scatter_peers(epoch)
            torch.cuda.synchronize()
            b, x = plan.heads(rank)
            r = shape.r
            ok &= torch.equal(step.buf.q_shard, q_full[:, b:b + x])
            ok &= torch.equal(step.buf.k_new, k_full[:, b // r:(b + x) // r])
            ok &= torch.equal(step.buf.v_new, v_full[:, b // r:(b + x) // r])
            ok &= int(step.qsig[0].item()) == epoch
            barrier.wait(timeout=120)                # nobody changes the root's buffers while others pull
        res.put((rank, bool(ok)))
        barrier.wait(timeout=120)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape_args,split", [((64, 8, 128, 16, "bf16"), (48, 16)),
                                              ((40, 40, 128, 16, "bf16"), (24, 16))])
def test_scatter_pull_two_ranks_one_gpu(shape_args, split):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import tempfile
    port = os.path.join(tempfile.mkdtemp(), "rendezvous")
    ctx = mp.get_context("spawn")
    res, barrier = ctx.Queue(), ctx.Barrier(2)
    ps = [ctx.Process(target=_pull_rank, args=(r, port, shape_args, split, res, barrier)) for r in range(2)]
    for p in ps:
        p.start()
    out = [res.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, ok in out:
        assert ok, rank
