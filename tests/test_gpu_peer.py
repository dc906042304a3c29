"""The N > 1 step over peer memory -- hetis_scatter_pull -> hetis_attn_partial_append ->
hetis_attn_combine_peers -> hetis_peer_wait -- run by N processes.

Only one GPU is reachable, so the N ranks are N processes on cuda:0 that map each
other's exchange state and o_full, and the root's input buffers, through CUDA
IPC (the same peer-pointer code path an 8-GPU NVSwitch box uses over NVLink,
with the data staying on one device).  Nothing orders the processes on the host
during the steps: every wait is the library's device-side epoch protocol
(kernels of different processes time-slice on the GPU, so a spinning wait yields
to the peer it waits for).  Several steps run eagerly, then more steps replayed
from a captured CUDA graph (no per-step host argument); the root flips the sign
of q before every step, so each step's O differs and a stale row would show.
Every receiving rank must end with the single-device result of the final q, bit
for bit (head-partition invariance; Eq. 2a Concat at the global
head index), for even, uneven (16/8/8/4/4) and gather-to-root
plans.
"""
from __future__ import annotations

import os
import tempfile

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

LENS = (300, 17, 1029, 2048, 5, 256, 1)
EAGER_STEPS, GRAPH_STEPS, GRAPH_REPLAYS = 3, 2, 2


def _rank(rank, world, rendezvous, shape_args, split, gather_root, merge_fused, pull, flags, res):
    import torch
    import torch.distributed as dist
    from paper_2509_08309_b200 import hetis, workload
    from paper_2509_08309_b200.step import DecodeStep
    dist.init_process_group("gloo", init_method="file://" + rendezvous, rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        shape = workload.Shape(*shape_args)
        lens = torch.tensor(LENS, dtype=torch.int32)
        B, H, D = len(LENS), shape.num_q_heads, shape.head_dim
        plan = hetis.plan_create(hetis.make_shape(shape), world, split)
        begin, count = plan.heads(rank)
        mine = workload.make_decode_batch(shape, lens, 13, dev, q_begin=begin, q_count=count, rank_salt=rank + 1)
        full = workload.make_decode_batch(shape, lens, 13, dev)       # the unsplit problem (reference + root inputs)
        step = DecodeStep(shape, plan, rank, B, int(lens.max()), dev)
        receives = gather_root < 0 or gather_root == rank
        o_full = torch.full((B, H, D), float("nan"), device=dev) if receives else None
        if rank == 0:
            q_full, kn_full, vn_full = full.q.clone(), full.k_new.clone(), full.v_new.clone()
            step.setup_peers(o_full, q_full, kn_full, vn_full, gather_root=gather_root)
        else:
            step.setup_peers(o_full, gather_root=gather_root)

        def one_step():
            if rank == 0:
                q_full.neg_()                   # the step's new inputs, written before the root's pull
            step.step_peers(mine.k_pool, mine.v_pool, mine.block_table, mine.seq_lens, merge_fused=merge_fused,
                            pull=pull, flags=flags)

        for _ in range(EAGER_STEPS):
            one_step()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(graph, stream=s):
                for _ in range(GRAPH_STEPS):
                    one_step()
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(GRAPH_REPLAYS):
            graph.replay()
        torch.cuda.synchronize()
        n_steps = EAGER_STEPS + GRAPH_STEPS * GRAPH_REPLAYS
        got = o_full.clone() if receives else None
        dist.barrier()                          # every rank is done writing into peers' o_full
        # reference: the unsplit problem with the final q, same launch (append fused) on this process
        cs = hetis.make_shape(shape)
        if n_steps % 2:
            full.q.neg_()
        ws = hetis.alloc_workspace(hetis.attn_decode_workspace(cs, B, H, int(lens.max())), dev)
        ref = torch.empty((B, H, D), device=dev)
        hetis.attn_decode_append(cs, full.q, full.k_new, full.v_new, full.k_pool, full.v_pool, full.block_table,
                                 full.seq_lens, int(lens.max()), ref, ws)
        torch.cuda.synchronize()
        state = step.peer_state.cpu()
        ok_eq = bool(torch.equal(got, ref)) if receives else True
        diff = float((got - ref).abs().nan_to_num(1e9).max()) if receives else 0.0
        # with the separate pull kernel, this rank's shard of the last step is a bit-exact copy of the root's
        # range (with the pull folded into the attention kernel there is no shard)
        r = shape.r
        q_last = full.q[:, begin:begin + count]
        ok_pull = pull is not False or (bool(torch.equal(step.buf.q_shard, q_last)) and bool(
            torch.equal(step.buf.k_new, full.k_new[:, begin // r:(begin + count) // r])))
        res.put((rank, receives, ok_eq, diff, ok_pull, int(state[0]), n_steps))
        dist.barrier()                          # keep the shared buffers alive until everyone has compared
    finally:
        dist.destroy_process_group()


# merge_fused: True = hetis_attn_decode_peers (attention, split merge and the stores into every rank's
# o_full in ONE kernel), False = partial kernel + hetis_attn_combine_peers, None = the default (fused where
# the launch runs in group mode -- every GQA case below: 7 requests, L <= 2048 -- else the combine).
# pull: None = the attention kernel reads q / new k, v from the Primary (the default), False = the
# separate hetis_scatter_pull kernel first.  NG = HETIS_ATTN_NO_GROUP_MODE (the last-arriver merge)
NG = 0x40
CASES = [
    ((64, 8, 128, 16, "bf16"), (32, 32), -1, None, None, 0),        # default: pull + group merge, ONE kernel
    ((64, 8, 128, 16, "bf16"), (32, 32), -1, False, None, 0),       # pull in the kernel, separate combine
    ((64, 8, 128, 16, "bf16"), (32, 32), -1, False, False, 0),      # ... and the separate pull kernel
    ((64, 8, 128, 16, "bf16"), (32, 32), -1, True, False, 0),       # separate pull, group merge + gather fused
    ((64, 8, 128, 16, "bf16"), (32, 32), -1, True, False, NG),      # ... last-arriver merge through L2
    ((64, 8, 128, 16, "bf16"), (32, 32), -1, True, None, NG),       # pull + last-arriver merge, one kernel
    ((40, 40, 128, 16, "bf16"), (16, 8, 8, 4, 4), -1, None, None, 0),  # c4's uneven split (CUDA-core MHA)
    ((40, 40, 128, 16, "bf16"), (16, 8, 8, 4, 4), -1, None, False, 0),
    ((64, 8, 128, 16, "bf16"), (16, 16, 24, 8), 0, None, None, 0),  # uneven GQA, gather to the Primary (paper)
    ((64, 8, 128, 16, "bf16"), (16, 16, 24, 8), 0, False, None, 0),
    ((64, 8, 128, 16, "bf16"), (16, 16, 24, 8), 0, True, False, 0),
    ((16, 2, 64, 16, "bf16"), (8, 8), -1, None, None, 0),           # GQA d = 64, pull + group merge
    ((16, 2, 64, 16, "bf16"), (8, 8), -1, True, False, NG),         # GQA d = 64, last-arriver
    ((8, 8, 64, 16, "f32"), (4, 4), -1, None, None, 0),             # c1 shape, fp32, pull in the kernel
]


@pytest.mark.parametrize("shape_args,split,gather_root,merge_fused,pull,flags", CASES)
def test_peer_step_n_ranks_one_gpu(shape_args, split, gather_root, merge_fused, pull, flags):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    world = len(split)
    rendezvous = os.path.join(tempfile.mkdtemp(), "rendezvous")
    ctx = mp.get_context("spawn")
    res = ctx.Queue()
    ps = [ctx.Process(target=_rank, args=(r, world, rendezvous, shape_args, split, gather_root, merge_fused, pull,
                                          flags, res))
          for r in range(world)]
    for p in ps:
        p.start()
    out = [res.get(timeout=900) for _ in ps]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, receives, ok_eq, diff, ok_pull, steps_done, n_steps in out:
        assert steps_done == n_steps, (rank, steps_done)
        assert ok_pull, rank
        assert ok_eq, (rank, diff)
    assert sum(o[1] for o in out) == (world if gather_root < 0 else 1)


def test_peer_access_contract():
    """hetis_peer_access: the current device itself is OK (no-op), a device index outside the box is
    HETIS_E_INVALID, and every other device of the box is enabled or reported unsupported."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_08309_b200 import hetis
    torch.cuda.set_device(0)
    hetis.peer_access(0)
    with pytest.raises(hetis.HetisError) as e:
        hetis.peer_access(torch.cuda.device_count())
    assert e.value.name == "HETIS_E_INVALID"
    for d in range(1, torch.cuda.device_count()):
        try:
            hetis.peer_access(d)
            hetis.peer_access(d)                   # already enabled: still OK
        except hetis.HetisError as exc:
            assert exc.name == "HETIS_E_UNSUPPORTED"
