"""The NCCL scatter / gather entry points through the C ABI on one GPU
(world size 1 -- the only NCCL world this round's single-GPU boxes allow).

Checks that hetis_scatter_q delivers the plan's head range of q_full and of the
new k, v rows, and that hetis_gather (all-gather and gather-to-root) places the
shard at its global head index (Eq. 2a Concat; reading 4) -- the
assembled O equals the directly computed O bit for bit.
"""
from __future__ import annotations

import os
import socket

import pytest
import torch

from paper_2509_08309_b200 import hetis, workload
from paper_2509_08309_b200.step import DecodeStep

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_world1():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    dist.barrier()
    comm = dist.group.WORLD._get_backend(dev)._comm_ptr()
    yield comm
    dist.destroy_process_group()


@pytest.mark.parametrize("shape", [workload.LLAMA2_13B, workload.LLAMA2_70B])
def test_scatter_and_gather_world1(nccl_world1, shape):
    comm = nccl_world1
    lens = torch.tensor([300, 17, 1, 1029], dtype=torch.int32)
    b = workload.make_decode_batch(shape, lens, 9, "cuda")
    plan = hetis.plan_create(hetis.make_shape(shape), 1, [shape.num_q_heads])
    step = DecodeStep(shape, plan, 0, len(lens), int(lens.max()), torch.device("cuda", 0), comm_ptr=comm)
    # scatter from the root's full tensors
    step.scatter(b.q, b.k_new, b.v_new)
    torch.cuda.synchronize()
    assert torch.equal(step.buf.q_shard, b.q)
    assert torch.equal(step.buf.k_new, b.k_new) and torch.equal(step.buf.v_new, b.v_new)
    step.append(b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    o = step.attention(b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    for root in (-1, 0):
        o_full = torch.full_like(o, float("nan"))
        step.gather(o_full, root=root)
        torch.cuda.synchronize()
        assert torch.equal(o_full, o), root


def test_gather_rejects_mismatched_communicator(nccl_world1):
    plan = hetis.plan_create(hetis.make_shape(workload.LLAMA2_13B), 2, [20, 20])
    o = torch.zeros((2, 20, 128), device="cuda")
    full = torch.zeros((2, 40, 128), device="cuda")
    ws = hetis.alloc_workspace(plan.comm_workspace(0, 2), "cuda")
    with pytest.raises(hetis.HetisError) as e:
        hetis.gather(plan, nccl_world1, 0, -1, 2, o, full, ws)
    assert e.value.name == "HETIS_E_INVALID"          # 2-device plan on a 1-rank communicator


@pytest.mark.parametrize("shape", [workload.LLAMA2_13B, workload.LLAMA2_70B])
def test_seq_split_broadcast_and_allgather_merge_world1(nccl_world1, shape):
    """Sequence split (row f3) through its NCCL entry points: hetis_seq_broadcast_q delivers q / new k, v
    in place and hetis_seq_allgather_merge of one device's (o, lse) record reproduces o bit for bit."""
    from paper_2509_08309_b200 import seqsplit
    lens = torch.tensor([300, 17, 1, 1029], dtype=torch.int32)
    b = workload.make_decode_batch(shape, lens, 11, "cuda")
    st = seqsplit.SeqSplitStep(shape, 1, 0, len(lens), int(lens.max()), torch.device("cuda", 0),
                               comm_ptr=nccl_world1)
    st.q.copy_(b.q)
    st.k_new.copy_(b.k_new)
    st.v_new.copy_(b.v_new)
    st.broadcast()
    torch.cuda.synchronize()
    assert torch.equal(st.q, b.q) and torch.equal(st.k_new, b.k_new) and torch.equal(st.v_new, b.v_new)
    lbt = seqsplit.local_block_table(b.block_table, 1, 0)
    o = torch.full_like(b.q, float("nan"), dtype=torch.float32)
    st.run(b.k_pool, b.v_pool, lbt, b.seq_lens, o)
    staging = torch.empty((1, st.part.numel()), dtype=torch.float32, device="cuda")
    o2 = torch.full_like(o, float("nan"))
    hetis.seq_allgather_merge(st.cshape, nccl_world1, 1, 0, len(lens), st.part, staging, o2)
    torch.cuda.synchronize()
    assert torch.equal(staging[0], st.part)
    assert torch.equal(o2, o) and torch.equal(o, st.part_o)
