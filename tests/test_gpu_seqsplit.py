"""GPU parity of the sequence-wise split (row f3) through the C ABI.

N virtual devices on one GPU share the physical pools; device r reads only its
striped pages (columns r, r + N, ... of the block table).  Each device runs
hetis_seq_split_lens -> hetis_kv_append (owner of the newest page only) ->
hetis_attn_partial -> hetis_attn_combine_lse on its local problem, and
hetis_seq_merge combines the N records.  Checked against the fp64 oracle:
  * O of the merged result vs the unsplit oracle (north-star tolerance),
  * every device's lse vs the oracle's lse on that device's local problem,
  * local lengths bit-exact vs the host bookkeeping (seqsplit.local_len),
  * N = 1 reproduces hetis_attn_decode bit for bit (one part: weight 2^0 = 1),
  * a device holding no token of a request returns o = 0, lse = -inf.
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import oracle
from paper_2509_08309_b200 import hetis, seqsplit, workload
from paper_2509_08309_b200.seqsplit import SeqSplitStep
from tests.helpers import dtype_code, err_stats, host_batch, host_batch_once

pytestmark = pytest.mark.gpu

ATOL, RTOL = 2e-3, 1e-2
LSE_ATOL = 1e-3


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    hetis.lib()


def _run_split(b: workload.DecodeBatch, N: int, o_dtype="f32"):
    """All N devices' steps on one GPU; returns (merged o, per-device (local_bt, local_lens, o, lse))."""
    shape = b.shape
    cs = hetis.make_shape(shape, o_dtype)
    B, H, D = b.q.shape
    dev = b.q.device
    steps, rec = [], []
    for r in range(N):
        st = SeqSplitStep(shape, N, r, B, b.max_seq_len, dev, o_dtype=o_dtype)
        st.q.copy_(b.q)
        st.k_new.copy_(b.k_new)
        st.v_new.copy_(b.v_new)
        steps.append(st)
    # appends first (every request's new row lands exactly once, on its owner), then attention
    lbts = [seqsplit.local_block_table(b.block_table, N, r) for r in range(N)]
    for r, st in enumerate(steps):
        hetis.seq_split_lens(N, r, shape.page_size, b.seq_lens, st.local_lens, st.append_lens)
        hetis.kv_append(cs, st.k_new, st.v_new, b.k_pool, b.v_pool, lbts[r], st.append_lens)
    for r, st in enumerate(steps):
        hetis.attn_partial(cs, st.q, b.k_pool, b.v_pool, lbts[r], st.local_lens, st.max_local, st.workspace)
        hetis.attn_combine_lse(cs, st.local_lens, st.max_local, st.part_o, st.part_lse, st.workspace)
    o_parts = torch.stack([st.part_o for st in steps])
    lse_parts = torch.stack([st.part_lse for st in steps])
    odt = torch.bfloat16 if o_dtype == "bf16" else torch.float32
    o = torch.full((B, H, D), float("nan"), dtype=odt, device=dev)
    hetis.seq_merge(cs, o_parts, lse_parts, o)
    torch.cuda.synchronize()
    return o, [(lbts[r], steps[r].local_lens, steps[r].part_o, steps[r].part_lse) for r in range(N)]


def _assert_close(got, ref, what):
    st = err_stats(got.float().cpu().numpy(), ref)
    assert st["nonfinite"] == 0, (what, st)
    assert st["max_abs"] <= ATOL and st["rel_fro"] <= RTOL, (what, st)


CASES = [
    (workload.Shape(40, 40, 128, 16, "bf16"), (1, 15, 16, 17, 33, 300, 1029, 4096)),
    (workload.Shape(64, 8, 128, 16, "bf16"), (1, 16, 17, 255, 257, 2048)),
    (workload.Shape(8, 8, 64, 16, "f32"), (128, 128, 5, 700)),
]


@pytest.mark.parametrize("shape,lens", CASES)
@pytest.mark.parametrize("N", [2, 3, 8])
def test_seq_split_matches_oracle(shape, lens, N):
    b = workload.make_decode_batch(shape, torch.tensor(lens, dtype=torch.int32), 17 + N, "cuda")
    hb = host_batch(b)   # host copy before the GPU appends; the oracle places the new rows itself
    ref = oracle.decode(hb["q"], hb["k_pool"], hb["v_pool"], hb["block_table"], hb["seq_lens"],
                        num_kv_heads=shape.num_kv_heads, dtype=dtype_code(shape))
    o, per_dev = _run_split(b, N)
    _assert_close(o, ref, f"seq split N={N}")
    P = shape.page_size
    for r, (lbt, ll, po, pl) in enumerate(per_dev):
        ll_h = ll.cpu().numpy()
        assert ll_h.tolist() == [seqsplit.local_len(L, N, r, P) for L in lens], r
        lse = pl.cpu().numpy()
        po_h = po.cpu().numpy()
        lbt_h = lbt.cpu().numpy()
        for j in range(len(lens)):
            if ll_h[j] == 0:
                assert np.all(np.isneginf(lse[j])) and np.all(po_h[j] == 0.0), (r, j)
                continue
            for h in range(0, shape.num_q_heads, max(1, shape.num_q_heads // 5)):
                o_ref, lse_ref = oracle.decode_range(hb["q"], hb["k_pool"], hb["v_pool"], lbt_h, ll_h, j, h, 0,
                                                     int(ll_h[j]), num_kv_heads=shape.num_kv_heads,
                                                     dtype=dtype_code(shape))
                assert abs(float(lse[j, h]) - lse_ref) <= LSE_ATOL, (r, j, h, float(lse[j, h]), lse_ref)
                assert np.max(np.abs(po_h[j, h] - o_ref)) <= ATOL, (r, j, h)


@pytest.mark.parametrize("shape,lens", CASES[:2])
def test_seq_split_one_device_is_bit_exact_vs_attn_decode(shape, lens):
    lens_t = torch.tensor(lens, dtype=torch.int32)
    b1 = workload.make_decode_batch(shape, lens_t, 5, "cuda")
    b2 = workload.make_decode_batch(shape, lens_t, 5, "cuda")
    o_split, _ = _run_split(b1, 1)
    s = hetis.make_shape(shape)
    B, H, D = b2.q.shape
    hetis.kv_append(s, b2.k_new, b2.v_new, b2.k_pool, b2.v_pool, b2.block_table, b2.seq_lens)
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, H, b2.max_seq_len), "cuda")
    o = torch.empty((B, H, D), dtype=torch.float32, device="cuda")
    hetis.attn_decode(s, b2.q, b2.k_pool, b2.v_pool, b2.block_table, b2.seq_lens, b2.max_seq_len, o, ws)
    torch.cuda.synchronize()
    assert torch.equal(o_split, o)


def test_seq_merge_edge_cases_and_bf16_output():
    shape = workload.Shape(8, 8, 128, 16, "bf16")
    cs32, cs16 = hetis.make_shape(shape, "f32"), hetis.make_shape(shape, "bf16")
    B, H, D, N = 3, 8, 128, 4
    g = torch.Generator(device="cuda").manual_seed(3)
    o_parts = torch.randn((N, B, H, D), generator=g, device="cuda")
    lse = torch.randn((N, B, H), generator=g, device="cuda") * 5
    lse[1:, 0] = -math.inf          # request 0: only device 0 holds tokens
    o_parts[1:, 0] = 0.0
    o = torch.empty((B, H, D), device="cuda")
    hetis.seq_merge(cs32, o_parts, lse, o)
    o16 = torch.empty((B, H, D), dtype=torch.bfloat16, device="cuda")
    hetis.seq_merge(cs16, o_parts, lse, o16)
    torch.cuda.synchronize()
    assert torch.equal(o[0], o_parts[0, 0])                    # one live part: bit for bit
    assert torch.equal(o16, o.to(torch.bfloat16))              # bf16 O = RNE(fp32 O) (reading 9)
    op, lp = o_parts.double().cpu().numpy(), lse.double().cpu().numpy()
    for j in (1, 2):
        for h in range(H):
            ref, _ = oracle.lse_merge(op[:, j, h], lp[:, j, h])
            assert np.max(np.abs(o[j, h].double().cpu().numpy() - ref)) <= 1e-5


def test_seq_split_c5_shape_whole_output():
    """c5 (LLaMA2-13B heads, B = 16 x 32k tokens) split over 8 devices by sequence: every element of O against
    the fp64 oracle."""
    cfg = workload.CONFIGS["c5"]
    b = workload.make_decode_batch(cfg.shape, cfg.seq_lens(), cfg.seed, "cuda")
    hb = host_batch_once(b)
    o, _ = _run_split(b, 8)
    ref = oracle.decode(hb["q"], hb["k_pool"], hb["v_pool"], hb["block_table"], hb["seq_lens"],
                        num_kv_heads=cfg.shape.num_kv_heads, dtype=dtype_code(cfg.shape))
    del hb
    st = err_stats(o.cpu().numpy(), ref)
    print("parity c5 sequence split N=8", st)
    assert st["nonfinite"] == 0 and st["max_abs"] <= ATOL and st["rel_fro"] <= RTOL, st
