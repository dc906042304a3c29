"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Tolerance (north star / DESIGN.md §5): max |O - O_ref| <= 2e-3 and
||O - O_ref||_F / ||O_ref||_F <= 1e-2 over the whole fp32 O, no NaN/Inf.
Index and byte work is bit-exact: kv_append (memcmp against the oracle's host
placement), page-permutation and head-partition invariance of the GPU output,
L = 1 returning the V row, bf16 O == RNE(fp32 O).
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2509_08309_b200 import hetis, workload
from tests.helpers import dtype_code, err_stats, host_batch, host_batch_once, oracle_full, to_f64

pytestmark = pytest.mark.gpu

ATOL, RTOL = 2e-3, 1e-2
C = 256


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    hetis.lib()


def run_gpu(b: workload.DecodeBatch, o_dtype="f32", flags=0, append=True, o_stride_heads=None):
    s = hetis.make_shape(b.shape, o_dtype)
    B, x, D = b.q.shape
    if append:
        hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    L = b.max_seq_len
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), b.q.device)
    odt = torch.bfloat16 if o_dtype == "bf16" else torch.float32
    if o_stride_heads is None:
        o = torch.full((B, x, D), float("nan"), dtype=odt, device=b.q.device)
        hetis.attn_decode(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, o, ws, q_head_begin=b.q_begin,
                          flags=flags)
    else:
        big = torch.full((B, o_stride_heads, D), float("nan"), dtype=odt, device=b.q.device)
        hetis.attn_partial(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, ws, q_head_begin=b.q_begin,
                           flags=flags)
        view = big[:, b.q_begin:b.q_begin + x]
        hetis.attn_combine(s, b.seq_lens, L, view, ws, q_head_count=x, o_seq_stride=big.stride(0))
        o = big
    torch.cuda.synchronize()
    return o


def run_gpu_fused(b: workload.DecodeBatch, flags=0):
    """The bench's per-device step: hetis_attn_decode_append (append fused into the attention kernel) + combine."""
    s = hetis.make_shape(b.shape)
    B, x, D = b.q.shape
    L = b.max_seq_len
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), b.q.device)
    o = torch.full((B, x, D), float("nan"), dtype=torch.float32, device=b.q.device)
    hetis.attn_decode_append(s, b.q, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, o, ws,
                             flags=flags)
    torch.cuda.synchronize()
    del ws
    return o


def log_parity(tag: str, b: workload.DecodeBatch, st: dict):
    rec = {"case": tag, "q_heads": b.q_count, "q_begin": b.q_begin, "batch": int(b.q.shape[0]),
           "max_seq_len": b.max_seq_len, "elements": int(b.q.numel()), **st}
    print("parity", json.dumps(rec))
    path = os.environ.get("HETIS_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def assert_close(got, ref, what=""):
    st = err_stats(got.float().cpu().numpy() if isinstance(got, torch.Tensor) else got, ref)
    assert st["nonfinite"] == 0, (what, st)
    assert st["max_abs"] <= ATOL and st["rel_fro"] <= RTOL, (what, st)
    return st


def gpu_batch(H, Hkv, D, dtype, lens, seed, q_begin=0, q_count=None, rank_salt=0):
    shape = workload.Shape(H, Hkv, D, 16, dtype)
    return workload.make_decode_batch(shape, torch.tensor(lens, dtype=torch.int32), seed, "cuda", q_begin=q_begin,
                                      q_count=q_count, rank_salt=rank_salt)


EDGE_LENS = (1, 2, 15, 16, 17, 31, 33, C - 1, C, C + 1, 2 * C + 5, 1000)


# ------------------------------------------------------------------ c1: the parity config
def test_c1_two_virtual_devices_match_oracle_and_unsplit():
    cfg = workload.CONFIGS["c1"]
    full = workload.make_decode_batch(cfg.shape, cfg.seq_lens(), cfg.seed, "cuda")
    ref = oracle_full(full)
    o_full = run_gpu(full)
    assert_close(o_full, ref, "c1 unsplit")
    parts = []
    begin = 0
    for i, x in enumerate(cfg.split):
        part = workload.make_decode_batch(cfg.shape, cfg.seq_lens(), cfg.seed, "cuda", q_begin=begin, q_count=x,
                                          rank_salt=i + 1)
        parts.append(run_gpu(part))
        begin += x
    o_split = torch.cat(parts, dim=1)
    st = assert_close(o_split, ref, "c1 split")
    assert st["max_abs"] < 1e-5            # fp32 path: far inside the budget
    assert torch.equal(o_split, o_full)    # head partition invariance, bit-exact


# ------------------------------------------------------------------ edge lengths, all kernels
@pytest.mark.parametrize("H,Hkv,D,dtype", [(8, 8, 128, "bf16"), (16, 2, 128, "bf16"), (8, 8, 64, "f32"),
                                           (16, 4, 64, "bf16"), (8, 1, 128, "bf16"), (4, 2, 128, "f32"),
                                           (8, 4, 128, "bf16"), (8, 8, 64, "bf16")])
def test_edge_lengths_ragged(H, Hkv, D, dtype):
    b = gpu_batch(H, Hkv, D, dtype, EDGE_LENS, seed=H * 7 + D + Hkv)
    o = run_gpu(b)
    assert_close(o, oracle_full(b), f"{H}/{Hkv}/{D}/{dtype}")
    # L = 1: the output is the new token's V row, bit for bit
    j1 = EDGE_LENS.index(1)
    v = b.v_new[j1].float()
    for h in range(H):
        assert torch.equal(o[j1, h], v[h // (H // Hkv)])


def test_single_sequence_and_all_length_one():
    for lens in [(4096,), (1,) * 37]:
        b = gpu_batch(64, 8, 128, "bf16", lens, seed=len(lens))
        assert_close(run_gpu(b), oracle_full(b), str(lens[:2]))


# ------------------------------------------------------------------ closed-form cases on the GPU
def test_q_zero_and_identical_keys_give_mean():
    b = gpu_batch(16, 2, 128, "bf16", (300, 17, 1), seed=5)
    b.q.zero_()
    o = run_gpu(b)
    ref = oracle_full(b)
    assert_close(o, ref, "q=0")
    b2 = gpu_batch(8, 8, 128, "bf16", (700, 33), seed=6)
    key = b2.k_pool[b2.block_table[0, 0, 0].long(), 0].clone()      # history token 0 of request 0
    b2.k_pool.copy_(key.expand_as(b2.k_pool))
    b2.k_new.copy_(key.expand_as(b2.k_new))
    assert_close(run_gpu(b2), oracle_full(b2), "identical keys")


@pytest.mark.parametrize("H,Hkv", [(8, 8), (64, 8)])
def test_peaked_attention_catches_low_precision_p(H, Hkv):
    """K x 4 and one key = 8 q: a few tokens dominate; bf16-rounded P would miss 2e-3."""
    b = gpu_batch(H, Hkv, 128, "bf16", (2048, 513, 64), seed=77)
    b.k_pool.mul_(4)          # exact in bf16 (power of two)
    b.k_new.mul_(4)
    r = H // Hkv
    for j in range(3):
        for g in range(Hkv):
            page = b.block_table[j, g, 3].long()
            b.k_pool[page, 5] = (b.q[j, g * r] * 8)
    st = assert_close(run_gpu(b), oracle_full(b), "peaked")
    assert st["max_abs"] < 1e-3


# ------------------------------------------------------------------ bit-exact invariances
@pytest.mark.parametrize("H,Hkv", [(40, 40), (64, 8)])
def test_page_permutation_bit_identical(H, Hkv):
    b = gpu_batch(H, Hkv, 128, "bf16", (777, 2048, 16), seed=12)
    hetis.kv_append(hetis.make_shape(b.shape), b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    o1 = run_gpu(b, append=False)
    n = b.k_pool.shape[0]
    perm = torch.randperm(n, generator=torch.Generator().manual_seed(3)).cuda()
    kp = torch.empty_like(b.k_pool)
    vp = torch.empty_like(b.v_pool)
    kp[perm] = b.k_pool
    vp[perm] = b.v_pool
    bt = b.block_table.clone()
    m = bt >= 0
    bt[m] = perm[bt[m].long()].int()
    b2 = workload.DecodeBatch(b.shape, 0, H, b.q, b.k_new, b.v_new, kp, vp, bt, b.seq_lens)
    o2 = run_gpu(b2, append=False)
    assert torch.equal(o1, o2)


@pytest.mark.parametrize("H,Hkv,splits", [(40, 40, [(16, 8, 8, 4, 4), (20, 20), (5,) * 8]),
                                          (64, 8, [(32, 32), (16,) * 4, (8,) * 8, (48, 16)])])
def test_head_partition_bit_identical(H, Hkv, splits):
    shape = workload.Shape(H, Hkv, 128, 16, "bf16")
    lens = torch.tensor([600, 5, 1300, 256], dtype=torch.int32)
    full = workload.make_decode_batch(shape, lens, 21, "cuda")
    o_full = run_gpu(full)
    for split in splits:
        begin, outs = 0, []
        for i, x in enumerate(split):
            part = workload.make_decode_batch(shape, lens, 21, "cuda", q_begin=begin, q_count=x, rank_salt=i + 1)
            outs.append(run_gpu(part))
            begin += x
        assert torch.equal(torch.cat(outs, 1), o_full), split


def test_deterministic_repeat():
    b = gpu_batch(64, 8, 128, "bf16", (2048, 999, 1), seed=31)
    o1 = run_gpu(b)
    o2 = run_gpu(b, append=False)
    assert torch.equal(o1, o2)


@pytest.mark.parametrize("lens", [(1500, 40, 257), (2048,) * 300, (700, 1, 4095) * 40])
def test_tensor_core_vs_cuda_core_gqa(lens):
    """Both tensor-core work decompositions (whole items per warp; shared ring + CTA merge) and the
    CUDA-core kernel agree with the oracle and with each other (different summation order only)."""
    b = gpu_batch(64, 8, 128, "bf16", lens, seed=41)
    o_tc = run_gpu(b)
    o_ring = run_gpu(b, flags=hetis.ATTN_TC_SHARED_RING, append=False)
    o_simt = run_gpu(b, flags=hetis.ATTN_FORCE_SIMT, append=False)
    ref = oracle_full(b)                          # every batch, incl. 300 x 2048 and (700, 1, 4095) x 40
    log_parity(f"gqa-batch-{len(lens)}/tc", b, assert_close(o_tc, ref, "tc"))
    assert_close(o_ring, ref, "tc shared ring")
    assert_close(o_simt, ref, "simt")
    assert torch.isfinite(o_tc).all() and torch.isfinite(o_ring).all()
    assert (o_tc - o_ring).abs().max().item() < 1e-5
    assert (o_tc - o_simt).abs().max().item() < 1e-4


def test_gqa_equals_expanded_mha_on_gpu():
    b = gpu_batch(16, 2, 128, "bf16", (900, 31), seed=44)
    o_gqa = run_gpu(b)
    r = 8
    bt = b.block_table.repeat_interleave(r, dim=1).contiguous()
    shape = workload.Shape(16, 16, 128, 16, "bf16")
    b2 = workload.DecodeBatch(shape, 0, 16, b.q, b.k_new.repeat_interleave(r, 1).contiguous(),
                              b.v_new.repeat_interleave(r, 1).contiguous(), b.k_pool, b.v_pool, bt, b.seq_lens)
    o_mha = run_gpu(b2, append=False)
    assert (o_gqa - o_mha).abs().max().item() < 1e-4


def test_bf16_output_is_rne_of_fp32():
    b = gpu_batch(64, 8, 128, "bf16", (1024, 77), seed=51)
    o32 = run_gpu(b)
    o16 = run_gpu(b, o_dtype="bf16", append=False)
    assert torch.equal(o16, o32.to(torch.bfloat16))


def test_strided_output_places_heads_in_full_tensor():
    b = gpu_batch(40, 40, 128, "bf16", (300, 1), seed=52, q_begin=16, q_count=8)
    o = run_gpu(b, o_stride_heads=40)
    dense = run_gpu(b, append=False)
    assert torch.equal(o[:, 16:24], dense)
    assert torch.isnan(o[:, :16]).all() and torch.isnan(o[:, 24:]).all()


# ------------------------------------------------------------------ kv append bit-exactness
@pytest.mark.parametrize("dtype,D,Hkv", [("bf16", 128, 8), ("f32", 64, 4), ("bf16", 64, 2)])
def test_kv_append_memcmp_against_oracle_placement(dtype, D, Hkv):
    b = gpu_batch(Hkv, Hkv, D, dtype, (1, 16, 17, 33, 4096, 255), seed=61)
    before = workload.to_numpy_bits(b.k_pool).copy()
    hb = host_batch(b)                         # oracle placement on host copies
    hetis.kv_append(hetis.make_shape(b.shape), b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    torch.cuda.synchronize()
    gk = workload.to_numpy_bits(b.k_pool)
    gv = workload.to_numpy_bits(b.v_pool)
    assert np.array_equal(gk.view(np.uint8), hb["k_pool"].view(np.uint8))
    assert np.array_equal(gv.view(np.uint8), hb["v_pool"].view(np.uint8))
    changed = np.any(gk.view(np.uint8).reshape(gk.shape[0], 16, -1) != before.view(np.uint8).reshape(
        gk.shape[0], 16, -1), axis=2)
    assert changed.sum() == 6 * Hkv


# ------------------------------------------------------------------ full-size configs, whole O against the oracle
FULL_SIZE_CASES = [("c2", 1, 0), ("c3", 1, 0), ("c3", 8, 5), ("c4", 5, 0), ("c4", 5, 1), ("c4", 5, 2), ("c4", 5, 3),
                   ("c4", 5, 4), ("c5", 8, 3)]


@pytest.mark.parametrize("name,n_dev,rank", FULL_SIZE_CASES)
def test_full_size_config_whole_output(name, n_dev, rank):
    """T10: one rank's share of a config at FULL size (c2 and c3 whole; every share of c4's
    16/8/8/4/4 split; an 8-GPU share of c3 and c5), run with the bench's launch (kv_append fused into the
    attention kernel, then the combine), compared with the fp64 oracle on EVERY element of O.  The max-abs
    location (request, local head, dim) is logged (HETIS_PARITY_LOG) and printed."""
    cfg = workload.CONFIGS[name]
    split = cfg.head_split(n_dev)
    begin = sum(split[:rank])
    b = workload.make_decode_batch(cfg.shape, cfg.seq_lens(), cfg.seed, "cuda", q_begin=begin,
                                   q_count=split[rank], rank_salt=rank)
    hb = host_batch_once(b)                       # host copies taken BEFORE the GPU append; oracle places the row
    o = run_gpu_fused(b)
    ref = oracle.decode(hb["q"], hb["k_pool"], hb["v_pool"], hb["block_table"], hb["seq_lens"],
                        num_kv_heads=b.kv_count, dtype=dtype_code(b.shape))
    del hb
    st = assert_close(o, ref, f"{name} N={n_dev} rank {rank}")
    log_parity(f"{name}/N{n_dev}/rank{rank}", b, st)


# ------------------------------------------------------------------ per-request (dispatcher) plans via work units
def _random_per_request_plan(B, H, r, N, seed):
    """x[j][i]: a random composition of request j's H / r kv groups over N devices (multiples of r, sum H)."""
    g = np.random.default_rng(seed)
    x = np.zeros((B, N), dtype=np.int32)
    for j in range(B):
        cuts = np.sort(g.integers(0, H // r + 1, size=N - 1))
        x[j] = np.diff(np.concatenate([[0], cuts, [H // r]])) * r
    return x


def _units_tensor(plan, dev):
    units = plan.units(dev)
    return torch.tensor(units, dtype=torch.int32, device="cuda").reshape(-1, 2), len(units)


def test_per_request_plan_units_bit_identical_to_unsplit():
    """A ragged per-request plan from the Eq. 7 dispatcher, each device's units run by
    hetis_attn_decode_units -- ONE attention launch + ONE combine on the full [B][H][d] q / o, no
    caller-side gathers -- reassembles to exactly the unsplit result and matches the oracle."""
    from paper_2509_08309_b200 import dispatch as dp
    shape = workload.LLAMA2_70B
    lens = (600, 5, 1300, 256, 2048, 77)
    full = gpu_batch(64, 8, 128, "bf16", lens, seed=91)
    o_full = run_gpu(full)                                       # appends the new tokens, then attends
    devs = [dp.DeviceState(0, 0, 1e12, True, dp.AttentionCost(1e-8, 1e-11, 5e-6)),
            dp.DeviceState(0, 0, 1e12, False, dp.AttentionCost(2e-8, 3e-11, 5e-6, gamma=1e-9, beta=2e-6)),
            dp.DeviceState(0, 0, 1e12, True, dp.AttentionCost(1.5e-8, 2e-11, 5e-6))]
    out = dp.dispatch(devs, list(lens), H=64, r=8)
    s = hetis.make_shape(shape)
    plan = hetis.plan_create(s, 3, dp.plan_rows(out.x), per_request=True, num_seqs=len(lens))
    assembled = torch.full_like(o_full, float("nan"))
    seen = 0
    for dev in range(3):
        units, U = _units_tensor(plan, dev)
        if U == 0:
            continue
        ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, U, shape.r, full.max_seq_len), "cuda")
        mine = torch.full_like(o_full, float("nan"))
        hetis.attn_decode_units(s, units, full.q, full.k_pool, full.v_pool, full.block_table, full.seq_lens,
                                full.max_seq_len, mine, ws)
        torch.cuda.synchronize()
        owned = torch.zeros(o_full.shape[:2], dtype=torch.bool, device="cuda")
        for j, g in plan.units(dev):
            owned[j, g * shape.r:(g + 1) * shape.r] = True
        assert torch.isnan(mine[~owned]).all(), dev                 # nothing outside the device's units is written
        assembled[owned] = mine[owned]
        seen += U
    assert seen == len(lens) * 8
    assert torch.equal(assembled, o_full)
    assert_close(assembled, oracle_full(full), "per-request plan")


@pytest.mark.parametrize("H,Hkv,D,dtype,fused,flags", [(64, 8, 128, "bf16", True, 0), (40, 40, 128, "bf16", True, 0),
                                                       (16, 4, 64, "bf16", False, 0), (8, 8, 64, "f32", False, 0),
                                                       (16, 2, 128, "f32", False, 0),
                                                       (64, 8, 128, "bf16", True, hetis.ATTN_FUSED_MERGE),
                                                       (16, 4, 64, "bf16", False, hetis.ATTN_FUSED_MERGE)])
def test_units_random_plans_all_kernels(H, Hkv, D, dtype, fused, flags):
    """hetis_attn_decode_units on random per-request plans over 3 devices, every kernel family (per-warp
    tensor-core GQA, CUDA-core MHA, fp32): the union of the devices' outputs is bit-identical to the unsplit
    single-launch result, and with the append fused the pools end bit-identical to hetis_kv_append's."""
    lens = (1, 17, 256, 257, 1000, 33, 700, 2)
    r = H // Hkv
    full = gpu_batch(H, Hkv, D, dtype, lens, seed=17)
    o_full = run_gpu(full)
    fresh = gpu_batch(H, Hkv, D, dtype, lens, seed=17)           # same bits, pools without the new token
    x = _random_per_request_plan(len(lens), H, r, 3, seed=H + D)
    s = hetis.make_shape(full.shape)
    plan = hetis.plan_create(s, 3, x.reshape(-1).tolist(), per_request=True, num_seqs=len(lens))
    out = torch.full_like(o_full, float("nan"))
    for dev in range(3):
        units, U = _units_tensor(plan, dev)
        ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, max(U, 1), r, full.max_seq_len), "cuda")
        b = fresh if fused else full
        hetis.attn_decode_units(s, units, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, b.max_seq_len, out, ws,
                                k_new=b.k_new if fused else None, v_new=b.v_new if fused else None, flags=flags)
    torch.cuda.synchronize()
    assert torch.equal(out, o_full)
    if fused:
        assert torch.equal(fresh.k_pool.view(torch.int16), full.k_pool.view(torch.int16))
        assert torch.equal(fresh.v_pool.view(torch.int16), full.v_pool.view(torch.int16))


def test_units_argument_errors():
    full = gpu_batch(64, 8, 128, "bf16", (5, 9), seed=3)
    s = hetis.make_shape(full.shape)
    units = torch.tensor([[0, 1], [1, 7]], dtype=torch.int32, device="cuda")
    o = torch.empty((2, 64, 128), device="cuda")
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, 2, 8, full.max_seq_len), "cuda")
    with pytest.raises(hetis.HetisError) as e:       # pipelined launches are not supported for units
        hetis.attn_decode_units(s, units, full.q, full.k_pool, full.v_pool, full.block_table, full.seq_lens,
                                full.max_seq_len, o, ws, flags=hetis.ATTN_PIPELINED)
    assert e.value.name == "HETIS_E_UNSUPPORTED"
    small = hetis.alloc_workspace(256, "cuda")
    with pytest.raises(hetis.HetisError) as e:
        hetis.attn_decode_units(s, units, full.q, full.k_pool, full.v_pool, full.block_table, full.seq_lens,
                                full.max_seq_len, o, small)
    assert e.value.name == "HETIS_E_WORKSPACE"
    with pytest.raises(ValueError):                  # q must hold every head
        hetis.attn_decode_units(s, units, full.q[:, :8].contiguous(), full.k_pool, full.v_pool, full.block_table,
                                full.seq_lens, full.max_seq_len, o, ws)


@pytest.mark.parametrize("name", ["c3", "c2"])
def test_head_partition_bit_identical_at_config_size(name):
    """The c3 / c2 batch split over 2, 4 and 8 ranks (each rank's share generated on its own) reassembles
    bit for bit to the single-device result: the per-warp work claiming and the CTA item dealing never
    change an item's arithmetic."""
    cfg = workload.CONFIGS[name]
    full = workload.make_decode_batch(cfg.shape, cfg.seq_lens(), cfg.seed, "cuda")
    o_full = run_gpu(full)
    del full
    for n in (2, 4, 8):
        split = cfg.head_split(n)
        begin, outs = 0, []
        for i, x in enumerate(split):
            part = workload.make_decode_batch(cfg.shape, cfg.seq_lens(), cfg.seed, "cuda", q_begin=begin, q_count=x,
                                              rank_salt=i + 1)
            outs.append(run_gpu(part))
            del part
            begin += x
        assert torch.equal(torch.cat(outs, 1), o_full), n


# ------------------------------------------------------------------ work distribution does not change bits
@pytest.mark.parametrize("lens", [(1, 255, 256, 257, 3000, 17), tuple([2048] * 96), (5,)])
def test_device_claim_flag_is_bit_identical(lens):
    """Device-wide item claiming (the default; HETIS_ATTN_DEVICE_CLAIM forces it and turns group mode off),
    the CTA-local deal with stealing of the last 5% (HETIS_ATTN_STATIC_DEAL) and group mode hand items to
    different warps; an item's arithmetic depends on L_j only, so O is identical -- also over back-to-back
    launches, which exercises the self-resetting device-wide counter."""
    b = gpu_batch(64, 8, 128, "bf16", lens, 71)
    s = hetis.make_shape(b.shape)
    hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    B, x, D = b.q.shape
    L = b.max_seq_len
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), "cuda")
    outs = []
    SD, DC = hetis.ATTN_STATIC_DEAL, hetis.ATTN_DEVICE_CLAIM
    for flags in (0, DC, SD, DC, 0, SD, SD, 0):
        o = torch.full((B, x, D), float("nan"), device="cuda")
        hetis.attn_decode(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, o, ws, flags=flags)
        outs.append(o)
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


# ------------------------------------------------------------------ combine arithmetic is launch-shape independent
@pytest.mark.parametrize("H,Hkv,D", [(40, 40, 128), (64, 8, 128), (8, 8, 64)])
def test_combine_narrow_and_wide_launches_give_identical_rows(H, Hkv, D):
    """The combine folds a request with <= 16 splits with one thread group whatever the launch shape: a
    batch whose longest request has > 16 splits launches one block per row (wide), a batch without one
    launches four rows per block (narrow).  The same requests must get bit-identical rows either way."""
    dt = "f32" if D == 64 else "bf16"
    lens = (300, 1029, 17, 4096, 5000)          # 2, 5, 1, 16 and 20 splits of 256
    b = gpu_batch(H, Hkv, D, dt, lens, 83)
    s = hetis.make_shape(b.shape)
    hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    wide = run_gpu(b, append=False)                                          # 20 splits present: wide launch
    first4 = workload.DecodeBatch(b.shape, 0, H, b.q[:4].contiguous(), b.k_new[:4].contiguous(),
                                  b.v_new[:4].contiguous(), b.k_pool, b.v_pool, b.block_table[:4].contiguous(),
                                  b.seq_lens[:4].contiguous())
    narrow = run_gpu(first4, append=False)                                   # <= 16 splits: narrow launch
    assert torch.equal(wide[:4], narrow)
    assert_close(wide, oracle_full(b), "combine (wide launch) vs oracle")


def test_combine_shared_memory_staged_matches_register_staged():
    """Launches with more rows than one wave of the register-staged combine use the shared-memory staged
    one (bulk copies of the split rows, the same fold code): a 5120-row batch (staged) and its first 6
    requests (384 rows, register-staged) give bit-identical rows for those requests, for f32 and bf16 O."""
    lens = tuple(int(v) for v in (1 + (torch.arange(80) * 977) % 4000))    # 1 .. 16 splits, ragged
    b = gpu_batch(64, 8, 128, "bf16", lens, 29)
    hetis.kv_append(hetis.make_shape(b.shape), b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    for odt in ("f32", "bf16"):
        big = run_gpu(b, o_dtype=odt, append=False)
        sub = workload.DecodeBatch(b.shape, 0, 64, b.q[:6].contiguous(), b.k_new[:6].contiguous(),
                                   b.v_new[:6].contiguous(), b.k_pool, b.v_pool, b.block_table[:6].contiguous(),
                                   b.seq_lens[:6].contiguous())
        small = run_gpu(sub, o_dtype=odt, append=False)
        assert torch.equal(big[:6].view(torch.int16), small.view(torch.int16)), odt
        if odt == "f32":
            assert_close(big, oracle_full(b), "staged combine vs oracle")


# ------------------------------------------------------------------ MHA on tensor cores (HETIS_ATTN_MHA_TC)
@pytest.mark.parametrize("D", [128, 64])
@pytest.mark.parametrize("peaked", [False, True])
def test_mha_on_tensor_cores_matches_oracle(D, peaked):
    """r = 1 on the per-warp tensor-core kernel (one valid MMA row, P carried as P_hi + P_lo): within the
    north-star tolerance of the oracle, including peaked keys (K x 4) that would fail a bf16-rounded P."""
    lens = (1, 15, 16, 17, 255, 256, 257, 1029)
    b = gpu_batch(8, 8, D, "bf16", lens, seed=91)
    if peaked:
        b.k_pool.mul_(4)
        b.k_new.mul_(4)
    o_tc = run_gpu(b, flags=hetis.ATTN_MHA_TC)
    o_simt = run_gpu(b, append=False)
    ref = oracle_full(b)
    assert_close(o_tc, ref, "mha tc")
    assert (o_tc - o_simt).abs().max().item() < 1e-3
    # L = 1 returns the V row bit for bit on the tensor-core path too
    v_row = b.v_new[0].float()
    assert torch.equal(o_tc[0], v_row)


@pytest.mark.parametrize("D", [128, 64])
@pytest.mark.parametrize("peaked", [False, True])
def test_mha_per_warp_cuda_cores_matches_oracle(D, peaked):
    """bf16 MHA's default: the per-warp kernel with the CUDA-core consumer (swizzled TMA pages, one warp per
    16-page item, consumer refill, device-wide claiming), d = 128 and 64: within the north-star tolerance of
    the oracle (peaked keys too) and of the shared-ring CUDA-core kernel; L = 1 returns the V row bit for bit;
    the launch is bit-identical whatever claims the items (default, forced device claim, static deal)."""
    lens = (1, 15, 16, 17, 255, 256, 257, 1029, 4096, 700)
    b = gpu_batch(8, 8, D, "bf16", lens, seed=93)
    if peaked:
        b.k_pool.mul_(4)
        b.k_new.mul_(4)
    o_pw = run_gpu(b)
    o_ring = run_gpu(b, append=False, flags=hetis.ATTN_TC_SHARED_RING)
    ref = oracle_full(b)
    assert_close(o_pw, ref, "mha per-warp cuda cores")
    assert (o_pw - o_ring).abs().max().item() < 1e-3
    assert torch.equal(o_pw[0], b.v_new[0].float())
    for flags in (hetis.ATTN_DEVICE_CLAIM, hetis.ATTN_STATIC_DEAL):
        assert torch.equal(run_gpu(b, append=False, flags=flags), o_pw), flags


def test_mha_per_warp_head_partition_bit_identical():
    """Head partition (c4's uneven 16/8/8/4/4) reproduces the unsplit result bit for bit on the default MHA
    kernel (an item's arithmetic depends on L_j only)."""
    shape = workload.Shape(40, 40, 128, 16, "bf16")
    lens = torch.tensor([600, 5, 1300, 256, 3000], dtype=torch.int32)
    full = workload.make_decode_batch(shape, lens, 29, "cuda")
    o_full = run_gpu(full)
    begin, outs = 0, []
    for i, x in enumerate((16, 8, 8, 4, 4)):
        part = workload.make_decode_batch(shape, lens, 29, "cuda", q_begin=begin, q_count=x, rank_salt=i + 1)
        outs.append(run_gpu(part))
        begin += x
    assert torch.equal(torch.cat(outs, 1), o_full)


def test_mha_tc_head_partition_bit_identical():
    shape = workload.Shape(40, 40, 128, 16, "bf16")
    lens = torch.tensor([600, 5, 1300, 256], dtype=torch.int32)
    full = workload.make_decode_batch(shape, lens, 23, "cuda")
    o_full = run_gpu(full, flags=hetis.ATTN_MHA_TC)
    begin, outs = 0, []
    for i, x in enumerate((16, 8, 8, 4, 4)):
        part = workload.make_decode_batch(shape, lens, 23, "cuda", q_begin=begin, q_count=x, rank_salt=i + 1)
        outs.append(run_gpu(part, flags=hetis.ATTN_MHA_TC))
        begin += x
    assert torch.equal(torch.cat(outs, 1), o_full)


# ------------------------------------------------------------------ kv_append fused into the attention kernel
@pytest.mark.parametrize("H,Hkv,D,dtype,flags", [
    (40, 40, 128, "bf16", 0),                          # CUDA-core MHA
    (64, 8, 128, "bf16", 0),                           # per-warp tensor-core GQA
    (16, 4, 64, "bf16", 0),
    (8, 8, 64, "f32", 0),                              # fp32 CUDA-core
    (4, 2, 128, "f32", 0),
    (40, 40, 128, "bf16", hetis.ATTN_MHA_TC),          # MHA on the per-warp tensor-core kernel
    (64, 8, 128, "bf16", hetis.ATTN_TC_SHARED_RING),   # shared-ring tensor-core kernel
    (16, 2, 128, "bf16", hetis.ATTN_FORCE_SIMT),
])
def test_fused_append_bit_identical_to_append_then_attention(H, Hkv, D, dtype, flags):
    """hetis_attn_decode_append (the new rows patched into the landed page in shared memory and stored into
    the pool by the same kernel) == hetis_kv_append + hetis_attn_decode: O and both pools bit for bit."""
    lens = EDGE_LENS
    a = gpu_batch(H, Hkv, D, dtype, lens, seed=97)
    b = gpu_batch(H, Hkv, D, dtype, lens, seed=97)
    s = hetis.make_shape(a.shape)
    B, x, _ = a.q.shape
    L = a.max_seq_len
    o_ref = run_gpu(a, flags=flags)                                   # kv_append, then attention + combine
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), "cuda")
    o = torch.full((B, x, D), float("nan"), device="cuda")
    hetis.attn_decode_append(s, b.q, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, o, ws,
                             flags=flags)
    torch.cuda.synchronize()
    assert torch.equal(o, o_ref)
    bits = lambda t: t.view(torch.int16) if t.dtype == torch.bfloat16 else t.view(torch.int32)
    assert torch.equal(bits(b.k_pool), bits(a.k_pool)) and torch.equal(bits(b.v_pool), bits(a.v_pool))
    # a second step reads the appended rows from the pools like any other token
    o2 = torch.full_like(o, float("nan"))
    hetis.attn_decode(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, o2, ws, flags=flags)
    torch.cuda.synchronize()
    assert torch.equal(o2, o_ref)


FM = hetis.ATTN_FUSED_MERGE


@pytest.mark.parametrize("H,Hkv,D,flags,odt", [(64, 8, 128, FM, "f32"), (16, 2, 128, FM, "f32"), (16, 4, 64, FM, "f32"),
                                              (8, 1, 128, FM, "bf16"), (40, 40, 128, FM | hetis.ATTN_MHA_TC, "f32"),
                                              (8, 4, 128, FM | hetis.ATTN_DEVICE_CLAIM, "bf16")])
def test_merge_fused_into_attention_bit_identical_to_combine_kernel(H, Hkv, D, flags, odt):
    """hetis_attn_decode with HETIS_ATTN_FUSED_MERGE and the per-warp tensor-core kernel is ONE launch: the
    last warp of a (request, kv head) pair folds the pair's splits (one split: the rows straight from registers).  Its O is bit-identical
    to the two-kernel path (hetis_attn_partial + hetis_attn_combine) for one split, the narrow fold (<= 16
    splits) and the wide fold (17, 20, 36 splits), and a second launch on the same workspace (the per-pair
    counters returned to zero) repeats it."""
    lens = EDGE_LENS + (4097, 5000, 9000)
    b = gpu_batch(H, Hkv, D, "bf16", lens, seed=123)
    s = hetis.make_shape(b.shape, odt)
    assert hetis.attn_decode_launches(s, flags) == 1
    B, x, _ = b.q.shape
    L = b.max_seq_len
    hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    odtype = torch.bfloat16 if odt == "bf16" else torch.float32
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), "cuda")
    ref = torch.full((B, x, D), float("nan"), dtype=odtype, device="cuda")
    hetis.attn_partial(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, ws, flags=flags)
    hetis.attn_combine(s, b.seq_lens, L, ref, ws)
    for rep in range(2):
        got = torch.full_like(ref, float("nan"))
        n0 = hetis.launch_count()
        hetis.attn_decode(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, got, ws, flags=flags)
        assert hetis.launch_count() - n0 == 1
        torch.cuda.synchronize()
        assert torch.equal(got.view(torch.int16), ref.view(torch.int16)), rep
    if odt == "f32":
        assert_close(got, oracle_full(b), "fused merge")


GROUP_LENS = (1, 15, 16, 17, 255, 256, 257, 511, 1000, 1024, 1500, 1793, 2000, 2047, 2048, 700)


@pytest.mark.parametrize("H,Hkv,D,odt,B", [(64, 8, 128, "f32", 16), (16, 2, 128, "bf16", 64), (16, 4, 64, "f32", 37),
                                           (8, 1, 128, "f32", 148), (8, 1, 128, "bf16", 149), (64, 8, 128, "f32", 19)])
def test_group_mode_bit_identical_to_combine_kernel(H, Hkv, D, odt, B):
    """Merge-fused launches with at most one (request, kv head) pair per SM and <= 8 splits per pair run in
    group mode (CTA c = pair c, warp w = split w, partials staged in shared memory and folded after one CTA
    barrier; 148 pairs is the boundary, 149 and 152 fall back to the last-arriver merge).  Every form is
    bit-identical to hetis_attn_partial + hetis_attn_combine, including ragged tails, one-split pairs
    (L <= 256) and the full 8 splits (L = 2048), for f32 and bf16 O; the append-fused form too; the oracle
    agrees within tolerance."""
    lens = [GROUP_LENS[i % len(GROUP_LENS)] for i in range(B)]
    fresh = gpu_batch(H, Hkv, D, "bf16", lens, seed=321)
    b = gpu_batch(H, Hkv, D, "bf16", lens, seed=321)
    s = hetis.make_shape(b.shape, odt)
    x = b.q.shape[1]
    L = 2048
    hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    odtype = torch.bfloat16 if odt == "bf16" else torch.float32
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), "cuda")
    ref = torch.full((B, x, D), float("nan"), dtype=odtype, device="cuda")
    hetis.attn_partial(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, ws)
    hetis.attn_combine(s, b.seq_lens, L, ref, ws)
    group = B * (x // (H // Hkv)) <= 148   # B200: one pair per SM
    assert hetis.attn_decode_launches_for(s, B, x, L, 0) == (1 if group else 2)
    assert hetis.attn_decode_launches_for(s, B, x, L, hetis.ATTN_NO_GROUP_MODE) == 2
    for flags in (0, FM, FM | hetis.ATTN_NO_GROUP_MODE):
        for rep in range(2):
            got = torch.full_like(ref, float("nan"))
            n0 = hetis.launch_count()
            hetis.attn_decode(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, got, ws, flags=flags)
            assert hetis.launch_count() - n0 == hetis.attn_decode_launches_for(s, B, x, L, flags)
            torch.cuda.synchronize()
            assert torch.equal(got.view(torch.int16), ref.view(torch.int16)), (flags, rep)
    # the append fused as well (the bench's one-kernel step): same O, same pools
    got = torch.full_like(ref, float("nan"))
    hetis.attn_decode_append(s, fresh.q, fresh.k_new, fresh.v_new, fresh.k_pool, fresh.v_pool, fresh.block_table,
                             fresh.seq_lens, L, got, ws)
    torch.cuda.synchronize()
    assert torch.equal(got.view(torch.int16), ref.view(torch.int16))
    assert torch.equal(fresh.k_pool.view(torch.int16), b.k_pool.view(torch.int16))
    assert torch.equal(fresh.v_pool.view(torch.int16), b.v_pool.view(torch.int16))
    if odt == "f32":
        assert_close(got, oracle_full(b), "group mode")


def test_group_mode_randomized_shapes_bit_identical():
    """30 seeded random launches around the group-mode boundary (r in {2, 4, 8}, d in {64, 128}, 1..160
    pairs, ragged lengths up to 2048 with 1-split and 8-split pairs, f32 / bf16 O): the default one-call
    decode (group mode where it qualifies, else attention + combine), the last-arriver merge and the
    two-kernel path give the same bits."""
    import random
    rnd = random.Random(2509)
    for case in range(30):
        r = rnd.choice([2, 4, 8])
        D = rnd.choice([64, 128])
        Hkv = rnd.choice([1, 2, 4])
        B = rnd.randint(1, max(1, 160 // Hkv))
        lens = [rnd.choice([1, rnd.randint(1, 256), rnd.randint(1, 2048), 2048]) for _ in range(B)]
        odt = rnd.choice(["f32", "bf16"])
        b = gpu_batch(Hkv * r, Hkv, D, "bf16", lens, seed=1000 + case)
        s = hetis.make_shape(b.shape, odt)
        x = b.q.shape[1]
        L = max(lens)
        hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
        ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), "cuda")
        odtype = torch.bfloat16 if odt == "bf16" else torch.float32
        ref = torch.full((B, x, D), float("nan"), dtype=odtype, device="cuda")
        hetis.attn_partial(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, ws)
        hetis.attn_combine(s, b.seq_lens, L, ref, ws)
        for flags in (0, FM | hetis.ATTN_NO_GROUP_MODE):
            got = torch.full_like(ref, float("nan"))
            hetis.attn_decode(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, got, ws, flags=flags)
            torch.cuda.synchronize()
            assert torch.equal(got.view(torch.int16), ref.view(torch.int16)), (case, r, D, Hkv, B, odt, flags)


def test_claim_modes_randomized_launches_bit_identical():
    """24 seeded random launches from one item per worker to several (r in {1, 2, 4, 8}: bf16 MHA on the
    per-warp CUDA-core consumer and GQA on the tensor-core one; d in {64, 128}; up to ~6000 items): the
    default (consumer refill + device-wide claiming), HETIS_ATTN_STATIC_DEAL and HETIS_ATTN_DEVICE_CLAIM hand
    items to different warps and CTAs and give the same bits, twice in a row on one workspace."""
    import random
    rnd = random.Random(830)
    for case in range(24):
        r = rnd.choice([1, 2, 4, 8])
        D = rnd.choice([64, 128])
        Hkv = rnd.choice([2, 4, 8])
        B = rnd.randint(1, 96)
        lens = [rnd.randint(1, 4096) for _ in range(B)]
        b = gpu_batch(Hkv * r, Hkv, D, "bf16", lens, seed=2000 + case)
        s = hetis.make_shape(b.shape)
        x = b.q.shape[1]
        L = max(lens)
        hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
        ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), "cuda")
        outs = []
        for flags in (0, hetis.ATTN_STATIC_DEAL, hetis.ATTN_DEVICE_CLAIM, 0):
            o = torch.full((B, x, D), float("nan"), device="cuda")
            hetis.attn_partial(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, ws, flags=flags)
            hetis.attn_combine(s, b.seq_lens, L, o, ws)
            outs.append(o)
        torch.cuda.synchronize()
        for k, o in enumerate(outs[1:]):
            assert torch.equal(o, outs[0]), (case, r, D, Hkv, B, k)
        assert torch.isfinite(outs[0]).all()


@pytest.mark.parametrize("H,Hkv,D,B", [(64, 8, 128, 9), (16, 4, 64, 40), (64, 8, 128, 40)])
def test_fused_merge_empty_requests_write_zeros(H, Hkv, D, B):
    """L_j = 0 (a device holding none of request j's tokens under a sequence split): the combine kernel writes
    o = 0; the one-kernel forms must too -- group mode (9 x 8 = 72 pairs) and the last-arriver merge (flag
    NO_GROUP_MODE, and 40 x 8 = 320 pairs where group mode does not apply) -- bit-identical to the two-kernel
    path on a batch mixing empty and non-empty requests."""
    lens = [(1 if i % 3 == 1 else GROUP_LENS[i % len(GROUP_LENS)]) for i in range(B)]
    b = gpu_batch(H, Hkv, D, "bf16", lens, seed=77)
    b.seq_lens[1::3] = 0      # the generator needs L >= 1 (the new token); these requests now hold no token
    s = hetis.make_shape(b.shape, "f32")
    x = b.q.shape[1]
    L = max(lens)
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), "cuda")
    ref = torch.full((B, x, D), float("nan"), device="cuda")
    hetis.attn_partial(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, ws)
    hetis.attn_combine(s, b.seq_lens, L, ref, ws)
    torch.cuda.synchronize()
    assert torch.all(ref[1::3] == 0)
    for flags in (0, FM, FM | hetis.ATTN_NO_GROUP_MODE):
        got = torch.full_like(ref, float("nan"))
        hetis.attn_decode(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, got, ws, flags=flags)
        torch.cuda.synchronize()
        assert torch.equal(got.view(torch.int32), ref.view(torch.int32)), flags


def test_decode_step_fused_append_matches_separate_calls():
    from paper_2509_08309_b200.step import DecodeStep
    shape = workload.LLAMA2_70B
    lens = torch.tensor([300, 17, 1, 1029], dtype=torch.int32)
    a = workload.make_decode_batch(shape, lens, 5, "cuda")
    b = workload.make_decode_batch(shape, lens, 5, "cuda")
    plan = hetis.plan_create(hetis.make_shape(shape), 1, [shape.num_q_heads])
    outs = []
    for batch, fused in ((a, False), (b, True)):
        st = DecodeStep(shape, plan, 0, len(lens), int(lens.max()), torch.device("cuda", 0))
        st.buf.q_shard.copy_(batch.q)
        st.buf.k_new.copy_(batch.k_new)
        st.buf.v_new.copy_(batch.v_new)
        if fused:
            o = st.append_attention(batch.k_pool, batch.v_pool, batch.block_table, batch.seq_lens)
        else:
            st.append(batch.k_pool, batch.v_pool, batch.block_table, batch.seq_lens)
            o = st.attention(batch.k_pool, batch.v_pool, batch.block_table, batch.seq_lens)
        outs.append(o.clone())
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    assert torch.equal(a.k_pool.view(torch.int16), b.k_pool.view(torch.int16))


# ------------------------------------------------------------------ pipelined steps (HETIS_ATTN_PIPELINED)
@pytest.mark.parametrize("H,Hkv,D,dtype,extra,large", [(64, 8, 128, "bf16", 0, False), (40, 40, 128, "bf16", 0, False),
                                                       (8, 8, 64, "f32", 0, False),
                                                       (40, 40, 128, "bf16", hetis.ATTN_MHA_TC, False),
                                                       (16, 4, 64, "bf16", 0, False), (64, 8, 128, "bf16", 0, True)])
def test_pipelined_steps_match_serial_steps(H, Hkv, D, dtype, extra, large):
    """Several decode steps (each appends one token) back to back on one stream, pipelined with two
    alternating workspaces, as a CUDA graph so consecutive kernels really overlap: every step's O and the
    final pools are bit-identical to the same steps run with the default (fully ordered) launches.
    large: 96 ragged requests (~5000 GQA items, >= 2 per worker), so pipelined launches also steal."""
    if large:
        lens0 = torch.tensor([200 + (i * 97) % 2800 for i in range(96)], dtype=torch.int32)
    else:
        lens0 = torch.tensor([1, 15, 16, 17, 255, 256, 900, 2047], dtype=torch.int32)
    n_steps = 6
    lens_max = lens0 + n_steps
    outs = {}
    for mode in ("serial", "pipelined"):
        shape = workload.Shape(H, Hkv, D, 16, dtype)
        b = workload.make_decode_batch(shape, lens_max, 111, "cuda")      # pages for every step's token
        s = hetis.make_shape(shape)
        B, x, _ = b.q.shape
        L = int(lens_max.max())
        ws = [hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, x, L), "cuda") for _ in range(2)]
        g = torch.Generator(device="cuda").manual_seed(7)
        kn = [torch.randn(b.k_new.shape, generator=g, device="cuda").to(b.k_new.dtype) for _ in range(n_steps)]
        vn = [torch.randn(b.v_new.shape, generator=g, device="cuda").to(b.v_new.dtype) for _ in range(n_steps)]
        sl = [(lens0 + i + 1).to("cuda") for i in range(n_steps)]
        o = [torch.empty((B, x, D), device="cuda") for _ in range(n_steps)]
        flags = (hetis.ATTN_PIPELINED if mode == "pipelined" else 0) | extra
        if mode == "serial" and H == Hkv and dtype == "bf16" and not extra & hetis.ATTN_MHA_TC:
            flags |= hetis.ATTN_TC_SHARED_RING   # pipelined bf16 MHA runs the shared-ring kernel: same arithmetic

        def run():
            for i in range(n_steps):
                w_ = ws[i % 2] if mode == "pipelined" else ws[0]
                hetis.attn_partial_append(s, b.q, kn[i], vn[i], b.k_pool, b.v_pool, b.block_table, sl[i], L, w_,
                                          flags=flags)
                hetis.attn_combine(s, sl[i], L, o[i], w_)

        k0, v0 = b.k_pool.clone(), b.v_pool.clone()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            run()
        for rep in range(3):                      # replays start from the same pools
            b.k_pool.copy_(k0)
            b.v_pool.copy_(v0)
            graph.replay()
            torch.cuda.synchronize()
            outs.setdefault(mode, []).append(([t.clone() for t in o], b.k_pool.clone(), b.v_pool.clone()))
    bits = lambda t: t.view(torch.int16) if t.dtype == torch.bfloat16 else t.view(torch.int32)   # NaN slack
    ref_o, ref_k, ref_v = outs["serial"][0]
    for mode in ("serial", "pipelined"):
        for os_, k, v in outs[mode]:
            for i in range(n_steps):
                assert torch.equal(os_[i], ref_o[i]), (mode, i)
            assert torch.equal(bits(k), bits(ref_k)) and torch.equal(bits(v), bits(ref_v)), mode


def test_check_tables_counts_contract_violations():
    b = gpu_batch(16, 4, 128, "bf16", (1, 17, 300, 1029), seed=7)
    s = hetis.make_shape(b.shape)
    assert hetis.check_tables(s, b.k_pool, b.block_table, b.seq_lens) == 0
    bt = b.block_table.clone()
    bt[2, 1, 3] = b.k_pool.shape[0]            # page id out of range, inside the request's pages
    bt[0, 0, 5] = 10 ** 6                      # beyond request 0's only page: never read -> not a violation
    assert hetis.check_tables(s, b.k_pool, bt, b.seq_lens) == 1
    sl = b.seq_lens.clone()
    sl[1] = 0                                  # empty request (reading 10)
    sl[3] = b.block_table.shape[2] * 16 + 1    # longer than its table
    assert hetis.check_tables(s, b.k_pool, b.block_table, sl) == 2
