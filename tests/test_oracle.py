"""Pins for the fp64 oracle (CPU only, `-m "not gpu"`).

The oracle (oracle/oracle.c) is the plain definition of Eq. 2b
read through head-granular pages.  Nothing here re-types its
loop: each test pins it to something else --
  * brute force with mpmath at 50 digits on tiny inputs (independent gather),
  * torch's fp64 scaled_dot_product_attention (library special case),
  * closed forms: L = 1, L = 2 (logistic), q = 0 / identical keys (mean of V),
    affine equivariance in V, the peaked (one-hot) limit, a hand-worked golden
    example (tests/golden/decode_l2_worked_example.json),
  * invariants: page permutation, head partition, joint token
    permutation, GQA == MHA with repeated kv heads, token split + LSE merge,
  * head-granular placement worked examples (tests/golden/kv_append_positions.json).
A plausible mistake (dropped 1/sqrt(d), wrong kv head h*r instead of h//r,
transposed pool index, off-by-one in the slot, missing max subtraction on
large scores, V/K swapped) fails at least one of them.
"""
from __future__ import annotations

import json
import math
import os

import mpmath as mp
import numpy as np
import pytest
import torch

import oracle
from paper_2509_08309_b200 import accounting, workload
from tests.helpers import dense_logical_kv, dtype_code, host_batch, small_batch, to_f64

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _oracle(hb, s: workload.Shape, kv_heads=None):
    return oracle.decode(hb["q"], hb["k_pool"], hb["v_pool"], hb["block_table"], hb["seq_lens"],
                         num_kv_heads=kv_heads or s.num_kv_heads, dtype=dtype_code(s))


def _brute_force(hb, s: workload.Shape):
    """mpmath (50 digits) softmax without max subtraction over an independently gathered dense cache."""
    mp.mp.dps = 50
    ks, vs = dense_logical_kv(hb, s.page_size)
    q = to_f64(hb["q"])
    B, H, D = q.shape
    r = s.num_q_heads // s.num_kv_heads
    out = np.zeros((B, H, D))
    for j in range(B):
        for h in range(H):
            K, V = ks[j, h // r], vs[j, h // r]
            scale = 1 / mp.sqrt(D)
            e = [mp.exp(mp.fsum(mp.mpf(q[j, h, k]) * mp.mpf(K[t, k]) for k in range(D)) * scale)
                 for t in range(K.shape[0])]
            Z = mp.fsum(e)
            for k in range(D):
                out[j, h, k] = float(mp.fsum(e[t] * mp.mpf(V[t, k]) for t in range(K.shape[0])) / Z)
    return out


@pytest.mark.parametrize("H,Hkv,D,dtype", [(4, 4, 4, "f32"), (8, 4, 8, "bf16"), (8, 2, 4, "f32"),
                                           (8, 1, 8, "bf16")])
def test_brute_force_tiny(H, Hkv, D, dtype):
    b = small_batch(H=H, Hkv=Hkv, D=D, P=4, dtype=dtype, lens=(1, 7, 40), seed=11 + H + D)
    hb = host_batch(b)
    got = _oracle(hb, b.shape)
    ref = _brute_force(hb, b.shape)
    assert np.max(np.abs(got - ref)) <= 1e-12


def test_torch_sdpa_fp64_c1_full_size():
    """Library special case: dense fp64 SDPA on the exact c1 config (fp32, d = 64, B = 4, L = 128)."""
    cfg = workload.CONFIGS["c1"]
    b = workload.make_decode_batch(cfg.shape, cfg.seq_lens(), cfg.seed, "cpu")
    hb = host_batch(b)
    got = _oracle(hb, cfg.shape)
    P = cfg.shape.page_size
    K = torch.from_numpy(to_f64(hb["k_pool"]))
    V = torch.from_numpy(to_f64(hb["v_pool"]))
    q = torch.from_numpy(to_f64(hb["q"]))
    bt = torch.from_numpy(hb["block_table"]).long()
    r = cfg.shape.r
    for j in range(cfg.batch):
        L = int(hb["seq_lens"][j])
        t = torch.arange(L)
        pages = bt[j][:, t // P]                      # [Hkv][L]
        Kd = K[pages, t % P]                          # [Hkv][L][D]
        Vd = V[pages, t % P]
        Kd = Kd.repeat_interleave(r, 0)
        Vd = Vd.repeat_interleave(r, 0)
        o = torch.nn.functional.scaled_dot_product_attention(q[j][:, None, :], Kd, Vd,
                                                             scale=1.0 / math.sqrt(cfg.shape.head_dim))
        assert torch.max(torch.abs(o[:, 0, :] - torch.from_numpy(got[j]))).item() <= 1e-12


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_torch_sdpa_fp64_gqa_ragged(dtype):
    b = small_batch(H=16, Hkv=2, D=64, P=16, dtype=dtype, lens=(1, 15, 16, 17, 33, 300), seed=5)
    hb = host_batch(b)
    got = _oracle(hb, b.shape)
    ks, vs = dense_logical_kv(hb, 16)
    q = torch.from_numpy(to_f64(hb["q"]))
    for j in range(6):
        for h in range(16):
            o = torch.nn.functional.scaled_dot_product_attention(
                q[j, h][None, None, :], torch.from_numpy(ks[j, h // 8])[None], torch.from_numpy(vs[j, h // 8])[None],
                scale=1.0 / 8.0)
            assert np.max(np.abs(o[0, 0].numpy() - got[j, h])) <= 1e-12


def test_golden_worked_example_l2():
    with open(os.path.join(GOLDEN, "decode_l2_worked_example.json")) as f:
        gx = json.load(f)
    # re-derive the fixture's digits from its closed form (guards the fixture itself)
    mp.mp.dps = 50
    w0 = 1 / (1 + mp.exp(-1 / mp.sqrt(2)))
    assert abs(w0 - mp.mpf(gx["expected_o"][0])) < mp.mpf("1e-45")
    D, P = gx["head_dim"], gx["page_size"]
    q = np.array([[gx["q"]]], dtype=np.float32)
    kp = np.full((2, P, D), np.nan, dtype=np.float32)
    vp = np.full((2, P, D), np.nan, dtype=np.float32)
    kp[1, :2] = gx["k"]
    vp[1, :2] = gx["v"]
    bt = np.array([[[1]]], dtype=np.int32)
    out = oracle.decode(q, kp, vp, bt, np.array([2], np.int32), num_kv_heads=1, dtype=oracle.F32)
    exp = np.array([float(x) for x in gx["expected_o"]])
    assert np.max(np.abs(out[0, 0] - exp)) <= 1e-15


def test_closed_form_L1_returns_v_row_exactly():
    b = small_batch(H=4, Hkv=2, D=8, dtype="bf16", lens=(1, 1, 1), seed=9)
    hb = host_batch(b)
    got = _oracle(hb, b.shape)
    v_new = to_f64(hb["v_new"])
    for h in range(4):
        assert np.array_equal(got[:, h], v_new[:, h // 2])


def test_closed_form_L2_logistic():
    b = small_batch(H=2, Hkv=2, D=8, dtype="f32", lens=(2, 2), seed=21)
    hb = host_batch(b)
    got = _oracle(hb, b.shape)
    ks, vs = dense_logical_kv(hb, b.shape.page_size)
    q = to_f64(hb["q"])
    mp.mp.dps = 40
    for j in range(2):
        for h in range(2):
            K, V = ks[j, h], vs[j, h]
            ds = (mp.fsum(mp.mpf(q[j, h, k]) * (mp.mpf(K[0, k]) - mp.mpf(K[1, k])) for k in range(8))
                  / mp.sqrt(8))
            w = 1 / (1 + mp.exp(-ds))
            ref = [float(w * mp.mpf(V[0, k]) + (1 - w) * mp.mpf(V[1, k])) for k in range(8)]
            assert np.max(np.abs(got[j, h] - np.array(ref))) <= 1e-14


def test_closed_form_q_zero_and_identical_keys_give_mean_of_v():
    b = small_batch(H=4, Hkv=4, D=8, dtype="f32", lens=(37, 5), seed=33)
    hb = host_batch(b)
    ks, vs = dense_logical_kv(hb, b.shape.page_size)
    # q = 0
    hb0 = dict(hb, q=np.zeros_like(hb["q"]))
    got = _oracle(hb0, b.shape)
    for j in range(2):
        for h in range(4):
            assert np.max(np.abs(got[j, h] - vs[j, h].mean(axis=0))) <= 1e-14
    # all keys identical (every used K row = the same vector)
    kp = hb["k_pool"].copy()
    kp[:] = kp[hb["block_table"][0, 0, 0], 0]
    got = _oracle(dict(hb, k_pool=kp), b.shape)
    for j in range(2):
        for h in range(4):
            assert np.max(np.abs(got[j, h] - vs[j, h].mean(axis=0))) <= 1e-14


def test_affine_equivariance_in_v():
    b = small_batch(H=4, Hkv=2, D=8, dtype="bf16", lens=(19, 3, 40), seed=41)
    hb = host_batch(b)
    # run in fp32 storage so that a*v + c of a bf16 value is exactly representable
    hb = dict(hb, q=to_f64(hb["q"]).astype(np.float32), k_pool=to_f64(hb["k_pool"]).astype(np.float32),
              v_pool=to_f64(hb["v_pool"]).astype(np.float32))
    s32 = workload.Shape(4, 2, 8, 4, "f32")
    base = _oracle(hb, s32)
    a, c = 2.0, 0.25
    vp64 = hb["v_pool"].astype(np.float64) * a + c
    vp = vp64.astype(np.float32)
    fin = np.isfinite(vp64)
    assert np.array_equal(vp[fin].astype(np.float64), vp64[fin])   # the transform itself is exact
    got = _oracle(dict(hb, v_pool=vp), s32)
    assert np.max(np.abs(got - (a * base + c))) <= 1e-13


def test_peaked_limit_one_hot():
    """One key = alpha * q with large alpha: the weight of that token -> 1, O -> its V row."""
    b = small_batch(H=1, Hkv=1, D=8, dtype="f32", lens=(24,), seed=55)
    hb = host_batch(b)
    q = to_f64(hb["q"])[0, 0]
    page, slot = hb["block_table"][0, 0, 1], 3            # token 7 (P = 4)
    kp = hb["k_pool"].copy()
    kp[page, slot] = (40.0 * q).astype(np.float32)
    got = _oracle(dict(hb, k_pool=kp), b.shape)
    v7 = to_f64(hb["v_pool"])[page, slot]
    ks, _ = dense_logical_kv(dict(hb, k_pool=kp), 4)
    s = ks[0, 0] @ q / math.sqrt(8)
    gap = s[7] - np.max(np.delete(s, 7))
    assert gap > 60
    assert np.max(np.abs(got[0, 0] - v7)) <= 24 * math.exp(-gap) * 10 + 1e-15


def test_large_scores_do_not_overflow():
    """Scores of order 1e3 would overflow exp() without max subtraction (reading 16)."""
    b = small_batch(H=2, Hkv=2, D=8, dtype="f32", lens=(9,), seed=60)
    hb = host_batch(b)
    hb = dict(hb, q=(hb["q"] * np.float32(512.0)))
    got = _oracle(hb, b.shape)
    assert np.all(np.isfinite(got))
    ref = _brute_force(hb, b.shape)
    assert np.max(np.abs(got - ref)) <= 1e-10


def test_page_permutation_invariance_exact():
    b = small_batch(H=8, Hkv=2, D=8, dtype="bf16", lens=(1, 16, 17, 40), seed=70)
    hb = host_batch(b)
    base = _oracle(hb, b.shape)
    n = hb["k_pool"].shape[0]
    perm = np.random.default_rng(0).permutation(n)         # new id of old page p = perm[p]
    kp = np.empty_like(hb["k_pool"])
    vp = np.empty_like(hb["v_pool"])
    kp[perm] = hb["k_pool"]
    vp[perm] = hb["v_pool"]
    bt = hb["block_table"].copy()
    bt[bt >= 0] = perm[bt[bt >= 0]]
    got = _oracle(dict(hb, k_pool=kp, v_pool=vp, block_table=bt), b.shape)
    assert np.array_equal(got, base)


def test_head_partition_invariance_exact():
    """Any head split reproduces the unsplit result: ranks generate their own shares."""
    shape = workload.Shape(16, 4, 8, 4, "bf16")
    lens = torch.tensor([3, 17, 40], dtype=torch.int32)
    full = workload.make_decode_batch(shape, lens, 99, "cpu")
    ref = _oracle(host_batch(full), shape)
    for split in [(8, 8), (4, 8, 4), (12, 4), (4, 4, 4, 4)]:
        begin = 0
        for i, x in enumerate(split):
            part = workload.make_decode_batch(shape, lens, 99, "cpu", q_begin=begin, q_count=x, rank_salt=i + 1)
            got = oracle.decode(*[host_batch(part)[k] for k in ("q", "k_pool", "v_pool", "block_table",
                                                                "seq_lens")],
                                num_kv_heads=x // 4, dtype=oracle.BF16)
            assert np.array_equal(got, ref[:, begin:begin + x])
            begin += x


def test_token_permutation_invariance():
    b = small_batch(H=2, Hkv=1, D=8, dtype="f32", lens=(40,), seed=80)
    hb = host_batch(b)
    base = _oracle(hb, b.shape)
    P = 4
    perm = np.random.default_rng(1).permutation(40)
    kp, vp = hb["k_pool"].copy(), hb["v_pool"].copy()
    bt = hb["block_table"][0, 0]
    for t_new, t_old in enumerate(perm):
        kp[bt[t_new // P], t_new % P] = hb["k_pool"][bt[t_old // P], t_old % P]
        vp[bt[t_new // P], t_new % P] = hb["v_pool"][bt[t_old // P], t_old % P]
    got = _oracle(dict(hb, k_pool=kp, v_pool=vp), b.shape)
    assert np.max(np.abs(got - base)) <= 1e-14


def test_gqa_equals_expanded_mha_exact():
    b = small_batch(H=8, Hkv=2, D=8, dtype="bf16", lens=(5, 23), seed=90)
    hb = host_batch(b)
    gqa = _oracle(hb, b.shape)
    # expand: kv head g -> heads 4g..4g+3 each with its own table row pointing at the same pages
    bt = np.repeat(hb["block_table"], 4, axis=1)
    mha = oracle.decode(hb["q"], hb["k_pool"], hb["v_pool"], bt, hb["seq_lens"], num_kv_heads=8,
                        dtype=oracle.BF16)
    assert np.array_equal(gqa, mha)


def test_token_split_lse_merge():
    """Any token split of one head + LSE merge equals the unsplit result (reading 12)."""
    b = small_batch(H=2, Hkv=2, D=8, dtype="bf16", lens=(40, 33), seed=95)
    hb = host_batch(b)
    full = _oracle(hb, b.shape)
    args = [hb[k] for k in ("q", "k_pool", "v_pool", "block_table", "seq_lens")]
    for j, L in enumerate((40, 33)):
        for cuts in ([0, L], [0, 16, L], [0, 1, 17, 32, L], [0, 5, 6, 20, L]):
            for h in range(2):
                parts = [oracle.decode_range(*args, j, h, a, c, num_kv_heads=2, dtype=oracle.BF16)
                         for a, c in zip(cuts[:-1], cuts[1:])]
                o, lse = oracle.lse_merge(np.stack([p[0] for p in parts]), np.array([p[1] for p in parts]))
                assert np.max(np.abs(o - full[j, h])) <= 1e-13
                o_all, lse_all = oracle.decode_range(*args, j, h, 0, L, num_kv_heads=2, dtype=oracle.BF16)
                assert abs(lse - lse_all) <= 1e-12


def test_kv_append_positions_golden():
    with open(os.path.join(GOLDEN, "kv_append_positions.json")) as f:
        gx = json.load(f)
    P = gx["page_size"]
    D = 4
    for case in gx["cases"]:
        L = case["seq_len"]
        npg = (L + P - 1) // P
        assert (npg - 1 == case["page_index"]) and ((L - 1) % P == case["slot"])
        assert ((L - 1) % P == 0) == case["new_page_needed"]
        pool_k = np.zeros((npg + 3, P, D), np.float32)
        pool_v = np.zeros((npg + 3, P, D), np.float32)
        bt = np.arange(npg, dtype=np.int32)[::-1].copy() + 2      # reversed, offset ids
        bt = bt.reshape(1, 1, npg)
        kn = np.full((1, 1, D), 7.0, np.float32)
        vn = np.full((1, 1, D), -3.0, np.float32)
        oracle.kv_append(kn, vn, pool_k, pool_v, bt, np.array([L], np.int32))
        page = bt[0, 0, case["page_index"]]
        assert np.all(pool_k[page, case["slot"]] == 7.0) and np.all(pool_v[page, case["slot"]] == -3.0)
        assert np.count_nonzero(pool_k) == D and np.count_nonzero(pool_v) == D


def test_kv_append_fills_only_the_new_slots():
    b = small_batch(H=4, Hkv=2, D=8, dtype="bf16", lens=(1, 4, 5, 40), seed=101)
    before_k = workload.to_numpy_bits(b.k_pool).copy()
    hb = host_batch(b)
    changed = np.any(hb["k_pool"] != before_k, axis=2)         # [pages][P]
    assert changed.sum() == 4 * 2
    # every previously-NaN slot that was not the new token is still the NaN pattern
    nan_bits = before_k == workload.NAN_BF16
    still = hb["k_pool"] == workload.NAN_BF16
    assert np.array_equal(np.all(nan_bits, axis=2) & ~changed, np.all(still, axis=2) & ~changed)


def test_oracle_rejects_empty_sequence_and_bad_pages():
    b = small_batch(H=2, Hkv=2, D=4, dtype="f32", lens=(3, 2), seed=111)
    hb = host_batch(b)
    with pytest.raises(oracle.OracleError):
        _oracle(dict(hb, seq_lens=np.array([3, 0], np.int32)), b.shape)
    bt = hb["block_table"].copy()
    bt[1, 0, 0] = hb["k_pool"].shape[0]
    with pytest.raises(oracle.OracleError):
        _oracle(dict(hb, block_table=bt), b.shape)


def test_nan_poison_never_reaches_output():
    """Slack pages, tail slots and unused table entries are NaN / -1; the oracle never touches them."""
    b = small_batch(H=4, Hkv=4, D=8, dtype="bf16", lens=(1, 2, 3, 17, 31), seed=120)
    got = _oracle(host_batch(b), b.shape)
    assert np.all(np.isfinite(got))


def test_generator_is_deterministic_by_seed():
    a = small_batch(seed=7, dtype="bf16")
    c = small_batch(seed=7, dtype="bf16")
    d = small_batch(seed=8, dtype="bf16")
    for name in ("q", "k_new", "v_new", "k_pool", "v_pool", "block_table"):
        x, y = getattr(a, name), getattr(c, name)
        assert torch.equal(x.view(torch.int16) if x.dtype == torch.bfloat16 else x,
                           y.view(torch.int16) if y.dtype == torch.bfloat16 else y)
    assert not torch.equal(a.q.float(), d.q.float())


def test_kv_bytes_closed_form_p64():
    with open(os.path.join(GOLDEN, "kv_bytes_p64.json")) as f:
        gx = json.load(f)
    got = accounting.kv_cache_bytes(gx["layers"], gx["kv_heads"], gx["head_dim"], gx["elem_bytes"], gx["tokens"])
    assert got == gx["expected_bytes"] and got > gx["paper_lower_bound_bytes"]


def test_comm_volume_eq4():
    # Eq. 4: d = (2 + 2/r) h; MHA r = 1 -> 4h, GQA r = 8 -> 2.25h
    assert accounting.comm_head_vectors(8, 8) == 18.0
    assert accounting.comm_head_vectors(5, 1) == 20.0


def test_kv_migrate_hand_worked_example():
    """Token-order-preserving head-granular migration against a hand-derived result (golden)."""
    with open(os.path.join(GOLDEN, "kv_migrate_example.json")) as f:
        gx = json.load(f)
    src_k = np.array(gx["src_k"], np.float32)[..., None]            # [pages][P][1]
    src_v = -src_k
    dst_k = np.full((4, gx["page_size"], 1), gx["dst_init"], np.float32)
    dst_v = dst_k.copy()
    oracle.kv_migrate(np.array(gx["entries"], np.int32), src_k, src_v, np.array(gx["src_bt"], np.int32),
                      dst_k, dst_v, np.array(gx["dst_bt"], np.int32))
    exp = np.array(gx["expected_dst_k"], np.float32)
    assert np.array_equal(dst_k[..., 0], exp)
    assert np.array_equal(dst_v[..., 0], -exp)


def test_kv_migrate_then_decode_equals_decode_in_place():
    """Moving every (request, kv head) to a freshly permuted pool leaves Eq. 2b's result unchanged."""
    b = small_batch(H=8, Hkv=2, D=8, dtype="bf16", lens=(1, 16, 17, 40), seed=55)
    hb = host_batch(b)
    B, G, mp = hb["block_table"].shape
    rng = np.random.default_rng(3)
    npg = hb["k_pool"].shape[0]
    perm = rng.permutation(npg).astype(np.int32)
    dst_bt = np.where(hb["block_table"] >= 0, perm[np.maximum(hb["block_table"], 0)], -1).astype(np.int32)
    dst_bt = dst_bt[::-1].copy()                                   # requests stored in reverse row order
    lens = hb["seq_lens"]
    entries = [[j * G + g, (B - 1 - j) * G + g, int(lens[j])] for j in range(B) for g in range(G)]
    dk = np.full_like(hb["k_pool"], workload.NAN_BF16)
    dv = np.full_like(hb["v_pool"], workload.NAN_BF16)
    oracle.kv_migrate(np.array(entries, np.int32), hb["k_pool"], hb["v_pool"], hb["block_table"], dk, dv, dst_bt)
    ref = oracle.decode(hb["q"], hb["k_pool"], hb["v_pool"], hb["block_table"], lens, num_kv_heads=G,
                        dtype=oracle.BF16)
    got = oracle.decode(hb["q"][::-1].copy(), dk, dv, dst_bt, lens[::-1].copy(), num_kv_heads=G, dtype=oracle.BF16)
    assert np.array_equal(got[::-1], ref)


# ------------------------------------------------------------------ oracle_decode_pairs_f64 (sampled outputs)
@pytest.mark.parametrize("H,Hkv,D,dtype", [(8, 4, 8, "bf16"), (4, 4, 4, "f32"), (8, 1, 8, "f32")])
def test_pairs_brute_force_tiny(H, Hkv, D, dtype):
    """decode_pairs on shuffled (seq, head) pairs, with repeats, against the mpmath brute force (independent
    gather, no max subtraction) -- the same pin as the full output, applied to the pairs entry point."""
    b = small_batch(H=H, Hkv=Hkv, D=D, P=4, dtype=dtype, lens=(1, 7, 40), seed=29 + H + D)
    hb = host_batch(b)
    ref = _brute_force(hb, b.shape)
    rng = np.random.default_rng(3)
    pairs = [(int(rng.integers(3)), int(rng.integers(H))) for _ in range(20)] + [(2, H - 1), (0, 0), (2, H - 1)]
    got = oracle.decode_pairs(hb["q"], hb["k_pool"], hb["v_pool"], hb["block_table"], hb["seq_lens"], pairs,
                              num_kv_heads=Hkv, dtype=dtype_code(b.shape))
    for i, (j, h) in enumerate(pairs):
        assert np.max(np.abs(got[i] - ref[j, h])) <= 1e-12, (j, h)


@pytest.mark.parametrize("H,Hkv,D,dtype", [(16, 2, 64, "bf16"), (8, 8, 32, "f32"), (12, 4, 16, "bf16")])
def test_pairs_equal_full_output_rows(H, Hkv, D, dtype):
    """Every sampled pair equals the pinned full output's row bit for bit (same per-output arithmetic), for
    GQA and MHA, bf16 and fp32, ragged lengths over several pages and random page ids."""
    b = small_batch(H=H, Hkv=Hkv, D=D, P=16, dtype=dtype, lens=(1, 16, 17, 300, 65, 2), seed=31 + H)
    hb = host_batch(b)
    full = _oracle(hb, b.shape)
    rng = np.random.default_rng(H * D)
    pairs = sorted({(int(rng.integers(6)), int(rng.integers(H))) for _ in range(40)} | {(0, 0), (5, H - 1)})
    got = oracle.decode_pairs(hb["q"], hb["k_pool"], hb["v_pool"], hb["block_table"], hb["seq_lens"], pairs,
                              num_kv_heads=Hkv, dtype=dtype_code(b.shape), nthreads=3)
    for i, (j, h) in enumerate(pairs):
        assert np.array_equal(got[i], full[j, h]), (j, h)
    # a head's row depends on its own kv group only: a wrong h -> g mapping in the pairs path would differ
    assert not np.array_equal(full[1, 0], full[1, H - 1])


def test_pairs_rejects_out_of_range_pairs():
    b = small_batch(H=4, Hkv=2, D=8, P=4, dtype="f32", lens=(3, 5), seed=2)
    hb = host_batch(b)
    for bad in ([(2, 0)], [(0, 4)], [(-1, 0)]):
        with pytest.raises(oracle.OracleError):
            oracle.decode_pairs(hb["q"], hb["k_pool"], hb["v_pool"], hb["block_table"], hb["seq_lens"], bad,
                                num_kv_heads=2, dtype=oracle.F32)
