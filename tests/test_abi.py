"""C-ABI tests that need no GPU: the library loads, exports every symbol
include/hetis.h declares, and validates arguments exactly as documented
(plans: Eq. 5 / Eq. 6 / group integrality; attention: shapes, alignment,
workspace).  No call here reaches a kernel launch."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

from paper_2509_08309_b200 import build as hbuild
from paper_2509_08309_b200 import hetis, workload

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    hbuild.build()
    return hetis.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hetis.h")).read()
    return sorted(set(re.findall(r"^HETIS_API [^;(]*?\b(hetis_\w+)\s*\(", src, flags=re.M)))


def test_every_declared_symbol_is_exported(L):
    syms = declared_symbols()
    assert len(syms) == 40
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(hetis.EXPORTED)


def test_exported_symbols_match_nm():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", hetis.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (hetis_\w+)", out))
    assert exported == set(declared_symbols())


def test_status_strings_and_constants(L):
    for code, name in hetis.STATUS.items():
        assert hetis.status_str(code) == name
    assert hetis.abi_version() == 4
    assert hetis.split_tokens() % 16 == 0


SHAPE_13B = hetis.make_shape(workload.LLAMA2_13B)
SHAPE_70B = hetis.make_shape(workload.LLAMA2_70B)


def test_plan_even_and_uneven_ranges(L):
    p = hetis.plan_create(SHAPE_13B, 5, [16, 8, 8, 4, 4])
    assert [p.heads(i) for i in range(5)] == [(0, 16), (16, 8), (24, 8), (32, 4), (36, 4)]
    p = hetis.plan_create(SHAPE_70B, 8, [8] * 8)
    assert [p.heads(i) for i in range(8)] == [(8 * i, 8) for i in range(8)]
    p = hetis.plan_create(SHAPE_70B, 3, [0, 48, 16])          # a device may hold no heads
    assert p.heads(0) == (0, 0) and p.heads(2) == (48, 16)


def test_plan_head_integrity_eq5(L):
    with pytest.raises(hetis.HetisError) as e:
        hetis.plan_create(SHAPE_13B, 2, [20, 19])
    assert e.value.name == "HETIS_E_HEAD_INTEGRITY"
    with pytest.raises(hetis.HetisError) as e:
        hetis.plan_create(SHAPE_13B, 2, [0, 0])                 # Sigma = 0 rejected (reading 14)
    assert e.value.name == "HETIS_E_HEAD_INTEGRITY"


def test_plan_group_integrality(L):
    with pytest.raises(hetis.HetisError) as e:
        hetis.plan_create(SHAPE_70B, 2, [36, 28])                # 36 / 8 not integral
    assert e.value.name == "HETIS_E_GROUP_ALIGN"
    with pytest.raises(hetis.HetisError) as e:
        hetis.plan_create(SHAPE_13B, 2, [-1, 41])
    assert e.value.name == "HETIS_E_INVALID"


def test_plan_per_request(L):
    x = [32, 32,
         64, 0,
         8, 56]
    p = hetis.plan_create(SHAPE_70B, 2, x, per_request=True, num_seqs=3)
    assert p.heads(1, seq=0) == (32, 32) and p.heads(0, seq=1) == (0, 64) and p.heads(1, seq=2) == (8, 56)
    with pytest.raises(hetis.HetisError) as e:
        hetis.plan_create(SHAPE_70B, 2, [32, 32, 64, 8], per_request=True, num_seqs=2)
    assert e.value.name == "HETIS_E_HEAD_INTEGRITY"


def test_plan_units_for_per_request_plans(L):
    x = [32, 32,
         64, 0,
         8, 56]
    p = hetis.plan_create(SHAPE_70B, 2, x, per_request=True, num_seqs=3)
    assert p.units(0) == [(0, 0), (0, 1), (0, 2), (0, 3), (1, 0), (1, 1), (1, 2), (1, 3), (1, 4), (1, 5), (1, 6),
                          (1, 7), (2, 0)]
    assert p.units(1) == [(0, 4), (0, 5), (0, 6), (0, 7), (2, 1), (2, 2), (2, 3), (2, 4), (2, 5), (2, 6), (2, 7)]
    # every (request, kv head) appears on exactly one device (Eq. 5 head integrity)
    allu = sorted(p.units(0) + p.units(1))
    assert allu == [(j, g) for j in range(3) for g in range(8)]
    with pytest.raises(hetis.HetisError):
        hetis.plan_create(SHAPE_70B, 2, [32, 32]).units(0)          # global plans have no units


def test_plan_capacity_eq6_in_pages(L):
    p = hetis.plan_create(SHAPE_13B, 5, [16, 8, 8, 4, 4])
    lens = [512, 10240, 17]
    pages = sum((n + 15) // 16 for n in lens)                     # per kv head
    need = [pages * x for x in (16, 8, 8, 4, 4)]                  # r = 1
    p.check_capacity(lens, need)
    with pytest.raises(hetis.HetisError) as e:
        p.check_capacity(lens, [need[0], need[1], need[2] - 1, need[3], need[4]])
    assert e.value.name == "HETIS_E_CAPACITY"
    p70 = hetis.plan_create(SHAPE_70B, 2, [48, 16])
    p70.check_capacity([2048], [128 * 6, 128 * 2])                 # x / r kv heads per device
    with pytest.raises(hetis.HetisError):
        p70.check_capacity([2048], [128 * 6, 128 * 2 - 1])


def test_comm_workspace_sizes(L):
    p = hetis.plan_create(SHAPE_70B, 4, [16] * 4)
    ws = p.comm_workspace(0, 128)
    # scatter: 4 ranks x (q 128x16x128x2 + k,v 128x2x128x2) ; gather (fp32 o): 4 x 128x16x128x4
    assert ws == max(4 * (128 * 16 * 256 + 2 * 128 * 2 * 256), 4 * 128 * 16 * 512)
    with pytest.raises(hetis.HetisError):
        hetis.plan_create(SHAPE_70B, 2, [32, 32, 64, 0], per_request=True, num_seqs=2).comm_workspace(0, 2)


def test_workspace_formula(L):
    C = hetis.split_tokens()
    n = hetis.attn_decode_workspace(SHAPE_13B, 64, 40, 4096)
    items = 64 * (4096 // C) * 40
    r256 = lambda b: (b + 255) // 256 * 256
    # split offsets + partial lse + partial o + work-claim counters + per-pair split counters (fused merge)
    assert n == r256(65 * 4) + r256(items * 4) + r256(items * 128 * 4) + 256 + r256(64 * 40 * 4)
    with pytest.raises(hetis.HetisError) as e:
        hetis.attn_decode_workspace(SHAPE_70B, 64, 12, 4096)     # 12 heads = 1.5 kv groups
    assert e.value.name == "HETIS_E_GROUP_ALIGN"


def _raw_partial(L, shape, B=4, begin=0, count=8, q=256, kp=1024, vp=1024, ws=512, ws_bytes=1 << 30, bt=64, sl=64,
                 max_seq=128, max_pages=8, num_pages=100):
    vp_ = ctypes.c_void_p
    return L.hetis_attn_partial(ctypes.byref(shape), B, begin, count, vp_(q), vp_(kp), vp_(vp), num_pages, vp_(bt),
                                max_pages, vp_(sl), max_seq, vp_(ws), ws_bytes, 0, vp_(0))


def test_attn_validation_before_launch(L):
    s = hetis.make_shape(workload.Shape(8, 8, 64, 16, "f32"))
    bad_d = hetis.make_shape(workload.Shape(8, 8, 96, 16, "f32"))
    assert _raw_partial(L, bad_d) == 5                                      # UNSUPPORTED head_dim
    bad_p = hetis.make_shape(workload.Shape(8, 8, 64, 32, "f32"))
    assert _raw_partial(L, bad_p) == 5                                      # UNSUPPORTED page size
    g = hetis.make_shape(workload.Shape(16, 4, 128, 16, "bf16"))
    assert _raw_partial(L, g, begin=2, count=8) == 3                        # GROUP_ALIGN begin
    assert _raw_partial(L, g, begin=0, count=6) == 3                        # GROUP_ALIGN count
    assert _raw_partial(L, s, begin=4, count=8) == 1                        # range past H
    assert _raw_partial(L, s, q=0) == 1                                     # NULL
    assert _raw_partial(L, s, q=258) == 1                                   # misaligned q
    assert _raw_partial(L, s, kp=1024 + 64) == 1                            # misaligned pool
    assert _raw_partial(L, s, ws=512 + 16) == 6                             # misaligned workspace
    assert _raw_partial(L, s, ws_bytes=100) == 6                            # workspace too small
    assert _raw_partial(L, s, max_pages=4, max_seq=128) == 1                # table cannot hold max_seq
    assert _raw_partial(L, s, B=5000) == 5                                  # batch above the smem table
    assert _raw_partial(L, s, B=0) == 0                                     # empty batch: no-op
    assert b"head range" in L.hetis_last_error() or True


def test_kv_append_and_combine_validation(L):
    vp_ = ctypes.c_void_p
    s = hetis.make_shape(workload.Shape(8, 8, 64, 16, "f32"))
    rc = L.hetis_kv_append(ctypes.byref(s), 4, 8, vp_(1024), vp_(1024 + 8), vp_(4096), vp_(8192), 10, vp_(64), 8,
                           vp_(64), vp_(0))
    assert rc == 1                                                          # misaligned v_new
    rc = L.hetis_kv_append(ctypes.byref(s), 0, 8, None, None, None, None, 10, None, 8, None, vp_(0))
    assert rc == 0                                                          # empty batch
    rc = L.hetis_attn_combine(ctypes.byref(s), 4, 8, vp_(64), 128, vp_(4096), 8 * 64 - 1, vp_(512), 1 << 30, vp_(0))
    assert rc == 1                                                          # stride below a dense row


def test_kv_migrate_validation(L):
    vp_ = ctypes.c_void_p
    s = hetis.make_shape(workload.Shape(8, 8, 128, 16, "bf16"))
    ok = [vp_(4096), vp_(8192), vp_(1 << 20), vp_(64), 8, vp_(2 << 20), vp_(3 << 20), vp_(128), 8, 0, vp_(0)]
    assert L.hetis_kv_migrate(ctypes.byref(s), 0, None, *([None] * 3), 8, None, None, None, 8, 0, vp_(0)) == 0
    assert L.hetis_kv_migrate(ctypes.byref(s), 16385, *ok) == 1               # above the entry cap
    assert L.hetis_kv_migrate(ctypes.byref(s), -1, *ok) == 1
    bad = list(ok)
    bad[1] = vp_(8192 + 8)
    assert L.hetis_kv_migrate(ctypes.byref(s), 4, *bad) == 1                 # misaligned source K pool
    bad = list(ok)
    bad[6] = None
    assert L.hetis_kv_migrate(ctypes.byref(s), 4, *bad) == 1                 # NULL destination V pool
    bad = list(ok)
    bad[9] = -1
    assert L.hetis_kv_migrate(ctypes.byref(s), 4, *bad) == 1                 # negative CTA budget
    s2 = hetis.make_shape(workload.Shape(8, 8, 96, 16, "bf16"))
    assert L.hetis_kv_migrate(ctypes.byref(s2), 4, *ok) == 5                 # head_dim not built


def test_nccl_calls_validate_plan_and_comm(L):
    p = hetis.plan_create(SHAPE_70B, 2, [32, 32])
    vp_ = ctypes.c_void_p
    rc = L.hetis_gather(p.handle, vp_(0), 0, -1, 4, vp_(256), vp_(512), vp_(1024), 1 << 20, vp_(0))
    assert rc == 1                                                          # NULL communicator
    rc = L.hetis_gather(p.handle, vp_(1234), 2, -1, 4, vp_(256), vp_(512), vp_(1024), 1 << 20, vp_(0))
    assert rc == 1                                                          # rank outside the plan
    rc = L.hetis_scatter_q(p.handle, vp_(1234), 0, -1, 4, *([vp_(256)] * 6), vp_(1024), 1 << 20, vp_(0))
    assert rc == 1                                                          # scatter needs a root


def test_binding_refuses_host_tensors(L):
    import torch
    s = hetis.make_shape(workload.Shape(8, 8, 64, 16, "f32"))
    t = torch.zeros(4, 8, 64)
    with pytest.raises(ValueError):
        hetis.attn_decode(s, t, t, t, torch.zeros(4, 8, 8, dtype=torch.int32), torch.ones(4, dtype=torch.int32), 1,
                          t, torch.zeros(1024, dtype=torch.uint8))


def test_seq_split_entry_points_validate(L):
    """Row f3 entry points: argument validation happens before any launch (no GPU needed)."""
    vp_ = ctypes.c_void_p
    s = hetis.make_shape(workload.LLAMA2_13B)
    # split lengths: rank outside [0, N), nothing to do for 0 requests, NULL outputs
    assert L.hetis_seq_split_lens(2, 2, 16, 4, vp_(256), vp_(512), None, vp_(0)) == 1
    assert L.hetis_seq_split_lens(0, 0, 16, 4, vp_(256), vp_(512), None, vp_(0)) == 1
    assert L.hetis_seq_split_lens(2, 1, 16, 0, None, None, None, vp_(0)) == 0
    assert L.hetis_seq_split_lens(2, 1, 16, 4, vp_(256), None, None, vp_(0)) == 1
    # merge: part strides below one part, misaligned parts, unsupported head_dim
    B, H, D = 4, 40, 128
    ok = (2, B, H, vp_(1 << 20), B * H * D, vp_(1 << 22), B * H, vp_(1 << 24), H * D, vp_(0))
    bad = list(ok)
    bad[4] = B * H * D - 1
    assert L.hetis_seq_merge(ctypes.byref(s), *bad) == 1
    bad = list(ok)
    bad[3] = vp_((1 << 20) + 8)
    assert L.hetis_seq_merge(ctypes.byref(s), *bad) == 1
    bad = list(ok)
    bad[8] = H * D - 4
    assert L.hetis_seq_merge(ctypes.byref(s), *bad) == 1
    assert L.hetis_seq_merge(ctypes.byref(s), 0, *ok[1:]) == 1
    s96 = hetis.make_shape(workload.Shape(40, 40, 96, 16, "bf16"))
    assert L.hetis_seq_merge(ctypes.byref(s96), *ok) == 5
    # combine with lse: the lse pointer is required
    assert L.hetis_attn_combine_lse(ctypes.byref(s), 4, H, vp_(256), 64, vp_(1024), H * D, None, vp_(4096),
                                    1 << 20, vp_(0)) == 1
    # NCCL exchange: NULL communicator / rank outside the world
    assert L.hetis_seq_allgather_merge(ctypes.byref(s), vp_(0), 2, 0, 4, vp_(256), vp_(512), vp_(1024), H * D,
                                       vp_(0)) == 1
    assert L.hetis_seq_broadcast_q(ctypes.byref(s), vp_(1234), 2, 3, 0, 4, vp_(256), vp_(512), vp_(768),
                                   vp_(0)) == 1


# ------------------------------------------------------------------ peer-memory exchange group (no launch)
def _group(plan, rank=0, root=0, gather_root=-1, states=None, outs=None, stride=None, root_bufs=None):
    n = plan.num_devices
    states = states if states is not None else [0x100000 * (p + 1) for p in range(n)]
    outs = outs if outs is not None else [0x4000000 * (p + 1) for p in range(n)]
    root_bufs = root_bufs if root_bufs is not None else (0x7000000, 0x7100000, 0x7200000)
    stride = stride if stride is not None else plan.shape.num_q_heads * plan.shape.head_dim
    return hetis.PeerGroup(plan, rank, root, gather_root, states, outs, stride, *root_bufs)


def test_peer_state_bytes(L):
    assert hetis.peer_state_bytes() == 512


def test_peer_group_validation(L):
    p = hetis.plan_create(SHAPE_13B, 5, [16, 8, 8, 4, 4])
    g = _group(p, rank=3)                                   # valid: no launch, pointers only recorded
    assert g.handle.value
    g2 = _group(p, rank=2, gather_root=0, outs=[0x4000000, None, None, None, None])   # only the receiver's o_full
    assert g2.handle.value
    bad = [dict(rank=5), dict(root=-1), dict(gather_root=5), dict(gather_root=-2),
           dict(states=[0x100000, 0, 0x300000, 0x400000, 0x500000]),             # NULL state
           dict(states=[0x100008, 0x200000, 0x300000, 0x400000, 0x500000]),      # state not 64-B aligned
           dict(outs=[0x4000000, None, 0x4000000, 0x4000000, 0x4000000]),         # a receiver without o_full
           dict(stride=40 * 128 - 1),                                            # stride below H * d
           dict(root_bufs=(0x7000004, 0x7100000, 0x7200000))]                     # misaligned root q
    for kw in bad:
        with pytest.raises(hetis.HetisError) as ei:
            _group(p, **kw)
        assert ei.value.name == "HETIS_E_INVALID", kw
    pr = hetis.plan_create(SHAPE_70B, 2, [64, 0, 32, 32], per_request=True, num_seqs=2)
    with pytest.raises(hetis.HetisError) as ei:
        _group(pr)
    assert ei.value.name == "HETIS_E_UNSUPPORTED"


def test_decode_launches_for_group_mode_selection(L):
    """hetis_attn_decode_launches_for (host logic, no launch): the one-kernel form where the launch qualifies for
    group mode -- bf16 GQA, <= one (request, kv head) pair per SM (148 on B200; also the CPU box's fallback), <= 8
    splits of 256 tokens -- or with HETIS_ATTN_FUSED_MERGE; two kernels otherwise; -1 on invalid arguments."""
    from paper_2509_08309_b200 import hetis, workload
    gqa = hetis.make_shape(workload.Shape(64, 8, 128, 16, "bf16"))
    mha = hetis.make_shape(workload.Shape(40, 40, 128, 16, "bf16"))
    f32 = hetis.make_shape(workload.Shape(8, 2, 64, 16, "f32"))
    n = hetis.attn_decode_launches_for
    assert n(gqa, 128, 8, 2048) == 1             # c3's 8-GPU share: 128 pairs, 8 splits
    assert n(gqa, 148, 8, 2048) == 1             # the boundary
    assert n(gqa, 149, 8, 2048) == 2
    assert n(gqa, 128, 8, 2049) == 2             # 9 splits
    assert n(gqa, 128, 16, 1024) == 2            # 256 pairs
    assert n(gqa, 128, 64, 2048) == 2            # c3 at N = 1
    assert n(gqa, 128, 64, 2048, hetis.ATTN_FUSED_MERGE) == 1
    assert n(gqa, 128, 8, 2048, hetis.ATTN_NO_GROUP_MODE) == 2
    assert n(gqa, 128, 8, 2048, hetis.ATTN_DEVICE_CLAIM) == 2
    assert n(gqa, 128, 8, 2048, hetis.ATTN_PIPELINED) == 2
    assert n(mha, 2, 40, 512) == 2               # MHA stays off the tensor cores: no fused merge
    assert n(f32, 4, 8, 512) == 2
    with pytest.raises(ValueError):
        n(gqa, 0, 8, 2048)
    with pytest.raises(ValueError):
        n(gqa, 4, 6, 2048)                       # not whole kv groups
