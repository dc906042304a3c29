"""Head-granular KV migration on the GPU (hetis_kv_migrate; the Hauler, PAPER.md:522, :545;
SURVEY.md §8(f) row f4).

A request re-dispatched from one per-request plan row to another moves only the
kv groups whose device changes (`dispatch.plan_migration`: every device keeps
min(old, new) / r of its groups, so ownership becomes non-contiguous).  Here
the devices are "virtual devices" on one GPU: each has its own K/V pools and a
block table with one row per (request, kv group) unit (`dispatch.owner_units`
order).  After the kernel copies the moved groups' pages:

* every destination pool equals the oracle's token-by-token migration bit for
  bit on every cached token (and untouched pages keep their bytes);
* attention executed on the NEW plan from the migrated pools -- each device's
  unit list in one hetis_attn_decode_units call -- reassembles to the
  single-device result bit for bit (the chunking depends on L_j only): the
  migrated cache is the cache.
A two-process test pushes the pages into another process's pools through CUDA
IPC mappings: the peer-pointer path an NVSwitch box uses over NVLink.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from paper_2509_08309_b200 import dispatch, hetis, workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    hetis.lib()


def _bits(a: np.ndarray) -> np.ndarray:
    return a.view(np.uint32) if a.dtype == np.float32 else a


def _full_batch(H, Hkv, D, dtype, lens, seed):
    shape = workload.Shape(H, Hkv, D, 16, dtype)
    b = workload.make_decode_batch(shape, torch.tensor(lens, dtype=torch.int32), seed, "cuda")
    s = hetis.make_shape(shape)
    hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    return shape, s, b


def _decode_full(s, b):
    B, H, D = b.q.shape
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, B, H, b.max_seq_len), "cuda")
    o = torch.empty((B, H, D), device="cuda")
    hetis.attn_decode(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, b.max_seq_len, o, ws)
    return o


def _random_rows(rng, J, G, N):
    """Per-request allocations of G kv groups over N devices (some devices may get none)."""
    rows = np.zeros((J, N), dtype=np.int64)
    for j in range(J):
        cuts = np.sort(rng.integers(0, G + 1, size=N - 1))
        rows[j] = np.diff(np.concatenate([[0], cuts, [G]]))
    return rows


def _contiguous_owners(rows, r):
    """Every request's group owners under contiguous head ranges (reading 3)."""
    return [dispatch.group_owners(rows[j] * r, r) for j in range(rows.shape[0])]


class VirtualDevice:
    """Pools + unit-row block table of one device, pages taken from a shuffled free list."""

    def __init__(self, b, capacity, rng):
        P, D = b.k_pool.shape[1], b.k_pool.shape[2]
        self.k = torch.full((capacity, P, D), float("nan"), dtype=b.k_pool.dtype, device="cuda")
        self.v = torch.full_like(self.k, float("nan"))
        self.free = list(rng.permutation(capacity))
        self.max_pages = b.block_table.shape[2]

    def alloc(self, n):
        out, self.free = self.free[:n], self.free[n:]
        return out

    def table(self, units, lens, keep=None):
        """[U][max_pages] rows; units found in `keep` (unit -> page list) reuse their pages."""
        t = torch.full((max(len(units), 1), self.max_pages), -1, dtype=torch.int32)
        pages = {}
        for u, (j, g) in enumerate(units):
            pg = keep[(j, g)] if keep and (j, g) in keep else self.alloc((int(lens[j]) + 15) // 16)
            pages[(j, g)] = pg
            t[u, :len(pg)] = torch.tensor(pg, dtype=torch.int32)
        return t.cuda(), pages


def _fill_from_full(dev, b, pages):
    """Old placement: copy each unit's pages out of the single-device pools (torch indexing)."""
    for (j, g), pg in pages.items():
        n = len(pg)
        src = b.block_table[j, g, :n].long()
        dst = torch.tensor(pg, dtype=torch.long, device="cuda")
        dev.k[dst] = b.k_pool[src]
        dev.v[dst] = b.v_pool[src]


def _run_units(s, b, dev, units, table, o):
    """The device's units on the full layouts in one attention launch + one combine
    (hetis_attn_decode_units): its unit-row table is scattered into a [B][H_kv][max_pages] table."""
    B, Hkv = b.block_table.shape[:2]
    full_tab = torch.full((B, Hkv, table.shape[1]), -1, dtype=torch.int32, device="cuda")
    for u, (j, g) in enumerate(units):
        full_tab[j, g] = table[u]
    ut = torch.tensor(units, dtype=torch.int32, device="cuda").reshape(-1, 2)
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, len(units), s.num_q_heads // s.num_kv_heads,
                                                           b.max_seq_len), "cuda")
    hetis.attn_decode_units(s, ut, b.q, dev.k, dev.v, full_tab, b.seq_lens, b.max_seq_len, o, ws)
    torch.cuda.synchronize()


@pytest.mark.parametrize("H,Hkv,D,dtype,max_ctas", [(64, 8, 128, "bf16", 0), (40, 40, 128, "bf16", 7),
                                                    (8, 8, 64, "f32", 1), (16, 4, 64, "bf16", 0)])
def test_redispatch_migration_bit_exact(H, Hkv, D, dtype, max_ctas):
    lens = (600, 5, 1300, 256, 17, 77, 1)
    N = 3
    shape, s, b = _full_batch(H, Hkv, D, dtype, lens, seed=171 + H)
    o_ref = _decode_full(s, b)
    rng = np.random.default_rng(H + D)
    G, r, J = Hkv, H // Hkv, len(lens)
    old = _random_rows(rng, J, G, N)
    new = old.copy()
    for j in (0, 2, 4, 6):                                       # the Hauler re-dispatches these requests
        new[j] = _random_rows(rng, 1, G, N)[0]
    migs = {j: dispatch.plan_migration(old[j] * r, new[j] * r, r) for j in range(J)
            if not np.array_equal(old[j], new[j])}
    old_own = _contiguous_owners(old, r)
    new_own = [migs[j].new_owner if j in migs else old_own[j] for j in range(J)]   # maximal reuse: not contiguous
    old_units, new_units = dispatch.owner_units(old_own, N), dispatch.owner_units(new_own, N)
    for j, m in migs.items():                                    # only the set difference moves
        assert len(m.moves) == G - int(np.minimum(old[j], new[j]).sum())
    capacity = sum(G * ((L + 15) // 16) for L in lens) + 8
    devs = [VirtualDevice(b, capacity, rng) for _ in range(N)]
    old_tab, new_tab = [], []
    for d in range(N):
        t, pages = devs[d].table(old_units[d], lens)
        _fill_from_full(devs[d], b, pages)
        old_tab.append((t, pages))
    for d in range(N):
        t, pages = devs[d].table(new_units[d], lens, keep=old_tab[d][1])
        new_tab.append((t, pages))
    torch.cuda.synchronize()
    host_before = [(workload.to_numpy_bits(dv.k).copy(), workload.to_numpy_bits(dv.v).copy()) for dv in devs]

    entries = dispatch.migration_entries(old_units, new_units, migs, lens)
    moved = sum(len(m.moves) for m in migs.values())
    assert sum(len(e) for e in entries.values()) == moved
    for (src, dst), e in entries.items():
        hetis.kv_migrate(s, torch.from_numpy(e).cuda(), devs[src].k, devs[src].v, old_tab[src][0], devs[dst].k,
                         devs[dst].v, new_tab[dst][0], max_ctas=max_ctas)
    torch.cuda.synchronize()

    # bytes: the oracle's token-by-token migration on host copies of the same pools
    expect = [(k.copy(), v.copy()) for k, v in host_before]
    for (src, dst), e in entries.items():
        oracle.kv_migrate(e, host_before[src][0], host_before[src][1], old_tab[src][0].cpu().numpy(),
                          expect[dst][0], expect[dst][1], new_tab[dst][0].cpu().numpy())
    for d in range(N):
        got_k, got_v = workload.to_numpy_bits(devs[d].k), workload.to_numpy_bits(devs[d].v)
        cached = np.zeros(got_k.shape[:2], dtype=bool)          # [pages][P]: slots holding a cached token
        for (j, g), pg in new_tab[d][1].items():
            for t in range(lens[j]):
                cached[pg[t // 16], t % 16] = True
        incoming = {p for (src, dst), e in entries.items() if dst == d
                    for row in e for p in new_tab[d][0][row[1], :(row[2] + 15) // 16].tolist()}
        untouched = np.ones(got_k.shape[0], dtype=bool)
        untouched[list(incoming)] = False
        for got, exp in ((got_k, expect[d][0]), (got_v, expect[d][1])):
            got, exp = _bits(got), _bits(exp)                    # NaN sentinels compare as bits
            assert np.array_equal(got[cached], exp[cached]), d
            assert np.array_equal(got[untouched], exp[untouched]), d

    # the migrated cache serves the new (non-contiguous) plan: every device runs its unit list with
    # hetis_attn_decode_units into the shared O; bit-identical to the single-device result
    assembled = torch.full_like(o_ref, float("nan"))
    for d in range(N):
        if new_units[d]:
            _run_units(s, b, devs[d], new_units[d], new_tab[d][0], assembled)
    assert torch.equal(assembled, o_ref)


def test_many_entries_and_empty_caches():
    """16384 entries (the shared-memory prefix above 48 KiB), lengths 0..40 incl. empty caches: every
    cached token lands in its destination slot (against torch gathers of the logical rows)."""
    shape = workload.Shape(8, 8, 128, 16, "bf16")
    s = hetis.make_shape(shape)
    n = 16384
    g = torch.Generator().manual_seed(7)
    lens = torch.randint(0, 41, (n,), generator=g)
    lens[::97] = 0
    npg = (lens + 15) // 16
    tot = int(npg.sum())
    src_k = torch.randn((tot + 5, 16, 128), generator=g).to(torch.bfloat16).cuda()
    src_v = torch.randn((tot + 5, 16, 128), generator=g).to(torch.bfloat16).cuda()
    perm_s = torch.randperm(tot + 5, generator=g)[:tot]
    perm_d = torch.randperm(tot + 11, generator=g)[:tot]
    src_bt = torch.full((n, 3), -1, dtype=torch.int32)
    dst_bt = torch.full((n, 3), -1, dtype=torch.int32)
    order = torch.randperm(n, generator=g)                      # destination rows are a permutation
    off = 0
    for i in range(n):
        k = int(npg[i])
        src_bt[i, :k] = perm_s[off:off + k].int()
        dst_bt[int(order[i]), :k] = perm_d[off:off + k].int()
        off += k
    entries = torch.stack([torch.arange(n), order, lens], dim=1).int().contiguous()
    dst_k = torch.zeros((tot + 11, 16, 128), dtype=torch.bfloat16, device="cuda")
    dst_v = torch.zeros_like(dst_k)
    hetis.kv_migrate(s, entries.cuda(), src_k, src_v, src_bt.cuda(), dst_k, dst_v, dst_bt.cuda())
    torch.cuda.synchronize()
    # logical token rows of every entry, gathered with torch on both sides
    rows = [(i, t) for i in range(0, n, 13) for t in range(int(lens[i]))]
    si = torch.tensor([int(src_bt[i, t // 16]) for i, t in rows])
    di = torch.tensor([int(dst_bt[int(order[i]), t // 16]) for i, t in rows])
    sl = torch.tensor([t % 16 for _, t in rows])
    assert torch.equal(dst_k[di, sl].cpu(), src_k[si, sl].cpu())
    assert torch.equal(dst_v[di, sl].cpu(), src_v[si, sl].cpu())
    # pages no entry maps to stay zero
    used = torch.zeros(tot + 11, dtype=torch.bool)
    used[perm_d] = True
    assert not dst_k[~used.cuda()].any()


# ---------------------------------------------------------------- two processes: push over peer mappings
def _rank(rank, q_in, q_out, barrier, res):
    import numpy as np
    import torch
    from paper_2509_08309_b200 import hetis, workload
    torch.cuda.set_device(0)
    shape = workload.Shape(64, 8, 128, 16, "bf16")
    s = hetis.make_shape(shape)
    lens = torch.tensor([700, 33, 2049], dtype=torch.int32)
    b = workload.make_decode_batch(shape, lens, 5, "cuda")
    hetis.kv_append(s, b.k_new, b.v_new, b.k_pool, b.v_pool, b.block_table, b.seq_lens)
    G = 8
    if rank == 1:                               # destination: an empty pool and a table for groups 4..7
        dst_k = torch.zeros_like(b.k_pool)
        dst_v = torch.zeros_like(b.v_pool)
        perm = torch.randperm(b.k_pool.shape[0], generator=torch.Generator().manual_seed(1))
        dst_bt = torch.full((3 * 4, b.block_table.shape[2]), -1, dtype=torch.int32)
        off = 0
        for j in range(3):
            n = (int(lens[j]) + 15) // 16
            for gg in range(4):
                dst_bt[j * 4 + gg, :n] = perm[off:off + n].int()
                off += n
        dst_bt = dst_bt.cuda()
        q_out.put((dst_k, dst_v, dst_bt))
        barrier.wait(timeout=120)               # rank 0 pushed and synchronised
        torch.cuda.synchronize()
        ok = True
        for j in range(3):
            for gg in range(4):
                n = int(lens[j])
                t = torch.arange(n)
                sp = b.block_table[j, 4 + gg, t // 16].long().cpu()
                dp_ = dst_bt[j * 4 + gg, t // 16].long().cpu()
                ok &= torch.equal(dst_k[dp_.cuda(), (t % 16).cuda()], b.k_pool[sp.cuda(), (t % 16).cuda()])
                ok &= torch.equal(dst_v[dp_.cuda(), (t % 16).cuda()], b.v_pool[sp.cuda(), (t % 16).cuda()])
        res.put((rank, bool(ok)))
        barrier.wait(timeout=120)
    else:                                       # source: push groups 4..7 of every request to rank 1
        dst_k, dst_v, dst_bt = q_in.get(timeout=120)
        src_bt = b.block_table.reshape(3 * G, -1).contiguous()
        entries = torch.tensor([[j * G + 4 + gg, j * 4 + gg, int(lens[j])] for j in range(3) for gg in range(4)],
                               dtype=torch.int32, device="cuda")
        hetis.kv_migrate(s, entries, b.k_pool, b.v_pool, src_bt, dst_k, dst_v, dst_bt)
        torch.cuda.synchronize()
        barrier.wait(timeout=120)
        res.put((rank, True))
        barrier.wait(timeout=120)


def test_push_migration_into_peer_process_pools():
    ctx = mp.get_context("spawn")
    a2b, b2a, res = ctx.Queue(), ctx.Queue(), ctx.Queue()
    barrier = ctx.Barrier(2)
    ps = [ctx.Process(target=_rank, args=(0, b2a, a2b, barrier, res)),
          ctx.Process(target=_rank, args=(1, a2b, b2a, barrier, res))]
    for p in ps:
        p.start()
    out = [res.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, ok in out), out
