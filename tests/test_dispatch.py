"""Cost models (Eq. 3, Eq. 4) and the Eq. 7 dispatcher (CPU only).

Worked examples follow SPEC.md's dispatcher interface with the
paper's formulas; optimality is pinned by exhaustive
enumeration on small instances.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from paper_2509_08309_b200 import dispatch
from paper_2509_08309_b200 import dispatch as dp
from paper_2509_08309_b200 import hetis


def test_fit_recovers_known_coefficients():
    rng = np.random.default_rng(0)
    h = np.repeat(np.arange(1, 9) * 40.0, 8)
    g = np.tile(np.arange(1, 9) * 1e6, 8)
    tau = 2e-8 * h + 1.5e-12 * g + 4e-6
    noisy = tau * (1 + 1e-3 * rng.standard_normal(tau.shape))
    m = dp.fit_attention_cost(h, g, noisy)
    assert abs(m.a - 2e-8) / 2e-8 < 0.05 and abs(m.b - 1.5e-12) / 1.5e-12 < 0.01 and abs(m.c - 4e-6) / 4e-6 < 0.05
    acc = dp.model_accuracy([m.attention_time(a, b) for a, b in zip(h, g)], tau)
    assert acc.min() > 0.99
    gamma, beta = dp.fit_transfer_cost([1, 2, 3, 4], [3.0, 5.0, 7.0, 9.0])
    assert abs(gamma - 2.0) < 1e-12 and abs(beta - 1.0) < 1e-12


def test_fit_rejects_rank_deficient_or_short_designs():
    with pytest.raises(dp.FitError):
        dp.fit_attention_cost([1, 2], [1, 2], [1, 2])                      # fewer samples than coefficients
    with pytest.raises(dp.FitError):
        dp.fit_attention_cost([1, 2, 3, 4], [2, 4, 6, 8], [1, 2, 3, 4])    # g proportional to h
    with pytest.raises(dp.FitError):
        dp.fit_attention_cost([5, 5, 5], [1, 2, 3], [1, 2, 3])             # h never varies


def test_eval_f_worked_examples():
    # primary, nothing added -> pure Eq. 3
    k = dp.AttentionCost(a=1e-4, b=1e-7, c=2e-5)
    d = dp.DeviceState(h=8, g=1000, mem=1e9, primary=True, cost=k)
    assert dp.eval_f(d, [0], [100], 1) == pytest.approx(1e-4 * 8 + 1e-7 * 1000 + 2e-5)
    # attention worker, h = 0, one request x = r = 1, l = 100:
    # (a + (2 + 2/r) gamma) * 1 + b * (2/r) * 100 + c + beta
    kw = dp.AttentionCost(a=1e-4, b=1e-7, c=0.0, gamma=1e-6, beta=1e-4)
    w = dp.DeviceState(h=0, g=0, mem=1e9, primary=False, cost=kw)
    assert dp.eval_f(w, [1], [100], 1) == pytest.approx(2.24e-4)


def test_transfer_and_beta_only_for_loaded_workers():
    """rho = 0 for h = 0; an Attention worker holding no heads pays no beta
    (SPEC.md:160, :299), and the dispatcher leaves a worker idle when its beta outweighs its help."""
    k = dp.AttentionCost(a=1e-4, b=1e-7, c=0.0, gamma=1e-6, beta=1e-4)
    assert k.transfer_time(0, 1) == 0.0
    assert k.transfer_time(2, 1) == pytest.approx(1e-6 * 4 * 2 + 1e-4)
    idle = dp.DeviceState(h=0, g=0, mem=1e9, primary=False, cost=k)
    assert dp.eval_f(idle, [0, 0], [100, 50], 1) == 0.0
    prim = dp.DeviceState(0, 0, 1e12, True, dp.AttentionCost(1e-6, 1e-9, 1e-6))
    slow_link = dp.DeviceState(0, 0, 1e12, False, dp.AttentionCost(1e-6, 1e-9, 1e-6, gamma=1e-9, beta=1.0))
    out = dp.dispatch([prim, slow_link], [100], H=8, r=1)
    assert out.x[1].sum() == 0 and out.x[0].sum() == 8
    assert out.objective == pytest.approx(dp.eval_f(prim, [8], [100], 1))
    assert out.objective == pytest.approx(dp.brute_force_optimum([prim, slow_link], [100], 8, 1))
    fast_link = dp.DeviceState(0, 0, 1e12, False, dp.AttentionCost(1e-6, 1e-9, 1e-6, gamma=1e-9, beta=1e-7))
    out = dp.dispatch([prim, fast_link], [100], H=8, r=1)
    assert out.x[1].sum() > 0                                  # a cheap link is worth using


def test_fit_clamps_negative_coefficients_and_refits():
    """a negative fitted coefficient is clamped to 0 and the rest refitted."""
    h = np.repeat(np.arange(1, 9) * 40.0, 8)
    g = np.tile(np.arange(1, 9) * 1e6, 8)
    tau = -3e-9 * h + 1.5e-12 * g + 4e-6                       # planted negative per-head cost
    m = dp.fit_attention_cost(h, g, tau)
    assert m.a == 0.0 and m.b > 0 and m.c > 0
    X = np.stack([g, np.ones_like(g)], axis=1)
    b_ref, c_ref = np.linalg.lstsq(X, tau, rcond=None)[0]      # the refit on the remaining terms
    assert m.b == pytest.approx(b_ref, rel=1e-12) and m.c == pytest.approx(c_ref, rel=1e-12)
    gamma, beta = dp.fit_transfer_cost([1, 2, 3, 4], [1.0, 1.0, 1.0, 1.0])
    assert gamma == pytest.approx(0.0, abs=1e-15) and beta == pytest.approx(1.0)
    gamma, beta = dp.fit_transfer_cost([1, 2, 3, 4], [3.0, 2.0, 1.0, 0.5])   # negative slope -> clamped
    assert gamma == 0.0 and beta == pytest.approx(1.625)


def _devs(n, mem=1e12, primary=True, a=1e-6, b=1e-9, c=0.0):
    return [dp.DeviceState(0, 0, mem, primary, dp.AttentionCost(a, b, c)) for _ in range(n)]


def test_dispatch_single_device_and_even_split():
    one = dp.dispatch(_devs(1), [500], H=8, r=1)
    assert one.x.tolist() == [[8]]
    two = dp.dispatch(_devs(2), [500], H=8, r=1)
    assert sorted(two.x[:, 0].tolist()) == [4, 4]
    assert two.objective == pytest.approx(1e-6 * 4 + 1e-9 * 2 * 4 * 500)


def test_dispatch_budget_binding():
    # device A can hold only 2 heads' cache: 2 heads x 100 tokens x 2 (K, V) = 400 head-vectors (r = 1)
    devs = [dp.DeviceState(0, 0, 400, True, dp.AttentionCost(1e-6, 1e-9, 0.0)),
            dp.DeviceState(0, 0, 1e9, True, dp.AttentionCost(1e-6, 1e-9, 0.0))]
    out = dp.dispatch(devs, [100], H=8, r=1)
    assert out.x[:, 0].tolist() == [2, 6]


def test_dispatch_heterogeneous_speed_and_groups():
    # device 1 twice as slow per head and per byte -> about 2:1 split, in whole kv groups (r = 8)
    fast = dp.DeviceState(0, 0, 1e12, True, dp.AttentionCost(1e-7, 1e-10, 0.0))
    slow = dp.DeviceState(0, 0, 1e12, True, dp.AttentionCost(2e-7, 2e-10, 0.0))
    out = dp.dispatch([fast, slow], [2048] * 4, H=64, r=8)
    assert (out.x % 8 == 0).all() and (out.x.sum(axis=0) == 64).all()
    share_fast = out.x[0].sum() / out.x.sum()
    assert 0.6 <= share_fast <= 0.72
    plan = hetis.plan_create(hetis.make_shape(__import__("paper_2509_08309_b200.workload", fromlist=["x"]).LLAMA2_70B),
                             2, dp.plan_rows(out.x), per_request=True, num_seqs=4)
    assert plan.heads(1, seq=0) == (int(out.x[0, 0]), int(out.x[1, 0]))


def test_transfer_cost_moves_load_to_primary():
    prim = dp.DeviceState(0, 0, 1e12, True, dp.AttentionCost(1e-7, 1e-10, 0.0))
    att = dp.DeviceState(0, 0, 1e12, False, dp.AttentionCost(1e-7, 1e-10, 0.0, gamma=5e-8, beta=1e-5))
    out = dp.dispatch([prim, att], [1000], H=40, r=1)
    assert out.x[0, 0] > out.x[1, 0]                    # network cost makes the attention worker pricier


def test_commit_eq8_and_conservation():
    devs = _devs(2)
    x = np.array([[8, 0], [0, 8]])
    new = dp.commit(devs, x, [50, 10], r=2)
    assert new[0].h == 8 and new[0].g == pytest.approx((2 / 2) * 8 * 50)       # SPEC.md:322 example
    assert new[1].h == 8 and new[1].g == pytest.approx((2 / 2) * 8 * 10)
    rng = np.random.default_rng(3)
    states = _devs(3)
    total = 0.0
    for _ in range(20):
        lens = rng.integers(1, 500, size=2)
        out = dp.dispatch(states, lens, H=8, r=2)
        states = dp.commit(states, out.x, lens, r=2)
        total += (2 / 2) * 8 * float(lens.sum())
        assert (out.x.sum(axis=0) == 8).all()
    assert sum(s.g for s in states) == pytest.approx(total)


def test_infeasible_reports_shortfall():
    devs = _devs(2, mem=100)
    with pytest.raises(dp.InfeasibleError):
        dp.dispatch(devs, [1000], H=8, r=1)


def test_small_instance_optimality_against_exhaustive_enumeration():
    """<= 3 devices, <= 3 requests, H <= 8, r in {1, 2}: over 1000 random instances the rounded LP solution is
    within the rounding slack of the exhaustive optimum always, and equal to it in >= 95%."""
    rng = np.random.default_rng(7)
    exact = 0
    trials = 1000
    for _ in range(trials):
        N = int(rng.integers(1, 4))
        J = int(rng.integers(1, 4))
        r = int(rng.choice([1, 2]))
        H = int(rng.choice([4, 8]))
        devs = []
        for _i in range(N):
            k = dp.AttentionCost(a=float(rng.uniform(1e-7, 1e-6)), b=float(rng.uniform(1e-10, 1e-9)),
                                 c=float(rng.uniform(0, 1e-6)), gamma=float(rng.uniform(0, 1e-7)),
                                 beta=float(rng.uniform(0, 1e-6)))
            devs.append(dp.DeviceState(float(rng.integers(0, 64)), float(rng.integers(0, 10000)), 1e12,
                                       bool(rng.integers(0, 2)), k))
        lens = rng.integers(16, 2048, size=J)
        out = dp.dispatch(devs, lens, H, r)
        opt = dp.brute_force_optimum(devs, lens, H, r)
        slack = max(d.cost.a + (2 + 2 / r) * d.cost.gamma + d.cost.b * (2 / r) * float(lens.max()) for d in devs) \
            * r * J
        assert out.lp_objective <= opt + 1e-12
        assert out.objective <= opt + slack + 1e-12
        exact += out.objective <= opt * (1 + 1e-9)
    assert exact / trials >= 0.95, exact / trials      # SPEC.md:338 / :573; measured 0.958


# ---------------------------------------------------------------- re-dispatch migration (f4)
def test_plan_migration_golden_examples():
    """SPEC.md:407-418 examples (identity, full move with its byte count, overlap count)."""
    with open(os.path.join(os.path.dirname(__file__), "golden", "migration_plans.json")) as f:
        gx = json.load(f)
    for c in gx["cases"]:
        m = dispatch.plan_migration(c["old"], c["new"], c["r"])
        assert len(m.moves) == c["moved"] and m.reused == c["reused"], c
        pairs = {}
        for _, s, d in m.moves:
            pairs[f"{s}->{d}"] = pairs.get(f"{s}->{d}", 0) + 1
        assert pairs == c["pairs"], c
        if "moved_bytes" in c:
            assert m.moved_bytes(c["seq_len"], c["head_dim"], c["elem_bytes"], c["n_layers"]) == c["moved_bytes"]


def _owners_brute(x, r):
    """Owner of each kv group by walking the heads one by one (independent of group_owners)."""
    own, dev, left = [], 0, list(x)
    for h in range(sum(x)):
        while left[dev] == 0:
            dev += 1
        left[dev] -= 1
        if h % r == 0:
            own.append(dev)
    return own


def test_plan_migration_moves_exactly_the_set_difference():
    """SPEC.md:418 / :580: moved groups == H/r - sum_i min(old_i, new_i)/r for every allocation pair (the
    maximum reuse), each device keeps min(old_i, new_i)/r of its own groups, ends with new_i/r groups, and
    the moves are exactly the groups whose owner changes -- checked on every pair of small instances,
    against owners walked head by head."""
    import itertools
    for N, H, r in ((2, 8, 1), (2, 16, 4), (3, 6, 1), (4, 8, 2), (3, 12, 2)):
        rows = [x for x in itertools.product(range(0, H + 1, r), repeat=N) if sum(x) == H]
        for old in rows:
            for new in rows:
                m = dispatch.plan_migration(old, new, r)
                ob = _owners_brute(old, r)
                own = m.new_owner
                assert [sum(1 for d in own if d == i) for i in range(N)] == [x // r for x in new]
                assert m.moves == [(g, ob[g], own[g]) for g in range(H // r) if ob[g] != own[g]]
                bound = sum(min(a, b) for a, b in zip(old, new)) // r
                assert m.reused == bound and len(m.moves) == H // r - bound
                for i in range(N):                                   # per device reuse = min(old, new) / r
                    kept = sum(1 for g in range(H // r) if ob[g] == i and own[g] == i)
                    assert kept == min(old[i], new[i]) // r
                # chaining: a second re-dispatch starts from the non-contiguous owners
                m2 = dispatch.plan_migration(new, old, r, old_owner=own)
                assert m2.reused == bound


def test_plan_migration_rejects_inconsistent_rows():
    with pytest.raises(ValueError):
        dispatch.plan_migration([8, 0], [4, 2], 1)         # sums differ (Eq. 5)
    with pytest.raises(ValueError):
        dispatch.plan_migration([6, 2], [4, 4], 4)         # not multiples of r


def test_migration_entries_follow_plan_unit_rows():
    """Entries index the units of the old plan on the source and of the new plan on the destination
    (hetis_plan_units order: requests ascending, kv groups ascending)."""
    r = 1
    old = np.array([[4, 0], [2, 2], [0, 4]]).T                 # [N][J]
    new = old.copy()
    new[:, 1] = [0, 4]                                         # request 1 re-dispatched to device 1
    units = lambda x: [[(j, g) for j in range(x.shape[1]) for g in range(4)
                        if dispatch.group_owners(x[:, j], r)[g] == i] for i in range(2)]
    mig = {1: dispatch.plan_migration(old[:, 1], new[:, 1], r)}
    ent = dispatch.migration_entries(units(old), units(new), mig, [10, 33, 7])
    assert list(ent) == [(0, 1)]
    # old device 0 units: (0,0..3), (1,0), (1,1) -> rows 4, 5; new device 1 units: (1,0..3), (2,0..3)
    assert ent[(0, 1)].tolist() == [[4, 0, 33], [5, 1, 33]]
