"""Hetis' head-wise dispatching on top of the measured B200 kernel.

* Cost models (§5.1): attention time tau_i = a_i h_i + b_i g_i + c_i (Eq. 3,
  PAPER.md:419-423) and transfer time rho_i = gamma_i d_i + beta_i with
  d_i = (2 + 2/r) h_i head-vectors (Eq. 4), fitted by ordinary
  least squares (the paper fits on an 8 x 8 grid).
* Dispatch (§5.2.2): the min-max program of Eq. 7 solved as a
  linear program ("reformulated as a linear programming
  problem"; the paper used cvxpy + MOSEK, PAPER.md:549 -- here scipy's HiGHS),
  then rounded to whole kv groups (x / r in N) by largest-remainder
  apportionment so every request keeps exactly H heads (Eq. 7c), with a repair
  pass for the cache budget.
* State update (Eq. 8): h_i += sum_j x_i^j,
  g_i += (2/r) sum_j x_i^j l_j.

Units (reading 13 in DESIGN.md): g and the capacity M are counted in cached
K/V head-vectors (one token of one kv head = 2 vectors, K and V), which is the
unit Eq. 8 accumulates in; the budget is then g_i + (2/r) sum_j x_i^j l_j <= M_i
(Eq. 6 / 7b rewritten in Eq. 8's units).  The plan a dispatch returns feeds
`hetis_plan_create(per_request=1)` or, for a uniform split, a global plan.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field, replace

import numpy as np


# ---------------------------------------------------------------- cost models (Eq. 3, Eq. 4)
class FitError(ValueError):
    pass


def fit_linear(X: np.ndarray, y: np.ndarray, nonneg: bool = False) -> np.ndarray:
    """Ordinary least squares y ~ X @ beta with an explicit rank check (no silent pseudo-inverse).

    nonneg: a negative fitted coefficient is clamped to 0 and the model refitted with the remaining
    terms, repeatedly -- a time model with a negative per-head or per-byte cost
    would reward the dispatcher for loading a device."""
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if X.ndim != 2 or y.shape != (X.shape[0],):
        raise FitError("shape mismatch")
    if X.shape[0] < X.shape[1]:
        raise FitError(f"need at least {X.shape[1]} samples, got {X.shape[0]}")
    if np.linalg.matrix_rank(X) < X.shape[1]:
        raise FitError("design matrix is rank deficient: vary every regressor independently")
    beta, *_ = np.linalg.lstsq(X, y, rcond=None)
    if not nonneg:
        return beta
    keep = np.ones(X.shape[1], dtype=bool)
    while (beta < 0).any():
        keep[int(np.argmin(np.where(keep, beta, np.inf)))] = False   # clamp the most negative term to 0
        beta = np.zeros(X.shape[1])
        if keep.any():
            beta[keep], *_ = np.linalg.lstsq(X[:, keep], y, rcond=None)
    return beta


@dataclass(frozen=True)
class AttentionCost:
    """tau = a h + b g + c (Eq. 3); for an Attention worker also gamma, beta of Eq. 4."""
    a: float
    b: float
    c: float
    gamma: float = 0.0
    beta: float = 0.0

    def attention_time(self, h: float, g: float) -> float:
        return self.a * h + self.b * g + self.c

    def transfer_time(self, h: float, r: int) -> float:
        """rho = gamma d + beta, d = (2 + 2/r) h (Eq. 4); 0 for h = 0: a worker holding no heads receives
        no message."""
        if h <= 0:
            return 0.0
        return self.gamma * (2.0 + 2.0 / r) * h + self.beta


def fit_attention_cost(h, g, tau) -> AttentionCost:
    """Fit Eq. 3 on measured (heads, cache, seconds) samples."""
    h = np.asarray(h, dtype=np.float64)
    X = np.stack([h, np.asarray(g, dtype=np.float64), np.ones_like(h)], axis=1)
    a, b, c = fit_linear(X, tau, nonneg=True)
    return AttentionCost(float(a), float(b), float(c))


def fit_transfer_cost(d, rho) -> tuple[float, float]:
    """Fit Eq. 4 rho = gamma d + beta on (head-vectors moved, seconds) samples."""
    d = np.asarray(d, dtype=np.float64)
    gamma, beta = fit_linear(np.stack([d, np.ones_like(d)], axis=1), rho, nonneg=True)
    return float(gamma), float(beta)


def model_accuracy(pred, meas) -> np.ndarray:
    """Per-sample accuracy 1 - |pred - meas| / meas (the paper reports 'up to 93.8%')."""
    pred = np.asarray(pred, dtype=np.float64)
    meas = np.asarray(meas, dtype=np.float64)
    return 1.0 - np.abs(pred - meas) / meas


# ---------------------------------------------------------------- device state and f_i (Eq. 7)
@dataclass(frozen=True)
class DeviceState:
    """h: resident query heads; g: resident cache (K/V head-vectors); mem: capacity M_i in the same unit."""
    h: float
    g: float
    mem: float
    primary: bool
    cost: AttentionCost


def eval_f(dev: DeviceState, x_row, lens, r: int) -> float:
    """f_i of Eq. 7 for adding x_row[j] heads of new request j (length lens[j]) to device `dev`.

    Primary:   a (h + sum x) + b (g + (2/r) sum l x) + c
    Attention: (a + (2 + 2/r) gamma) (h + sum x) + b (g + (2/r) sum l x) + c + beta,
               beta charged only when the worker holds heads (h + sum x > 0)
    """
    x = np.asarray(x_row, dtype=np.float64)
    l = np.asarray(lens, dtype=np.float64)
    heads = dev.h + x.sum()
    cache = dev.g + (2.0 / r) * float((l * x).sum())
    k = dev.cost
    if dev.primary:
        return k.a * heads + k.b * cache + k.c
    return (k.a + (2.0 + 2.0 / r) * k.gamma) * heads + k.b * cache + k.c + (k.beta if heads > 0 else 0.0)


def _coeffs(dev: DeviceState, r: int, loaded: bool = True):
    """f_i(x) = sum_j (alpha + b (2/r) l_j) x_j + const, for a worker that is (loaded) or is not
    (idle: it receives nothing, so no beta) carrying heads."""
    k = dev.cost
    alpha = k.a if dev.primary else k.a + (2.0 + 2.0 / r) * k.gamma
    const = alpha * dev.h + k.b * dev.g + k.c + (k.beta if (not dev.primary and loaded) else 0.0)
    return alpha, const


class InfeasibleError(RuntimeError):
    pass


@dataclass
class Dispatch:
    x: np.ndarray               # [N][J] integer heads, multiples of r, columns sum to H
    objective: float            # max_i f_i of the rounded allocation
    lp_objective: float         # optimum of the continuous relaxation
    per_device_f: list = field(default_factory=list)


def dispatch(devices: list[DeviceState], lens, H: int, r: int) -> Dispatch:
    """Solve Eq. 7 for the new requests `lens` (tokens each) over `devices`."""
    lens = np.asarray(lens, dtype=np.float64)
    N, J = len(devices), len(lens)
    if H % r:
        raise ValueError("H must be a multiple of r")
    if J == 0:
        f = [eval_f(d, np.zeros(0), lens, r) for d in devices]
        return Dispatch(np.zeros((N, 0), dtype=np.int64), max(f), max(f), f)
    # beta is charged only to a worker that receives heads: a fixed charge, so the LP is
    # solved once per set of idle Attention workers allowed to take heads (the others stay idle, x = 0),
    # and the best rounded allocation over the sets is kept.  2^k LPs for k idle workers with beta > 0.
    optional = [i for i, d in enumerate(devices) if not d.primary and d.h <= 0 and d.cost.beta > 0]
    if len(optional) > 10:
        optional = []                          # too many subsets: every worker may take heads
    best, lp_best, last_msg = None, np.inf, ""
    for mask in range(1 << len(optional)):
        active = [True] * N
        for k, i in enumerate(optional):
            active[i] = bool(mask >> k & 1)
        res = _solve_lp(devices, lens, H, r, active)
        if res.status != 0:
            last_msg = res.message
            continue
        lp_best = min(lp_best, float(res.x[-1]))
        try:
            x = _round_groups(res.x[:-1].reshape(N, J), H, r)
            x = _repair_budget(devices, x, lens, r)
        except InfeasibleError as exc:
            last_msg = str(exc)
            continue
        x = _improve(devices, x, lens, r)
        f = [eval_f(d, x[i], lens, r) for i, d in enumerate(devices)]
        if best is None or max(f) < max(best[1]) * (1 - 1e-12):
            best = (x, f)
    if best is None:
        need = (2.0 / r) * H * float(lens.sum())
        free = sum(d.mem - d.g for d in devices)
        raise InfeasibleError(f"no feasible dispatch (cache needed {need:.0f} head-vectors, free {free:.0f}): "
                              f"{last_msg}")
    x, f = best
    return Dispatch(x, max(f), lp_best, f)


def _solve_lp(devices, lens, H: int, r: int, active):
    """The Eq. 7 relaxation with the workers marked inactive held at x = 0 (and charged no beta)."""
    from scipy.optimize import linprog
    N, J = len(devices), len(lens)
    # variables: x[i, j] (row major) then T
    nv = N * J + 1
    cvec = np.zeros(nv)
    cvec[-1] = 1.0
    A_ub, b_ub = [], []
    for i, d in enumerate(devices):
        alpha, const = _coeffs(d, r, loaded=active[i])
        row = np.zeros(nv)
        row[i * J:(i + 1) * J] = alpha + d.cost.b * (2.0 / r) * lens
        row[-1] = -1.0
        A_ub.append(row)                      # f_i(x) - T <= 0   (Eq. 7a)
        b_ub.append(-const)
        cap = np.zeros(nv)
        cap[i * J:(i + 1) * J] = (2.0 / r) * lens
        A_ub.append(cap)                      # cache budget      (Eq. 7b, Eq. 8 units)
        b_ub.append(d.mem - d.g)
    A_eq, b_eq = [], []
    for j in range(J):
        row = np.zeros(nv)
        row[[i * J + j for i in range(N)]] = 1.0
        A_eq.append(row)                      # sum_i x_i^j = H   (Eq. 7c)
        b_eq.append(float(H))
    bounds = []
    for i in range(N):
        bounds += [(0.0, float(H) if active[i] else 0.0)] * J
    bounds.append((None, None))
    return linprog(cvec, A_ub=np.array(A_ub), b_ub=np.array(b_ub), A_eq=np.array(A_eq), b_eq=np.array(b_eq),
                   bounds=bounds, method="highs")


def _round_groups(xr: np.ndarray, H: int, r: int) -> np.ndarray:
    """Largest-remainder apportionment of each request's H / r kv groups (sum preserved exactly)."""
    N, J = xr.shape
    groups = H // r
    x = np.zeros((N, J), dtype=np.int64)
    for j in range(J):
        q = np.clip(xr[:, j], 0.0, None) / r
        base = np.floor(q + 1e-9).astype(np.int64)
        rem = groups - int(base.sum())
        frac = q - base
        for i in np.argsort(-frac, kind="stable")[:max(rem, 0)]:
            base[i] += 1
        while base.sum() > groups:             # numerical overshoot guard
            base[int(np.argmax(base))] -= 1
        x[:, j] = base * r
    return x


def _repair_budget(devices, x, lens, r):
    """Move r-head chunks off devices over their cache budget to the feasible device with the smallest f."""
    x = x.copy()
    N, J = x.shape

    def used(i):
        return devices[i].g + (2.0 / r) * float((lens * x[i]).sum())

    for _ in range(N * int(x.sum() // max(r, 1)) + 1):
        over = [i for i in range(N) if used(i) > devices[i].mem + 1e-9]
        if not over:
            return x
        i = over[0]
        js = [j for j in range(J) if x[i, j] > 0]
        j = max(js, key=lambda jj: lens[jj])   # the largest request frees the most cache per move
        best, best_f = None, None
        for k in range(N):
            if k == i or used(k) + (2.0 / r) * lens[j] * r > devices[k].mem + 1e-9:
                continue
            trial = x[k].copy()
            trial[j] += r
            fk = eval_f(devices[k], trial, lens, r)
            if best_f is None or fk < best_f:
                best, best_f = k, fk
        if best is None:
            raise InfeasibleError("rounded allocation cannot be repaired within the cache budgets")
        x[i, j] -= r
        x[best, j] += r
    raise InfeasibleError("budget repair did not converge")


def _improve(devices, x, lens, r, max_moves: int = 256):
    """Post-rounding local search on whole r-head chunks (the LP relaxation is the lower bound it approaches):
    a move of one chunk of request j from device i to k, or a swap of a chunk of j1 (i -> k) with a chunk
    of j2 (k -> i), is taken when it keeps every cache budget and lowers the vector of per-device times
    sorted in decreasing order (lexicographic min-max: a move that cannot lower the maximum yet but lowers
    the runner-up opens the next one)."""
    x = x.copy()
    N, J = x.shape

    def key(xx):
        return sorted((eval_f(d, xx[i], lens, r) for i, d in enumerate(devices)), reverse=True)

    def fits(xx, i):
        return devices[i].g + (2.0 / r) * float((lens * xx[i]).sum()) <= devices[i].mem + 1e-9

    def better(a, b):
        for u, v in zip(a, b):
            if u < v * (1 - 1e-12):
                return True
            if u > v * (1 + 1e-12):
                return False
        return False

    cur = key(x)
    for _ in range(max_moves):
        best_x, best_key = None, cur
        for i in range(N):
            for k in range(N):
                if k == i:
                    continue
                for j in range(J):
                    if x[i, j] < r:
                        continue
                    trial = x.copy()
                    trial[i, j] -= r
                    trial[k, j] += r
                    if fits(trial, k):
                        kk = key(trial)
                        if better(kk, best_key):
                            best_x, best_key = trial, kk
                    for j2 in range(J):                     # swap: a chunk of j2 goes back k -> i
                        if j2 == j or trial[k, j2] < r:
                            continue
                        t2 = trial.copy()
                        t2[k, j2] -= r
                        t2[i, j2] += r
                        if fits(t2, k) and fits(t2, i):
                            kk = key(t2)
                            if better(kk, best_key):
                                best_x, best_key = t2, kk
        if best_x is None:
            return x
        x, cur = best_x, best_key
    return x


def commit(devices: list[DeviceState], x: np.ndarray, lens, r: int) -> list[DeviceState]:
    """Eq. 8: h_i += sum_j x_i^j; g_i += (2/r) sum_j x_i^j l_j."""
    lens = np.asarray(lens, dtype=np.float64)
    out = []
    for i, d in enumerate(devices):
        out.append(replace(d, h=d.h + float(x[i].sum()), g=d.g + (2.0 / r) * float((lens * x[i]).sum())))
    return out


def brute_force_optimum(devices: list[DeviceState], lens, H: int, r: int) -> float:
    """Exhaustive optimum over all integral allocations (multiples of r) within the budgets -- test oracle
    for small instances (<= 3 devices, <= 3 requests).  Every allocation is enumerated (as one numpy
    array) and evaluated with the same f_i as eval_f, term by term."""
    lens = np.asarray(lens, dtype=np.float64)
    N, J = len(devices), len(lens)
    groups = H // r
    per_req = np.array([c for c in itertools.product(range(groups + 1), repeat=N) if sum(c) == groups],
                       dtype=np.float64) * r                                        # [P][N]
    idx = np.array(list(itertools.product(range(len(per_req)), repeat=J)), dtype=np.int64).reshape(-1, J)
    X = per_req[idx]                                                                # [C][J][N]
    worst = np.full(X.shape[0], -np.inf)
    ok = np.ones(X.shape[0], dtype=bool)
    for i, d in enumerate(devices):
        xi = X[:, :, i]                                                             # [C][J]
        heads = d.h + xi.sum(axis=1)
        cache = d.g + (2.0 / r) * (xi * lens[None, :]).sum(axis=1)
        ok &= cache <= d.mem + 1e-9
        k = d.cost
        if d.primary:
            f = k.a * heads + k.b * cache + k.c
        else:
            f = (k.a + (2.0 + 2.0 / r) * k.gamma) * heads + k.b * cache + k.c + np.where(heads > 0, k.beta, 0.0)
        worst = np.maximum(worst, f)
    return float(worst[ok].min()) if ok.any() else np.inf


def plan_rows(x: np.ndarray) -> list[int]:
    """Flatten a [N][J] allocation into hetis_plan_create(per_request=1)'s [J][N] row-major x."""
    return [int(v) for v in np.asarray(x).T.reshape(-1)]


# ---------------------------------------------------------------- re-dispatch migration (row f4)
def group_owners(x_row, r: int) -> np.ndarray:
    """Device of every kv group of one request under a plan row x_i (i = device): device i owns the
    contiguous head range [b_i, b_i + x_i), b_i = sum_{i' < i} x_i' (reading 3), i.e. groups
    [b_i / r, (b_i + x_i) / r)."""
    x = np.asarray(x_row, dtype=np.int64)
    if (x < 0).any() or (x % r).any():
        raise ValueError("head counts must be non-negative multiples of r (PAPER.md:454)")
    return np.repeat(np.arange(len(x)), x // r)


@dataclass
class Migration:
    """KV movement of one re-dispatched request ("only partial cache transmission").

    moves     : (kv group g, source device, destination device), ascending g -- the groups whose
                owner changes; every other group's pages stay where they are (reused)
    reused    : number of kv groups that stay on their device
    new_owner : device of every kv group after the move (groups of one device need not be contiguous:
                the kernels take any (request, kv head) unit list, hetis_attn_decode_units)
    """
    moves: list[tuple[int, int, int]]
    reused: int
    new_owner: list[int] = field(default_factory=list)

    def moved_bytes(self, seq_len: int, head_dim: int, elem_bytes: int, n_layers: int = 1) -> int:
        """K and V bytes the moves transfer: groups x L tokens x 2 x d x elem x layers."""
        return len(self.moves) * seq_len * 2 * head_dim * elem_bytes * n_layers


def plan_migration(old_row, new_row, r: int, old_owner=None) -> Migration:
    """Groups of one request that must move when its allocation changes from old_row to new_row heads
    per device ("leverages the overlap in head distribution").

    Every device keeps min(old_i, new_i) / r of the groups it holds -- the maximum reuse, so exactly
    H / r - sum_i min(old_i, new_i) / r groups move.  A device with a surplus releases its
    lowest-index groups first; devices with a deficit, in device-id order, take the released groups in
    ascending order.  old_owner: device of every kv group now (default: the contiguous ranges of
    old_row, reading 3).  The result's new_owner is in general not contiguous per device."""
    old, new = np.asarray(old_row, dtype=np.int64), np.asarray(new_row, dtype=np.int64)
    if old.shape != new.shape:
        raise ValueError("plans cover different device counts")
    if old.sum() != new.sum():
        raise ValueError("old and new rows must both sum to H (Eq. 5)")
    o = group_owners(old, r) if old_owner is None else np.asarray(old_owner, dtype=np.int64)
    group_owners(new, r)                                   # validates new_row (multiples of r)
    if len(o) != old.sum() // r or any(int((o == i).sum()) != old[i] // r for i in range(len(old))):
        raise ValueError("old_owner does not match old_row")
    owner = o.copy()
    released = []
    for i in range(len(old)):
        surplus = (old[i] - new[i]) // r
        if surplus > 0:
            released += [int(g) for g in np.flatnonzero(o == i)[:surplus]]
    released.sort()
    k = 0
    for i in range(len(new)):
        for _ in range(max(0, (new[i] - old[i]) // r)):
            owner[released[k]] = i
            k += 1
    moves = [(int(g), int(o[g]), int(owner[g])) for g in range(len(o)) if o[g] != owner[g]]
    return Migration(moves=moves, reused=int((o == owner).sum()), new_owner=[int(v) for v in owner])


def owner_units(owners, num_devices: int) -> list[list[tuple[int, int]]]:
    """Per device, its (request, kv group) units in ascending (request, group) order -- the block-table row
    order of the device and the unit list hetis_attn_decode_units runs -- from every request's group
    owners (owners[j][g] = device)."""
    out: list[list[tuple[int, int]]] = [[] for _ in range(num_devices)]
    for j, own in enumerate(owners):
        for g, d in enumerate(own):
            out[int(d)].append((j, g))
    return out


def migration_entries(old_units: list[list[tuple[int, int]]], new_units: list[list[tuple[int, int]]],
                      migrations: dict[int, Migration], seq_lens) -> dict[tuple[int, int], np.ndarray]:
    """hetis_kv_migrate entries per (source, destination) device pair.

    old_units / new_units: per device, the (request, global kv group) units of the old / new
    per-request plan (hetis_plan_units order = block-table row order, one row per unit).
    migrations: request -> Migration.  Returns {(src, dst): int32 [n][3] (src_row, dst_row, L_j)}."""
    old_row = [{u: k for k, u in enumerate(units)} for units in old_units]
    new_row = [{u: k for k, u in enumerate(units)} for units in new_units]
    out: dict[tuple[int, int], list[list[int]]] = {}
    for j in sorted(migrations):
        for g, src, dst in migrations[j].moves:
            out.setdefault((src, dst), []).append([old_row[src][(j, g)], new_row[dst][(j, g)], int(seq_lens[j])])
    return {k: np.asarray(v, dtype=np.int32) for k, v in out.items()}
