#!/usr/bin/env python
"""Benchmark of the Hetis head-partitioned paged decode-attention hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One step = one layer's decode step for the whole batch on every rank:
    N = 1:  hetis_attn_partial_append (kv_append fused) -> hetis_attn_combine
    N > 1 (default, --exchange peer): hetis_attn_partial_pull (the attention kernel
            reads the rank's q / new k, v straight from the Primary's buffers over
            NVLink, append fused) -> hetis_attn_combine_peers (the combine storing
            every O row into every rank's o_full) -> hetis_peer_wait; where the rank's
            launch runs in group mode (<= one (request, kv head) pair per SM, L <= 2048:
            c3 at 8 GPUs) the merge and the stores are in the attention kernel too
            (hetis_attn_decode_peers, pull form) -> hetis_peer_wait.  --pull 0: a separate
            hetis_scatter_pull kernel first.  --exchange nccl: hetis_scatter_q -> ... ->
            hetis_attn_combine -> hetis_gather (NCCL over NVLink)
Metric (BASELINE.json): decode attention tokens/s (= batch / step time, one
layer, all heads, max over ranks) and achieved HBM GB/s of the dominant kernel
(% of the measured copy peak).  Default workload: config c2 (LLaMA2-13B, 40
heads x 128, batch 64, context 4096, bf16 paged KV) -- BASELINE.json configs[1];
at N > 1 the heads are partitioned over the ranks (strong scaling, same total
problem).  A sub-record for c3 (LLaMA2-70B GQA, the config the >= 6x scaling
target is stated on) is measured in the same run and printed inside the line.

After timing, the step is run once more and rank 0 checks the gathered O against
the fp64 oracle (every element) and against the unsplit single-device result
(bit for bit); a mismatch exits with rc 3.

Rank 0 prints ONE JSON line.  `--impl reference` times the fp64 CPU oracle
(oracle/, the only reference this tier has) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2509_08309_b200 import accounting, workload  # noqa: E402

L2_BYTES = 126 * 1024 * 1024
METRIC = "decode attention tokens/s and achieved HBM GB/s (% of peak) at 1/2/4/8 B200"
UNIT = "tokens/s"
ATOL, RTOL = 2e-3, 1e-2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2", choices=sorted(workload.CONFIGS))
    ap.add_argument("--sub-config", default="auto",
                    help="second workload measured in the same run ('auto': c3 unless --config is c3; 'none')")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-seqs", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the post-timing oracle / unsplit check")
    ap.add_argument("--o-dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--attn-flags", type=int, default=0, help="HETIS_ATTN_* flags (diagnostics)")
    ap.add_argument("--graph", type=int, default=1, help="replay the K timed steps as one CUDA graph")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="N > 1: peer-memory scatter/gather kernels (default) or NCCL scatter_q / gather")
    ap.add_argument("--gather-root", type=int, default=-1,
                    help="-1: every rank receives O (all-gather); r >= 0: only rank r (gather to the Primary)")
    ap.add_argument("--pull", type=int, default=1,
                    help="N > 1 peer exchange: the attention kernel reads q / new k, v from the Primary "
                         "(hetis_attn_partial_pull) instead of a separate pull-scatter kernel")
    ap.add_argument("--fused-append", type=int, default=1,
                    help="1: kv_append fused into the attention kernel (hetis_attn_partial_append); 0: separate")
    ap.add_argument("--force-dist", action="store_true",
                    help="debug: run the N > 1 code path (process group, exchanges) at N = 1")
    ap.add_argument("--share-gpu", action="store_true",
                    help="debug: every rank on cuda:0 with a gloo bootstrap group (correctness of the N > 1 peer "
                         "path on a one-GPU box; timings are meaningless)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profiles(key: str):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        v = d.get(key)
        return None if v is None else float(v)
    except Exception:
        return None


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------- clocks sampled during the timed region
class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
               0x2: "applications_clocks_setting"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- CPU oracle timing
def cpu_oracle_sample(cfg: workload.Config, n_seqs: int, budget_s: float = 20.0):
    """Time the fp64 oracle (as it stands) on a CPU-generated batch of the workload's first n_seqs requests
    and ALL heads, at the workload's lengths: once on all host cores and once on one thread (the one-thread
    run on fewer requests if the all-core time says it would exceed budget_s)."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    lens_all = cfg.seq_lens()
    dt = oracle.BF16 if cfg.shape.dtype == "bf16" else oracle.F32

    def timed(n, threads):
        lens = lens_all[:n]
        b = workload.make_decode_batch(cfg.shape, lens, cfg.seed, "cpu")
        h = {k: workload.to_numpy_bits(getattr(b, k)).copy() for k in ("q", "k_new", "v_new", "k_pool", "v_pool")}
        bt, sl = b.block_table.numpy(), b.seq_lens.numpy()
        t0 = time.perf_counter()
        oracle.kv_append(h["k_new"], h["v_new"], h["k_pool"], h["v_pool"], bt, sl)
        oracle.decode(h["q"], h["k_pool"], h["v_pool"], bt, sl, num_kv_heads=cfg.shape.num_kv_heads, dtype=dt,
                      nthreads=threads)
        return time.perf_counter() - t0, int(lens.sum())

    n = min(n_seqs, cfg.batch)
    sec_all, tok_all = timed(n, cores)
    n1 = max(1, min(n, int(n * budget_s / max(sec_all * cores, 1e-9))))
    sec_1, tok_1 = timed(n1, 1)
    return {"value": n / sec_all, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": (f"{n} of {cfg.batch} requests x {cfg.shape.num_q_heads} heads at the workload's lengths "
                       f"(sum L = {tok_all}), kv_append + fp64 oracle decode, {cores} threads; one-thread run on "
                       f"{n1} requests (sum L = {tok_1})"),
            "value_1thread": n1 / sec_1, "cpu_model": cpu_model(),
            "gbs_all_cores": tok_all * cfg.shape.num_kv_heads * cfg.shape.head_dim * 2 * cfg.shape.elem_bytes
            / sec_all / 1e9}


def run_reference(args, world, rank, budget_s: float = 150.0):
    """The oracle as it stands, on this box's host cores.  The sample (requests
    per step) is sized so that warm-up + K steps take about `budget_s`."""
    import oracle
    cfg = workload.CONFIGS[args.config]
    if rank != 0:
        return 0
    n_max = min(args.cpu_sample_seqs, cfg.batch)
    lens = cfg.seq_lens()[:n_max]
    b = workload.make_decode_batch(cfg.shape, lens, cfg.seed, "cpu")
    h = {k: workload.to_numpy_bits(getattr(b, k)).copy() for k in ("q", "k_new", "v_new", "k_pool", "v_pool")}
    bt, sl = b.block_table.numpy(), b.seq_lens.numpy()
    oracle.kv_append(h["k_new"], h["v_new"], h["k_pool"], h["v_pool"], bt, sl)
    cores = len(os.sched_getaffinity(0))
    dt = oracle.BF16 if cfg.shape.dtype == "bf16" else oracle.F32

    def run(n):
        t0 = time.perf_counter()
        oracle.decode(h["q"][:n], h["k_pool"], h["v_pool"], bt[:n], sl[:n], num_kv_heads=b.kv_count, dtype=dt,
                      nthreads=cores)
        return time.perf_counter() - t0

    t1 = run(1)                                   # calibration = warm-up
    per_step = budget_s / max(args.steps + args.warmup, 1)
    n = int(max(1, min(n_max, per_step // max(t1, 1e-6))))
    for _ in range(args.warmup):
        run(n)
    times = [run(n) for _ in range(max(args.steps, 1))]
    sec = sum(times) / len(times)
    value = n / sec
    sample = (f"{n} of {cfg.batch} requests x {cfg.shape.num_q_heads} heads at the workload's lengths "
              f"(sum L = {int(sl[:n].sum())}), fp64 oracle decode, {cores} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.description}", "batch_sampled": n, "batch": cfg.batch},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample + " per step", "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm
class Dist:
    """Process-group plumbing: barrier, max over ranks, object broadcast (NCCL, or gloo with --share-gpu)."""

    def __init__(self, active: bool, world: int, local: int, device, backend: str):
        self.active, self.world, self.local, self.device, self.backend = active, world, local, device, backend

    def barrier(self):
        if self.active:
            import torch.distributed as dist
            if self.backend == "nccl":
                dist.barrier(device_ids=[self.local])
            else:
                dist.barrier()
        torch.cuda.synchronize(self.device)

    def max(self, x: float) -> float:
        if not self.active or self.world == 1:
            return x
        import torch.distributed as dist
        dev = self.device if self.backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.active or self.world == 1:
            return x
        import torch.distributed as dist
        dev = self.device if self.backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())


def measure(args, cfg_name: str, D: Dist, rank: int, world: int, comm_ptr, headline: bool):
    """Time cfg_name's step on this rank's share; returns the record (meaningful on rank 0)."""
    from paper_2509_08309_b200 import hetis
    from paper_2509_08309_b200.step import DecodeStep

    device = D.device
    cfg = workload.CONFIGS[cfg_name]
    shape = cfg.shape
    split = cfg.head_split(world)
    dist_mode = D.active
    peer = dist_mode and args.exchange == "peer"
    exchange_note = args.exchange
    B = cfg.batch
    seq_lens = cfg.seq_lens()
    max_len = int(seq_lens.max())
    cs = hetis.make_shape(shape, args.o_dtype)
    plan = hetis.plan_create(cs, world, split)
    q_begin, q_count = plan.heads(rank)
    batch = workload.make_decode_batch(shape, seq_lens, cfg.seed, device, q_begin=q_begin, q_count=q_count,
                                       rank_salt=rank)
    step = DecodeStep(shape, plan, rank, B, max_len, device, o_dtype=args.o_dtype,
                      comm_ptr=comm_ptr if dist_mode else None)
    kv_bytes_rank = accounting.step_bytes(seq_lens.tolist(), q_count, shape.r, shape.head_dim, shape.page_size,
                                          shape.elem_bytes, shape.elem_bytes, 4).kv
    # rotate layer pools so the per-step KV stream never sits in L2
    n_layers = max(1, math.ceil(4 * L2_BYTES / max(kv_bytes_rank, 1)))
    free = torch.cuda.mem_get_info(device)[0]
    pool_bytes = 2 * batch.k_pool.numel() * batch.k_pool.element_size()
    n_layers = max(1, min(n_layers, int(0.5 * free // max(pool_bytes * (world if args.share_gpu else 1), 1)) + 1))
    k_pools = [batch.k_pool] + [batch.k_pool.clone() for _ in range(n_layers - 1)]
    v_pools = [batch.v_pool] + [batch.v_pool.clone() for _ in range(n_layers - 1)]
    odt = torch.bfloat16 if args.o_dtype == "bf16" else torch.float32
    is_root = rank == 0
    gather_root = args.gather_root
    receives = gather_root < 0 or gather_root == rank
    q_full = kn_full = vn_full = None
    if dist_mode:
        if is_root:     # the Primary holds the step's inputs for every head (the logical problem's q, new k, v)
            q_full = workload.make_q(shape, B, cfg.seed, device)
            kn_full, vn_full = workload.make_new_rows(shape, seq_lens, cfg.seed, device)
        o_full = torch.empty((B, shape.num_q_heads, shape.head_dim), dtype=odt, device=device) if receives else None
        if peer:
            # the peer mappings need peer access between every pair of GPUs; if setting them up fails on
            # every rank, the step falls back to the NCCL exchange (same plan, same parity check)
            try:
                step.setup_peers(o_full, q_full, kn_full, vn_full, gather_root=gather_root)
                ok = 1.0
            except Exception as exc:  # noqa: BLE001
                print(f"rank {rank}: peer-memory exchange unavailable ({type(exc).__name__}: {exc})",
                      file=sys.stderr, flush=True)
                ok = 0.0
            if D.max(1.0 - ok) > 0 and comm_ptr is not None:
                peer = False
                exchange_note = "nccl (peer-memory setup failed on some rank)"
                if o_full is None:
                    o_full = torch.empty((B, shape.num_q_heads, shape.head_dim), dtype=odt, device=device)
            elif D.max(1.0 - ok) > 0:
                raise SystemExit("peer-memory exchange setup failed and no NCCL communicator to fall back to")
        if not peer and o_full is None:
            o_full = torch.empty((B, shape.num_q_heads, shape.head_dim), dtype=odt, device=device)
    else:
        step.buf.q_shard.copy_(batch.q)
        step.buf.k_new.copy_(batch.k_new)
        step.buf.v_new.copy_(batch.v_new)
        o_full = step.buf.o_shard
    stream = torch.cuda.current_stream(device)
    if peer and q_count > 0:   # the roofline's attention-only launches read the dense shard: this rank's inputs
        step.buf.q_shard.copy_(batch.q)
        step.buf.k_new.copy_(batch.k_new)
        step.buf.v_new.copy_(batch.v_new)
    # the local step (N = 1, and the NCCL exchange) through the library's one-call step,
    # hetis_attn_decode_append: the attention kernel with the append fused, then the combine kernel -- or ONE
    # kernel with the merge fused: automatically in group mode (<= one (request, kv head) pair per SM, <= 8
    # splits), opt-in elsewhere with --attn-flags 0x20 (measured slower there)
    fused = (not peer) and bool(args.fused_append)
    merge_in_kernel = fused and hetis.attn_decode_launches_for(step.cshape, B, q_count, max_len,
                                                               args.attn_flags) == 1

    # over peer memory the merge (+ the stores into every rank's o_full) is fused into the attention kernel where
    # this rank's launch runs in group mode (or with --attn-flags 0x20)
    fused_peer = peer and bool(args.fused_append) and step.merge_fused_default(args.attn_flags)
    # the scatter folded into the attention kernel (it reads q / new k, v from the Primary): the default
    pull = peer and bool(args.fused_append) and bool(args.pull) and step.pull_supported(args.attn_flags)

    def attention(li):
        if pull and fused_peer:   # pull + append + attention + split merge + the stores into every rank's o_full
            hetis.attn_decode_peers_pull(step.group, B, k_pools[li], v_pools[li], batch.block_table,
                                         batch.seq_lens, max_len, step.buf.workspace, flags=args.attn_flags)
        elif pull:
            hetis.attn_partial_pull(step.group, B, k_pools[li], v_pools[li], batch.block_table, batch.seq_lens,
                                    max_len, step.buf.workspace, flags=args.attn_flags & ~hetis.ATTN_FUSED_MERGE)
        elif fused_peer:          # append + attention + split merge + the stores into every rank's o_full
            hetis.attn_decode_peers(step.group, step.buf.q_shard, k_pools[li], v_pools[li], batch.block_table,
                                    batch.seq_lens, max_len, step.buf.workspace, k_new_shard=step.buf.k_new,
                                    v_new_shard=step.buf.v_new, flags=args.attn_flags)
        elif fused:             # append + attention + split merge, O straight into the shard
            hetis.attn_decode_append(step.cshape, step.buf.q_shard, step.buf.k_new, step.buf.v_new, k_pools[li],
                                     v_pools[li], batch.block_table, batch.seq_lens, max_len, step.buf.o_shard,
                                     step.buf.workspace, q_head_begin=q_begin, flags=args.attn_flags)
        elif args.fused_append:   # the append happens inside the attention kernel
            hetis.attn_partial_append(step.cshape, step.buf.q_shard, step.buf.k_new, step.buf.v_new, k_pools[li],
                                      v_pools[li], batch.block_table, batch.seq_lens, max_len, step.buf.workspace,
                                      q_head_begin=q_begin, flags=args.attn_flags)
        else:
            step.append(k_pools[li], v_pools[li], batch.block_table, batch.seq_lens)
            hetis.attn_partial(step.cshape, step.buf.q_shard, k_pools[li], v_pools[li], batch.block_table,
                               batch.seq_lens, max_len, step.buf.workspace, q_head_begin=q_begin,
                               flags=args.attn_flags)

    def attention_only(li):
        # the dominant kernel alone (roofline): with the merge + gather fused over peer memory that kernel needs
        # the step's scatter_pull (it waits for every rank's acknowledgement of the previous o_full), so it is
        # timed as the same kernel writing the local o shard (identical arithmetic and K/V traffic)
        if fused_peer:
            hetis.attn_decode_append(step.cshape, step.buf.q_shard, step.buf.k_new, step.buf.v_new, k_pools[li],
                                     v_pools[li], batch.block_table, batch.seq_lens, max_len, step.buf.o_shard,
                                     step.buf.workspace, q_head_begin=q_begin, flags=args.attn_flags)
        elif pull or (fused and not merge_in_kernel):   # the attention kernel alone (same K/V traffic)
            hetis.attn_partial_append(step.cshape, step.buf.q_shard, step.buf.k_new, step.buf.v_new, k_pools[li],
                                      v_pools[li], batch.block_table, batch.seq_lens, max_len, step.buf.workspace,
                                      q_head_begin=q_begin, flags=args.attn_flags)
        else:
            attention(li)

    def one_step(i, ev=None):
        """ev: optional 5 events recorded between the phases (scatter | attention | combine(+gather) | wait)."""
        li = i % n_layers
        rec = (lambda k: ev[k].record(torch.cuda.current_stream(device))) if ev is not None else (lambda k: None)
        rec(0)
        if peer:
            if not pull:                 # with the pull folded into the attention kernel there is no scatter
                step.scatter_peers()
        elif dist_mode:
            step.scatter(q_full, kn_full, vn_full)
        rec(1)
        attention(li)
        rec(2)
        if peer:
            if not fused_peer:
                hetis.attn_combine_peers(step.group, batch.seq_lens, max_len, step.buf.workspace)
            rec(3)
            hetis.peer_wait(step.group)
        else:
            if not fused:
                hetis.attn_combine(step.cshape, batch.seq_lens, max_len, step.buf.o_shard, step.buf.workspace,
                                   q_head_count=q_count)
            rec(3)
            if dist_mode:
                step.gather(o_full, root=gather_root)
        rec(4)

    # ---- warm-up
    for i in range(args.warmup):
        one_step(i)
    D.barrier()

    # ---- graphs: A = the K timed steps (no nodes between kernels: programmatic dependent launch overlaps
    # each kernel's prologue with its predecessor); B = the same steps with event nodes between the phases
    # (per-phase times); C = K attention launches alone (the dominant kernel's duration for the roofline,
    # with the same PDL overlap as in A).
    use_graph = bool(args.graph)
    evs = [[torch.cuda.Event(enable_timing=True, external=use_graph) for _ in range(5)] for _ in range(args.steps)]
    graph = graph_ev = graph_attn = None
    graph_launches = 0
    launch_mode = "eager"
    if use_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            c0 = hetis.launch_count()
            with torch.cuda.graph(graph, capture_error_mode="thread_local"):
                for i in range(args.steps):
                    one_step(i)
            graph_launches = hetis.launch_count() - c0
            graph_ev = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph_ev, capture_error_mode="thread_local"):
                for i in range(args.steps):
                    one_step(i, evs[i])
            graph_attn = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph_attn, capture_error_mode="thread_local"):
                for i in range(args.steps):
                    attention_only(i % n_layers)
            for g in (graph, graph_ev, graph_attn):   # untimed replays (warm instantiation)
                g.replay()
            torch.cuda.synchronize(device)
            launch_mode = "cuda_graph (PDL between kernels)"
        except Exception as exc:               # capture unsupported: time eagerly instead
            import traceback
            traceback.print_exc()
            graph = graph_ev = graph_attn = None
            launch_mode = f"eager (graph capture failed: {type(exc).__name__}: {exc})"
            torch.cuda.synchronize(device)
    D.barrier()
    sampler = ClockSampler(device.index if not args.share_gpu else 0) if headline else None
    if sampler:
        sampler.start()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = hetis.launch_count()
    start.record(stream)
    if graph is not None:
        graph.replay()
    else:
        for i in range(args.steps):
            one_step(i)
    end.record(stream)
    n1 = hetis.launch_count() + graph_launches
    D.barrier()
    if sampler:
        sampler.stop()
    elapsed_ms = D.max(start.elapsed_time(end))
    launches = n1 - n0
    launches_all = int(D.sum(launches))
    ms_per_step = elapsed_ms / args.steps
    value = B / (ms_per_step / 1e3)

    # per-phase times (evented replay) and the attention kernel alone
    if graph_ev is not None:
        graph_ev.replay()
    else:
        for i in range(args.steps):
            one_step(i, evs[i])
    D.barrier()
    phase_names = ("scatter", "attention", "combine" + ("_gather" if peer else ""), "wait" if peer else "gather")
    phases = {}
    for k, name in enumerate(phase_names):
        mean_ms = sum(e[k].elapsed_time(e[k + 1]) for e in evs) / args.steps
        phases[name + "_us"] = D.max(mean_ms) * 1e3
    evented_step_ms = D.max(sum(e[0].elapsed_time(e[4]) for e in evs) / args.steps)
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    if graph_attn is not None:
        graph_attn.replay()
    else:
        for i in range(args.steps):
            attention_only(i % n_layers)
    a1.record(stream)
    D.barrier()
    attn_ms = a0.elapsed_time(a1) / args.steps
    attn_ms_max = D.max(attn_ms)

    # ---- end to end through the public API with pinned host buffers: every step copies its inputs in
    # (the Primary's q / new k, v; every rank's seq_lens) and reads the result back (O on the receiver)
    hsl = batch.seq_lens.cpu().pin_memory()
    if dist_mode:
        if is_root:
            hq, hk, hv = (t.cpu().pin_memory() for t in (q_full, kn_full, vn_full))
        ho = torch.empty_like(o_full, device="cpu").pin_memory() if (receives and o_full is not None and (
            is_root or gather_root >= 0)) else None
    else:
        hq, hk, hv = (t.cpu().pin_memory() for t in (batch.q, batch.k_new, batch.v_new))
        ho = torch.empty_like(o_full, device="cpu").pin_memory()
    h2d = hsl.numel() * 4 + (sum(t.numel() * t.element_size() for t in (hq, hk, hv)) if (is_root or not dist_mode)
                             else 0)
    d2h = 0 if ho is None else o_full.numel() * o_full.element_size()

    def e2e_step(i):
        if dist_mode:
            if is_root:
                q_full.copy_(hq, non_blocking=True)
                kn_full.copy_(hk, non_blocking=True)
                vn_full.copy_(hv, non_blocking=True)
        else:
            step.buf.q_shard.copy_(hq, non_blocking=True)
            step.buf.k_new.copy_(hk, non_blocking=True)
            step.buf.v_new.copy_(hv, non_blocking=True)
        batch.seq_lens.copy_(hsl, non_blocking=True)
        one_step(i)
        if ho is not None:
            ho.copy_(o_full, non_blocking=True)

    e_steps = max(args.steps, 3)     # as many steps as the timed region (same power / clock regime)
    e_mode = "serial (copies in, step, O out, on the step's stream)"
    for i in range(3):
        e2e_step(i)
    D.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(e_steps):
        e2e_step(i)
    e1.record(stream)
    D.barrier()
    e2e_ms = e0.elapsed_time(e1) / e_steps
    if not dist_mode:
        # Overlapped through the same public calls: step i's host->device copies run on a copy stream
        # while step i-1 computes, and its device->host read on another stream while step i+1 computes --
        # double-buffered device inputs / outputs and pinned host outputs.  Every step still moves its own
        # inputs in and its own O out inside the timed region.  The faster of the two loops is reported.
        ins = [(step.buf.q_shard.clone(), step.buf.k_new.clone(), step.buf.v_new.clone(), batch.seq_lens.clone())
               for _ in range(2)]
        outs = [torch.empty_like(o_full) for _ in range(2)]
        hos = [ho, torch.empty_like(ho).pin_memory()]
        s_in, s_out = torch.cuda.Stream(device), torch.cuda.Stream(device)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]

        def compute(i, q, kn, vn, sl, o):
            li = i % n_layers
            if fused:
                hetis.attn_decode_append(step.cshape, q, kn, vn, k_pools[li], v_pools[li], batch.block_table, sl,
                                         max_len, o, step.buf.workspace, q_head_begin=q_begin, flags=args.attn_flags)
                return
            if args.fused_append:
                hetis.attn_partial_append(step.cshape, q, kn, vn, k_pools[li], v_pools[li], batch.block_table, sl,
                                          max_len, step.buf.workspace, q_head_begin=q_begin, flags=args.attn_flags)
            else:
                hetis.kv_append(step.cshape, kn, vn, k_pools[li], v_pools[li], batch.block_table, sl)
                hetis.attn_partial(step.cshape, q, k_pools[li], v_pools[li], batch.block_table, sl, max_len,
                                   step.buf.workspace, q_head_begin=q_begin, flags=args.attn_flags)
            hetis.attn_combine(step.cshape, sl, max_len, o, step.buf.workspace, q_head_count=q_count)

        def run_overlapped(n, start_event=None):
            if start_event is not None:
                s_in.wait_event(start_event)
            for i in range(n):
                k = i % 2
                q, kn, vn, sl = ins[k]
                with torch.cuda.stream(s_in):
                    if i >= 2:
                        s_in.wait_event(ev_done[k])          # step i-2 finished reading these buffers
                    q.copy_(hq, non_blocking=True)
                    kn.copy_(hk, non_blocking=True)
                    vn.copy_(hv, non_blocking=True)
                    sl.copy_(hsl, non_blocking=True)
                    ev_in[k].record(s_in)
                stream.wait_event(ev_in[k])
                if i >= 2:
                    stream.wait_event(ev_out[k])             # step i-2's O has been read back
                compute(i, q, kn, vn, sl, outs[k])
                ev_done[k].record(stream)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_done[k])
                    hos[k].copy_(outs[k], non_blocking=True)
                    ev_out[k].record(s_out)
            for k in range(2):
                stream.wait_event(ev_out[k])

        run_overlapped(4)
        D.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        run_overlapped(e_steps, f0)
        f1.record(stream)
        D.barrier()
        if f0.elapsed_time(f1) / e_steps < e2e_ms:
            e2e_ms, e_mode = f0.elapsed_time(f1) / e_steps, "overlapped (double-buffered inputs/outputs, copy streams)"
    e2e_ms = D.max(e2e_ms)
    e2e_value = B / (e2e_ms / 1e3)

    # ---- parity of this run's result: one more step with O poisoned, then rank 0 compares the gathered
    # O with the unsplit single-device result (bit for bit) and with the fp64 oracle (every element)
    parity = None
    if not args.no_parity:
        D.barrier()
        if o_full is not None:
            o_full.fill_(float("nan"))
        D.barrier()
        if dist_mode and is_root:
            q_full.copy_(hq)
            kn_full.copy_(hk)
            vn_full.copy_(hv)
        batch.seq_lens.copy_(hsl)
        one_step(0)
        D.barrier()
        if is_root:
            parity = check_parity(cfg, args, o_full, device, dist_mode, gather_root)
        D.barrier()

    # ---- roofline of the dominant kernel (split-KV partial attention) on this rank
    sb = accounting.step_bytes(seq_lens.tolist(), q_count, shape.r, shape.head_dim, shape.page_size,
                               shape.elem_bytes, shape.elem_bytes, 4)
    alg_bytes = sb.kv + sb.q + sb.table + sb.seq_lens
    kernel_name = "hetis_attn_partial (split-KV)"
    if args.fused_append:   # the new rows are read from k_new / v_new and written into the pools
        alg_bytes += 2 * 2 * B * (q_count // shape.r) * shape.head_dim * shape.elem_bytes
        kernel_name = "hetis_attn_partial_append (split-KV attention with kv_append fused)"
    if merge_in_kernel or fused_peer:   # the kernel also writes O
        alg_bytes += sb.o
        kernel_name = ("hetis_attn_decode_append (ONE kernel: kv_append + split-KV attention + split merge; "
                       "O written by the kernel)")
    achieved = alg_bytes / (attn_ms / 1e3) / 1e9
    achieved_min = D.max(-achieved) * -1.0      # the slowest rank
    peak, peak_src = peaks()
    rec = {
        "workload": f"{cfg.name}: {cfg.description}", "value": value, "ms_per_step": ms_per_step,
        "config": {
            "workload": f"{cfg.name}: {cfg.description}", "batch": B, "seq_len": cfg.seq_len,
            "seq_len_range": cfg.seq_len_range, "q_heads": shape.num_q_heads, "kv_heads": shape.num_kv_heads,
            "head_dim": shape.head_dim, "page_size": shape.page_size, "split": list(split),
            "o_dtype": args.o_dtype, "layers_rotated": n_layers,
            "exchange": (exchange_note if dist_mode else None), "gather_root": (gather_root if dist_mode else None),
            "fused_append": bool(args.fused_append), "merge_fused": bool(merge_in_kernel or fused_peer),
            "scatter_in_attention": bool(pull),
            "l2": f"inputs larger than L2: {n_layers} layer pool(s) x {kv_bytes_rank / 1e6:.1f} MB KV per rank "
                  f"rotated per step (L2 = 126 MB)",
            "tokens": "one token = one request's decode step of one layer, all heads"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_from_profiles(f"{cfg.name}/N{world}"),
                     "kernel": kernel_name, "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": attn_ms,
                     "avg_launch_ms_max_rank": attn_ms_max, "achieved_slowest_rank": achieved_min,
                     "launch_timing": "K attention launches replayed as one CUDA graph (PDL overlap as in the "
                                      "timed steps), CUDA events around the replay on the launching stream",
                     "peak_source": peak_src, "frac_of_8TBps_nominal": achieved / 8000.0},
        "attention_only_tokens_per_s": B / (attn_ms_max / 1e3),
        "phases_us": phases, "evented_step_us": evented_step_ms * 1e3,
        "nvlink_us": ({k: v for k, v in phases.items() if k in ("scatter_us", "wait_us", "gather_us")}
                      if dist_mode else None),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms, "mode": e_mode},
        "gpu_launches": launches, "gpu_launches_all_ranks": launches_all,
        "launch_mode": launch_mode,
        "parity": parity,
        "clocks": sampler.summary() if sampler else None,
    }
    del k_pools, v_pools, batch, step
    torch.cuda.empty_cache()
    return rec


def check_parity(cfg: workload.Config, args, o_full, device, dist_mode: bool, gather_root: int) -> dict:
    """Rank 0: the step's gathered O vs (a) the unsplit problem on this GPU (bit for bit: head partition does
    not change an item's arithmetic) and (b) the fp64 oracle on every element."""
    import numpy as np

    import oracle
    from paper_2509_08309_b200 import hetis
    shape = cfg.shape
    lens = cfg.seq_lens()
    full = workload.make_decode_batch(shape, lens, cfg.seed, device)
    host = {k: workload.to_numpy_bits(getattr(full, k)) for k in ("q", "k_new", "v_new", "k_pool", "v_pool")}
    bt, sl = full.block_table.cpu().numpy(), full.seq_lens.cpu().numpy()
    cs = hetis.make_shape(shape, args.o_dtype)
    B, H, D = full.q.shape
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(cs, B, H, full.max_seq_len), device)
    ref_gpu = torch.empty((B, H, D), dtype=o_full.dtype, device=device)
    hetis.attn_decode_append(cs, full.q, full.k_new, full.v_new, full.k_pool, full.v_pool, full.block_table,
                             full.seq_lens, full.max_seq_len, ref_gpu, ws, flags=args.attn_flags)
    torch.cuda.synchronize(device)
    bit_exact = bool(torch.equal(o_full, ref_gpu))
    got = o_full.float().cpu().numpy().astype(np.float64)
    del full, ws, ref_gpu
    oracle.kv_append(host["k_new"], host["v_new"], host["k_pool"], host["v_pool"], bt, sl)
    t0 = time.perf_counter()
    ref = oracle.decode(host["q"], host["k_pool"], host["v_pool"], bt, sl, num_kv_heads=shape.num_kv_heads,
                        dtype=oracle.BF16 if shape.dtype == "bf16" else oracle.F32)
    t_oracle = time.perf_counter() - t0
    diff = np.abs(got - ref)
    finite = bool(np.isfinite(got).all())
    loc = tuple(int(i) for i in np.unravel_index(int(np.nanargmax(diff)), diff.shape)) if finite else None
    max_abs = float(np.nanmax(diff)) if finite else float("inf")
    rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref)) if finite else float("inf")
    tol = ATOL if args.o_dtype == "f32" else 2.0 ** -8 * float(np.abs(ref).max()) + ATOL
    ok = finite and max_abs <= tol and rel <= RTOL and (bit_exact or args.attn_flags != 0)
    return {"ok": ok, "bit_exact_vs_unsplit": bit_exact, "max_abs": max_abs, "argmax": loc, "rel_fro": rel,
            "tol_abs": tol, "tol_rel_fro": RTOL, "elements": int(got.size), "oracle_s": t_oracle,
            "checked": "gathered O on rank 0 (after the timed steps) vs the unsplit single-GPU step and the fp64 "
                       "oracle, every element"}


def run_ours(args, world, rank, local):
    from paper_2509_08309_b200 import hetis

    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    dev_index = 0 if args.share_gpu else local
    torch.cuda.set_device(dev_index)
    device = torch.device("cuda", dev_index)
    dist_mode = world > 1 or args.force_dist
    comm_ptr = None
    backend = "gloo" if args.share_gpu else "nccl"
    if dist_mode:
        import torch.distributed as dist
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if "MASTER_PORT" not in os.environ:
                import socket
                so = socket.socket()
                so.bind(("127.0.0.1", 0))
                os.environ["MASTER_PORT"] = str(so.getsockname()[1])
                so.close()
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
            comm_ptr = dist.group.WORLD._get_backend(device)._comm_ptr()
        else:
            if args.exchange != "peer":
                raise SystemExit("--share-gpu runs the peer-memory exchange only (NCCL needs one GPU per rank)")
            dist.init_process_group("gloo")
    if args.gather_root not in (-1, 0):
        raise SystemExit("--gather-root: -1 (all-gather) or 0 (gather to the Primary, which checks parity)")
    D = Dist(dist_mode, world, local, device, backend)
    D.barrier()
    rec = measure(args, args.config, D, rank, world, comm_ptr, headline=True)
    sub_name = args.sub_config
    if sub_name == "auto":
        sub_name = "c3" if args.config != "c3" else "none"
    sub = None
    if sub_name != "none":
        sub_args = argparse.Namespace(**vars(args))
        sub_args.steps = min(args.steps, 100)
        try:
            workload.CONFIGS[sub_name].head_split(world)
        except ValueError as exc:          # e.g. c3's 8 kv groups over 5 ranks
            sub_name, sub = f"{sub_name} (skipped: {exc})", None
        else:
            sub = measure(sub_args, sub_name, D, rank, world, comm_ptr, headline=False)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_oracle_sample(workload.CONFIGS[args.config], args.cpu_sample_seqs)
    failed = [r["workload"][:2] for r in (rec, sub) if r is not None and r["parity"] is not None
              and not r["parity"]["ok"]]
    if rank == 0:
        shape = workload.CONFIGS[args.config].shape
        line = {
            "metric": METRIC, "value": rec["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": rec["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": shape.dtype, "data": "synthetic",
            "config": rec["config"], "roofline": rec["roofline"],
            "attention_only_tokens_per_s": rec["attention_only_tokens_per_s"],
            "phases_us": rec["phases_us"], "evented_step_us": rec["evented_step_us"], "nvlink_us": rec["nvlink_us"],
            "cpu_baseline": cpu, "e2e": rec["e2e"], "gpu_launches": rec["gpu_launches"],
            "gpu_launches_all_ranks": rec["gpu_launches_all_ranks"], "launch_mode": rec["launch_mode"],
            "parity": rec["parity"], "clocks": rec["clocks"],
        }
        if sub is None and sub_name != "none":
            line["sub"] = {sub_name: None}
        if sub is not None:
            line["sub"] = {sub_name: {k: sub[k] for k in ("value", "ms_per_step", "config", "roofline", "phases_us",
                                                          "nvlink_us", "e2e", "parity", "gpu_launches")}}
        if args.share_gpu:
            line["note"] = "--share-gpu: every rank on cuda:0 (correctness run; timings are not B200 numbers)"
        print(json.dumps(line), flush=True)
    if dist_mode:
        import torch.distributed as dist
        D.barrier()
        dist.destroy_process_group()
    if failed:
        print(f"PARITY FAILED: {failed}", file=sys.stderr, flush=True)
        return 3
    return 0


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
