#!/usr/bin/env python
"""Benchmark of the Hetis head-partitioned paged decode-attention hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One step = one layer's decode step for the whole batch on every rank:
    [N > 1] hetis_scatter_q (NCCL)  -> hetis_kv_append -> hetis_attn_partial
    -> hetis_attn_combine -> [N > 1] hetis_gather (NCCL all-gather of O)
Metric (BASELINE.json): decode attention tokens/s (= batch / step time, one
layer, all heads) and achieved HBM GB/s of the dominant kernel (% of the
measured copy peak).  Default workload: config c2 (LLaMA2-13B, 40 heads x 128,
batch 64, context 4096, bf16 paged KV) -- BASELINE.json configs[1]; at N > 1 the
40 heads are partitioned over the ranks (strong scaling, same total problem).

Rank 0 prints ONE JSON line.  `--impl reference` times the fp64 CPU oracle
(oracle/, the only reference this tier has) on the same workload shape.
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2", choices=sorted(workload.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-seqs", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--o-dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--attn-flags", type=int, default=0, help="HETIS_ATTN_* flags (diagnostics)")
    ap.add_argument("--graph", type=int, default=1, help="N = 1: replay the K timed steps as one CUDA graph")
    ap.add_argument("--gather", default="nccl", choices=["nccl", "peer"],
                    help="N > 1: NCCL all-gather of O (default) or the combine kernel's peer-memory stores")
    ap.add_argument("--fused-append", type=int, default=1,
                    help="1: kv_append fused into the attention kernel (hetis_attn_partial_append); 0: separate")
    ap.add_argument("--force-dist", action="store_true",
                    help="debug: run the N > 1 code path (NCCL process group, scatter, gather) at N = 1")
    ap.add_argument("--graph-dist", type=int, default=1,
                    help="N > 1: replay the timed steps as a CUDA graph too (NCCL calls captured; not with the "
                         "peer-memory exchanges, whose epochs change every step)")
    ap.add_argument("--scatter", default="nccl", choices=["nccl", "peer"],
                    help="N > 1: 'peer' = every rank pulls its q / new k, v shard from the root's buffers over "
                         "NVLink (hetis_peer_signal + hetis_scatter_pull) instead of NCCL send/recv")
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


def traffic_from_profiles(workload_name: str):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        v = d.get(workload_name)
        return None if v is None else float(v)
    except Exception:
        return None


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
def cpu_oracle_sample(cfg: workload.Config, split, rank: int, n_seqs: int):
    """Time the fp64 oracle (as it stands) on a CPU-generated batch of the workload's first n_seqs requests,
    all of this rank's heads, at the workload's lengths.  Returns (tokens/s, seconds, cores, sample text)."""
    import oracle
    lens = cfg.seq_lens()[:n_seqs]
    begin = sum(split[:rank])
    b = workload.make_decode_batch(cfg.shape, lens, cfg.seed, "cpu", q_begin=begin, q_count=split[rank],
                                   rank_salt=rank)
    h = {k: workload.to_numpy_bits(getattr(b, k)).copy() for k in ("q", "k_new", "v_new", "k_pool", "v_pool")}
    bt = b.block_table.numpy()
    sl = b.seq_lens.numpy()
    cores = len(os.sched_getaffinity(0))
    dt = oracle.BF16 if cfg.shape.dtype == "bf16" else oracle.F32
    t0 = time.perf_counter()
    oracle.kv_append(h["k_new"], h["v_new"], h["k_pool"], h["v_pool"], bt, sl)
    oracle.decode(h["q"], h["k_pool"], h["v_pool"], bt, sl, num_kv_heads=b.kv_count, dtype=dt, nthreads=cores)
    sec = time.perf_counter() - t0
    sample = (f"{n_seqs} of {cfg.batch} requests x {split[rank]} heads at the workload's lengths "
              f"(sum L = {int(lens.sum())}), kv_append + fp64 oracle decode, {cores} threads")
    return n_seqs / sec, sec, cores, sample


def run_reference(args, world, rank, budget_s: float = 150.0):
    """The oracle as it stands, on this box's host cores.  The sample (requests
    per step) is sized so that warm-up + K steps take about `budget_s`."""
    import oracle
    cfg = workload.CONFIGS[args.config]
    if rank != 0:
        return 0
    split = cfg.head_split(1)
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
    sample = (f"{n} of {cfg.batch} requests x {split[0]} heads at the workload's lengths "
              f"(sum L = {int(sl[:n].sum())}), fp64 oracle decode, {cores} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.description}", "batch_sampled": n, "batch": cfg.batch},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample + " per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm
def run_ours(args, world, rank, local):
    from paper_2509_08309_b200 import hetis
    from paper_2509_08309_b200.step import DecodeStep

    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    cfg = workload.CONFIGS[args.config]
    shape = cfg.shape
    split = cfg.head_split(world)
    comm_ptr = None
    pg = None
    dist_mode = world > 1 or args.force_dist
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
        dist.init_process_group("nccl", device_id=device)
        pg = dist.group.WORLD
        dist.barrier()
        comm_ptr = pg._get_backend(device)._comm_ptr()
    B = cfg.batch
    seq_lens = cfg.seq_lens()
    max_len = int(seq_lens.max())
    cs = hetis.make_shape(shape, args.o_dtype)
    plan = hetis.plan_create(cs, world, split)
    q_begin, q_count = plan.heads(rank)
    batch = workload.make_decode_batch(shape, seq_lens, cfg.seed, device, q_begin=q_begin, q_count=q_count,
                                       rank_salt=rank)
    step = DecodeStep(shape, plan, rank, B, max_len, device, o_dtype=args.o_dtype, comm_ptr=comm_ptr)
    kv_bytes_rank = accounting.step_bytes(seq_lens.tolist(), q_count, shape.r, shape.head_dim, shape.page_size,
                                          shape.elem_bytes, shape.elem_bytes, 4).kv
    # rotate layer pools so the per-step KV stream never sits in L2
    n_layers = max(1, math.ceil(4 * L2_BYTES / max(kv_bytes_rank, 1)))
    free = torch.cuda.mem_get_info(device)[0]
    pool_bytes = 2 * batch.k_pool.numel() * batch.k_pool.element_size()
    n_layers = max(1, min(n_layers, int(0.6 * free // max(pool_bytes, 1)) + 1))
    k_pools = [batch.k_pool] + [batch.k_pool.clone() for _ in range(n_layers - 1)]
    v_pools = [batch.v_pool] + [batch.v_pool.clone() for _ in range(n_layers - 1)]
    odt = torch.bfloat16 if args.o_dtype == "bf16" else torch.float32
    is_root = rank == 0
    if dist_mode:
        gq = torch.Generator(device=device).manual_seed(cfg.seed + 17)
        q_full = workload.make_q(shape, B, cfg.seed, device) if is_root else None
        kn_full = (torch.randn((B, shape.num_kv_heads, shape.head_dim), generator=gq, device=device)
                   .to(shape.torch_dtype) if is_root else None)
        vn_full = (torch.randn((B, shape.num_kv_heads, shape.head_dim), generator=gq, device=device)
                   .to(shape.torch_dtype) if is_root else None)
        o_full = torch.empty((B, shape.num_q_heads, shape.head_dim), dtype=odt, device=device)
        if args.gather == "peer" or args.scatter == "peer":
            step.setup_peers(o_full, q_full, kn_full, vn_full)
    else:
        step.buf.q_shard.copy_(batch.q)
        step.buf.k_new.copy_(batch.k_new)
        step.buf.v_new.copy_(batch.v_new)
        o_full = step.buf.o_shard
    stream = torch.cuda.current_stream(device)

    def one_step(i, ev_a=None, ev_b=None):
        li = i % n_layers
        if dist_mode and (args.gather == "peer" or args.scatter == "peer"):
            step.epoch += 1
        if dist_mode and args.scatter == "peer":
            step.scatter_peers(step.epoch)
        elif dist_mode:
            step.scatter(q_full, kn_full, vn_full)
        if not args.fused_append:
            step.append(k_pools[li], v_pools[li], batch.block_table, batch.seq_lens)
        if ev_a is not None:
            ev_a.record(torch.cuda.current_stream(device))
        if args.fused_append:   # the append happens inside the attention kernel
            hetis.attn_partial_append(step.cshape, step.buf.q_shard, step.buf.k_new, step.buf.v_new, k_pools[li],
                                      v_pools[li], batch.block_table, batch.seq_lens, max_len, step.buf.workspace,
                                      q_head_begin=q_begin, flags=args.attn_flags)
        else:
            hetis.attn_partial(step.cshape, step.buf.q_shard, k_pools[li], v_pools[li], batch.block_table,
                               batch.seq_lens, max_len, step.buf.workspace, q_head_begin=q_begin,
                               flags=args.attn_flags)
        if ev_b is not None:
            ev_b.record(torch.cuda.current_stream(device))
        if dist_mode and args.gather == "peer":
            # one kernel merges the splits and stores O into every rank's o_full over NVLink
            hetis.attn_combine_peers(step.cshape, batch.seq_lens, max_len, step.o_peers, step.sig_peers, rank,
                                     step.epoch, step.buf.workspace, q_head_begin=q_begin, q_head_count=q_count)
            hetis.peer_wait(step.sig, step.epoch)
            return
        hetis.attn_combine(step.cshape, batch.seq_lens, max_len, step.buf.o_shard, step.buf.workspace,
                           q_head_count=q_count)
        if dist_mode:
            step.gather(o_full, root=-1)

    def barrier():
        if dist_mode:
            import torch.distributed as dist
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(device)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up
    for i in range(args.warmup):
        one_step(i)
    barrier()

    # ---- timed: K steps, CUDA events on the launching stream.  At N = 1 the K steps
    # are captured once into a CUDA graph (the same kernels, no host launch gaps) and
    # the graph is replayed once inside the timed region; per-step events are graph nodes.
    sampler = ClockSampler(local)
    # external=True: inside a capture the records become event-record graph nodes
    # N > 1: only the NCCL exchanges can be captured -- the peer-memory ones carry a per-step epoch
    use_graph = bool(args.graph) and (not dist_mode or (bool(args.graph_dist) and args.gather == "nccl"
                                                         and args.scatter == "nccl"))
    evs_a = [torch.cuda.Event(enable_timing=True, external=use_graph) for _ in range(args.steps)]
    evs_b = [torch.cuda.Event(enable_timing=True, external=use_graph) for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launch_mode = "eager"
    # At N = 1 the K timed steps are captured as CUDA graphs: graph A (the headline
    # number) has no nodes between the kernels, so programmatic dependent launch
    # overlaps each kernel's prologue with its predecessor; graph B is the same K
    # steps with event nodes around every attention kernel (per-launch durations
    # for the roofline), replayed in a second timed region.
    graph = graph_ev = None
    graph_launches = 0
    if use_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            c0 = hetis.launch_count()
            with torch.cuda.graph(graph):
                for i in range(args.steps):
                    one_step(i)
            graph_launches = hetis.launch_count() - c0
            graph_ev = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph_ev):
                for i in range(args.steps):
                    one_step(i, evs_a[i], evs_b[i])
            graph.replay()                      # untimed replays (warm instantiation)
            graph_ev.replay()
            torch.cuda.synchronize(device)
            launch_mode = "cuda_graph (PDL between kernels); roofline from a second replay with event nodes"
        except Exception as exc:               # capture unsupported: time eagerly instead
            graph = graph_ev = None
            launch_mode = f"eager (graph capture failed: {type(exc).__name__})"
    barrier()
    sampler.start()
    n0 = hetis.launch_count()
    start.record(stream)
    if graph is not None:
        graph.replay()
    else:
        for i in range(args.steps):
            one_step(i, evs_a[i], evs_b[i])
    end.record(stream)
    n1 = hetis.launch_count() + graph_launches
    barrier()
    if graph_ev is not None:
        graph_ev.replay()
        barrier()
    sampler.stop()
    elapsed_ms = max_over_ranks(start.elapsed_time(end))
    attn_ms = sum(a.elapsed_time(b) for a, b in zip(evs_a, evs_b)) / args.steps
    attn_ms_max = max_over_ranks(attn_ms)
    launches = n1 - n0
    ms_per_step = elapsed_ms / args.steps
    value = B / (ms_per_step / 1e3)

    # ---- end to end through the public API with pinned host buffers
    h2d = d2h = 0
    if dist_mode:
        if is_root:
            hq = q_full.cpu().pin_memory()
            hk = kn_full.cpu().pin_memory()
            hv = vn_full.cpu().pin_memory()
            h2d = sum(t.numel() * t.element_size() for t in (hq, hk, hv))
        ho = torch.empty_like(o_full, device="cpu").pin_memory() if is_root else None
        d2h = o_full.numel() * o_full.element_size() if is_root else 0
    else:
        hq = batch.q.cpu().pin_memory()
        hk = batch.k_new.cpu().pin_memory()
        hv = batch.v_new.cpu().pin_memory()
        ho = torch.empty_like(o_full, device="cpu").pin_memory()
        h2d = sum(t.numel() * t.element_size() for t in (hq, hk, hv))
        d2h = o_full.numel() * o_full.element_size()
    hsl = batch.seq_lens.cpu().pin_memory()
    h2d += hsl.numel() * 4

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

    e_steps = max(min(args.steps, 50), 3)
    e_mode = "serial"
    if not dist_mode:
        # Overlapped through the same public calls: step i's host->device copies run on a copy stream
        # while step i-1 computes, and its device->host read on another stream while step i+1
        # computes -- double-buffered device inputs / outputs and pinned host outputs.  Every step
        # still moves its own inputs in and its own O out inside the timed region.
        e_mode = "overlapped (double-buffered inputs/outputs, copy streams)"
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
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_overlapped(e_steps, e0)
        e1.record(stream)
        barrier()
        # tiny steps (c1) are host-bound: the extra stream/event calls cost more than the overlap
        # saves, so the plain serial loop is timed too and the faster of the two is reported
        for i in range(3):
            e2e_step(i)
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for i in range(e_steps):
            e2e_step(i)
        f1.record(stream)
        barrier()
        if f0.elapsed_time(f1) < e0.elapsed_time(e1):
            e0, e1, e_mode = f0, f1, "serial (faster than the overlapped loop for this step size)"
    else:
        for i in range(3):
            e2e_step(i)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(e_steps):
            e2e_step(i)
        e1.record(stream)
        barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / e_steps
    e2e_value = B / (e2e_ms / 1e3)

    # ---- roofline of the dominant kernel (split-KV partial attention) on this rank
    sb = accounting.step_bytes(seq_lens.tolist(), q_count, shape.r, shape.head_dim, shape.page_size,
                               shape.elem_bytes, shape.elem_bytes, 4)
    alg_bytes = sb.kv + sb.q + sb.table + sb.seq_lens
    kernel_name = "hetis_attn_partial (split-KV)"
    if args.fused_append:   # the new rows are read from k_new / v_new and written into the pools
        alg_bytes += 2 * 2 * B * (q_count // shape.r) * shape.head_dim * shape.elem_bytes
        kernel_name = "hetis_attn_partial_append (split-KV attention with kv_append fused)"
    achieved = alg_bytes / (attn_ms / 1e3) / 1e9
    peak, peak_src = peaks()
    clocks = sampler.summary()
    traffic = traffic_from_profiles(f"{cfg.name}/N{world}")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tps, sec, cores, sample = cpu_oracle_sample(cfg, split, rank, min(args.cpu_sample_seqs, B))
        cpu = {"value": tps, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": shape.dtype, "data": "synthetic",
            "config": {
                "workload": f"{cfg.name}: {cfg.description}", "batch": B, "seq_len": cfg.seq_len,
                "seq_len_range": cfg.seq_len_range, "q_heads": shape.num_q_heads, "kv_heads": shape.num_kv_heads,
                "head_dim": shape.head_dim, "page_size": shape.page_size, "split": list(split),
                "o_dtype": args.o_dtype, "layers_rotated": n_layers,
                "gather": (args.gather if dist_mode else None),
                "scatter": (args.scatter if dist_mode else None),
                "fused_append": bool(args.fused_append),
                "l2": f"inputs larger than L2: {n_layers} layer pool(s) x {kv_bytes_rank / 1e6:.1f} MB KV per rank "
                      f"rotated per step (L2 = 126 MB)",
                "tokens": "one token = one request's decode step of one layer, all heads"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": kernel_name,
                         "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": attn_ms,
                         "avg_launch_ms_max_rank": attn_ms_max, "peak_source": peak_src,
                         "frac_of_8TBps_nominal": achieved / 8000.0},
            "attention_only_tokens_per_s": B / (attn_ms_max / 1e3),
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms, "mode": e_mode},
            "gpu_launches": launches,
            "launch_mode": launch_mode,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if dist_mode:
        import torch.distributed as dist
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
