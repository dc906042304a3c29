#!/usr/bin/env python
"""Timeline of the per-warp GQA kernel phases (needs a -DHETIS_TRACE build).

    HETIS_LIB=/tmp/libhetis_trace.so HETIS_NVCC_FLAGS=-DHETIS_TRACE python -m paper_2509_08309_b200.build
    HETIS_LIB=/tmp/libhetis_trace.so python scripts/trace_kernel.py [--heads 8] [--batch 128] [--len 2048]

Per CTA (%globaltimer, ns): 0 entry, 1 split offsets built, 2 producer past
griddepcontrol.wait, 3 first page issued, 4 first page landed at consumer 0,
5 last consumer warp done.  Prints min / median / max over CTAs relative to the
earliest entry.
"""
from __future__ import annotations

import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_08309_b200 import hetis, workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--len", type=int, default=2048)
    ap.add_argument("--flags", type=int, default=0)
    a = ap.parse_args()
    shape = workload.LLAMA2_70B
    lens = torch.full((a.batch,), a.len, dtype=torch.int32)
    b = workload.make_decode_batch(shape, lens, 3, "cuda", q_begin=0, q_count=a.heads)
    s = hetis.make_shape(shape)
    ws = hetis.alloc_workspace(hetis.attn_decode_workspace(s, a.batch, a.heads, a.len), "cuda")
    L = hetis.lib()
    L.hetis_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    buf = np.zeros((1024, 8), dtype=np.uint64)
    for rep in range(4):
        L.hetis_trace_read(buf.ctypes.data, buf.nbytes, 1)          # clear
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        hetis.attn_partial(s, b.q, b.k_pool, b.v_pool, b.block_table, b.seq_lens, a.len, ws, flags=a.flags)
        ev1.record()
        torch.cuda.synchronize()
    L.hetis_trace_read(buf.ctypes.data, buf.nbytes, 0)
    n = torch.cuda.get_device_properties(0).multi_processor_count
    t = buf[:n].astype(np.int64)
    t0 = t[:, 0].min()
    names = ["entry", "offsets built", "producer past wait", "first page issued", "first page landed",
             "last consumer done"]
    kv = a.batch * a.len * (a.heads // 8) * 128 * 4
    print(f"batch {a.batch} x len {a.len}, {a.heads} heads: KV {kv / 1e6:.1f} MB, event time "
          f"{ev0.elapsed_time(ev1) * 1e3:.1f} us, floor at 6.5 TB/s {kv / 6.5e12 * 1e6:.1f} us")
    for k, name in enumerate(names):
        v = (t[:, k] - t0) / 1e3
        print(f"  {name:22s} min {v.min():8.2f} us  median {np.median(v):8.2f} us  max {v.max():8.2f} us")
    done = (t[:, 5] - t0) / 1e3
    smid, items = buf[:n, 6].astype(np.int64), buf[:n, 7].astype(np.int64)
    print("  finish deciles (us):", " ".join(f"{x:.1f}" for x in np.percentile(done, np.arange(0, 101, 10))))
    print(f"  items per CTA: min {items.min()} median {int(np.median(items))} max {items.max()} total {items.sum()}")
    rate = items / np.maximum(done - (t[:, 4] - t0) / 1e3, 1e-3)     # items per us after the first page
    order = np.argsort(done)
    print("  slowest CTAs (smid, items, done us):", [(int(smid[i]), int(items[i]), round(float(done[i]), 1))
                                                    for i in order[-8:]])
    print("  fastest CTAs (smid, items, done us):", [(int(smid[i]), int(items[i]), round(float(done[i]), 1))
                                                    for i in order[:8]])
    # per-SM throughput by SM id bands (two dies: 0..73 / 74..147 if numbered that way)
    for lo in range(0, n, 37):
        m = (smid >= lo) & (smid < lo + 37)
        if m.any():
            print(f"  smid {lo:3d}-{lo + 36:3d}: items/us median {np.median(rate[m]):.3f}, done median "
                  f"{np.median(done[m]):.1f} us")


if __name__ == "__main__":
    main()

