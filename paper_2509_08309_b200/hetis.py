"""Thin Python binding of libhetis.so (include/hetis.h), same names as the C ABI.

Argument marshalling only: torch tensors -> raw pointers, sizes and the current
CUDA stream.  Every step of the decode path runs in the library's kernels; if
the library is missing this module raises at import-time use -- there is no
CPU or eager fallback.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import workload

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HETIS_LIB") or os.path.join(_PKG, "libhetis.so")

HETIS_OK = 0
STATUS = {0: "HETIS_OK", 1: "HETIS_E_INVALID", 2: "HETIS_E_HEAD_INTEGRITY", 3: "HETIS_E_GROUP_ALIGN",
          4: "HETIS_E_CAPACITY", 5: "HETIS_E_UNSUPPORTED", 6: "HETIS_E_WORKSPACE", 7: "HETIS_E_CUDA",
          8: "HETIS_E_NCCL"}
F32, BF16 = 0, 1
ATTN_FORCE_SIMT = 0x1
ATTN_TC_SHARED_RING = 0x2
ATTN_DEVICE_CLAIM = 0x4
ATTN_MHA_TC = 0x8
ATTN_PIPELINED = 0x10
ATTN_FUSED_MERGE = 0x20
ATTN_NO_GROUP_MODE = 0x40
ATTN_STATIC_DEAL = 0x80
ATTN_DIAG_STREAM_ONLY = 0x100

EXPORTED = ("hetis_status_str", "hetis_last_error", "hetis_abi_version", "hetis_split_tokens",
            "hetis_plan_create", "hetis_plan_destroy", "hetis_plan_heads", "hetis_plan_num_devices", "hetis_plan_units",
            "hetis_plan_check_capacity", "hetis_kv_append", "hetis_attn_decode_workspace", "hetis_attn_partial",
            "hetis_attn_combine", "hetis_attn_decode", "hetis_attn_decode_launches_for", "hetis_attn_combine_peers", "hetis_peer_wait",
            "hetis_comm_workspace", "hetis_scatter_q", "hetis_gather", "hetis_kv_migrate",
            "hetis_attn_combine_lse", "hetis_seq_split_lens", "hetis_seq_merge", "hetis_seq_broadcast_q",
            "hetis_seq_allgather_merge", "hetis_peer_state_bytes", "hetis_peer_group_create",
            "hetis_peer_group_destroy", "hetis_scatter_pull", "hetis_attn_partial_append",
            "hetis_attn_decode_append", "hetis_check_tables", "hetis_launch_count", "hetis_attn_decode_units",
            "hetis_attn_decode_launches", "hetis_attn_decode_peers", "hetis_peer_access",
            "hetis_attn_partial_pull")


class HetisError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        self.name = STATUS.get(status, f"status {status}")
        super().__init__(f"{where}: {self.name}: {detail}")


class CShape(ctypes.Structure):
    _fields_ = [("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("page_size", ctypes.c_int32), ("kv_dtype", ctypes.c_int32), ("q_dtype", ctypes.c_int32),
                ("o_dtype", ctypes.c_int32)]


_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load the in-tree libhetis.so (built by paper_2509_08309_b200.build)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2509_08309_b200.build` "
                                  "(there is no fallback path)")
            L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
            vp, i32, i64, u32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_size_t
            P = ctypes.POINTER
            sp = P(CShape)
            sig = {
                "hetis_status_str": (ctypes.c_char_p, [ctypes.c_int]),
                "hetis_last_error": (ctypes.c_char_p, []),
                "hetis_abi_version": (i32, []),
                "hetis_split_tokens": (i32, []),
                "hetis_launch_count": (ctypes.c_uint64, []),
                "hetis_plan_create": (ctypes.c_int, [sp, i32, i32, P(i32), i32, P(vp)]),
                "hetis_plan_destroy": (None, [vp]),
                "hetis_plan_heads": (ctypes.c_int, [vp, i32, i32, P(i32), P(i32)]),
                "hetis_plan_num_devices": (i32, [vp]),
                "hetis_plan_units": (ctypes.c_int, [vp, i32, P(i32), P(i32)]),
                "hetis_plan_check_capacity": (ctypes.c_int, [vp, i32, P(i32), P(i64)]),
                "hetis_kv_append": (ctypes.c_int, [sp, i32, i32, vp, vp, vp, vp, i64, vp, i32, vp, vp]),
                "hetis_attn_decode_workspace": (ctypes.c_int, [sp, i32, i32, i32, P(sz)]),
                "hetis_attn_partial": (ctypes.c_int, [sp, i32, i32, i32, vp, vp, vp, i64, vp, i32, vp, i32, vp, sz,
                                                      u32, vp]),
                "hetis_attn_combine": (ctypes.c_int, [sp, i32, i32, vp, i32, vp, i64, vp, sz, vp]),
                "hetis_attn_decode": (ctypes.c_int, [sp, i32, i32, i32, vp, vp, vp, i64, vp, i32, vp, i32, vp, vp,
                                                     sz, u32, vp]),
                "hetis_peer_state_bytes": (sz, []),
                "hetis_peer_group_create": (ctypes.c_int, [vp, i32, i32, i32, P(vp), P(vp), i64, vp, vp, vp, P(vp)]),
                "hetis_peer_group_destroy": (None, [vp]),
                "hetis_attn_combine_peers": (ctypes.c_int, [vp, i32, vp, i32, vp, sz, vp]),
                "hetis_peer_wait": (ctypes.c_int, [vp, vp]),
                "hetis_comm_workspace": (ctypes.c_int, [vp, i32, i32, P(sz)]),
                "hetis_scatter_q": (ctypes.c_int, [vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
                "hetis_gather": (ctypes.c_int, [vp, vp, i32, i32, i32, vp, vp, vp, sz, vp]),
                "hetis_kv_migrate": (ctypes.c_int, [sp, i32, vp, vp, vp, vp, i32, vp, vp, vp, i32, i32, vp]),
                "hetis_attn_combine_lse": (ctypes.c_int, [sp, i32, i32, vp, i32, vp, i64, vp, vp, sz, vp]),
                "hetis_seq_split_lens": (ctypes.c_int, [i32, i32, i32, i32, vp, vp, vp, vp]),
                "hetis_seq_merge": (ctypes.c_int, [sp, i32, i32, i32, vp, i64, vp, i64, vp, i64, vp]),
                "hetis_seq_broadcast_q": (ctypes.c_int, [sp, vp, i32, i32, i32, i32, vp, vp, vp, vp]),
                "hetis_seq_allgather_merge": (ctypes.c_int, [sp, vp, i32, i32, i32, vp, vp, vp, i64, vp]),
                "hetis_check_tables": (ctypes.c_int, [sp, i32, i32, i64, vp, i32, vp, vp, vp]),
                "hetis_attn_partial_append": (ctypes.c_int, [sp, i32, i32, i32, vp, vp, vp, vp, vp, i64, vp, i32, vp,
                                                             i32, vp, sz, u32, vp]),
                "hetis_attn_decode_append": (ctypes.c_int, [sp, i32, i32, i32, vp, vp, vp, vp, vp, i64, vp, i32, vp,
                                                            i32, vp, vp, sz, u32, vp]),
                "hetis_scatter_pull": (ctypes.c_int, [vp, i32, vp, vp, vp, vp]),
                "hetis_attn_decode_launches": (i32, [sp, u32]),
                "hetis_attn_decode_launches_for": (i32, [sp, i32, i32, i32, u32]),
                "hetis_peer_access": (ctypes.c_int, [i32]),
                "hetis_attn_partial_pull": (ctypes.c_int, [vp, i32, vp, vp, i64, vp, i32, vp, i32, vp, sz, u32, vp]),
                "hetis_attn_decode_peers": (ctypes.c_int, [vp, i32, vp, vp, vp, vp, vp, i64, vp, i32, vp, i32, vp, sz,
                                                           u32, vp]),
                "hetis_attn_decode_units": (ctypes.c_int, [sp, i32, i32, vp, vp, vp, vp, vp, vp, i64, vp, i32, vp,
                                                           i32, vp, i64, vp, sz, u32, vp]),
            }
            for name, (res, args) in sig.items():
                # an older build loaded through HETIS_LIB (A/B runs) may lack newer entry points;
                # tests/test_abi.py checks that the in-tree library exports every declared one
                f = getattr(L, name, None)
                if f is None:
                    continue
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _check(rc: int, where: str):
    if rc != HETIS_OK:
        raise HetisError(rc, where, lib().hetis_last_error().decode())


def dtype_code(dt: torch.dtype | str) -> int:
    if dt in (torch.bfloat16, "bf16"):
        return BF16
    if dt in (torch.float32, "f32"):
        return F32
    raise ValueError(f"unsupported dtype {dt}")


def make_shape(shape: workload.Shape, o_dtype: str = "f32") -> CShape:
    c = dtype_code(shape.dtype)
    return CShape(shape.num_q_heads, shape.num_kv_heads, shape.head_dim, shape.page_size, c, c, dtype_code(o_dtype))


def _dev(t: torch.Tensor | None, name: str):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the library has no host path)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


_TORCH_OF = {F32: torch.float32, BF16: torch.bfloat16}


def _check_args(shape: CShape, q=None, o=None, k_pool=None, v_pool=None, block_table=None, seq_lens=None,
                k_new=None, v_new=None, kv_heads: int | None = None) -> None:
    """Host-side dtype / shape agreement with the CShape (the C ABI takes raw pointers and cannot check it):
    a bf16 o passed with an f32 o_dtype, or a block table with the wrong number of kv heads, would make the
    kernels read or write past the buffers."""
    r = shape.num_q_heads // shape.num_kv_heads
    kvt, qt, ot = _TORCH_OF[shape.kv_dtype], _TORCH_OF[shape.q_dtype], _TORCH_OF[shape.o_dtype]
    D, P = shape.head_dim, shape.page_size
    B = None
    if q is not None:
        if q.dtype != qt or q.dim() != 3 or q.shape[2] != D or q.shape[1] % r:
            raise ValueError(f"q must be {qt} [B][x][{D}] with x a multiple of r={r}, got {q.dtype} {tuple(q.shape)}")
        B, kv_heads = q.shape[0], q.shape[1] // r
    if o is not None:
        if o.dtype != ot or o.shape[-1] != D:
            raise ValueError(f"o must be {ot} [..][{D}] (shape.o_dtype), got {o.dtype} {tuple(o.shape)}")
        if q is not None and (o.shape[0] != q.shape[0] or o.shape[1] < q.shape[1]):
            raise ValueError(f"o {tuple(o.shape)} does not cover q {tuple(q.shape)}")
    for name, pool in (("k_pool", k_pool), ("v_pool", v_pool)):
        if pool is not None and (pool.dtype != kvt or pool.dim() != 3 or pool.shape[1] != P or pool.shape[2] != D):
            raise ValueError(f"{name} must be {kvt} [pages][{P}][{D}], got {pool.dtype} {tuple(pool.shape)}")
    if k_pool is not None and v_pool is not None and k_pool.shape != v_pool.shape:
        raise ValueError("k_pool and v_pool differ in shape")
    for name, t in (("k_new", k_new), ("v_new", v_new)):
        if t is not None:
            if t.dtype != kvt or t.dim() != 3 or t.shape[2] != D:
                raise ValueError(f"{name} must be {kvt} [B][kv][{D}], got {t.dtype} {tuple(t.shape)}")
            if B is not None and (t.shape[0] != B or t.shape[1] != kv_heads):
                raise ValueError(f"{name} {tuple(t.shape)} does not match q's [B][x/r] = [{B}][{kv_heads}]")
    if block_table is not None:
        if block_table.dtype != torch.int32 or block_table.dim() != 3:
            raise ValueError("block_table must be int32 [B][kv][max_pages]")
        if B is not None and (block_table.shape[0] != B or block_table.shape[1] != kv_heads):
            raise ValueError(f"block_table {tuple(block_table.shape)} does not match [B][x/r] = [{B}][{kv_heads}]")
    if seq_lens is not None:
        if seq_lens.dtype != torch.int32 or seq_lens.dim() != 1:
            raise ValueError("seq_lens must be int32 [B]")
        if B is not None and seq_lens.shape[0] != B:
            raise ValueError(f"seq_lens has {seq_lens.shape[0]} entries for {B} requests")


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def status_str(s: int) -> str:
    return lib().hetis_status_str(s).decode()


def abi_version() -> int:
    return lib().hetis_abi_version()


def split_tokens() -> int:
    return lib().hetis_split_tokens()


def launch_count() -> int:
    return int(lib().hetis_launch_count())


# ---------------------------------------------------------------- plans
class Plan:
    """Owned hetis_plan (Eq. 5 validated head -> device assignment)."""

    def __init__(self, shape: CShape, num_devices: int, x, per_request: bool = False, num_seqs: int = 0):
        arr = (ctypes.c_int32 * len(x))(*[int(v) for v in x])
        h = ctypes.c_void_p()
        _check(lib().hetis_plan_create(ctypes.byref(shape), num_devices, num_seqs, arr, int(per_request),
                                       ctypes.byref(h)), "hetis_plan_create")
        self._h = h
        self.shape = shape
        self.num_devices = num_devices
        self.num_seqs = num_seqs

    @property
    def handle(self):
        return self._h

    def heads(self, device: int, seq: int = 0) -> tuple[int, int]:
        b, c = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().hetis_plan_heads(self._h, device, seq, ctypes.byref(b), ctypes.byref(c)), "hetis_plan_heads")
        return b.value, c.value

    def units(self, device: int) -> list[tuple[int, int]]:
        """(request, global kv head) work units of `device` for a per-request plan (hetis_plan_units)."""
        n = ctypes.c_int32()
        _check(lib().hetis_plan_units(self._h, device, None, ctypes.byref(n)), "hetis_plan_units")
        buf = (ctypes.c_int32 * max(2 * n.value, 1))()
        _check(lib().hetis_plan_units(self._h, device, buf, ctypes.byref(n)), "hetis_plan_units")
        return [(buf[2 * u], buf[2 * u + 1]) for u in range(n.value)]

    def check_capacity(self, seq_lens, free_pages) -> None:
        sl = (ctypes.c_int32 * max(len(seq_lens), 1))(*[int(v) for v in seq_lens])
        fp = (ctypes.c_int64 * len(free_pages))(*[int(v) for v in free_pages])
        _check(lib().hetis_plan_check_capacity(self._h, len(seq_lens), sl, fp), "hetis_plan_check_capacity")

    def comm_workspace(self, rank: int, num_seqs: int) -> int:
        b = ctypes.c_size_t()
        _check(lib().hetis_comm_workspace(self._h, rank, num_seqs, ctypes.byref(b)), "hetis_comm_workspace")
        return b.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.hetis_plan_destroy(h)
            self._h = None


def plan_create(shape: CShape, num_devices: int, x, per_request: bool = False, num_seqs: int = 0) -> Plan:
    return Plan(shape, num_devices, x, per_request, num_seqs)


# ---------------------------------------------------------------- kernels
def kv_append(shape: CShape, k_new, v_new, k_pool, v_pool, block_table, seq_lens, stream=None) -> None:
    B, G, _ = k_new.shape
    _check_args(shape, k_pool=k_pool, v_pool=v_pool, k_new=k_new, v_new=v_new, block_table=block_table,
                seq_lens=seq_lens)
    if block_table.shape[:2] != k_new.shape[:2] or v_new.shape != k_new.shape or seq_lens.shape[0] != B:
        raise ValueError("k_new, v_new, block_table and seq_lens disagree on [B][kv]")
    _check(lib().hetis_kv_append(ctypes.byref(shape), B, G, _dev(k_new, "k_new"), _dev(v_new, "v_new"),
                                 _dev(k_pool, "k_pool"), _dev(v_pool, "v_pool"), k_pool.shape[0],
                                 _dev(block_table, "block_table"), block_table.shape[2], _dev(seq_lens, "seq_lens"),
                                 _stream(stream)), "hetis_kv_append")


def check_tables(shape: CShape, k_pool, block_table, seq_lens, stream=None) -> int:
    """Number of device-data contract violations (hetis_check_tables); synchronises the stream."""
    out = torch.empty(1, dtype=torch.int32, device=block_table.device)
    B, G, M = block_table.shape
    _check(lib().hetis_check_tables(ctypes.byref(shape), B, G, k_pool.shape[0], _dev(block_table, "block_table"), M,
                                    _dev(seq_lens, "seq_lens"), _dev(out, "violations"), _stream(stream)),
           "hetis_check_tables")
    return int(out.item())


def kv_migrate(shape: CShape, entries, src_k_pool, src_v_pool, src_block_table, dst_k_pool, dst_v_pool,
               dst_block_table, max_ctas: int = 0, stream=None) -> None:
    """Head-granular KV migration (hetis_kv_migrate).  entries: device int32 [n][3] rows of
    (src_row, dst_row, num_tokens); the block tables are viewed as [rows][max_pages] (their last
    dimension is max_pages).  Pools may be peer mappings (CUDA IPC) of another device's pools."""
    if entries.dtype != torch.int32 or entries.dim() != 2 or entries.shape[1] != 3 or not entries.is_contiguous():
        raise ValueError("entries must be a contiguous int32 [n][3] tensor")
    _check(lib().hetis_kv_migrate(ctypes.byref(shape), entries.shape[0], _dev(entries, "entries"),
                                  _dev(src_k_pool, "src_k_pool"), _dev(src_v_pool, "src_v_pool"),
                                  _dev(src_block_table, "src_block_table"), src_block_table.shape[-1],
                                  _dev(dst_k_pool, "dst_k_pool"), _dev(dst_v_pool, "dst_v_pool"),
                                  _dev(dst_block_table, "dst_block_table"), dst_block_table.shape[-1], max_ctas,
                                  _stream(stream)), "hetis_kv_migrate")


def attn_decode_workspace(shape: CShape, num_seqs: int, q_head_count: int, max_seq_len: int) -> int:
    b = ctypes.c_size_t()
    _check(lib().hetis_attn_decode_workspace(ctypes.byref(shape), num_seqs, q_head_count, max_seq_len,
                                             ctypes.byref(b)), "hetis_attn_decode_workspace")
    return b.value


def alloc_workspace(nbytes: int, device) -> torch.Tensor:
    """A zero-filled, 256-byte aligned uint8 device buffer (torch's caching allocator aligns to
    512).  Zero-filled because the attention workspace ends in work-claim counters that must start
    at zero; every completed launch leaves them zero again."""
    return torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)


def attn_partial(shape: CShape, q, k_pool, v_pool, block_table, seq_lens, max_seq_len: int, workspace,
                 q_head_begin: int = 0, flags: int = 0, stream=None) -> None:
    B, x, _ = q.shape
    _check_args(shape, q=q, k_pool=k_pool, v_pool=v_pool, block_table=block_table, seq_lens=seq_lens)
    _check(lib().hetis_attn_partial(ctypes.byref(shape), B, q_head_begin, x, _dev(q, "q"), _dev(k_pool, "k_pool"),
                                    _dev(v_pool, "v_pool"), k_pool.shape[0], _dev(block_table, "block_table"),
                                    block_table.shape[2], _dev(seq_lens, "seq_lens"), max_seq_len,
                                    _dev(workspace, "workspace"), workspace.numel() * workspace.element_size(),
                                    flags, _stream(stream)), "hetis_attn_partial")


def attn_combine(shape: CShape, seq_lens, max_seq_len: int, o, workspace, q_head_count: int | None = None,
                 o_seq_stride: int | None = None, stream=None) -> None:
    B = seq_lens.shape[0]
    if q_head_count is None:
        q_head_count = o.shape[1]
    if o_seq_stride is None:
        o_seq_stride = o.stride(0)
    if not o.is_cuda:
        raise ValueError("o must be a CUDA tensor")
    _check_args(shape, o=o, seq_lens=seq_lens)
    _check(lib().hetis_attn_combine(ctypes.byref(shape), B, q_head_count, _dev(seq_lens, "seq_lens"), max_seq_len,
                                    ctypes.c_void_p(o.data_ptr()), o_seq_stride, _dev(workspace, "workspace"),
                                    workspace.numel() * workspace.element_size(), _stream(stream)),
           "hetis_attn_combine")


def attn_combine_lse(shape: CShape, seq_lens, max_seq_len: int, o, lse, workspace, q_head_count: int | None = None,
                     o_seq_stride: int | None = None, stream=None) -> None:
    """hetis_attn_combine that also writes lse [B][q_head_count] (natural log) -- the sequence split's input."""
    B = seq_lens.shape[0]
    if q_head_count is None:
        q_head_count = o.shape[1]
    if o_seq_stride is None:
        o_seq_stride = o.stride(0)
    if not o.is_cuda or not lse.is_cuda or lse.dtype != torch.float32:
        raise ValueError("o and lse (float32) must be CUDA tensors")
    _check_args(shape, o=o, seq_lens=seq_lens)
    _check(lib().hetis_attn_combine_lse(ctypes.byref(shape), B, q_head_count, _dev(seq_lens, "seq_lens"), max_seq_len,
                                        ctypes.c_void_p(o.data_ptr()), o_seq_stride, ctypes.c_void_p(lse.data_ptr()),
                                        _dev(workspace, "workspace"), workspace.numel() * workspace.element_size(),
                                        _stream(stream)), "hetis_attn_combine_lse")


def attn_partial_append(shape: CShape, q, k_new, v_new, k_pool, v_pool, block_table, seq_lens, max_seq_len: int,
                        workspace, q_head_begin: int = 0, flags: int = 0, stream=None) -> None:
    """kv_append fused into the split-KV attention kernel (hetis_attn_partial_append)."""
    B, x, _ = q.shape
    _check_args(shape, q=q, k_pool=k_pool, v_pool=v_pool, block_table=block_table, seq_lens=seq_lens, k_new=k_new,
                v_new=v_new)
    _check(lib().hetis_attn_partial_append(ctypes.byref(shape), B, q_head_begin, x, _dev(q, "q"), _dev(k_new, "k_new"),
                                           _dev(v_new, "v_new"), _dev(k_pool, "k_pool"), _dev(v_pool, "v_pool"),
                                           k_pool.shape[0], _dev(block_table, "block_table"), block_table.shape[2],
                                           _dev(seq_lens, "seq_lens"), max_seq_len, _dev(workspace, "workspace"),
                                           workspace.numel() * workspace.element_size(), flags, _stream(stream)),
           "hetis_attn_partial_append")


def attn_decode_append(shape: CShape, q, k_new, v_new, k_pool, v_pool, block_table, seq_lens, max_seq_len: int, o,
                       workspace, q_head_begin: int = 0, flags: int = 0, stream=None) -> None:
    """The per-device step in two kernels: attention with the append fused, then the combine."""
    B, x, _ = q.shape
    _check_args(shape, q=q, o=o, k_pool=k_pool, v_pool=v_pool, block_table=block_table, seq_lens=seq_lens,
                k_new=k_new, v_new=v_new)
    _check(lib().hetis_attn_decode_append(ctypes.byref(shape), B, q_head_begin, x, _dev(q, "q"), _dev(k_new, "k_new"),
                                          _dev(v_new, "v_new"), _dev(k_pool, "k_pool"), _dev(v_pool, "v_pool"),
                                          k_pool.shape[0], _dev(block_table, "block_table"), block_table.shape[2],
                                          _dev(seq_lens, "seq_lens"), max_seq_len, _dev(o, "o"),
                                          _dev(workspace, "workspace"), workspace.numel() * workspace.element_size(),
                                          flags, _stream(stream)), "hetis_attn_decode_append")


def attn_decode_launches(shape: CShape, flags: int = 0) -> int:
    """1 when hetis_attn_decode(_append) fuses the split merge into the attention kernel, else 2."""
    n = lib().hetis_attn_decode_launches(ctypes.byref(shape), flags)
    if n < 0:
        raise ValueError("invalid shape")
    return n


def attn_decode_launches_for(shape: CShape, num_seqs: int, q_head_count: int, max_seq_len: int, flags: int = 0) -> int:
    """Kernels of one hetis_attn_decode(_append) launch (1: merge fused, opt-in or group mode; 2: + combine)."""
    n = lib().hetis_attn_decode_launches_for(ctypes.byref(shape), num_seqs, q_head_count, max_seq_len, flags)
    if n < 0:
        raise ValueError("invalid arguments")
    return n


def attn_decode_units(shape: CShape, units, q, k_pool, v_pool, block_table, seq_lens, max_seq_len: int, o,
                      workspace, k_new=None, v_new=None, flags: int = 0, stream=None) -> None:
    """A per-request plan's units on the full layouts in one attention launch + one combine
    (hetis_attn_decode_units).  units: device int32 [U][2] (request, global kv head); q, o
    [B][H][d]; block_table [B][H_kv][max_pages]; k_new, v_new [B][H_kv][d] or None."""
    if units.dtype != torch.int32 or units.dim() != 2 or units.shape[1] != 2 or not units.is_contiguous():
        raise ValueError("units must be a contiguous int32 [U][2] tensor")
    H, Hkv = shape.num_q_heads, shape.num_kv_heads
    if q.dim() != 3 or q.shape[1] != H:
        raise ValueError(f"q must be [B][{H}][d] (all heads), got {tuple(q.shape)}")
    _check_args(shape, q=q, o=o, k_pool=k_pool, v_pool=v_pool, block_table=block_table, seq_lens=seq_lens,
                k_new=k_new, v_new=v_new)
    if o.dim() != 3 or o.shape[1] != H:
        raise ValueError(f"o must be [B][{H}][d], got {tuple(o.shape)}")
    _check(lib().hetis_attn_decode_units(ctypes.byref(shape), q.shape[0], units.shape[0], _dev(units, "units"),
                                         _dev(q, "q"), _dev(k_new, "k_new"), _dev(v_new, "v_new"), _dev(k_pool, "k_pool"),
                                         _dev(v_pool, "v_pool"), k_pool.shape[0], _dev(block_table, "block_table"),
                                         block_table.shape[2], _dev(seq_lens, "seq_lens"), max_seq_len,
                                         ctypes.c_void_p(o.data_ptr()), o.stride(0), _dev(workspace, "workspace"),
                                         workspace.numel() * workspace.element_size(), flags, _stream(stream)),
           "hetis_attn_decode_units")


def attn_decode(shape: CShape, q, k_pool, v_pool, block_table, seq_lens, max_seq_len: int, o, workspace,
                q_head_begin: int = 0, flags: int = 0, stream=None) -> None:
    B, x, _ = q.shape
    _check_args(shape, q=q, o=o, k_pool=k_pool, v_pool=v_pool, block_table=block_table, seq_lens=seq_lens)
    _check(lib().hetis_attn_decode(ctypes.byref(shape), B, q_head_begin, x, _dev(q, "q"), _dev(k_pool, "k_pool"),
                                   _dev(v_pool, "v_pool"), k_pool.shape[0], _dev(block_table, "block_table"),
                                   block_table.shape[2], _dev(seq_lens, "seq_lens"), max_seq_len, _dev(o, "o"),
                                   _dev(workspace, "workspace"), workspace.numel() * workspace.element_size(), flags,
                                   _stream(stream)), "hetis_attn_decode")


# ---------------------------------------------------------------- the step's exchanges over peer memory
def peer_state_bytes() -> int:
    return int(lib().hetis_peer_state_bytes())


def peer_access(peer_device: int) -> None:
    """Enable kernels on the current device to dereference peer_device's memory (hetis_peer_access)."""
    _check(lib().hetis_peer_access(int(peer_device)), "hetis_peer_access")


def alloc_peer_state(device) -> torch.Tensor:
    """A zero-filled device state for hetis_peer_group_create (int64 slots; torch allocations are 512-B aligned)."""
    return torch.zeros(peer_state_bytes() // 8, dtype=torch.int64, device=device)


class PeerGroup:
    """Owned hetis_peer_group: this rank's view of every rank's state and o_full and of the root's inputs."""

    def __init__(self, plan: Plan, rank: int, root: int, gather_root: int, state_peers, o_full_peers,
                 o_seq_stride: int, q_full_root, k_new_full_root, v_new_full_root):
        n = plan.num_devices
        if len(state_peers) != n or len(o_full_peers) != n:
            raise ValueError("one state and one o_full (or None) per rank")
        ptr = lambda t: None if t is None else (t.data_ptr() if hasattr(t, "data_ptr") else int(t))
        st = (ctypes.c_void_p * n)(*[ptr(t) for t in state_peers])
        of = (ctypes.c_void_p * n)(*[ptr(t) for t in o_full_peers])
        h = ctypes.c_void_p()
        _check(lib().hetis_peer_group_create(plan.handle, rank, root, gather_root, st, of, o_seq_stride,
                                             ptr(q_full_root), ptr(k_new_full_root), ptr(v_new_full_root),
                                             ctypes.byref(h)), "hetis_peer_group_create")
        self._h = h
        self.plan = plan
        self.rank, self.root, self.gather_root = rank, root, gather_root
        self._keep = (state_peers, o_full_peers, q_full_root, k_new_full_root, v_new_full_root)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.hetis_peer_group_destroy(h)
            self._h = None


def scatter_pull(group: PeerGroup, num_seqs: int, q_shard, k_new_shard, v_new_shard, stream=None) -> None:
    """a2 over peer memory: (root) publish the step's inputs, acknowledge the previous o_full, wait for the
    root, copy this rank's range of q / new k, v straight from the root's buffers."""
    _check(lib().hetis_scatter_pull(group.handle, num_seqs, _dev(q_shard, "q_shard"), _dev(k_new_shard, "k_new_shard"),
                                    _dev(v_new_shard, "v_new_shard"), _stream(stream)), "hetis_scatter_pull")


def attn_combine_peers(group: PeerGroup, seq_lens, max_seq_len: int, workspace, stream=None) -> None:
    """a5 + a6 in one kernel: merge this rank's splits, store every row into every receiving rank's o_full at
    its global head index, publish the epoch."""
    _check(lib().hetis_attn_combine_peers(group.handle, seq_lens.shape[0], _dev(seq_lens, "seq_lens"), max_seq_len,
                                          _dev(workspace, "workspace"), workspace.numel() * workspace.element_size(),
                                          _stream(stream)), "hetis_attn_combine_peers")


def attn_partial_pull(group: PeerGroup, num_seqs: int, k_pool, v_pool, block_table, seq_lens, max_seq_len: int,
                      workspace, flags: int = 0, stream=None) -> None:
    """a2 + a3 + a4 in one kernel: the partial attention with the append fused, q and the new k, v rows
    read straight from the Primary's buffers (hetis_attn_partial_pull)."""
    _check(lib().hetis_attn_partial_pull(group.handle, num_seqs, _dev(k_pool, "k_pool"), _dev(v_pool, "v_pool"),
                                         k_pool.shape[0], _dev(block_table, "block_table"), block_table.shape[2],
                                         _dev(seq_lens, "seq_lens"), max_seq_len, _dev(workspace, "workspace"),
                                         workspace.numel() * workspace.element_size(), flags, _stream(stream)),
           "hetis_attn_partial_pull")


def attn_decode_peers(group: PeerGroup, q_shard, k_pool, v_pool, block_table, seq_lens, max_seq_len: int, workspace,
                      k_new_shard=None, v_new_shard=None, flags: int = 0, stream=None) -> None:
    """a3 + a4 + a5 + a6 in one kernel: attention (append fused when k/v_new_shard are given) whose split
    merge stores every row into every receiving rank's o_full and publishes the epoch (hetis_attn_decode_peers)."""
    _check(lib().hetis_attn_decode_peers(group.handle, q_shard.shape[0], _dev(q_shard, "q_shard"),
                                         _dev(k_new_shard, "k_new_shard"), _dev(v_new_shard, "v_new_shard"),
                                         _dev(k_pool, "k_pool"), _dev(v_pool, "v_pool"), k_pool.shape[0],
                                         _dev(block_table, "block_table"), block_table.shape[2],
                                         _dev(seq_lens, "seq_lens"), max_seq_len, _dev(workspace, "workspace"),
                                         workspace.numel() * workspace.element_size(), flags, _stream(stream)),
           "hetis_attn_decode_peers")


def attn_decode_peers_pull(group: PeerGroup, num_seqs: int, k_pool, v_pool, block_table, seq_lens, max_seq_len: int,
                           workspace, flags: int = 0, stream=None) -> None:
    """The pull form of hetis_attn_decode_peers (q_shard = NULL): the scatter, the append, the attention, the
    split merge and the stores into every receiving rank's o_full in ONE kernel (then hetis_peer_wait)."""
    _check(lib().hetis_attn_decode_peers(group.handle, num_seqs, None, None, None, _dev(k_pool, "k_pool"),
                                         _dev(v_pool, "v_pool"), k_pool.shape[0], _dev(block_table, "block_table"),
                                         block_table.shape[2], _dev(seq_lens, "seq_lens"), max_seq_len,
                                         _dev(workspace, "workspace"), workspace.numel() * workspace.element_size(),
                                         flags, _stream(stream)), "hetis_attn_decode_peers")


def peer_wait(group: PeerGroup, stream=None) -> None:
    """The step's last kernel: wait for every rank's rows of this step (receiving ranks), record the step."""
    _check(lib().hetis_peer_wait(group.handle, _stream(stream)), "hetis_peer_wait")


# ---------------------------------------------------------------- NCCL scatter / gather
def scatter_q(plan: Plan, comm_ptr: int, rank: int, root: int, num_seqs: int, q_full, k_new_full, v_new_full,
              q_shard, k_new_shard, v_new_shard, workspace, stream=None) -> None:
    _check(lib().hetis_scatter_q(plan.handle, ctypes.c_void_p(comm_ptr), rank, root, num_seqs,
                                 _dev(q_full, "q_full"), _dev(k_new_full, "k_new_full"), _dev(v_new_full, "v_new_full"),
                                 _dev(q_shard, "q_shard"), _dev(k_new_shard, "k_new_shard"),
                                 _dev(v_new_shard, "v_new_shard"), _dev(workspace, "workspace"),
                                 0 if workspace is None else workspace.numel() * workspace.element_size(),
                                 _stream(stream)), "hetis_scatter_q")


def gather(plan: Plan, comm_ptr: int, rank: int, root: int, num_seqs: int, o_shard, o_full, workspace,
           stream=None) -> None:
    _check(lib().hetis_gather(plan.handle, ctypes.c_void_p(comm_ptr), rank, root, num_seqs, _dev(o_shard, "o_shard"),
                              _dev(o_full, "o_full"), _dev(workspace, "workspace"),
                              0 if workspace is None else workspace.numel() * workspace.element_size(),
                              _stream(stream)), "hetis_gather")


# ---------------------------------------------------------------- sequence-wise split (row f3)
def seq_split_lens(num_ranks: int, rank: int, page_size: int, seq_lens, local_lens, append_lens=None,
                   stream=None) -> None:
    """Page-striped sequence split: this rank's token counts (and append lengths) from global lengths."""
    _check(lib().hetis_seq_split_lens(num_ranks, rank, page_size, seq_lens.shape[0], _dev(seq_lens, "seq_lens"),
                                      _dev(local_lens, "local_lens"), _dev(append_lens, "append_lens"),
                                      _stream(stream)), "hetis_seq_split_lens")


def seq_merge(shape: CShape, o_parts, lse_parts, o, stream=None) -> None:
    """o_parts float [N][B][x][D], lse_parts float [N][B][x] -> o [B][x][D] (o dtype; rows may be strided).
    Parts may sit at any stride (e.g. views into the all-gather's staging); each part must be dense."""
    n, B, x, D = o_parts.shape
    if not (o.is_cuda and o_parts.is_cuda and lse_parts.is_cuda):
        raise ValueError("o, o_parts and lse_parts must be CUDA tensors")
    if not (o_parts[0].is_contiguous() and lse_parts[0].is_contiguous()):
        raise ValueError("each part of o_parts / lse_parts must be dense")
    if o_parts.dtype != torch.float32 or lse_parts.dtype != torch.float32:
        raise ValueError("o_parts and lse_parts must be float32")
    _check(lib().hetis_seq_merge(ctypes.byref(shape), n, B, x, ctypes.c_void_p(o_parts.data_ptr()), o_parts.stride(0),
                                 ctypes.c_void_p(lse_parts.data_ptr()), lse_parts.stride(0),
                                 ctypes.c_void_p(o.data_ptr()), o.stride(0), _stream(stream)), "hetis_seq_merge")


def seq_broadcast_q(shape: CShape, comm_ptr: int, num_ranks: int, rank: int, root: int, q, k_new, v_new,
                    stream=None) -> None:
    _check(lib().hetis_seq_broadcast_q(ctypes.byref(shape), ctypes.c_void_p(comm_ptr), num_ranks, rank, root,
                                       q.shape[0], _dev(q, "q"), _dev(k_new, "k_new"), _dev(v_new, "v_new"),
                                       _stream(stream)), "hetis_seq_broadcast_q")


def seq_allgather_merge(shape: CShape, comm_ptr: int, num_ranks: int, rank: int, num_seqs: int, part, staging, o,
                        stream=None) -> None:
    """part: float [B*H*D + B*H] (o then lse); staging: float [N][same]; o: [B][H][D] (o dtype)."""
    _check(lib().hetis_seq_allgather_merge(ctypes.byref(shape), ctypes.c_void_p(comm_ptr), num_ranks, rank, num_seqs,
                                           _dev(part, "part"), _dev(staging, "staging"), _dev(o, "o"), o.stride(0),
                                           _stream(stream)), "hetis_seq_allgather_merge")
