"""One rank's decode step of one layer: the composition of
the C-ABI calls -- scatter (N > 1), kv_append, attention partial + combine,
gather (N > 1).  Buffers are torch tensors (device memory only); every step
runs in libhetis.so kernels or NCCL.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import hetis, workload


@dataclass
class RankBuffers:
    """Device buffers one rank owns for one layer."""
    q_shard: torch.Tensor       # [B][x][D]
    k_new: torch.Tensor         # [B][x/r][D]
    v_new: torch.Tensor
    o_shard: torch.Tensor       # [B][x][D] (o dtype)
    workspace: torch.Tensor     # attention workspace
    comm_ws: torch.Tensor | None


class DecodeStep:
    """Runs the hot path for one rank.

    shape      : global model shape (H, H_kv, d, P, dtype)
    plan       : hetis.Plan with the head split (global, per_request = 0)
    rank, comm : position in the plan and the raw ncclComm_t (None at N = 1)
    """

    def __init__(self, shape: workload.Shape, plan: hetis.Plan, rank: int, num_seqs: int, max_seq_len: int,
                 device, o_dtype: str = "f32", comm_ptr: int | None = None, root: int = 0):
        self.shape = shape
        self.cshape = hetis.make_shape(shape, o_dtype)
        self.plan = plan
        self.rank = rank
        self.world = plan.num_devices
        self.root = root
        self.comm_ptr = comm_ptr
        self.num_seqs = num_seqs
        self.max_seq_len = max_seq_len
        self.q_begin, self.q_count = plan.heads(rank)
        self.device = device
        D, r = shape.head_dim, shape.r
        dt = shape.torch_dtype
        odt = torch.bfloat16 if o_dtype == "bf16" else torch.float32
        ws = hetis.attn_decode_workspace(self.cshape, num_seqs, self.q_count, max_seq_len)
        comm_ws = None
        if comm_ptr is not None:
            comm_ws = hetis.alloc_workspace(plan.comm_workspace(rank, num_seqs), device)
        self.buf = RankBuffers(
            q_shard=torch.empty((num_seqs, self.q_count, D), dtype=dt, device=device),
            k_new=torch.empty((num_seqs, self.q_count // r, D), dtype=dt, device=device),
            v_new=torch.empty((num_seqs, self.q_count // r, D), dtype=dt, device=device),
            o_shard=torch.empty((num_seqs, self.q_count, D), dtype=odt, device=device),
            workspace=hetis.alloc_workspace(ws, device),
            comm_ws=comm_ws,
        )
        self.o_dtype = odt

    # kernels launched per step by this rank (for gpu_launches accounting)
    def launches_per_step(self) -> int:
        n = 3  # kv_append, attention partial, combine (2 with the fused append)
        if self.world > 1:
            x = [self.plan.heads(i)[1] for i in range(self.world)]
            if self.rank == self.root:
                n += 1                                    # one batched scatter pack (every rank's slices)
            n += 1                                        # one batched gather placement
        return n

    def scatter(self, q_full, k_new_full, v_new_full, stream=None):
        hetis.scatter_q(self.plan, self.comm_ptr, self.rank, self.root, self.num_seqs, q_full, k_new_full,
                        v_new_full, self.buf.q_shard, self.buf.k_new, self.buf.v_new, self.buf.comm_ws, stream)

    def append(self, k_pool, v_pool, block_table, seq_lens, k_new=None, v_new=None, stream=None):
        hetis.kv_append(self.cshape, self.buf.k_new if k_new is None else k_new,
                        self.buf.v_new if v_new is None else v_new, k_pool, v_pool, block_table, seq_lens, stream)

    def attention(self, k_pool, v_pool, block_table, seq_lens, q=None, o=None, stream=None, flags: int = 0):
        q = self.buf.q_shard if q is None else q
        o = self.buf.o_shard if o is None else o
        hetis.attn_partial(self.cshape, q, k_pool, v_pool, block_table, seq_lens, self.max_seq_len,
                           self.buf.workspace, q_head_begin=self.q_begin, flags=flags, stream=stream)
        hetis.attn_combine(self.cshape, seq_lens, self.max_seq_len, o, self.buf.workspace, q_head_count=self.q_count,
                           stream=stream)
        return o

    def append_attention(self, k_pool, v_pool, block_table, seq_lens, q=None, o=None, stream=None, flags: int = 0):
        """kv_append fused into the attention kernel, then the combine: the per-device step in two kernels
        (bit-identical to append() followed by attention())."""
        q = self.buf.q_shard if q is None else q
        o = self.buf.o_shard if o is None else o
        hetis.attn_partial_append(self.cshape, q, self.buf.k_new, self.buf.v_new, k_pool, v_pool, block_table, seq_lens,
                                  self.max_seq_len, self.buf.workspace, q_head_begin=self.q_begin, flags=flags,
                                  stream=stream)
        hetis.attn_combine(self.cshape, seq_lens, self.max_seq_len, o, self.buf.workspace, q_head_count=self.q_count,
                           stream=stream)
        return o

    def gather(self, o_full, root: int = -1, stream=None):
        hetis.gather(self.plan, self.comm_ptr, self.rank, root, self.num_seqs, self.buf.o_shard, o_full,
                     self.buf.comm_ws, stream)

    # ---- exchanges over peer memory (NVLink): pull scatter (hetis_scatter_pull), the combine fused with the
    # gather (hetis_attn_combine_peers) and the step's closing wait (hetis_peer_wait); epochs live on the device
    def setup_peers(self, o_full: torch.Tensor | None, q_full=None, k_new_full=None, v_new_full=None,
                    gather_root: int = -1) -> None:
        """Map every rank's exchange state and o_full, and the root's q_full / k_new_full / v_new_full, into
        this process (CUDA IPC handles exchanged over the default torch.distributed group -- gloo or NCCL; on
        one NVSwitch box the mappings are NVLink peer memory).  Collective.  Only the root passes the *_full
        tensors; o_full may be None on a rank that receives nothing (gather_root >= 0, not this rank)."""
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        self.o_full = o_full
        self.peer_state = hetis.alloc_peer_state(self.device)
        root_bufs = None
        if self.rank == self.root:
            root_bufs = tuple(reduce_tensor(t) for t in (q_full, k_new_full, v_new_full))
        mine = (reduce_tensor(self.peer_state), None if o_full is None else reduce_tensor(o_full), root_bufs)
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine)
        peer_devices = set()

        def open_here(red):
            # torch's rebuild opens the IPC handle (cudaIpcOpenMemHandle, cudaIpcMemLazyEnablePeerAccess) under the
            # device it is told; opening it under THIS rank's device maps the peer's memory into the context our
            # kernels run in (NVLink peer memory when the exporter is another GPU) -- the documented pattern, rather
            # than a mapping in the exporter device's context of this process.  The tensor is only used for its
            # pointer.  Rebuild args: (type, size, stride, offset, storage type, dtype, device, handle, ...).
            fn, args = red
            args = list(args)
            peer_devices.add(int(args[6]))
            args[6] = self.device.index
            return fn(*args)

        states, outs = [], []
        for i, (rs, ro, _) in enumerate(everyone):
            if i == self.rank:
                states.append(self.peer_state)
                outs.append(o_full)
            else:
                states.append(open_here(rs))
                outs.append(None if ro is None else open_here(ro))
        if self.rank == self.root:
            root = (q_full, k_new_full, v_new_full)
        else:
            root = tuple(open_here(red) for red in everyone[self.root][2])
        # the peers' buffers live on their own GPUs: this device's kernels load / store them over NVLink
        with torch.cuda.device(self.device):
            for d in sorted(peer_devices - {self.device.index}):
                hetis.peer_access(d)
        stride = (o_full.stride(0) if o_full is not None
                  else self.shape.num_q_heads * self.shape.head_dim)
        self.group = hetis.PeerGroup(self.plan, self.rank, self.root, gather_root, states, outs, stride, *root)

    def scatter_peers(self, stream=None):
        """Every rank pulls its heads' q and its kv heads' new k, v straight from the root's buffers (the root
        first publishes that this step's inputs are written).  One kernel."""
        hetis.scatter_pull(self.group, self.num_seqs, self.buf.q_shard, self.buf.k_new, self.buf.v_new, stream=stream)

    def merge_fused(self, flags: int = 0) -> bool:
        """True when the attention kernel itself merges the splits and stores O into every receiving rank
        (hetis_attn_decode_peers: the per-warp tensor-core kernel, a rank holding heads)."""
        return self.q_count > 0 and self.num_seqs > 0 and hetis.attn_decode_launches(
            self.cshape, flags | hetis.ATTN_FUSED_MERGE) == 1

    def merge_fused_default(self, flags: int = 0) -> bool:
        """The default choice: the merge fused into the attention kernel where the caller opts in
        (HETIS_ATTN_FUSED_MERGE) or where this rank's launch runs in group mode (<= one (request, kv head) pair
        per SM, <= 8 splits: the merge then runs in shared memory and is measured faster than the combine)."""
        return self.merge_fused(flags) and (bool(flags & hetis.ATTN_FUSED_MERGE) or hetis.attn_decode_launches_for(
            self.cshape, self.num_seqs, self.q_count, self.max_seq_len, flags) == 1)

    def attention_gather_peers(self, k_pool, v_pool, block_table, seq_lens, stream=None, flags: int = 0,
                               fused_append: bool = True, merge_fused: bool | None = None):
        """Attention (kv_append fused by default) whose split merge stores every row into every receiving
        rank's o_full -- ONE kernel (hetis_attn_decode_peers) where the per-warp kernel runs, else the partial
        kernel + hetis_attn_combine_peers -- then the step's closing wait.  Returns o_full."""
        if merge_fused is None:                 # opt-in, or group mode
            merge_fused = self.merge_fused_default(flags)
        if merge_fused:
            hetis.attn_decode_peers(self.group, self.buf.q_shard, k_pool, v_pool, block_table, seq_lens,
                                    self.max_seq_len, self.buf.workspace,
                                    k_new_shard=self.buf.k_new if fused_append else None,
                                    v_new_shard=self.buf.v_new if fused_append else None, flags=flags, stream=stream)
            hetis.peer_wait(self.group, stream=stream)
            return self.o_full
        if fused_append:
            hetis.attn_partial_append(self.cshape, self.buf.q_shard, self.buf.k_new, self.buf.v_new, k_pool, v_pool,
                                      block_table, seq_lens, self.max_seq_len, self.buf.workspace,
                                      q_head_begin=self.q_begin, flags=flags, stream=stream)
        else:
            hetis.attn_partial(self.cshape, self.buf.q_shard, k_pool, v_pool, block_table, seq_lens,
                               self.max_seq_len, self.buf.workspace, q_head_begin=self.q_begin, flags=flags,
                               stream=stream)
        hetis.attn_combine_peers(self.group, seq_lens, self.max_seq_len, self.buf.workspace, stream=stream)
        hetis.peer_wait(self.group, stream=stream)
        return self.o_full

    def pull_supported(self, flags: int = 0) -> bool:
        """hetis_attn_partial_pull applies: this rank holds heads and requests, an ordinary launch."""
        return self.q_count > 0 and self.num_seqs > 0 and not (
            flags & (hetis.ATTN_PIPELINED | hetis.ATTN_DIAG_STREAM_ONLY))

    def step_peers(self, k_pool, v_pool, block_table, seq_lens, stream=None, flags: int = 0,
                   merge_fused: bool | None = None, pull: bool | None = None):
        """The whole N > 1 step over peer memory, no NCCL and no per-step host argument (graph-capturable):
        by default the attention kernel itself pulls q and the new k, v rows from the Primary
        (hetis_attn_partial_pull), then combine + gather into every rank's o_full, then the closing wait --
        three kernels; where the merge is fused (group mode, or opt-in) the pull, the attention, the merge and
        the stores into every o_full are ONE kernel (hetis_attn_decode_peers with q_shard = NULL) + the wait;
        pull=False: the separate pull scatter kernel first."""
        if merge_fused is None:
            merge_fused = self.merge_fused_default(flags)
        if pull is None:
            pull = self.pull_supported(flags)
        if pull and merge_fused:
            hetis.attn_decode_peers_pull(self.group, self.num_seqs, k_pool, v_pool, block_table, seq_lens,
                                         self.max_seq_len, self.buf.workspace, flags=flags, stream=stream)
            hetis.peer_wait(self.group, stream=stream)
            return self.o_full
        if pull:
            hetis.attn_partial_pull(self.group, self.num_seqs, k_pool, v_pool, block_table, seq_lens,
                                    self.max_seq_len, self.buf.workspace, flags=flags & ~hetis.ATTN_FUSED_MERGE,
                                    stream=stream)
            hetis.attn_combine_peers(self.group, seq_lens, self.max_seq_len, self.buf.workspace, stream=stream)
            hetis.peer_wait(self.group, stream=stream)
            return self.o_full
        self.scatter_peers(stream)
        return self.attention_gather_peers(k_pool, v_pool, block_table, seq_lens, stream=stream, flags=flags,
                                           merge_fused=merge_fused)
