import os, sys, tempfile, time
sys.path.insert(0, os.getcwd())
import torch, torch.distributed as dist
from paper_2509_08309_b200 import hetis, workload
from paper_2509_08309_b200.step import DecodeStep
mode = sys.argv[3]
torch.cuda.set_device(0); dev = torch.device("cuda", 0)
if "nccl" in mode:
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29611")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
else:
    dist.init_process_group("gloo", init_method="file://" + os.path.join(tempfile.mkdtemp(), "rdv"), rank=0, world_size=1)
B = int(sys.argv[1]); L = int(sys.argv[2]); shape = workload.LLAMA2_70B
lens = torch.full((B,), L, dtype=torch.int32)
plan = hetis.plan_create(hetis.make_shape(shape), 1, [64])
b = workload.make_decode_batch(shape, lens, 3, dev)
st = DecodeStep(shape, plan, 0, B, L, dev)
o_full = torch.full((B, 64, 128), float("nan"), device=dev)
q_full, kn, vn = b.q.clone(), b.k_new.clone(), b.v_new.clone()
st.setup_peers(o_full, q_full, kn, vn, gather_root=-1)
sync = "sync" in mode
for i in range(6):
    st.scatter_peers()
    if sync: torch.cuda.synchronize()
    if "fused" in mode:
        hetis.attn_decode_peers(st.group, st.buf.q_shard, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L,
                                st.buf.workspace, k_new_shard=st.buf.k_new, v_new_shard=st.buf.v_new)
    else:
        hetis.attn_partial_append(st.cshape, st.buf.q_shard, st.buf.k_new, st.buf.v_new, b.k_pool, b.v_pool,
                                  b.block_table, b.seq_lens, L, st.buf.workspace)
        hetis.attn_combine_peers(st.group, b.seq_lens, L, st.buf.workspace)
    if sync: torch.cuda.synchronize()
    hetis.peer_wait(st.group)
    if sync: torch.cuda.synchronize()
t = time.time(); torch.cuda.synchronize(); print(mode, "done", round(time.time() - t, 3), st.peer_state.cpu()[:1].tolist(), "nan", torch.isnan(o_full).sum().item(), flush=True)
dist.destroy_process_group()
