import os, sys, tempfile
sys.path.insert(0, os.getcwd())
import torch, torch.distributed as dist
from paper_2509_08309_b200 import hetis, workload
from paper_2509_08309_b200.step import DecodeStep
dist.init_process_group("gloo", init_method="file://" + os.path.join(tempfile.mkdtemp(), "rdv"), rank=0, world_size=1)
torch.cuda.set_device(0); dev = torch.device("cuda", 0)
shape = workload.LLAMA2_70B; B, L = 16, 512
lens = torch.full((B,), L, dtype=torch.int32)
plan = hetis.plan_create(hetis.make_shape(shape), 1, [64])
b = workload.make_decode_batch(shape, lens, 3, dev)
st = DecodeStep(shape, plan, 0, B, L, dev)
o_full = torch.full((B, 64, 128), float("nan"), device=dev)
st.setup_peers(o_full, b.q.clone(), b.k_new.clone(), b.v_new.clone(), gather_root=-1)
for name, fn in [("pull", lambda: hetis.attn_partial_pull(st.group, B, b.k_pool, b.v_pool, b.block_table, b.seq_lens, L, st.buf.workspace)),
                 ("combine_peers", lambda: hetis.attn_combine_peers(st.group, b.seq_lens, L, st.buf.workspace)),
                 ("peer_wait", lambda: hetis.peer_wait(st.group)),
                 ("step_peers", lambda: st.step_peers(b.k_pool, b.v_pool, b.block_table, b.seq_lens))]:
    n0 = hetis.launch_count(); fn(); torch.cuda.synchronize(); print(name, hetis.launch_count() - n0, flush=True)
dist.destroy_process_group()
