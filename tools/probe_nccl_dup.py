import os, torch, torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("nccl")
t = torch.ones(4, device="cuda") * (dist.get_rank() + 1)
try:
    dist.all_reduce(t); torch.cuda.synchronize()
    print("rank", dist.get_rank(), "allreduce ok", t.tolist(), flush=True)
except Exception as e:
    print("rank", dist.get_rank(), "FAILED", repr(e)[:300], flush=True)
dist.destroy_process_group()
