"""Probe: torch symmetric memory on this box (world 1, NCCL): peer pointers, multicast."""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
g = dist.group.WORLD
for backend in (None, "CUDA", "NCCL"):
    try:
        if backend:
            symm.set_backend(backend)
        t = symm.empty(1024, dtype=torch.float32, device="cuda")
        h = symm.rendezvous(t, g.group_name)
        print(backend, "ok: world", h.world_size, "rank", h.rank, "buffer_ptrs", h.buffer_ptrs,
              "multicast_ptr", getattr(h, "multicast_ptr", None), "signal_pad", h.signal_pad_ptrs[:1])
        h.barrier(channel=0)
        torch.cuda.synchronize()
        print(backend, "barrier ok")
    except Exception as e:
        print(backend, "failed:", type(e).__name__, str(e)[:300])
dist.destroy_process_group()
