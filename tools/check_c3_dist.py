"""Exercise bench.c3_distributed through a 1-rank NCCL process group."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
import torch
import torch.distributed as dist
import bench

torch.cuda.set_device(0)
dist.init_process_group("nccl", world_size=1, rank=0)
print(bench.c3_distributed(torch, 1, 0))
dist.barrier()
dist.destroy_process_group()
