"""Does NCCL's PreMulSum apply the scalar on a one-rank communicator? (tools only)"""
import os
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
for n in (1000, 44032, 65536, 131072, 262144, 308228, 1 << 20):
    x = torch.ones(n, device="cuda")
    op = dist._make_nccl_premul_sum(0.7)
    dist.all_reduce(x, op=op)
    torch.cuda.synchronize()
    print(n, "mean", x.mean().item(), "frac scaled", (x - 0.7).abs().lt(1e-6).float().mean().item(), flush=True)
dist.destroy_process_group()
