"""Can two NCCL ranks share one GPU on this box?  (If yes, the NCCL expert-parallel transport can
be tested with W = 2 on a 1-GPU box.)  torchrun --nproc-per-node 2 tools/nccl_same_gpu_probe.py"""
import os
import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
try:
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    t = torch.ones(4, device="cuda") * (rank + 1)
    dist.all_reduce(t)
    torch.cuda.synchronize()
    print(f"rank {rank}: all_reduce ok {t.tolist()}", flush=True)
    dist.destroy_process_group()
except Exception as e:  # noqa: BLE001
    print(f"rank {rank}: NCCL with two ranks on one GPU failed: {str(e)[:300]}", flush=True)
