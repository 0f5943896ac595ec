"""Probe: which NCCL_* variables the box sets, and whether NCCL's INIT lines reach stderr."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
print("env:", {k: v for k, v in os.environ.items() if k.startswith("NCCL") or k.startswith("TORCH_NCCL")}, file=sys.stderr)
from bench import nccl_log_to_stderr  # noqa: E402
nccl_log_to_stderr()
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
t = torch.ones(4, device="cuda")
dist.all_reduce(t)
torch.cuda.synchronize()
print("rank", dist.get_rank(), "sum", t[0].item(), file=sys.stderr)
dist.destroy_process_group()
