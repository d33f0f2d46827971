"""Exercise bench.dp_leg (the N > 1 data-parallel headline) at world 1 on one
GPU under an NCCL process group: the code path the driver's multi-GPU run
takes, minus the other ranks."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import bench
r = bench.dp_leg(0, 0, 1, dist, steps=5, warmup=2, B_per=64)
print(json.dumps(r))
import argparse
args = argparse.Namespace(parallel="dp", mapping="heads", exchange_chunks=2)
print(json.dumps(bench.vitl_leg(steps=2, warmup=1, rank=0, world=1, dist=dist, args=args)))
dist.destroy_process_group()
