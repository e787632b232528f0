"""Multi-GPU check of the sharded path's NCCL collectives (one process per GPU):
torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/nccl_selftest.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2006_05874_b200 import ihs  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl")
uid = [ihs.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
comm = ihs.NcclComm(uid[0], world, rank, local)
bad = ihs.comm_selftest(comm, local, 1 << 16)
print(f"rank {rank}/{world}: mismatches {bad}", flush=True)
comm.close()
dist.destroy_process_group()
sys.exit(1 if bad else 0)
