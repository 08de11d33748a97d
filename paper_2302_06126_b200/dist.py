"""torch.distributed plumbing for one-process-per-GPU runs (plumbing only, no method arithmetic).

  init_from_env()     read RANK / LOCAL_RANK / WORLD_SIZE (torchrun) and init the process group
  bootstrap_comm()    rank 0 makes libtag's 128-byte NCCL id, torch.distributed broadcasts it,
                      every rank creates its libtag communicator
  max_over_ranks()    device-timed numbers are reported as the max over ranks
"""
import os

import torch
import torch.distributed as dist


def env_ranks():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def init_from_env(backend=None):
    """Returns (rank, local_rank, world). Initialises the default process group when world > 1."""
    rank, local_rank, world = env_ranks()
    if world > 1 and not dist.is_initialized():
        backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local_rank)
            dist.init_process_group(backend, device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    return rank, local_rank, world


def _comm_device():
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def broadcast_bytes(payload, nbytes=128, src=0):
    """Broadcast a fixed-size byte string from `src` (torch.distributed; any backend)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return payload
    t = torch.zeros(nbytes, dtype=torch.uint8, device=_comm_device())
    if dist.get_rank() == src:
        t.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().tolist())


def bootstrap_comm(tag, local_rank, loopback=False, multicast=False):
    """Create the libtag communicator over all ranks of the default group (n = world size).
    loopback: with one rank, still create a (one-rank) NCCL communicator so the collective code
    paths run; multicast: NVLS multicast stores in the fused push."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    if world == 1:
        return tag.Comm(1, 0, local_rank, loopback=loopback, multicast=multicast)
    uid = tag.unique_id() if rank == 0 else bytes(128)
    uid = broadcast_bytes(uid, 128, 0)
    return tag.Comm(world, rank, local_rank, uid, multicast=multicast)


def max_over_ranks(x):
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_comm_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_gather_object(obj):
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def barrier():
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
