"""Multi-GPU host logic: independent reconstructor replicas, one process per GPU.

The FEWHA frame (reconstructor.hpp:310-355) has no exchange step between
telescope instances, so N GPUs run N independent instance streams (SURVEY §8e,
BASELINE config 5) with no data-path collective.  The only collectives are the
timing barrier and the max-over-ranks reduction of the measured times.  The
same code runs with backend "nccl" on GPUs and "gloo" on CPU (tests).
"""
import os
from dataclasses import dataclass


@dataclass
class ReplicaContext:
    rank: int
    world: int
    local_rank: int
    dist: object  # torch.distributed or None

    @property
    def seed(self) -> int:
        """Per-replica slope-stream seed: every rank reconstructs its own instance."""
        return 1 + self.rank

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max_over_ranks(self, values, device=None):
        """Element-wise max of a list of floats over all ranks (fp64)."""
        vals = [float(v) for v in values]
        if self.dist is None:
            return vals
        import torch
        t = torch.tensor(vals, dtype=torch.float64, device=device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return [float(x) for x in t.tolist()]

    def sum_over_ranks(self, values, device=None):
        vals = [float(v) for v in values]
        if self.dist is None:
            return vals
        import torch
        t = torch.tensor(vals, dtype=torch.float64, device=device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return [float(x) for x in t.tolist()]

    def aggregate_throughput(self, frames_per_rank, max_ms):
        """Whole-job reconstructions/s: all ranks' frames over the slowest rank's time."""
        return self.world * frames_per_rank / (max_ms / 1000.0)

    def shutdown(self):
        if self.dist is not None and self.dist.is_initialized():
            self.dist.destroy_process_group()


def init_replicas(backend=None):
    """Read RANK/WORLD_SIZE/LOCAL_RANK (torchrun) and join the process group.

    backend None -> "nccl" (one GPU per rank, device = LOCAL_RANK); override with
    FEWHA_DIST_BACKEND=gloo for CPU runs.  world 1 -> no process group at all.
    """
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world <= 1:
        return ReplicaContext(rank=0, world=1, local_rank=local, dist=None)
    import torch
    import torch.distributed as dist
    backend = backend or os.environ.get("FEWHA_DIST_BACKEND", "nccl")
    if backend == "nccl":
        ndev = torch.cuda.device_count()
        if ndev == 0:
            raise RuntimeError("FEWHA replicas: backend nccl needs a CUDA device per rank")
        local = local % ndev
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return ReplicaContext(rank=rank, world=world, local_rank=local, dist=dist)


def share_nccl_id(rc: ReplicaContext, make_id) -> bytes | None:
    """Rank 0 makes a 128-byte NCCL unique id (make_id()) and every rank gets it
    over the process group (broadcast_object_list); world 1 -> None."""
    if rc.dist is None:
        return None
    obj = [make_id() if rc.rank == 0 else None]
    rc.dist.broadcast_object_list(obj, src=0)
    return obj[0]


def shard_frame(rec, rc: ReplicaContext):
    """Per-WFS sharding of ONE reconstruction frame over the ranks:
    rank r owns fewha_gpu_shard_range(r, world) and the partial adjoint layer
    sums are all-reduced through NCCL inside the frame graph.  Returns the
    owned WFS range."""
    import paper_2009_00946_b200 as fg
    nid = share_nccl_id(rc, fg.nccl_unique_id)
    rec.shard(rc.rank, rc.world, nid)
    return rec.shard_wfs()
