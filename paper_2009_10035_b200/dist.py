"""Multi-GPU Force2Vec epochs: vertex-partitioned shards, one process per GPU
(DESIGN.md "Multi-GPU").

Semantics (pinned by the oracle, oracle/f2v_oracle.c orc_train with G > 1):
shard g of G owns a contiguous row range cut at quantiles of the per-vertex
work deg(u) + s (``shard_layout``: R-MAT's hubs do not pile onto shard 0),
shuffles it every epoch with partition_epoch on (seed, {0x22, epoch, g})
(sampling.cpp:7-19, trainer.cpp:216-217), uses the local batch
ceil(|shard| / T) with T = ceil(n / (G batch)) steps (so per-step work is
balanced too), and draws the negatives of its t-th batch from
(seed, {0x33, epoch, t, g}) or Philox with shard = g.  Step t = the t-th
local batch of every shard: all gradients on ONE snapshot of Z
(trainer.cpp:227-233), then every update (trainer.cpp:235) -- synchronous
minibatch SGD with global batch ~G*b.  G = 1 is exactly the reference.

Two exchange paths, same results:

* ``ShardedDevice`` (the product, ``bench.py --gpus N``): every GPU keeps a
  full replica of Z and runs the dataflow epoch kernel over its own rows; the
  kernel's update epilogue stores each new row into every replica through
  CUDA IPC mappings over NVLink (f2v_shard.cu), so the all-gather is fused
  into the update, row by row, overlapped with the compute.  torch.distributed
  is only used once, to all-gather the IPC handles.
* ``train_allgather`` (the baseline at the reference's synchronisation
  granularity): per step, the local batch's gradient on the replica, a
  failure vote, the local update, then an all-gather of (ids, rows) through
  torch.distributed (NCCL over NVLink on GPUs; gloo in the CPU tests) and the
  peers' rows written into the replica.  Its compute is a ``StepBackend``:
  ``DeviceBackend`` (the CUDA per-step operators) in production.
"""
from __future__ import annotations

import dataclasses
import os
import re
from typing import List, Optional, Tuple

import numpy as np

from . import (CsrGraph, Device, NumericalError, TrainConfig, TrainCounters, UsageError,
               negatives, partition_shard, shard_layout)

__all__ = ["env_rank", "ShardedDevice", "AllgatherDevice", "StepBackend", "DeviceBackend",
           "train_allgather", "shard_steps"]


def env_rank() -> Tuple[int, int, int]:
    """(rank, world, local_rank) from torchrun's environment (1 process = 1 GPU)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_steps(g: CsrGraph, batch: int, shards: int, negatives: int
                ) -> Tuple[List[int], List[int], List[int], int]:
    """Row bounds lo[G+1], per-shard batch size and batch count, T = steps."""
    lo, bs, _, T = shard_layout(g, batch, shards, negatives)
    nb = [(int(lo[i + 1] - lo[i]) + int(bs[i]) - 1) // int(bs[i]) for i in range(shards)]
    return [int(x) for x in lo], [int(x) for x in bs], nb, T


def _all_gather_objects(obj, group=None) -> list:
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


# ------------------------------------------------------------ fused (NVLink)
class ShardedDevice:
    """One rank of a G-GPU run: a Device whose epoch kernel stores every
    updated row into all G replicas (f2v_shard_init/export/attach)."""

    def __init__(self, rank: Optional[int] = None, world: Optional[int] = None,
                 device: Optional[int] = None, group=None):
        r, w, local = env_rank()
        self.rank = r if rank is None else rank
        self.world = w if world is None else world
        self.group = group
        self.dev = Device(local if device is None else device)

    def close(self):
        self.dev.close()

    def setup(self, g: CsrGraph, z0: Optional[np.ndarray] = None, dim: int = 128,
              seed: int = 1, lo: float = -1.0, hi: float = 1.0):
        """Upload the graph and the SAME initial Z on every rank (z0, or the
        configs' U(lo, hi) from Rng(seed, 0) generated on each device), then
        exchange the replica handles."""
        self.dev.upload_graph(g)
        if z0 is not None:
            self.dev.set_embedding(z0)
        else:
            self.dev.uniform_embedding(g.num_vertices(), dim, seed, lo, hi)
        self.dev.shard_init(self.rank, self.world)
        if self.world > 1:
            import torch.distributed as dist

            handles = _all_gather_objects(self.dev.shard_export(), self.group)
            self.dev.shard_attach(handles)
            dist.barrier(group=self.group)  # every rank mapped every replica
        else:
            self.dev.shard_attach([self.dev.shard_export()])

    def train_epochs(self, cfg: TrainConfig, first_epoch: int = 0, run_epochs: int = 0,
                     counters: Optional[TrainCounters] = None,
                     failure: Optional[dict] = None) -> list:
        """Epochs of the G-shard schedule; every rank gets the same losses."""
        c = dataclasses.replace(cfg, shards=self.world)
        return self.dev.train_epochs(c, first_epoch, run_epochs, counters=counters,
                                     failure=failure)

    def get_embedding(self) -> np.ndarray:
        return self.dev.get_embedding()

    def last_timing(self) -> dict:
        return self.dev.last_timing()

    @property
    def kernel_launches(self) -> int:
        return self.dev.kernel_launches


# ------------------------------------ per-step ncclAllGather (in the library)
class AllgatherDevice:
    """One rank of the per-step all-gather baseline run inside the library
    (f2v_train_epochs_allgather): every step's updated rows are exchanged
    with ncclAllGather on the context stream, no host staging.  Rank 0's NCCL
    unique id is broadcast through torch.distributed (any backend)."""

    def __init__(self, rank: Optional[int] = None, world: Optional[int] = None,
                 device: Optional[int] = None, group=None):
        r, w, local = env_rank()
        self.rank = r if rank is None else rank
        self.world = w if world is None else world
        self.group = group
        self.dev = Device(local if device is None else device)

    def close(self):
        self.dev.close()

    def setup(self, g: CsrGraph, z0: Optional[np.ndarray] = None, dim: int = 128,
              seed: int = 1, lo: float = -1.0, hi: float = 1.0):
        self.dev.upload_graph(g)
        if z0 is not None:
            self.dev.set_embedding(z0)
        else:
            self.dev.uniform_embedding(g.num_vertices(), dim, seed, lo, hi)
        uid = Device.nccl_unique_id() if self.rank == 0 else None
        if self.world > 1:
            import torch.distributed as dist

            box = [uid]
            dist.broadcast_object_list(box, src=0, group=self.group)
            uid = box[0]
        self.dev.nccl_init(uid, self.rank, self.world)

    def train_epochs(self, cfg: TrainConfig, first_epoch: int = 0, run_epochs: int = 0,
                     counters: Optional[TrainCounters] = None,
                     failure: Optional[dict] = None) -> list:
        c = dataclasses.replace(cfg, shards=self.world)
        return self.dev.train_epochs_allgather(c, first_epoch, run_epochs, counters=counters,
                                               failure=failure)

    def get_embedding(self) -> np.ndarray:
        return self.dev.get_embedding()

    def last_timing(self) -> dict:
        return self.dev.last_timing()


# ---------------------------------------------- per-step all-gather baseline
class StepBackend:
    """The per-rank compute of one step over the rank's local replica of Z."""
    d: int

    def grad(self, ids: np.ndarray, negs: np.ndarray, cfg: TrainConfig) -> np.ndarray:
        """grad_minibatch (trainer.cpp:108-165); raises NumericalError naming
        the first non-finite vertex in batch order."""
        raise NotImplementedError

    def loss(self, ids: np.ndarray, negs: np.ndarray, cfg: TrainConfig) -> float:
        raise NotImplementedError

    def apply(self, ids: np.ndarray, grads: np.ndarray, eta: float):
        raise NotImplementedError

    def get_rows(self, ids: np.ndarray) -> np.ndarray:
        raise NotImplementedError

    def set_rows(self, ids: np.ndarray, rows: np.ndarray):
        raise NotImplementedError


class DeviceBackend(StepBackend):
    """The CUDA per-step operators (f2v_grad_minibatch / f2v_apply_update /
    f2v_batch_loss / f2v_get_rows / f2v_set_rows) on one device."""

    def __init__(self, dev: Device):
        self.dev = dev
        self.d = dev.d

    def grad(self, ids, negs, cfg):
        return self.dev.grad_minibatch(ids, negs, cfg.model)

    def loss(self, ids, negs, cfg):
        return self.dev.batch_loss(ids, negs, cfg.model)

    def apply(self, ids, grads, eta):
        self.dev.apply_update(ids, grads, eta)

    def get_rows(self, ids):
        return self.dev.get_rows(ids)

    def set_rows(self, ids, rows):
        self.dev.set_rows(ids, rows)


_NOFAIL = np.iinfo(np.int64).max


def _failed_vertex(e: NumericalError, ids: np.ndarray) -> Tuple[int, int]:
    m = re.search(r"vertex (\d+)", str(e))
    v = int(m.group(1)) if m else int(ids[0])
    hit = np.nonzero(ids == v)[0]
    return (int(hit[0]) if len(hit) else 0), v


def train_allgather(backend: StepBackend, g: CsrGraph, cfg: TrainConfig, rank: int, world: int,
                    first_epoch: int = 0, run_epochs: int = 0, group=None,
                    tensor_device=None, counters: Optional[TrainCounters] = None) -> list:
    """The G-shard schedule with an explicit all-gather of updated rows after
    every step.  Returns the epoch losses (identical on every rank; summed in
    (step, shard) order like orc_train) when cfg.monitor_loss."""
    import torch
    import torch.distributed as dist

    if world != dist.get_world_size(group):
        raise UsageError("world does not match the process group")
    d = backend.d
    n = g.num_vertices()
    s = cfg.negatives
    bounds, bs, nb, T = shard_steps(g, cfg.batch, world, s)
    lo, hi = bounds[rank], bounds[rank + 1]
    bmax = max(bs)
    end = min(cfg.epochs, first_epoch + run_epochs) if run_epochs else cfg.epochs
    tdev = tensor_device if tensor_device is not None else torch.device("cpu")
    losses = []
    for epoch in range(first_epoch, end):
        eta = cfg.lr
        if cfg.lr_decay == "linear_to_zero":  # trainer.cpp:212-214, fp32
            eta = float(np.float32(cfg.lr) * (np.float32(1) - np.float32(epoch) /
                                              np.float32(cfg.epochs)))
        perm = partition_shard(hi - lo, bs[rank], cfg.seed, epoch, rank, world) + np.uint32(lo)
        epoch_loss = 0.0
        for t in range(T):
            if t < nb[rank]:
                ids = perm[t * bs[rank]:min((t + 1) * bs[rank], hi - lo)]
                negs = negatives(cfg.sampler, cfg.seed, epoch, t, n, s, shard=rank,
                                 num_shards=world)
            else:
                ids = np.zeros(0, np.uint32)
                negs = np.zeros(0, np.uint32)
            # every shard's gradient on the same snapshot, then a failure vote
            # (the first failure in (step, shard, batch index) order wins and
            # no rank applies its update: trainer.cpp:149-152)
            fail_key, fail_v, grads, lossv = _NOFAIL, 0, None, 0.0
            if len(ids):
                try:
                    grads = backend.grad(ids, negs, cfg)
                except NumericalError as e:
                    i, fail_v = _failed_vertex(e, ids)
                    fail_key = rank * (1 << 32) + i
                if cfg.monitor_loss and fail_key == _NOFAIL:
                    lossv = backend.loss(ids, negs, cfg)
            vote = torch.tensor([fail_key, fail_v], dtype=torch.int64, device=tdev)
            votes = [torch.zeros_like(vote) for _ in range(world)]
            dist.all_gather(votes, vote, group=group)
            keys = [int(v[0]) for v in votes]
            k = int(np.argmin(keys))
            if keys[k] != _NOFAIL:
                raise NumericalError(f"non-finite gradient for vertex {int(votes[k][1])} "
                                     f"(epoch {epoch}, batch {t})")
            if len(ids):
                backend.apply(ids, grads, eta)
                rows = backend.get_rows(ids)
            else:
                rows = np.zeros((0, d), np.float32)
            # all-gather (count, ids, rows, loss) of every shard's step
            pack = np.zeros(1 + bmax + bmax * d + 2, np.int32)
            pack[0] = len(ids)
            pack[1:1 + len(ids)] = ids.view(np.int32)
            pack[1 + bmax:1 + bmax + len(ids) * d] = rows.reshape(-1).view(np.int32)
            pack[-2:] = np.array([lossv], np.float64).view(np.int32)
            mine = torch.from_numpy(pack).to(tdev)
            allp = [torch.zeros_like(mine) for _ in range(world)]
            dist.all_gather(allp, mine, group=group)
            for r in range(world):
                p = allp[r].cpu().numpy()
                cnt = int(p[0])
                if cnt and r != rank:
                    backend.set_rows(p[1:1 + cnt].view(np.uint32),
                                     p[1 + bmax:1 + bmax + cnt * d].view(np.float32).reshape(cnt, d))
                if cfg.monitor_loss and cnt:
                    epoch_loss += float(p[-2:].copy().view(np.float64)[0])
        if counters is not None:
            counters.attractive_evals += int(g.num_edges())
            counters.repulsive_evals += n * s
        if cfg.monitor_loss:
            losses.append(epoch_loss)
    return losses
