"""Data-parallel sharding of a synthesis batch over ranks (one process per GPU).

Grasps are independent (reference pipeline.cpp:444-446, batch-prefix
independence test_pipeline.cpp:414-420), so a global batch is split into
contiguous shards with no per-iteration collective; every rank draws the
same global init_poses stream and keeps its slice, and the results are
gathered once at the end. The same code path runs with NCCL on GPUs and
with gloo on CPU (tests/test_multigpu_gloo.py).
"""
from __future__ import annotations

from typing import Callable, Tuple

import numpy as np

from .api import RunConfig, SynthesisOutput, init_poses

FIELDS = ("x_p", "x", "x_s", "energy_total", "per_direction", "contact_forces", "contacts", "stage_energy",
          "failed", "qp_converged")


def shard_range(rank: int, world: int, global_batch: int) -> Tuple[int, int]:
    """Contiguous [start, stop) of rank in a balanced split."""
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_start_states(model, obj, cfg: RunConfig, rank: int, world: int) -> np.ndarray:
    """This rank's slice of the single global init_poses stream."""
    x0 = init_poses(model, obj, cfg.batch, cfg.seed, cfg.init)
    start, stop = shard_range(rank, world, cfg.batch)
    return np.ascontiguousarray(x0[start:stop])


def gather_outputs(local: SynthesisOutput, cfg: RunConfig, world: int, device=None) -> SynthesisOutput:
    """One all_gather of every record field: each rank packs its rows (all fields side by side,
    as float64 - the integer fields are small and exact in it) into one matrix padded to the
    largest shard, and every rank unpacks the global batch in input order."""
    import torch
    import torch.distributed as dist

    sizes = [shard_range(r, world, cfg.batch)[1] - shard_range(r, world, cfg.batch)[0] for r in range(world)]
    cap = max(sizes)
    cols = [getattr(local, name).reshape(local.failed.shape[0], -1) for name in FIELDS]
    widths = [c.shape[1] for c in cols]
    packed = np.zeros((cap, sum(widths)))
    packed[: local.failed.shape[0]] = np.concatenate([c.astype(np.float64) for c in cols], axis=1)
    t = torch.from_numpy(packed)
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    rows = np.concatenate([p.cpu().numpy()[:n] for p, n in zip(parts, sizes)])
    glob = SynthesisOutput.__new__(SynthesisOutput)
    off = 0
    for name, w in zip(FIELDS, widths):
        ref = getattr(local, name)
        block = rows[:, off:off + w].reshape((rows.shape[0],) + ref.shape[1:])
        setattr(glob, name, block.astype(ref.dtype))
        off += w
    return glob


def synthesize_sharded(model, obj, cfg: RunConfig, rank: int, world: int,
                       run_shard: Callable[[np.ndarray], SynthesisOutput], device=None) -> SynthesisOutput:
    """Shard -> run_shard(x0_slice) on this rank -> gather."""
    x0 = shard_start_states(model, obj, cfg, rank, world)
    local = run_shard(x0)
    return gather_outputs(local, cfg, world, device)
