"""World-size-2 coverage of the multi-GPU path on CPU (gloo).

Each rank takes its contiguous shard of one global init_poses stream, runs
the per-rank synthesis (here the CPU oracle stands in for the per-GPU
engine, which needs a device) and the ranks all_gather the records. The
gathered batch must be bitwise identical to a single-process run over the
whole batch: shards are independent and no collective touches the loop.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    import paper_2412_16490_b200 as G
    from paper_2412_16490_b200.dist import synthesize_sharded
    from oracle import oracle as O

    dist.init_process_group("gloo", rank=rank, world_size=world)
    hand = G.HandModel.builtin()
    obj = G.make_primitive("sphere", 0.1)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 5, 17
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 12, 6, 6
    out = synthesize_sharded(hand, obj, cfg, rank, world, lambda x0: O.synthesize(hand, obj, cfg, x0, workers=2))
    if rank == 0:
        np.savez(Path(out_dir) / "gathered.npz", **{k: getattr(out, k) for k in ("x", "x_p", "x_s",
                                                                                  "energy_total", "failed")})
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_partition_the_batch():
    from paper_2412_16490_b200.dist import shard_range
    for batch in (1, 5, 4096, 32768, 1001):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(r, world, batch) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == batch
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1


def test_two_rank_gloo_gather_equals_single_process(tmp_path, G, O):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    got = np.load(tmp_path / "gathered.npz")
    hand = G.HandModel.builtin()
    obj = G.make_primitive("sphere", 0.1)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 5, 17
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 12, 6, 6
    ref = O.synthesize(hand, obj, cfg, G.init_poses(hand, obj, 5, 17), workers=1)
    for k in ("x", "x_p", "x_s", "energy_total", "failed"):
        assert np.array_equal(got[k], getattr(ref, k), equal_nan=True), k
