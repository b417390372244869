#!/usr/bin/env python
"""BASELINE config 3: Leap-like hand, 16 objects = {sphere, box, cylinder, capsule} x
{0.06, 0.08, 0.10, 0.12}, 1024 grasps each (seed = object index), full 300/100/100 schedule.

Sharded by object: under torchrun rank r takes objects r, r + N, ... (results do not depend on
the split; grasps are independent). One step = every object of this rank synthesized on its
GPU. Default mode "single": all of the rank's objects in ONE batch of one context
(grasp_ctx_set_objects + grasp_synthesize_objects: object id per grasp, one set of kernel
launches for the 16 x 1024 grasps), host buffers in and out, timed as wall clock around the
synchronous call (it includes the host-device copies). Mode "streams": one synthesize per object
on 8 concurrent engine contexts/streams, device-resident (the round-1 path). value = all ranks'
grasps / max-over-ranks step time. The CPU oracle is timed on a bounded sample (object 0).
Prints one JSON line.

    python bench_multi.py [--steps K] [--warmup W] [--grasps 1024] [--mode single|streams]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench_multi.py --gpus N
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SHAPES = ("sphere", "box", "cylinder", "capsule")
SCALES = (0.06, 0.08, 0.10, 0.12)


def _objects(G):
    return [(i, s, sc, G.make_primitive(s, sc)) for i, (s, sc) in enumerate((s, sc) for s in SHAPES for sc in SCALES)]


def run(steps=2, warmup=2, grasps=1024, mode="single", rank=0, world=1, local=0, cpu=True):
    """Returns the config-3 result dict for this rank's objects (value = this rank's grasps/s;
    the caller takes the max-time over ranks)."""
    import torch

    import paper_2412_16490_b200 as G

    dev = torch.device("cuda", local)
    hand = G.HandModel.from_file(ROOT / "paper_2412_16490_b200/assets/hands/leap_like.json")
    objects = _objects(G)
    mine = [o for o in objects if o[0] % world == rank]
    cfg = G.RunConfig()
    B, D, m = grasps, hand.dims(), hand.n_tips
    n = m * cfg.contact.n_edges
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    failed = [0]
    if mode == "single":
        eng = G.Engine(local)
        eng.set_option("graphs", 1)  # one context: the synthesis replays as one CUDA graph
        eng.set_hand(hand)
        eng.set_objects([o[3] for o in mine])
        x0 = np.concatenate([G.init_poses(hand, o[3], B, o[0], cfg.init) for o in mine])
        idx = np.repeat(np.arange(len(mine), dtype=np.int32), B)
        c = dataclasses.replace(cfg, batch=B * len(mine))

        def step(record=False):
            out = eng.synthesize_objects(c, x0, idx)
            if record:
                failed[0] = int((out.failed != 0).sum())

        launches = eng.launch_count
        detail = "all of this rank's objects in one batch of one context (grasp_synthesize_objects)"
    else:
        S = min(8, len(mine))
        engs = [G.Engine(local) for _ in range(S)]
        for e in engs:
            e.set_hand(hand)
        streams = [torch.cuda.ExternalStream(e.stream_handle(), device=dev) for e in engs]
        per_obj = []
        for i, _, _, obj in mine:
            per_obj.append((obj, dataclasses.replace(cfg, batch=B, seed=i),
                            torch.from_numpy(G.init_poses(hand, obj, B, i, cfg.init)).to(dev)))

        def make_outs():
            shapes = {"x_p": (B, D), "x": (B, D), "x_s": (B, D), "energy_total": (B,), "per_direction": (B, 6),
                      "contact_forces": (B, 6 * n), "contacts": (B, m * 12), "stage_energy": (B, 6)}
            o = {k: torch.empty(v, dtype=torch.float64, device=dev) for k, v in shapes.items()}
            o["failed"] = torch.empty(B, dtype=torch.int32, device=dev)
            o["qp_converged"] = torch.empty(B, 6, dtype=torch.int32, device=dev)
            return o

        outs = [make_outs() for _ in range(S)]
        ptrs = [{k: v.data_ptr() for k, v in o.items()} for o in outs]

        def lane(k, record):
            e = engs[k]
            for j in range(k, len(per_obj), S):
                obj, c, x0 = per_obj[j]
                e.set_object(obj)
                e.synthesize_device(c, x0.data_ptr(), B, ptrs[k])
                if record:
                    failed[0] += int(outs[k]["failed"].sum().item())

        def step(record=False):
            threads = [threading.Thread(target=lane, args=(k, record)) for k in range(S)]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
            torch.cuda.synchronize(dev)

        launches = lambda: sum(e.launch_count() for e in engs)
        detail = "one synthesize per object on %d concurrent engine contexts/streams" % S
    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    l0 = launches()
    times = []
    for _ in range(steps):
        flush.fill_(1.0)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize(dev)
        times.append(1e3 * (time.perf_counter() - t0))
    n_launch = (launches() - l0) // max(1, steps)
    step(record=True)
    ms = statistics.mean(times)
    res = {"metric": "grasps/sec (Leap-like, 16 objects x 1024)", "value": round(len(mine) * B / (ms * 1e-3), 3),
           "unit": "grasps/s", "ms_per_step": round(ms, 2), "steps": steps, "warmup": warmup,
           "higher_is_better": True, "dtype": "f64",
           "data": "synthetic: init_poses(seed = object index) start states, generated hand, primitive objects",
           "config": {"workload": "BASELINE config 3", "objects": [f"{s}@{sc}" for s in SHAPES for sc in SCALES],
                      "grasps_per_object": B, "mode": mode, "detail": detail,
                      "iters": [cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters],
                      "timing": "wall clock around each synchronous step (host buffers and copies included in "
                                "mode single)", "l2": "flushed between timed steps (512 MiB device write)"},
           "gpu_launches_per_step": int(n_launch), "failed_grasps": failed[0]}
    if cpu and rank == 0:
        from oracle import oracle as O
        obj = mine[0][3]
        threads = os.cpu_count() or 1
        ns = 2 * threads
        x0 = G.init_poses(hand, obj, ns, 0, cfg.init)
        t0 = time.perf_counter()
        O.synthesize(hand, obj, dataclasses.replace(cfg, batch=ns, seed=0), x0, workers=threads)
        dt = time.perf_counter() - t0
        res["cpu_baseline"] = {"value": round(ns / dt, 4), "unit": "grasps/s", "cores": threads, "kind": "port",
                               "sample": f"{ns} grasps of object 0 (full schedule) on {threads} threads, {dt:.1f} s"}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--grasps", type=int, default=1024, help="grasps per object")
    ap.add_argument("--mode", choices=("single", "streams"), default="single")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    res = run(args.steps, args.warmup, args.grasps, args.mode, rank, world, local, not args.no_cpu_baseline)
    ms_t = torch.tensor([res["ms_per_step"]], dtype=torch.float64, device=torch.device("cuda", local))
    if world > 1:
        dist.barrier()
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    if rank == 0:
        res["n_gpus"] = world
        res["scaling"] = "strong"
        res["ms_per_step"] = round(float(ms_t.item()), 2)
        res["value"] = round(len(SHAPES) * len(SCALES) * args.grasps / (float(ms_t.item()) * 1e-3), 3)
        res["config"]["parallelism"] = f"objects sharded over {world} rank(s), no collective"
        print(json.dumps(res))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
