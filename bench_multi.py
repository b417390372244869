#!/usr/bin/env python
"""BASELINE config 3: Leap-like hand, 16 objects = {sphere, box, cylinder, capsule} x
{0.06, 0.08, 0.10, 0.12}, 1024 grasps each (seed = object index), full 300/100/100 schedule.

Sharded by object: under torchrun rank r takes objects r, r + N, ... (results do not depend on
the split; grasps are independent). One step = every object of this rank synthesized on its
GPU (one synthesize per object, device-resident start states and outputs). value = all ranks'
grasps / max-over-ranks device time. The CPU oracle is timed on a bounded sample (object 0).
Prints one JSON line.

    python bench_multi.py [--steps K] [--warmup W] [--grasps 1024]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench_multi.py --gpus N
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SHAPES = ("sphere", "box", "cylinder", "capsule")
SCALES = (0.06, 0.08, 0.10, 0.12)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--grasps", type=int, default=1024, help="grasps per object")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=8,
                    help="engine contexts (streams) per GPU, each driven by a host thread, objects round-robin")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2412_16490_b200 as G

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    hand = G.HandModel.from_file(ROOT / "paper_2412_16490_b200/assets/hands/leap_like.json")
    objects = [(i, s, sc) for i, (s, sc) in enumerate((s, sc) for s in SHAPES for sc in SCALES)]
    mine = [o for o in objects if o[0] % world == rank]
    cfg = G.RunConfig()
    B, D, m = args.grasps, hand.dims(), hand.n_tips
    n = m * cfg.contact.n_edges
    S = max(1, min(args.streams, len(mine)))
    engs = [G.Engine(local) for _ in range(S)]
    for e in engs:
        e.set_hand(hand)
    streams = [torch.cuda.ExternalStream(e.stream_handle(), device=dev) for e in engs]
    stream = streams[0]
    per_obj = []
    for idx, shape, scale in mine:
        obj = G.make_primitive(shape, scale)
        c = dataclasses.replace(cfg, batch=B, seed=idx)
        x0 = torch.from_numpy(G.init_poses(hand, obj, B, idx, cfg.init)).to(dev)
        per_obj.append((obj, c, x0))
    def make_outs():
        return {
            "x_p": torch.empty(B, D, dtype=torch.float64, device=dev),
            "x": torch.empty(B, D, dtype=torch.float64, device=dev),
            "x_s": torch.empty(B, D, dtype=torch.float64, device=dev),
            "energy_total": torch.empty(B, dtype=torch.float64, device=dev),
            "per_direction": torch.empty(B, 6, dtype=torch.float64, device=dev),
            "contact_forces": torch.empty(B, 6 * n, dtype=torch.float64, device=dev),
            "contacts": torch.empty(B, m * 12, dtype=torch.float64, device=dev),
            "stage_energy": torch.empty(B, 6, dtype=torch.float64, device=dev),
            "failed": torch.empty(B, dtype=torch.int32, device=dev),
            "qp_converged": torch.empty(B, 6, dtype=torch.int32, device=dev),
        }
    outs = [make_outs() for _ in range(S)]
    ptrs = [{k: v.data_ptr() for k, v in o.items()} for o in outs]
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    failed = []
    import threading

    def run_lane(k, record):
        e = engs[k]
        for j in range(k, len(per_obj), S):
            obj, c, x0 = per_obj[j]
            e.set_object(obj)
            e.synthesize_device(c, x0.data_ptr(), B, ptrs[k])
            if record:
                failed.append(int(outs[k]["failed"].sum().item()))

    def step(record=False):
        # every lane's stream starts after the main stream's start event
        start = torch.cuda.Event()
        start.record(streams[0])
        for st in streams[1:]:
            st.wait_event(start)
        threads = [threading.Thread(target=run_lane, args=(k, record)) for k in range(S)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        for st in streams[1:]:
            done = torch.cuda.Event()
            done.record(st)
            streams[0].wait_event(done)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    barrier()
    times = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        barrier()
        times.append(a.elapsed_time(b))
    ms = statistics.mean(times)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    total = len(objects) * B
    value = total / (ms_max * 1e-3)
    step(record=True)
    if rank == 0:
        line = {"metric": "grasps/sec (Leap-like, 16 objects x 1024)", "value": round(value, 3), "unit": "grasps/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 2),
                "higher_is_better": True, "scaling": "strong", "dtype": "f64",
                "data": "synthetic: init_poses(seed = object index) start states, generated hand, primitive objects",
                "config": {"workload": "BASELINE config 3", "objects": [f"{s}@{sc}" for s in SHAPES for sc in SCALES],
                           "grasps_per_object": B, "iters": [cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters,
                                                             cfg.pipeline.final_stage.iters],
                           "parallelism": f"objects sharded over {world} rank(s), {S} concurrent engine streams "
                                          "per GPU, no collective",
                           "l2": "flushed between timed steps (512 MiB device write)"},
                "failed_grasps_rank0": sum(failed)}
        if not args.no_cpu_baseline:
            from oracle import oracle as O
            obj = G.make_primitive(SHAPES[0], SCALES[0])
            threads = os.cpu_count() or 1
            ns = threads
            x0 = G.init_poses(hand, obj, ns, 0, cfg.init)
            t0 = time.perf_counter()
            O.synthesize(hand, obj, dataclasses.replace(cfg, batch=ns, seed=0), x0, workers=threads)
            dt = time.perf_counter() - t0
            line["cpu_baseline"] = {"value": round(ns / dt, 4), "unit": "grasps/s", "cores": threads, "kind": "port",
                                    "sample": f"{ns} grasps of object 0 (full schedule) on {threads} threads, {dt:.1f} s"}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
