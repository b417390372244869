#!/usr/bin/env python
"""Benchmark: batched bilevel grasp synthesis on B200 (BASELINE.json metric
"grasps/sec (Shadow, 1/2/4/8 B200) vs CPU ref").

One step = one full synthesize() over this rank's batch: the reference's
three-stage schedule (300 coarse / 100 fine / 100 final iterations), the
final cold-QP record and the squeeze pose, for every grasp. Workload =
BASELINE config 2 (Shadow-like hand, one multi-part convex mesh, 4096 grasps
per GPU); with torchrun each rank takes a contiguous shard of one global
init_poses stream (weak scaling: 4096 grasps per GPU, 32768 on 8 GPUs =
config 4). There is no per-iteration collective; results are gathered to
rank 0 once at the end (inside the e2e region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HAND = ROOT / "paper_2412_16490_b200" / "assets" / "hands" / "shadow_like.json"
OBJECT = ROOT / "paper_2412_16490_b200" / "assets" / "objects" / "drill_like.obj"
SCALE = 0.10
SEED = 17


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--batch", type=int, default=4096, help="grasps per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true", help="skip the config-3 / config-5 sub-results")
    ap.add_argument("--profile-json", default="", help="also dump the per-kernel profile here")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(G, batch_per_gpu, n_gpus):
    hand = G.HandModel.from_file(HAND)
    obj = G.load_object(OBJECT, SCALE)
    cfg = G.RunConfig()
    cfg.seed = SEED
    cfg.batch = batch_per_gpu * n_gpus
    return hand, obj, cfg


def config_dict(hand, obj, cfg, batch_per_gpu, n_gpus):
    return {
        "workload": "BASELINE config 2 (config 4 at 8 GPUs): shadow_like hand (22 DoF, 5 tips, 23 links) grasping "
                    "drill_like 6-part convex mesh (%d faces) at scale %.2f; full 300/100/100 schedule + final "
                    "record per grasp" % (len(obj.faces), SCALE),
        "hand": "assets/hands/shadow_like.json",
        "object": "assets/objects/drill_like.obj",
        "batch_per_gpu": batch_per_gpu,
        "global_batch": batch_per_gpu * n_gpus,
        "iters": [cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters],
        "seed": SEED,
        "l2": "flushed between timed steps (512 MiB device write); per-step working set ~40 MB",
        "parallelism": "dp%d: contiguous grasp shards, no per-iteration collective, one final gather" % n_gpus,
    }


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._thread = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.QUERY,
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([c.strip() for c in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._thread = threading.Thread(target=run, daemon=True)
        self._thread.start()

    def stop(self):
        self._stop.set()
        if self._thread:
            self._thread.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ncu --set full captures (profiles/) that give each kernel class's DRAM traffic per launch.
NCU_CAPTURES = {
    "pairs": "profiles/r02_ncu_pairs_list_full.json",
    "qp": "profiles/r02_ncu_qp_full.json",
    "point_query": "profiles/r02_ncu_point_query_full.json",
    "step_coarse": "profiles/r02_ncu_step_coarse_full.json",
    "step_mesh": "profiles/r02_ncu_step_mesh_full.json",
}


def class_flops(ops, hand, cfg, n_steps_iters):
    """Algorithmic flops per kernel class: SURVEY.md 8(d) constants x this run's op counters
    (FMA = 2). Step kernels: FK 160/link + proxy transform 20/proxy + self pair 10/pair +
    apply_step 5D per grasp-iteration (their point-Jacobian work is replaced by wrench sums)."""
    m = hand.n_tips
    n = m * cfg.contact.n_edges
    M = m + 1 + n
    L, S, D = hand.n_links, len(hand.proxies), hand.dims()
    nsp = int(getattr(hand, "n_sphere_pairs", 0))
    per_grasp_iter = 160.0 * L + 20.0 * S + 10.0 * nsp + 5.0 * D
    coarse_gi, mesh_gi = n_steps_iters
    return {
        "point_query": 7.0 * ops["plane_tests"] + 64.0 * ops["triangle_tests"],
        "qp": (45.0 * n + 6.0 * M + 100.0 + 3.0 * n) * ops["qp_column_sweeps"] + (80.0 * n + 400.0) * ops["qp_solves"],
        "pairs": 6.0 * ops["support_verts"] + 200.0 * ops["gjk_iters"] + 200.0 * ops["epa_iters"],
        "step_coarse": per_grasp_iter * coarse_gi,
        "step_mesh": per_grasp_iter * mesh_gi,
    }


def roofline(prof, hand, cfg, peak_tflops, batch):
    """Per kernel class: achieved = algorithmic flops / its CUDA-event time; the dominant class
    (by device time) is the headline block, every class is listed under "kernels"."""
    ms = prof["ms"]
    ops = prof["ops"]
    it = (cfg.pipeline.coarse.iters + 1, cfg.pipeline.fine.iters + cfg.pipeline.final_stage.iters + 2)
    flops = class_flops(ops, hand, cfg, (batch * it[0], batch * it[1]))
    total_ms = sum(ms.values())
    kernels = {}
    for cls, f in flops.items():
        t = ms.get(cls, 0.0)
        if t <= 0:
            continue
        achieved = f / (t * 1e-3) / 1e12
        traffic = None
        cap = NCU_CAPTURES.get(cls)
        if cap and (ROOT / cap).exists():
            traffic = json.loads((ROOT / cap).read_text()).get("traffic_bytes_per_launch")
        kernels[cls] = {"achieved": round(achieved, 3), "frac": round(achieved / peak_tflops, 4),
                        "ms": round(t, 2), "share_of_step": round(t / total_ms, 3), "traffic": traffic,
                        "traffic_source": cap if traffic is not None else None}
    dom = max((c for c in kernels), key=lambda c: kernels[c]["ms"])
    k = kernels[dom]
    return dom, {
        "bound": "fp64",
        "kernel": dom,
        "achieved": k["achieved"],
        "peak": round(peak_tflops, 3),
        "unit": "TFLOP/s",
        "frac": k["frac"],
        "traffic": k["traffic"],
        "traffic_source": (k["traffic_source"] + " (dram__bytes_read.sum + dram__bytes_write.sum, bytes per "
                           "launch)") if k["traffic_source"] else None,
        "share_of_step": k["share_of_step"],
        "peak_source": "measured fp64 FMA micro-benchmark on this GPU (MEASURED_PEAKS.json has no fp64 entry)",
        "flop_model": "SURVEY 8(d): plane test 7, closest-on-triangle 64, ADMM column-sweep 45n+6M+100+3n, "
                      "QP setup 80n+400, support vertex 6, GJK/EPA iteration 200; step kernels FK 160/link, "
                      "proxy 20, self pair 10, apply_step 5D per grasp-iteration",
        "kernels": kernels,
        "kernel_ms": {c: round(v, 2) for c, v in ms.items()},
        "ops": ops,
    }


def cpu_baseline(G, hand, obj, cfg, threads):
    """The oracle port on the host: 4 grasps per host thread on all threads (the reference's
    strided std::thread scheme, pipeline.cpp:443-455), plus a workers = 1 figure on 2 grasps."""
    from oracle import oracle as O
    n_grasps = 4 * threads
    x0 = G.init_poses(hand, obj, n_grasps, SEED)
    t0 = time.perf_counter()
    O.synthesize(hand, obj, cfg, x0, workers=threads)
    dt = time.perf_counter() - t0
    t1 = time.perf_counter()
    O.synthesize(hand, obj, cfg, x0[:2], workers=1)
    dt1 = time.perf_counter() - t1
    return {"value": round(n_grasps / dt, 4), "unit": "grasps/s", "cores": threads, "kind": "port",
            "sample": "%d grasps (full schedule) of the same workload on %d host threads, %.1f s" % (
                n_grasps, threads, dt),
            "workers_1": {"value": round(2 / dt1, 4), "unit": "grasps/s", "cores": 1,
                          "sample": "2 grasps (full schedule) on one host thread, %.1f s" % dt1}}


def run_reference(args):
    """--impl reference: the reference algorithm's CPU implementation (the
    fp64 oracle port; the C++ reference needs Eigen3 and does not build
    here), all host threads, bounded sample per step. Rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import paper_2412_16490_b200 as G
    hand, obj, cfg = workload(G, args.batch, args.gpus)
    threads = os.cpu_count() or 1
    # two grasps per host thread (strided as in pipeline.cpp:443-455), so a step is
    # not just the slowest single grasp, and 20 steps still finish in a few minutes
    per_step = 2 * threads
    from oracle import oracle as O
    x0 = G.init_poses(hand, obj, per_step, SEED)
    for _ in range(args.warmup):
        O.synthesize(hand, obj, cfg, x0[: max(1, threads // 4)], workers=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.synthesize(hand, obj, cfg, x0, workers=threads)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.mean(times)
    value = per_step / (ms * 1e-3)
    line = {
        "metric": "grasps/sec", "value": round(value, 4), "unit": "grasps/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (init_poses seed 17)",
        "impl": "reference",
        "config": config_dict(hand, obj, cfg, args.batch, args.gpus),
        "cpu_baseline": {"value": round(value, 4), "unit": "grasps/s", "cores": threads, "kind": "port",
                         "sample": "%d grasps per step (two per host thread), full schedule" % per_step},
        "e2e": {"value": round(value, 4), "unit": "grasps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2412_16490_b200 as G
    from paper_2412_16490_b200 import _native as N

    rank, world, local = dist_env()
    if world != args.gpus:
        args.gpus = world if world > 1 else args.gpus
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    hand, obj, cfg = workload(G, args.batch, world)
    B, D, m = args.batch, hand.dims(), hand.n_tips
    n = m * cfg.contact.n_edges

    # One global init_poses stream; this rank's contiguous shard (dist.py).
    from paper_2412_16490_b200.dist import shard_start_states, synthesize_sharded
    x0_host = shard_start_states(hand, obj, cfg, rank, world)
    import dataclasses
    shard_cfg = dataclasses.replace(cfg, batch=B)

    eng = G.Engine(local)
    eng.set_option("graphs", 1)  # one context per GPU: the synthesis replays as one CUDA graph
    eng.set_hand(hand)
    eng.set_object(obj)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=dev)

    x0 = torch.from_numpy(x0_host).to(dev)
    outs = {
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
    ptrs = {k: v.data_ptr() for k, v in outs.items()}
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        eng.synthesize_device(shard_cfg, x0.data_ptr(), B, ptrs)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    barrier()

    # ---- device-resident timed region (value)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = eng.launch_count()
    ev = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        ev.append((a, b))
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    launches = eng.launch_count() - launches0
    clk = clocks.stop()
    ms = statistics.mean(step_ms)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = B * world / (ms_max * 1e-3)

    # ---- end-to-end through the C ABI with host buffers (value e2e):
    # init_poses (global stream, this rank's slice) + grasp_synthesize with
    # host buffers + (N > 1) one all_gather of every record field.
    import ctypes as C
    host_out = G.SynthesisOutput(B, D, m, cfg.contact.n_edges)

    def run_shard(x0_shard):
        s = host_out.as_struct()
        N.check(N.lib().grasp_synthesize(eng._ctx, C.byref(shard_cfg.to_params()), B,
                                         np.ascontiguousarray(x0_shard).ctypes.data_as(C.POINTER(C.c_double)),
                                         C.byref(s)))
        return host_out

    e2e_times = []
    for _ in range(max(1, args.steps)):
        barrier()
        t0 = time.perf_counter()
        if world > 1:
            synthesize_sharded(hand, obj, cfg, rank, world, run_shard, device=dev)
            torch.cuda.synchronize(dev)
        else:
            run_shard(shard_start_states(hand, obj, cfg, rank, world))
        e2e_times.append(time.perf_counter() - t0)
    e2e_t = torch.tensor([statistics.mean(e2e_times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = B * world / float(e2e_t.item())
    h2d = B * D * 8
    d2h = sum(a.nbytes for a in (host_out.x_p, host_out.x, host_out.x_s, host_out.energy_total,
                                 host_out.per_direction, host_out.contact_forces, host_out.contacts,
                                 host_out.stage_energy, host_out.failed, host_out.qp_converged))

    # ---- profiling pass (not timed): per-kernel share + roofline
    rl = None
    prof = None
    if rank == 0:
        peak = C_double_fp64_peak(N, local)
        eng.set_profiling(True)
        step()
        torch.cuda.synchronize(dev)
        prof = eng.profile()
        eng.set_profiling(False)
        _, rl = roofline(prof, hand, shard_cfg, peak, B)
        if args.profile_json:
            Path(args.profile_json).write_text(json.dumps({"profile": prof, "fp64_peak_tflops": peak,
                                                            "step_ms": step_ms}, indent=1))

    if rank == 0:
        failed = int((outs["failed"] != 0).sum().item())
        line = {
            "metric": "grasps/sec", "value": round(value, 3), "unit": "grasps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: init_poses(seed 17) start states, generated hand/object assets",
            "config": config_dict(hand, obj, cfg, B, world),
            "e2e": {"value": round(e2e_value, 3), "unit": "grasps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": "init_poses + grasp_synthesize (C ABI, host buffers)" + (
                        " + NCCL all_gather of every record field" if world > 1 else "")},
            "gpu_launches": launches,
            "clocks": clk,
            "failed_grasps": failed,
        }
        if rl:
            line["roofline"] = rl
        if world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            line["cpu_baseline"] = cpu_baseline(G, hand, obj, cfg, threads)
        if world == 1 and not args.no_other_configs:
            line["other_configs"] = other_configs(not args.no_cpu_baseline)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def other_configs(cpu=True):
    """The other BASELINE configs measured in the same run (not the headline): config 3 (Leap-like,
    16 objects x 1024 in one multi-object batch, bench_multi.py) and config 5 (batched lower-level
    QP at 256k columns, cold as BASELINE defines it and warm-started, bench_qp.py)."""
    import bench_multi
    import bench_qp
    out = {}
    c3 = bench_multi.run(steps=2, warmup=1, mode="single", cpu=cpu)
    out["config3"] = {k: c3[k] for k in ("metric", "value", "unit", "ms_per_step", "gpu_launches_per_step",
                                         "failed_grasps") if k in c3}
    out["config3"]["config"] = c3["config"]
    if "cpu_baseline" in c3:
        out["config3"]["cpu_baseline"] = c3["cpu_baseline"]
    for name, warm in (("config5", False), ("config5_warm", True)):
        q = bench_qp.run(sizes=(256000,), steps=3, warmup=2, warm=warm, cpu=cpu and not warm)
        out[name] = {"metric": q["metric"], "value": q["value"], "unit": q["unit"], "result": q["results"][-1],
                     "config": q["config"]}
        if "cpu_baseline" in q:
            out[name]["cpu_baseline"] = q["cpu_baseline"]
    return out


def C_double_fp64_peak(N, device):
    import ctypes as C
    v = C.c_double()
    N.check(N.lib().grasp_measure_fp64_peak(device, C.byref(v)))
    return v.value


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
