#!/usr/bin/env python
"""BASELINE config 5: batched lower-level QP micro-benchmark ("batched QP solves/sec").

W from random contact frames as in the reference's test_energy.cpp:82-91 (p on a 0.4-1.2 x
scale shell, n roughly inward), m contacts, k = 8 edges, beta = 10, gamma = 0.1 m, the 6
closure targets, cold start, default QpParams. N QP columns = N / 6 grasps. One step = one
grasp_qp_batch over device-resident frames and outputs (CUDA events on the engine's stream, L2
flushed between steps); the CPU oracle (qp_batch restated from qpsolve.cpp:45-120, all host
threads) is timed on a bounded sample of the same frames. Prints one JSON line.

    python bench_qp.py [--m 5] [--sizes 1000,4000,16000,64000,256000] [--steps 3] [--warmup 3]
"""
from __future__ import annotations

import argparse
import ctypes as C
import dataclasses
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def random_frames(rng, g, m, scale=0.1):
    u = rng.normal(size=(g, m, 3))
    u /= np.linalg.norm(u, axis=-1, keepdims=True)
    p = scale * rng.uniform(0.4, 1.2, size=(g, m, 1)) * u
    w = rng.normal(size=(g, m, 3))
    w /= np.linalg.norm(w, axis=-1, keepdims=True)
    n = -u + 0.4 * w
    n /= np.linalg.norm(n, axis=-1, keepdims=True)
    seed = np.where(np.abs(n[..., :1]) > 0.99, np.array([0.0, 1.0, 0.0]), np.array([1.0, 0.0, 0.0]))
    d = np.cross(n, seed)
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    e = np.cross(n, d)
    return np.concatenate([p, n, d, e], axis=-1)


def run(sizes=(1000, 4000, 16000, 64000, 256000), m=5, steps=3, warmup=3, cpu_columns=6000, warm=False,
        cpu=True):
    """Times grasp_qp_batch on device-resident data; returns the result dict (see module doc).
    warm=True: each batch is warm-started from a 20000-sweep solve of the same frames before a
    1e-3 m perturbation of the contact points, so columns freeze at check sweeps spread over
    10..500 (the pipeline's warm-started coarse QPs) instead of all running to the cap."""
    import torch

    import paper_2412_16490_b200 as G
    from paper_2412_16490_b200 import _native as N

    cfg = G.RunConfig()
    k = cfg.contact.n_edges
    n = m * k
    M = m + 1 + n
    eng = G.Engine(0)
    eng.set_hand(G.HandModel.builtin())
    dev = torch.device("cuda:0")
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    rng = np.random.default_rng(5)
    params = cfg.to_params()
    long_params = dataclasses.replace(cfg, qp=dataclasses.replace(cfg.qp, max_iters=20000)).to_params()
    lib = N.lib()
    dp = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_double)) if t is not None else None
    ip = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_int))
    results = []
    for cols in sizes:
        g = max(1, cols // 6)
        fr_np = random_frames(rng, g, m)
        frames = torch.from_numpy(fr_np).to(dev)
        X = torch.empty((g, 6, n), dtype=torch.float64, device=dev)
        Y = torch.empty((g, 6, M), dtype=torch.float64, device=dev)
        Z = torch.empty((g, 6, M), dtype=torch.float64, device=dev)
        it = torch.empty((g, 6), dtype=torch.int32, device=dev)
        conv = torch.empty((g, 6), dtype=torch.int32, device=dev)
        per = torch.empty((g, 6), dtype=torch.float64, device=dev)
        WX = WY = None
        if warm:
            N.check(lib.grasp_qp_batch(eng._ctx, C.byref(long_params), g, m, dp(frames), None, None, dp(X), dp(Y),
                                       dp(Z), ip(it), ip(conv), dp(per), 1))
            WX, WY = X.clone(), Y.clone()
            fr_np = fr_np.copy()
            fr_np[:, :, 0:3] += rng.normal(size=fr_np[:, :, 0:3].shape) * 1e-3
            frames = torch.from_numpy(fr_np).to(dev)

        def step():
            if warm:  # the solver overwrites its warm start with the snapshot; restart from the same one
                X.copy_(WX)
                Y.copy_(WY)
            N.check(lib.grasp_qp_batch(eng._ctx, C.byref(params), g, m, dp(frames), dp(X if warm else None),
                                       dp(Y if warm else None), dp(X), dp(Y), dp(Z), ip(it), ip(conv), dp(per), 1))

        for _ in range(warmup):
            with torch.cuda.stream(stream):
                step()
        torch.cuda.synchronize()
        times = []
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                step()
                b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        ms = float(np.median(times))
        sweeps = int(it.sum().item())
        results.append({"columns": 6 * g, "grasps": g, "ms": round(ms, 3),
                        "qp_columns_per_s": round(6 * g / (ms * 1e-3), 1),
                        "admm_column_sweeps_per_s": round(sweeps / (ms * 1e-3), 1),
                        "mean_sweeps": round(sweeps / (6 * g), 1),
                        "converged_frac": round(float(conv.float().mean().item()), 4)})
    out = {"metric": "batched QP solves/sec (QP columns/s)", "value": results[-1]["qp_columns_per_s"],
           "unit": "QP columns/s", "n_gpus": 1, "steps": steps, "warmup": warmup, "higher_is_better": True,
           "dtype": "f64", "data": "synthetic: random contact frames",
           "config": {"workload": "BASELINE config 5" + (" (warm-started variant)" if warm else ""), "m": m, "k": k,
                      "beta": cfg.energy.beta, "cold_start": not warm,
                      "l2": "flushed between steps (512 MiB write)"},
           "results": results}
    if cpu:
        # CPU oracle on a bounded sample (all host threads), cold start like the device run
        from oracle import oracle as O
        threads = os.cpu_count() or 1
        gs = max(1, cpu_columns // 6)
        fr = random_frames(rng, gs, m)
        t0 = time.perf_counter()
        ref = O.qp_batch(cfg, fr, m, threads=threads)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"qp_columns_per_s": round(6 * gs / dt, 1),
                               "admm_column_sweeps_per_s": round(float(np.asarray(ref["iters"]).sum()) / dt, 1),
                               "cores": threads, "kind": "port",
                               "sample": f"{6 * gs} columns (m={m}, cold) in {dt:.2f} s"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=5)
    ap.add_argument("--sizes", default="1000,4000,16000,64000,256000")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-columns", type=int, default=6000, help="CPU oracle sample (columns)")
    ap.add_argument("--warm", action="store_true", help="warm-started variant (columns freeze at check sweeps)")
    args = ap.parse_args()
    print(json.dumps(run([int(x) for x in args.sizes.split(",")], args.m, args.steps, args.warmup,
                         args.cpu_columns, args.warm)))


if __name__ == "__main__":
    main()
