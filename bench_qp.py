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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=5)
    ap.add_argument("--sizes", default="1000,4000,16000,64000,256000")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-columns", type=int, default=6000, help="CPU oracle sample (columns)")
    args = ap.parse_args()
    import torch

    import paper_2412_16490_b200 as G
    from paper_2412_16490_b200 import _native as N
    from oracle import oracle as O

    m = args.m
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
    lib = N.lib()
    results = []
    for cols in [int(s) for s in args.sizes.split(",")]:
        g = max(1, cols // 6)
        frames = torch.from_numpy(random_frames(rng, g, m)).to(dev)
        X = torch.empty((g, 6, n), dtype=torch.float64, device=dev)
        Y = torch.empty((g, 6, M), dtype=torch.float64, device=dev)
        Z = torch.empty((g, 6, M), dtype=torch.float64, device=dev)
        it = torch.empty((g, 6), dtype=torch.int32, device=dev)
        conv = torch.empty((g, 6), dtype=torch.int32, device=dev)
        per = torch.empty((g, 6), dtype=torch.float64, device=dev)

        def step():
            N.check(lib.grasp_qp_batch(eng._ctx, C.byref(params), g, m,
                                       C.cast(C.c_void_p(frames.data_ptr()), C.POINTER(C.c_double)), None, None,
                                       C.cast(C.c_void_p(X.data_ptr()), C.POINTER(C.c_double)),
                                       C.cast(C.c_void_p(Y.data_ptr()), C.POINTER(C.c_double)),
                                       C.cast(C.c_void_p(Z.data_ptr()), C.POINTER(C.c_double)),
                                       C.cast(C.c_void_p(it.data_ptr()), C.POINTER(C.c_int)),
                                       C.cast(C.c_void_p(conv.data_ptr()), C.POINTER(C.c_int)),
                                       C.cast(C.c_void_p(per.data_ptr()), C.POINTER(C.c_double)), 1))

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        times = []
        for _ in range(args.steps):
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
                        "converged_frac": round(float(conv.float().mean().item()), 4)})
    # CPU oracle on a bounded sample (all host threads)
    threads = os.cpu_count() or 1
    gs = max(1, args.cpu_columns // 6)
    fr = random_frames(rng, gs, m)
    t0 = time.perf_counter()
    ref = O.qp_batch(cfg, fr, m, threads=threads)
    dt = time.perf_counter() - t0
    cpu = {"qp_columns_per_s": round(6 * gs / dt, 1),
           "admm_column_sweeps_per_s": round(float(np.asarray(ref["iters"]).sum()) / dt, 1),
           "cores": threads, "kind": "port", "sample": f"{6 * gs} columns (m={m}, cold) in {dt:.2f} s"}
    big = results[-1]
    print(json.dumps({"metric": "batched QP solves/sec (QP columns/s)", "value": big["qp_columns_per_s"],
                      "unit": "QP columns/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                      "higher_is_better": True, "dtype": "f64", "data": "synthetic: random contact frames",
                      "config": {"workload": "BASELINE config 5", "m": m, "k": k, "beta": cfg.energy.beta,
                                 "cold_start": True, "l2": "flushed between steps (512 MiB write)"},
                      "results": results, "cpu_baseline": cpu}))


if __name__ == "__main__":
    main()
