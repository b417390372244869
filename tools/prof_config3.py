"""Kernel-class profile of BASELINE config 3 (Leap-like, 16 primitives x 1024 in one
multi-object batch) (dev tool)."""
import dataclasses
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2412_16490_b200 as G  # noqa: E402

hand = G.HandModel.from_file(ROOT / "paper_2412_16490_b200/assets/hands/leap_like.json")
objs = [G.make_primitive(s, sc) for s in ("sphere", "box", "cylinder", "capsule") for sc in (0.06, 0.08, 0.10, 0.12)]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = G.RunConfig()
eng = G.Engine(0)
eng.set_hand(hand)
eng.set_objects(objs)
x0 = np.concatenate([G.init_poses(hand, o, B, i, cfg.init) for i, o in enumerate(objs)])
idx = np.repeat(np.arange(len(objs), dtype=np.int32), B)
c = dataclasses.replace(cfg, batch=B * len(objs))
eng.synthesize_objects(c, x0, idx)
t = time.perf_counter()
eng.synthesize_objects(c, x0, idx)
dt = time.perf_counter() - t
print(f"config 3: {len(objs) * B / dt:.1f} grasps/s ({dt:.3f} s)")
eng.set_profiling(True)
eng.synthesize_objects(c, x0, idx)
prof = eng.profile()
print(json.dumps({k: round(v, 1) for k, v in prof["ms"].items()}), "total", round(sum(prof["ms"].values()), 1))
o = prof["ops"]
print(json.dumps({k: o[k] for k in ("point_queries", "plane_tests", "triangle_tests", "pairs_needed", "gjk_iters", "epa_iters", "epa_overflow", "epa_max_iters", "epa_long_jobs", "qp_column_sweeps")}))
