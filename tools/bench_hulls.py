"""Load-time convex parts: device builder (grasp_build_convex_parts, one thread
per part) vs the host builder (ObjectModel.from_points, one part after another) on many random
point clouds (dev tool). Prints one JSON line."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2412_16490_b200 as G  # noqa: E402

n_parts = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
n_pts = int(sys.argv[2]) if len(sys.argv) > 2 else 300
rng = np.random.default_rng(0)
parts = [rng.normal(size=(n_pts, 3)) * rng.uniform(0.01, 0.05, 3) for _ in range(n_parts)]
G.build_convex_parts(parts[:64])  # warm-up (context, module load)
t = time.perf_counter()
dev = G.build_convex_parts(parts)
t_dev = time.perf_counter() - t
k = min(n_parts, 256)
t = time.perf_counter()
host = [G.ObjectModel.from_points([p]) for p in parts[:k]]
t_host = (time.perf_counter() - t) * n_parts / k
same = all(np.array_equal(d["vertices"], h.part_vertices(0)) and np.array_equal(d["faces"], h.part_faces(0))
           for d, h in zip(dev[:k], host))
print(json.dumps({"parts": n_parts, "points_per_part": n_pts, "device_s": round(t_dev, 4),
                  "device_parts_per_s": round(n_parts / t_dev, 1), "host_s_est": round(t_host, 3),
                  "host_parts_per_s": round(n_parts / t_host, 1), "host_sample_parts": k,
                  "bitwise_equal_on_sample": same, "faces_mean": float(np.mean([len(d["faces"]) for d in dev]))}))
