"""Column/warp/block imbalance of the coarse-stage QP (dev tool): per traced
iteration, the sweeps a warp runs (max over its 6 columns) against the
columns' own sweeps, and a 4-warp block's (max over its 4 grasps)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2412_16490_b200 as G  # noqa: E402

hand = G.HandModel.from_file(ROOT / "paper_2412_16490_b200/assets/hands/shadow_like.json")
obj = G.load_object(ROOT / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)
cfg = G.RunConfig()
cfg.seed = 17
B = 4096
cfg.batch = B
cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 300, 100, 100
eng = G.Engine(0)
eng.set_hand(hand)
eng.set_object(obj)
its = [0, 1, 2, 5, 10, 50, 100, 200, 299]
_, t = eng.synthesize_traced(cfg, G.init_poses(hand, obj, B, 17), [(0, i) for i in its])
rows = []
for k, i in enumerate(its):
    q = t["qp_iters"][k].astype(np.float64)  # [B, 6]
    live = t["failed"][k] == 0
    q = q[live]
    col = q.sum()
    warp = 6 * q.max(axis=1).sum()
    nb = (len(q) // 4) * 4
    blk = 24 * q[:nb].max(axis=1).reshape(-1, 4).max(axis=1).sum()
    rows.append({"iter": i, "mean_col_sweeps": round(q.mean(), 1), "mean_warp_sweeps": round(q.max(axis=1).mean(), 1),
                 "col_over_warp": round(col / warp, 3), "col_over_block": round(q[:nb].sum() / blk, 3),
                 "capped_cols": int((q >= 500).sum())})
print(json.dumps(rows, indent=1))
