"""Quick GPU timing + kernel profile for a given hand/object/batch (dev tool)."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2412_16490_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--hand", default="shadow_like")
ap.add_argument("--object", default="drill_like")
ap.add_argument("--batch", type=int, default=512)
ap.add_argument("--coarse", type=int, default=300)
ap.add_argument("--fine", type=int, default=100)
ap.add_argument("--final", type=int, default=100)
ap.add_argument("--option", action="append", default=[], help="engine option name=value (repeatable)")
ap.add_argument("--shards", type=int, default=1, help="contexts on device 0 splitting the batch")
args = ap.parse_args()

hand = G.HandModel.builtin() if args.hand == "trident" else G.HandModel.from_file(
    ROOT / f"paper_2412_16490_b200/assets/hands/{args.hand}.json")
obj = G.load_object(ROOT / f"paper_2412_16490_b200/assets/objects/{args.object}.obj", 0.10) \
    if args.object == "drill_like" else G.make_primitive(args.object, 0.10)
cfg = G.RunConfig()
cfg.seed = 17
cfg.batch = args.batch
cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = args.coarse, args.fine, args.final
x0 = G.init_poses(hand, obj, args.batch, 17)
eng = G.Engine(0, devices=[0] * args.shards if args.shards > 1 else None)
eng.set_hand(hand)
eng.set_object(obj)
for o in args.option:
    k, v = o.split("=")
    eng.set_option(k, int(v))
eng.synthesize(cfg, x0[:64])
t = time.perf_counter()
out = eng.synthesize(cfg, x0)
dt = time.perf_counter() - t
print(f"{args.hand} x {args.object} batch {args.batch}: {dt:.3f} s -> {args.batch / dt:.1f} grasps/s; "
      f"failed {int((out.failed != 0).sum())}")
eng.set_profiling(True)
eng.synthesize(cfg, x0)
prof = eng.profile()
tot = sum(prof["ms"].values())
print(json.dumps({k: round(v, 1) for k, v in prof["ms"].items()}), "total ms", round(tot, 1))
print(json.dumps(prof["launches"]))
print(json.dumps(prof["ops"]))
