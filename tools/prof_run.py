"""Short synthesis run for ncu captures (dev tool): Shadow-like + drill,
batch 1024, 20/10/10 iterations (argv: batch [coarse fine final])."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2412_16490_b200 as G  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
hand = G.HandModel.from_file(ROOT / "paper_2412_16490_b200/assets/hands/shadow_like.json")
obj = G.load_object(ROOT / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)
cfg = G.RunConfig()
cfg.seed = 17
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg.batch = batch
sched = [int(a) for a in sys.argv[2:5]] if len(sys.argv) > 4 else [20, 10, 10]
cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = sched
eng = G.Engine(0)
eng.set_hand(hand)
eng.set_object(obj)
k0 = eng.launch_count()
out = eng.synthesize(cfg, G.init_poses(hand, obj, batch, 17))
print("ok failed", int((out.failed != 0).sum()), "kernels", eng.launch_count() - k0)
