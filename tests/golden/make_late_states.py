"""Generates tests/golden/late_states_shadow_drill.npz: final hand states of a full-schedule
oracle run (shadow_like + drill_like @ 0.10, 16 grasps, seed 17).

These are test INPUTS for the pair parity test on late-stage geometry (near-contact link/part
pairs, where the reference's GJK cycles until its iteration cap); expected outputs are always
recomputed by the oracle at test time. Run from the repo root: python tests/golden/make_late_states.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2412_16490_b200 as G  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main() -> None:
    hand = G.HandModel.from_file(ROOT / "paper_2412_16490_b200/assets/hands/shadow_like.json")
    obj = G.load_object(ROOT / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)
    cfg = G.RunConfig()
    cfg.seed = 17
    n = 16
    cfg.batch = n
    x0 = G.init_poses(hand, obj, n, 17)
    out = O.synthesize(hand, obj, cfg, x0, workers=16)
    np.savez_compressed(Path(__file__).with_name("late_states_shadow_drill.npz"), x=out.x, x0=x0,
                        failed=out.failed)
    print("saved", out.x.shape, "failed", int((out.failed != 0).sum()))


if __name__ == "__main__":
    main()
