"""Diagnostic: dump signed-distance pairs where GPU and oracle disagree."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import paper_2412_16490_b200 as G  # noqa: E402
from oracle import oracle as O  # noqa: E402
from test_gpu_parity import gpu_pairs, random_link_poses  # noqa: E402

hand = G.HandModel.builtin()
obj = G.make_primitive(sys.argv[1] if len(sys.argv) > 1 else "sphere", 0.1)
eng = G.Engine(0)
eng.set_hand(hand)
eng.set_object(obj)
rng = np.random.default_rng(7)
n = 3000
links = rng.integers(0, hand.n_links, size=n)
parts = np.zeros(n, dtype=np.int32)
poses = random_link_poses(rng, n, 0.16)
ref = O.signed_distance(hand, obj, links, parts, poses)
got = gpu_pairs(eng, links, parts, poses)
bad = np.where(np.abs(got[:, :10] - ref[:, :10]).max(axis=1) > 1e-9)[0]
print("bad", len(bad))
np.savez("gpurun_out/diag_pairs.npz", links=links, poses=poses, ref=ref, got=got, bad=bad)
for i in bad[:20]:
    print(i, "link", links[i], "d", ref[i, 0], got[i, 0], "flags", ref[i, 10], got[i, 10],
          "dpa", np.abs(got[i, 1:4] - ref[i, 1:4]).max(), "dn", np.abs(got[i, 7:10] - ref[i, 7:10]).max())
