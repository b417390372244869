"""Diagnostic: fine_contact_query GPU vs oracle mismatches (box object)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import paper_2412_16490_b200 as G  # noqa: E402
from oracle import oracle as O  # noqa: E402
from test_gpu_parity import gpu_fcq  # noqa: E402

hand = G.HandModel.builtin()
obj = G.make_primitive(sys.argv[1] if len(sys.argv) > 1 else "box", 0.1)
eng = G.Engine(0)
eng.set_hand(hand)
eng.set_object(obj)
x = G.init_poses(hand, obj, 128, 5)
x[:, 9:12] *= 0.6
ref = O.fine_contact_query(hand, obj, x)
got = gpu_fcq(eng, hand, x)
diff = np.abs(got[..., :10] - ref[..., :10]).max(axis=-1)
bad = np.argwhere(diff > 1e-9)
print("bad", len(bad))
for g, f in bad:
    r, q = ref[g, f], got[g, f]
    print(g, f, "d ref %.12g gpu %.12g" % (r[9], q[9]), "|cw-pw| ref %.9g gpu %.9g" % (
        np.linalg.norm(r[0:3] - r[3:6]), np.linalg.norm(q[0:3] - q[3:6])), "dn %.3g" % np.abs(r[6:9] - q[6:9]).max(),
        "dc %.3g" % np.abs(r[0:3] - q[0:3]).max())
