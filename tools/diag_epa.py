"""Diagnostic: EPA internals on GPU for the pairs listed in gpurun_out/diag_pairs.npz."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2412_16490_b200 as G  # noqa: E402
from paper_2412_16490_b200 import _native as N  # noqa: E402


class EpaDebug(C.Structure):
    _fields_ = [("iters", C.c_int), ("nv", C.c_int), ("nf", C.c_int), ("v", C.c_int * 3), ("n", C.c_double * 3),
                ("d", C.c_double), ("tri_w", C.c_double * 9), ("tri_a", C.c_double * 9), ("wts", C.c_double * 3),
                ("keep", C.c_int * 3), ("nkeep", C.c_int)]


def run(fn, ctx_or_descs, links, parts, poses):
    n = len(links)
    out = np.zeros((n, 11))
    dbg = (EpaDebug * n)()
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))
    fn(*ctx_or_descs, n, ip(links), ip(parts), dp(poses), dp(out), C.cast(dbg, C.c_void_p))
    return out, dbg


if __name__ == "__main__":
    d = np.load("tools/_scratch/diag_pairs.npz")
    bad = d["bad"]
    links = np.ascontiguousarray(d["links"][bad].astype(np.int32))
    poses = np.ascontiguousarray(d["poses"][bad])
    parts = np.zeros(len(bad), np.int32)
    hand = G.HandModel.builtin()
    obj = G.make_primitive("sphere", 0.1)
    if len(sys.argv) > 1 and sys.argv[1] == "host":
        L = C.CDLL("/tmp/host_gjk.so")
        out, dbg = run(L.host_signed_distance, (C.byref(hand.desc), C.byref(obj.desc)), links, parts, poses)
        tag = "host"
    else:
        eng = G.Engine(0)
        eng.set_hand(hand)
        eng.set_object(obj)
        N.lib().grasp_debug_epa.restype = C.c_int
        out, dbg = run(N.lib().grasp_debug_epa, (eng._ctx,), links, parts, poses)
        tag = "gpu"
    rows = []
    for i in range(len(bad)):
        b = dbg[i]
        rows.append(dict(nv=b.nv, nf=b.nf, v=list(b.v), n=list(b.n), d=b.d, tri_w=list(b.tri_w), tri_a=list(b.tri_a),
                         wts=list(b.wts), keep=list(b.keep), nkeep=b.nkeep, out=out[i].tolist()))
    import json
    Path("gpurun_out").mkdir(exist_ok=True)
    Path(f"gpurun_out/epa_{tag}.json").write_text(json.dumps(rows))
    for r in rows[:4]:
        print(tag, r["nv"], r["nf"], r["v"], r["nkeep"], r["keep"], r["wts"], r["d"])
