"""Diagnostic: closest_on_simplex on the GPU for the EPA triangles in tools/_scratch/epa_gpu.json."""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2412_16490_b200 import _native as N  # noqa: E402

rows = json.load(open("tools/_scratch/epa_gpu.json"))
w = np.ascontiguousarray(np.array([r["tri_w"] for r in rows]))
out = np.zeros((len(rows), 8))
dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
print("status", N.lib().grasp_debug_cos(len(rows), dp(w), dp(out)))
for r, o in zip(rows, out):
    k = int(o[0])
    print("isolated gpu:", k, o[1:1 + k], np.round(o[4:4 + k], 4), " in-epa gpu:", r["keep"][:r["nkeep"]],
          np.round(r["wts"][:r["nkeep"]], 4))
