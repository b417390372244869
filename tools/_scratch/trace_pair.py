import ctypes as C, sys, numpy as np
sys.path.insert(0, '.')
import paper_2412_16490_b200 as G
exec(open('tools/_scratch/sat_check.py').read().split("x = np.load('tests/golden")[0])
x = np.load('tests/golden/late_states_shadow_drill.npz')['x']
rng = np.random.default_rng(0)
xs = np.concatenate([x] + [x + np.concatenate([np.zeros((len(x), 9)), rng.normal(size=(len(x), 3)) * 0.003, np.zeros((len(x), x.shape[1]-12))], 1) for _ in range(30)])
world = G.forward_kinematics(hand, xs[278:279])
pose = np.ascontiguousarray(world[0, 6])
Lb = C.CDLL('tools/_scratch/host_gjk_trace.so')
out = np.zeros(11)
links = np.array([6], np.int32); parts = np.array([3], np.int32)
Lb.host_signed_distance(C.byref(hand.desc), C.byref(obj.desc), 1, links.ctypes.data_as(C.c_void_p), parts.ctypes.data_as(C.c_void_p), pose.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p), None)
print(out)
