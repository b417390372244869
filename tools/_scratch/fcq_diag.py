import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2412_16490_b200 as G
from oracle import oracle as O
from test_gpu_parity import gpu_fcq
hand = G.HandModel.from_file('paper_2412_16490_b200/assets/hands/shadow_like.json')
obj = G.load_object('paper_2412_16490_b200/assets/objects/drill_like.obj', 0.10)
eng = G.Engine(0); eng.set_hand(hand); eng.set_object(obj)
x = np.load('tests/golden/late_states_shadow_drill.npz')['x']
rng = np.random.default_rng(0)
xs = np.concatenate([x] + [x + np.concatenate([np.zeros((len(x), 9)), rng.normal(size=(len(x), 3)) * 0.003, np.zeros((len(x), x.shape[1]-12))], 1) for _ in range(30)])[256:320]
got = gpu_fcq(eng, hand, xs); ref = O.fine_contact_query(hand, obj, xs)
d = np.abs(got[..., 9] - ref[..., 9])
for i, f in zip(*np.where(d > 1e-9)):
    print(i + 256, f, got[i, f, 9], ref[i, f, 9], got[i, f, 10] if got.shape[-1] > 10 else None)
