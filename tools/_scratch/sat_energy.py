import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2412_16490_b200 as G
from test_gpu_parity import gpu_energy, gpu_fcq
hand = G.HandModel.from_file('paper_2412_16490_b200/assets/hands/shadow_like.json')
obj = G.load_object('paper_2412_16490_b200/assets/objects/drill_like.obj', 0.10)
eng = G.Engine(0); eng.set_hand(hand); eng.set_object(obj)
x = np.load('tests/golden/late_states_shadow_drill.npz')['x']
rng = np.random.default_rng(0)
xs = np.concatenate([x] + [x + np.concatenate([np.zeros((len(x), 9)), rng.normal(size=(len(x), 3)) * 0.003, np.zeros((len(x), x.shape[1]-12))], 1) for _ in range(30)])
cfg = G.RunConfig()
out = []
for stage in (1, 2):
    anchors = np.random.default_rng(1).normal(size=(len(xs), hand.n_tips, 3)) * 0.05
    e, g = gpu_energy(eng, cfg, stage, xs, anchors=anchors)
    out.append(np.concatenate([e[:, None], g], 1))
out.append(gpu_fcq(eng, hand, xs).reshape(len(xs), -1))
np.save(sys.argv[1], np.concatenate(out, 1))
