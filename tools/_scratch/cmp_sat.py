import os, sys, numpy as np
sys.path.insert(0, '.')
import paper_2412_16490_b200 as G
hand = G.HandModel.from_file('paper_2412_16490_b200/assets/hands/shadow_like.json')
obj = G.load_object('paper_2412_16490_b200/assets/objects/drill_like.obj', 0.10)
cfg = G.RunConfig(); cfg.seed = 17; cfg.batch = 512
x0 = G.init_poses(hand, obj, 512, 17)
eng = G.Engine(0); eng.set_hand(hand); eng.set_object(obj)
out = eng.synthesize(cfg, x0)
np.save(sys.argv[1], np.concatenate([out.x, out.contacts.reshape(512, -1), out.energy_total[:, None]], axis=1))
