import sys, numpy as np, time
sys.path.insert(0, '.')
exec(open('tools/_scratch/sat_check.py').read().split("x = np.load('tests/golden")[0])
def sat_gap(Rw, tw, la, pbx):
    # vectorized over n: max separation gap over 15 axes (unnormalised cross axes normalised here)
    A = np.einsum('nij,kj->nki', Rw, la[:, 6:15].reshape(-1, 3, 3)[0] if False else None) if False else None
    return None
x = np.load('tests/golden/late_states_shadow_drill.npz')['x']
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
fps = []
tot = 0
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    noise = rng.choice([0.002, 0.005, 0.01, 0.02])
    xs = x.copy()
    xs[:, 9:12] += rng.normal(size=(len(x), 3)) * noise
    xs[:, 12:] += rng.normal(size=(len(x), x.shape[1] - 12)) * 0.05
    world = G.forward_kinematics(hand, xs)
    n = world.shape[0]
    links = np.tile(np.repeat(np.arange(L), P), n); parts = np.tile(np.arange(P), n * L)
    poses = np.repeat(world.reshape(n * L, 12), P, axis=0)
    ref = O.signed_distance(hand, obj, links, parts, poses)
    tot += len(links)
    for t in np.where(ref[:, 0] < 0)[0]:
        Rw = poses[t, :9].reshape(3, 3).T; tw = poses[t, 9:]
        la, pbx = lb[links[t]], pb[parts[t]]
        A = (Rw @ la[6:15].reshape(3, 3).T).T; B = pbx[6:15].reshape(3, 3)
        hv = (Rw @ lv[lvb[links[t]]:lvb[links[t] + 1]].T).T + tw
        pvv = pv[pvb[parts[t]]:pvb[parts[t] + 1]]
        axes = [A[i] for i in range(3)] + [B[j] for j in range(3)] + [np.cross(A[i], B[j]) for i in range(3) for j in range(3)]
        best = -1
        for Lx in axes:
            nl = np.linalg.norm(Lx)
            if nl < 1e-9: continue
            Lx = Lx / nl
            a, b = hv @ Lx, pvv @ Lx
            best = max(best, a.min() - b.max(), b.min() - a.max())
        if best > 0:
            fps.append((best, ref[t, 0], links[t], parts[t]))
print('pairs', tot, 'false positives', len(fps))
for f in sorted(fps, reverse=True)[:15]: print('gap %.6f refd %.6f link %d part %d' % f)
