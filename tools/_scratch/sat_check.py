import sys, numpy as np
sys.path.insert(0, '.')
import paper_2412_16490_b200 as G
from oracle import oracle as O
from paper_2412_16490_b200.api import _arr
hand = G.HandModel.from_file('paper_2412_16490_b200/assets/hands/shadow_like.json')
obj = G.load_object('paper_2412_16490_b200/assets/objects/drill_like.obj', 0.10)
hd, od = hand.desc, obj.desc
L, P = hand.n_links, obj.n_parts
lobb = _arr(hd.link_obb, 15 * L, np.float64).reshape(L, 15); lv = _arr(hd.verts, 3 * hd.n_verts, np.float64).reshape(-1, 3)
lvb = _arr(hd.link_vert_begin, L + 1, np.int32)
pobb = _arr(od.part_obb, 15 * P, np.float64).reshape(P, 15); pv = _arr(od.verts, 3 * od.n_verts, np.float64).reshape(-1, 3)
pvb = _arr(od.part_vert_begin, P + 1, np.int32)
def boxes(obb, verts, vb):
    out = obb.copy()
    for i in range(len(obb)):
        ax = obb[i, 6:15].reshape(3, 3)  # rows = columns of col-major matrix = axes
        r = verts[vb[i]:vb[i+1]] - obb[i, :3]
        h = np.abs(r @ ax.T).max(axis=0)
        out[i, 3:6] = h * (1 + 1e-12) + 1e-12
    return out
lb, pb = boxes(lobb, lv, lvb), boxes(pobb, pv, pvb)
def sep(la, Rw, tw, pbx, margin=1e-9):
    A = (Rw @ la[6:15].reshape(3, 3).T).T; B = pbx[6:15].reshape(3, 3)
    ah, bh = la[3:6], pbx[3:6]
    T = pbx[:3] - (Rw @ la[:3] + tw)
    R = A @ B.T; AR = np.abs(R) + 1e-12; t = A @ T
    for i in range(3):
        if abs(t[i]) > ah[i] + bh @ AR[i] + margin: return True
    for j in range(3):
        if abs(t @ R[:, j]) > ah @ AR[:, j] + bh[j] + margin: return True
    for i in range(3):
        i1, i2 = (i+1) % 3, (i+2) % 3
        for j in range(3):
            j1, j2 = (j+1) % 3, (j+2) % 3
            ra = ah[i1]*AR[i2, j] + ah[i2]*AR[i1, j]; rb = bh[j1]*AR[i, j2] + bh[j2]*AR[i, j1]
            if abs(t[i2]*R[i1, j] - t[i1]*R[i2, j]) > ra + rb + margin: return True
    return False
x = np.load('tests/golden/late_states_shadow_drill.npz')['x']
rng = np.random.default_rng(0)
xs = [x] + [x + np.concatenate([np.zeros((len(x), 9)), rng.normal(size=(len(x), 3)) * 0.01, np.zeros((len(x), x.shape[1]-12))], 1) for _ in range(10)]
world = G.forward_kinematics(hand, np.concatenate(xs))
n = world.shape[0]
links = np.tile(np.repeat(np.arange(L), P), n); parts = np.tile(np.arange(P), n * L)
poses = np.repeat(world.reshape(n * L, 12), P, axis=0)
ref = O.signed_distance(hand, obj, links, parts, poses)
bad = 0; nsep = 0
for t in range(len(links)):
    Rw = poses[t, :9].reshape(3, 3).T; tw = poses[t, 9:]
    if sep(lb[links[t]], Rw, tw, pb[parts[t]]):
        nsep += 1
        if ref[t, 0] <= 0: bad += 1; print('BAD', t, links[t], parts[t], ref[t, 0])
print('pairs', len(links), 'sat separated', nsep, 'bad', bad)

# state 278 of sat_energy.py
rng = np.random.default_rng(0)
xs = np.concatenate([x] + [x + np.concatenate([np.zeros((len(x), 9)), rng.normal(size=(len(x), 3)) * 0.003, np.zeros((len(x), x.shape[1]-12))], 1) for _ in range(30)])
xr = xs[278:279]
world = G.forward_kinematics(hand, xr)
links = np.repeat(np.arange(L), P); parts = np.tile(np.arange(P), L)
poses = np.repeat(world.reshape(L, 12), P, axis=0)
ref = O.signed_distance(hand, obj, links, parts, poses)
for t in range(len(links)):
    Rw = poses[t, :9].reshape(3, 3).T; tw = poses[t, 9:]
    s = sep(lb[links[t]], Rw, tw, pb[parts[t]])
    if s and ref[t, 0] <= 1e-3: print('sep but close', links[t], parts[t], ref[t, 0])
    if ref[t, 0] < 0: print('penetrating', links[t], parts[t], ref[t, 0], 'sat', s)

print('part3 obb', pobb[3]); print('part3 box', pb[3])
ax = pobb[3, 6:15].reshape(3, 3); print('orth', ax @ ax.T)
print('link6 obb', lobb[6]); print('link6 box', lb[6]); axl = lobb[6, 6:15].reshape(3, 3); print('orth', axl @ axl.T)
print('link6 verts range', lv[lvb[6]:lvb[7]].min(0), lv[lvb[6]:lvb[7]].max(0))
print('part3 verts range', pv[pvb[3]:pvb[4]].min(0), pv[pvb[3]:pvb[4]].max(0))

t = 6 * P + 3
Rw = poses[t, :9].reshape(3, 3).T; tw = poses[t, 9:]
la, pbx = lb[6], pb[3]
def corners(c, h, axes):
    out = []
    for sx in (-1, 1):
        for sy in (-1, 1):
            for sz in (-1, 1):
                out.append(c + sx * h[0] * axes[0] + sy * h[1] * axes[1] + sz * h[2] * axes[2])
    return np.array(out)
A = (Rw @ la[6:15].reshape(3, 3).T).T; B = pbx[6:15].reshape(3, 3)
ca = corners(Rw @ la[:3] + tw, la[3:6], A); cb = corners(pbx[:3], pbx[3:6], B)
axes = [A[i] for i in range(3)] + [B[j] for j in range(3)] + [np.cross(A[i], B[j]) for i in range(3) for j in range(3)]
for k, L in enumerate(axes):
    if np.linalg.norm(L) < 1e-9: continue
    pa, pbb = ca @ L, cb @ L
    gap = max(pa.min() - pbb.max(), pbb.min() - pa.max())
    if gap > 0: print('axis', k, 'separates by', gap)
print('Rw det', np.linalg.det(Rw), 'A orth', A @ A.T)
# link hull in world vs part verts: true min distance sanity via hull vertices
hv = (Rw @ lv[lvb[6]:lvb[7]].T).T + tw
print('link verts inside part box?', ((np.abs((hv - pbx[:3]) @ B.T) <= pbx[3:6]).all(1)).sum())

L6 = np.cross(A[0], B[0]); L6 /= np.linalg.norm(L6)
pv3 = pv[pvb[3]:pvb[4]]
print('hull projections link', (hv @ L6).min(), (hv @ L6).max(), 'part', (pv3 @ L6).min(), (pv3 @ L6).max())
print('oracle result', ref[t])
