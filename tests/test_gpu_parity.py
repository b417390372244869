"""GPU parity: the sm_100a kernels vs the fp64 CPU oracle on identical inputs.

Tolerances (fp64 on both sides; differences come only from operation order,
FMA contraction and device libm):
  * discrete selections (part index, inside/outside, witness part, EPA use,
    failure flags): exact, except where the oracle's own top-2 gap is within
    1e-12 (rounding-level tie), which is reported separately;
  * distances / points / normals: 1e-9 abs;
  * energies and gradients: 1e-7 relative (teacher-forced, one iteration);
  * QP: iteration counts exact, lambda 1e-7 abs (teacher-forced);
  * end-to-end after 20/10/10 iterations: |dx| <= 1e-5 (ulp-level FK differences from device
    sin/cos grow through the optimisation), stage energies 1e-4.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import use

pytestmark = pytest.mark.gpu


def gpu_points(engine, pts):
    from paper_2412_16490_b200 import _native as N
    from paper_2412_16490_b200.api import dptr
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    out = np.zeros((len(pts), 8))
    N.check(N.lib().grasp_point_to_mesh(engine._ctx, len(pts), dptr(pts), dptr(out)))
    return out


def gpu_pairs(engine, links, parts, poses):
    from paper_2412_16490_b200 import _native as N
    from paper_2412_16490_b200.api import dptr, iptr
    links = np.ascontiguousarray(links, dtype=np.int32)
    parts = np.ascontiguousarray(parts, dtype=np.int32)
    poses = np.ascontiguousarray(poses, dtype=np.float64)
    out = np.zeros((len(links), 11))
    N.check(N.lib().grasp_signed_distance(engine._ctx, len(links), iptr(links), iptr(parts), dptr(poses), dptr(out)))
    return out


def gpu_energy(engine, cfg, stage, x, anchors=None, warm_x=None, warm_y=None):
    from paper_2412_16490_b200 import _native as N
    from paper_2412_16490_b200.api import dptr
    x = np.ascontiguousarray(x, dtype=np.float64)
    e = np.zeros(len(x))
    g = np.zeros_like(x)
    anc = None if anchors is None else np.ascontiguousarray(anchors, dtype=np.float64)
    N.check(N.lib().grasp_total_energy(engine._ctx, C.byref(cfg.to_params()), stage, len(x), dptr(x), dptr(anc),
                                       dptr(warm_x), dptr(warm_y), dptr(e), dptr(g)))
    return e, g


def gpu_fcq(engine, hand, x):
    from paper_2412_16490_b200 import _native as N
    from paper_2412_16490_b200.api import dptr
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros((len(x), hand.n_tips, 11))
    N.check(N.lib().grasp_fine_contact_query(engine._ctx, len(x), dptr(x), dptr(out)))
    return out


def gpu_qp(engine, cfg, frames, m, warm_x=None, warm_y=None):
    from paper_2412_16490_b200 import _native as N
    from paper_2412_16490_b200.api import dptr, iptr
    frames = np.ascontiguousarray(frames, dtype=np.float64)
    g = frames.size // (m * 12)
    n = m * cfg.contact.n_edges
    M = m + 1 + n
    X, Y, Z = np.zeros((g, 6, n)), np.zeros((g, 6, M)), np.zeros((g, 6, M))
    it, conv, per = np.zeros((g, 6), np.int32), np.zeros((g, 6), np.int32), np.zeros((g, 6))
    N.check(N.lib().grasp_qp_batch(engine._ctx, C.byref(cfg.to_params()), g, m, dptr(frames), dptr(warm_x),
                                   dptr(warm_y), dptr(X), dptr(Y), dptr(Z), iptr(it), iptr(conv), dptr(per), 0))
    return dict(X=X, Y=Y, Z=Z, iters=it, converged=conv, per_direction=per)


def random_frames(rng, g, m, scale=0.1):
    """test_energy.cpp:82-91 style contacts: p on a shell, n roughly inward."""
    out = np.zeros((g, m, 12))
    for i in range(g):
        for c in range(m):
            u = rng.normal(size=3)
            u /= np.linalg.norm(u)
            p = scale * rng.uniform(0.4, 1.2) * u
            w = rng.normal(size=3)
            w /= np.linalg.norm(w)
            n = -u + 0.4 * w
            n /= np.linalg.norm(n)
            seed = np.array([0.0, 1.0, 0.0]) if abs(n[0]) > 0.99 else np.array([1.0, 0.0, 0.0])
            d = np.cross(n, seed)
            d /= np.linalg.norm(d)
            e = np.cross(n, d)
            out[i, c] = np.concatenate([p, n, d, e])
    return out


# ------------------------------------------------------------ point queries
@pytest.mark.parametrize("name", ["sphere", "box", "capsule"])
def test_point_queries_match_oracle(G, O, trident, engine, name):
    obj = G.make_primitive(name, 0.1)
    use(engine, trident, obj)
    rng = np.random.default_rng(5)
    pts = rng.normal(size=(4000, 3)) * 0.08
    ref = O.point_to_mesh(obj, pts)
    got = gpu_points(engine, pts)
    assert (got[:, 7] == ref[:, 7]).all()
    assert np.array_equal(got[:, 0] < 0, ref[:, 0] < 0)
    np.testing.assert_allclose(got[:, :7], ref[:, :7], atol=1e-9, rtol=0)


def test_point_queries_multipart(G, O, trident, engine):
    from test_models import three_box_obj
    obj = G.parse_object_text(three_box_obj(), 0.12, "three_boxes")
    use(engine, trident, obj)
    rng = np.random.default_rng(6)
    pts = rng.normal(size=(4000, 3)) * 0.1
    ref = O.point_to_mesh(obj, pts)
    got = gpu_points(engine, pts)
    assert (got[:, 7] == ref[:, 7]).all()
    np.testing.assert_allclose(got[:, :7], ref[:, :7], atol=1e-9, rtol=0)


def test_point_queries_drill_match_oracle(G, O, trident):
    """The drill mesh (6 parts, long strip faces) through the spatial point-query face order and
    the normal plane groups: points on shells from inside to 0.3 m out, plus a cloud near the
    surface; part index and values agree with the oracle's index-order scan."""
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    obj = G.load_object(root / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)
    eng = G.Engine(0)
    eng.set_hand(trident)
    eng.set_object(obj)
    rng = np.random.default_rng(12)
    d = rng.normal(size=(8000, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    pts = np.concatenate([d * rng.uniform(0.0, 0.3, 8000)[:, None], rng.normal(size=(4000, 3)) * 0.03])
    ref = O.point_to_mesh(obj, pts)
    got = gpu_points(eng, pts)
    assert (got[:, 7] == ref[:, 7]).all()
    assert np.array_equal(got[:, 0] < 0, ref[:, 0] < 0)
    np.testing.assert_allclose(got[:, :7], ref[:, :7], atol=1e-9, rtol=0)


WARM_START_SCRIPT = r'''
import ctypes as C, sys
import numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import paper_2412_16490_b200 as G
from paper_2412_16490_b200 import _native as N
from oracle import oracle as O
from test_gpu_parity import gpu_points, warm_start_checks
assert N.LIB_PATH.name == "libgrasp_b200_debug.so"
eng = G.Engine(0)
warm_start_checks(G, O, eng, G.HandModel.builtin())
print("warm start ok")
'''


def test_point_queries_warm_start_exact(tmp_path):
    """Warm-start seeds (the slot's previous closest face, used as an exact upper bound) must not
    change any result. Runs in a subprocess on the debug library (libgrasp_b200_debug.so: the
    engine plus grasp_debug_point_to_mesh_warm; the product library carries no debug surface)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    lib = root / "paper_2412_16490_b200/_lib/libgrasp_b200_debug.so"
    script = tmp_path / "warm.py"
    script.write_text(WARM_START_SCRIPT)
    r = subprocess.run([sys.executable, str(script), str(root)], capture_output=True, text=True,
                       env=dict(os.environ, GRASP_LIB=str(lib)), timeout=600)
    assert r.returncode == 0 and "warm start ok" in r.stdout, r.stdout + r.stderr


def warm_start_checks(G, O, engine, trident):
    """Random and nearest-face seeds vs no seed, bitwise, and vs the oracle, on the drill mesh."""
    from pathlib import Path
    from paper_2412_16490_b200 import _native as N
    from paper_2412_16490_b200.api import dptr, iptr
    root = Path(__file__).resolve().parents[1]
    obj = G.load_object(root / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)
    use(engine, trident, obj)
    rng = np.random.default_rng(11)
    pts = rng.normal(size=(6000, 3)) * 0.06 + np.array([0.02, 0.0, 0.0])
    nf = int(obj.desc.n_faces)
    cold = gpu_points(engine, pts)
    ref = O.point_to_mesh(obj, pts)
    assert (cold[:, 7] == ref[:, 7]).all()
    np.testing.assert_allclose(cold[:, :7], ref[:, :7], atol=1e-9, rtol=0)
    lib = N.lib()
    fn = getattr(lib, "grasp_debug_point_to_mesh_warm")
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_double)]
    for warm in (rng.integers(0, nf, size=len(pts)).astype(np.int32),
                 np.full(len(pts), -1, np.int32), np.full(len(pts), nf + 5, np.int32)):
        out = np.zeros((len(pts), 8))
        N.check(fn(engine._ctx, len(pts), dptr(pts), iptr(warm), dptr(out)))
        assert np.array_equal(out, cold), "warm start changed a point query"
    # seeds from the neighbours' answers (the solver's real use): shifted points
    pts2 = pts + rng.normal(size=pts.shape) * 1e-3
    cold2 = gpu_points(engine, pts2)
    out = np.zeros((len(pts), 8))
    seeds = np.full(len(pts), -1, np.int32)
    N.check(fn(engine._ctx, len(pts), dptr(pts), iptr(seeds), dptr(out)))
    # no face output on this surface; use random faces of the winning part instead
    fb = np.asarray(obj.part_face_begin)
    part = cold[:, 7].astype(int)
    seeds = (fb[part] + rng.integers(0, 1 << 30, size=len(pts)) % (fb[part + 1] - fb[part])).astype(np.int32)
    N.check(fn(engine._ctx, len(pts2), dptr(pts2), iptr(seeds), dptr(out)))
    assert np.array_equal(out, cold2)


# ---------------------------------------------------------------- GJK / EPA
def random_link_poses(rng, n, span):
    from scipy.spatial.transform import Rotation
    R = Rotation.random(n, random_state=int(rng.integers(1 << 30))).as_matrix()
    poses = np.zeros((n, 12))
    poses[:, :9] = R.transpose(0, 2, 1).reshape(n, 9)  # column-major
    poses[:, 9:] = rng.uniform(-span, span, size=(n, 3))
    return poses


def test_signed_distance_matches_oracle(G, O, trident, engine):
    obj = G.make_primitive("sphere", 0.1)
    use(engine, trident, obj)
    rng = np.random.default_rng(7)
    n = 3000
    links = rng.integers(0, trident.n_links, size=n)
    parts = np.zeros(n, dtype=np.int32)
    poses = random_link_poses(rng, n, 0.16)
    ref = O.signed_distance(trident, obj, links, parts, poses)
    got = gpu_pairs(engine, links, parts, poses)
    assert ((got[:, 10] % 2) == ref[:, 10]).all(), "EPA usage differs"
    assert (ref[:, 0] < 0).sum() > 100 and (ref[:, 0] > 0).sum() > 100
    # Poses are fed directly (no FK, no sin/cos): GJK and EPA follow the oracle's operation
    # order (--fmad=false), so every pair -- distance, witnesses, normal -- is bit-exact.
    assert np.array_equal(got[:, :10], ref[:, :10]), np.where((got[:, :10] != ref[:, :10]).any(axis=1))[0][:10]


def assert_witnesses_match_or_tie(got, ref, budget=0.0):
    """Witnesses agree except on EPA faces lying on a flat hull face, where
    the support scan has an exact tie (any point of the contact patch is a
    valid witness and rounding picks one). There both witness pairs must
    realize the same depth along the same normal."""
    bad = np.abs(got[:, 1:7] - ref[:, 1:7]).max(axis=1) > 1e-9
    assert (ref[bad, 10] == 1).all(), "witness mismatch outside EPA"
    assert bad.mean() <= budget, f"{bad.mean():.4f} of pairs hit witness ties"
    for r in (got[bad], ref[bad]):
        sep = r[:, 1:4] - r[:, 4:7]
        np.testing.assert_allclose(np.linalg.norm(sep, axis=1), -r[:, 0], atol=1e-9)
        np.testing.assert_allclose(np.einsum("ij,ij->i", sep, r[:, 7:10]), r[:, 0], atol=1e-9)


def test_signed_distance_late_stage_matches_oracle(G, O, engine):
    """Pairs from the final states of a full-schedule oracle run (tests/golden/
    make_late_states.py) and 1-2 mm shifts of them: near-contact geometry where the
    reference's GJK enters exact cycles and runs to its 128-iteration cap. The device
    fast-forwards those cycles (Brent detection on support-vertex keys); results must
    still be the oracle's."""
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    hand = G.HandModel.from_file(root / "paper_2412_16490_b200/assets/hands/shadow_like.json")
    obj = G.load_object(root / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)
    use(engine, hand, obj)
    x = np.load(root / "tests/golden/late_states_shadow_drill.npz")["x"]
    rng = np.random.default_rng(3)
    xs = [x]
    for _ in range(4):
        xp = x.copy()
        xp[:, 9:12] += rng.uniform(-2e-3, 2e-3, size=(len(x), 3))
        xs.append(xp)
    world = G.forward_kinematics(hand, np.concatenate(xs))  # (n, L, 12)
    n, L, _ = world.shape
    P = obj.n_parts
    links = np.tile(np.repeat(np.arange(L), P), n)
    parts = np.tile(np.arange(P), n * L)
    poses = np.repeat(world.reshape(n * L, 12), P, axis=0)
    ref = O.signed_distance(hand, obj, links, parts, poses)
    engine.set_profiling(True)
    try:
        got = gpu_pairs(engine, links, parts, poses)
        ops = engine.profile()["ops"]
    finally:
        engine.set_profiling(False)
    assert ops["gjk_cycle_jumps"] > 0, "no cycling pair exercised"
    assert ((got[:, 10] % 2) == ref[:, 10]).all(), "EPA usage differs"
    # identical poses: every pair (separated, capped-cycling and EPA) is bit-exact
    assert np.array_equal(got[:, :10], ref[:, :10]), np.where((got[:, :10] != ref[:, :10]).any(axis=1))[0][:10]


# ---------------------------------------------------------------------- QP
@pytest.mark.parametrize("m", [3, 4, 5])
def test_qp_batch_cold_capped_matches_oracle(G, O, engine, m):
    """Cold starts from test_energy.cpp:82-91-style frames: at beta = 10 none of these columns
    reaches the 1e-5 tolerance within 500 sweeps (the oracle agrees), so this pins the
    capped path: every column reports 500 sweeps, unconverged, and the same iterate."""
    cfg = G.RunConfig()
    rng = np.random.default_rng(100 + m)
    frames = random_frames(rng, 200, m)
    ref = O.qp_batch(cfg, frames, m)
    got = gpu_qp(engine, cfg, frames, m)
    assert (ref["iters"] == 500).all() and not ref["converged"].any()
    assert np.array_equal(got["iters"], ref["iters"]) and np.array_equal(got["converged"], ref["converged"])
    np.testing.assert_allclose(got["X"], ref["X"], atol=1e-7)
    np.testing.assert_allclose(got["per_direction"], ref["per_direction"], rtol=1e-7, atol=1e-9)


def warm_qp_batch(G, O, m, g, pert, seed):
    """Contacts on spheres of radius 3-12 cm with noisy inward normals, warm-started from a
    long (20k-sweep) cold solve of the unperturbed frames, then solved at default settings on
    frames moved by `pert` m: the columns freeze at every check sweep from 10 to 500
    (qpsolve.cpp:99-117), like the pipeline's warm-started coarse QPs."""
    rng = np.random.default_rng(seed)
    fr = np.zeros((g, m, 12))
    for i in range(g):
        r = rng.uniform(0.03, 0.12)
        for c in range(m):
            u = rng.normal(size=3)
            u /= np.linalg.norm(u)
            n = -u + rng.normal(size=3) * rng.uniform(0, 0.3)
            n /= np.linalg.norm(n)
            seed_v = np.array([0.0, 1.0, 0.0]) if abs(n[0]) > 0.99 else np.array([1.0, 0.0, 0.0])
            d = np.cross(n, seed_v)
            d /= np.linalg.norm(d)
            fr[i, c] = np.concatenate([r * u, n, d, np.cross(n, d)])
    long = G.RunConfig()
    long.qp.max_iters = 20000
    base = O.qp_batch(long, fr, m, threads=8)
    fr2 = fr.copy()
    fr2[:, :, 0:3] += rng.normal(size=fr2[:, :, 0:3].shape) * pert
    return fr2, np.ascontiguousarray(base["X"]), np.ascontiguousarray(base["Y"])


@pytest.mark.parametrize("m,pert", [(3, 1e-3), (4, 1e-3), (5, 1e-3), (4, 1e-2), (5, 1e-2)])
def test_qp_warm_freeze_semantics_match_oracle(G, O, engine, m, pert):
    """Discriminating QP parity: columns converge at different check sweeps, so the per-column
    freeze and snapshot (qpsolve.cpp:99-117) are compared, not just the 500-sweep cap. Sweep
    counts and convergence flags must be identical on every column; forces and duals agree to
    rounding (Woodbury sweep vs the reference's dense LLT)."""
    cfg = G.RunConfig()
    fr, wx, wy = warm_qp_batch(G, O, m, 300, pert, 7 + m)
    ref = O.qp_batch(cfg, fr, m, warm_x=wx.copy(), warm_y=wy.copy(), threads=8)
    got = gpu_qp(engine, cfg, fr, m, warm_x=wx.copy(), warm_y=wy.copy())
    its = ref["iters"].ravel()
    assert len(np.unique(its)) >= 10, "freeze sweeps not spread"
    assert ref["converged"].mean() >= 0.8
    mism = got["iters"] != ref["iters"]
    assert not mism.any(), (f"{mism.sum()} / {mism.size} columns froze at a different sweep",
                            got["iters"][mism][:8], ref["iters"][mism][:8])
    assert np.array_equal(got["converged"], ref["converged"])
    np.testing.assert_allclose(got["X"], ref["X"], atol=1e-7, rtol=0)
    np.testing.assert_allclose(got["Y"], ref["Y"], atol=1e-7, rtol=0)
    np.testing.assert_allclose(got["per_direction"], ref["per_direction"], rtol=1e-7, atol=1e-9)


# ------------------------------------------------------ teacher-forced energy
def test_coarse_energy_and_gradient_match_oracle(G, O, trident, engine):
    obj = G.make_primitive("sphere", 0.1)
    use(engine, trident, obj)
    cfg = G.RunConfig()
    x = G.init_poses(trident, obj, 64, 3)
    e_ref, g_ref = O.total_energy(trident, obj, cfg, 0, x)
    e_got, g_got = gpu_energy(engine, cfg, 0, x)
    np.testing.assert_allclose(e_got, e_ref, rtol=1e-7)
    scale = np.maximum(1.0, np.abs(g_ref).max(axis=1, keepdims=True))
    assert np.abs(g_got - g_ref).max() / scale.max() < 1e-6


def witness_ties(got, ref):
    """Per-(grasp, tip) witness rows that differ while distance and normal
    agree: flat-face EPA ties, decided by ulp-level differences in FK (device
    vs glibc sin/cos). Returns the boolean tie mask after asserting that no
    other kind of difference exists and that both witnesses are valid."""
    wdiff = np.abs(got[..., 0:6] - ref[..., 0:6]).max(axis=-1) > 1e-9
    np.testing.assert_allclose(got[..., 9], ref[..., 9], atol=1e-9)       # signed distance
    np.testing.assert_allclose(got[..., 6:9], ref[..., 6:9], atol=1e-9)   # normal
    assert (got[..., 10] == ref[..., 10]).all()                           # link
    for r in (got[wdiff], ref[wdiff]):
        # EPA witnesses realize the penetration along the normal.
        np.testing.assert_allclose(np.einsum("ij,ij->i", r[:, 0:3] - r[:, 3:6], r[:, 6:9]), r[:, 9], atol=1e-9)
    return wdiff


def gpu_fk(engine, hand, x):
    from paper_2412_16490_b200 import _native as N
    from paper_2412_16490_b200.api import dptr
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros((len(x), hand.n_links, 12))
    N.check(N.lib().grasp_device_forward_kinematics(engine._ctx, len(x), dptr(x), dptr(out)))
    return out


@pytest.mark.parametrize("hand_name", ["trident", "allegro_like", "shadow_like"])
def test_device_fk_matches_oracle(G, O, engine, hand_name):
    """Device FK (hand.cpp:108-153; correctly rounded sin/cos, reference operation order) vs the
    oracle's (glibc sin/cos): within 1e-15 m / 1e-15 rotation entries (8(d) asks 1e-6 m), and
    bitwise on the large majority of link transforms."""
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    hand = G.HandModel.builtin() if hand_name == "trident" else \
        G.HandModel.from_file(root / f"paper_2412_16490_b200/assets/hands/{hand_name}.json")
    obj = G.make_primitive("sphere", 0.1)
    use(engine, hand, obj)
    x = G.init_poses(hand, obj, 2000, 31)
    rng = np.random.default_rng(31)
    x[:, :9] += rng.normal(size=(len(x), 9)) * 0.05  # raw (unprojected) rotation blocks, as in the loop
    got = gpu_fk(engine, hand, x)
    ref = O.forward_kinematics(hand, x)
    assert np.abs(got - ref).max() <= 1e-15
    assert (got == ref).all(axis=2).mean() >= 0.95


def test_mesh_energy_and_gradient_match_oracle(G, O, trident, engine):
    """Teacher-forced mesh-stage total_energy (pipeline.cpp:175-210) at contact-rich states. With
    the device's link transforms fed to the oracle (world=...), every grasp agrees: energy 1e-12
    relative, gradient 1e-9 (the only differences left are summation order in the gradient)."""
    obj = G.make_primitive("sphere", 0.1)
    use(engine, trident, obj)
    cfg = G.RunConfig()
    rng = np.random.default_rng(9)
    x = G.init_poses(trident, obj, 64, 4)
    x[:, 9:12] *= 0.62  # pull the palms in so fingers touch / penetrate
    anchors = rng.normal(size=(64, trident.n_tips, 3)) * 0.05
    world = gpu_fk(engine, trident, x)
    for stage in (1, 2):
        e_ref, g_ref = O.total_energy(trident, obj, cfg, stage, x, anchors=anchors, world=world)
        e_got, g_got = gpu_energy(engine, cfg, stage, x, anchors=anchors)
        np.testing.assert_allclose(e_got, e_ref, rtol=1e-12, atol=0)
        row_err = np.abs(g_got - g_ref).max(axis=1) / np.abs(g_ref).max(axis=1)
        assert row_err.max() <= 1e-9, row_err.max()


def test_mesh_energy_late_stage_matches_oracle(G, O, engine):
    """Teacher-forced mesh-stage energies on late-stage Shadow/drill states
    (tests/golden/make_late_states.py + 3 mm shifts). The batch includes a pair the
    reference's GJK reports as overlapping although the hulls are 0.4 mm apart
    (coplanar 4-point simplex); the default engine computes every pair
    like the reference, so the spurious hinge term is reproduced."""
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    hand = G.HandModel.from_file(root / "paper_2412_16490_b200/assets/hands/shadow_like.json")
    obj = G.load_object(root / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)
    use(engine, hand, obj)
    x = np.load(root / "tests/golden/late_states_shadow_drill.npz")["x"]
    rng = np.random.default_rng(0)
    xs = np.concatenate([x] + [x + np.concatenate([np.zeros((len(x), 9)), rng.normal(size=(len(x), 3)) * 0.003,
                                                   np.zeros((len(x), x.shape[1] - 12))], 1) for _ in range(30)])
    xs = xs[256:320]  # includes state 278 (link 6 / part 3 spurious overlap)
    anchors = np.random.default_rng(1).normal(size=(len(xs), hand.n_tips, 3)) * 0.05
    cfg = G.RunConfig()
    world = gpu_fk(engine, hand, xs)
    e_ref, g_ref = O.total_energy(hand, obj, cfg, 1, xs, anchors=anchors, world=world)
    e_got, g_got = gpu_energy(engine, cfg, 1, xs, anchors=anchors)
    np.testing.assert_allclose(e_got, e_ref, rtol=1e-12, atol=0)
    assert (np.abs(g_got - g_ref).max(axis=1) / np.abs(g_ref).max(axis=1)).max() <= 1e-9
    # the spurious-overlap state also matches with the oracle's own FK
    e_own, _ = O.total_energy(hand, obj, cfg, 1, xs[278 - 256:279 - 256], anchors=anchors[278 - 256:279 - 256])
    assert abs(e_got[278 - 256] - e_own[0]) <= 1e-12 * abs(e_own[0]), "spurious-overlap state differs"


def test_eval_matches_oracle(G, O, engine):
    """Grasp evaluation on the device (eval.cpp:51-158) vs the oracle on
    late-stage Shadow/drill states: penetration / self-penetration depths and contact-distance
    consistency to 1e-6 mm, contact counts and success flags exact, gravity residuals to the
    QP tolerance."""
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    hand = G.HandModel.from_file(root / "paper_2412_16490_b200/assets/hands/shadow_like.json")
    obj = G.load_object(root / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)
    use(engine, hand, obj)
    d = np.load(root / "tests/golden/late_states_shadow_drill.npz")
    x = d["x"]
    x_s = np.array([G.squeeze_pose(hand, x[i], d["x0"][i]) for i in range(len(x))])
    x_s2 = x.copy()
    x_s2[:, 9:12] += 0.002
    xs_all = np.concatenate([x_s, x_s2, x])
    x_all = np.concatenate([x, x, x])
    cfg = G.RunConfig()
    ref = O.evaluate(hand, obj, cfg, x_all, xs_all)
    got = engine.evaluate(cfg, x_all, xs_all)
    np.testing.assert_allclose(got["pd_mm"], ref["pd_mm"], atol=1e-6, rtol=0)
    np.testing.assert_allclose(got["spd_mm"], ref["spd_mm"], atol=1e-6, rtol=0)
    np.testing.assert_allclose(got["cdc_mm"], ref["cdc_mm"], atol=1e-6, rtol=0)
    assert (got["contact_count"] == ref["contact_count"]).all()
    assert (got["success"] == ref["success"]).all()
    assert (got["note_flags"] == ref["note_flags"]).all()
    mg = cfg.eval.mass * cfg.eval.gravity
    np.testing.assert_allclose(got["residuals"], ref["residuals"], atol=1e-6 * mg, rtol=1e-6)


def ball_points(r, n=300):
    golden = np.pi * (3.0 - np.sqrt(5.0))
    k = np.arange(n)
    z = 1.0 - 2.0 * (k + 0.5) / n
    rr = np.sqrt(np.maximum(1.0 - z * z, 0.0))
    return np.stack([r * rr * np.cos(golden * k), r * rr * np.sin(golden * k), r * z], 1)


def test_eval_self_pairs_with_large_epa_polytopes(G, O, engine):
    """Self-penetration depth (eval.cpp:63-72) between two deeply overlapping 300-vertex round
    links: EPA needs far more than the 64-vertex per-thread polytope, so those pairs go through
    the full-capacity retry (k_eval_self_pairs_big) and still match the oracle."""
    import json
    ball = ball_points(0.03).round(6).tolist()
    tiny = [[x * 0.004, y * 0.004, z * 0.004] for x in (-1, 1) for y in (-1, 1) for z in (-1, 1)]
    doc = {"format_version": 1, "name": "balls", "links": [
        {"name": "palm", "vertices": ball, "proxies": [{"center": [0, 0, 0], "radius": 0.03}]},
        {"name": "stem", "vertices": tiny, "joint": {"parent": "palm", "origin": [0, 0, 0.05], "axis": [1, 0, 0],
                                                      "lower": -0.5, "upper": 0.5}},
        {"name": "tip", "vertices": ball, "proxies": [{"center": [0, 0, 0], "radius": 0.03}], "tip_proxy": 0,
         "joint": {"parent": "stem", "origin": [0, 0, -0.03], "axis": [1, 0, 0], "lower": -0.5, "upper": 0.5}}]}
    hand = G.HandModel.from_json(json.dumps(doc))
    assert hand.n_pairs == 1
    obj = G.make_primitive("sphere", 0.1)
    use(engine, hand, obj)
    rng = np.random.default_rng(12)
    x = np.zeros((64, hand.dims()))
    x[:, [0, 4, 8]] = 1.0
    x[:, 9:12] = [0.0, 0.0, 0.5]
    x[:, 12:] = rng.uniform(-0.3, 0.3, size=(64, 2))
    ref = O.evaluate(hand, obj, G.RunConfig(), x, x)
    got = engine.evaluate(G.RunConfig(), x, x)
    assert (ref["spd_mm"] > 30).all()
    np.testing.assert_allclose(got["spd_mm"], ref["spd_mm"], atol=1e-6, rtol=0)


def test_fine_contact_query_matches_oracle(G, O, trident, engine):
    obj = G.make_primitive("box", 0.1)
    use(engine, trident, obj)
    x = G.init_poses(trident, obj, 128, 5)
    x[:, 9:12] *= 0.6
    ref = O.fine_contact_query(trident, obj, x)
    got = gpu_fcq(engine, trident, x)
    # With the oracle's own FK (glibc sin/cos) a few box-on-box witnesses sit on flat-face
    # ties that an ulp decides; distance, normal and link always agree.
    ties = witness_ties(got, ref)
    assert ties.mean() <= 0.03, f"{ties.mean():.3f} of box-on-box witnesses hit ties"
    # On the device's own link poses the pair results are the oracle's bit for bit.
    world = gpu_fk(engine, trident, x)
    m, P = trident.n_tips, obj.n_parts
    links = np.tile(np.repeat(trident.fingertip_links, P), len(x))
    parts = np.tile(np.arange(P), len(x) * m)
    poses = np.repeat(world[:, trident.fingertip_links].reshape(-1, 12), P, axis=0)
    assert np.array_equal(gpu_pairs(engine, links, parts, poses)[:, :10],
                          O.signed_distance(trident, obj, links, parts, poses)[:, :10])


# ---------------------------------------------------------------- end to end
def test_synthesize_short_schedule_matches_oracle(G, O, trident, engine):
    obj = G.make_primitive("sphere", 0.1)
    use(engine, trident, obj)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 8, 17
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 20, 10, 10
    x0 = G.init_poses(trident, obj, cfg.batch, cfg.seed, cfg.init)
    gpu = engine.synthesize(cfg, x0)
    cpu = O.synthesize(trident, obj, cfg, x0, workers=8)
    assert (gpu.failed == cpu.failed).all()
    # 40 coupled nonconvex steps: QP solver rounding (Woodbury vs LLT) and
    # convergence-check timing accumulate to ~1e-6 on a few coordinates.
    np.testing.assert_allclose(gpu.x, cpu.x, atol=1e-5)
    np.testing.assert_allclose(gpu.x_p, cpu.x_p, atol=1e-5)
    np.testing.assert_allclose(gpu.x_s, cpu.x_s, atol=1e-5)
    np.testing.assert_allclose(gpu.energy_total, cpu.energy_total, rtol=1e-4)
    # Mesh-stage energies are ~1e-2; the 1e-5-level pose differences above
    # move them by ~1e-5 absolute.
    np.testing.assert_allclose(gpu.stage_energy, cpu.stage_energy, rtol=1e-4, atol=1e-4)


# ----------------------------------------------------------- KATs on device
BOX_HAND = """{"format_version": 1, "name": "box", "links": [{"name": "box", "vertices":
 [[-0.5,-0.5,-0.5],[-0.5,-0.5,0.5],[-0.5,0.5,-0.5],[-0.5,0.5,0.5],[0.5,-0.5,-0.5],[0.5,-0.5,0.5],[0.5,0.5,-0.5],
  [0.5,0.5,0.5]], "proxies": [{"center": [0,0,0], "radius": 0.5}], "tip_proxy": 0}]}"""


@pytest.mark.parametrize("p,d,pb", [((0.9, 0.1, 0.05), 0.4, (0.5, 0.1, 0.05)),
                                    ((0.8, 0.7, 0.0), 0.42426406871192851, (0.5, 0.4, 0.0)),
                                    ((1.5, 1.4, 1.3), 1.7320508075688772, (0.5, 0.4, 0.3)),
                                    ((0.1, 0.0, 0.2), -0.1, (0.1, 0.0, 0.3))])
def test_point_query_box_kats_on_device(G, trident, engine, p, d, pb):
    # test_geometry.cpp:274-305 on the sm_100a kernel.
    box = G.ObjectModel.from_points([np.array([(sx * 0.5, sy * 0.4, sz * 0.3) for sx in (-1, 1) for sy in (-1, 1)
                                               for sz in (-1, 1)])])
    use(engine, trident, box)
    r = gpu_points(engine, [p])[0]
    assert r[0] == pytest.approx(d, abs=1e-12)
    np.testing.assert_allclose(r[1:4], pb, atol=1e-12)


def test_gjk_epa_box_kats_on_device(G, engine):
    # test_geometry.cpp:147-167, 215-247 (link = unit box, object = unit box).
    hand = G.HandModel.from_json(BOX_HAND)
    box = G.ObjectModel.from_points([np.array([(sx * 0.5, sy * 0.5, sz * 0.5) for sx in (-1, 1) for sy in (-1, 1)
                                               for sz in (-1, 1)])])
    use(engine, hand, box)
    shifts = [1.0 + g for g in (1e-6, 0.01, 0.3, 2.0)] + [1.0 - d for d in (0.05, 0.2, 0.45)] + [0.0]
    poses = np.zeros((len(shifts), 12))
    poses[:, [0, 4, 8]] = 1.0
    poses[:, 9] = -np.array(shifts)  # move the link so the object sits at +shift
    r = gpu_pairs(engine, np.zeros(len(shifts)), np.zeros(len(shifts)), poses)
    for i, g in enumerate((1e-6, 0.01, 0.3, 2.0)):
        assert r[i, 0] == pytest.approx(g, rel=1e-10)
    for i, dep in enumerate((0.05, 0.2, 0.45)):
        assert r[4 + i, 0] == pytest.approx(-dep, rel=1e-9)
        np.testing.assert_allclose(r[4 + i, 7:10], (-1, 0, 0), atol=1e-9)
    assert r[7, 0] == pytest.approx(-1.0, rel=1e-9)  # concentric: depth 1, deterministic


def test_energy_kats_on_device(G, engine):
    # test_energy.cpp:152-217 through grasp_qp_batch.
    def frame(p, n):
        n = np.asarray(n, float)
        seed = np.array([0.0, 1.0, 0.0]) if abs(n[0]) > 0.99 else np.array([1.0, 0.0, 0.0])
        d = np.cross(n, seed)
        d /= np.linalg.norm(d)
        return np.concatenate([p, n, d, np.cross(n, d)])

    def tight(beta, gamma):
        cfg = G.RunConfig()
        cfg.qp.eps_primal = cfg.qp.eps_dual = 1e-9
        cfg.qp.max_iters = 200000
        cfg.energy.beta, cfg.energy.gamma_per_contact = beta, gamma
        return cfg

    pair = np.array([[frame((1.0, 0, 0), (-1, 0, 0)), frame((-1.0, 0, 0), (1, 0, 0))]])
    for gamma in (0.0, 0.1):
        r = gpu_qp(engine, tight(0.8, gamma), pair, 2)
        assert r["converged"].all() and r["per_direction"].sum() <= 1e-6
    one = np.array([[frame((0.3, 0, 0), (-1, 0, 0))]])
    r = gpu_qp(engine, tight(0.0, 0.1), one, 1)
    np.testing.assert_allclose(r["per_direction"][0], 0.01, rtol=1e-4)


# --------------------------------------------------- full schedule, statistics
def test_full_schedule_matches_oracle_statistics(G, O, trident, engine):
    """Default 300/100/100 schedule: per-grasp trajectories stay within
    rounding of the oracle for most grasps; where ties or QP convergence
    timing let them drift, the batch statistics (failure flags, final grasp
    energy distribution, fine-stage energy) still agree."""
    obj = G.make_primitive("sphere", 0.1)
    use(engine, trident, obj)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 24, 17
    x0 = G.init_poses(trident, obj, cfg.batch, cfg.seed, cfg.init)
    gpu = engine.synthesize(cfg, x0)
    cpu = O.synthesize(trident, obj, cfg, x0, workers=8)
    assert (gpu.failed == cpu.failed).all()
    close = np.abs(gpu.x - cpu.x).max(axis=1) <= 1e-4
    assert close.mean() >= 0.75, close
    ok = cpu.failed == 0
    for a, b in ((gpu.energy_total[ok], cpu.energy_total[ok]), (gpu.stage_energy[ok, 1, 1], cpu.stage_energy[ok, 1, 1])):
        assert abs(np.median(a) - np.median(b)) <= 0.05 * abs(np.median(b)) + 1e-3


@pytest.mark.parametrize("shape", ["sphere", "box"])
def test_config1_allegro_end_to_end_statistics(G, O, engine, shape):
    """BASELINE config 1 (Allegro-like hand, primitive object at 0.08, batch 64, 4 contacts,
    seed 17, default 300/100/100 schedule): GPU synthesis vs the oracle on the same x0 -
    identical failure flags, matching final-energy statistics, and matching evaluation
    statistics (quasi-static success rate and median penetration, eval.cpp:91-158), each
    side evaluated with its own evaluator."""
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    hand = G.HandModel.from_file(root / "paper_2412_16490_b200/assets/hands/allegro_like.json")
    obj = G.make_primitive(shape, 0.08)
    use(engine, hand, obj)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 64, 17
    x0 = G.init_poses(hand, obj, cfg.batch, cfg.seed, cfg.init)
    gpu = engine.synthesize(cfg, x0)
    cpu = O.synthesize(hand, obj, cfg, x0, workers=16)
    assert (gpu.failed == cpu.failed).all()
    ok = cpu.failed == 0
    assert ok.sum() >= 48
    for a, b in ((gpu.energy_total[ok], cpu.energy_total[ok]), (gpu.stage_energy[ok, 1, 1], cpu.stage_energy[ok, 1, 1])):
        assert abs(np.median(a) - np.median(b)) <= 0.1 * abs(np.median(b)) + 1e-3
    eg = engine.evaluate(cfg, gpu.x[ok], gpu.x_s[ok])
    ec = O.evaluate(hand, obj, cfg, cpu.x[ok], cpu.x_s[ok])
    n = ok.sum()
    assert abs(eg["success"].mean() - ec["success"].mean()) <= 3.0 / np.sqrt(n) + 0.05
    assert abs(np.median(eg["pd_mm"]) - np.median(ec["pd_mm"])) <= 0.25 * np.median(ec["pd_mm"]) + 0.5


@pytest.mark.parametrize("single_launch", [True, False])
def test_synthesize_objects_equals_per_object_runs(G, trident, engine, single_launch):
    """Multi-object synthesis (config 3 path): one batch over several objects in
    one context (object id per grasp, parts packed, one set of launches) -- including a
    multi-part mesh next to single-part primitives of different batch sizes -- and the
    concurrent-context fallback both return, per object, bitwise the records of a plain
    per-object synthesize."""
    import dataclasses
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    objs = [G.make_primitive(n, 0.09) for n in ("sphere", "box", "cylinder")]
    objs.insert(1, G.load_object(root / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10))
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 8, 3
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 30, 10, 10
    cfgs = [dataclasses.replace(cfg, seed=i, batch=6 + 3 * i) for i in range(len(objs))]
    many = G.synthesize_objects(trident, objs, cfgs, streams=3, single_launch=single_launch)
    for obj, c, recs in zip(objs, cfgs, many):
        one = G.synthesize(trident, obj, c)
        assert len(one) == len(recs) == c.batch
        for a, b in zip(one, recs):
            assert np.array_equal(a.x, b.x) and np.array_equal(a.x_s, b.x_s) and np.array_equal(a.x_p, b.x_p)
            assert a.energy_total == b.energy_total or (np.isnan(a.energy_total) and np.isnan(b.energy_total))
            assert a.failed == b.failed and a.object_id == b.object_id


def test_optional_pair_cull_runs_and_agrees(G):
    """The opt-in separation cull (option "pair_cull") runs and, on well-separated
    starts, gives the reference-exact default's results except for the grasps where the
    reference's spurious GJK overlaps matter (most grasps identical)."""
    hand = G.HandModel.builtin()
    obj = G.make_primitive("box", 0.1)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 32, 5
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 40, 20, 20
    x0 = G.init_poses(hand, obj, cfg.batch, cfg.seed, cfg.init)
    eng = G.Engine(0)
    eng.set_hand(hand)
    eng.set_object(obj)
    a = eng.synthesize(cfg, x0).x
    eng.set_option("pair_cull", 1)
    b = eng.synthesize(cfg, x0).x
    same = (a == b).all(axis=1)
    assert same.mean() >= 0.75, same.mean()
    with pytest.raises(G.InvalidArgument):
        eng.set_option("no_such_option", 1)


def test_group_point_queries_bitwise_equal_thread_queries(G):
    """The lane-group point query (tip-centre queries of the fine/final stages, 4 lanes per query by
    default) merges its split scans with order-free reductions; any group size must give
    the thread-per-query kernel's results bit for bit, on the tips and on all query slots."""
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    hand = G.HandModel.from_file(root / "paper_2412_16490_b200/assets/hands/shadow_like.json")
    obj = G.load_object(root / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 96, 23
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 30, 10, 10
    x0 = G.init_poses(hand, obj, cfg.batch, cfg.seed, cfg.init)
    eng = G.Engine(0)
    eng.set_hand(hand)
    eng.set_object(obj)
    outs = {}
    for tips, full in ((1, 1), (4, 1), (8, 2), (32, 4)):
        eng.set_option("tip_query_lanes", tips)
        eng.set_option("query_lanes", full)
        outs[(tips, full)] = eng.synthesize(cfg, x0)
    ref = outs[(1, 1)]
    for k, o in outs.items():
        assert np.array_equal(o.x, ref.x), k
        assert np.array_equal(o.x_s, ref.x_s), k
        assert np.array_equal(o.failed, ref.failed), k
        assert np.array_equal(o.contacts, ref.contacts, equal_nan=True), k


@pytest.mark.parametrize("case", ["shadow_drill", "trident_box"])
def test_bucketed_point_queries_bitwise(G, case):
    """The coarse stage's point queries listed by spatial bucket (k_pq_count / k_pq_scatter /
    k_point_query_list) give bitwise the records of the slot-order launch (query_buckets = 0)."""
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    if case == "shadow_drill":
        hand = G.HandModel.from_file(root / "paper_2412_16490_b200/assets/hands/shadow_like.json")
        obj = G.load_object(root / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)
    else:
        hand, obj = G.HandModel.builtin(), G.make_primitive("box", 0.08)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 256, 31
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 300, 5, 5
    x0 = G.init_poses(hand, obj, cfg.batch, cfg.seed, cfg.init)
    outs = []
    for flag in (0, 1):
        eng = G.Engine(0)
        eng.set_hand(hand)
        eng.set_object(obj)
        eng.set_option("query_buckets", flag)
        outs.append(eng.synthesize(cfg, x0))
    for f in ("x", "x_p", "x_s", "energy_total", "stage_energy", "failed", "contact_forces"):
        assert np.array_equal(getattr(outs[0], f), getattr(outs[1], f), equal_nan=True), f


@pytest.mark.parametrize("case", ["shadow_drill", "trident_box"])
def test_early_epa_pass_bitwise(G, case):
    """Pairs whose last EPA ran long take the early pass (k_pairs_early: GJK + EPA per thread on a
    side stream, option "pair_early"); every threshold, from all overlapping pairs (0) to none
    (255), gives bitwise the same records as the two-pass GJK -> EPA path."""
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    if case == "shadow_drill":
        hand = G.HandModel.from_file(root / "paper_2412_16490_b200/assets/hands/shadow_like.json")
        obj = G.load_object(root / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)
    else:
        hand, obj = G.HandModel.builtin(), G.make_primitive("box", 0.08)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 128, 37
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 40, 30, 30
    x0 = G.init_poses(hand, obj, cfg.batch, cfg.seed, cfg.init)
    outs = {}
    for thr in (255, 0, 4, 24):
        eng = G.Engine(0)
        eng.set_hand(hand)
        eng.set_object(obj)
        eng.set_option("pair_early", thr)
        outs[thr] = eng.synthesize(cfg, x0)
    ref = outs[255]
    for thr, o in outs.items():
        for f in ("x", "x_p", "x_s", "energy_total", "stage_energy", "failed", "contacts"):
            assert np.array_equal(getattr(o, f), getattr(ref, f), equal_nan=True), (thr, f)


def test_graph_replay_bitwise_equals_eager(G):
    """Synthesis through a captured CUDA graph (option "graphs", default on: captured once per
    hand/object/buffers/parameters, then replayed) gives bitwise the eager launches' records,
    on a replay and after a recapture for new parameters; the kernel count is the same."""
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    hand = G.HandModel.from_file(root / "paper_2412_16490_b200/assets/hands/shadow_like.json")
    obj = G.load_object(root / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 96, 41
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 24, 12, 12
    fields = ("x", "x_p", "x_s", "energy_total", "stage_energy", "failed", "contacts", "contact_forces")

    def runs(flag, seeds):
        eng = G.Engine(0)
        eng.set_hand(hand)
        eng.set_object(obj)
        eng.set_option("graphs", flag)
        outs, counts = [], []
        for sd in seeds:
            c = G.RunConfig.from_params(cfg.to_params())
            c.seed = sd
            k0 = eng.launch_count()
            outs.append(eng.synthesize(c, G.init_poses(hand, obj, c.batch, sd, c.init)))
            counts.append(eng.launch_count() - k0)
        return outs, counts

    seeds = (41, 41, 7)
    eager, k_eager = runs(0, seeds)
    graph, k_graph = runs(1, seeds)
    assert k_eager == k_graph
    for e, g in zip(eager, graph):
        for f in fields:
            assert np.array_equal(getattr(e, f), getattr(g, f), equal_nan=True), f


def test_synthesis_deterministic_and_batch_prefix_independent(G, trident, engine):
    """test_pipeline.cpp:399-421 on the device: the same start states give bitwise-equal
    records on a rerun, and a grasp's record does not depend on the batch it is in
    (a prefix of the batch, and a batch of one)."""
    obj = G.make_primitive("box", 0.08)
    use(engine, trident, obj)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 12, 5
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 15, 6, 6
    x0 = G.init_poses(trident, obj, cfg.batch, cfg.seed, cfg.init)
    a = engine.synthesize(cfg, x0)
    b = engine.synthesize(cfg, x0)
    for f in ("x", "x_p", "x_s", "energy_total", "stage_energy", "failed"):
        assert np.array_equal(getattr(a, f), getattr(b, f), equal_nan=True), f
    for k in (5, 1):
        cfg.batch = k
        p = engine.synthesize(cfg, np.ascontiguousarray(x0[:k]))
        for f in ("x", "x_p", "x_s", "energy_total", "failed"):
            assert np.array_equal(getattr(p, f), getattr(a, f)[:k], equal_nan=True), (k, f)


def test_multi_device_context_equals_single_device(G, trident, engine):
    """grasp_ctx_create_devices: contiguous shards on their own host threads
    and streams (here three shards on cuda:0) give bitwise the single-context records."""
    obj = G.make_primitive("capsule", 0.09)
    use(engine, trident, obj)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 13, 9
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 40, 15, 15
    x0 = G.init_poses(trident, obj, cfg.batch, cfg.seed, cfg.init)
    one = engine.synthesize(cfg, x0)
    multi = G.Engine(devices=[0, 0, 0])
    multi.set_hand(trident)
    multi.set_object(obj)
    many = multi.synthesize(cfg, x0)
    for f in ("x", "x_p", "x_s", "energy_total", "per_direction", "contact_forces", "contacts", "stage_energy",
              "failed", "qp_converged"):
        assert np.array_equal(getattr(one, f), getattr(many, f), equal_nan=True), f


def test_failed_rows_masked_on_device_outputs(G, trident, engine):
    """Failed grasps report NaN energy / forces / contacts and unconverged flags on the
    device-pointer path too (pipeline.cpp:312-314), not stale buffer contents."""
    import torch
    sphere = G.make_primitive("sphere", 0.1)
    use(engine, trident, sphere)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 4, 17
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 30, 10, 10
    x0 = G.init_poses(trident, sphere, 4, 17, cfg.init)
    engine.synthesize(cfg, x0)  # leaves finite values in the engine's buffers
    cfg.pipeline.coarse.step_translation = 1e5
    D, m, n = trident.dims(), trident.n_tips, trident.n_tips * cfg.contact.n_edges
    dev = torch.device("cuda:0")
    xd = torch.from_numpy(x0).to(dev)
    outs = dict(energy_total=torch.zeros(4, dtype=torch.float64, device=dev),
                contact_forces=torch.zeros(4 * n * 6, dtype=torch.float64, device=dev),
                contacts=torch.zeros(4 * m * 12, dtype=torch.float64, device=dev),
                failed=torch.zeros(4, dtype=torch.int32, device=dev),
                qp_converged=torch.ones(4 * 6, dtype=torch.int32, device=dev))
    engine.synthesize_device(cfg, xd.data_ptr(), 4, {k: v.data_ptr() for k, v in outs.items()})
    torch.cuda.synchronize()
    assert (outs["failed"].cpu().numpy() != 0).all()
    assert torch.isnan(outs["energy_total"]).all() and torch.isnan(outs["contact_forces"]).all()
    assert torch.isnan(outs["contacts"]).all() and (outs["qp_converged"] == 0).all()


def test_diverging_grasps_are_flagged_on_device(G, O, trident, engine):
    """test_pipeline.cpp:475-488 on the device: a huge translation step diverges every
    grasp; each is flagged failed (as the oracle flags it) with finite state and NaN energy."""
    sphere = G.make_primitive("sphere", 0.1)
    use(engine, trident, sphere)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 3, 17
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 120, 50, 50
    cfg.pipeline.coarse.step_translation = 1e5
    x0 = G.init_poses(trident, sphere, 3, 17, cfg.init)
    gpu = engine.synthesize(cfg, x0)
    cpu = O.synthesize(trident, sphere, cfg, x0, workers=3)
    assert (gpu.failed != 0).all()
    assert np.array_equal(gpu.failed, cpu.failed)
    assert np.isfinite(gpu.x).all()
    assert np.isnan(gpu.energy_total).all()


def _finger_hand_json(lengths):
    """A palm box with one chain of revolute box links per finger (lengths[i] links), the last
    link of each finger carrying a tip proxy."""
    import json
    box = [[x, y, z] for x in (-0.005, 0.005) for y in (-0.005, 0.005) for z in (0.0, 0.02)]
    prox = [{"center": [0, 0, 0.01], "radius": 0.005}]
    links = [{"name": "palm", "vertices": box, "proxies": prox}]
    for f, n in enumerate(lengths):
        parent = "palm"
        for i in range(n):
            name = f"f{f}_{i}"
            origin = [0.012 * (f - len(lengths) / 2), 0, 0.02] if i == 0 else [0, 0, 0.02]
            link = {"name": name, "joint": {"name": f"j{f}_{i}", "parent": parent, "origin": origin,
                                            "axis": [1, 0, 0], "lower": -0.5, "upper": 0.5},
                    "vertices": box, "proxies": prox}
            if i == n - 1:
                link["tip_proxy"] = 0
            links.append(link)
            parent = name
    return json.dumps({"format_version": 1, "name": "fingers", "links": links})


def test_device_capacity_limits_are_invalid_arguments(G, engine):
    """The engine's fixed capacities (32 links, 1..5 fingertips, chains up to 12 joints deep,
    64 parts per object) and an empty batch are reported as invalid arguments (the reference's
    std::invalid_argument), never truncated; a hand at the limits runs."""
    ok = G.HandModel.from_json(_finger_hand_json([7, 6, 6, 6, 6]))  # 32 links, 31 joints, 5 tips
    obj = G.make_primitive("sphere", 0.1)
    engine.set_hand(ok)
    engine.set_object(obj)
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = 4, 3
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 3, 2, 2
    out = engine.synthesize(cfg, G.init_poses(ok, obj, cfg.batch, cfg.seed, cfg.init))
    assert out.x.shape[0] == 4
    for lengths in ([7, 7, 6, 6, 6], [2] * 6, [13]):  # 33 links; 6 tips; a chain deeper than 12
        h = G.HandModel.from_json(_finger_hand_json(lengths))
        with pytest.raises(G.InvalidArgument):
            engine.set_hand(h)
    engine.set_hand(ok)
    many = G.ObjectModel.from_points([np.random.default_rng(i).normal(size=(8, 3)) * 0.01 + [0.05 * i, 0, 0]
                                      for i in range(65)])
    with pytest.raises(G.InvalidArgument):
        engine.set_object(many)
    engine.set_object(obj)
    cfg.batch = 0
    with pytest.raises(G.InvalidArgument):
        engine.synthesize(cfg, np.zeros((0, ok.dims())))
