"""The fp64 CPU oracle against the reference's own known-answer tests.

The reference (proj/) cannot be built here (Eigen3/doctest/nlohmann absent),
so these KATs -- copied as expectations, not code, from proj/tests/*.cpp --
are what pins the oracle to the reference's behaviour.
"""
import math

import numpy as np
import pytest


def box_points(hx, hy, hz, c=(0.0, 0.0, 0.0)):
    return np.array([(c[0] + sx * hx, c[1] + sy * hy, c[2] + sz * hz) for sx in (-1, 1) for sy in (-1, 1)
                     for sz in (-1, 1)])


def pose12(R=None, t=(0.0, 0.0, 0.0)):
    R = np.eye(3) if R is None else np.asarray(R)
    return np.concatenate([R.T.reshape(9), np.asarray(t, dtype=float)])  # column-major R, t


@pytest.fixture(scope="module")
def box543(G):
    return G.ObjectModel.from_points([box_points(0.5, 0.4, 0.3)])


# ------------------------------------------------------------ point queries
@pytest.mark.parametrize("p,d,pb,n", [
    ((0.9, 0.1, 0.05), 0.4, (0.5, 0.1, 0.05), (1, 0, 0)),          # face region
    ((0.8, 0.7, 0.0), math.hypot(0.3, 0.3), (0.5, 0.4, 0.0), None),  # edge region
    ((1.5, 1.4, 1.3), math.sqrt(3.0), (0.5, 0.4, 0.3), None),       # corner region
    ((0.1, 0.0, 0.2), -0.1, (0.1, 0.0, 0.3), (0, 0, 1)),            # interior: signed, nearest face
])
def test_point_query_box_kats(O, box543, p, d, pb, n):
    # test_geometry.cpp:274-305.
    r = O.point_to_mesh(box543, [p])[0]
    assert r[0] == pytest.approx(d, abs=1e-12)
    np.testing.assert_allclose(r[1:4], pb, atol=1e-12)
    if n is not None:
        np.testing.assert_allclose(r[4:7], n, atol=1e-12)
    assert r[7] == 0


def test_point_query_surface_is_zero(O, box543):
    assert abs(O.point_to_mesh(box543, [(0.5, 0.0, 0.0)])[0][0]) < 1e-12


def test_multipart_nearest_and_low_ties(G, O):
    # test_geometry.cpp:307-319.
    box = box_points(0.5, 0.5, 0.5)
    two = G.ObjectModel.from_points([box, box + np.array([2.0, 0, 0])])
    assert O.point_to_mesh(two, [(-1.0, 0, 0)])[0][7] == 0
    assert O.point_to_mesh(two, [(3.5, 0, 0)])[0][7] == 1
    twins = G.ObjectModel.from_points([box, box])
    assert O.point_to_mesh(twins, [(0.9, 0.2, 0.1)])[0][7] == 0
    assert O.point_to_mesh(twins, [(0.1, 0.0, 0.0)])[0][7] == 0


# ------------------------------------------------------------------ GJK/EPA
@pytest.fixture(scope="module")
def unit_boxes(G):
    b = G.ObjectModel.from_points([box_points(0.5, 0.5, 0.5)])
    return b, b


@pytest.mark.parametrize("gap", [1e-6, 0.01, 0.3, 2.0])
def test_gjk_box_gap_is_exact(O, unit_boxes, gap):
    # test_geometry.cpp:147-167.
    a, b = unit_boxes
    r = O.part_pairs(a, b, [0], [0], [pose12()], [pose12(t=(1.0 + gap, 0, 0))], kind=1)[0]
    assert r[0] == pytest.approx(gap, rel=1e-10)
    assert np.linalg.norm(r[1:4] - r[4:7]) == pytest.approx(gap, rel=1e-9)
    assert r[1] == pytest.approx(0.5, rel=1e-9)
    assert r[4] == pytest.approx(0.5 + gap, rel=1e-9)


def test_gjk_touch_and_overlap_report_zero(O, unit_boxes):
    a, b = unit_boxes
    for t in (1.0, 0.7):
        r = O.part_pairs(a, b, [0], [0], [pose12()], [pose12(t=(t, 0, 0))], kind=1)[0]
        assert r[0] == pytest.approx(0.0, abs=1e-12)


@pytest.mark.parametrize("depth", [0.05, 0.2, 0.45])
def test_epa_depth_on_shifted_boxes(O, unit_boxes, depth):
    # test_geometry.cpp:215-233.
    a, b = unit_boxes
    e = O.part_pairs(a, b, [0], [0], [pose12()], [pose12(t=(1.0 - depth, 0, 0))], kind=2)[0]
    assert e[0] == pytest.approx(depth, rel=1e-9)
    np.testing.assert_allclose(e[7:10], (-1, 0, 0), atol=1e-9)
    s = O.part_pairs(a, b, [0], [0], [pose12()], [pose12(t=(1.0 - depth, 0, 0))], kind=0)[0]
    assert s[0] == pytest.approx(-depth, rel=1e-9)
    assert s[10] == 1


def test_epa_concentric_tie_is_deterministic(O, unit_boxes):
    # test_geometry.cpp:235-247.
    a, b = unit_boxes
    first = O.part_pairs(a, b, [0], [0], [pose12()], [pose12()], kind=2)[0]
    assert first[0] == pytest.approx(1.0, rel=1e-9)
    assert np.abs(first[7:10]).max() == pytest.approx(1.0, rel=1e-9)
    for _ in range(3):
        again = O.part_pairs(a, b, [0], [0], [pose12()], [pose12()], kind=2)[0]
        assert again[0] == first[0] and (again[7:10] == first[7:10]).all()


def test_epa_on_disjoint_parts_raises(G, O, unit_boxes):
    a, b = unit_boxes
    with pytest.raises(G.GeometryError):
        O.part_pairs(a, b, [0], [0], [pose12()], [pose12(t=(3.0, 0, 0))], kind=2)


def test_ball_hull_distance(G, O):
    # test_geometry.cpp:435-444 (inscribed 400-point ball hulls).
    golden = math.pi * (3.0 - math.sqrt(5.0))
    pts = []
    for k in range(400):
        z = 1.0 - 2.0 * (k + 0.5) / 400
        r = math.sqrt(max(1.0 - z * z, 0.0))
        pts.append((0.1 * r * math.cos(golden * k), 0.1 * r * math.sin(golden * k), 0.1 * z))
    ball = G.ObjectModel.from_points([np.array(pts)])
    r = O.part_pairs(ball, ball, [0], [0], [pose12()], [pose12(t=(0.5, 0, 0))], kind=1)[0]
    assert 0.3 <= r[0] <= 0.302


# ------------------------------------------------------- lower QP / energies
def frame(p, n):
    n = np.asarray(n, float)
    seed = np.array([0.0, 1.0, 0.0]) if abs(n[0]) > 0.99 else np.array([1.0, 0.0, 0.0])
    d = np.cross(n, seed)
    d /= np.linalg.norm(d)
    return np.concatenate([p, n, d, np.cross(n, d)])


def tight_cfg(G, beta, gamma):
    cfg = G.RunConfig()
    cfg.qp.eps_primal = cfg.qp.eps_dual = 1e-9
    cfg.qp.max_iters = 200000
    cfg.energy.beta, cfg.energy.gamma_per_contact = beta, gamma
    return cfg


@pytest.mark.parametrize("gamma", [0.0, 0.1])
def test_antipodal_pair_achieves_every_closure_target(G, O, gamma):
    # test_energy.cpp:152-173.
    frames = np.array([[frame((1.0, 0, 0), (-1, 0, 0)), frame((-1.0, 0, 0), (1, 0, 0))]])
    r = O.qp_batch(tight_cfg(G, 0.8, gamma), frames, 2)
    assert r["converged"].all()
    assert 0.0 <= r["per_direction"].sum() <= 1e-6


def test_beta_zero_floor_costs_gamma_squared(G, O):
    # test_energy.cpp:198-217.
    one = np.array([[frame((0.3, 0, 0), (-1, 0, 0))]])
    r = O.qp_batch(tight_cfg(G, 0.0, 0.1), one, 1)
    assert r["converged"].all()
    np.testing.assert_allclose(r["per_direction"][0], 0.01, rtol=1e-4)
    assert np.abs(r["per_direction"][0] - r["per_direction"][0, 0]).max() <= 1e-12
    pair = np.array([[frame((1.0, 0, 0), (-1, 0, 0)), frame((-1.0, 0, 0), (1, 0, 0))]])
    r2 = O.qp_batch(tight_cfg(G, 0.0, 0.1), pair, 2)
    assert r2["converged"].all() and r2["per_direction"].sum() <= 1e-8


def test_qp_cap_propagates_nonconvergence(G, O):
    # test_energy.cpp:566-580: a strangled solve reports converged = false.
    rng = np.random.default_rng(3)
    frames = np.array([[frame(p, -p / np.linalg.norm(p)) for p in rng.normal(size=(3, 3))]])
    cfg = G.RunConfig()
    cfg.qp.max_iters = 2
    r = O.qp_batch(cfg, frames, 3)
    assert not r["converged"].all()
    assert (r["iters"] == 2).all()


def test_infeasible_floor_rejected(G, O):
    cfg = G.RunConfig()
    cfg.energy.gamma_per_contact = 1.5  # > caps (qpsolve.cpp:215-217)
    with pytest.raises(G.InvalidArgument):
        O.qp_batch(cfg, np.zeros((1, 1, 12)) + np.array(frame((1, 0, 0), (-1, 0, 0))), 1)


# --------------------------------------------------------------- pipeline
def plain_state(hand, t, q):
    x = np.zeros(hand.dims())
    x[0] = x[4] = x[8] = 1.0
    x[9:12] = t
    x[12:] = q
    return x


def aabb_distance(p, lo, hi):
    outside = np.maximum.reduce([lo - p, np.zeros(3), p - hi])
    out = np.linalg.norm(outside)
    return out if out > 0 else max(np.max(lo - p), np.max(p - hi))


def test_coarse_distance_energy_matches_box_arithmetic(G, O, trident):
    # test_pipeline.cpp:107-134, with fingertip centers from the host FK.
    box = G.make_primitive("box", 0.1)
    lo, hi = box.bounding_box()
    q = 0.5 * (trident.lower + trident.upper)
    tip_r = trident.proxies[trident.link_proxy_begin[trident.fingertip_links] +
                            trident.link_tip_proxy[trident.fingertip_links], 3]
    x0 = plain_state(trident, np.zeros(3), q)
    tips0 = tip_centers(O, trident, box, x0)
    for offset in (0.0, 0.01):
        for beyond in (0.0, 0.004, -0.003):
            target = np.array([0.0, 0.0, hi[2] + tip_r[0] + offset + beyond])
            x = plain_state(trident, target - tips0[0], q)
            tips = tip_centers(O, trident, box, x)
            expected = sum((aabb_distance(tips[f], lo, hi) - tip_r[f] - offset) ** 2 for f in range(3))
            e, _ = O.coarse_distance_energy(trident, box, x, offset, 1e-6, with_grad=False)
            assert e[0] == pytest.approx(expected, rel=1e-9)


def tip_centers(O, hand, obj, x):
    """Fingertip centers by an independent numpy FK (hand.cpp:126-153)."""
    R = x[:9].reshape(3, 3).T  # column-major raw block; plain states are exact rotations
    t = x[9:12]
    pb = hand.link_proxy_begin
    centers = []
    chain = {}
    lpj = hand.link_parent_joint
    d = hand.desc
    jo = np.ctypeslib.as_array(d.joint_origin, shape=(3 * hand.dof(),)).reshape(-1, 3)
    ja = np.ctypeslib.as_array(d.joint_axis, shape=(3 * hand.dof(),)).reshape(-1, 3)
    jpl = np.ctypeslib.as_array(d.joint_parent_link, shape=(hand.dof(),))
    for link in range(hand.n_links):
        j = lpj[link]
        if j < 0:
            chain[link] = (np.eye(3), np.zeros(3))
            continue
        Rp, tp = chain[jpl[j]]
        a = ja[j]
        c, s = math.cos(x[12 + j]), math.sin(x[12 + j])
        K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
        Rs = c * np.eye(3) + s * K + (1 - c) * np.outer(a, a)
        chain[link] = (Rp @ Rs, Rp @ jo[j] + tp)
    for link in hand.fingertip_links:
        Rc, tc = chain[link]
        p = hand.proxies[pb[link] + hand.link_tip_proxy[link], :3]
        centers.append(R @ (Rc @ p + tc) + t)
    return np.array(centers)


def short_cfg(G, batch=4):
    cfg = G.RunConfig()
    cfg.batch, cfg.seed = batch, 17
    cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters = 120, 50, 50
    return cfg


@pytest.mark.slow
def test_synthesis_is_deterministic_and_worker_independent(G, O, trident):
    # test_pipeline.cpp:399-421.
    sphere = G.make_primitive("sphere", 0.1)
    cfg = short_cfg(G)
    x0 = G.init_poses(trident, sphere, 4, 17)
    a = O.synthesize(trident, sphere, cfg, x0, workers=1)
    b = O.synthesize(trident, sphere, cfg, x0, workers=3)
    for f in ("x", "x_p", "x_s", "energy_total", "stage_energy", "contact_forces"):
        assert np.array_equal(getattr(a, f), getattr(b, f), equal_nan=True), f
    c = O.synthesize(trident, sphere, cfg, x0[:3], workers=2)
    assert np.array_equal(a.x[:3], c.x)


@pytest.mark.slow
def test_synthesis_records_are_structurally_sound(G, O, trident):
    # test_pipeline.cpp:423-473.
    sphere = G.make_primitive("sphere", 0.1)
    cfg = short_cfg(G, 6)
    x0 = G.init_poses(trident, sphere, 6, 17)
    out = O.synthesize(trident, sphere, cfg, x0, workers=6)
    ok = out.failed == 0
    assert ok.sum() >= 4
    assert np.isfinite(out.energy_total[ok]).all()
    for g in np.where(ok)[0]:
        np.testing.assert_allclose(G.squeeze_pose(trident, out.x[g], out.x_p[g]), out.x_s[g], atol=1e-12)
    assert np.median(out.stage_energy[:, 1, 1]) <= np.median(out.stage_energy[:, 0, 1])
    clear = O.fine_contact_query(trident, sphere, out.x_p[ok])[..., 9].ravel()
    assert 0.005 <= np.median(clear) <= 0.015


def test_diverging_grasps_are_flagged(G, O, trident):
    # test_pipeline.cpp:475-488.
    sphere = G.make_primitive("sphere", 0.1)
    cfg = short_cfg(G, 3)
    cfg.pipeline.coarse.step_translation = 1e5
    x0 = G.init_poses(trident, sphere, 3, 17)
    out = O.synthesize(trident, sphere, cfg, x0, workers=3)
    assert (out.failed != 0).all()
    assert np.isfinite(out.x).all()
    assert np.isnan(out.energy_total).all()
