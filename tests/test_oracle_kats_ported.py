"""The reference's own known-answer and property tests for the gradient, kinematics, contact and
QP paths, run against the fp64 CPU oracle.

The reference cannot be compiled here (Eigen3/doctest absent), so these ports -- the
expectations and tolerances of proj/tests/test_hand.cpp, test_contact.cpp, test_qpsolve.cpp,
test_energy.cpp and test_pipeline.cpp, with their random draws replaced by numpy draws -- are
what pins the oracle's restatement of the hot path's derivative and QP math to the
reference's behaviour. Each test cites the reference TEST_CASE it ports. The oracle is test
infrastructure (oracle/src/kats.cpp exposes its internals); nothing here touches the product.
"""
import math

import numpy as np
import pytest


def rand_rotation(rng, n=None):
    """shapes.hpp:39-44: normalized Gaussian quaternion -> rotation matrix."""
    q = rng.normal(size=(1 if n is None else n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    R = np.stack([np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
                  np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
                  np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)], -2)
    return R[0] if n is None else R


def axis_angle(w):
    a = np.linalg.norm(w)
    if a < 1e-12:
        return np.eye(3)
    k = w / a
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    return np.eye(3) + math.sin(a) * K + (1 - math.cos(a)) * K @ K


def state(hand, R, t, q):
    x = np.zeros(hand.dims())
    x[:9] = np.asarray(R).T.reshape(9)  # column-major raw block
    x[9:12] = t
    x[12:] = q
    return x


def random_state(hand, rng):
    """test_hand.cpp:48-59."""
    q = rng.uniform(hand.lower, hand.upper)
    return state(hand, rand_rotation(rng), rng.normal(0.0, 0.1, 3), q)


def fd_jacobian(f, x, h=1e-6):
    """oracles/fd_check.hpp:28-43 (central differences)."""
    cols = []
    for i in range(len(x)):
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        cols.append((np.asarray(f(xp)) - np.asarray(f(xm))) / (2 * h))
    return np.stack(cols, axis=-1)


def link_transform(O, hand, x, link):
    w = O.forward_kinematics(hand, x)[0, link]
    return w[:9].reshape(3, 3).T, w[9:]


# ----------------------------------------------------------------- test_hand.cpp
def test_rotation_projection_returns_nearest_proper_rotation(O):
    # test_hand.cpp:62-93.
    rng = np.random.default_rng(41)
    M = rng.normal(size=(4000, 3, 3))
    R, fb = O.project_rotation(M)
    assert np.abs(R.transpose(0, 2, 1) @ R - np.eye(3)).max() < 1e-12
    np.testing.assert_allclose(np.linalg.det(R), 1.0, rtol=1e-12)
    R2, _ = O.project_rotation(R[~fb])
    assert np.linalg.norm(R2 - R[~fb], axis=(1, 2)).max() < 1e-12  # idempotent
    for k in range(50):
        m = M[k]
        if fb[k]:
            continue
        best = np.linalg.norm(m - R[k])
        Q = rand_rotation(rng, 200)
        assert (best <= np.linalg.norm(m - Q, axis=(1, 2)) + 1e-9).all()
        for _ in range(50):
            w = rng.normal(0.0, 0.05, 3)
            assert best <= np.linalg.norm(m - R[k] @ axis_angle(w)) + 1e-12


def test_rotation_projection_fixes_improper_and_degenerate_blocks(O):
    # test_hand.cpp:95-110.
    rng = np.random.default_rng(43)
    Rs = rand_rotation(rng, 200)
    P, _ = O.project_rotation(Rs)
    assert np.linalg.norm(P - Rs, axis=(1, 2)).max() < 1e-13
    improper = Rs.copy()
    improper[:, :, 2] *= -1.0
    P, _ = O.project_rotation(improper)
    np.testing.assert_allclose(np.linalg.det(P), 1.0, rtol=1e-12)
    rank1 = np.outer([1, 2, 3], [0.5, -1, 2])
    P, fb = O.project_rotation(rank1)
    assert fb[0]
    assert np.abs(P[0].T @ P[0] - np.eye(3)).max() < 1e-12
    assert np.linalg.det(P[0]) == pytest.approx(1.0, rel=1e-12)


def test_rotation_tangent_jacobian_matches_numeric_projection_derivatives(O):
    # test_hand.cpp:112-135.
    rng = np.random.default_rng(47)
    M = rand_rotation(rng, 200) + rng.normal(0.0, 0.15, size=(200, 3, 3))
    R, ai, dg, J = O.pose_state(M)
    assert (~dg).sum() >= 150
    h = 1e-6
    checked = 0
    for k in np.where(~dg)[0]:
        plus, minus = [], []
        for c in range(9):
            dm = np.zeros((3, 3))
            dm[c % 3, c // 3] = 1.0
            plus.append(M[k] + h * dm)
            minus.append(M[k] - h * dm)
        rp, _ = O.project_rotation(np.array(plus))
        rm, _ = O.project_rotation(np.array(minus))
        for c in range(9):
            s = R[k].T @ ((rp[c] - rm[c]) / (2 * h))
            w = 0.5 * np.array([s[2, 1] - s[1, 2], s[0, 2] - s[2, 0], s[1, 0] - s[0, 1]])
            assert np.linalg.norm(J[k][:, c] - w) < 1e-5 * (1.0 + np.linalg.norm(w))
        checked += 1
    assert checked >= 150


def naive_link_pose(hand, x, link):
    """test_hand.cpp:30-46: Translation(t) * R, then Translation(origin_j) * AngleAxis(q_j, axis_j)
    along the chain (numpy, shares no code with the oracle)."""
    d = hand.desc
    jo = np.ctypeslib.as_array(d.joint_origin, shape=(3 * hand.dof(),)).reshape(-1, 3)
    ja = np.ctypeslib.as_array(d.joint_axis, shape=(3 * hand.dof(),)).reshape(-1, 3)
    jpl = np.ctypeslib.as_array(d.joint_parent_link, shape=(hand.dof(),))
    chain = []
    l = link
    while l >= 0:
        chain.append(l)
        j = hand.link_parent_joint[l]
        l = -1 if j < 0 else jpl[j]
    T = np.eye(4)
    T[:3, :3] = x[:9].reshape(3, 3).T
    T[:3, 3] = x[9:12]
    for l in reversed(chain):
        j = hand.link_parent_joint[l]
        if j < 0:
            continue
        S = np.eye(4)
        S[:3, :3] = axis_angle(ja[j] * x[12 + j]) if x[12 + j] != 0 else np.eye(3)
        S[:3, 3] = jo[j]
        T = T @ S
    return T


def test_forward_kinematics_matches_naive_chain(O, trident):
    # test_hand.cpp:137-150.
    rng = np.random.default_rng(53)
    for _ in range(100):
        x = random_state(trident, rng)
        w = O.forward_kinematics(trident, x)[0]
        for l in range(trident.n_links):
            T = naive_link_pose(trident, x, l)
            assert np.linalg.norm(w[l, :9].reshape(3, 3).T - T[:3, :3]) < 1e-12
            assert np.linalg.norm(w[l, 9:] - T[:3, 3]) < 1e-12


def test_point_and_direction_jacobians_match_finite_differences(O, trident):
    # test_hand.cpp:152-183.
    rng = np.random.default_rng(59)
    for _ in range(30):
        x = random_state(trident, rng)
        link = int(rng.integers(trident.n_links))
        p_local = rng.normal(0.0, 0.02, 3)

        def world_point(xs):
            R, t = link_transform(O, trident, xs, link)
            return R @ p_local + t

        def world_dir(xs):
            R, _ = link_transform(O, trident, xs, link)
            return R[:, 2]

        J = O.hand_jacobian(trident, x, link, world_point(x))
        assert np.abs(J - fd_jacobian(world_point, x)).max() < 5e-6
        Jd = O.hand_jacobian(trident, x, link, world_dir(x), direction=True)
        assert np.abs(Jd - fd_jacobian(world_dir, x)).max() < 5e-6
        assert np.abs(Jd[:, 9:12]).max() == 0.0  # no translation columns


def test_limit_energy_is_a_smooth_hinge_with_exact_gradient(O, trident):
    # test_hand.cpp:185-212.
    q = np.zeros(trident.dof())
    e, _ = O.limit_energy(trident, state(trident, np.eye(3), np.zeros(3), q))
    assert e[0] == 0.0
    q[0] = trident.upper[0] + 0.2
    q[3] = trident.lower[3] - 0.1
    e, g = O.limit_energy(trident, state(trident, np.eye(3), np.zeros(3), q))
    assert e[0] == pytest.approx(0.05, rel=1e-12)
    assert g[0, 12] == pytest.approx(0.4, rel=1e-12)
    assert g[0, 15] == pytest.approx(-0.2, rel=1e-12)
    rng = np.random.default_rng(61)
    for _ in range(10):
        x = random_state(trident, rng)
        x[12:] += 0.5
        _, g = O.limit_energy(trident, x)
        fd = fd_jacobian(lambda xs: O.limit_energy(trident, xs)[0][0], x)
        assert np.abs(g[0] - fd).max() < 1e-6


def test_self_penetration_zero_at_rest_and_differentiable_when_engaged(O, trident):
    # test_hand.cpp:214-252.
    rest = state(trident, np.eye(3), np.zeros(3), np.zeros(trident.dof()))
    assert O.self_penetration_energy(trident, rest)[0][0] == 0.0
    curled = state(trident, np.eye(3), np.zeros(3), trident.upper)
    assert O.self_penetration_energy(trident, curled)[0][0] > 0.0
    rng = np.random.default_rng(67)
    checked = 0
    for _ in range(40):
        if checked == 5:
            break
        x = random_state(trident, rng)
        x[12:] = 0.75 * trident.upper + 0.25 * x[12:]
        e, g = O.self_penetration_energy(trident, x)
        if e[0] < 1e-8:
            continue
        checked += 1
        fd = fd_jacobian(lambda xs: O.self_penetration_energy(trident, xs)[0][0], x)
        assert np.abs(g[0] - fd).max() < 1e-5 * (1.0 + np.linalg.norm(fd))
    assert checked == 5


def test_builtin_hand_tips_are_symmetric(O, trident):
    # test_hand.cpp:254-277.
    assert trident.dof() == 6 and trident.n_links == 7 and trident.n_tips == 3 and trident.n_pairs == 15
    pb = trident.link_proxy_begin

    def tips(q):
        w = O.forward_kinematics(trident, state(trident, np.eye(3), np.zeros(3), q))[0]
        out = []
        for link in trident.fingertip_links:
            c = trident.proxies[pb[link] + trident.link_tip_proxy[link], :3]
            out.append(w[link, :9].reshape(3, 3).T @ c + w[link, 9:])
        return np.array(out)

    t = tips(np.zeros(6))
    assert np.linalg.norm(t[0, :2]) == pytest.approx(np.linalg.norm(t[1, :2]), rel=1e-12)
    assert t[0, 2] == pytest.approx(t[1, 2], rel=1e-12)
    rot = axis_angle(np.array([0.0, 0.0, 2.0 * math.pi / 3.0]))
    assert np.linalg.norm(rot @ t[0] - t[1]) < 1e-12
    assert np.linalg.norm(rot @ t[1] - t[2]) < 1e-12
    assert np.linalg.norm(tips(np.full(6, 0.5))[0, :2]) < np.linalg.norm(t[0, :2])


# -------------------------------------------------------------- test_contact.cpp
def rand_unit(rng, n):
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def test_contact_frame_is_right_handed_orthonormal_and_deterministic(O):
    # test_contact.cpp:34-59.
    rng = np.random.default_rng(71001)
    normals = np.concatenate([rand_unit(rng, 200), [[1, 0, 0], [-1, 0, 0]],
                              [np.array([0.9995, 0.02, 0.0]) / np.linalg.norm([0.9995, 0.02, 0.0])]])
    p = rand_unit(rng, len(normals)) * 0.1
    f = O.build_frame(p, normals)
    assert (f[:, :3] == p).all() and (f[:, 3:6] == normals).all()
    d, e = f[:, 6:9], f[:, 9:12]
    assert np.abs(np.linalg.norm(d, axis=1) - 1).max() < 1e-12
    assert np.abs(np.linalg.norm(e, axis=1) - 1).max() < 1e-12
    for a, b in ((d, normals), (e, normals), (d, e)):
        assert np.abs(np.einsum("ij,ij->i", a, b)).max() < 1e-12
    assert np.abs(np.cross(d, e) - normals).max() < 1e-12
    assert (O.build_frame(p, normals) == f).all()


def test_pyramid_edges_and_wrench_columns(G, O):
    # test_contact.cpp:61-117, 162-185 (grasp_matrix / pyramid_edges are the wrench-basis blocks).
    rng = np.random.default_rng(71003)
    for t in range(50):
        f = O.build_frame(np.zeros(3), rand_unit(rng, 1))[0]
        mu = 0.2 + 0.8 * (t % 5) / 4.0
        k = 3 + t % 8
        W = O.wrench_basis(f, mu, k)
        edges, n, d = W[:3], f[3:6], f[6:9]
        assert np.abs(edges.T @ n - 1.0).max() < 1e-12
        assert np.abs(np.linalg.norm(edges - n[:, None], axis=0) - mu).max() < 1e-12
        assert np.linalg.norm(edges[:, 0] - (n + mu * d)) < 1e-12
        assert np.linalg.norm(edges.sum(axis=1) - k * n) < 1e-10
    f = O.build_frame(np.zeros(3), [0.0, 0.0, 1.0])[0]
    for mu, k in ((0.5, 2), (0.0, 8), (-0.3, 8)):
        with pytest.raises(G.InvalidArgument):
            O.wrench_basis(f, mu, k)
    # torque rows are p x edge; the basis is linear in the weights
    frames = O.build_frame(rng.normal(size=(3, 3)) * 0.1, rand_unit(rng, 3))
    W = O.wrench_basis(frames, 0.6, 8)
    for i in range(3):
        blk = W[:, 8 * i:8 * i + 8]
        assert np.abs(blk[3:] - np.cross(frames[i, :3], blk[:3].T).T).max() < 1e-13
    lam = np.abs(rng.normal(size=24))
    expect = np.zeros(6)
    for i in range(3):
        force = W[:3, 8 * i:8 * i + 8] @ lam[8 * i:8 * i + 8]
        expect[:3] += force
        expect[3:] += np.cross(frames[i, :3], force)
    assert np.linalg.norm(W @ lam - expect) < 1e-12


def test_weighted_edge_forces_stay_in_the_friction_cone(O):
    # test_contact.cpp:119-141.
    rng = np.random.default_rng(71004)
    for _ in range(100):
        f = O.build_frame(np.zeros(3), rand_unit(rng, 1))[0]
        W = O.wrench_basis(f, 0.6, 8)
        lam = rng.uniform(0.0, 1.0, 8)
        force = W[:3] @ lam
        fn = force @ f[3:6]
        assert abs(fn - lam.sum()) < 1e-12
        assert np.linalg.norm(force - fn * f[3:6]) <= 0.6 * fn + 1e-12


# -------------------------------------------------------------- test_qpsolve.cpp
def tight(G, eps, max_iters):
    cfg = G.RunConfig()
    cfg.qp.eps_primal = cfg.qp.eps_dual = eps
    cfg.qp.max_iters = max_iters
    return cfg


def test_separable_box_qp_clamps_the_unconstrained_minimum(G, O):
    # test_qpsolve.cpp:101-120.
    rng = np.random.default_rng(81001)
    n = 8
    for _ in range(20):
        q = rng.normal(0.0, 2.0, n)
        s = O.solve_shared(np.eye(n), np.eye(n), q, np.zeros(n), np.ones(n), tight(G, 1e-9, 100000))
        assert s["converged"][0]
        assert np.abs(s["X"][:, 0] - np.clip(-q, 0.0, 1.0)).max() < 1e-7


def test_pure_equality_constraints_reproduce_the_kkt_solution(G, O):
    # test_qpsolve.cpp:122-156.
    rng = np.random.default_rng(81002)
    n, m = 6, 3
    for _ in range(20):
        b = rng.normal(size=(n, n))
        P = b.T @ b / n + 0.5 * np.eye(n)
        P = 0.5 * (P + P.T)
        q = rng.normal(size=n)
        A = rng.normal(size=(m, n))
        rhs = rng.normal(size=m)
        kkt = np.block([[P, A.T], [A, np.zeros((m, m))]])
        sol = np.linalg.solve(kkt, np.concatenate([-q, rhs]))
        s = O.solve_shared(P, A, q, rhs, rhs, tight(G, 1e-9, 200000))
        assert s["converged"][0]
        assert np.abs(s["X"][:, 0] - sol[:n]).max() < 1e-6
        assert np.abs(A @ s["X"][:, 0] - rhs).max() < 1e-7


def random_shared(rng, n, m, B, delta):
    """test_qpsolve.cpp:39-66."""
    b = rng.normal(size=(n, n))
    P = b.T @ b / n + delta * np.eye(n)
    P = 0.5 * (P + P.T)
    A = rng.normal(size=(m, n))
    Q, L, U = np.zeros((n, B)), np.zeros((m, B)), np.zeros((m, B))
    for c in range(B):
        x_ref = rng.normal(size=n)
        Q[:, c] = rng.normal(size=n)
        z = A @ x_ref
        L[:, c] = z - 0.05 - np.abs(rng.normal(size=m))
        U[:, c] = z + 0.05 + np.abs(rng.normal(size=m))
    return P, A, Q, L, U


def test_batched_solve_tracks_sequential_solves(G, O):
    # test_qpsolve.cpp:207-221: per-column freeze makes every column of the batch identical to
    # its own single-column solve, including the sweep at which it froze.
    rng = np.random.default_rng(81005)
    cfg = tight(G, 1e-8, 100000)
    P, A, Q, L, U = random_shared(rng, 12, 18, 40, 0.3)
    b = O.solve_shared(P, A, Q, L, U, cfg)
    assert len(np.unique(b["iters"])) > 5
    for c in range(40):
        assert b["converged"][c]
        s = O.solve_shared(P, A, Q[:, c], L[:, c], U[:, c], cfg)
        assert s["converged"][0]
        assert np.abs(b["X"][:, c] - s["X"][:, 0]).max() <= 1e-9
        assert np.abs(b["Y"][:, c] - s["Y"][:, 0]).max() <= 1e-9
        assert b["iters"][c] == s["iters"][0]


def test_repeated_solves_are_bitwise_identical(G, O):
    # test_qpsolve.cpp:223-235.
    rng = np.random.default_rng(81006)
    P, A, Q, L, U = random_shared(rng, 10, 14, 8, 0.3)
    a = O.solve_shared(P, A, Q, L, U, tight(G, 1e-8, 100000))
    b = O.solve_shared(P, A, Q, L, U, tight(G, 1e-8, 100000))
    assert (a["X"] == b["X"]).all() and (a["Y"] == b["Y"]).all() and (a["iters"] == b["iters"]).all()


def test_warm_start_at_the_solution_converges_at_the_first_check(G, O):
    # test_qpsolve.cpp:237-250 (random strictly convex problems, x0 = cold solution).
    rng = np.random.default_rng(81007)
    cfg = tight(G, 1e-8, 100000)
    for _ in range(30):
        P, A, Q, L, U = random_shared(rng, 6, 9, 1, 0.3)
        cold = O.solve_shared(P, A, Q, L, U, cfg)
        assert cold["converged"][0]
        warm = O.solve_shared(P, A, Q, L, U, cfg, warm_x=cold["X"], warm_y=cold["Y"])
        assert warm["converged"][0]
        assert warm["iters"][0] <= cfg.qp.check_interval
        assert np.abs(warm["X"] - cold["X"]).max() < 1e-6


def test_iteration_cap_reports_nonconvergence(G, O):
    # test_qpsolve.cpp:280-288.
    rng = np.random.default_rng(81009)
    P, A, Q, L, U = random_shared(rng, 10, 14, 1, 0.1)
    s = O.solve_shared(P, A, Q, L, U, tight(G, 1e-12, 3))
    assert not s["converged"][0] and s["iters"][0] == 3


def test_input_validation_rejects_malformed_problems(G, O):
    # test_qpsolve.cpp:290-299.
    P = np.eye(3)
    P[0, 1] = 0.5
    with pytest.raises(G.InvalidArgument):
        O.solve_shared(P, np.eye(3), np.zeros(3), np.zeros(3), np.ones(3), G.RunConfig())
    with pytest.raises(G.InvalidArgument):
        O.solve_shared(np.eye(3), np.eye(3), np.zeros(3), np.zeros(2), np.ones(2), G.RunConfig())


def ring_frames(O, m, radius):
    """test_qpsolve.cpp:79-88: m inward contacts on a circle."""
    phi = 2.0 * np.pi * np.arange(m) / m
    p = np.stack([radius * np.cos(phi), radius * np.sin(phi), np.zeros(m)], 1)
    return O.build_frame(p, -p / np.linalg.norm(p, axis=1, keepdims=True))


def closure_targets():
    t = np.zeros((6, 6))
    for a in range(3):
        t[a, 2 * a], t[a, 2 * a + 1] = 1.0, -1.0
    return t


def test_lower_qp_assembly_layout(G, O):
    # test_qpsolve.cpp:301-333.
    m, k = 3, 8
    W = O.wrench_basis(ring_frames(O, m, 0.05), 0.6, k)
    b = O.assemble_lower_qp(W, m, closure_targets(), 10.0, 0.3)
    assert b["A"].shape == (m + 1 + m * k, m * k) and b["Q"].shape[1] == 6
    assert np.abs(b["P"] - 2.0 * W.T @ W).max() < 1e-12
    for i in range(m):
        assert b["A"][i].sum() == pytest.approx(k)
        assert b["L"][i, 0] == 0.0 and b["U"][i, 0] == 1.0
    assert b["L"][m, 0] == pytest.approx(0.3) and np.isinf(b["U"][m, 0])
    assert np.linalg.norm(b["A"][m + 1:] - np.eye(m * k)) == 0.0
    assert np.linalg.norm(b["Q"][:, 0] + 2.0 * 10.0 * W.T @ closure_targets()[:, 0]) < 1e-12
    for gamma in (3.5, -0.1):
        with pytest.raises(G.InvalidArgument):
            O.assemble_lower_qp(W, m, closure_targets(), 10.0, gamma)


def test_lower_qp_solutions_are_feasible(G, O):
    # test_qpsolve.cpp:335-383 (feasibility part; the certified bracket needs the reference's
    # active-set oracle, replaced here by the floor/caps/nonnegativity checks it also makes).
    m, k, gamma = 3, 8, 0.3
    W = O.wrench_basis(ring_frames(O, m, 0.05), 0.6, k)
    b = O.assemble_lower_qp(W, m, closure_targets(), 10.0, gamma)
    s = O.solve_shared(b["P"], b["A"], b["Q"], b["L"], b["U"], tight(G, 1e-10, 400000))
    assert s["converged"].all()
    lam = s["X"]
    assert lam.min() >= -1e-8
    blocks = lam.reshape(m, k, 6).sum(axis=1)
    assert blocks.min() >= -1e-8 and blocks.max() <= 1.0 + 1e-8
    assert lam.sum(axis=0).min() >= gamma - 1e-8


def test_positive_floor_forces_nonzero_weights(G, O):
    # test_qpsolve.cpp:385-395.
    m, k = 3, 8
    W = O.wrench_basis(ring_frames(O, m, 0.05), 0.6, k)
    b = O.assemble_lower_qp(W, m, np.zeros((6, 1)), 10.0, 0.3)
    s = O.solve_shared(b["P"], b["A"], b["Q"], b["L"], b["U"], tight(G, 1e-9, 200000))
    assert s["converged"][0]
    assert s["X"][:, 0].sum() >= 0.3 - 1e-7 and s["X"][:, 0].min() >= -1e-8


# --------------------------------------------------------------- test_energy.cpp
def energy_cfg(G, beta, gamma):
    cfg = G.RunConfig()
    cfg.qp.eps_primal = cfg.qp.eps_dual = 1e-9
    cfg.qp.max_iters = 200000
    cfg.energy.beta, cfg.energy.gamma_per_contact = beta, gamma
    return cfg


def random_contacts(O, rng, m):
    """test_energy.cpp:82-91."""
    p = rng.uniform(0.4, 1.2, (m, 1)) * rand_unit(rng, m)
    n = -p + 0.4 * rand_unit(rng, m)
    return O.build_frame(p, n / np.linalg.norm(n, axis=1, keepdims=True))


def test_per_direction_energies_sum_to_the_total(G, O):
    # test_energy.cpp:224-251.
    rng = np.random.default_rng(91004)
    for trial in range(12):
        m = 1 + trial % 5
        beta = (0.0, 0.5, 10.0)[trial % 3]
        fr = random_contacts(O, rng, m)
        r = O.grasp_energy(energy_cfg(G, beta, 0.1), fr)
        assert r["converged"].all()
        assert r["per_direction"].min() >= 0.0
        assert abs(r["total"] - r["per_direction"].sum()) <= 1e-9
        W = O.wrench_basis(fr, 0.6, 8)
        for j in range(6):
            res = beta * closure_targets()[:, j] - W @ r["forces"][:, j]
            assert np.linalg.norm(res - r["residuals"][:, j]) <= 1e-12
            assert r["per_direction"][j] == pytest.approx(res @ res, rel=1e-12)


def test_rotating_contacts_and_targets_preserves_every_energy(G, O):
    # test_energy.cpp:253-282.
    rng = np.random.default_rng(91005)
    for _ in range(8):
        fr = random_contacts(O, rng, 3)
        rot = axis_angle(1.5 * rand_unit(rng, 1)[0])
        turned = fr.copy()
        for s in range(4):
            turned[:, 3 * s:3 * s + 3] = fr[:, 3 * s:3 * s + 3] @ rot.T
        T = closure_targets()
        TT = np.concatenate([rot @ T[:3], rot @ T[3:]])
        a = O.grasp_energy(energy_cfg(G, 10.0, 0.1), fr)
        b = O.grasp_energy(energy_cfg(G, 10.0, 0.1), turned, targets=TT)
        assert a["converged"].all() and b["converged"].all()
        assert np.abs(a["per_direction"] - b["per_direction"]).max() <= 1e-8


def test_pure_torque_target_on_zero_moment_arm_costs_beta_squared(G, O):
    # test_energy.cpp:284-297.
    fr = O.build_frame(np.zeros(3), [0.0, 0.0, 1.0])
    r = O.grasp_energy(energy_cfg(G, 0.8, 0.0), fr, targets=np.array([[0, 0, 0, 1, 0, 0]], float).T)
    assert r["converged"].all()
    assert r["total"] == pytest.approx(0.64, rel=1e-8)


def test_closure_energy_zero_while_targets_reachable(G, O):
    # test_energy.cpp:299-322 (sphere tripod; the grid certificate is replaced by the energy itself).
    c = []
    for i in range(3):
        az, el = 2.0 * np.pi * i / 3.0, (0.7 if i == 0 else -0.35)
        c.append([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az), np.sin(el)])
    p = np.array(c)
    fr = O.build_frame(p, -p)
    for beta in (0.05, 0.2, 0.5):
        r = O.grasp_energy(energy_cfg(G, beta, 0.0), fr)
        assert r["converged"].all() and r["total"] <= 1e-6
    assert O.grasp_energy(energy_cfg(G, 10.0, 0.0), fr)["total"] > 1.0


def frames_at(O, p0, u0, x):
    m = len(p0)
    p = p0 + x.reshape(m, 6)[:, :3]
    n = u0 + x.reshape(m, 6)[:, 3:]
    return O.build_frame(p, n / np.linalg.norm(n, axis=1, keepdims=True))


def test_envelope_gradient_matches_finite_differences(G, O):
    # test_energy.cpp:324-376: d(total)/d(contact points, normals) with lambda* fixed vs central
    # differences of the bilevel value (h = 1e-4); one active-set switch tolerated.
    rng = np.random.default_rng(91008)
    cfg = energy_cfg(G, 10.0, 0.1)
    ok = trials = 0
    for t in range(12):
        m = 2 + t % 2
        base = random_contacts(O, rng, m)
        p0, u0 = base[:, :3], base[:, 3:6]
        dims = 6 * m
        fr = frames_at(O, p0, u0, np.zeros(dims))
        rep = O.grasp_energy(cfg, fr)
        assert rep["converged"].all()
        jp, jn = np.zeros((m, 3, dims)), np.zeros((m, 3, dims))
        for i in range(m):
            jp[i][:, 6 * i:6 * i + 3] = np.eye(3)
            n = fr[i, 3:6]
            jn[i][:, 6 * i + 3:6 * i + 6] = (np.eye(3) - np.outer(n, n)) / np.linalg.norm(u0[i])
        grad = O.grasp_energy_gradient(cfg, fr, rep, jp, jn)
        fd = fd_jacobian(lambda xx: O.grasp_energy(cfg, frames_at(O, p0, u0, xx))["total"], np.zeros(dims), 1e-4)
        trials += 1
        ok += np.linalg.norm(grad - fd) / max(np.linalg.norm(fd), 1e-6) <= 1e-2
    assert ok >= trials - 1


def test_gradient_vanishes_at_a_symmetric_closure_optimum(G, O):
    # test_energy.cpp:378-395.
    rng = np.random.default_rng(91009)
    fr = O.build_frame([[1.0, 0, 0], [-1.0, 0, 0]], [[-1.0, 0, 0], [1.0, 0, 0]])
    rep = O.grasp_energy(energy_cfg(G, 0.8, 0.0), fr)
    assert rep["converged"].all() and rep["total"] <= 1e-8
    g = O.grasp_energy_gradient(energy_cfg(G, 0.8, 0.0), fr, rep, rng.normal(size=(2, 3, 9)), rng.normal(size=(2, 3, 9)))
    assert np.linalg.norm(g) <= 1e-6


def test_uniform_translation_gradient_equals_the_torque_row_term(G, O):
    # test_energy.cpp:397-435.
    rng = np.random.default_rng(91010)
    cfg = energy_cfg(G, 10.0, 0.1)
    fr = random_contacts(O, rng, 3)
    rep = O.grasp_energy(cfg, fr)
    assert rep["converged"].all()
    g = O.grasp_energy_gradient(cfg, fr, rep, np.tile(np.eye(3), (3, 1, 1)), np.zeros((3, 3, 3)))
    W = O.wrench_basis(fr, 0.6, 8)
    expect = np.zeros(3)
    for j in range(6):
        rt = rep["residuals"][3:, j]
        for i in range(3):
            f = W[:3, 8 * i:8 * i + 8] @ rep["forces"][8 * i:8 * i + 8, j]
            expect -= 2.0 * np.cross(f, rt)
    assert np.linalg.norm(g - expect) <= 1e-10 * max(1.0, np.linalg.norm(expect))
    h = 1e-4
    fd = np.zeros(3)
    for a in range(3):
        up, dn = fr.copy(), fr.copy()
        up[:, a] += h
        dn[:, a] -= h
        fd[a] = (O.grasp_energy(cfg, up)["total"] - O.grasp_energy(cfg, dn)["total"]) / (2 * h)
    assert np.linalg.norm(g - fd) <= 1e-2 * max(np.linalg.norm(fd), 1e-6)


def test_fine_stage_surrogate_value_and_rigid_motion_gradient(O):
    # test_energy.cpp:516-564.
    same = np.tile([0.2, -0.1, 0.4], (3, 1))
    assert O.stage_surrogate(same, same)[0] == 0.0
    moved = same.copy()
    moved[1, 2] += 1.0
    assert O.stage_surrogate(moved, same)[0] == pytest.approx(1.0)
    rng = np.random.default_rng(91014)
    for _ in range(10):
        body, anchors = rng.normal(size=(4, 3)), rng.normal(size=(4, 3))

        def points_at(x):
            return body @ axis_angle(x[:3]).T + x[3:]

        jac = np.zeros((4, 3, 6))
        for i, b in enumerate(body):
            jac[i][:, :3] = np.array([[0, b[2], -b[1]], [-b[2], 0, b[0]], [b[1], -b[0], 0]])
            jac[i][:, 3:] = np.eye(3)
        _, g = O.stage_surrogate(points_at(np.zeros(6)), anchors, jac)
        fd = fd_jacobian(lambda xx: O.stage_surrogate(points_at(xx), anchors)[0], np.zeros(6), 1e-5)
        assert np.linalg.norm(g - fd) <= 1e-6 * max(np.linalg.norm(fd), 1.0)


def test_warm_start_at_previous_solution_reproduces_it(G, O):
    # test_energy.cpp:584-600.
    c = []
    for i in range(3):
        az, el = 2.0 * np.pi * i / 3.0, (0.7 if i == 0 else -0.35)
        c.append([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az), np.sin(el)])
    p = np.array(c)
    fr = O.build_frame(p, -p)
    cfg = energy_cfg(G, 10.0, 0.1)
    cold = O.grasp_energy(cfg, fr)
    warm = O.grasp_energy(cfg, fr, warm_x=cold["forces"], warm_y=cold["duals"])
    assert cold["converged"].all() and warm["converged"].all()
    assert np.abs(warm["forces"] - cold["forces"]).max() <= 1e-9
    assert abs(warm["total"] - cold["total"]) <= 1e-6


# ------------------------------------------------------------- test_pipeline.cpp
def tip_center(O, hand, x, f):
    link = hand.fingertip_links[f]
    R, t = link_transform(O, hand, x, link)
    c = hand.proxies[hand.link_proxy_begin[link] + hand.link_tip_proxy[link], :3]
    return R @ c + t


def test_coarse_distance_gradient_matches_central_differences(G, O, trident):
    # test_pipeline.cpp:136-174.
    box = G.make_primitive("box", 0.1)
    lo, hi = box.bounding_box()
    rng = np.random.default_rng(331)
    mid = 0.5 * (trident.lower + trident.upper)
    tested = 0
    for _ in range(400):
        if tested == 20:
            break
        q = mid + 0.2 * rng.uniform(-1, 1, trident.dof())
        tip0 = tip_center(O, trident, state(trident, np.eye(3), np.zeros(3), q), 0)
        target = np.array([0.01 * rng.uniform(-1, 1), 0.01 * rng.uniform(-1, 1),
                           hi[2] + 0.012 + 0.012 * (rng.uniform(-1, 1) + 1.2)])
        x = state(trident, np.eye(3), target - tip0, q)
        interior = all(c[2] > hi[2] + 2e-3 and abs(c[0]) < 0.8 * hi[0] and abs(c[1]) < 0.8 * hi[1]
                       for c in (tip_center(O, trident, x, f) for f in range(3)))
        if not interior:
            continue
        tested += 1
        _, g = O.coarse_distance_energy(trident, box, x, 0.01, 1e-6)
        fd = fd_jacobian(lambda xx: O.coarse_distance_energy(trident, box, xx, 0.01, 1e-6, with_grad=False)[0][0], x)
        assert np.linalg.norm(g[0] - fd) <= 1e-3 * max(1.0, np.linalg.norm(fd))
    assert tested == 20


def flipped_state(hand, angle, t):
    return state(hand, axis_angle(np.array([angle, 0.0, 0.0])), t, np.zeros(hand.dof()))


def test_fine_contact_query_reports_aligned_witnesses(G, O, trident):
    # test_pipeline.cpp:176-216.
    sphere = G.make_primitive("sphere", 0.1)
    radius = sphere.bounding_radius()
    for drop in (0.175, 0.160, 0.148):
        x = flipped_state(trident, np.pi, [0.0, 0.0, drop])
        w = O.fine_contact_query(trident, sphere, x)[0]
        for f in range(3):
            c = tip_center(O, trident, x, f)
            cw, pw, n, d, link = w[f, 0:3], w[f, 3:6], w[f, 6:9], w[f, 9], w[f, 10]
            assert link == trident.fingertip_links[f]
            assert abs(d - (np.linalg.norm(c) - radius - 0.010)) <= 0.004
            u = c / np.linalg.norm(c)
            assert np.linalg.norm(pw - (pw @ u) * u) <= 0.008
            assert np.linalg.norm(cw - (cw @ u) * u) <= 0.008
            assert n @ u >= 0.9
            assert np.linalg.norm(cw - pw) == pytest.approx(abs(d), rel=1e-9)
    deep = O.fine_contact_query(trident, sphere, flipped_state(trident, np.pi, [0.0, 0.0, 0.130]))[0]
    assert (deep[:, 9] < 0).sum() >= 1


def test_culled_query_equals_the_exhaustive_query(G, O, trident):
    # test_pipeline.cpp:218-260 (200 scenes; three separated boxes).
    from test_models import three_box_obj
    obj = G.parse_object_text(three_box_obj(), 0.12, "three_boxes")
    assert obj.n_parts == 3
    rng = np.random.default_rng(77)
    mid = 0.5 * (trident.lower + trident.upper)
    xs = np.array([state(trident, rand_rotation(rng), rng.uniform(-1, 1, 3) * 0.12,
                         mid + 0.3 * rng.uniform(-1, 1, trident.dof())) for _ in range(200)])
    fast = O.fine_contact_query(trident, obj, xs)
    world = O.forward_kinematics(trident, xs)
    links = np.repeat(trident.fingertip_links, 3)
    parts = np.tile(np.arange(3), 3)
    disagreements = 0
    for s in range(200):
        r = O.signed_distance(trident, obj, links, parts, world[s][links])
        for f in range(3):
            rows = r[3 * f:3 * f + 3]
            best = int(np.argmin(rows[:, 0]))  # first minimum: smallest index wins ties
            same = fast[s, f, 9] == rows[best, 0] and (fast[s, f, 0:3] == rows[best, 1:4]).all() and \
                (fast[s, f, 3:6] == rows[best, 4:7]).all()
            disagreements += not same
    assert disagreements == 0


def test_surrogate_gradient_uses_detached_witnesses(G, O, trident):
    # test_pipeline.cpp:262-311.
    sphere = G.make_primitive("sphere", 0.1)
    radius = sphere.bounding_radius()
    x = flipped_state(trident, 0.5 * np.pi, [0.0, -(radius + 0.020), -0.06])
    w = O.fine_contact_query(trident, sphere, x)[0]
    links = w[:, 10].astype(np.int32)
    anchors = w[:, 3:6] + np.array([0.02, 0.01, -0.015])
    value, grad = O.fine_grasp_surrogate(trident, x, w[:, 0:3], links, anchors)
    world = O.forward_kinematics(trident, x)[0]
    frozen = [world[l, :9].reshape(3, 3) @ (w[i, 0:3] - world[l, 9:]) for i, l in enumerate(links)]

    def fixed_value(xx):
        ww = O.forward_kinematics(trident, xx)[0]
        return sum(np.sum((ww[l, :9].reshape(3, 3).T @ frozen[i] + ww[l, 9:] - anchors[i]) ** 2)
                   for i, l in enumerate(links))

    assert abs(fixed_value(x) - value) <= 1e-12 * max(1.0, value)
    fd_fixed = fd_jacobian(fixed_value, x)
    assert np.linalg.norm(grad - fd_fixed) <= 1e-5 * max(1.0, np.linalg.norm(fd_fixed))

    def requery_value(xx):
        ws = O.fine_contact_query(trident, sphere, xx)[0]
        return float(np.sum((ws[:, 0:3] - anchors) ** 2))

    fd_requery = fd_jacobian(requery_value, x)
    assert np.linalg.norm(fd_requery - grad) > 1e-2 * max(1.0, np.linalg.norm(grad))
