"""Host-side pipeline pieces: init_poses and squeeze_pose (pipeline.cpp:388-434),
RunConfig parsing/validation (config.cpp:139-229). Expectations follow
proj/tests/test_pipeline.cpp:313-397 and test_records/config behaviour."""
import json
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation


def test_init_poses_aim_at_the_object_and_cover_directions(G, trident):
    sphere = G.make_primitive("sphere", 0.08)
    params = G.InitParams()
    states = G.init_poses(trident, sphere, 1000, 99, params)
    lo, hi = sphere.bounding_box()
    ring = sphere.bounding_radius() + params.standoff
    octants = np.zeros(8, int)
    for x in states:
        R = x[:9].reshape(3, 3).T
        t = x[9:12]
        assert np.linalg.norm(t) == pytest.approx(ring, rel=1e-9)
        assert ((t < lo) | (t > hi)).any()
        assert R[:, 2] @ (-t / np.linalg.norm(t)) == pytest.approx(1.0, rel=1e-9)
        assert np.linalg.norm(R.T @ R - np.eye(3)) <= 1e-9
        q = x[12:]
        assert (q >= trident.lower - 1e-12).all() and (q <= trident.upper + 1e-12).all()
        mid = 0.5 * (trident.lower + trident.upper)
        assert (np.abs(q - mid) <= 0.5 * params.joint_span_fraction * (trident.upper - trident.lower) + 1e-12).all()
        octants[int(t[0] > 0) + 2 * int(t[1] > 0) + 4 * int(t[2] > 0)] += 1
    chi2 = ((octants - 125.0) ** 2 / 125.0).sum()
    assert chi2 < 18.4753
    again = G.init_poses(trident, sphere, 1000, 99, params)
    assert np.array_equal(states, again)
    assert not np.array_equal(G.init_poses(trident, sphere, 10, 100, params)[0], states[0])


def test_init_poses_prefix_independent(G, trident):
    sphere = G.make_primitive("sphere", 0.1)
    a = G.init_poses(trident, sphere, 64, 17)
    b = G.init_poses(trident, sphere, 16, 17)
    assert np.array_equal(a[:16], b)


def state(trident, R, t, q):
    x = np.zeros(trident.dims())
    x[:9] = np.asarray(R).T.reshape(9)
    x[9:12] = t
    x[12:] = q
    return x


def test_squeeze_pose_extrapolates_and_clamps(G, trident):
    # test_pipeline.cpp:358-397.
    Rz = lambda a: Rotation.from_rotvec([0, 0, a]).as_matrix()
    n = trident.dof()
    x_p = state(trident, Rz(0.3), (0.01, -0.02, 0.03), np.full(n, 0.2))
    x = state(trident, Rz(0.5), (0.03, -0.02, 0.01), np.full(n, 0.3))
    s = G.squeeze_pose(trident, x, x_p)
    np.testing.assert_allclose(s[9:12], (0.05, -0.02, -0.01), atol=1e-12)
    np.testing.assert_allclose(s[12:], 0.4, rtol=1e-12)
    np.testing.assert_allclose(s[:9].reshape(3, 3).T, Rz(0.7), atol=1e-9)
    same = G.squeeze_pose(trident, x, x)
    np.testing.assert_allclose(same, x, atol=1e-12)
    hi_q = trident.upper - 0.01
    clamped = G.squeeze_pose(trident, state(trident, Rz(0.5), (0, 0, 0), hi_q),
                             state(trident, Rz(0.5), (0, 0, 0), hi_q - 0.5))
    np.testing.assert_allclose(clamped[12:], trident.upper, rtol=1e-12)


def test_run_config_defaults_match_reference(G):
    cfg = G.RunConfig()
    assert (cfg.qp.rho, cfg.qp.sigma, cfg.qp.alpha, cfg.qp.max_iters) == (0.1, 1e-6, 1.6, 500)
    assert (cfg.qp.eps_primal, cfg.qp.eps_dual, cfg.qp.check_interval) == (1e-5, 1e-5, 10)
    assert (cfg.contact.mu, cfg.contact.n_edges) == (0.6, 8)
    assert (cfg.energy.beta, cfg.energy.gamma_per_contact) == (10.0, 0.1)
    assert (cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters) == (300, 100, 100)
    assert cfg.pipeline.contact_offset == 0.01 and cfg.pipeline.fd_step == 1e-6
    assert (cfg.seed, cfg.batch, cfg.workers) == (0, 64, 1)
    G.validate(cfg)


def test_run_config_parse_is_strict(G):
    cfg = G.parse_run_config(json.dumps({"qp": {"rho": 0.2}, "pipeline": {"coarse": {"iters": 7}}, "batch": 9}))
    assert cfg.qp.rho == 0.2 and cfg.pipeline.coarse.iters == 7 and cfg.batch == 9
    assert cfg.qp.sigma == 1e-6  # untouched default
    for bad in ({"qp": {"rhoo": 1}}, {"unknown": 1}, {"pipeline": {"coarse": {"iterz": 3}}}):
        with pytest.raises(G.InvalidArgument):
            G.parse_run_config(json.dumps(bad))


@pytest.mark.parametrize("path,value", [("qp.rho", 0.0), ("qp.alpha", 2.0), ("contact.n_edges", 2),
                                        ("energy.gamma_per_contact", 1.5), ("pipeline.fd_step", 0.0),
                                        ("batch", 0), ("pipeline.coarse.step_floor", 0.0)])
def test_validate_rejects_out_of_range(G, path, value):
    cfg = G.RunConfig()
    obj = cfg
    parts = path.split(".")
    for p in parts[:-1]:
        obj = getattr(obj, p)
    setattr(obj, parts[-1], value)
    with pytest.raises(G.InvalidArgument):
        G.validate(cfg)
