"""ORACLE bindings (test infrastructure only).

ctypes access to oracle/_build/liboracle_grasp.so, the fp64 CPU restatement
of the reference hot path. Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module; the
product path (paper_2412_16490_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
LIB_PATH = ROOT / "_build" / "liboracle_grasp.so"

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_longlong)
_vp = C.c_void_p

STAT_NAMES = ("point_queries", "inside_faces", "outside_faces", "gjk_calls", "gjk_iters", "gjk_support_verts",
              "epa_calls", "epa_iters", "epa_face_scans", "qp_solves", "qp_sweeps", "qp_column_sweeps",
              "jacobians", "self_pairs", "obb_tests")

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(ROOT)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        sig = {
            "oracle_last_error": (C.c_char_p, []),
            "oracle_point_to_mesh": (C.c_int, [_vp, C.c_int, _dp, _dp]),
            "oracle_part_pairs": (C.c_int, [_vp, _vp, C.c_int, _ip, _ip, _dp, _dp, C.c_int, _dp]),
            "oracle_signed_distance": (C.c_int, [_vp, _vp, C.c_int, _ip, _ip, _dp, _dp]),
            "oracle_total_energy": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _ip, _dp, _dp,
                                              _dp, _ip, _ip, C.c_int]),
            "oracle_forward_kinematics": (C.c_int, [_vp, C.c_int, _dp, _dp]),
            "oracle_project_rotation": (C.c_int, [C.c_int, _dp, _dp, _ip]),
            "oracle_pose_state": (C.c_int, [C.c_int, _dp, _dp, _dp, _ip, _dp]),
            "oracle_hand_jacobian": (C.c_int, [_vp, _dp, C.c_int, _dp, C.c_int, _dp]),
            "oracle_hand_energy": (C.c_int, [_vp, C.c_int, C.c_int, _dp, _dp, _dp]),
            "oracle_build_frame": (C.c_int, [C.c_int, _dp, _dp, _dp]),
            "oracle_wrench_basis": (C.c_int, [C.c_int, _dp, C.c_double, C.c_int, _dp]),
            "oracle_assemble_lower_qp": (C.c_int, [_dp, C.c_int, C.c_int, _dp, C.c_int, C.c_double, C.c_double,
                                                   _dp, _dp, _dp, _dp, _dp]),
            "oracle_solve_shared": (C.c_int, [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, _ip, _vp, _dp,
                                              _dp, _dp, _dp, _dp, _ip, _ip]),
            "oracle_grasp_energy": (C.c_int, [_vp, C.c_int, _dp, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                              _ip, _ip]),
            "oracle_grasp_energy_gradient": (C.c_int, [_vp, C.c_int, _dp, _dp, _dp, C.c_int, _dp, _dp, _dp]),
            "oracle_stage_surrogate": (C.c_int, [C.c_int, _dp, _dp, C.c_int, _dp, _dp, _dp]),
            "oracle_fine_grasp_surrogate": (C.c_int, [_vp, _dp, C.c_int, _dp, _ip, _dp, _dp, _dp]),
            "oracle_apply_step": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _dp, _dp]),
            "oracle_coarse_distance_energy": (C.c_int, [_vp, _vp, C.c_int, _dp, C.c_double, C.c_double, _dp, _dp]),
            "oracle_fine_contact_query": (C.c_int, [_vp, _vp, C.c_int, _dp, _dp]),
            "oracle_qp_batch": (C.c_int, [_vp, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _ip, _ip, _dp,
                                          C.c_int]),
            "oracle_synthesize": (C.c_int, [_vp, _vp, _vp, C.c_int, _dp, C.c_int, _vp, _lp]),
            "oracle_eval": (C.c_int, [_vp, _vp, _vp, _dp, C.c_int, _dp, _dp, _dp, _ip]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status):
    if status != 0:
        msg = lib().oracle_last_error().decode(errors="replace")
        from paper_2412_16490_b200.errors import raise_for
        raise_for(status, msg)


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _i(a):
    return None if a is None else a.ctypes.data_as(_ip)


def ref(s):
    return C.cast(C.pointer(s), _vp)


def point_to_mesh(obj, points) -> np.ndarray:
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    out = np.zeros((len(pts), 8))
    _check(lib().oracle_point_to_mesh(ref(obj.desc), len(pts), _d(pts), _d(out)))
    return out


def part_pairs(obj_a, obj_b, ia, ib, poses_a, poses_b, kind=0) -> np.ndarray:
    ia = np.ascontiguousarray(ia, dtype=np.int32)
    ib = np.ascontiguousarray(ib, dtype=np.int32)
    pa = np.ascontiguousarray(poses_a, dtype=np.float64).reshape(-1, 12)
    pb = np.ascontiguousarray(poses_b, dtype=np.float64).reshape(-1, 12)
    out = np.zeros((len(ia), 11))
    _check(lib().oracle_part_pairs(ref(obj_a.desc), ref(obj_b.desc), len(ia), _i(ia), _i(ib), _d(pa), _d(pb), kind,
                                   _d(out)))
    return out


def signed_distance(hand, obj, link_ids, part_ids, poses) -> np.ndarray:
    li = np.ascontiguousarray(link_ids, dtype=np.int32)
    pi = np.ascontiguousarray(part_ids, dtype=np.int32)
    ps = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 12)
    out = np.zeros((len(li), 11))
    _check(lib().oracle_signed_distance(ref(hand.desc), ref(obj.desc), len(li), _i(li), _i(pi), _d(ps), _d(out)))
    return out


def total_energy(hand, obj, cfg, stage, x, anchors=None, warm_x=None, warm_y=None, with_grad=True,
                 warm_ready=None, qp_stats=False, threads=None, world=None):
    """total_energy (pipeline.cpp:96-210) per grasp. warm_x/warm_y (updated in place) are
    the coarse QP's warm start, used for grasps with warm_ready != 0 (all when None).
    With qp_stats, also returns the coarse QP's per-column (iters, converged). world
    ((n, L, 12), R column-major) teacher-forces the link transforms instead of the oracle's FK."""
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, hand.dims())
    n = len(x)
    energy = np.zeros(n)
    grad = np.zeros_like(x) if with_grad else None
    anc = None if anchors is None else np.ascontiguousarray(anchors, dtype=np.float64)
    rdy = None if warm_ready is None else np.ascontiguousarray(warm_ready, dtype=np.int32)
    its = np.zeros((n, 6), np.int32) if qp_stats else None
    conv = np.zeros((n, 6), np.int32) if qp_stats else None
    for a in (warm_x, warm_y):
        assert a is None or (a.flags.c_contiguous and a.dtype == np.float64)
    p = cfg.to_params()
    nt = threads if threads is not None else (os.cpu_count() or 1)
    wd = None if world is None else np.ascontiguousarray(world, dtype=np.float64)
    _check(lib().oracle_total_energy(ref(hand.desc), ref(obj.desc), ref(p), stage, n, _d(x), _d(anc), _d(warm_x),
                                     _d(warm_y), _i(rdy), _d(wd), _d(energy), _d(grad), _i(its), _i(conv), int(nt)))
    if qp_stats:
        return energy, grad, its, conv
    return energy, grad


def forward_kinematics(hand, x) -> np.ndarray:
    """forward_kinematics(pose_from_state(x)) (hand.cpp:108-153) -> (n, L, 12) world R (column-major), t."""
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, hand.dims())
    out = np.zeros((len(x), hand.n_links, 12))
    _check(lib().oracle_forward_kinematics(ref(hand.desc), len(x), _d(x), _d(out)))
    return out


def apply_step(hand, stage_params, it, grad, x):
    from paper_2412_16490_b200 import _native as N
    s = stage_params
    sp = N.StageParams(s.iters, s.step_rotation, s.step_translation, s.step_joints, s.step_floor)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, hand.dims()).copy()
    g = np.ascontiguousarray(grad, dtype=np.float64).reshape(-1, hand.dims())
    _check(lib().oracle_apply_step(ref(hand.desc), ref(sp), int(it), len(x), _d(g), _d(x)))
    return x


def coarse_distance_energy(hand, obj, x, offset, fd_step, with_grad=True):
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, hand.dims())
    e = np.zeros(len(x))
    g = np.zeros_like(x) if with_grad else None
    _check(lib().oracle_coarse_distance_energy(ref(hand.desc), ref(obj.desc), len(x), _d(x), offset, fd_step, _d(e),
                                               _d(g)))
    return e, g


def fine_contact_query(hand, obj, x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, hand.dims())
    out = np.zeros((len(x), hand.n_tips, 11))
    _check(lib().oracle_fine_contact_query(ref(hand.desc), ref(obj.desc), len(x), _d(x), _d(out)))
    return out


def qp_batch(cfg, frames, m, warm_x=None, warm_y=None, threads=1):
    frames = np.ascontiguousarray(frames, dtype=np.float64)
    g = frames.size // (m * 12)
    n = m * cfg.contact.n_edges
    M = m + 1 + n
    X = np.zeros((g, 6, n))
    Y = np.zeros((g, 6, M))
    Z = np.zeros((g, 6, M))
    iters = np.zeros((g, 6), dtype=np.int32)
    conv = np.zeros((g, 6), dtype=np.int32)
    per = np.zeros((g, 6))
    p = cfg.to_params()
    _check(lib().oracle_qp_batch(ref(p), g, m, _d(frames), _d(warm_x), _d(warm_y), _d(X), _d(Y), _d(Z), _i(iters),
                                 _i(conv), _d(per), int(threads)))
    return dict(X=X, Y=Y, Z=Z, iters=iters, converged=conv, per_direction=per)


def evaluate(hand, obj, cfg, x, x_s):
    """quasi_static_check per grasp (eval.cpp:91-158) -> dict of arrays; notes as flags
    (1 no contacts, 2 qp unconverged, 4 residual above tol, 8 < 2 contacts, 16 penetration)."""
    x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
    x_s = np.ascontiguousarray(np.atleast_2d(x_s), dtype=np.float64)
    n = len(x)
    e = cfg.eval
    ev = np.array([e.mass, e.gravity, e.residual_rel_tol, e.force_budget_factor, e.contact_tol, e.penetration_tol,
                   e.qp_eps])
    real = np.zeros((n, 9))
    ints = np.zeros((n, 3), dtype=np.int32)
    p = cfg.to_params()
    _check(lib().oracle_eval(ref(hand.desc), ref(obj.desc), ref(p), _d(ev), n, _d(x), _d(x_s), _d(real), _i(ints)))
    return dict(pd_mm=real[:, 0], spd_mm=real[:, 1], cdc_mm=real[:, 2], residuals=real[:, 3:9],
                contact_count=ints[:, 0], success=ints[:, 1].astype(bool), note_flags=ints[:, 2])


def synthesize(hand, obj, cfg, x0, workers=1, with_stats=False):
    """oracle run over caller x0 -> SynthesisOutput (+ op counters)."""
    from paper_2412_16490_b200.api import SynthesisOutput
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    out = SynthesisOutput(len(x0), hand.dims(), hand.n_tips, cfg.contact.n_edges)
    s = out.as_struct()
    stats = np.zeros(len(STAT_NAMES), dtype=np.int64) if with_stats else None
    p = cfg.to_params()
    _check(lib().oracle_synthesize(ref(hand.desc), ref(obj.desc), ref(p), len(x0), _d(x0), int(workers), ref(s),
                                   None if stats is None else stats.ctypes.data_as(_lp)))
    if with_stats:
        return out, dict(zip(STAT_NAMES, (int(v) for v in stats)))
    return out


# ------------------------------------------------------------------------------
# Fine-grained entry points for the reference's own KATs (oracle/src/kats.cpp).
def _f(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


def _colmajor(M):
    """3x3 (or (n, 3, 3)) row-index matrices -> column-major 9-vectors."""
    M = np.asarray(M, dtype=np.float64)
    return np.ascontiguousarray(M.swapaxes(-1, -2).reshape(M.shape[:-2] + (9,)))


def _from_colmajor(v):
    v = np.asarray(v)
    return v.reshape(v.shape[:-1] + (3, 3)).swapaxes(-1, -2)


def project_rotation(raw):
    """hand.cpp:45-73 on (n, 3, 3) -> (R (n, 3, 3), fallback (n,))."""
    raw = np.asarray(raw, dtype=np.float64).reshape(-1, 3, 3)
    n = len(raw)
    R = np.zeros((n, 9))
    fb = np.zeros(n, np.int32)
    _check(lib().oracle_project_rotation(n, _d(_colmajor(raw)), _d(R), _i(fb)))
    return _from_colmajor(R), fb.astype(bool)


def pose_state(raw):
    """make_pose_state + rotation_tangent_jacobian (hand.cpp:75-106) -> R, a_inv, degenerate, J (n, 3, 9)."""
    raw = np.asarray(raw, dtype=np.float64).reshape(-1, 3, 3)
    n = len(raw)
    R, ai, J = np.zeros((n, 9)), np.zeros((n, 9)), np.zeros((n, 3, 9))
    dg = np.zeros(n, np.int32)
    _check(lib().oracle_pose_state(n, _d(_colmajor(raw)), _d(R), _d(ai), _i(dg), _d(J)))
    return _from_colmajor(R), _from_colmajor(ai), dg.astype(bool), J


def hand_jacobian(hand, x, link, vec, direction=False):
    """point_jacobian (hand.cpp:155-169) or direction_jacobian (:171-183) -> (3, D)."""
    x = _f(x)
    J = np.zeros((3, hand.dims()))
    _check(lib().oracle_hand_jacobian(ref(hand.desc), _d(x), int(link), _d(_f(vec)), 1 if direction else 0, _d(J)))
    return J


def limit_energy(hand, x):
    """hand.cpp:207-218 on states (n, D) -> (e, grad)."""
    x = _f(x).reshape(-1, hand.dims())
    e, g = np.zeros(len(x)), np.zeros_like(x)
    _check(lib().oracle_hand_energy(ref(hand.desc), 0, len(x), _d(x), _d(e), _d(g)))
    return e, g


def self_penetration_energy(hand, x):
    """hand.cpp:220-245 on states (n, D) -> (e, grad)."""
    x = _f(x).reshape(-1, hand.dims())
    e, g = np.zeros(len(x)), np.zeros_like(x)
    _check(lib().oracle_hand_energy(ref(hand.desc), 1, len(x), _d(x), _d(e), _d(g)))
    return e, g


def build_frame(p, n):
    """contact.cpp:13-21 -> (k, 12) rows p n d e."""
    p = _f(p).reshape(-1, 3)
    n = _f(n).reshape(-1, 3)
    out = np.zeros((len(p), 12))
    _check(lib().oracle_build_frame(len(p), _d(p), _d(n), _d(out)))
    return out


def wrench_basis(frames, mu, k):
    """contact.cpp:47-53 -> W (6, m*k)."""
    fr = _f(frames).reshape(-1, 12)
    m = len(fr)
    W = np.zeros((m * k, 6))
    _check(lib().oracle_wrench_basis(m, _d(fr), float(mu), int(k), _d(W)))
    return W.T.copy()


def assemble_lower_qp(W, m, targets, beta, gamma_total):
    """qpsolve.cpp:193-235 -> dict P, A, Q, L, U (numpy, row-index)."""
    W = np.asarray(W, dtype=np.float64)
    nv = W.shape[1]
    T = np.asarray(targets, dtype=np.float64).reshape(6, -1)
    B = T.shape[1]
    M = m + 1 + nv
    P, A, Q, L, U = np.zeros(nv * nv), np.zeros(M * nv), np.zeros(nv * B), np.zeros(M * B), np.zeros(M * B)
    _check(lib().oracle_assemble_lower_qp(_d(_f(W.T)), int(m), nv, _d(_f(T.T)), B, float(beta), float(gamma_total),
                                          _d(P), _d(A), _d(Q), _d(L), _d(U)))
    cm = lambda v, r, c: v.reshape(c, r).T
    return dict(P=cm(P, nv, nv), A=cm(A, M, nv), Q=cm(Q, nv, B), L=cm(L, M, B), U=cm(U, M, B))


def solve_shared(P, A, Q, L, U, cfg, warm_x=None, warm_y=None):
    """qpsolve.cpp:45-120 on a general batch (numpy, row-index; Q/L/U (rows, B)) -> dict."""
    P, A = np.asarray(P, float), np.asarray(A, float)
    Q, L, U = (np.asarray(v, float).reshape(len(v), -1) for v in (Q, L, U))
    n, M, B = P.shape[0], A.shape[0], Q.shape[1]
    X, Y, Z = np.zeros(n * B), np.zeros(M * B), np.zeros(M * B)
    it, cv = np.zeros(B, np.int32), np.zeros(B, np.int32)
    p = cfg.to_params()
    wx = None if warm_x is None else _f(np.asarray(warm_x, float).reshape(n, B).T)
    wy = None if warm_y is None else _f(np.asarray(warm_y, float).reshape(M, B).T)
    rows = np.array([Q.shape[0], L.shape[0], U.shape[0]], np.int32)
    _check(lib().oracle_solve_shared(n, M, B, _d(_f(P.T)), _d(_f(A.T)), _d(_f(Q.T)), _d(_f(L.T)), _d(_f(U.T)),
                                     _i(rows), ref(p), _d(wx), _d(wy), _d(X), _d(Y), _d(Z), _i(it), _i(cv)))
    cm = lambda v, r: v.reshape(B, r).T
    return dict(X=cm(X, n), Y=cm(Y, M), Z=cm(Z, M), iters=it, converged=cv.astype(bool))


def grasp_energy(cfg, frames, targets=None, warm_x=None, warm_y=None):
    """energy.cpp:60-92 with targets (6, B) (None = the six closure directions) -> dict."""
    fr = _f(frames).reshape(-1, 12)
    m = len(fr)
    nv = m * cfg.contact.n_edges
    M = m + 1 + nv
    T = None if targets is None else np.asarray(targets, float).reshape(6, -1)
    B = 6 if T is None else T.shape[1]
    tot = C.c_double()
    per, conv, its = np.zeros(B), np.zeros(B, np.int32), np.zeros(B, np.int32)
    F, R, Yd = np.zeros(nv * B), np.zeros(6 * B), np.zeros(M * B)
    p = cfg.to_params()
    _check(lib().oracle_grasp_energy(ref(p), m, _d(fr), B, None if T is None else _d(_f(T.T)),
                                     None if warm_x is None else _d(_f(np.asarray(warm_x).T)),
                                     None if warm_y is None else _d(_f(np.asarray(warm_y).T)),
                                     C.byref(tot), _d(per), _d(F), _d(R), _d(Yd), _i(conv), _i(its)))
    return dict(total=tot.value, per_direction=per, forces=F.reshape(B, nv).T, residuals=R.reshape(B, 6).T,
                duals=Yd.reshape(B, M).T, converged=conv.astype(bool), iters=its)


def grasp_energy_gradient(cfg, frames, report, jac_p, jac_n):
    """energy.cpp:94-145: jac_p/jac_n (m, 3, D) -> grad (D,)."""
    fr = _f(frames).reshape(-1, 12)
    m = len(fr)
    jp, jn = _f(jac_p).reshape(m, 3, -1), _f(jac_n).reshape(m, 3, -1)
    D = jp.shape[2]
    g = np.zeros(D)
    p = cfg.to_params()
    _check(lib().oracle_grasp_energy_gradient(ref(p), m, _d(fr), _d(_f(report["forces"].T)),
                                              _d(_f(report["residuals"].T)), D, _d(jp), _d(jn), _d(g)))
    return g


def stage_surrogate(points, anchors, jacobians=None):
    """fine_stage_surrogate (energy.cpp:208-229) -> (value, grad or None)."""
    pts, anc = _f(points).reshape(-1, 3), _f(anchors).reshape(-1, 3)
    v = C.c_double()
    if jacobians is None:
        _check(lib().oracle_stage_surrogate(len(pts), _d(pts), _d(anc), 0, None, C.byref(v), None))
        return v.value, None
    J = _f(jacobians).reshape(len(pts), 3, -1)
    g = np.zeros(J.shape[2])
    _check(lib().oracle_stage_surrogate(len(pts), _d(pts), _d(anc), J.shape[2], _d(J), C.byref(v), _d(g)))
    return v.value, g


def fine_grasp_surrogate(hand, x, c_w, links, anchors):
    """pipeline.cpp:54-65 / 382-386 (witnesses rigid on their links) -> (value, grad)."""
    x = _f(x)
    cw, anc = _f(c_w).reshape(-1, 3), _f(anchors).reshape(-1, 3)
    lk = np.ascontiguousarray(links, dtype=np.int32)
    v = C.c_double()
    g = np.zeros(hand.dims())
    _check(lib().oracle_fine_grasp_surrogate(ref(hand.desc), _d(x), len(cw), _d(cw), _i(lk), _d(anc), C.byref(v), _d(g)))
    return v.value, g
