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
                                              _ip, _ip, C.c_int]),
            "oracle_forward_kinematics": (C.c_int, [_vp, C.c_int, _dp, _dp]),
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
                 warm_ready=None, qp_stats=False, threads=None):
    """total_energy (pipeline.cpp:96-210) per grasp. warm_x/warm_y (updated in place) are
    the coarse QP's warm start, used for grasps with warm_ready != 0 (all when None).
    With qp_stats, also returns the coarse QP's per-column (iters, converged)."""
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
    _check(lib().oracle_total_energy(ref(hand.desc), ref(obj.desc), ref(p), stage, n, _d(x), _d(anc), _d(warm_x),
                                     _d(warm_y), _i(rdy), _d(energy), _d(grad), _i(its), _i(conv), int(nt)))
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
