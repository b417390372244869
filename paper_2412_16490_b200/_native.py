"""ctypes mirror of include/grasp_b200.h (the product C ABI).

The shared library is built in-tree by __graft_entry__.build() (nvcc for
sm_100a + g++ for the host half). Loading fails loudly when it is missing:
there is no CPU fallback for the hot path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "_lib"
LIB_PATH = Path(os.environ.get("GRASP_LIB", str(LIB_DIR / "libgrasp_b200.so")))

GRASP_OK = 0
GRASP_EINVAL = 1
GRASP_EGEOM = 2
GRASP_EHAND = 3
GRASP_EOBJECT = 4
GRASP_ECUDA = 5
GRASP_ENOMEM = 6

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class HandDesc(C.Structure):
    _fields_ = [
        ("n_links", C.c_int), ("dof", C.c_int), ("n_tips", C.c_int), ("n_proxies", C.c_int),
        ("n_pairs", C.c_int), ("n_verts", C.c_int), ("n_faces", C.c_int),
        ("link_parent_joint", _ip), ("link_tip_proxy", _ip), ("link_vert_begin", _ip),
        ("link_face_begin", _ip), ("link_proxy_begin", _ip), ("verts", _dp), ("faces", _ip),
        ("link_obb", _dp), ("link_centroid", _dp), ("link_volume", _dp), ("proxies", _dp),
        ("joint_parent_link", _ip), ("joint_child_link", _ip), ("joint_origin", _dp),
        ("joint_axis", _dp), ("joint_lower", _dp), ("joint_upper", _dp), ("tip_links", _ip),
        ("collision_pairs", _ip),
    ]


class ObjectDesc(C.Structure):
    _fields_ = [
        ("n_parts", C.c_int), ("n_verts", C.c_int), ("n_faces", C.c_int),
        ("part_vert_begin", _ip), ("part_face_begin", _ip), ("verts", _dp), ("faces", _ip),
        ("part_obb", _dp), ("part_centroid", _dp), ("part_volume", _dp),
        ("scale", C.c_double), ("bbox_diagonal", C.c_double), ("mass_center", C.c_double * 3),
        ("source", C.c_char_p),
    ]


class StageParams(C.Structure):
    _fields_ = [("iters", C.c_int), ("step_rotation", C.c_double), ("step_translation", C.c_double),
                ("step_joints", C.c_double), ("step_floor", C.c_double)]


class EvalParamsStruct(C.Structure):
    _fields_ = [("mass", C.c_double), ("gravity", C.c_double), ("residual_rel_tol", C.c_double),
                ("force_budget_factor", C.c_double), ("contact_tol", C.c_double), ("penetration_tol", C.c_double),
                ("qp_eps", C.c_double)]


class RunParams(C.Structure):
    _fields_ = [
        ("qp_rho", C.c_double), ("qp_sigma", C.c_double), ("qp_alpha", C.c_double),
        ("qp_max_iters", C.c_int), ("qp_eps_primal", C.c_double), ("qp_eps_dual", C.c_double),
        ("qp_check_interval", C.c_int), ("mu", C.c_double), ("n_edges", C.c_int),
        ("beta", C.c_double), ("gamma_per_contact", C.c_double),
        ("w_grasp", C.c_double), ("w_distance", C.c_double), ("w_joint_limit", C.c_double),
        ("w_self_penetration", C.c_double), ("w_object_penetration", C.c_double),
        ("coarse", StageParams), ("fine", StageParams), ("final_stage", StageParams),
        ("contact_offset", C.c_double), ("fd_step", C.c_double), ("skip_fine_stages", C.c_int),
        ("standoff", C.c_double), ("joint_span_fraction", C.c_double),
        ("seed", C.c_uint64), ("batch", C.c_int), ("workers", C.c_int),
    ]


class Out(C.Structure):
    _fields_ = [("x_p", _dp), ("x", _dp), ("x_s", _dp), ("energy_total", _dp), ("per_direction", _dp),
                ("contact_forces", _dp), ("contacts", _dp), ("stage_energy", _dp), ("failed", _ip),
                ("qp_converged", _ip)]


class Trace(C.Structure):
    _fields_ = [("n_snap", C.c_int), ("stage", _ip), ("iter", _ip), ("x_in", _dp), ("world_in", _dp),
                ("warm_x_in", _dp), ("warm_y_in", _dp), ("warm_ready_in", _ip), ("anchors", _dp),
                ("energy", _dp), ("grad", _dp), ("x_out", _dp), ("warm_x_out", _dp), ("warm_y_out", _dp),
                ("qp_iters", _ip), ("qp_converged", _ip), ("failed", _ip)]


# Every symbol include/grasp_b200.h declares, with its ctypes signature.
SIGNATURES = {
    "grasp_last_error": (C.c_char_p, []),
    "grasp_version": (C.c_char_p, []),
    "grasp_hand_builtin": (C.c_int, [C.POINTER(C.c_void_p)]),
    "grasp_hand_parse": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "grasp_hand_free": (None, [C.c_void_p]),
    "grasp_hand_builtin_json": (C.c_int64, [C.c_char_p, C.c_int64]),
    "grasp_object_primitive": (C.c_int, [C.c_char_p, C.c_double, C.POINTER(C.c_void_p)]),
    "grasp_object_parse": (C.c_int, [C.c_char_p, C.c_double, C.c_char_p, C.POINTER(C.c_void_p)]),
    "grasp_object_from_points": (C.c_int, [C.c_int, _ip, _dp, C.POINTER(C.c_void_p)]),
    "grasp_build_convex_parts": (C.c_int, [C.c_int, _dp, _ip, C.c_int, C.c_double, _dp, _ip, _ip, _ip, _dp, _dp, _dp,
                                           _ip]),
    "grasp_object_free": (None, [C.c_void_p]),
    "grasp_object_bounding_radius": (C.c_double, [C.c_void_p]),
    "grasp_hand_describe": (C.c_int, [C.c_void_p, C.POINTER(HandDesc)]),
    "grasp_object_describe": (C.c_int, [C.c_void_p, C.POINTER(ObjectDesc)]),
    "grasp_run_params_default": (None, [C.POINTER(RunParams)]),
    "grasp_run_params_parse": (C.c_int, [C.c_char_p, C.POINTER(RunParams)]),
    "grasp_run_params_validate": (C.c_int, [C.POINTER(RunParams)]),
    "grasp_init_poses": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, C.c_double, C.c_double, _dp]),
    "grasp_squeeze_pose": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "grasp_forward_kinematics": (C.c_int, [C.c_void_p, C.c_int, _dp, _dp]),
    "grasp_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "grasp_ctx_create_devices": (C.c_int, [_ip, C.c_int, C.POINTER(C.c_void_p)]),
    "grasp_ctx_destroy": (None, [C.c_void_p]),
    "grasp_ctx_set_hand": (C.c_int, [C.c_void_p, C.POINTER(HandDesc)]),
    "grasp_ctx_set_object": (C.c_int, [C.c_void_p, C.POINTER(ObjectDesc)]),
    "grasp_synthesize": (C.c_int, [C.c_void_p, C.POINTER(RunParams), C.c_int, _dp, C.POINTER(Out)]),
    "grasp_synthesize_device": (C.c_int, [C.c_void_p, C.POINTER(RunParams), C.c_int, _dp, C.POINTER(Out)]),
    "grasp_ctx_set_objects": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.POINTER(ObjectDesc))]),
    "grasp_synthesize_objects": (C.c_int, [C.c_void_p, C.POINTER(RunParams), C.c_int, _dp, _ip, C.POINTER(Out)]),
    "grasp_eval_params_default": (None, [C.POINTER(EvalParamsStruct)]),
    "grasp_eval": (C.c_int, [C.c_void_p, C.POINTER(RunParams), C.POINTER(EvalParamsStruct), C.c_int, _dp, _dp, _dp,
                             C.POINTER(C.c_int)]),
    "grasp_qp_batch": (C.c_int, [C.c_void_p, C.POINTER(RunParams), C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp,
                                 _dp, _ip, _ip, _dp, C.c_int]),
    "grasp_point_to_mesh": (C.c_int, [C.c_void_p, C.c_int, _dp, _dp]),
    "grasp_signed_distance": (C.c_int, [C.c_void_p, C.c_int, _ip, _ip, _dp, _dp]),
    "grasp_total_energy": (C.c_int, [C.c_void_p, C.POINTER(RunParams), C.c_int, C.c_int, _dp, _dp, _dp, _dp,
                                     _dp, _dp]),
    "grasp_fine_contact_query": (C.c_int, [C.c_void_p, C.c_int, _dp, _dp]),
    "grasp_device_forward_kinematics": (C.c_int, [C.c_void_p, C.c_int, _dp, _dp]),
    "grasp_fine_contact_query_world": (C.c_int, [C.c_void_p, C.c_int, _dp, _dp]),
    "grasp_ctx_stream": (C.c_void_p, [C.c_void_p]),
    "grasp_ctx_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "grasp_ctx_profile": (C.c_int, [C.c_void_p, _dp, C.POINTER(C.c_longlong), C.POINTER(C.c_ulonglong)]),
    "grasp_ctx_launch_count": (C.c_longlong, [C.c_void_p]),
    "grasp_ctx_set_option": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int]),
    "grasp_ctx_set_trace": (C.c_int, [C.c_void_p, C.POINTER(Trace)]),
    "grasp_measure_fp64_peak": (C.c_int, [C.c_int, _dp]),
}

_lib = None


def lib() -> C.CDLL:
    """Loads the in-tree native library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc sm_100a). "
                "There is no CPU fallback for the grasp-synthesis engine.")
        handle = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int) -> None:
    if status != GRASP_OK:
        msg = lib().grasp_last_error().decode(errors="replace")
        from .errors import raise_for
        raise_for(status, msg)
