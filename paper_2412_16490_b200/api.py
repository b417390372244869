"""Python mirror of the reference C++ API (proj/include/grasp/*.hpp).

Names and argument meaning follow the reference: HandModel (hand.hpp:20-47),
ObjectModel (object.hpp:19-25), RunConfig (config.hpp:77-88),
init_poses / squeeze_pose / synthesize (pipeline.hpp:55-71), GraspRecord
(records.hpp:29-44). All compute goes through the native library
(include/grasp_b200.h); synthesize runs on a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import json
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp) if a is not None else None


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_ip) if a is not None else None


# --------------------------------------------------------------------- config
@dataclass
class QpParams:
    rho: float = 0.1
    sigma: float = 1e-6
    alpha: float = 1.6
    max_iters: int = 500
    eps_primal: float = 1e-5
    eps_dual: float = 1e-5
    check_interval: int = 10


@dataclass
class ContactParams:
    mu: float = 0.6
    n_edges: int = 8


@dataclass
class EnergyParams:
    beta: float = 10.0
    gamma_per_contact: float = 0.1


@dataclass
class ObjectiveWeights:
    grasp: float = 1.0
    distance: float = 100.0
    joint_limit: float = 10.0
    self_penetration: float = 10.0
    object_penetration: float = 10.0


@dataclass
class StageSchedule:
    iters: int = 300
    step_rotation: float = 0.010
    step_translation: float = 0.0025
    step_joints: float = 0.010
    step_floor: float = 0.1


@dataclass
class PipelineParams:
    coarse: StageSchedule = field(default_factory=lambda: StageSchedule(300, 0.010, 0.0025, 0.010, 0.1))
    fine: StageSchedule = field(default_factory=lambda: StageSchedule(100, 0.004, 0.0010, 0.004, 0.1))
    final_stage: StageSchedule = field(default_factory=lambda: StageSchedule(100, 0.004, 0.0010, 0.004, 0.1))
    contact_offset: float = 0.01
    fd_step: float = 1e-6
    skip_fine_stages: bool = False


@dataclass
class InitParams:
    standoff: float = 0.10
    joint_span_fraction: float = 0.25


@dataclass
class EvalParams:
    mass: float = 0.03
    gravity: float = 9.8
    residual_rel_tol: float = 1e-3
    force_budget_factor: float = 20.0
    contact_tol: float = 0.002
    penetration_tol: float = 0.003
    qp_eps: float = 1e-8


@dataclass
class RunConfig:
    qp: QpParams = field(default_factory=QpParams)
    contact: ContactParams = field(default_factory=ContactParams)
    energy: EnergyParams = field(default_factory=EnergyParams)
    weights: ObjectiveWeights = field(default_factory=ObjectiveWeights)
    pipeline: PipelineParams = field(default_factory=PipelineParams)
    init: InitParams = field(default_factory=InitParams)
    eval: EvalParams = field(default_factory=EvalParams)
    seed: int = 0
    batch: int = 64
    workers: int = 1

    def to_params(self) -> N.RunParams:
        p = N.RunParams()
        p.qp_rho, p.qp_sigma, p.qp_alpha = self.qp.rho, self.qp.sigma, self.qp.alpha
        p.qp_max_iters, p.qp_eps_primal, p.qp_eps_dual = self.qp.max_iters, self.qp.eps_primal, self.qp.eps_dual
        p.qp_check_interval = self.qp.check_interval
        p.mu, p.n_edges = self.contact.mu, self.contact.n_edges
        p.beta, p.gamma_per_contact = self.energy.beta, self.energy.gamma_per_contact
        w = self.weights
        p.w_grasp, p.w_distance, p.w_joint_limit = w.grasp, w.distance, w.joint_limit
        p.w_self_penetration, p.w_object_penetration = w.self_penetration, w.object_penetration
        for name in ("coarse", "fine", "final_stage"):
            s = getattr(self.pipeline, name)
            setattr(p, name, N.StageParams(s.iters, s.step_rotation, s.step_translation, s.step_joints,
                                           s.step_floor))
        p.contact_offset, p.fd_step = self.pipeline.contact_offset, self.pipeline.fd_step
        p.skip_fine_stages = int(bool(self.pipeline.skip_fine_stages))
        p.standoff, p.joint_span_fraction = self.init.standoff, self.init.joint_span_fraction
        p.seed, p.batch, p.workers = int(self.seed), int(self.batch), int(self.workers)
        return p

    @staticmethod
    def from_params(p: N.RunParams, eval_params: Optional[EvalParams] = None) -> "RunConfig":
        st = lambda s: StageSchedule(s.iters, s.step_rotation, s.step_translation, s.step_joints, s.step_floor)
        return RunConfig(
            qp=QpParams(p.qp_rho, p.qp_sigma, p.qp_alpha, p.qp_max_iters, p.qp_eps_primal, p.qp_eps_dual,
                        p.qp_check_interval),
            contact=ContactParams(p.mu, p.n_edges),
            energy=EnergyParams(p.beta, p.gamma_per_contact),
            weights=ObjectiveWeights(p.w_grasp, p.w_distance, p.w_joint_limit, p.w_self_penetration,
                                     p.w_object_penetration),
            pipeline=PipelineParams(st(p.coarse), st(p.fine), st(p.final_stage), p.contact_offset, p.fd_step,
                                    bool(p.skip_fine_stages)),
            init=InitParams(p.standoff, p.joint_span_fraction),
            eval=eval_params or EvalParams(), seed=p.seed, batch=p.batch, workers=p.workers)


def parse_run_config(json_text: str) -> RunConfig:
    """config.cpp:139-156: strict parse + validate (eval block checked natively too)."""
    p = N.RunParams()
    N.check(N.lib().grasp_run_params_parse(json_text.encode(), C.byref(p)))
    ev = EvalParams()
    doc = json.loads(json_text)
    for k, v in doc.get("eval", {}).items():
        setattr(ev, k, v)
    return RunConfig.from_params(p, ev)


def validate(cfg: RunConfig) -> None:
    """config.cpp:196-229 (eval ranges checked here, the rest natively)."""
    N.check(N.lib().grasp_run_params_validate(C.byref(cfg.to_params())))
    e = cfg.eval
    for ok, what in ((e.mass > 0, "eval.mass must be positive"), (e.gravity > 0, "eval.gravity must be positive"),
                     (e.residual_rel_tol > 0, "eval.residual_rel_tol must be positive"),
                     (e.force_budget_factor > 0, "eval.force_budget_factor must be positive"),
                     (e.contact_tol >= 0, "eval.contact_tol must be nonnegative"),
                     (e.penetration_tol >= 0, "eval.penetration_tol must be nonnegative"),
                     (e.qp_eps > 0, "eval.qp_eps must be positive")):
        if not ok:
            from .errors import InvalidArgument
            raise InvalidArgument("config: " + what)


# --------------------------------------------------------------------- models
def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


class HandModel:
    """Owns a native grasp_hand; exposes the packed arrays (hand.hpp:20-47)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        self.desc = N.HandDesc()
        N.check(N.lib().grasp_hand_describe(self._h, C.byref(self.desc)))
        d = self.desc
        self.n_links, self.n_tips, self.n_pairs = d.n_links, d.n_tips, d.n_pairs
        self.fingertip_links = _arr(d.tip_links, d.n_tips, np.int32)
        self.lower = _arr(d.joint_lower, d.dof, np.float64)
        self.upper = _arr(d.joint_upper, d.dof, np.float64)
        self.link_vert_begin = _arr(d.link_vert_begin, d.n_links + 1, np.int32)
        self.link_face_begin = _arr(d.link_face_begin, d.n_links + 1, np.int32)
        self.link_proxy_begin = _arr(d.link_proxy_begin, d.n_links + 1, np.int32)
        self.proxies = _arr(d.proxies, 4 * d.n_proxies, np.float64).reshape(-1, 4)
        self.collision_pairs = _arr(d.collision_pairs, 2 * d.n_pairs, np.int32).reshape(-1, 2)
        self.link_parent_joint = _arr(d.link_parent_joint, d.n_links, np.int32)
        self.link_tip_proxy = _arr(d.link_tip_proxy, d.n_links, np.int32)
        per_link = np.diff(self.link_proxy_begin)
        # sphere pairs the self-penetration term visits (hand.cpp:225-231)
        self.n_sphere_pairs = int(sum(per_link[a] * per_link[b] for a, b in self.collision_pairs))

    @staticmethod
    def builtin() -> "HandModel":
        h = C.c_void_p()
        N.check(N.lib().grasp_hand_builtin(C.byref(h)))
        return HandModel(h)

    @staticmethod
    def from_json(text: str) -> "HandModel":
        h = C.c_void_p()
        N.check(N.lib().grasp_hand_parse(text.encode(), C.byref(h)))
        return HandModel(h)

    @staticmethod
    def from_file(path) -> "HandModel":
        with open(path) as f:
            return HandModel.from_json(f.read())

    def dof(self) -> int:
        return self.desc.dof

    def dims(self) -> int:
        return 12 + self.desc.dof

    def lower_limits(self):
        return self.lower.copy()

    def upper_limits(self):
        return self.upper.copy()

    def __del__(self):
        try:
            if self._h:
                N.lib().grasp_hand_free(self._h)
        except Exception:
            pass


def builtin_hand_json() -> str:
    n = N.lib().grasp_hand_builtin_json(None, 0)
    buf = C.create_string_buffer(int(n))
    N.lib().grasp_hand_builtin_json(buf, n)
    return buf.value.decode()


class ObjectModel:
    """Owns a native grasp_object (object.hpp:19-25)."""

    def __init__(self, handle):
        self._o = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        self.desc = N.ObjectDesc()
        N.check(N.lib().grasp_object_describe(self._o, C.byref(self.desc)))
        d = self.desc
        self.scale = d.scale
        self.bbox_diagonal = d.bbox_diagonal
        self.mass_center = np.array(list(d.mass_center))
        self.source = d.source.decode() if d.source else ""
        self.part_vert_begin = _arr(d.part_vert_begin, d.n_parts + 1, np.int32)
        self.part_face_begin = _arr(d.part_face_begin, d.n_parts + 1, np.int32)
        self.verts = _arr(d.verts, 3 * d.n_verts, np.float64).reshape(-1, 3)
        self.faces = _arr(d.faces, 3 * d.n_faces, np.int32).reshape(-1, 3)
        self.part_obb = _arr(d.part_obb, 15 * d.n_parts, np.float64).reshape(-1, 15)
        self.part_volume = _arr(d.part_volume, d.n_parts, np.float64)
        self.part_centroid = _arr(d.part_centroid, 3 * d.n_parts, np.float64).reshape(-1, 3)

    @property
    def n_parts(self) -> int:
        return self.desc.n_parts

    def part_vertices(self, i):
        return self.verts[self.part_vert_begin[i]:self.part_vert_begin[i + 1]]

    def part_faces(self, i):
        return self.faces[self.part_face_begin[i]:self.part_face_begin[i + 1]]

    @staticmethod
    def primitive(name: str, scale: float) -> "ObjectModel":
        o = C.c_void_p()
        N.check(N.lib().grasp_object_primitive(name.encode(), float(scale), C.byref(o)))
        return ObjectModel(o)

    @staticmethod
    def from_obj_text(text: str, scale: float, source: str = "mesh") -> "ObjectModel":
        o = C.c_void_p()
        N.check(N.lib().grasp_object_parse(text.encode(), float(scale), source.encode(), C.byref(o)))
        return ObjectModel(o)

    @staticmethod
    def load(path, scale: float) -> "ObjectModel":
        with open(path) as f:
            return ObjectModel.from_obj_text(f.read(), scale, str(path))

    @staticmethod
    def from_points(parts) -> "ObjectModel":
        """Raw convex parts (make_convex_part), no normalization."""
        counts = np.array([len(p) for p in parts], dtype=np.int32)
        pts = np.ascontiguousarray(np.concatenate([np.asarray(p, dtype=np.float64) for p in parts]))
        o = C.c_void_p()
        N.check(N.lib().grasp_object_from_points(len(parts), iptr(counts), dptr(pts), C.byref(o)))
        return ObjectModel(o)

    def bounding_radius(self) -> float:
        return N.lib().grasp_object_bounding_radius(self._o)

    def bounding_box(self):
        return self.verts.min(axis=0), self.verts.max(axis=0)

    def __del__(self):
        try:
            if self._o:
                N.lib().grasp_object_free(self._o)
        except Exception:
            pass


make_primitive = ObjectModel.primitive
parse_object_text = ObjectModel.from_obj_text
load_object = ObjectModel.load
PRIMITIVE_NAMES = ("sphere", "box", "cylinder", "capsule", "flat_box")


def build_convex_parts(parts, merge_tol: float = 1e-9, device: int = 0) -> List[dict]:
    """make_convex_part (geometry.cpp:414-466) of many point clouds on the device, one thread per
    part (grasp_build_convex_parts), bit-identical to the host builder (ObjectModel.from_points).
    Returns per part: vertices (V, 3), faces (F, 3) local indices, volume, centroid (3,),
    obb (15,) = center, half extents, rotation column-major, status (0 ok, 1 degenerate,
    2 workspace overflow)."""
    arrs = [np.asarray(p, dtype=np.float64).reshape(-1, 3) for p in parts]
    begin = np.zeros(len(arrs) + 1, dtype=np.int32)
    begin[1:] = np.cumsum([len(a) for a in arrs])
    n_pts, n = int(begin[-1]), len(arrs)
    pts = np.ascontiguousarray(np.concatenate(arrs) if n_pts else np.zeros((0, 3)))
    verts = np.zeros((max(n_pts, 1), 3))
    faces = np.zeros((max(2 * n_pts, 1), 3), dtype=np.int32)
    nv, nf, status = (np.zeros(max(n, 1), dtype=np.int32) for _ in range(3))
    vol, cen, obb = np.zeros(max(n, 1)), np.zeros((max(n, 1), 3)), np.zeros((max(n, 1), 15))
    N.check(N.lib().grasp_build_convex_parts(int(device), dptr(pts), iptr(begin), n, float(merge_tol), dptr(verts),
                                             iptr(nv), iptr(faces), iptr(nf), dptr(vol), dptr(cen), dptr(obb),
                                             iptr(status)))
    out = []
    for p in range(n):
        b = int(begin[p])
        out.append(dict(vertices=verts[b:b + nv[p]].copy(), faces=faces[2 * b:2 * b + nf[p]].copy(),
                        volume=float(vol[p]), centroid=cen[p].copy(), obb=obb[p].copy(), status=int(status[p])))
    return out


def init_poses(model: HandModel, obj: ObjectModel, n: int, seed: int, params: InitParams = None) -> np.ndarray:
    """pipeline.cpp:388-424 -> (n, D) array."""
    params = params or InitParams()
    out = np.zeros((n, model.dims()), dtype=np.float64)
    N.check(N.lib().grasp_init_poses(model._h, obj._o, int(n), int(seed), params.standoff,
                                     params.joint_span_fraction, dptr(out)))
    return out


def squeeze_pose(model: HandModel, x, x_p) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    x_p = np.ascontiguousarray(x_p, dtype=np.float64)
    out = np.zeros(model.dims())
    N.check(N.lib().grasp_squeeze_pose(model._h, dptr(x), dptr(x_p), dptr(out)))
    return out


def forward_kinematics(model: HandModel, x) -> np.ndarray:
    """hand::forward_kinematics (hand.hpp:100) of (n, D) states -> (n, n_links, 12) world link
    transforms: R (9, column-major), t (3). Host-side."""
    x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
    out = np.zeros((x.shape[0], model.n_links, 12))
    N.check(N.lib().grasp_forward_kinematics(model._h, int(x.shape[0]), dptr(x), dptr(out)))
    return out


# -------------------------------------------------------------------- records
@dataclass
class ContactFrame:
    p: np.ndarray
    n: np.ndarray
    d: np.ndarray
    e: np.ndarray


@dataclass
class StageTrace:
    stage: str
    iterations: int
    energy_start: float
    energy_end: float


@dataclass
class GraspRecord:
    x_p: np.ndarray
    x: np.ndarray
    x_s: np.ndarray
    energy_total: float
    per_direction: np.ndarray
    contact_forces: np.ndarray
    contacts: List[ContactFrame]
    object_id: str
    object_scale: float
    seed: int
    index: int
    failed: bool
    note: str
    stages: List[StageTrace]


_NOTES = {0: "", 1: "non-finite energy", 2: "diverged"}


class SynthesisOutput:
    """SoA result buffers laid out like grasp_out (host numpy arrays)."""

    def __init__(self, batch: int, dims: int, m: int, n_edges: int):
        n = m * n_edges
        self.x_p = np.zeros((batch, dims))
        self.x = np.zeros((batch, dims))
        self.x_s = np.zeros((batch, dims))
        self.energy_total = np.zeros(batch)
        self.per_direction = np.zeros((batch, 6))
        self.contact_forces = np.zeros((batch, 6, n))  # per grasp column-major (n x 6) == row-major (6, n)
        self.contacts = np.zeros((batch, m, 12))
        self.stage_energy = np.zeros((batch, 3, 2))
        self.failed = np.zeros(batch, dtype=np.int32)
        self.qp_converged = np.zeros((batch, 6), dtype=np.int32)

    def as_struct(self) -> N.Out:
        return N.Out(dptr(self.x_p), dptr(self.x), dptr(self.x_s), dptr(self.energy_total),
                     dptr(self.per_direction), dptr(self.contact_forces), dptr(self.contacts),
                     dptr(self.stage_energy), iptr(self.failed), iptr(self.qp_converged))

    def subset(self, lo: int, hi: int) -> "SynthesisOutput":
        """Rows [lo, hi) as their own output (views)."""
        out = SynthesisOutput.__new__(SynthesisOutput)
        for k in ("x_p", "x", "x_s", "energy_total", "per_direction", "contact_forces", "contacts", "stage_energy",
                  "failed", "qp_converged"):
            setattr(out, k, getattr(self, k)[lo:hi])
        return out

    def records(self, cfg: RunConfig, obj: ObjectModel, index_offset: int = 0) -> List[GraspRecord]:
        names = ("coarse", "fine", "final")
        iters = (cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters)
        n_stages = 1 if cfg.pipeline.skip_fine_stages else 3
        out = []
        for g in range(self.x.shape[0]):
            failed = int(self.failed[g])
            contacts = [] if failed else [ContactFrame(c[0:3].copy(), c[3:6].copy(), c[6:9].copy(), c[9:12].copy())
                                          for c in self.contacts[g]]
            out.append(GraspRecord(
                x_p=self.x_p[g].copy(), x=self.x[g].copy(), x_s=self.x_s[g].copy(),
                energy_total=float(self.energy_total[g]),
                per_direction=np.zeros(0) if failed else self.per_direction[g].copy(),
                contact_forces=np.zeros((0, 0)) if failed else self.contact_forces[g].T.copy(),
                contacts=contacts, object_id=obj.source, object_scale=obj.scale, seed=int(cfg.seed),
                index=index_offset + g, failed=bool(failed), note=_NOTES.get(failed, "failed"),
                stages=[StageTrace(names[s], iters[s], float(self.stage_energy[g, s, 0]),
                                   float(self.stage_energy[g, s, 1])) for s in range(n_stages)]))
        return out


# --------------------------------------------------------------------- engine
class Engine:
    """One CUDA device, one stream (grasp_ctx). Hand/object uploaded once."""

    def __init__(self, device: int = 0, devices: Optional[List[int]] = None):
        """devices: shard synthesize over these CUDA devices (grasp_ctx_create_devices)."""
        self._ctx = C.c_void_p()
        if devices:
            ids = np.ascontiguousarray(devices, dtype=np.int32)
            N.check(N.lib().grasp_ctx_create_devices(iptr(ids), len(ids), C.byref(self._ctx)))
        else:
            N.check(N.lib().grasp_ctx_create(int(device), C.byref(self._ctx)))
        self.hand: Optional[HandModel] = None
        self.obj: Optional[ObjectModel] = None

    def set_hand(self, hand: HandModel):
        N.check(N.lib().grasp_ctx_set_hand(self._ctx, C.byref(hand.desc)))
        self.hand = hand

    def set_object(self, obj: ObjectModel):
        N.check(N.lib().grasp_ctx_set_object(self._ctx, C.byref(obj.desc)))
        self.obj = obj

    def synthesize(self, cfg: RunConfig, x0: np.ndarray) -> SynthesisOutput:
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        batch = x0.shape[0]
        out = SynthesisOutput(batch, self.hand.dims(), self.hand.n_tips, cfg.contact.n_edges)
        s = out.as_struct()
        N.check(N.lib().grasp_synthesize(self._ctx, C.byref(cfg.to_params()), batch, dptr(x0), C.byref(s)))
        return out

    def set_objects(self, objects: List[ObjectModel]):
        """Several objects in this context (grasp_ctx_set_objects)."""
        arr = (C.POINTER(N.ObjectDesc) * len(objects))(*[C.pointer(o.desc) for o in objects])
        N.check(N.lib().grasp_ctx_set_objects(self._ctx, len(objects), arr))
        self.objects = list(objects)
        self.obj = objects[0]

    def synthesize_objects(self, cfg: RunConfig, x0: np.ndarray, object_index) -> SynthesisOutput:
        """One batch over grasps of the objects of set_objects (grasp_synthesize_objects)."""
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        idx = np.ascontiguousarray(object_index, dtype=np.int32)
        batch = x0.shape[0]
        out = SynthesisOutput(batch, self.hand.dims(), self.hand.n_tips, cfg.contact.n_edges)
        s = out.as_struct()
        N.check(N.lib().grasp_synthesize_objects(self._ctx, C.byref(cfg.to_params()), batch, dptr(x0), iptr(idx),
                                                 C.byref(s)))
        return out

    def synthesize_traced(self, cfg: RunConfig, x0: np.ndarray, snaps) -> tuple:
        """synthesize with a per-iteration trace (grasp_ctx_set_trace): snaps is a list of
        (stage, iter); returns (SynthesisOutput, dict of snapshot-major arrays)."""
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        B, D, m, L = x0.shape[0], self.hand.dims(), self.hand.n_tips, self.hand.n_links
        nv = m * cfg.contact.n_edges
        M = m + 1 + nv
        S = len(snaps)
        stage = np.array([s for s, _ in snaps], dtype=np.int32)
        it = np.array([i for _, i in snaps], dtype=np.int32)
        t = dict(x_in=np.zeros((S, B, D)), world_in=np.zeros((S, B, L, 12)), warm_x_in=np.zeros((S, B, 6, nv)),
                 warm_y_in=np.zeros((S, B, 6, M)), warm_ready_in=np.zeros((S, B), np.int32),
                 anchors=np.zeros((S, B, m, 3)), energy=np.zeros((S, B)), grad=np.zeros((S, B, D)),
                 x_out=np.zeros((S, B, D)), warm_x_out=np.zeros((S, B, 6, nv)), warm_y_out=np.zeros((S, B, 6, M)),
                 qp_iters=np.zeros((S, B, 6), np.int32), qp_converged=np.zeros((S, B, 6), np.int32),
                 failed=np.zeros((S, B), np.int32))
        ptr = {k: (iptr(v) if v.dtype == np.int32 else dptr(v)) for k, v in t.items()}
        spec = N.Trace(S, iptr(stage), iptr(it), ptr["x_in"], ptr["world_in"], ptr["warm_x_in"], ptr["warm_y_in"],
                       ptr["warm_ready_in"], ptr["anchors"], ptr["energy"], ptr["grad"], ptr["x_out"],
                       ptr["warm_x_out"], ptr["warm_y_out"], ptr["qp_iters"], ptr["qp_converged"], ptr["failed"])
        N.check(N.lib().grasp_ctx_set_trace(self._ctx, C.byref(spec)))
        try:
            out = self.synthesize(cfg, x0)
        finally:
            N.check(N.lib().grasp_ctx_set_trace(self._ctx, None))
        # device link transforms store R row-major; report column-major like forward_kinematics
        w = t["world_in"]
        w[..., :9] = w[..., :9].reshape(w.shape[:-1] + (3, 3)).swapaxes(-1, -2).reshape(w.shape[:-1] + (9,))
        t["stage"], t["iter"] = stage, it
        return out, t

    def synthesize_device(self, cfg: RunConfig, x0_ptr: int, batch: int, out_ptrs: dict) -> None:
        """grasp_synthesize_device: x0 and outputs are device pointers (ints)."""
        vp = lambda k: C.cast(C.c_void_p(out_ptrs[k]), _dp) if out_ptrs.get(k) else None
        ip = lambda k: C.cast(C.c_void_p(out_ptrs[k]), _ip) if out_ptrs.get(k) else None
        s = N.Out(vp("x_p"), vp("x"), vp("x_s"), vp("energy_total"), vp("per_direction"), vp("contact_forces"),
                  vp("contacts"), vp("stage_energy"), ip("failed"), ip("qp_converged"))
        N.check(N.lib().grasp_synthesize_device(self._ctx, C.byref(cfg.to_params()), int(batch),
                                                C.cast(C.c_void_p(x0_ptr), _dp), C.byref(s)))

    def stream_handle(self) -> int:
        return N.lib().grasp_ctx_stream(self._ctx) or 0

    def set_option(self, name: str, value: int) -> None:
        """grasp_ctx_set_option: "query_buckets", "query_lanes", "tip_query_lanes", "pair_cull", "pair_sat",
        "pair_early" (EPA-iteration threshold for the early GJK+EPA pass; >= 255 turns it off),
        "graphs" (1: synthesis as a captured CUDA graph; 0, the default: eager launches)."""
        N.check(N.lib().grasp_ctx_set_option(self._ctx, name.encode(), int(value)))

    def set_profiling(self, on: bool) -> None:
        N.check(N.lib().grasp_ctx_set_profiling(self._ctx, int(bool(on))))

    KERNEL_CLASSES = ("point_query", "qp", "step_coarse", "pairs", "step_mesh", "fk", "finalize", "pairs_big")
    OP_NAMES = ("plane_tests", "triangle_tests", "qp_column_sweeps", "qp_solves", "gjk_iters", "support_verts",
                "epa_iters", "point_queries", "pairs_needed", "epa_overflow",
                "gjk_pairs_le4", "gjk_pairs_le8", "gjk_pairs_le16", "gjk_pairs_le32", "gjk_pairs_le64",
                "gjk_pairs_gt64", "gjk_cycle_jumps", "gjk_iters_skipped", "epa_max_iters", "epa_long_jobs")

    def evaluate(self, config: RunConfig, x, x_s) -> dict:
        """quasi_static_check (eval.cpp:91-158) for each grasp on the device: pd_mm, spd_mm, cdc_mm,
        residuals (6), contact_count, success, note_flags (1 no contacts, 2 resistance qp unconverged,
        4 gravity residual above tolerance, 8 fewer than two contacts, 16 penetration above tolerance)."""
        x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
        x_s = np.ascontiguousarray(np.atleast_2d(x_s), dtype=np.float64)
        n = len(x)
        e = N.EvalParamsStruct(config.eval.mass, config.eval.gravity, config.eval.residual_rel_tol,
                               config.eval.force_budget_factor, config.eval.contact_tol,
                               config.eval.penetration_tol, config.eval.qp_eps)
        real = np.zeros((n, 9))
        ints = np.zeros((n, 3), dtype=np.int32)
        N.check(N.lib().grasp_eval(self._ctx, C.byref(config.to_params()), C.byref(e), n, dptr(x), dptr(x_s),
                                   dptr(real), iptr(ints)))
        return dict(pd_mm=real[:, 0], spd_mm=real[:, 1], cdc_mm=real[:, 2], residuals=real[:, 3:9],
                    contact_count=ints[:, 0], success=ints[:, 1].astype(bool), note_flags=ints[:, 2])

    def profile(self) -> dict:
        ms = (C.c_double * 8)()
        launches = (C.c_longlong * 8)()
        ops = (C.c_ulonglong * 20)()
        N.check(N.lib().grasp_ctx_profile(self._ctx, ms, launches, ops))
        return {"ms": dict(zip(self.KERNEL_CLASSES, list(ms))),
                "launches": dict(zip(self.KERNEL_CLASSES, list(launches))),
                "ops": dict(zip(self.OP_NAMES, list(ops)))}

    def launch_count(self) -> int:
        return int(N.lib().grasp_ctx_launch_count(self._ctx))

    def close(self):
        if self._ctx:
            N.lib().grasp_ctx_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def synthesize(model: HandModel, obj: ObjectModel, cfg: RunConfig, device: int = 0,
               engine: Optional[Engine] = None) -> List[GraspRecord]:
    """pipeline.cpp:436-457 on a B200: validate, init_poses (host, one RNG
    stream), the three-stage loop on the GPU, records in input order."""
    validate(cfg)
    x0 = init_poses(model, obj, cfg.batch, cfg.seed, cfg.init)
    eng = engine or Engine(device)
    if eng.hand is not model:
        eng.set_hand(model)
    if eng.obj is not obj:
        eng.set_object(obj)
    return eng.synthesize(cfg, x0).records(cfg, obj)


def synthesize_objects(model: HandModel, objects: List[ObjectModel], configs, device: int = 0,
                       streams: int = 8, single_launch: bool = True) -> List[List[GraspRecord]]:
    """Many objects on one GPU (BASELINE config 3). `configs` is one RunConfig
    or one per object (each object's start states come from its own init_poses stream,
    pipeline.cpp:388-424). When the configs differ only in seed and batch (config 3), all
    objects run as ONE batch in one context (grasp_synthesize_objects: object id per grasp,
    parts packed on the device, one set of launches); otherwise one synthesize per object is
    issued from `streams` host threads on their own contexts and streams. Either way each
    object's records equal a plain per-object synthesize."""
    import threading
    from .errors import InvalidArgument
    if isinstance(configs, RunConfig):
        configs = [configs] * len(objects)
    if len(configs) != len(objects):
        raise InvalidArgument("one RunConfig per object")
    for c in configs:
        validate(c)
    shared = all(dataclasses.replace(c, seed=0, batch=0) == dataclasses.replace(configs[0], seed=0, batch=0)
                 for c in configs)
    if single_launch and shared:
        eng = Engine(device)
        eng.set_hand(model)
        eng.set_objects(list(objects))
        x0 = np.concatenate([init_poses(model, o, c.batch, c.seed, c.init) for o, c in zip(objects, configs)])
        idx = np.concatenate([np.full(c.batch, k, np.int32) for k, c in enumerate(configs)])
        res = eng.synthesize_objects(configs[0], x0, idx)
        recs, lo = [], 0
        for o, c in zip(objects, configs):
            recs.append(res.subset(lo, lo + c.batch).records(c, o))
            lo += c.batch
        return recs
    S = max(1, min(int(streams), len(objects)))
    engines = [Engine(device) for _ in range(S)]
    for e in engines:
        e.set_hand(model)
    out: List[Optional[List[GraspRecord]]] = [None] * len(objects)
    errors: list = []

    def lane(k):
        try:
            e = engines[k]
            for j in range(k, len(objects), S):
                obj, cfg = objects[j], configs[j]
                x0 = init_poses(model, obj, cfg.batch, cfg.seed, cfg.init)
                e.set_object(obj)
                out[j] = e.synthesize(cfg, x0).records(cfg, obj)
        except Exception as exc:  # surfaced on the caller's thread below
            errors.append(exc)

    threads = [threading.Thread(target=lane, args=(k,)) for k in range(S)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return out  # type: ignore[return-value]
