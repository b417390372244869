"""B200-native batched bilevel grasp synthesis (BODex, arXiv 2412.16490).

Drop-in for the reference's hot path grasp::pipeline::synthesize
(proj/src/pipeline.cpp:436-457): C++ host code + hand-written sm_100a CUDA
kernels behind the C ABI in include/grasp_b200.h.
"""
from .api import (  # noqa: F401
    ContactFrame, ContactParams, Engine, EnergyParams, EvalParams, GraspRecord, HandModel, InitParams,
    ObjectiveWeights, ObjectModel, PipelineParams, QpParams, RunConfig, StageSchedule, StageTrace,
    SynthesisOutput, build_convex_parts, builtin_hand_json, init_poses, load_object, make_primitive, parse_object_text,
    parse_run_config, squeeze_pose, synthesize, synthesize_objects, validate, PRIMITIVE_NAMES, forward_kinematics,
)
from .errors import CudaError, GeometryError, GraspError, HandError, InvalidArgument, ObjectError  # noqa: F401
