"""Exception types mirroring the reference's error classes.

reference: std::invalid_argument (config.cpp:133-135), geom::GeometryError
(geometry.hpp:64-66), hand::HandError (hand.hpp:134-136),
object::ObjectError (object.hpp:27-29).
"""


class GraspError(RuntimeError):
    pass


class InvalidArgument(GraspError, ValueError):
    pass


class GeometryError(GraspError):
    pass


class HandError(GraspError):
    pass


class ObjectError(GraspError):
    pass


class CudaError(GraspError):
    pass


_BY_CODE = {1: InvalidArgument, 2: GeometryError, 3: HandError, 4: ObjectError, 5: CudaError, 6: MemoryError}


def raise_for(status: int, msg: str):
    raise _BY_CODE.get(status, GraspError)(msg)
