// The debug/test library libgrasp_b200_debug.so: the whole engine plus the debug surfaces
// (grasp_debug_epa, grasp_debug_point_to_mesh_warm, grasp_debug_cos). Tests that need them load
// this library in a subprocess (GRASP_LIB); the product libgrasp_b200.so carries none of them.
#define GRASP_DEBUG_SURFACES
#include "engine.cu"
