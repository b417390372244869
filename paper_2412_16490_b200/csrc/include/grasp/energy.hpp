// Mesh-stage surrogate (reference proj/include/grasp/energy.hpp, SurrogateResult and
// fine_stage_surrogate, energy.cpp:208-229). The lower-level grasp energy and its
// envelope gradient run batched on the GPU (qp.cuh); this header carries the
// single-call surrogate the pipeline API exposes.
#pragma once

#include "grasp/la.hpp"

#include <span>
#include <vector>

namespace grasp::energy {

struct SurrogateResult {
  double value = 0.0;
  std::vector<double> gradient;  // state layout; empty when no Jacobians were given
};

/// value = sum |p_i - a_i|^2; gradient = sum 2 J_i^T (p_i - a_i) when Jacobians are given.
SurrogateResult fine_stage_surrogate(std::span<const Vec3> points, std::span<const Vec3> anchors,
                                     std::span<const MatrixXd> jacobians);

}  // namespace grasp::energy
