// Grasp evaluation API (reference include/grasp/eval.hpp:16-60), computed on the
// device through grasp_eval (include/grasp_b200.h). Vectors are std::vector/Vec
// instead of Eigen; names, fields and semantics follow the reference.
#pragma once

#include <array>
#include <string>
#include <vector>

#include "grasp/config.hpp"
#include "grasp/hand.hpp"
#include "grasp/object.hpp"
#include "grasp/records.hpp"

namespace grasp::eval {

using VectorXd = std::vector<double>;

struct EvalResult {
  bool success = false;
  std::array<double, 6> per_direction_residuals{};  // unresisted wrench norms [N]
  double pd_mm = 0.0;
  double spd_mm = 0.0;
  double cdc_mm = 0.0;
  int contact_count = 0;
  std::string notes;
};

/// eval.cpp:91-158 for one record (x, x_s).
EvalResult quasi_static_check(const hand::HandModel& model, const records::GraspRecord& record,
                              const object::ObjectModel& object, const RunConfig& cfg, int device = 0);
/// The same for a batch of records in one device pass.
std::vector<EvalResult> quasi_static_check(const hand::HandModel& model,
                                           const std::vector<records::GraspRecord>& records,
                                           const object::ObjectModel& object, const RunConfig& cfg,
                                           int device = 0);
/// eval.cpp:51-61 [mm].
double penetration_depth(const hand::HandModel& model, const VectorXd& x, const object::ObjectModel& object,
                         int device = 0);
/// eval.cpp:63-72 [mm].
double self_penetration_depth(const hand::HandModel& model, const VectorXd& x, const object::ObjectModel& object,
                              int device = 0);
/// eval.cpp:84-89 [mm].
double contact_distance_consistency(const hand::HandModel& model, const VectorXd& x,
                                    const object::ObjectModel& object, int device = 0);

}  // namespace grasp::eval
