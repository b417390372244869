// A reference-style C++ caller: same calls as proj/tests/test_pipeline.cpp
// (builtin_hand, make_primitive, RunConfig, synthesize), linked against
// libgrasp_b200.so instead of the reference's static library.
#include "grasp/config.hpp"
#include "grasp/eval.hpp"
#include "grasp/hand.hpp"
#include "grasp/object.hpp"
#include "grasp/pipeline.hpp"

#include <cmath>
#include <cstdio>

int main() {
  using namespace grasp;
  const hand::HandModel& model = hand::builtin_hand();
  const object::ObjectModel sphere = object::make_primitive("sphere", 0.1);
  RunConfig cfg;
  cfg.batch = 6;
  cfg.seed = 17;
  cfg.pipeline.coarse.iters = 120;
  cfg.pipeline.fine.iters = 50;
  cfg.pipeline.final_stage.iters = 50;
  const auto recs = pipeline::synthesize(model, sphere, cfg);
  int ok = 0;
  for (const auto& r : recs) {
    if (r.failed) continue;
    ++ok;
    if (r.contacts.size() != 3 || r.per_direction.size() != 6 || !std::isfinite(r.energy_total)) return 2;
    const auto xs = pipeline::squeeze_pose(model, r.x, r.x_p);
    for (size_t i = 0; i < xs.size(); ++i)
      if (std::abs(xs[i] - r.x_s[i]) > 1e-9) return 3;
  }
  std::printf("records %zu ok %d stages %zu object %s\n", recs.size(), ok, recs[0].stages.size(),
              recs[0].object_id.c_str());
  // grasp evaluation (eval.hpp): one device pass over all records
  const auto evals = eval::quasi_static_check(model, recs, sphere, cfg);
  if (evals.size() != recs.size()) return 5;
  for (const auto& e : evals)
    if (!(e.pd_mm >= 0.0) || !(e.spd_mm >= 0.0) || !(e.cdc_mm >= 0.0) || e.contact_count < 0 || e.contact_count > 3)
      return 6;
  std::printf("eval: success %d contacts %d pd %.3f mm notes '%s'\n", (int)evals[0].success, evals[0].contact_count,
              evals[0].pd_mm, evals[0].notes.c_str());
  try {
    RunConfig bad = cfg;
    bad.qp.alpha = 2.5;
    pipeline::synthesize(model, sphere, bad);
    return 4;
  } catch (const std::invalid_argument&) {
  }
  return ok >= 4 ? 0 : 1;
}
