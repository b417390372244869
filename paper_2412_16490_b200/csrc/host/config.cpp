// RunConfig JSON and validation (reference proj/src/config.cpp:13-229).
#include "grasp/config.hpp"

#include "json_lite.hpp"

#include <map>
#include <sstream>
#include <stdexcept>

namespace grasp {
namespace {

// Applies present keys onto defaults and rejects unknown keys (config.cpp:13-47).
class Fields {
 public:
  Fields(const json::Value& j, std::string scope) : j_(j), scope_(std::move(scope)) {
    if (!j_.is_object()) throw std::invalid_argument(scope_ + " must be a JSON object");
    for (const auto& kv : j_.members()) seen_[kv.first] = false;
  }
  void get(const char* key, double& out) {
    if (const json::Value* v = take(key)) out = v->as_double();
  }
  void get(const char* key, int& out) {
    if (const json::Value* v = take(key)) out = static_cast<int>(v->as_int());
  }
  void get(const char* key, std::uint64_t& out) {
    if (const json::Value* v = take(key)) out = v->as_uint64();
  }
  void get(const char* key, bool& out) {
    if (const json::Value* v = take(key)) out = v->as_bool();
  }
  const json::Value* sub(const char* key) { return take(key); }
  void finish() const {
    for (const auto& [key, used] : seen_)
      if (!used) throw std::invalid_argument("unknown field '" + key + "' in " + scope_);
  }

 private:
  const json::Value* take(const char* key) {
    const json::Value* v = j_.find(key);
    if (v) seen_[key] = true;
    return v;
  }
  const json::Value& j_;
  std::string scope_;
  std::map<std::string, bool> seen_;
};

void read_stage(const json::Value& j, const char* name, StageSchedule& s) {
  Fields r(j, name);
  r.get("iters", s.iters);
  r.get("step_rotation", s.step_rotation);
  r.get("step_translation", s.step_translation);
  r.get("step_joints", s.step_joints);
  r.get("step_floor", s.step_floor);
  r.finish();
}

void require(bool cond, const char* what) {
  if (!cond) throw std::invalid_argument(std::string("config: ") + what);
}

std::string num(double v) { return json::format_double(v); }

std::string stage_json(const StageSchedule& s) {
  std::ostringstream o;
  o << "{\"iters\": " << s.iters << ", \"step_floor\": " << num(s.step_floor)
    << ", \"step_joints\": " << num(s.step_joints) << ", \"step_rotation\": " << num(s.step_rotation)
    << ", \"step_translation\": " << num(s.step_translation) << "}";
  return o.str();
}

}  // namespace

RunConfig parse_run_config(const std::string& json_text) {
  json::Value j;
  try {
    j = json::parse(json_text);
  } catch (const json::ParseError& e) {
    throw std::invalid_argument(e.what());
  }
  RunConfig cfg;
  try {
    Fields r(j, "config");
    if (const json::Value* s = r.sub("qp")) {
      Fields q(*s, "qp");
      q.get("rho", cfg.qp.rho);
      q.get("sigma", cfg.qp.sigma);
      q.get("alpha", cfg.qp.alpha);
      q.get("max_iters", cfg.qp.max_iters);
      q.get("eps_primal", cfg.qp.eps_primal);
      q.get("eps_dual", cfg.qp.eps_dual);
      q.get("check_interval", cfg.qp.check_interval);
      q.finish();
    }
    if (const json::Value* s = r.sub("contact")) {
      Fields q(*s, "contact");
      q.get("mu", cfg.contact.mu);
      q.get("n_edges", cfg.contact.n_edges);
      q.finish();
    }
    if (const json::Value* s = r.sub("energy")) {
      Fields q(*s, "energy");
      q.get("beta", cfg.energy.beta);
      q.get("gamma_per_contact", cfg.energy.gamma_per_contact);
      q.finish();
    }
    if (const json::Value* s = r.sub("weights")) {
      Fields q(*s, "weights");
      q.get("grasp", cfg.weights.grasp);
      q.get("distance", cfg.weights.distance);
      q.get("joint_limit", cfg.weights.joint_limit);
      q.get("self_penetration", cfg.weights.self_penetration);
      q.get("object_penetration", cfg.weights.object_penetration);
      q.finish();
    }
    if (const json::Value* s = r.sub("pipeline")) {
      Fields q(*s, "pipeline");
      if (const json::Value* t = q.sub("coarse")) read_stage(*t, "pipeline.coarse", cfg.pipeline.coarse);
      if (const json::Value* t = q.sub("fine")) read_stage(*t, "pipeline.fine", cfg.pipeline.fine);
      if (const json::Value* t = q.sub("final")) read_stage(*t, "pipeline.final", cfg.pipeline.final_stage);
      q.get("contact_offset", cfg.pipeline.contact_offset);
      q.get("fd_step", cfg.pipeline.fd_step);
      q.get("skip_fine_stages", cfg.pipeline.skip_fine_stages);
      q.finish();
    }
    if (const json::Value* s = r.sub("init")) {
      Fields q(*s, "init");
      q.get("standoff", cfg.init.standoff);
      q.get("joint_span_fraction", cfg.init.joint_span_fraction);
      q.finish();
    }
    if (const json::Value* s = r.sub("eval")) {
      Fields q(*s, "eval");
      q.get("mass", cfg.eval.mass);
      q.get("gravity", cfg.eval.gravity);
      q.get("residual_rel_tol", cfg.eval.residual_rel_tol);
      q.get("force_budget_factor", cfg.eval.force_budget_factor);
      q.get("contact_tol", cfg.eval.contact_tol);
      q.get("penetration_tol", cfg.eval.penetration_tol);
      q.get("qp_eps", cfg.eval.qp_eps);
      q.finish();
    }
    r.get("seed", cfg.seed);
    r.get("batch", cfg.batch);
    r.get("workers", cfg.workers);
    r.finish();
  } catch (const json::TypeError& e) {
    throw std::invalid_argument(std::string("config: ") + e.what());
  }
  validate(cfg);
  return cfg;
}

std::string dump_run_config(const RunConfig& cfg) {
  std::ostringstream o;
  o << "{\"batch\": " << cfg.batch << ", \"contact\": {\"mu\": " << num(cfg.contact.mu)
    << ", \"n_edges\": " << cfg.contact.n_edges << "}, \"energy\": {\"beta\": " << num(cfg.energy.beta)
    << ", \"gamma_per_contact\": " << num(cfg.energy.gamma_per_contact) << "}, \"eval\": {\"contact_tol\": "
    << num(cfg.eval.contact_tol) << ", \"force_budget_factor\": " << num(cfg.eval.force_budget_factor)
    << ", \"gravity\": " << num(cfg.eval.gravity) << ", \"mass\": " << num(cfg.eval.mass)
    << ", \"penetration_tol\": " << num(cfg.eval.penetration_tol) << ", \"qp_eps\": " << num(cfg.eval.qp_eps)
    << ", \"residual_rel_tol\": " << num(cfg.eval.residual_rel_tol) << "}, \"init\": {\"joint_span_fraction\": "
    << num(cfg.init.joint_span_fraction) << ", \"standoff\": " << num(cfg.init.standoff)
    << "}, \"pipeline\": {\"coarse\": " << stage_json(cfg.pipeline.coarse)
    << ", \"contact_offset\": " << num(cfg.pipeline.contact_offset) << ", \"fd_step\": " << num(cfg.pipeline.fd_step)
    << ", \"final\": " << stage_json(cfg.pipeline.final_stage) << ", \"fine\": " << stage_json(cfg.pipeline.fine)
    << ", \"skip_fine_stages\": " << (cfg.pipeline.skip_fine_stages ? "true" : "false")
    << "}, \"qp\": {\"alpha\": " << num(cfg.qp.alpha) << ", \"check_interval\": " << cfg.qp.check_interval
    << ", \"eps_dual\": " << num(cfg.qp.eps_dual) << ", \"eps_primal\": " << num(cfg.qp.eps_primal)
    << ", \"max_iters\": " << cfg.qp.max_iters << ", \"rho\": " << num(cfg.qp.rho)
    << ", \"sigma\": " << num(cfg.qp.sigma) << "}, \"seed\": " << cfg.seed << ", \"weights\": {\"distance\": "
    << num(cfg.weights.distance) << ", \"grasp\": " << num(cfg.weights.grasp) << ", \"joint_limit\": "
    << num(cfg.weights.joint_limit) << ", \"object_penetration\": " << num(cfg.weights.object_penetration)
    << ", \"self_penetration\": " << num(cfg.weights.self_penetration) << "}, \"workers\": " << cfg.workers << "}";
  return o.str();
}

void validate(const RunConfig& cfg) {
  require(cfg.qp.rho > 0, "qp.rho must be positive");
  require(cfg.qp.sigma > 0, "qp.sigma must be positive");
  require(cfg.qp.alpha > 0 && cfg.qp.alpha < 2, "qp.alpha must lie in (0, 2)");
  require(cfg.qp.max_iters > 0, "qp.max_iters must be positive");
  require(cfg.qp.eps_primal > 0 && cfg.qp.eps_dual > 0, "qp tolerances must be positive");
  require(cfg.qp.check_interval > 0, "qp.check_interval must be positive");
  require(cfg.contact.mu > 0, "contact.mu must be positive");
  require(cfg.contact.n_edges >= 3, "contact.n_edges must be at least 3");
  require(cfg.energy.beta >= 0, "energy.beta must be nonnegative");
  require(cfg.energy.gamma_per_contact >= 0 && cfg.energy.gamma_per_contact <= 1,
          "energy.gamma_per_contact must lie in [0, 1]");
  for (const StageSchedule* s : {&cfg.pipeline.coarse, &cfg.pipeline.fine, &cfg.pipeline.final_stage}) {
    require(s->iters >= 0, "stage iters must be nonnegative");
    require(s->step_rotation >= 0 && s->step_translation >= 0 && s->step_joints >= 0,
            "stage steps must be nonnegative");
    require(s->step_floor > 0 && s->step_floor <= 1, "stage step_floor must lie in (0, 1]");
  }
  require(cfg.pipeline.contact_offset >= 0, "pipeline.contact_offset must be nonnegative");
  require(cfg.pipeline.fd_step > 0, "pipeline.fd_step must be positive");
  require(cfg.init.standoff >= 0, "init.standoff must be nonnegative");
  require(cfg.init.joint_span_fraction >= 0 && cfg.init.joint_span_fraction <= 1,
          "init.joint_span_fraction must lie in [0, 1]");
  require(cfg.eval.mass > 0, "eval.mass must be positive");
  require(cfg.eval.gravity > 0, "eval.gravity must be positive");
  require(cfg.eval.residual_rel_tol > 0, "eval.residual_rel_tol must be positive");
  require(cfg.eval.force_budget_factor > 0, "eval.force_budget_factor must be positive");
  require(cfg.eval.contact_tol >= 0, "eval.contact_tol must be nonnegative");
  require(cfg.eval.penetration_tol >= 0, "eval.penetration_tol must be nonnegative");
  require(cfg.eval.qp_eps > 0, "eval.qp_eps must be positive");
  require(cfg.batch > 0, "batch must be positive");
  require(cfg.workers > 0, "workers must be positive");
}

}  // namespace grasp
