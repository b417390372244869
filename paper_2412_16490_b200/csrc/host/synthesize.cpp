// C++ drop-in for grasp::pipeline::synthesize (reference pipeline.cpp:436-457):
// validate -> init_poses (host, one RNG stream) -> GPU three-stage loop via
// the C ABI -> std::vector<GraspRecord> in input order.
#include "../../../include/grasp_b200.h"

#include "capi_common.hpp"
#include "grasp/pipeline.hpp"

#include <cmath>
#include <limits>
#include <map>
#include <memory>
#include <stdexcept>

namespace grasp::pipeline {
namespace {

struct CtxDeleter {
  void operator()(grasp_ctx* c) const { grasp_ctx_destroy(c); }
};

// One device context per (thread, device); models are re-uploaded only when
// the caller passes different model objects.
struct CachedCtx {
  std::unique_ptr<grasp_ctx, CtxDeleter> ctx;
  const hand::HandModel* hand = nullptr;
  const object::ObjectModel* object = nullptr;
  capi::PackedHand packed_hand;
  capi::PackedObject packed_object;
};

void check(int status) {
  if (status == GRASP_OK) return;
  const std::string msg = grasp_last_error();
  switch (status) {
    case GRASP_EINVAL: throw std::invalid_argument(msg);
    case GRASP_EGEOM: throw geom::GeometryError(msg);
    case GRASP_EHAND: throw hand::HandError(msg);
    case GRASP_EOBJECT: throw object::ObjectError(msg);
    default: throw std::runtime_error(msg);
  }
}

CachedCtx& context_for(int device) {
  thread_local std::map<int, CachedCtx> cache;
  CachedCtx& c = cache[device];
  if (!c.ctx) {
    grasp_ctx* raw = nullptr;
    check(grasp_ctx_create(device, &raw));
    c.ctx.reset(raw);
  }
  return c;
}

}  // namespace

std::vector<records::GraspRecord> synthesize(const hand::HandModel& model, const object::ObjectModel& object,
                                             const RunConfig& cfg, int device) {
  validate(cfg);
  CachedCtx& c = context_for(device);
  if (c.hand != &model) {
    c.packed_hand = capi::pack_hand(model);
    check(grasp_ctx_set_hand(c.ctx.get(), &c.packed_hand.desc));
    c.hand = &model;
  }
  if (c.object != &object) {
    c.packed_object = capi::pack_object(object);
    c.packed_object.desc.source = c.packed_object.source.c_str();
    check(grasp_ctx_set_object(c.ctx.get(), &c.packed_object.desc));
    c.object = &object;
  }
  const int B = cfg.batch, D = 12 + model.dof(), m = static_cast<int>(model.fingertip_links.size());
  const int n = m * cfg.contact.n_edges;
  const std::vector<VectorXd> starts = init_poses(model, object, B, cfg.seed, cfg.init);
  std::vector<double> x0(static_cast<size_t>(B) * D);
  for (int g = 0; g < B; ++g) std::copy(starts[g].begin(), starts[g].end(), x0.begin() + static_cast<size_t>(g) * D);

  std::vector<double> x_p(x0.size()), x(x0.size()), x_s(x0.size()), energy(B), per(6 * B),
      forces(static_cast<size_t>(B) * n * 6), contacts(static_cast<size_t>(B) * m * 12), stage(6 * B);
  std::vector<int> failed(B), conv(6 * B);
  grasp_out out{x_p.data(), x.data(), x_s.data(), energy.data(), per.data(), forces.data(),
                contacts.data(), stage.data(), failed.data(), conv.data()};
  grasp_run_params p;
  capi::from_config(cfg, &p);
  check(grasp_synthesize(c.ctx.get(), &p, B, x0.data(), &out));

  static const char* kNames[3] = {"coarse", "fine", "final"};
  const int iters[3] = {cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters};
  const int n_stages = cfg.pipeline.skip_fine_stages ? 1 : 3;
  std::vector<records::GraspRecord> recs(B);
  for (int g = 0; g < B; ++g) {
    records::GraspRecord& r = recs[g];
    auto slice = [&](const std::vector<double>& v) {
      return VectorXd(v.begin() + static_cast<size_t>(g) * D, v.begin() + static_cast<size_t>(g + 1) * D);
    };
    r.x_p = slice(x_p);
    r.x = slice(x);
    r.x_s = slice(x_s);
    r.index = g;
    r.seed = cfg.seed;
    r.object_id = object.source;
    r.object_scale = object.scale;
    r.failed = failed[g] != 0;
    r.note = failed[g] == 1 ? "non-finite energy" : (failed[g] == 2 ? "diverged" : "");
    for (int s = 0; s < n_stages; ++s)
      r.stages.push_back({kNames[s], iters[s], stage[6 * g + 2 * s], stage[6 * g + 2 * s + 1]});
    if (r.failed) {
      r.energy_total = std::numeric_limits<double>::quiet_NaN();
      continue;
    }
    r.energy_total = energy[g];
    r.per_direction.assign(per.begin() + 6 * g, per.begin() + 6 * g + 6);
    r.contact_force_rows = n;
    r.contact_force_cols = 6;
    r.contact_forces.assign(forces.begin() + static_cast<size_t>(g) * n * 6,
                            forces.begin() + static_cast<size_t>(g + 1) * n * 6);
    for (int f = 0; f < m; ++f) {
      const double* cf = contacts.data() + (static_cast<size_t>(g) * m + f) * 12;
      contact::ContactFrame fr;
      fr.p = Vec3(cf[0], cf[1], cf[2]);
      fr.n = Vec3(cf[3], cf[4], cf[5]);
      fr.d = Vec3(cf[6], cf[7], cf[8]);
      fr.e = Vec3(cf[9], cf[10], cf[11]);
      r.contacts.push_back(fr);
    }
  }
  return recs;
}

}  // namespace grasp::pipeline
