// Host half of the C ABI (include/grasp_b200.h): model handles, packing,
// run-parameter parsing/validation, init poses and squeeze.
#include "../../../include/grasp_b200.h"

#include "capi_common.hpp"
#include "grasp/config.hpp"
#include "grasp/hand.hpp"
#include "grasp/object.hpp"
#include "grasp/pipeline.hpp"

#include <cstring>

using namespace grasp;

namespace grasp::capi {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

RunConfig to_config(const grasp_run_params* p) {
  RunConfig c;
  c.qp.rho = p->qp_rho;
  c.qp.sigma = p->qp_sigma;
  c.qp.alpha = p->qp_alpha;
  c.qp.max_iters = p->qp_max_iters;
  c.qp.eps_primal = p->qp_eps_primal;
  c.qp.eps_dual = p->qp_eps_dual;
  c.qp.check_interval = p->qp_check_interval;
  c.contact.mu = p->mu;
  c.contact.n_edges = p->n_edges;
  c.energy.beta = p->beta;
  c.energy.gamma_per_contact = p->gamma_per_contact;
  c.weights.grasp = p->w_grasp;
  c.weights.distance = p->w_distance;
  c.weights.joint_limit = p->w_joint_limit;
  c.weights.self_penetration = p->w_self_penetration;
  c.weights.object_penetration = p->w_object_penetration;
  auto stage = [](const grasp_stage_params& s) {
    return StageSchedule{s.iters, s.step_rotation, s.step_translation, s.step_joints, s.step_floor};
  };
  c.pipeline.coarse = stage(p->coarse);
  c.pipeline.fine = stage(p->fine);
  c.pipeline.final_stage = stage(p->final_stage);
  c.pipeline.contact_offset = p->contact_offset;
  c.pipeline.fd_step = p->fd_step;
  c.pipeline.skip_fine_stages = p->skip_fine_stages != 0;
  c.init.standoff = p->standoff;
  c.init.joint_span_fraction = p->joint_span_fraction;
  c.seed = p->seed;
  c.batch = p->batch;
  c.workers = p->workers;
  return c;
}

void from_config(const RunConfig& c, grasp_run_params* p) {
  std::memset(p, 0, sizeof(*p));
  p->qp_rho = c.qp.rho;
  p->qp_sigma = c.qp.sigma;
  p->qp_alpha = c.qp.alpha;
  p->qp_max_iters = c.qp.max_iters;
  p->qp_eps_primal = c.qp.eps_primal;
  p->qp_eps_dual = c.qp.eps_dual;
  p->qp_check_interval = c.qp.check_interval;
  p->mu = c.contact.mu;
  p->n_edges = c.contact.n_edges;
  p->beta = c.energy.beta;
  p->gamma_per_contact = c.energy.gamma_per_contact;
  p->w_grasp = c.weights.grasp;
  p->w_distance = c.weights.distance;
  p->w_joint_limit = c.weights.joint_limit;
  p->w_self_penetration = c.weights.self_penetration;
  p->w_object_penetration = c.weights.object_penetration;
  auto stage = [](const StageSchedule& s) {
    return grasp_stage_params{s.iters, s.step_rotation, s.step_translation, s.step_joints, s.step_floor};
  };
  p->coarse = stage(c.pipeline.coarse);
  p->fine = stage(c.pipeline.fine);
  p->final_stage = stage(c.pipeline.final_stage);
  p->contact_offset = c.pipeline.contact_offset;
  p->fd_step = c.pipeline.fd_step;
  p->skip_fine_stages = c.pipeline.skip_fine_stages ? 1 : 0;
  p->standoff = c.init.standoff;
  p->joint_span_fraction = c.init.joint_span_fraction;
  p->seed = c.seed;
  p->batch = c.batch;
  p->workers = c.workers;
}

PackedHand pack_hand(const hand::HandModel& m) {
  PackedHand p;
  const int L = static_cast<int>(m.links.size());
  p.link_vert_begin.push_back(0);
  p.link_face_begin.push_back(0);
  p.link_proxy_begin.push_back(0);
  for (int l = 0; l < L; ++l) {
    const auto& ln = m.links[l];
    p.link_parent_joint.push_back(ln.parent_joint);
    p.link_tip_proxy.push_back(ln.tip_proxy);
    for (const Vec3& v : ln.part.vertices) {
      p.verts.push_back(v.x);
      p.verts.push_back(v.y);
      p.verts.push_back(v.z);
    }
    for (const auto& f : ln.part.faces)
      for (int k = 0; k < 3; ++k) p.faces.push_back(f[k]);
    p.link_vert_begin.push_back(p.link_vert_begin.back() + static_cast<int>(ln.part.vertices.size()));
    p.link_face_begin.push_back(p.link_face_begin.back() + static_cast<int>(ln.part.faces.size()));
    const auto& o = ln.part.obb;
    const double obb[15] = {o.center.x, o.center.y, o.center.z, o.half_extents.x, o.half_extents.y,
                            o.half_extents.z, o.rotation.m[0], o.rotation.m[1], o.rotation.m[2],
                            o.rotation.m[3], o.rotation.m[4], o.rotation.m[5], o.rotation.m[6],
                            o.rotation.m[7], o.rotation.m[8]};
    p.link_obb.insert(p.link_obb.end(), obb, obb + 15);
    p.link_centroid.push_back(ln.part.centroid.x);
    p.link_centroid.push_back(ln.part.centroid.y);
    p.link_centroid.push_back(ln.part.centroid.z);
    p.link_volume.push_back(ln.part.volume);
    for (const auto& s : ln.proxies) {
      p.proxies.push_back(s.center_local.x);
      p.proxies.push_back(s.center_local.y);
      p.proxies.push_back(s.center_local.z);
      p.proxies.push_back(s.radius);
    }
    p.link_proxy_begin.push_back(p.link_proxy_begin.back() + static_cast<int>(ln.proxies.size()));
  }
  for (const auto& j : m.joints) {
    p.joint_parent_link.push_back(j.parent_link);
    p.joint_child_link.push_back(j.child_link);
    p.joint_origin.insert(p.joint_origin.end(), {j.origin.x, j.origin.y, j.origin.z});
    p.joint_axis.insert(p.joint_axis.end(), {j.axis.x, j.axis.y, j.axis.z});
    p.joint_lower.push_back(j.lower);
    p.joint_upper.push_back(j.upper);
  }
  p.tip_links = m.fingertip_links;
  for (const auto& [a, b] : m.collision_pairs) {
    p.collision_pairs.push_back(a);
    p.collision_pairs.push_back(b);
  }
  grasp_hand_desc& d = p.desc;
  d.n_links = L;
  d.dof = m.dof();
  d.n_tips = static_cast<int>(m.fingertip_links.size());
  d.n_proxies = p.link_proxy_begin.back();
  d.n_pairs = static_cast<int>(m.collision_pairs.size());
  d.n_verts = p.link_vert_begin.back();
  d.n_faces = p.link_face_begin.back();
  d.link_parent_joint = p.link_parent_joint.data();
  d.link_tip_proxy = p.link_tip_proxy.data();
  d.link_vert_begin = p.link_vert_begin.data();
  d.link_face_begin = p.link_face_begin.data();
  d.link_proxy_begin = p.link_proxy_begin.data();
  d.verts = p.verts.data();
  d.faces = p.faces.data();
  d.link_obb = p.link_obb.data();
  d.link_centroid = p.link_centroid.data();
  d.link_volume = p.link_volume.data();
  d.proxies = p.proxies.data();
  d.joint_parent_link = p.joint_parent_link.data();
  d.joint_child_link = p.joint_child_link.data();
  d.joint_origin = p.joint_origin.data();
  d.joint_axis = p.joint_axis.data();
  d.joint_lower = p.joint_lower.data();
  d.joint_upper = p.joint_upper.data();
  d.tip_links = p.tip_links.data();
  d.collision_pairs = p.collision_pairs.data();
  return p;
}

PackedObject pack_object(const object::ObjectModel& m) {
  PackedObject p;
  p.source = m.source;
  p.part_vert_begin.push_back(0);
  p.part_face_begin.push_back(0);
  for (const auto& part : m.parts) {
    for (const Vec3& v : part.vertices) p.verts.insert(p.verts.end(), {v.x, v.y, v.z});
    for (const auto& f : part.faces) p.faces.insert(p.faces.end(), {f[0], f[1], f[2]});
    p.part_vert_begin.push_back(p.part_vert_begin.back() + static_cast<int>(part.vertices.size()));
    p.part_face_begin.push_back(p.part_face_begin.back() + static_cast<int>(part.faces.size()));
    const auto& o = part.obb;
    const double obb[15] = {o.center.x, o.center.y, o.center.z, o.half_extents.x, o.half_extents.y,
                            o.half_extents.z, o.rotation.m[0], o.rotation.m[1], o.rotation.m[2],
                            o.rotation.m[3], o.rotation.m[4], o.rotation.m[5], o.rotation.m[6],
                            o.rotation.m[7], o.rotation.m[8]};
    p.part_obb.insert(p.part_obb.end(), obb, obb + 15);
    p.part_centroid.insert(p.part_centroid.end(), {part.centroid.x, part.centroid.y, part.centroid.z});
    p.part_volume.push_back(part.volume);
  }
  grasp_object_desc& d = p.desc;
  d.n_parts = static_cast<int>(m.parts.size());
  d.n_verts = p.part_vert_begin.back();
  d.n_faces = p.part_face_begin.back();
  d.part_vert_begin = p.part_vert_begin.data();
  d.part_face_begin = p.part_face_begin.data();
  d.verts = p.verts.data();
  d.faces = p.faces.data();
  d.part_obb = p.part_obb.data();
  d.part_centroid = p.part_centroid.data();
  d.part_volume = p.part_volume.data();
  d.scale = m.scale;
  d.bbox_diagonal = m.bbox_diagonal;
  d.mass_center[0] = m.mass_center.x;
  d.mass_center[1] = m.mass_center.y;
  d.mass_center[2] = m.mass_center.z;
  d.source = p.source.c_str();
  return p;
}

}  // namespace grasp::capi

using namespace grasp::capi;

struct grasp_hand {
  hand::HandModel model;
  PackedHand packed;
};

struct grasp_object {
  object::ObjectModel model;
  PackedObject packed;
};

namespace {

template <class F>
int guard(F&& f) {
  try {
    f();
    return GRASP_OK;
  } catch (const hand::HandError& e) {
    return fail(GRASP_EHAND, e.what());
  } catch (const object::ObjectError& e) {
    return fail(GRASP_EOBJECT, e.what());
  } catch (const geom::GeometryError& e) {
    return fail(GRASP_EGEOM, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(GRASP_EINVAL, e.what());
  } catch (const std::bad_alloc&) {
    return fail(GRASP_ENOMEM, "out of host memory");
  } catch (const std::exception& e) {
    return fail(GRASP_EINVAL, e.what());
  }
}

grasp_hand* wrap_hand(hand::HandModel m) {
  auto* h = new grasp_hand{std::move(m), {}};
  h->packed = pack_hand(h->model);
  return h;
}

grasp_object* wrap_object(object::ObjectModel m) {
  auto* o = new grasp_object{std::move(m), {}};
  o->packed = pack_object(o->model);
  o->packed.desc.source = o->packed.source.c_str();  // SSO strings move with the object
  return o;
}

}  // namespace

const hand::HandModel& grasp::capi::hand_model(const grasp_hand* h) { return h->model; }
const object::ObjectModel& grasp::capi::object_model(const grasp_object* o) { return o->model; }

extern "C" {

const char* grasp_last_error(void) { return g_last_error.c_str(); }
const char* grasp_version(void) { return "paper_2412_16490_b200 0.1 (sm_100a, fp64)"; }

int grasp_hand_builtin(grasp_hand** out) {
  return guard([&] { *out = wrap_hand(hand::builtin_hand()); });
}

int grasp_hand_parse(const char* json_text, grasp_hand** out) {
  return guard([&] {
    if (!json_text) throw std::invalid_argument("null hand spec");
    *out = wrap_hand(hand::parse_hand_spec(json_text));
  });
}

void grasp_hand_free(grasp_hand* h) { delete h; }

int64_t grasp_hand_builtin_json(char* buf, int64_t cap) {
  const std::string& s = hand::builtin_hand_json();
  const int64_t need = static_cast<int64_t>(s.size()) + 1;
  if (buf && cap >= need) std::memcpy(buf, s.c_str(), static_cast<size_t>(need));
  return need;
}

int grasp_object_primitive(const char* name, double scale, grasp_object** out) {
  return guard([&] { *out = wrap_object(object::make_primitive(name ? name : "", scale)); });
}

int grasp_object_parse(const char* obj_text, double scale, const char* source, grasp_object** out) {
  return guard([&] {
    if (!obj_text) throw std::invalid_argument("null mesh text");
    *out = wrap_object(object::parse_object_text(obj_text, scale, source ? source : "mesh"));
  });
}

int grasp_object_from_points(int n_parts, const int* counts, const double* points, grasp_object** out) {
  return guard([&] {
    object::ObjectModel m;
    m.source = "points";
    size_t off = 0;
    for (int i = 0; i < n_parts; ++i) {
      std::vector<Vec3> pts;
      for (int k = 0; k < counts[i]; ++k, ++off) pts.emplace_back(points[3 * off], points[3 * off + 1], points[3 * off + 2]);
      m.parts.push_back(geom::make_convex_part(pts));
    }
    *out = wrap_object(std::move(m));
  });
}

void grasp_object_free(grasp_object* o) { delete o; }

double grasp_object_bounding_radius(const grasp_object* o) { return object::bounding_radius(o->model); }

int grasp_hand_describe(const grasp_hand* h, grasp_hand_desc* out) {
  if (!h || !out) return fail(GRASP_EINVAL, "null argument");
  *out = h->packed.desc;
  return GRASP_OK;
}

int grasp_object_describe(const grasp_object* o, grasp_object_desc* out) {
  if (!o || !out) return fail(GRASP_EINVAL, "null argument");
  *out = o->packed.desc;
  return GRASP_OK;
}

void grasp_run_params_default(grasp_run_params* p) { from_config(RunConfig{}, p); }

int grasp_run_params_parse(const char* json_text, grasp_run_params* out) {
  return guard([&] { from_config(parse_run_config(json_text ? json_text : ""), out); });
}

int grasp_run_params_validate(const grasp_run_params* p) {
  return guard([&] { validate(to_config(p)); });
}

int grasp_init_poses(const grasp_hand* h, const grasp_object* o, int n, uint64_t seed, double standoff,
                     double joint_span_fraction, double* out) {
  return guard([&] {
    InitParams ip;
    ip.standoff = standoff;
    ip.joint_span_fraction = joint_span_fraction;
    const auto states = pipeline::init_poses(h->model, o->model, n, seed, ip);
    const size_t D = 12 + static_cast<size_t>(h->model.dof());
    for (int i = 0; i < n; ++i) std::memcpy(out + i * D, states[i].data(), sizeof(double) * D);
  });
}

int grasp_forward_kinematics(const grasp_hand* h, int n, const double* x, double* out) {
  return guard([&] {
    if (!h || n < 0 || (n > 0 && (!x || !out))) throw std::invalid_argument("null argument");
    const size_t D = 12 + static_cast<size_t>(h->model.dof());
    const size_t L = h->model.links.size();
    for (int i = 0; i < n; ++i) {
      const std::vector<double> xv(x + i * D, x + (i + 1) * D);
      const auto fk = hand::forward_kinematics(h->model, hand::pose_from_state(h->model, xv));
      for (size_t l = 0; l < L; ++l) {
        double* o = out + (i * L + l) * 12;
        std::memcpy(o, fk.world[l].R.m, sizeof(double) * 9);
        o[9] = fk.world[l].t.x;
        o[10] = fk.world[l].t.y;
        o[11] = fk.world[l].t.z;
      }
    }
  });
}

int grasp_squeeze_pose(const grasp_hand* h, const double* x, const double* x_p, double* out) {
  return guard([&] {
    const size_t D = 12 + static_cast<size_t>(h->model.dof());
    const std::vector<double> xv(x, x + D), xp(x_p, x_p + D);
    const auto s = pipeline::squeeze_pose(h->model, xv, xp);
    std::memcpy(out, s.data(), sizeof(double) * D);
  });
}

}  // extern "C"
