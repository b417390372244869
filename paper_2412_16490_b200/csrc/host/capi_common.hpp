// Shared helpers between the host and device halves of the C ABI.
#pragma once

#include "../../../include/grasp_b200.h"
#include "grasp/config.hpp"
#include "grasp/hand.hpp"
#include "grasp/object.hpp"

#include <string>
#include <vector>

namespace grasp::capi {

extern thread_local std::string g_last_error;
int fail(int code, const std::string& msg);

RunConfig to_config(const grasp_run_params* p);
void from_config(const RunConfig& c, grasp_run_params* p);

struct PackedHand {
  std::vector<int> link_parent_joint, link_tip_proxy, link_vert_begin, link_face_begin, link_proxy_begin;
  std::vector<double> verts;
  std::vector<int> faces;
  std::vector<double> link_obb, link_centroid, link_volume, proxies;
  std::vector<int> joint_parent_link, joint_child_link;
  std::vector<double> joint_origin, joint_axis, joint_lower, joint_upper;
  std::vector<int> tip_links, collision_pairs;
  grasp_hand_desc desc{};
};

struct PackedObject {
  std::vector<int> part_vert_begin, part_face_begin;
  std::vector<double> verts;
  std::vector<int> faces;
  std::vector<double> part_obb, part_centroid, part_volume;
  std::string source;
  grasp_object_desc desc{};
};

PackedHand pack_hand(const hand::HandModel& m);
PackedObject pack_object(const object::ObjectModel& m);

const hand::HandModel& hand_model(const grasp_hand* h);
const object::ObjectModel& object_model(const grasp_object* o);

}  // namespace grasp::capi
