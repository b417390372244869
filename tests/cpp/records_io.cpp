// Writes records with tricky doubles through grasp::records::write_records, reads them back
// and checks the to_line round trip (tests/test_records_jsonl.py compares the bytes with the
// oracle's restatement of nlohmann's dump).
#include "grasp/records.hpp"

#include <cmath>
#include <cstdio>
#include <limits>
#include <vector>

int main(int argc, char** argv) {
  using namespace grasp;
  if (argc < 2) return 2;
  const double vals[] = {0.0, -0.0, 1.0, -1.0, 0.1, 1e-4, 1e-5, 9.999e-5, 1234.5678, 1e15, 1e16, 123456789012345.0,
                         1234567890123456.0, 3.141592653589793, -2.5e-300, 1.7976931348623157e308, 5e-324, 0.30000000000000004,
                         100.0, 1e21, 6.02214076e23, std::numeric_limits<double>::quiet_NaN()};
  std::vector<records::GraspRecord> recs(3);
  for (int i = 0; i < 3; ++i) {
    auto& r = recs[i];
    for (double v : vals) r.x.push_back(v * (i + 1));
    r.x_p = {0.25, -0.125, 7.0};
    r.x_s = {1e-10, 2e10};
    r.energy_total = i == 1 ? std::numeric_limits<double>::quiet_NaN() : 0.0123456789 * (i + 1);
    r.per_direction = {1.5, 2.25, 3.0, 4e-7, 5e7, 6.0};
    r.contact_force_rows = 2;
    r.contact_force_cols = 3;
    r.contact_forces = {0.1, 0.2, 0.3, 0.4, 0.5, 0.6};
    contact::ContactFrame f;
    f.p = Vec3(0.01, -0.02, 0.03);
    r.contacts = {f, f};
    r.object_id = i == 2 ? "quote\"back\\slash\ttab\x01" : "drill_like";
    r.object_scale = 0.1;
    r.seed = 18446744073709551615ull;
    r.index = i;
    r.failed = i == 1;
    r.note = i == 1 ? "non-finite energy" : "";
    r.stages = {{"coarse", 300, 1.25, 0.5}, {"fine", 100, 0.5, 0.25}};
  }
  records::write_records(argv[1], recs);
  const auto back = records::read_records(argv[1]);
  if (back.size() != recs.size()) return 3;
  for (size_t i = 0; i < recs.size(); ++i)
    if (records::to_line(back[i]) != records::to_line(recs[i])) return 4;
  std::printf("ok %zu\n", back.size());
  return 0;
}
