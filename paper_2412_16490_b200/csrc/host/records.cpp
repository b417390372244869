// Record JSONL I/O (reference proj/src/records.cpp:65-152). The reference
// dumps with nlohmann/json 3.11 (object keys sorted, compact, doubles through
// its Grisu2 to_chars and format_buffer layout); here the same layout is
// produced from std::to_chars' shortest round-trip digits, and lines are
// parsed with json_lite.
#include "grasp/records.hpp"

#include "json_lite.hpp"

#include <charconv>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <limits>
#include <sstream>

namespace grasp::records {

std::string format_json_double(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
  std::string s(buf, r.ptr);
  const bool neg = s[0] == '-';
  if (neg) s.erase(0, 1);
  const size_t epos = s.find('e');
  std::string digits;
  for (size_t i = 0; i < epos; ++i)
    if (s[i] != '.') digits += s[i];
  const int k = static_cast<int>(digits.size());
  const int n = std::stoi(s.substr(epos + 1)) + 1;  // value = 0.d1..dk x 10^n
  std::string out;
  if (k <= n && n <= 15) {
    out = digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string(-n, '0') + digits;
  } else {
    out = digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    int e = n - 1;
    out += 'e';
    out += e < 0 ? '-' : '+';
    e = std::abs(e);
    if (e < 10) out += '0';
    out += std::to_string(e);
  }
  return neg ? "-" + out : out;
}

namespace {

// nlohmann's escape rules with ensure_ascii = false.
std::string quote(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof(b), "\\u%04x", c);
          o += b;
        } else {
          o += static_cast<char>(c);
        }
    }
  }
  return o + "\"";
}

std::string vec(const double* v, size_t n) {
  std::string o = "[";
  for (size_t i = 0; i < n; ++i) {
    if (i) o += ",";
    o += format_json_double(v[i]);
  }
  return o + "]";
}
std::string vec(const std::vector<double>& v) { return vec(v.data(), v.size()); }
std::string vec3(const Vec3& v) {
  const double a[3] = {v.x, v.y, v.z};
  return vec(a, 3);
}

double num(const json::Value& v) { return v.is_null() ? std::numeric_limits<double>::quiet_NaN() : v.as_double(); }
std::vector<double> load_vec(const json::Value& a) {
  std::vector<double> out;
  for (const auto& x : a.items()) out.push_back(num(x));
  return out;
}
Vec3 load_vec3(const json::Value& a) {
  const auto v = load_vec(a);
  if (v.size() != 3) throw RecordError("record line is missing fields: frame vector size");
  return Vec3(v[0], v[1], v[2]);
}

}  // namespace

std::string to_line(const GraspRecord& r) {
  // keys in sorted order (nlohmann::json objects are std::map)
  std::string o = "{";
  o += "\"contact_forces\":[";
  for (int c = 0; c < r.contact_force_cols; ++c) {
    if (c) o += ",";
    o += vec(r.contact_forces.data() + static_cast<size_t>(c) * r.contact_force_rows,
             static_cast<size_t>(r.contact_force_rows));
  }
  o += "],\"contacts\":[";
  for (size_t i = 0; i < r.contacts.size(); ++i) {
    const auto& f = r.contacts[i];
    if (i) o += ",";
    o += "{\"d\":" + vec3(f.d) + ",\"e\":" + vec3(f.e) + ",\"n\":" + vec3(f.n) + ",\"p\":" + vec3(f.p) + "}";
  }
  o += "],\"energy_total\":" + format_json_double(r.energy_total);
  o += ",\"failed\":" + std::string(r.failed ? "true" : "false");
  o += ",\"index\":" + std::to_string(r.index);
  o += ",\"note\":" + quote(r.note);
  o += ",\"object_id\":" + quote(r.object_id);
  o += ",\"object_scale\":" + format_json_double(r.object_scale);
  o += ",\"per_direction\":" + vec(r.per_direction);
  o += ",\"seed\":" + std::to_string(r.seed);
  o += ",\"stages\":[";
  for (size_t i = 0; i < r.stages.size(); ++i) {
    const auto& s = r.stages[i];
    if (i) o += ",";
    o += "{\"energy_end\":" + format_json_double(s.energy_end) + ",\"energy_start\":" +
         format_json_double(s.energy_start) + ",\"iterations\":" + std::to_string(s.iterations) +
         ",\"stage\":" + quote(s.stage) + "}";
  }
  o += "],\"version\":" + std::to_string(kFormatVersion);
  o += ",\"x\":" + vec(r.x) + ",\"x_p\":" + vec(r.x_p) + ",\"x_s\":" + vec(r.x_s) + "}";
  return o;
}

GraspRecord from_line(const std::string& line) {
  json::Value j;
  try {
    j = json::parse(line);
  } catch (const std::exception& e) {
    throw RecordError(std::string("record line is not valid JSON: ") + e.what());
  }
  try {
    const int version = static_cast<int>(j.at("version").as_int());
    if (version != kFormatVersion)
      throw RecordError("record version " + std::to_string(version) + " does not match reader version " +
                        std::to_string(kFormatVersion));
    GraspRecord r;
    r.x_p = load_vec(j.at("x_p"));
    r.x = load_vec(j.at("x"));
    r.x_s = load_vec(j.at("x_s"));
    r.energy_total = num(j.at("energy_total"));
    r.per_direction = load_vec(j.at("per_direction"));
    const auto& cols = j.at("contact_forces");
    r.contact_force_cols = static_cast<int>(cols.size());
    for (size_t c = 0; c < cols.size(); ++c) {
      const auto col = load_vec(cols.at(c));
      if (c == 0) r.contact_force_rows = static_cast<int>(col.size());
      r.contact_forces.insert(r.contact_forces.end(), col.begin(), col.end());
    }
    for (const auto& f : j.at("contacts").items()) {
      contact::ContactFrame fr;
      fr.p = load_vec3(f.at("p"));
      fr.n = load_vec3(f.at("n"));
      fr.d = load_vec3(f.at("d"));
      fr.e = load_vec3(f.at("e"));
      r.contacts.push_back(fr);
    }
    r.object_id = j.at("object_id").as_string();
    r.object_scale = num(j.at("object_scale"));
    r.seed = j.at("seed").as_uint64();
    r.index = static_cast<int>(j.at("index").as_int());
    r.failed = j.at("failed").as_bool();
    r.note = j.at("note").as_string();
    for (const auto& s : j.at("stages").items())
      r.stages.push_back({s.at("stage").as_string(), static_cast<int>(s.at("iterations").as_int()),
                          num(s.at("energy_start")), num(s.at("energy_end"))});
    return r;
  } catch (const RecordError&) {
    throw;
  } catch (const std::exception& e) {
    throw RecordError(std::string("record line is missing fields: ") + e.what());
  }
}

void write_records(const std::string& path, std::span<const GraspRecord> records) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw RecordError(path + ": cannot open for writing");
  for (const auto& r : records) out << to_line(r) << "\n";
  out.flush();
  if (!out) throw RecordError(path + ": write failed");
}

std::vector<GraspRecord> read_records(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw RecordError(path + ": cannot open records file");
  std::vector<GraspRecord> records;
  std::string line;
  int line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty()) continue;
    try {
      records.push_back(from_line(line));
    } catch (const RecordError& e) {
      throw RecordError(path + ":" + std::to_string(line_no) + ": " + e.what());
    }
  }
  return records;
}

}  // namespace grasp::records
