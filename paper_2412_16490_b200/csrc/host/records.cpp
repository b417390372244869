// Record JSONL I/O (reference proj/src/records.cpp:65-152). The reference
// dumps with nlohmann/json 3.11 (object keys sorted, compact, doubles through
// its Grisu2 to_chars and format_buffer layout). The Grisu2 digits are NOT
// always the shortest-nearest ones std::to_chars gives (e.g. ...705.13 vs
// ...705.12), so the digit generation is restated here (boundaries, cached
// powers of ten, digit generation, round step) for byte-identical lines;
// tests/test_records_jsonl.py pins it to the real nlohmann 3.11.3. Lines are
// parsed with json_lite.
#include "grasp/records.hpp"

#include "json_lite.hpp"

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>

namespace grasp::records {
namespace {

// A 64-bit significand and binary exponent: f * 2^e.
struct Fp {
  std::uint64_t f;
  int e;
};

// High 64 bits of the 128-bit product, rounded half up on bits 32..63.
Fp fp_mul(Fp x, Fp y) {
  const std::uint64_t u_lo = x.f & 0xFFFFFFFFu, u_hi = x.f >> 32, v_lo = y.f & 0xFFFFFFFFu, v_hi = y.f >> 32;
  const std::uint64_t p0 = u_lo * v_lo, p1 = u_lo * v_hi, p2 = u_hi * v_lo, p3 = u_hi * v_hi;
  std::uint64_t q = (p0 >> 32) + (p1 & 0xFFFFFFFFu) + (p2 & 0xFFFFFFFFu);
  q += std::uint64_t{1} << 31;
  return {p3 + (p2 >> 32) + (p1 >> 32) + (q >> 32), x.e + y.e + 64};
}

Fp fp_normalize(Fp x) {
  while ((x.f >> 63) == 0) {
    x.f <<= 1;
    --x.e;
  }
  return x;
}

// 10^k ~ f * 2^e, k = -300, -292, ..., 324 (tools/gen_cached_powers.py: exact, rounded to nearest).
struct CachedPower {
  std::uint64_t f;
  int e, k;
};
constexpr CachedPower kCachedPowers[] = {
    {0xAB70FE17C79AC6CA, -1060, -300}, {0xFF77B1FCBEBCDC4F, -1034, -292}, {0xBE5691EF416BD60C, -1007, -284},
    {0x8DD01FAD907FFC3C, -980, -276}, {0xD3515C2831559A83, -954, -268}, {0x9D71AC8FADA6C9B5, -927, -260},
    {0xEA9C227723EE8BCB, -901, -252}, {0xAECC49914078536D, -874, -244}, {0x823C12795DB6CE57, -847, -236},
    {0xC21094364DFB5637, -821, -228}, {0x9096EA6F3848984F, -794, -220}, {0xD77485CB25823AC7, -768, -212},
    {0xA086CFCD97BF97F4, -741, -204}, {0xEF340A98172AACE5, -715, -196}, {0xB23867FB2A35B28E, -688, -188},
    {0x84C8D4DFD2C63F3B, -661, -180}, {0xC5DD44271AD3CDBA, -635, -172}, {0x936B9FCEBB25C996, -608, -164},
    {0xDBAC6C247D62A584, -582, -156}, {0xA3AB66580D5FDAF6, -555, -148}, {0xF3E2F893DEC3F126, -529, -140},
    {0xB5B5ADA8AAFF80B8, -502, -132}, {0x87625F056C7C4A8B, -475, -124}, {0xC9BCFF6034C13053, -449, -116},
    {0x964E858C91BA2655, -422, -108}, {0xDFF9772470297EBD, -396, -100}, {0xA6DFBD9FB8E5B88F, -369, -92},
    {0xF8A95FCF88747D94, -343, -84}, {0xB94470938FA89BCF, -316, -76}, {0x8A08F0F8BF0F156B, -289, -68},
    {0xCDB02555653131B6, -263, -60}, {0x993FE2C6D07B7FAC, -236, -52}, {0xE45C10C42A2B3B06, -210, -44},
    {0xAA242499697392D3, -183, -36}, {0xFD87B5F28300CA0E, -157, -28}, {0xBCE5086492111AEB, -130, -20},
    {0x8CBCCC096F5088CC, -103, -12}, {0xD1B71758E219652C, -77, -4}, {0x9C40000000000000, -50, 4},
    {0xE8D4A51000000000, -24, 12}, {0xAD78EBC5AC620000, 3, 20}, {0x813F3978F8940984, 30, 28},
    {0xC097CE7BC90715B3, 56, 36}, {0x8F7E32CE7BEA5C70, 83, 44}, {0xD5D238A4ABE98068, 109, 52},
    {0x9F4F2726179A2245, 136, 60}, {0xED63A231D4C4FB27, 162, 68}, {0xB0DE65388CC8ADA8, 189, 76},
    {0x83C7088E1AAB65DB, 216, 84}, {0xC45D1DF942711D9A, 242, 92}, {0x924D692CA61BE758, 269, 100},
    {0xDA01EE641A708DEA, 295, 108}, {0xA26DA3999AEF774A, 322, 116}, {0xF209787BB47D6B85, 348, 124},
    {0xB454E4A179DD1877, 375, 132}, {0x865B86925B9BC5C2, 402, 140}, {0xC83553C5C8965D3D, 428, 148},
    {0x952AB45CFA97A0B3, 455, 156}, {0xDE469FBD99A05FE3, 481, 164}, {0xA59BC234DB398C25, 508, 172},
    {0xF6C69A72A3989F5C, 534, 180}, {0xB7DCBF5354E9BECE, 561, 188}, {0x88FCF317F22241E2, 588, 196},
    {0xCC20CE9BD35C78A5, 614, 204}, {0x98165AF37B2153DF, 641, 212}, {0xE2A0B5DC971F303A, 667, 220},
    {0xA8D9D1535CE3B396, 694, 228}, {0xFB9B7CD9A4A7443C, 720, 236}, {0xBB764C4CA7A44410, 747, 244},
    {0x8BAB8EEFB6409C1A, 774, 252}, {0xD01FEF10A657842C, 800, 260}, {0x9B10A4E5E9913129, 827, 268},
    {0xE7109BFBA19C0C9D, 853, 276}, {0xAC2820D9623BF429, 880, 284}, {0x80444B5E7AA7CF85, 907, 292},
    {0xBF21E44003ACDD2D, 933, 300}, {0x8E679C2F5E44FF8F, 960, 308}, {0xD433179D9C8CB841, 986, 316},
    {0x9E19DB92B4E31BA9, 1013, 324},
};

// Digits d (ASCII, len) and decimal exponent with v = d * 10^dec, v > 0 finite.
void grisu2(double value, char* buf, int& len, int& dec) {
  std::uint64_t bits;
  std::memcpy(&bits, &value, sizeof bits);
  const std::uint64_t E = bits >> 52, F = bits & ((std::uint64_t{1} << 52) - 1);
  const Fp v = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (std::uint64_t{1} << 52), static_cast<int>(E) - 1075};
  const bool closer = F == 0 && E > 1;
  const Fp m_plus = fp_normalize({2 * v.f + 1, v.e - 1});
  Fp m_minus = closer ? Fp{4 * v.f - 1, v.e - 2} : Fp{2 * v.f - 1, v.e - 1};
  m_minus = {m_minus.f << (m_minus.e - m_plus.e), m_plus.e};
  const Fp w0 = fp_normalize(v);
  // cached power with alpha = -60 <= e_c + e + 64 <= gamma = -32
  const int fk = -60 - m_plus.e - 1;
  const int k = (fk * 78913) / (1 << 18) + (fk > 0 ? 1 : 0);
  const CachedPower c = kCachedPowers[(300 + k + 7) / 8];
  const Fp cp{c.f, c.e};
  const Fp w = fp_mul(w0, cp), wm = fp_mul(m_minus, cp), wp = fp_mul(m_plus, cp);
  const Fp Mm{wm.f + 1, wm.e}, Mp{wp.f - 1, wp.e};
  dec = -c.k;
  std::uint64_t delta = Mp.f - Mm.f, dist = Mp.f - w.f;
  const int sh = -Mp.e;
  const std::uint64_t one = std::uint64_t{1} << sh;
  std::uint32_t p1 = static_cast<std::uint32_t>(Mp.f >> sh);
  std::uint64_t p2 = Mp.f & (one - 1);
  std::uint32_t pow10 = 1;
  int n = 1;
  for (std::uint32_t t = 1000000000, d = 10; t >= 10; t /= 10, --d)
    if (p1 >= t) {
      pow10 = t;
      n = static_cast<int>(d);
      break;
    }
  len = 0;
  auto round_step = [&](std::uint64_t rest, std::uint64_t ten_k) {
    while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
      --buf[len - 1];
      rest += ten_k;
    }
  };
  while (n > 0) {
    const std::uint32_t d = p1 / pow10, r = p1 % pow10;
    buf[len++] = static_cast<char>('0' + d);
    p1 = r;
    --n;
    const std::uint64_t rest = (std::uint64_t{p1} << sh) + p2;
    if (rest <= delta) {
      dec += n;
      round_step(rest, std::uint64_t{pow10} << sh);
      return;
    }
    pow10 /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    const std::uint64_t d = p2 >> sh, r = p2 & (one - 1);
    buf[len++] = static_cast<char>('0' + d);
    p2 = r;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  dec -= m;
  round_step(p2, one);
}

}  // namespace

std::string format_json_double(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  const bool neg = std::signbit(v);
  char buf[32];
  int len = 0, dec = 0;
  grisu2(std::fabs(v), buf, len, dec);
  const std::string digits(buf, len);
  const int k = len;
  const int n = len + dec;  // value = 0.d1..dk x 10^n
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
