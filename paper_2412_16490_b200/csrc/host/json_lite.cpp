#include "json_lite.hpp"

#include <cctype>
#include <cerrno>
#include <charconv>
#include <locale.h>
#include <stdlib.h>
#include <cmath>
#include <cstdlib>
#include <cstring>

namespace grasp::json {

double Value::as_double() const {
  if (kind_ != Kind::Number) throw TypeError("json: value is not a number");
  return d_;
}

std::int64_t Value::as_int() const {
  if (kind_ != Kind::Number) throw TypeError("json: value is not a number");
  if (is_int_) return i_;
  if (is_uint_) throw TypeError("json: integer out of range");
  // nlohmann get<int> on a float truncates; keep that behaviour.
  return static_cast<std::int64_t>(d_);
}

std::uint64_t Value::as_uint64() const {
  if (kind_ != Kind::Number) throw TypeError("json: value is not a number");
  if (is_uint_) return u_;
  if (is_int_) return static_cast<std::uint64_t>(i_);
  return static_cast<std::uint64_t>(d_);
}

bool Value::as_bool() const {
  if (kind_ != Kind::Bool) throw TypeError("json: value is not a boolean");
  return b_;
}

const std::string& Value::as_string() const {
  if (kind_ != Kind::String) throw TypeError("json: value is not a string");
  return s_;
}

std::size_t Value::size() const {
  if (kind_ == Kind::Array) return arr_.size();
  if (kind_ == Kind::Object) return obj_.size();
  if (kind_ == Kind::Null) return 0;
  return 1;
}

const Value& Value::at(std::size_t i) const {
  if (kind_ != Kind::Array) throw TypeError("json: value is not an array");
  if (i >= arr_.size()) throw TypeError("json: array index out of range");
  return arr_[i];
}

const Value* Value::find(const std::string& key) const {
  if (kind_ != Kind::Object) return nullptr;
  for (auto it = obj_.rbegin(); it != obj_.rend(); ++it)
    if (it->first == key) return &it->second;
  return nullptr;
}

const Value& Value::at(const std::string& key) const {
  if (kind_ != Kind::Object) throw TypeError("json: value is not an object");
  const Value* v = find(key);
  if (!v) throw TypeError("json: key '" + key + "' not found");
  return *v;
}

void Value::set(const std::string& key, Value v) {
  if (kind_ == Kind::Null) kind_ = Kind::Object;
  for (auto& kv : obj_)
    if (kv.first == key) { kv.second = std::move(v); return; }
  obj_.emplace_back(key, std::move(v));
}

class Parser {
 public:
  explicit Parser(const std::string& t) : s_(t) {}

  Value run() {
    skip_ws();
    Value v = value(0);
    skip_ws();
    if (pos_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const char* what) const {
    throw ParseError(std::string("json parse error at byte ") + std::to_string(pos_) + ": " + what);
  }
  void skip_ws() {
    while (pos_ < s_.size() && (s_[pos_] == ' ' || s_[pos_] == '\t' || s_[pos_] == '\n' || s_[pos_] == '\r'))
      ++pos_;
  }
  bool eat(char c) {
    if (pos_ < s_.size() && s_[pos_] == c) { ++pos_; return true; }
    return false;
  }
  void expect_word(const char* w) {
    const std::size_t n = std::strlen(w);
    if (s_.compare(pos_, n, w) != 0) fail("invalid literal");
    pos_ += n;
  }

  Value value(int depth) {
    if (depth > 256) fail("nesting too deep");
    if (pos_ >= s_.size()) fail("unexpected end of input");
    const char c = s_[pos_];
    if (c == '{') return object(depth);
    if (c == '[') return array(depth);
    if (c == '"') return Value::make_string(string());
    if (c == 't') { expect_word("true"); return Value::make_bool(true); }
    if (c == 'f') { expect_word("false"); return Value::make_bool(false); }
    if (c == 'n') { expect_word("null"); return Value::make_null(); }
    return number();
  }

  Value object(int depth) {
    ++pos_;
    Value v = Value::make_object();
    skip_ws();
    if (eat('}')) return v;
    for (;;) {
      skip_ws();
      if (pos_ >= s_.size() || s_[pos_] != '"') fail("expected object key");
      std::string key = string();
      skip_ws();
      if (!eat(':')) fail("expected ':'");
      skip_ws();
      v.set(key, value(depth + 1));
      skip_ws();
      if (eat(',')) continue;
      if (eat('}')) return v;
      fail("expected ',' or '}'");
    }
  }

  Value array(int depth) {
    ++pos_;
    Value v = Value::make_array();
    skip_ws();
    if (eat(']')) return v;
    for (;;) {
      skip_ws();
      v.push_back(value(depth + 1));
      skip_ws();
      if (eat(',')) continue;
      if (eat(']')) return v;
      fail("expected ',' or ']'");
    }
  }

  static void put_utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) out += static_cast<char>(cp);
    else if (cp < 0x800) { out += static_cast<char>(0xC0 | (cp >> 6)); out += static_cast<char>(0x80 | (cp & 0x3F)); }
    else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }

  unsigned hex4() {
    if (pos_ + 4 > s_.size()) fail("truncated \\u escape");
    unsigned v = 0;
    for (int k = 0; k < 4; ++k) {
      const char h = s_[pos_++];
      v <<= 4;
      if (h >= '0' && h <= '9') v |= static_cast<unsigned>(h - '0');
      else if (h >= 'a' && h <= 'f') v |= static_cast<unsigned>(h - 'a' + 10);
      else if (h >= 'A' && h <= 'F') v |= static_cast<unsigned>(h - 'A' + 10);
      else fail("bad \\u escape");
    }
    return v;
  }

  std::string string() {
    ++pos_;  // opening quote
    std::string out;
    for (;;) {
      if (pos_ >= s_.size()) fail("unterminated string");
      const char c = s_[pos_++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') { out += c; continue; }
      if (pos_ >= s_.size()) fail("unterminated escape");
      const char e = s_[pos_++];
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (!(eat('\\') && eat('u'))) fail("unpaired surrogate");
            const unsigned lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("bad surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          put_utf8(out, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
  }

  Value number() {
    const std::size_t start = pos_;
    if (eat('-')) {}
    if (pos_ >= s_.size()) fail("bad number");
    if (s_[pos_] == '0') ++pos_;
    else if (s_[pos_] >= '1' && s_[pos_] <= '9') while (pos_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[pos_]))) ++pos_;
    else fail("bad number");
    bool integral = true;
    if (eat('.')) {
      integral = false;
      if (pos_ >= s_.size() || !std::isdigit(static_cast<unsigned char>(s_[pos_]))) fail("bad fraction");
      while (pos_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[pos_]))) ++pos_;
    }
    if (pos_ < s_.size() && (s_[pos_] == 'e' || s_[pos_] == 'E')) {
      integral = false;
      ++pos_;
      if (pos_ < s_.size() && (s_[pos_] == '+' || s_[pos_] == '-')) ++pos_;
      if (pos_ >= s_.size() || !std::isdigit(static_cast<unsigned char>(s_[pos_]))) fail("bad exponent");
      while (pos_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[pos_]))) ++pos_;
    }
    const std::string tok = s_.substr(start, pos_ - start);
    // Locale-free and correctly rounded (like nlohmann's lexer, whatever
    // LC_NUMERIC the host application set); out-of-range magnitudes saturate
    // like strtod in the "C" locale.
    double d = 0.0;
    const auto fr = std::from_chars(tok.data(), tok.data() + tok.size(), d);
    if (fr.ec == std::errc::result_out_of_range) {
      static const locale_t c_locale = newlocale(LC_ALL_MASK, "C", static_cast<locale_t>(0));
      d = strtod_l(tok.c_str(), nullptr, c_locale);
    } else if (fr.ec != std::errc()) {
      fail("bad number");
    }
    Value v = Value::make_number(d, false, 0);
    if (integral) {
      std::int64_t i = 0;
      auto r = std::from_chars(tok.data(), tok.data() + tok.size(), i);
      if (r.ec == std::errc()) {
        v.is_int_ = true;
        v.i_ = i;
      } else {
        std::uint64_t u = 0;
        auto r2 = std::from_chars(tok.data(), tok.data() + tok.size(), u);
        if (r2.ec == std::errc()) { v.is_uint_ = true; v.u_ = u; }
      }
    }
    return v;
  }

  const std::string& s_;
  std::size_t pos_ = 0;
};

Value parse(const std::string& text) { return Parser(text).run(); }

std::string format_double(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

}  // namespace grasp::json
