// Minimal JSON DOM for the host boundary: hand specs (reference
// proj/src/hand.cpp:259-363) and run configs (proj/src/config.cpp:139-194).
// The reference uses nlohmann/json 3.11 (not shipped, proj/.gitignore:2);
// numbers here are parsed with strtod, which is correctly rounded like
// nlohmann's parser, so every double in a spec reaches the model unchanged.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace grasp::json {

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct TypeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Value {
 public:
  enum class Kind { Null, Bool, Number, String, Array, Object };

  Value() = default;
  static Value make_null() { return Value(); }
  static Value make_bool(bool b) { Value v; v.kind_ = Kind::Bool; v.b_ = b; return v; }
  static Value make_number(double d, bool is_int, std::int64_t i) {
    Value v; v.kind_ = Kind::Number; v.d_ = d; v.is_int_ = is_int; v.i_ = i; return v;
  }
  static Value make_string(std::string s) { Value v; v.kind_ = Kind::String; v.s_ = std::move(s); return v; }
  static Value make_array() { Value v; v.kind_ = Kind::Array; return v; }
  static Value make_object() { Value v; v.kind_ = Kind::Object; return v; }

  Kind kind() const { return kind_; }
  bool is_object() const { return kind_ == Kind::Object; }
  bool is_array() const { return kind_ == Kind::Array; }
  bool is_number() const { return kind_ == Kind::Number; }
  bool is_string() const { return kind_ == Kind::String; }
  bool is_bool() const { return kind_ == Kind::Bool; }
  bool is_null() const { return kind_ == Kind::Null; }

  double as_double() const;
  std::int64_t as_int() const;
  std::uint64_t as_uint64() const;
  bool as_bool() const;
  const std::string& as_string() const;

  // Arrays
  std::size_t size() const;
  bool empty() const { return size() == 0; }
  const Value& at(std::size_t i) const;
  void push_back(Value v) { arr_.push_back(std::move(v)); }
  const std::vector<Value>& items() const { return arr_; }

  // Objects (insertion order kept; duplicate keys: last wins like nlohmann)
  bool contains(const std::string& key) const { return find(key) != nullptr; }
  const Value* find(const std::string& key) const;
  const Value& at(const std::string& key) const;
  void set(const std::string& key, Value v);
  const std::vector<std::pair<std::string, Value>>& members() const { return obj_; }

 private:
  Kind kind_ = Kind::Null;
  bool b_ = false;
  double d_ = 0.0;
  bool is_int_ = false;
  std::int64_t i_ = 0;
  std::uint64_t u_ = 0;
  bool is_uint_ = false;
  std::string s_;
  std::vector<Value> arr_;
  std::vector<std::pair<std::string, Value>> obj_;
  friend Value parse(const std::string&);
  friend class Parser;
};

Value parse(const std::string& text);

/// Shortest round-trip decimal for a double (std::to_chars), JSON style:
/// integral values keep a ".0" suffix like nlohmann's serializer.
std::string format_double(double v);

}  // namespace grasp::json
