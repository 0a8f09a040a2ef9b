// Minimal JSON values with the reference's exact text conventions:
// `json.dumps(..., sort_keys=True)` output (", " / ": " separators, keys in
// code-point order, ensure_ascii escaping, Python float repr), and a parser
// for the documents the reference writes (`src/ir.py:708-715`,
// `src/trace.py:80-86`).  Host-side only (trace replay, src/trace.py).
#pragma once

#include <cstdint>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace lsb {
namespace pj {

struct Value {
  enum Type : uint8_t { Null, Bool, Int, Float, Str, Arr, Obj } t = Null;
  bool b = false;
  int64_t i = 0;
  bool big = false;   // integer outside int64: kept verbatim in `s`
  double d = 0;
  std::string s;      // Str payload (UTF-8), or the digits of a big Int
  std::vector<Value> a;
  std::vector<std::pair<std::string, Value>> o;  // insertion order

  const Value* get(std::string_view k) const {
    for (const auto& kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  static Value integer(int64_t v) { Value x; x.t = Int; x.i = v; return x; }
  static Value real(double v) { Value x; x.t = Float; x.d = v; return x; }
  static Value str(std::string v) { Value x; x.t = Str; x.s = std::move(v); return x; }
  static Value arr() { Value x; x.t = Arr; return x; }
  static Value obj() { Value x; x.t = Obj; return x; }
  void put(std::string k, Value v) { o.emplace_back(std::move(k), std::move(v)); }
};

// Parses one JSON document (Python's json.loads grammar incl. NaN/Infinity);
// false on malformed input.
bool parse(std::string_view text, Value* out);

// json.dumps(v, sort_keys=True)
void dump(const Value& v, std::string* out);
std::string dumps(const Value& v);

// Python's repr(float) (shortest round-trip digits, fixed vs exponent rule).
void float_repr(double x, std::string* out);
// json.dumps of a str (ensure_ascii=True)
void dump_string(std::string_view s, std::string* out);
// Python repr() of a str (single-quoted; the identifiers of a program)
std::string py_repr(std::string_view s);

}  // namespace pj
}  // namespace lsb
