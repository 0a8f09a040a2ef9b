// See pyjson.hpp.
#include "pyjson.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace lsb {
namespace pj {

namespace {

struct Parser {
  std::string_view t;
  size_t p = 0;
  bool ok = true;

  void ws() {
    while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\r' || t[p] == '\t')) ++p;
  }
  bool lit(const char* w) {
    size_t n = std::strlen(w);
    if (t.substr(p, n) == w) {
      p += n;
      return true;
    }
    return false;
  }
  static void put_utf8(uint32_t cp, std::string* s) {
    if (cp < 0x80) {
      s->push_back(static_cast<char>(cp));
    } else if (cp < 0x800) {
      s->push_back(static_cast<char>(0xC0 | (cp >> 6)));
      s->push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else if (cp < 0x10000) {
      s->push_back(static_cast<char>(0xE0 | (cp >> 12)));
      s->push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      s->push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else {
      s->push_back(static_cast<char>(0xF0 | (cp >> 18)));
      s->push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
      s->push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      s->push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    }
  }
  bool hex4(uint32_t* v) {
    if (p + 4 > t.size()) return false;
    uint32_t x = 0;
    for (int k = 0; k < 4; ++k) {
      char c = t[p + k];
      x <<= 4;
      if (c >= '0' && c <= '9') x |= static_cast<uint32_t>(c - '0');
      else if (c >= 'a' && c <= 'f') x |= static_cast<uint32_t>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') x |= static_cast<uint32_t>(c - 'A' + 10);
      else return false;
    }
    p += 4;
    *v = x;
    return true;
  }
  bool string(std::string* out) {
    if (p >= t.size() || t[p] != '"') return false;
    ++p;
    while (p < t.size()) {
      char c = t[p++];
      if (c == '"') return true;
      if (c != '\\') {
        out->push_back(c);
        continue;
      }
      if (p >= t.size()) return false;
      char e = t[p++];
      switch (e) {
        case '"': out->push_back('"'); break;
        case '\\': out->push_back('\\'); break;
        case '/': out->push_back('/'); break;
        case 'b': out->push_back('\b'); break;
        case 'f': out->push_back('\f'); break;
        case 'n': out->push_back('\n'); break;
        case 'r': out->push_back('\r'); break;
        case 't': out->push_back('\t'); break;
        case 'u': {
          uint32_t cp;
          if (!hex4(&cp)) return false;
          if (cp >= 0xD800 && cp < 0xDC00 && p + 6 <= t.size() && t[p] == '\\' && t[p + 1] == 'u') {
            size_t save = p;
            p += 2;
            uint32_t lo;
            if (hex4(&lo) && lo >= 0xDC00 && lo < 0xE000) cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            else p = save;
          }
          put_utf8(cp, out);
          break;
        }
        default: return false;
      }
    }
    return false;
  }
  bool number(Value* v) {
    size_t s = p;
    if (lit("-Infinity")) {
      v->t = Value::Float;
      v->d = -INFINITY;
      return true;
    }
    if (p < t.size() && t[p] == '-') ++p;
    size_t digits0 = p;
    while (p < t.size() && t[p] >= '0' && t[p] <= '9') ++p;
    if (p == digits0) return false;
    bool flt = false;
    if (p < t.size() && t[p] == '.') {
      flt = true;
      ++p;
      while (p < t.size() && t[p] >= '0' && t[p] <= '9') ++p;
    }
    if (p < t.size() && (t[p] == 'e' || t[p] == 'E')) {
      flt = true;
      ++p;
      if (p < t.size() && (t[p] == '+' || t[p] == '-')) ++p;
      while (p < t.size() && t[p] >= '0' && t[p] <= '9') ++p;
    }
    std::string tok(t.substr(s, p - s));
    if (flt) {
      v->t = Value::Float;
      v->d = std::strtod(tok.c_str(), nullptr);
      return true;
    }
    v->t = Value::Int;
    errno = 0;
    char* end = nullptr;
    long long x = std::strtoll(tok.c_str(), &end, 10);
    if (errno == ERANGE) {
      v->big = true;
      v->s = tok;
    } else {
      v->i = x;
    }
    return true;
  }
  bool value(Value* v, int depth) {
    if (depth > 256) return false;
    ws();
    if (p >= t.size()) return false;
    char c = t[p];
    if (c == '{') {
      ++p;
      v->t = Value::Obj;
      ws();
      if (p < t.size() && t[p] == '}') {
        ++p;
        return true;
      }
      for (;;) {
        ws();
        std::string k;
        if (!string(&k)) return false;
        ws();
        if (p >= t.size() || t[p] != ':') return false;
        ++p;
        Value x;
        if (!value(&x, depth + 1)) return false;
        // json.loads keeps the last of duplicate keys
        bool dup = false;
        for (auto& kv : v->o)
          if (kv.first == k) {
            kv.second = std::move(x);
            dup = true;
            break;
          }
        if (!dup) v->o.emplace_back(std::move(k), std::move(x));
        ws();
        if (p < t.size() && t[p] == ',') {
          ++p;
          continue;
        }
        if (p < t.size() && t[p] == '}') {
          ++p;
          return true;
        }
        return false;
      }
    }
    if (c == '[') {
      ++p;
      v->t = Value::Arr;
      ws();
      if (p < t.size() && t[p] == ']') {
        ++p;
        return true;
      }
      for (;;) {
        Value x;
        if (!value(&x, depth + 1)) return false;
        v->a.push_back(std::move(x));
        ws();
        if (p < t.size() && t[p] == ',') {
          ++p;
          continue;
        }
        if (p < t.size() && t[p] == ']') {
          ++p;
          return true;
        }
        return false;
      }
    }
    if (c == '"') {
      v->t = Value::Str;
      return string(&v->s);
    }
    if (lit("true")) {
      v->t = Value::Bool;
      v->b = true;
      return true;
    }
    if (lit("false")) {
      v->t = Value::Bool;
      v->b = false;
      return true;
    }
    if (lit("null")) {
      v->t = Value::Null;
      return true;
    }
    if (lit("NaN")) {
      v->t = Value::Float;
      v->d = NAN;
      return true;
    }
    if (lit("Infinity")) {
      v->t = Value::Float;
      v->d = INFINITY;
      return true;
    }
    return number(v);
  }
};

// decode one UTF-8 code point at s[i] (invalid bytes map to themselves)
uint32_t next_cp(std::string_view s, size_t* i) {
  unsigned char c = static_cast<unsigned char>(s[*i]);
  int n = c < 0x80 ? 0 : (c >> 5) == 6 ? 1 : (c >> 4) == 14 ? 2 : (c >> 3) == 30 ? 3 : 0;
  uint32_t cp = n == 0 ? c : n == 1 ? (c & 0x1F) : n == 2 ? (c & 0x0F) : (c & 0x07);
  if (*i + n >= s.size() + (n ? 0 : 1)) n = 0;
  for (int k = 1; k <= n; ++k) cp = (cp << 6) | (static_cast<unsigned char>(s[*i + k]) & 0x3F);
  *i += static_cast<size_t>(n) + 1;
  return cp;
}

}  // namespace

bool parse(std::string_view text, Value* out) {
  Parser ps{text};
  *out = Value();
  if (!ps.value(out, 0)) return false;
  ps.ws();
  return ps.p == text.size();
}

void dump_string(std::string_view s, std::string* out) {
  static const char* hex = "0123456789abcdef";
  out->push_back('"');
  size_t i = 0;
  while (i < s.size()) {
    uint32_t cp = next_cp(s, &i);
    switch (cp) {
      case '"': out->append("\\\""); continue;
      case '\\': out->append("\\\\"); continue;
      case '\n': out->append("\\n"); continue;
      case '\r': out->append("\\r"); continue;
      case '\t': out->append("\\t"); continue;
      case '\b': out->append("\\b"); continue;
      case '\f': out->append("\\f"); continue;
      default: break;
    }
    if (cp >= 0x20 && cp < 0x7F) {
      out->push_back(static_cast<char>(cp));
      continue;
    }
    auto u4 = [&](uint32_t u) {
      out->append("\\u");
      for (int k = 3; k >= 0; --k) out->push_back(hex[(u >> (4 * k)) & 0xF]);
    };
    if (cp >= 0x10000) {
      cp -= 0x10000;
      u4(0xD800 | (cp >> 10));
      u4(0xDC00 | (cp & 0x3FF));
    } else {
      u4(cp);
    }
  }
  out->push_back('"');
}

void float_repr(double x, std::string* out) {
  if (std::isnan(x)) {
    out->append("NaN");
    return;
  }
  if (std::isinf(x)) {
    out->append(x > 0 ? "Infinity" : "-Infinity");
    return;
  }
  if (x == 0) {
    out->append(std::signbit(x) ? "-0.0" : "0.0");
    return;
  }
  // shortest correctly rounded digit string that reads back to x
  char buf[64];
  std::string digits;
  int exp10 = 0;
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*e", prec - 1, x);
    if (std::strtod(buf, nullptr) == x || prec == 17) {
      const char* q = buf;
      if (*q == '-') ++q;
      digits.clear();
      for (; *q && *q != 'e'; ++q)
        if (*q != '.') digits.push_back(*q);
      exp10 = std::atoi(q + 1);
      break;
    }
  }
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  if (x < 0) out->push_back('-');
  const int decpt = exp10 + 1;  // x = 0.DIGITS * 10^decpt
  const int nd = static_cast<int>(digits.size());
  if (decpt <= -4 || decpt > 16) {
    out->push_back(digits[0]);
    if (nd > 1) {
      out->push_back('.');
      out->append(digits, 1, std::string::npos);
    }
    int e = decpt - 1;
    std::snprintf(buf, sizeof buf, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    out->append(buf);
  } else if (decpt <= 0) {
    out->append("0.");
    out->append(static_cast<size_t>(-decpt), '0');
    out->append(digits);
  } else if (decpt >= nd) {
    out->append(digits);
    out->append(static_cast<size_t>(decpt - nd), '0');
    out->append(".0");
  } else {
    out->append(digits, 0, static_cast<size_t>(decpt));
    out->push_back('.');
    out->append(digits, static_cast<size_t>(decpt), std::string::npos);
  }
}

void dump(const Value& v, std::string* out) {
  switch (v.t) {
    case Value::Null: out->append("null"); return;
    case Value::Bool: out->append(v.b ? "true" : "false"); return;
    case Value::Int:
      if (v.big) out->append(v.s);
      else out->append(std::to_string(v.i));
      return;
    case Value::Float: float_repr(v.d, out); return;
    case Value::Str: dump_string(v.s, out); return;
    case Value::Arr:
      out->push_back('[');
      for (size_t k = 0; k < v.a.size(); ++k) {
        if (k) out->append(", ");
        dump(v.a[k], out);
      }
      out->push_back(']');
      return;
    case Value::Obj: {
      std::vector<const std::pair<std::string, Value>*> kv;
      kv.reserve(v.o.size());
      for (const auto& x : v.o) kv.push_back(&x);
      std::sort(kv.begin(), kv.end(), [](auto* a, auto* b) { return a->first < b->first; });
      out->push_back('{');
      for (size_t k = 0; k < kv.size(); ++k) {
        if (k) out->append(", ");
        dump_string(kv[k]->first, out);
        out->append(": ");
        dump(kv[k]->second, out);
      }
      out->push_back('}');
      return;
    }
  }
}

std::string dumps(const Value& v) {
  std::string s;
  dump(v, &s);
  return s;
}

std::string py_repr(std::string_view s) {
  const bool dq = s.find('\'') != std::string_view::npos && s.find('"') == std::string_view::npos;
  const char q = dq ? '"' : '\'';
  std::string out(1, q);
  for (char c : s) {
    if (c == '\\') out.append("\\\\");
    else if (c == q) { out.push_back('\\'); out.push_back(c); }
    else if (c == '\n') out.append("\\n");
    else if (c == '\t') out.append("\\t");
    else if (c == '\r') out.append("\\r");
    else out.push_back(c);
  }
  out.push_back(q);
  return out;
}

}  // namespace pj
}  // namespace lsb
