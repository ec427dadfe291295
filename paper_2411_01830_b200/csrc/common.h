// Shared helpers for the decision side of libfaastube: error plumbing,
// CPython-compatible float arithmetic (so results are bit-identical to the
// reference simulator), an insertion-ordered map (Python dict order), and a
// small JSON reader/writer for topology documents and state dumps.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "../../include/faastube.h"

namespace ft {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
void set_last_error(const std::string& msg);
const char* g_last_error_cstr();

// ------------------------------------------------ CPython float semantics
// sum() over floats in CPython >= 3.12 (Neumaier compensation,
// Python/bltinmodule.c builtin_sum_impl): start is int 0, so the first float
// item becomes the running value exactly (0 + x), later items are
// compensated, and the compensation is added once at the end.
struct PySum {
  double f = 0.0, c = 0.0;
  bool any = false;
  void add(double x) {
    if (!any) {
      f = 0.0 + x;
      any = true;
      return;
    }
    double t = f + x;
    if (std::fabs(f) >= std::fabs(x))
      c += (f - t) + x;
    else
      c += (x - t) + f;
    f = t;
  }
  double value() const {
    if (!any) return 0.0;
    double r = f;
    if (c != 0.0 && std::isfinite(c)) r += c;
    return r;
  }
};
template <class It, class F>
double py_sum(It b, It e, F get) {
  PySum s;
  for (; b != e; ++b) s.add(get(*b));
  return s.value();
}

// float.__floordiv__ (Objects/floatobject.c _float_div_mod)
inline double py_floordiv(double vx, double wx) {
  double mod = std::fmod(vx, wx);
  double div = (vx - mod) / wx;
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) {
      mod += wx;
      div -= 1.0;
    }
  }
  double floordiv;
  if (div != 0.0) {
    floordiv = std::floor(div);
    if (div - floordiv > 0.5) floordiv += 1.0;
  } else {
    floordiv = std::copysign(0.0, vx / wx);
  }
  return floordiv;
}

// math.ceil on a float, returned as an integer-valued double / int64
inline int64_t py_ceil(double x) { return (int64_t)std::ceil(x); }

inline double none() { return std::nan(""); }
inline bool is_none(double x) { return std::isnan(x); }

// ------------------------------------------------------- ordered dict
template <class V>
struct ODict {
  std::vector<std::pair<std::string, V>> items;
  std::unordered_map<std::string, size_t> pos;
  V* find(const std::string& k) {
    auto it = pos.find(k);
    return it == pos.end() ? nullptr : &items[it->second].second;
  }
  const V* find(const std::string& k) const {
    auto it = pos.find(k);
    return it == pos.end() ? nullptr : &items[it->second].second;
  }
  V& set(const std::string& k, V v) {  // dict[k] = v (keeps position of existing key)
    auto it = pos.find(k);
    if (it != pos.end()) {
      items[it->second].second = std::move(v);
      return items[it->second].second;
    }
    pos[k] = items.size();
    items.emplace_back(k, std::move(v));
    return items.back().second;
  }
  bool erase(const std::string& k) {  // dict.pop(k, None)
    auto it = pos.find(k);
    if (it == pos.end()) return false;
    size_t i = it->second;
    items.erase(items.begin() + i);
    pos.erase(it);
    for (auto& p : pos)
      if (p.second > i) --p.second;
    return true;
  }
  size_t size() const { return items.size(); }
  bool empty() const { return items.empty(); }
};

// --------------------------------------------------------- JSON writer
struct JsonOut {
  std::string s;
  void num(double x) {
    if (std::isnan(x)) {
      s += "null";
      return;
    }
    if (std::isinf(x)) {
      s += x > 0 ? "1e999" : "-1e999";
      return;
    }
    char b[40];
    snprintf(b, sizeof b, "%.17g", x);
    s += b;
  }
  void inum(int64_t x) { s += std::to_string(x); }
  void str(const std::string& x) {
    s += '"';
    for (char c : x) {
      if (c == '"' || c == '\\') s += '\\';
      s += c;
    }
    s += '"';
  }
  void raw(const char* x) { s += x; }
};
int emit_json(const std::string& s, char* buf, size_t cap, size_t* need);

// ---------------------------------------------------------- JSON reader
struct JVal {
  enum T { NUL, BOOL, NUM, STR, ARR, OBJ } t = NUL;
  bool b = false;
  double n = 0;
  bool is_int = false;
  std::string s;
  std::vector<JVal> a;
  std::vector<std::pair<std::string, JVal>> o;
  const JVal* get(const std::string& k) const {
    for (auto& kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};
JVal json_parse(const std::string& text);

}  // namespace ft
