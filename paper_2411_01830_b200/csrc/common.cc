#include "common.h"

#include <cctype>
#include <cstdlib>

namespace ft {

static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* g_last_error_cstr() { return g_last_error.c_str(); }

int emit_json(const std::string& s, char* buf, size_t cap, size_t* need) {
  if (need) *need = s.size() + 1;
  if (!buf || cap < s.size() + 1) {
    set_last_error("json output buffer too small");
    return FT_E_TRUNCATED;
  }
  memcpy(buf, s.data(), s.size());
  buf[s.size()] = 0;
  return FT_OK;
}

namespace {
struct Parser {
  const std::string& t;
  size_t i = 0;
  explicit Parser(const std::string& s) : t(s) {}
  void ws() {
    while (i < t.size() && isspace((unsigned char)t[i])) ++i;
  }
  [[noreturn]] void bad(const char* what) {
    fail(FT_E_TOPOLOGY, std::string("malformed topology document: json ") + what + " at offset " +
                            std::to_string(i));
  }
  JVal value() {
    ws();
    if (i >= t.size()) bad("unexpected end");
    char c = t[i];
    JVal v;
    if (c == '{') {
      v.t = JVal::OBJ;
      ++i;
      ws();
      if (i < t.size() && t[i] == '}') {
        ++i;
        return v;
      }
      for (;;) {
        ws();
        if (i >= t.size() || t[i] != '"') bad("expected key");
        std::string k = string();
        ws();
        if (i >= t.size() || t[i] != ':') bad("expected ':'");
        ++i;
        v.o.emplace_back(k, value());
        ws();
        if (i < t.size() && t[i] == ',') {
          ++i;
          continue;
        }
        if (i < t.size() && t[i] == '}') {
          ++i;
          return v;
        }
        bad("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.t = JVal::ARR;
      ++i;
      ws();
      if (i < t.size() && t[i] == ']') {
        ++i;
        return v;
      }
      for (;;) {
        v.a.push_back(value());
        ws();
        if (i < t.size() && t[i] == ',') {
          ++i;
          continue;
        }
        if (i < t.size() && t[i] == ']') {
          ++i;
          return v;
        }
        bad("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.t = JVal::STR;
      v.s = string();
      return v;
    }
    if (t.compare(i, 4, "true") == 0) {
      i += 4;
      v.t = JVal::BOOL;
      v.b = true;
      return v;
    }
    if (t.compare(i, 5, "false") == 0) {
      i += 5;
      v.t = JVal::BOOL;
      return v;
    }
    if (t.compare(i, 4, "null") == 0) {
      i += 4;
      return v;
    }
    size_t st = i;
    if (t[i] == '-' || t[i] == '+') ++i;
    bool frac = false;
    while (i < t.size() && (isdigit((unsigned char)t[i]) || t[i] == '.' || t[i] == 'e' || t[i] == 'E' ||
                            t[i] == '-' || t[i] == '+')) {
      if (t[i] == '.' || t[i] == 'e' || t[i] == 'E') frac = true;
      ++i;
    }
    if (i == st) bad("unexpected character");
    std::string num = t.substr(st, i - st);
    v.t = JVal::NUM;
    v.n = strtod(num.c_str(), nullptr);
    v.is_int = !frac;
    return v;
  }
  std::string string() {
    ++i;  // opening quote
    std::string out;
    while (i < t.size() && t[i] != '"') {
      if (t[i] == '\\') {
        ++i;
        if (i >= t.size()) bad("bad escape");
        char e = t[i];
        if (e == 'n') out += '\n';
        else if (e == 't') out += '\t';
        else if (e == 'u') {
          if (i + 4 >= t.size()) bad("bad \\u escape");
          unsigned cp = strtoul(t.substr(i + 1, 4).c_str(), nullptr, 16);
          if (cp < 0x80) out += (char)cp;
          else out += '?';
          i += 4;
        } else out += e;
        ++i;
        continue;
      }
      out += t[i++];
    }
    if (i >= t.size()) bad("unterminated string");
    ++i;
    return out;
  }
};
}  // namespace

JVal json_parse(const std::string& text) {
  Parser p(text);
  JVal v = p.value();
  p.ws();
  if (p.i != text.size()) p.bad("trailing data");
  return v;
}

}  // namespace ft

extern "C" const char* ft_last_error(void) { return ft::g_last_error_cstr(); }
