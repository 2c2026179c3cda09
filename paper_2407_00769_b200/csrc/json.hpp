// Minimal JSON reader for the plan format (objects, arrays, numbers, strings, true/false/null).
// Numbers are parsed with strtod (exact round trip of the shortest-repr doubles Python writes).
#pragma once
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace tnjson {

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Value {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;

  const Value* get(const char* key) const {
    if (kind != Obj) return nullptr;
    for (auto& kv : obj)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
  bool is_arr() const { return kind == Arr; }
  bool is_num() const { return kind == Num; }
  bool is_obj() const { return kind == Obj; }
};

class Parser {
 public:
  Parser(const char* s, size_t n) : p_(s), end_(s + n) {}
  Value parse() {
    Value v = value();
    ws();
    if (p_ != end_) fail("trailing characters");
    return v;
  }

 private:
  const char* p_;
  const char* end_;
  int depth_ = 0;

  [[noreturn]] void fail(const char* what) {
    throw ParseError(std::string("json: ") + what);
  }
  void ws() {
    while (p_ < end_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\t' || *p_ == '\r')) ++p_;
  }
  Value value() {
    ws();
    if (p_ >= end_) fail("unexpected end");
    char c = *p_;
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') {
      Value v;
      v.kind = Value::Str;
      v.str = string();
      return v;
    }
    if (c == 't' || c == 'f' || c == 'n') return literal();
    return number();
  }
  Value literal() {
    Value v;
    auto match = [&](const char* w) {
      size_t n = strlen(w);
      if ((size_t)(end_ - p_) >= n && memcmp(p_, w, n) == 0) {
        p_ += n;
        return true;
      }
      return false;
    };
    if (match("true")) { v.kind = Value::Bool; v.b = true; return v; }
    if (match("false")) { v.kind = Value::Bool; v.b = false; return v; }
    if (match("null")) { v.kind = Value::Null; return v; }
    fail("bad literal");
  }
  Value number() {
    char buf[64];
    size_t n = 0;
    while (p_ < end_ && n < sizeof(buf) - 1 &&
           (isdigit((unsigned char)*p_) || *p_ == '-' || *p_ == '+' || *p_ == '.' || *p_ == 'e' ||
            *p_ == 'E' || *p_ == 'I' || *p_ == 'n' || *p_ == 'f' || *p_ == 'i' || *p_ == 't' ||
            *p_ == 'y' || *p_ == 'N' || *p_ == 'a'))
      buf[n++] = *p_++;
    buf[n] = 0;
    if (n == 0) fail("bad value");
    char* e = nullptr;
    double d = strtod(buf, &e);
    if (e != buf + n) fail("bad number");
    Value v;
    v.kind = Value::Num;
    v.num = d;
    return v;
  }
  std::string string() {
    ++p_;  // opening quote
    std::string s;
    while (p_ < end_ && *p_ != '"') {
      if (*p_ == '\\') {
        ++p_;
        if (p_ >= end_) fail("bad escape");
        char c = *p_++;
        switch (c) {
          case 'n': s += '\n'; break;
          case 't': s += '\t'; break;
          case 'r': s += '\r'; break;
          case 'b': s += '\b'; break;
          case 'f': s += '\f'; break;
          case 'u': {
            if (end_ - p_ < 4) fail("bad \\u escape");
            p_ += 4;  // plan strings are ASCII; non-ASCII code points are replaced
            s += '?';
            break;
          }
          default: s += c;
        }
      } else {
        s += *p_++;
      }
    }
    if (p_ >= end_) fail("unterminated string");
    ++p_;
    return s;
  }
  Value array() {
    if (++depth_ > 256) fail("nesting too deep");
    ++p_;
    Value v;
    v.kind = Value::Arr;
    ws();
    if (p_ < end_ && *p_ == ']') {
      ++p_;
      --depth_;
      return v;
    }
    for (;;) {
      v.arr.push_back(value());
      ws();
      if (p_ >= end_) fail("unterminated array");
      if (*p_ == ',') { ++p_; continue; }
      if (*p_ == ']') { ++p_; break; }
      fail("expected , or ]");
    }
    --depth_;
    return v;
  }
  Value object() {
    if (++depth_ > 256) fail("nesting too deep");
    ++p_;
    Value v;
    v.kind = Value::Obj;
    ws();
    if (p_ < end_ && *p_ == '}') {
      ++p_;
      --depth_;
      return v;
    }
    for (;;) {
      ws();
      if (p_ >= end_ || *p_ != '"') fail("expected key");
      std::string k = string();
      ws();
      if (p_ >= end_ || *p_ != ':') fail("expected :");
      ++p_;
      v.obj.emplace_back(std::move(k), value());
      ws();
      if (p_ >= end_) fail("unterminated object");
      if (*p_ == ',') { ++p_; continue; }
      if (*p_ == '}') { ++p_; break; }
      fail("expected , or }");
    }
    --depth_;
    return v;
  }
};

inline Value parse(const char* s, size_t n) { return Parser(s, n).parse(); }

}  // namespace tnjson
