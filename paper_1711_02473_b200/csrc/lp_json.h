// Minimal JSON reader for the reference's serialized LoopProgram
// (scheduling.serialize_program, reference scheduling.py:465-532): objects,
// arrays, strings, numbers (incl. Python's NaN / Infinity spellings), true /
// false / null.  Numbers keep their source text so that table values and
// literals are parsed with strtod exactly once (Python writes floats with
// repr(), which round-trips, so the doubles are bit-identical to the
// reference's).
#pragma once

#include <cmath>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace sfk {
namespace json {

struct Value {
  enum Kind { NUL, BOOL, NUM, STR, ARR, OBJ } kind = NUL;
  bool b = false;
  double num = 0.0;
  std::string str;                       // STR: the string; NUM: source text
  std::vector<Value> arr;
  std::map<std::string, Value> obj;

  bool is_arr() const { return kind == ARR; }
  bool is_str() const { return kind == STR; }
  bool is_num() const { return kind == NUM; }
  const Value& at(size_t i) const {
    if (kind != ARR || i >= arr.size()) throw std::runtime_error("json: bad array access");
    return arr[i];
  }
  const Value& at(const std::string& k) const {
    auto it = obj.find(k);
    if (kind != OBJ || it == obj.end()) throw std::runtime_error("json: missing key '" + k + "'");
    return it->second;
  }
  size_t size() const { return arr.size(); }
  const std::string& s() const {
    if (kind != STR) throw std::runtime_error("json: expected string");
    return str;
  }
  double d() const {
    if (kind != NUM) throw std::runtime_error("json: expected number");
    return num;
  }
  long long i() const {
    const double v = d();
    if (v != std::floor(v)) throw std::runtime_error("json: expected integer");
    return (long long)v;
  }
};

class Parser {
 public:
  Parser(const char* p, size_t n) : p_(p), end_(p + n) {}

  Value parse() {
    Value v = value();
    ws();
    if (p_ != end_) throw std::runtime_error("json: trailing characters");
    return v;
  }

 private:
  const char* p_;
  const char* end_;

  void ws() {
    while (p_ < end_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\r' || *p_ == '\t')) ++p_;
  }
  bool lit(const char* w) {
    const char* q = p_;
    for (; *w; ++w, ++q)
      if (q >= end_ || *q != *w) return false;
    p_ = q;
    return true;
  }
  Value value() {
    ws();
    if (p_ >= end_) throw std::runtime_error("json: unexpected end");
    Value v;
    const char c = *p_;
    if (c == '{') {
      v.kind = Value::OBJ;
      ++p_;
      ws();
      if (p_ < end_ && *p_ == '}') { ++p_; return v; }
      for (;;) {
        ws();
        std::string k = string();
        ws();
        if (p_ >= end_ || *p_ != ':') throw std::runtime_error("json: expected ':'");
        ++p_;
        v.obj[k] = value();
        ws();
        if (p_ < end_ && *p_ == ',') { ++p_; continue; }
        if (p_ < end_ && *p_ == '}') { ++p_; return v; }
        throw std::runtime_error("json: expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = Value::ARR;
      ++p_;
      ws();
      if (p_ < end_ && *p_ == ']') { ++p_; return v; }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (p_ < end_ && *p_ == ',') { ++p_; continue; }
        if (p_ < end_ && *p_ == ']') { ++p_; return v; }
        throw std::runtime_error("json: expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = Value::STR;
      v.str = string();
      return v;
    }
    if (lit("true")) { v.kind = Value::BOOL; v.b = true; return v; }
    if (lit("false")) { v.kind = Value::BOOL; return v; }
    if (lit("null")) return v;
    v.kind = Value::NUM;
    if (lit("NaN")) { v.num = std::nan(""); v.str = "NaN"; return v; }
    if (lit("Infinity")) { v.num = INFINITY; v.str = "Infinity"; return v; }
    if (lit("-Infinity")) { v.num = -INFINITY; v.str = "-Infinity"; return v; }
    const char* s = p_;
    while (p_ < end_ && (std::isdigit((unsigned char)*p_) || *p_ == '-' || *p_ == '+' ||
                         *p_ == '.' || *p_ == 'e' || *p_ == 'E'))
      ++p_;
    if (p_ == s) throw std::runtime_error(std::string("json: unexpected character '") + c + "'");
    v.str.assign(s, p_);
    char* e = nullptr;
    v.num = std::strtod(v.str.c_str(), &e);
    if (!e || *e) throw std::runtime_error("json: bad number '" + v.str + "'");
    return v;
  }
  std::string string() {
    if (p_ >= end_ || *p_ != '"') throw std::runtime_error("json: expected string");
    ++p_;
    std::string out;
    while (p_ < end_ && *p_ != '"') {
      char c = *p_++;
      if (c == '\\') {
        if (p_ >= end_) break;
        const char e = *p_++;
        switch (e) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {  // names are ASCII; keep \uXXXX below 0x80 only
            if (end_ - p_ < 4) throw std::runtime_error("json: bad \\u escape");
            const int code = (int)std::strtol(std::string(p_, p_ + 4).c_str(), nullptr, 16);
            p_ += 4;
            if (code >= 0x80) throw std::runtime_error("json: non-ASCII name");
            out += (char)code;
            break;
          }
          default: out += e;
        }
      } else {
        out += c;
      }
    }
    if (p_ >= end_) throw std::runtime_error("json: unterminated string");
    ++p_;
    return out;
  }
};

inline Value parse(const char* text, size_t n) { return Parser(text, n).parse(); }

}  // namespace json
}  // namespace sfk
