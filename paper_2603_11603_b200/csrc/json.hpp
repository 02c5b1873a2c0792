// Minimal JSON reader for the space descriptor (objects, arrays, strings, numbers, bools, null).
// Numbers are parsed with strtod (correctly rounded), so "0.82" yields the same double as
// Python's json module.
#pragma once
#include <cctype>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace asj {

struct Value {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  bool b = false;
  double num = 0.0;
  bool is_int = false;  // literal had no fraction/exponent
  std::string str;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;

  const Value* get(const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  bool has(const std::string& k) const { return get(k) != nullptr; }
};

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Parser {
 public:
  explicit Parser(const char* s) : p_(s) {}
  Value parse() {
    Value v = value();
    ws();
    if (*p_) throw ParseError("trailing characters after JSON document");
    return v;
  }

 private:
  const char* p_;
  void ws() {
    while (*p_ && std::isspace(static_cast<unsigned char>(*p_))) ++p_;
  }
  Value value() {
    ws();
    Value v;
    char c = *p_;
    if (c == '{') {
      v.kind = Value::Object;
      ++p_;
      ws();
      if (*p_ == '}') { ++p_; return v; }
      for (;;) {
        ws();
        if (*p_ != '"') throw ParseError("expected object key");
        std::string k = string();
        ws();
        if (*p_ != ':') throw ParseError("expected ':'");
        ++p_;
        v.obj.emplace_back(k, value());
        ws();
        if (*p_ == ',') { ++p_; continue; }
        if (*p_ == '}') { ++p_; break; }
        throw ParseError("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.kind = Value::Array;
      ++p_;
      ws();
      if (*p_ == ']') { ++p_; return v; }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (*p_ == ',') { ++p_; continue; }
        if (*p_ == ']') { ++p_; break; }
        throw ParseError("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.kind = Value::String;
      v.str = string();
    } else if (c == 't' && std::string(p_, 4) == "true") {
      v.kind = Value::Bool; v.b = true; p_ += 4;
    } else if (c == 'f' && std::string(p_, 5) == "false") {
      v.kind = Value::Bool; v.b = false; p_ += 5;
    } else if (c == 'n' && std::string(p_, 4) == "null") {
      v.kind = Value::Null; p_ += 4;
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      const char* s = p_;
      char* e = nullptr;
      v.num = std::strtod(s, &e);
      if (e == s) throw ParseError("bad number");
      v.kind = Value::Number;
      v.is_int = true;
      for (const char* q = s; q < e; ++q)
        if (*q == '.' || *q == 'e' || *q == 'E') v.is_int = false;
      p_ = e;
    } else {
      throw ParseError(std::string("unexpected character in JSON: ") + (c ? c : '0'));
    }
    return v;
  }
  std::string string() {
    std::string out;
    ++p_;  // opening quote
    while (*p_ && *p_ != '"') {
      if (*p_ == '\\') {
        ++p_;
        switch (*p_) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            unsigned cp = std::strtoul(std::string(p_ + 1, 4).c_str(), nullptr, 16);
            if (cp < 0x80) out += static_cast<char>(cp);
            else if (cp < 0x800) { out += static_cast<char>(0xC0 | (cp >> 6)); out += static_cast<char>(0x80 | (cp & 0x3F)); }
            else { out += static_cast<char>(0xE0 | (cp >> 12)); out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F)); out += static_cast<char>(0x80 | (cp & 0x3F)); }
            p_ += 4;
            break;
          }
          default: throw ParseError("bad escape");
        }
        ++p_;
      } else {
        out += *p_++;
      }
    }
    if (*p_ != '"') throw ParseError("unterminated string");
    ++p_;
    return out;
  }
};

inline Value parse(const char* s) { return Parser(s).parse(); }

}  // namespace asj
