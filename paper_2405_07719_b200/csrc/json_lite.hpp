// json_lite.hpp — the small JSON subset the request/report boundary needs.
//
// The reference's public C ABI (include/uspsim.h:33-40) takes a JSON request
// and returns a JSON report; it uses nlohmann::json (3.11.x, header-only).
// This is a self-contained restatement of the parts of that library the
// `simulate` command touches:
//   * parse: RFC 8259 documents; integers without sign -> unsigned, with a
//     sign -> signed, anything with '.', 'e' or overflow -> double;
//     objects are ordered maps (duplicate keys: last wins);
//   * dump: compact form, object keys sorted, doubles printed as the
//     shortest round-trip digits in nlohmann's layout (dtoa_impl::
//     format_buffer: "1.0", "0.001", "1e-05", "1e+16"), strings escaped as
//     nlohmann does with ensure_ascii = false. The reference hashes this dump
//     (config_digest, commands.cpp:27-33), so the digest matches only if the
//     bytes do;
//   * typed access with nlohmann's conversions and type_error messages
//     ("[json.exception.type_error.302] type must be number, but is string").
#pragma once

#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace uspb200::json {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};

class Value {
 public:
  enum class Kind { kNull, kBool, kInt, kUint, kDouble, kString, kArray, kObject };
  using Object = std::map<std::string, Value>;
  using Array = std::vector<Value>;

  Value() = default;
  Value(std::nullptr_t) {}
  Value(bool b) : kind_(Kind::kBool), b_(b) {}
  Value(int v) : Value(static_cast<int64_t>(v)) {}
  Value(int64_t v) {
    if (v >= 0) {
      kind_ = Kind::kUint;
      u_ = static_cast<uint64_t>(v);
    } else {
      kind_ = Kind::kInt;
      i_ = v;
    }
  }
  Value(uint64_t v) : kind_(Kind::kUint), u_(v) {}
  Value(double v) : kind_(Kind::kDouble), d_(v) {}
  Value(const char* s) : kind_(Kind::kString), s_(s) {}
  Value(std::string s) : kind_(Kind::kString), s_(std::move(s)) {}
  Value(Array a) : kind_(Kind::kArray), a_(std::make_shared<Array>(std::move(a))) {}
  Value(Object o) : kind_(Kind::kObject), o_(std::make_shared<Object>(std::move(o))) {}

  static Value object() { return Value(Object{}); }
  static Value array() { return Value(Array{}); }

  Kind kind() const { return kind_; }
  bool is_object() const { return kind_ == Kind::kObject; }
  bool is_number() const { return kind_ == Kind::kInt || kind_ == Kind::kUint || kind_ == Kind::kDouble; }

  const char* type_name() const {
    switch (kind_) {
      case Kind::kNull: return "null";
      case Kind::kBool: return "boolean";
      case Kind::kString: return "string";
      case Kind::kArray: return "array";
      case Kind::kObject: return "object";
      default: return "number";
    }
  }

  // ---- objects
  bool contains(const std::string& key) const { return is_object() && o_->count(key) != 0; }
  const Value& at(const std::string& key) const {
    if (!is_object())
      throw Error(std::string("[json.exception.type_error.304] cannot use at() with ") + type_name());
    auto it = o_->find(key);
    if (it == o_->end()) throw Error("[json.exception.out_of_range.403] key '" + key + "' not found");
    return it->second;
  }
  Value& operator[](const std::string& key) {
    if (kind_ == Kind::kNull) *this = object();
    if (!is_object())
      throw Error(std::string("[json.exception.type_error.305] cannot use operator[] with a string argument with ") +
                  type_name());
    if (o_.use_count() > 1) o_ = std::make_shared<Object>(*o_);  // copy on write
    return (*o_)[key];
  }
  const Object& items() const { return *o_; }
  void push_back(Value v) {
    if (kind_ == Kind::kNull) *this = array();
    if (a_.use_count() > 1) a_ = std::make_shared<Array>(*a_);
    a_->push_back(std::move(v));
  }

  // ---- conversions (nlohmann get<T>() semantics)
  int64_t get_int() const {
    switch (kind_) {
      case Kind::kInt: return i_;
      case Kind::kUint: return static_cast<int64_t>(u_);
      case Kind::kDouble: return static_cast<int64_t>(d_);
      default: throw type_error("number");
    }
  }
  uint64_t get_uint() const {
    switch (kind_) {
      case Kind::kInt: return static_cast<uint64_t>(i_);
      case Kind::kUint: return u_;
      case Kind::kDouble: return static_cast<uint64_t>(d_);
      default: throw type_error("number");
    }
  }
  double get_double() const {
    switch (kind_) {
      case Kind::kInt: return static_cast<double>(i_);
      case Kind::kUint: return static_cast<double>(u_);
      case Kind::kDouble: return d_;
      default: throw type_error("number");
    }
  }
  bool get_bool() const {
    if (kind_ != Kind::kBool) throw type_error("boolean");
    return b_;
  }
  const std::string& get_string() const {
    if (kind_ != Kind::kString) throw type_error("string");
    return s_;
  }

  // value(key, default) (nlohmann basic_json::value): type_error.306 on a
  // non-object, the default when the key is absent, get<T>() otherwise.
  int64_t value(const std::string& key, int64_t def) const { return lookup(key) ? lookup(key)->get_int() : def; }
  int value(const std::string& key, int def) const {
    return lookup(key) ? static_cast<int>(lookup(key)->get_int()) : def;
  }
  uint64_t value(const std::string& key, uint64_t def) const {
    return lookup(key) ? lookup(key)->get_uint() : def;
  }
  double value(const std::string& key, double def) const { return lookup(key) ? lookup(key)->get_double() : def; }
  bool value(const std::string& key, bool def) const { return lookup(key) ? lookup(key)->get_bool() : def; }
  std::string value(const std::string& key, const std::string& def) const {
    return lookup(key) ? lookup(key)->get_string() : def;
  }

  std::string dump() const {
    std::string out;
    dump_to(out);
    return out;
  }

 private:
  Error type_error(const char* want) const {
    return Error(std::string("[json.exception.type_error.302] type must be ") + want + ", but is " + type_name());
  }
  const Value* lookup(const std::string& key) const {
    if (!is_object())
      throw Error(std::string("[json.exception.type_error.306] cannot use value() with ") + type_name());
    auto it = o_->find(key);
    return it == o_->end() ? nullptr : &it->second;
  }

  static void dump_string(std::string& out, const std::string& s) {
    out += '"';
    for (unsigned char c : s) {
      switch (c) {
        case '"': out += "\\\""; break;
        case '\\': out += "\\\\"; break;
        case '\b': out += "\\b"; break;
        case '\f': out += "\\f"; break;
        case '\n': out += "\\n"; break;
        case '\r': out += "\\r"; break;
        case '\t': out += "\\t"; break;
        default:
          if (c < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof(buf), "\\u%04x", c);
            out += buf;
          } else {
            out += static_cast<char>(c);
          }
      }
    }
    out += '"';
  }

  // nlohmann dtoa_impl::format_buffer layout over the shortest digits.
  static void dump_double(std::string& out, double v) {
    if (!std::isfinite(v)) {
      out += "null";
      return;
    }
    if (v == 0) {
      out += std::signbit(v) ? "-0.0" : "0.0";
      return;
    }
    char sci[64];
    auto res = std::to_chars(sci, sci + sizeof(sci), v, std::chars_format::scientific);
    std::string s(sci, res.ptr);
    std::string sign;
    if (s[0] == '-') {
      sign = "-";
      s = s.substr(1);
    }
    const size_t epos = s.find('e');
    const int e10 = std::atoi(s.c_str() + epos + 1);
    std::string digits;
    for (size_t i = 0; i < epos; ++i)
      if (s[i] != '.') digits += s[i];
    const int k = static_cast<int>(digits.size());
    const int n = e10 + 1;  // value = 0.d1d2..dk * 10^n
    constexpr int kMinExp = -4, kMaxExp = 15;
    out += sign;
    if (k <= n && n <= kMaxExp) {
      out += digits + std::string(n - k, '0') + ".0";
    } else if (0 < n && n <= kMaxExp) {
      out += digits.substr(0, n) + "." + digits.substr(n);
    } else if (kMinExp < n && n <= 0) {
      out += "0." + std::string(-n, '0') + digits;
    } else {
      out += digits.substr(0, 1);
      if (k > 1) out += "." + digits.substr(1);
      int e = n - 1;
      out += e < 0 ? "e-" : "e+";
      e = std::abs(e);
      if (e < 10) out += '0';
      out += std::to_string(e);
    }
  }

  void dump_to(std::string& out) const {
    switch (kind_) {
      case Kind::kNull: out += "null"; break;
      case Kind::kBool: out += b_ ? "true" : "false"; break;
      case Kind::kInt: out += std::to_string(i_); break;
      case Kind::kUint: out += std::to_string(u_); break;
      case Kind::kDouble: dump_double(out, d_); break;
      case Kind::kString: dump_string(out, s_); break;
      case Kind::kArray: {
        out += '[';
        bool first = true;
        for (const auto& x : *a_) {
          if (!first) out += ',';
          first = false;
          x.dump_to(out);
        }
        out += ']';
        break;
      }
      case Kind::kObject: {
        out += '{';
        bool first = true;
        for (const auto& [key, x] : *o_) {
          if (!first) out += ',';
          first = false;
          dump_string(out, key);
          out += ':';
          x.dump_to(out);
        }
        out += '}';
        break;
      }
    }
  }

  Kind kind_ = Kind::kNull;
  bool b_ = false;
  int64_t i_ = 0;
  uint64_t u_ = 0;
  double d_ = 0;
  std::string s_;
  std::shared_ptr<Array> a_;
  std::shared_ptr<Object> o_;
};

// ------------------------------------------------------------------ parser
class Parser {
 public:
  explicit Parser(const std::string& text) : t_(text) {}

  Value parse_document() {
    Value v = parse_value();
    skip_ws();
    if (i_ != t_.size()) fail("unexpected trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& what) const {
    throw Error("[json.exception.parse_error.101] parse error at byte " + std::to_string(i_ + 1) + ": " + what);
  }
  void skip_ws() {
    while (i_ < t_.size() && (t_[i_] == ' ' || t_[i_] == '\t' || t_[i_] == '\n' || t_[i_] == '\r')) ++i_;
  }
  bool consume(const char* lit) {
    size_t n = std::char_traits<char>::length(lit);
    if (t_.compare(i_, n, lit) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }

  Value parse_value() {
    skip_ws();
    if (i_ >= t_.size()) fail("unexpected end of input");
    const char c = t_[i_];
    if (c == '{') return parse_object();
    if (c == '[') return parse_array();
    if (c == '"') return Value(parse_string());
    if (consume("true")) return Value(true);
    if (consume("false")) return Value(false);
    if (consume("null")) return Value(nullptr);
    if (c == '-' || (c >= '0' && c <= '9')) return parse_number();
    fail("syntax error while parsing value");
  }

  Value parse_object() {
    ++i_;
    Value obj = Value::object();
    skip_ws();
    if (i_ < t_.size() && t_[i_] == '}') {
      ++i_;
      return obj;
    }
    for (;;) {
      skip_ws();
      if (i_ >= t_.size() || t_[i_] != '"') fail("object key must be a string");
      std::string key = parse_string();
      skip_ws();
      if (i_ >= t_.size() || t_[i_] != ':') fail("expected ':'");
      ++i_;
      obj[key] = parse_value();
      skip_ws();
      if (i_ < t_.size() && t_[i_] == ',') {
        ++i_;
        continue;
      }
      if (i_ < t_.size() && t_[i_] == '}') {
        ++i_;
        return obj;
      }
      fail("expected ',' or '}'");
    }
  }

  Value parse_array() {
    ++i_;
    Value arr = Value::array();
    skip_ws();
    if (i_ < t_.size() && t_[i_] == ']') {
      ++i_;
      return arr;
    }
    for (;;) {
      arr.push_back(parse_value());
      skip_ws();
      if (i_ < t_.size() && t_[i_] == ',') {
        ++i_;
        continue;
      }
      if (i_ < t_.size() && t_[i_] == ']') {
        ++i_;
        return arr;
      }
      fail("expected ',' or ']'");
    }
  }

  static void put_utf8(std::string& out, uint32_t cp) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
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

  uint32_t hex4() {
    if (i_ + 4 > t_.size()) fail("truncated \\u escape");
    uint32_t v = 0;
    for (int j = 0; j < 4; ++j) {
      const char c = t_[i_++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= c - '0';
      else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
      else fail("invalid \\u escape");
    }
    return v;
  }

  std::string parse_string() {
    ++i_;  // opening quote
    std::string out;
    for (;;) {
      if (i_ >= t_.size()) fail("missing closing quote");
      const char c = t_[i_++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (i_ >= t_.size()) fail("truncated escape");
      const char e = t_[i_++];
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
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00) {
            if (!consume("\\u")) fail("unpaired surrogate");
            const uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("invalid surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          put_utf8(out, cp);
          break;
        }
        default: fail("invalid escape");
      }
    }
  }

  Value parse_number() {
    const size_t start = i_;
    bool neg = false, is_float = false;
    if (t_[i_] == '-') {
      neg = true;
      ++i_;
    }
    if (i_ >= t_.size() || !(t_[i_] >= '0' && t_[i_] <= '9')) fail("invalid number");
    if (t_[i_] == '0') {
      ++i_;
    } else {
      while (i_ < t_.size() && t_[i_] >= '0' && t_[i_] <= '9') ++i_;
    }
    if (i_ < t_.size() && t_[i_] == '.') {
      is_float = true;
      ++i_;
      if (i_ >= t_.size() || !(t_[i_] >= '0' && t_[i_] <= '9')) fail("invalid number");
      while (i_ < t_.size() && t_[i_] >= '0' && t_[i_] <= '9') ++i_;
    }
    if (i_ < t_.size() && (t_[i_] == 'e' || t_[i_] == 'E')) {
      is_float = true;
      ++i_;
      if (i_ < t_.size() && (t_[i_] == '+' || t_[i_] == '-')) ++i_;
      if (i_ >= t_.size() || !(t_[i_] >= '0' && t_[i_] <= '9')) fail("invalid number");
      while (i_ < t_.size() && t_[i_] >= '0' && t_[i_] <= '9') ++i_;
    }
    const std::string tok = t_.substr(start, i_ - start);
    if (!is_float) {
      if (neg) {
        int64_t v = 0;
        auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
        if (r.ec == std::errc()) return Value(v);
      } else {
        uint64_t v = 0;
        auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
        if (r.ec == std::errc()) return Value(v);
      }
    }
    return Value(std::strtod(tok.c_str(), nullptr));
  }

  const std::string& t_;
  size_t i_ = 0;
};

inline Value parse(const std::string& text) { return Parser(text).parse_document(); }

}  // namespace uspb200::json
