#include "json.h"

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "util.h"

namespace tpx {

namespace {

struct Reader {
  const char* p;
  const char* end;

  [[noreturn]] void bad(const char* what) {
    fail(std::string("malformed plan document: ") + what);
  }
  void ws() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  bool lit(const char* s) {
    size_t n = std::strlen(s);
    if (size_t(end - p) >= n && std::memcmp(p, s, n) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  static void utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) {
      out += char(cp);
    } else if (cp < 0x800) {
      out += char(0xC0 | (cp >> 6));
      out += char(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += char(0xE0 | (cp >> 12));
      out += char(0x80 | ((cp >> 6) & 0x3F));
      out += char(0x80 | (cp & 0x3F));
    } else {
      out += char(0xF0 | (cp >> 18));
      out += char(0x80 | ((cp >> 12) & 0x3F));
      out += char(0x80 | ((cp >> 6) & 0x3F));
      out += char(0x80 | (cp & 0x3F));
    }
  }
  unsigned hex4() {
    if (end - p < 4) bad("truncated \\u escape");
    unsigned v = 0;
    for (int i = 0; i < 4; ++i) {
      char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= unsigned(c - '0');
      else if (c >= 'a' && c <= 'f') v |= unsigned(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= unsigned(c - 'A' + 10);
      else bad("bad \\u escape");
    }
    return v;
  }
  std::string string() {
    if (p >= end || *p != '"') bad("expected string");
    ++p;
    std::string out;
    while (true) {
      if (p >= end) bad("unterminated string");
      char c = *p++;
      if (c == '"') break;
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p >= end) bad("unterminated escape");
      char e = *p++;
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
          if (cp >= 0xD800 && cp < 0xDC00 && end - p >= 6 && p[0] == '\\' && p[1] == 'u') {
            p += 2;
            unsigned lo = hex4();
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          utf8(out, cp);
          break;
        }
        default: bad("bad escape");
      }
    }
    return out;
  }
  Json value(int depth) {
    if (depth > 256) bad("nesting too deep");
    ws();
    if (p >= end) bad("unexpected end of input");
    Json j;
    char c = *p;
    if (c == '{') {
      ++p;
      j.type = Json::Object;
      ws();
      if (p < end && *p == '}') {
        ++p;
        return j;
      }
      while (true) {
        ws();
        std::string k = string();
        ws();
        if (p >= end || *p != ':') bad("expected ':'");
        ++p;
        j.obj.emplace_back(std::move(k), value(depth + 1));
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == '}') {
          ++p;
          break;
        }
        bad("expected ',' or '}'");
      }
      return j;
    }
    if (c == '[') {
      ++p;
      j.type = Json::Array;
      ws();
      if (p < end && *p == ']') {
        ++p;
        return j;
      }
      while (true) {
        j.arr.push_back(value(depth + 1));
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == ']') {
          ++p;
          break;
        }
        bad("expected ',' or ']'");
      }
      return j;
    }
    if (c == '"') {
      j.type = Json::String;
      j.str = string();
      return j;
    }
    if (lit("true")) {
      j.type = Json::Bool;
      j.b = true;
      return j;
    }
    if (lit("false")) {
      j.type = Json::Bool;
      return j;
    }
    if (lit("null")) return j;
    if (c == '-' || (c >= '0' && c <= '9')) {
      const char* s = p;
      bool integral = true;
      if (*p == '-') ++p;
      while (p < end && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' ||
                         *p == '+' || *p == '-')) {
        if (*p == '.' || *p == 'e' || *p == 'E') integral = false;
        ++p;
      }
      std::string tok(s, p);
      j.type = Json::Number;
      char* e = nullptr;
      j.num = std::strtod(tok.c_str(), &e);
      if (!e || *e) bad("bad number");
      if (integral) {
        j.inum = std::strtoll(tok.c_str(), &e, 10);
        j.is_int = true;
      } else {
        j.inum = (long long)j.num;
      }
      return j;
    }
    bad("unexpected character");
  }
};

}  // namespace

Json Json::parse(const std::string& text) {
  Reader r{text.data(), text.data() + text.size()};
  Json j = r.value(0);
  r.ws();
  if (r.p != r.end) r.bad("trailing characters");
  return j;
}

bool Json::has(const std::string& key) const { return find(key) != nullptr; }

const Json* Json::find(const std::string& key) const {
  if (type != Object) return nullptr;
  for (const auto& kv : obj)
    if (kv.first == key) return &kv.second;
  return nullptr;
}

const Json& Json::at(const std::string& key) const {
  const Json* j = find(key);
  if (!j) fail("malformed plan document: missing key '" + key + "'");
  return *j;
}

long long Json::as_int() const {
  if (type != Number) fail("malformed plan document: expected a number");
  if (!is_int && std::floor(num) != num) fail("malformed plan document: expected an integer");
  return is_int ? inum : (long long)num;
}

double Json::as_double() const {
  if (type != Number) fail("malformed plan document: expected a number");
  return num;
}

const std::string& Json::as_string() const {
  if (type != String) fail("malformed plan document: expected a string");
  return str;
}

bool Json::as_bool() const {
  if (type != Bool) fail("malformed plan document: expected a boolean");
  return b;
}

std::string json_quote(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\n': o += "\\n"; break;
      case '\t': o += "\\t"; break;
      default:
        if ((unsigned char)c < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", c);
          o += buf;
        } else {
          o += c;
        }
    }
  }
  return o + "\"";
}

}  // namespace tpx
