// Minimal JSON reader for plan documents (the wire format of export_plan,
// proj/src/execgraph.cpp:323-361).  Objects keep insertion order.
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace tpx {

struct Json {
  enum Type { Null, Bool, Number, String, Array, Object } type = Null;
  bool b = false;
  double num = 0;
  long long inum = 0;
  bool is_int = false;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;

  static Json parse(const std::string& text);  // throws Error("malformed ... document")

  bool has(const std::string& key) const;
  const Json& at(const std::string& key) const;  // throws when missing
  const Json* find(const std::string& key) const;
  long long as_int() const;
  double as_double() const;
  const std::string& as_string() const;
  bool as_bool() const;
};

// JSON string escaping for the describe / report documents the library emits.
std::string json_quote(const std::string& s);

}  // namespace tpx
