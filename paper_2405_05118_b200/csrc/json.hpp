// Minimal JSON value + parser + writer for the md_hom spec/config dialect.
// (The reference uses nlohmann/json, proj/src/json_io.cpp:6; the product keeps
// no third-party dependency, so this is a small self-contained reader.)
#pragma once

#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

namespace mdhb::json {

struct Value {
  enum Kind { Null, Bool, Int, Real, Str, Arr, Obj } kind = Null;
  bool b = false;
  int64_t i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Value> a;
  std::vector<std::pair<std::string, Value>> o;  // insertion order kept

  bool is_null() const { return kind == Null; }
  bool is_int() const { return kind == Int; }
  bool is_num() const { return kind == Int || kind == Real; }
  bool is_str() const { return kind == Str; }
  bool is_arr() const { return kind == Arr; }
  bool is_obj() const { return kind == Obj; }
  size_t size() const { return kind == Arr ? a.size() : kind == Obj ? o.size() : 0; }

  const Value* find(const std::string& key) const {
    if (kind != Obj) return nullptr;
    for (auto& kv : o)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
  bool has(const std::string& key) const { return find(key) != nullptr; }
  const Value& at(const std::string& key) const;
  const Value& operator[](size_t k) const;
  int64_t as_int() const;
  double as_num() const;
  const std::string& as_str() const;

  static Value make_int(int64_t v) { Value x; x.kind = Int; x.i = v; return x; }
  static Value make_real(double v) { Value x; x.kind = Real; x.d = v; return x; }
  static Value make_str(std::string v) { Value x; x.kind = Str; x.s = std::move(v); return x; }
  static Value make_arr() { Value x; x.kind = Arr; return x; }
  static Value make_obj() { Value x; x.kind = Obj; return x; }
  Value& push(Value v) { a.push_back(std::move(v)); return a.back(); }
  Value& set(const std::string& k, Value v) {
    for (auto& kv : o)
      if (kv.first == k) { kv.second = std::move(v); return kv.second; }
    o.emplace_back(k, std::move(v));
    return o.back().second;
  }
};

struct ParseFailure {
  std::string msg;
};

Value parse(const std::string& text);        // throws ParseFailure
std::string dump(const Value& v, int indent = -1);

}  // namespace mdhb::json
