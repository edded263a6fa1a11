#include "json.hpp"

#include <cmath>
#include <cstdio>

namespace mdhb::json {

namespace {

struct Reader {
  const std::string& t;
  size_t p = 0;

  [[noreturn]] void die(const std::string& m) const {
    int line = 1, col = 1;
    for (size_t k = 0; k < p && k < t.size(); ++k) {
      if (t[k] == '\n') { ++line; col = 1; } else { ++col; }
    }
    throw ParseFailure{m + " at line " + std::to_string(line) + ", column " + std::to_string(col)};
  }
  void ws() {
    while (p < t.size() && (t[p] == ' ' || t[p] == '\t' || t[p] == '\n' || t[p] == '\r')) ++p;
  }
  bool lit(const char* w) {
    size_t n = 0;
    while (w[n]) ++n;
    if (t.compare(p, n, w) == 0) { p += n; return true; }
    return false;
  }
  std::string str() {
    if (t[p] != '"') die("expected string");
    ++p;
    std::string out;
    while (p < t.size() && t[p] != '"') {
      char c = t[p++];
      if (c == '\\') {
        if (p >= t.size()) die("bad escape");
        char e = t[p++];
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
            if (p + 4 > t.size()) die("bad \\u escape");
            unsigned cp = static_cast<unsigned>(std::strtoul(t.substr(p, 4).c_str(), nullptr, 16));
            p += 4;
            if (cp < 0x80) out += static_cast<char>(cp);
            else if (cp < 0x800) { out += static_cast<char>(0xC0 | (cp >> 6)); out += static_cast<char>(0x80 | (cp & 0x3F)); }
            else { out += static_cast<char>(0xE0 | (cp >> 12)); out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F)); out += static_cast<char>(0x80 | (cp & 0x3F)); }
            break;
          }
          default: die("bad escape");
        }
      } else {
        out += c;
      }
    }
    if (p >= t.size()) die("unterminated string");
    ++p;
    return out;
  }
  Value num() {
    size_t s = p;
    bool real = false;
    if (t[p] == '-') ++p;
    while (p < t.size() && isdigit(static_cast<unsigned char>(t[p]))) ++p;
    if (p < t.size() && t[p] == '.') { real = true; ++p; while (p < t.size() && isdigit(static_cast<unsigned char>(t[p]))) ++p; }
    if (p < t.size() && (t[p] == 'e' || t[p] == 'E')) {
      real = true;
      ++p;
      if (p < t.size() && (t[p] == '+' || t[p] == '-')) ++p;
      while (p < t.size() && isdigit(static_cast<unsigned char>(t[p]))) ++p;
    }
    std::string tok = t.substr(s, p - s);
    if (tok.empty() || tok == "-") die("bad number");
    if (real) return Value::make_real(std::strtod(tok.c_str(), nullptr));
    return Value::make_int(std::strtoll(tok.c_str(), nullptr, 10));
  }
  Value val() {
    ws();
    if (p >= t.size()) die("unexpected end of input");
    char c = t[p];
    if (c == '{') {
      ++p;
      Value v = Value::make_obj();
      ws();
      if (t[p] == '}') { ++p; return v; }
      for (;;) {
        ws();
        std::string k = str();
        ws();
        if (t[p] != ':') die("expected ':'");
        ++p;
        v.o.emplace_back(std::move(k), val());
        ws();
        if (t[p] == ',') { ++p; continue; }
        if (t[p] == '}') { ++p; return v; }
        die("expected ',' or '}'");
      }
    }
    if (c == '[') {
      ++p;
      Value v = Value::make_arr();
      ws();
      if (t[p] == ']') { ++p; return v; }
      for (;;) {
        v.a.push_back(val());
        ws();
        if (t[p] == ',') { ++p; continue; }
        if (t[p] == ']') { ++p; return v; }
        die("expected ',' or ']'");
      }
    }
    if (c == '"') return Value::make_str(str());
    if (lit("true")) { Value v; v.kind = Value::Bool; v.b = true; return v; }
    if (lit("false")) { Value v; v.kind = Value::Bool; v.b = false; return v; }
    if (lit("null")) return Value{};
    return num();
  }
};

void write(const Value& v, std::string& out, int indent, int depth) {
  auto nl = [&](int d) {
    if (indent < 0) return;
    out += '\n';
    out.append(static_cast<size_t>(indent * d), ' ');
  };
  switch (v.kind) {
    case Value::Null: out += "null"; break;
    case Value::Bool: out += v.b ? "true" : "false"; break;
    case Value::Int: out += std::to_string(v.i); break;
    case Value::Real: {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.17g", v.d);
      out += buf;
      break;
    }
    case Value::Str: {
      out += '"';
      for (char c : v.s) {
        if (c == '"' || c == '\\') { out += '\\'; out += c; }
        else if (c == '\n') out += "\\n";
        else out += c;
      }
      out += '"';
      break;
    }
    case Value::Arr: {
      out += '[';
      for (size_t k = 0; k < v.a.size(); ++k) {
        if (k) out += indent < 0 ? ", " : ",";
        nl(depth + 1);
        write(v.a[k], out, indent, depth + 1);
      }
      if (!v.a.empty()) nl(depth);
      out += ']';
      break;
    }
    case Value::Obj: {
      out += '{';
      for (size_t k = 0; k < v.o.size(); ++k) {
        if (k) out += indent < 0 ? ", " : ",";
        nl(depth + 1);
        write(Value::make_str(v.o[k].first), out, indent, depth + 1);
        out += ": ";
        write(v.o[k].second, out, indent, depth + 1);
      }
      if (!v.o.empty()) nl(depth);
      out += '}';
      break;
    }
  }
}

}  // namespace

const Value& Value::at(const std::string& key) const {
  const Value* v = find(key);
  if (!v) throw ParseFailure{"missing key '" + key + "'"};
  return *v;
}

const Value& Value::operator[](size_t k) const {
  if (kind != Arr || k >= a.size()) throw ParseFailure{"array index out of range"};
  return a[k];
}

int64_t Value::as_int() const {
  if (kind == Int) return i;
  if (kind == Real && std::floor(d) == d) return static_cast<int64_t>(d);
  throw ParseFailure{"expected an integer"};
}

double Value::as_num() const {
  if (kind == Int) return static_cast<double>(i);
  if (kind == Real) return d;
  throw ParseFailure{"expected a number"};
}

const std::string& Value::as_str() const {
  if (kind != Str) throw ParseFailure{"expected a string"};
  return s;
}

Value parse(const std::string& text) {
  Reader r{text};
  Value v = r.val();
  r.ws();
  if (r.p != text.size()) r.die("trailing characters");
  return v;
}

std::string dump(const Value& v, int indent) {
  std::string out;
  write(v, out, indent, 0);
  return out;
}

}  // namespace mdhb::json
