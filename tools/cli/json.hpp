// json.hpp — a minimal ordered JSON value for the CLI reports (no third-party dependency).
// Objects keep insertion order; numbers print as integers or shortest round-trip doubles;
// dump(-1) is compact, dump(2) indents like the reference's report output.
#pragma once

#include <charconv>
#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

namespace cli {

class Json {
 public:
  enum class Kind { Null, Bool, Int, UInt, Double, String, Array, Object };

  Json() = default;
  Json(bool b) : kind_(Kind::Bool), b_(b) {}                          // NOLINT
  Json(int v) : kind_(Kind::Int), i_(v) {}                            // NOLINT
  Json(long v) : kind_(Kind::Int), i_(v) {}                           // NOLINT
  Json(long long v) : kind_(Kind::Int), i_(v) {}                      // NOLINT
  Json(unsigned v) : kind_(Kind::UInt), u_(v) {}                      // NOLINT
  Json(unsigned long v) : kind_(Kind::UInt), u_(v) {}                 // NOLINT
  Json(unsigned long long v) : kind_(Kind::UInt), u_(v) {}            // NOLINT
  Json(float v) : kind_(Kind::Double), d_(v) {}                       // NOLINT
  Json(double v) : kind_(Kind::Double), d_(v) {}                      // NOLINT
  Json(const char* s) : kind_(Kind::String), s_(s) {}                 // NOLINT
  Json(std::string s) : kind_(Kind::String), s_(std::move(s)) {}      // NOLINT

  static Json object() {
    Json j;
    j.kind_ = Kind::Object;
    return j;
  }
  static Json array() {
    Json j;
    j.kind_ = Kind::Array;
    return j;
  }

  Json& operator[](const std::string& key) {
    if (kind_ == Kind::Null) kind_ = Kind::Object;
    for (auto& kv : obj_)
      if (kv.first == key) return kv.second;
    obj_.emplace_back(key, Json());
    return obj_.back().second;
  }
  void push_back(Json v) {
    if (kind_ == Kind::Null) kind_ = Kind::Array;
    arr_.push_back(std::move(v));
  }
  void erase(const std::string& key) {
    for (auto it = obj_.begin(); it != obj_.end(); ++it)
      if (it->first == key) {
        obj_.erase(it);
        return;
      }
  }
  bool contains(const std::string& key) const {
    for (auto& kv : obj_)
      if (kv.first == key) return true;
    return false;
  }
  Kind kind() const { return kind_; }
  const std::vector<std::pair<std::string, Json>>& items() const { return obj_; }
  const std::vector<Json>& elements() const { return arr_; }

  std::string dump(int indent = -1) const {
    std::string out;
    write(out, indent, 0);
    return out;
  }

 private:
  static void esc(std::string& out, const std::string& s) {
    out += '"';
    for (char c : s) {
      switch (c) {
        case '"': out += "\\\""; break;
        case '\\': out += "\\\\"; break;
        case '\n': out += "\\n"; break;
        case '\t': out += "\\t"; break;
        case '\r': out += "\\r"; break;
        default:
          if (static_cast<unsigned char>(c) < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof(buf), "\\u%04x", c);
            out += buf;
          } else {
            out += c;
          }
      }
    }
    out += '"';
  }
  static void num(std::string& out, double d) {
    if (!std::isfinite(d)) {
      out += "null";  // JSON has no NaN / Inf
      return;
    }
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), d);  // shortest round-trip representation
    std::string s(buf, r.ptr);
    if (s.find_first_of(".eE") == std::string::npos) s += ".0";
    out += s;
  }
  void write(std::string& out, int indent, int depth) const {
    const bool pretty = indent >= 0;
    auto nl = [&](int dep) {
      if (pretty) {
        out += '\n';
        out.append(static_cast<std::size_t>(indent * dep), ' ');
      }
    };
    switch (kind_) {
      case Kind::Null: out += "null"; break;
      case Kind::Bool: out += b_ ? "true" : "false"; break;
      case Kind::Int: out += std::to_string(i_); break;
      case Kind::UInt: out += std::to_string(u_); break;
      case Kind::Double: num(out, d_); break;
      case Kind::String: esc(out, s_); break;
      case Kind::Array:
        if (arr_.empty()) {
          out += "[]";
          break;
        }
        out += '[';
        for (std::size_t i = 0; i < arr_.size(); ++i) {
          if (i) out += ',';
          nl(depth + 1);
          arr_[i].write(out, indent, depth + 1);
        }
        nl(depth);
        out += ']';
        break;
      case Kind::Object:
        if (obj_.empty()) {
          out += "{}";
          break;
        }
        out += '{';
        for (std::size_t i = 0; i < obj_.size(); ++i) {
          if (i) out += ',';
          nl(depth + 1);
          esc(out, obj_[i].first);
          out += pretty ? ": " : ":";
          obj_[i].second.write(out, indent, depth + 1);
        }
        nl(depth);
        out += '}';
        break;
    }
  }

  Kind kind_ = Kind::Null;
  bool b_ = false;
  long long i_ = 0;
  unsigned long long u_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<Json> arr_;
  std::vector<std::pair<std::string, Json>> obj_;
};

// 64-bit FNV-1a, hex (the reference's config_hash over the compact config echo).
inline std::string fnv1a_hex(const std::string& text) {
  std::uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char c : text) {
    h ^= c;
    h *= 0x100000001b3ull;
  }
  char buf[17];
  std::snprintf(buf, sizeof(buf), "%016llx", static_cast<unsigned long long>(h));
  return buf;
}

// CSV: one row per element of a top-level "cells" array (shared scalars repeated), else one row;
// nested keys flattened with '.', array members with [i]; cells are compact JSON so CSV text
// matches the JSON emission exactly.
inline void flatten(const Json& node, const std::string& prefix,
                    std::vector<std::pair<std::string, Json>>& out) {
  if (node.kind() == Json::Kind::Object) {
    for (const auto& kv : node.items())
      flatten(kv.second, prefix.empty() ? kv.first : prefix + "." + kv.first, out);
  } else if (node.kind() == Json::Kind::Array) {
    std::size_t i = 0;
    for (const auto& v : node.elements()) flatten(v, prefix + "[" + std::to_string(i++) + "]", out);
  } else {
    out.emplace_back(prefix, node);
  }
}

inline std::string to_csv(const Json& report) {
  Json shared = report;
  std::vector<Json> rows;
  if (report.contains("cells")) {
    shared.erase("cells");
    for (const auto& kv : report.items())
      if (kv.first == "cells")
        for (const auto& c : kv.second.elements()) rows.push_back(c);
  } else {
    rows.push_back(Json::object());
  }
  std::vector<std::pair<std::string, Json>> shared_flat;
  flatten(shared, "", shared_flat);
  std::vector<std::string> cols;
  for (const auto& kv : shared_flat) cols.push_back(kv.first);
  std::vector<std::vector<std::pair<std::string, Json>>> flats;
  for (const auto& r : rows) {
    flats.emplace_back();
    flatten(r, "", flats.back());
    for (const auto& kv : flats.back()) {
      bool seen = false;
      for (const auto& c : cols) seen = seen || c == kv.first;
      if (!seen) cols.push_back(kv.first);
    }
  }
  std::string out;
  for (std::size_t c = 0; c < cols.size(); ++c) out += (c ? "," : "") + cols[c];
  out += '\n';
  for (const auto& flat : flats) {
    std::map<std::string, std::string> cell;
    for (const auto& kv : flat) cell[kv.first] = kv.second.dump();
    for (const auto& kv : shared_flat) cell.emplace(kv.first, kv.second.dump());
    for (std::size_t c = 0; c < cols.size(); ++c) {
      if (c) out += ',';
      auto it = cell.find(cols[c]);
      if (it != cell.end()) out += it->second;
    }
    out += '\n';
  }
  return out;
}

}  // namespace cli
