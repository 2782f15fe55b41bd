// json.hpp — TEST INFRASTRUCTURE.  Self-written stand-in for the few nlohmann::json calls in
// the reference's LoglikResult::to_json (oracle/refshim/README.md): an ordered map of scalar
// values with dump(indent).
#pragma once

#include <cstdio>
#include <map>
#include <string>

namespace nlohmann {

class json {
 public:
  class value {
   public:
    value& operator=(double v) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.17g", v);
      text_ = buf;
      return *this;
    }
    value& operator=(int v) {
      text_ = std::to_string(v);
      return *this;
    }
    value& operator=(long long v) {
      text_ = std::to_string(v);
      return *this;
    }
    value& operator=(bool v) {
      text_ = v ? "true" : "false";
      return *this;
    }
    value& operator=(const std::string& v) {
      text_ = "\"" + v + "\"";
      return *this;
    }
    value& operator=(const char* v) { return *this = std::string(v); }
    const std::string& text() const { return text_; }

   private:
    std::string text_ = "null";
  };

  value& operator[](const std::string& key) { return items_[key]; }

  std::string dump(int indent = -1) const {
    const std::string nl = indent >= 0 ? "\n" : "", pad = indent > 0 ? std::string(indent, ' ') : "";
    std::string out = "{" + nl;
    bool first = true;
    for (const auto& [k, v] : items_) {
      if (!first) out += "," + nl;
      first = false;
      out += pad + "\"" + k + "\":" + (indent >= 0 ? " " : "") + v.text();
    }
    return out + nl + "}";
  }

 private:
  std::map<std::string, value> items_;
};

}  // namespace nlohmann
