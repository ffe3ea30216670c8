// colo_report.cpp -- host-side report formatting helpers.
//
// The reference writes its JSON-lines reports with nlohmann/json 3.11.3
// (metrics.hpp:191-226, `nlohmann::json::dump()`), whose double formatting
// (Grisu2 + its own exponent layout) is not always the shortest round-trip
// form.  To write byte-identical reports the export path formats doubles
// with the same library (the header ships in this image; MIT licensed).
#include <cstdint>
#include <cstring>
#include <string>

#include "json.hpp"

#include "colo_abi.h"

extern "C" int64_t colo_json_doubles(const double* v, size_t n, char* out, size_t cap) {
    std::string s;
    s.reserve(n * 20);
    for (size_t i = 0; i < n; ++i) {
        if (i) s += ',';
        s += nlohmann::json(v[i]).dump();
    }
    if (out && cap > s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
    return static_cast<int64_t>(s.size());
}
