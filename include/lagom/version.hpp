// lagom-b200 — API version. The public API tracks reference version 0.1.0
// (reference proj/include/lagom/version.hpp:6); reports embed this string.
#pragma once

namespace lagom {

inline constexpr const char* kVersion = "0.1.0";

}  // namespace lagom
