// sl_internal_host.h — the pieces of sl_internal.cuh that host-only translation units (g++)
// need: the thread-local error message behind sl_last_error().
#pragma once

#include <string>

namespace sl {
void set_error(const std::string& msg);
const std::string& get_error();
}  // namespace sl
