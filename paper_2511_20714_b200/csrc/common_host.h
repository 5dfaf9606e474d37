// common_host.h — thread-local last-error plumbing shared by every C-ABI entry point.
#pragma once
#include <string>

namespace ifx {
// Records `msg` as the calling thread's last error (ifx_last_error) and returns `code`.
int fail(int code, const std::string& msg);
}  // namespace ifx
