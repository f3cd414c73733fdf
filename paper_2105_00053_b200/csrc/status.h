// Shared C-ABI error state (pnn_last_error()).
#pragma once

#include <string>

namespace pnn_b200 {
void set_last_error(const std::string& msg);
int set_status(int code, const std::string& msg);  // sets the message, returns code
}  // namespace pnn_b200
