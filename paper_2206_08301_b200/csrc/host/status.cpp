#include "status.hpp"

namespace eb {

namespace {
thread_local std::string g_error;
}

void set_error(const std::string& msg) { g_error = msg; }
const char* error_cstr() { return g_error.c_str(); }

}  // namespace eb

extern "C" const char* eb_last_error(void) { return eb::error_cstr(); }
