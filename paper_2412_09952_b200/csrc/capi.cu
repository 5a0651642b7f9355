// Error plumbing and version of the b200moe C ABI.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace b200moe {
static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
}  // namespace b200moe

extern "C" {
const char* b200moe_last_error(void) { return b200moe::g_err; }
int b200moe_version(void) { return 1; }
}
