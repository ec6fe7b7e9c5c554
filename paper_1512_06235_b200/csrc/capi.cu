// C-ABI glue: error reporting and version (see include/msfm_b200.h).
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace msfm {
static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
}  // namespace msfm

extern "C" const char* msfm_last_error(void) { return msfm::g_err; }
extern "C" int msfm_version(void) { return 1; }
