// Thread-local last-error message behind nc_last_error().
#include <cstdarg>
#include <cstdio>
#include "nc_common.h"

static thread_local char g_nc_error[1024] = "";

void nc_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_nc_error, sizeof(g_nc_error), fmt, ap);
  va_end(ap);
}

extern "C" const char* nc_last_error(void) { return g_nc_error; }
extern "C" int nc_abi_version(void) { return NC_ABI_VERSION; }
