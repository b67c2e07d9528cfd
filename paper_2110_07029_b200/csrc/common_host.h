// Host-side helpers shared by the C-ABI translation units (error reporting).
#pragma once
#include <cstdarg>
#include <cstdio>

#include "adasgd.h"

// Thread-local message for as_last_error(); defined in api.cu.
extern thread_local char g_as_err[512];

static inline int as_fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_as_err, sizeof(g_as_err), fmt, ap);
  va_end(ap);
  return code;
}
