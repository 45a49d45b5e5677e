// Internal helpers shared by the library's translation units (not part of the ABI).
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include "lobra.h"

namespace lobra {

// Thread-local last-error string (lobra_last_error()).
void set_error(const char* fmt, ...);
void clear_error();

inline lobra_status fail(lobra_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  set_error("%s", buf);
  return st;
}

}  // namespace lobra
