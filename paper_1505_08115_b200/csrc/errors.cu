// Thread-local error message store behind rq_last_error().
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace rq {
static thread_local char g_msg[1024] = "";
int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_msg, sizeof(g_msg), fmt, ap);
  va_end(ap);
  return code;
}
const char* last_error() { return g_msg; }
void clear_error() { g_msg[0] = 0; }
}  // namespace rq
