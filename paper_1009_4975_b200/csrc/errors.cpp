// to_last_error() backing store (thread-local), shared by the host builder and
// the device library.
#include <cstdarg>
#include <cstdio>

#include "common.h"

namespace tomesh {
static thread_local char g_err[1024] = {0};

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void clear_error() { g_err[0] = 0; }
}  // namespace tomesh

extern "C" const char *to_last_error(void) { return tomesh::g_err; }
