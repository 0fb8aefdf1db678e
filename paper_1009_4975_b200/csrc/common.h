// Shared host-side helpers of libtomesh (error reporting, Morton keys).
#pragma once
#include <cstdint>
#include <cstdio>
#include <string>

namespace tomesh {

// Thread-local last-error message behind to_last_error() (tomesh.h).
void set_error(const char *fmt, ...);
void clear_error();

// Morton key: bit b of axis c -> bit dim*b + c (x least significant), SURVEY C2.
static inline uint64_t spread2(uint64_t v) {
  v &= 0x1fffffULL;
  v = (v | (v << 16)) & 0x0000ffff0000ffffULL;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffULL;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0fULL;
  v = (v | (v << 2)) & 0x3333333333333333ULL;
  v = (v | (v << 1)) & 0x5555555555555555ULL;
  return v;
}
static inline uint64_t spread3(uint64_t v) {
  v &= 0x1fffffULL;
  v = (v | (v << 32)) & 0x1f00000000ffffULL;
  v = (v | (v << 16)) & 0x1f0000ff0000ffULL;
  v = (v | (v << 8)) & 0x100f00f00f00f00fULL;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ULL;
  v = (v | (v << 2)) & 0x1249249249249249ULL;
  return v;
}
static inline uint64_t morton(int dim, const int32_t *c) {
  if (dim == 2) return spread2((uint64_t)c[0]) | (spread2((uint64_t)c[1]) << 1);
  return spread3((uint64_t)c[0]) | (spread3((uint64_t)c[1]) << 1) | (spread3((uint64_t)c[2]) << 2);
}

}  // namespace tomesh
