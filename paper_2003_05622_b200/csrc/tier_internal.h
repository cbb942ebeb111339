// Host-side internals shared by the translation units of libhps_gpu.so.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "hps_gpu.h"

namespace hpsgpu {

// Thread-local last-error message behind hps_last_error().
void set_error_message(const std::string& msg);
const char* error_message();

inline hps_status set_error(hps_status code, const char* fmt, ...) {
  char buf[768];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  set_error_message(buf);
  return code;
}

// replicate_dense(init_dense(cfg)) weights (model.hpp:42-53), host side.
void init_dense_host(const hps_config* cfg, float* out, std::uint64_t n);

}  // namespace hpsgpu
