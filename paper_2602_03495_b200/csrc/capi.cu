// Library-level C-ABI: error reporting, version, launch counter.
#include <cstdarg>

#include "common.cuh"

namespace dali {

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace dali

extern "C" const char* dali_last_error(void) { return dali::g_err; }
extern "C" int dali_version(void) { return 1; }
extern "C" int64_t dali_launch_count(void) { return dali::g_launches.load(); }
