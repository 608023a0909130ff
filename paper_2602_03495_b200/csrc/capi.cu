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

// ---------------------------------------------------------------------------
// Host expert store allocation.
// ---------------------------------------------------------------------------
#include <sys/mman.h>

#include <sys/syscall.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace {
// On a multi-socket host, spread the store's pages over every NUMA node
// before first touch (MPOL_INTERLEAVE): the CPU-expert workers of every
// local rank and the GPUs' H2D copies then draw on all memory controllers
// instead of the node local rank 0 happened to run on.  One node: no-op.
// DALI_NUMA_INTERLEAVE=0 turns it off.
void interleave_numa(void* p, size_t bytes) {
  const char* env = getenv("DALI_NUMA_INTERLEAVE");
  if (env && env[0] == '0') return;
  FILE* f = fopen("/sys/devices/system/node/online", "r");
  if (!f) return;
  char buf[256] = {0};
  const bool ok = fgets(buf, sizeof(buf), f) != nullptr;
  fclose(f);
  if (!ok) return;
  unsigned long mask[4] = {0, 0, 0, 0};           // nodes 0..255
  int n_nodes = 0;
  for (char* tok = strtok(buf, ",\n"); tok; tok = strtok(nullptr, ",\n")) {
    int a = 0, b = 0;
    if (sscanf(tok, "%d-%d", &a, &b) != 2) b = a = atoi(tok);
    for (int node = a; node <= b && node < 256; ++node, ++n_nodes)
      mask[node / 64] |= 1ul << (node % 64);
  }
  if (n_nodes < 2) return;
  constexpr int kMpolInterleave = 3;
  syscall(SYS_mbind, p, bytes, kMpolInterleave, mask, 256ul, 0u);   // best effort
}
}  // namespace

extern "C" int dali_host_alloc(size_t bytes, int32_t nthreads, void** out) {
  DALI_REQUIRE(out != nullptr && bytes > 0, DALI_ECUDA, "bad host allocation request");
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  DALI_REQUIRE(p != MAP_FAILED, DALI_ECUDA, "mmap of %zu bytes failed", bytes);
  madvise(p, bytes, MADV_HUGEPAGE);
  interleave_numa(p, bytes);
  if (nthreads < 1) nthreads = 1;
  std::vector<std::thread> th;
  const size_t chunk = (bytes + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    th.emplace_back([=] {
      const size_t a = (size_t)t * chunk;
      if (a >= bytes) return;
      const size_t b = a + chunk < bytes ? a + chunk : bytes;
      char* c = static_cast<char*>(p);
      for (size_t i = a; i < b; i += 4096) c[i] = 0;
    });
  }
  for (auto& x : th) x.join();
  cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    munmap(p, bytes);
    dali::set_error("cudaHostRegister(%zu bytes): %s", bytes, cudaGetErrorString(e));
    return DALI_ECUDA;
  }
  *out = p;
  return DALI_OK;
}

extern "C" int dali_host_free(void* p, size_t bytes) {
  if (!p) return DALI_OK;
  cudaHostUnregister(p);
  munmap(p, bytes);
  return DALI_OK;
}

#include <fcntl.h>

extern "C" int dali_host_alloc_shared(size_t bytes, int32_t nthreads, int32_t create, int32_t* fd,
                                      int32_t owner_pid, void** out) {
  DALI_REQUIRE(out != nullptr && fd != nullptr && bytes > 0, DALI_ECUDA, "bad shared alloc");
  int f = -1;
  if (create) {
    f = (int)syscall(SYS_memfd_create, "dali_expert_store", 0);
    DALI_REQUIRE(f >= 0, DALI_ECUDA, "memfd_create failed");
    DALI_REQUIRE(ftruncate(f, (off_t)bytes) == 0, DALI_ECUDA, "ftruncate(%zu) failed", bytes);
  } else if (owner_pid < 0) {
    f = *fd;                     // descriptor received over a Unix socket (SCM_RIGHTS)
  } else {
    char path[64];
    snprintf(path, sizeof(path), "/proc/%d/fd/%d", owner_pid, *fd);
    f = open(path, O_RDWR);
    DALI_REQUIRE(f >= 0, DALI_ECUDA, "open(%s) failed", path);
  }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, f, 0);
  DALI_REQUIRE(p != MAP_FAILED, DALI_ECUDA, "mmap of shared store failed");
  madvise(p, bytes, MADV_HUGEPAGE);
  if (create) {
    interleave_numa(p, bytes);
    if (nthreads < 1) nthreads = 1;
    std::vector<std::thread> th;
    const size_t chunk = (bytes + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t)
      th.emplace_back([=] {
        const size_t a = (size_t)t * chunk;
        if (a >= bytes) return;
        const size_t b = a + chunk < bytes ? a + chunk : bytes;
        char* c = static_cast<char*>(p);
        for (size_t i = a; i < b; i += 4096) c[i] = 0;
      });
    for (auto& x : th) x.join();
    *fd = f;
  }
  cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    munmap(p, bytes);
    dali::set_error("cudaHostRegister(shared, %zu bytes): %s", bytes, cudaGetErrorString(e));
    return DALI_ECUDA;
  }
  *out = p;
  return DALI_OK;
}
