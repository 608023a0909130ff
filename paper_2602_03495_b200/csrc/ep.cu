// Expert-parallel token exchange over peer memory (NVLink / NVSwitch on a
// B200 node): the dispatch and return all-to-alls of the EP MoE layer are
// fused with the permute / unpermute they bracket, as stores straight into
// the peer rank's receive buffers (CUDA IPC mappings), with a system-scope
// arrival counter per rank instead of a collective.
//
// Per rank, one IPC allocation holds (see dali_ep_layout):
//   recv  [G][cap][d]  bf16   rows other ranks send to my experts
//   ret   [G][cap][d]  f32    expert outputs my rows get back
//   cnt   [G][NL]      i32    rows each source sends to each of my experts
//   flags [2]          u64    dispatch / return arrival counters (monotonic)
// Source block s of recv/ret is written only by rank s; the row index inside
// the block is the row's index within the source's permuted rows for this
// destination, so no sender needs another sender's counts.  Each direction
// ends with __threadfence_system + one atomic increment of every peer's
// counter by the grid's last CTA; a receiver waits for counter >= epoch * G
// (bounded spin: a lost peer sets an error flag instead of hanging).
#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace dali {

__device__ __forceinline__ int find_bucket(const int32_t* __restrict__ offs, int n, int r) {
  int lo = 0, hi = n;                         // offs[lo] <= r < offs[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (offs[mid] <= r) lo = mid; else hi = mid;
  }
  return lo;
}

// Count arrivals of this grid; the last CTA bumps every peer's counter.
__device__ void signal_peers(unsigned int* done, const uint64_t* __restrict__ peer_flag,
                             int G) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(done, 1u);
    if (prev == gridDim.x - 1) {
      *done = 0u;
      __threadfence_system();
      for (int g = 0; g < G; ++g)
        atomicAdd_system(reinterpret_cast<unsigned long long*>(peer_flag[g]), 1ull);
    }
  }
}

// Dispatch: row r of this rank's permuted rows (grouped by global expert)
// goes to owner q = expert / NL at recv_q[rank][r - offsets[q*NL]].
__global__ void ep_dispatch_kernel(const uint4* __restrict__ x, const int32_t* __restrict__ perm,
                                   const int32_t* __restrict__ offsets, int N, int NL, int G,
                                   int rank, int64_t cap, int d8,
                                   const uint64_t* __restrict__ peer_recv,
                                   const uint64_t* __restrict__ peer_cnt,
                                   const uint64_t* __restrict__ peer_flag,
                                   unsigned int* done) {
  DALI_PDL_ENTRY();
  const int rows = offsets[N];
  const int64_t items = (int64_t)rows * d8;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(it / d8), c = (int)(it - (int64_t)r * d8);
    const int e = find_bucket(offsets, N, r);
    const int q = e / NL;
    const int64_t idx = r - offsets[q * NL];
    uint4* dst = reinterpret_cast<uint4*>(peer_recv[q]) + ((int64_t)rank * cap + idx) * d8;
    dst[c] = x[(int64_t)perm[r] * d8 + c];
  }
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const int q = i / NL, j = i % NL;
      reinterpret_cast<int32_t*>(peer_cnt[q])[rank * NL + j] = offsets[i + 1] - offsets[i];
    }
  signal_peers(done, peer_flag, G);
}

__global__ void ep_wait_kernel(const unsigned long long* flag, unsigned long long target,
                               long long max_spins, int32_t* err) {
  DALI_PDL_ENTRY();
  if (threadIdx.x != 0) return;
  long long spins = 0;
  unsigned long long v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= target) break;
    if (++spins > max_spins) {
      *err = 1;
      break;
    }
    __nanosleep(64);
  }
  __threadfence_system();
}

// Receive plan (one CTA): cnt[s][j] -> grouped order (local expert j, source
// s, t): offs_l (NL+1), perm2[i] = s*cap + sum_{j'<j} cnt[s][j'] + t,
// workloads[j] = sum_s cnt[s][j] (int64, the policy's global workloads),
// meta[0] = total rows.
__global__ void ep_recv_plan_kernel(const int32_t* __restrict__ cnt, int G, int NL, int64_t cap,
                                    int32_t* __restrict__ perm2, int32_t* __restrict__ offs_l,
                                    int64_t* __restrict__ workloads, int32_t* __restrict__ meta) {
  DALI_PDL_ENTRY();
  __shared__ int base[DALI_MAX_EXPERTS + 1];
  if (threadIdx.x == 0) {
    int run = 0;
    for (int j = 0; j < NL; ++j) {
      base[j] = run;
      offs_l[j] = run;
      int tot = 0;
      for (int s = 0; s < G; ++s) tot += cnt[s * NL + j];
      workloads[j] = tot;
      run += tot;
    }
    base[NL] = run;
    offs_l[NL] = run;
    meta[0] = run;
  }
  __syncthreads();
  // one warp per (j, s) pair writes its contiguous run
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int p = warp; p < NL * G; p += nw) {
    const int j = p / G, s = p % G;
    int dst = base[j];
    for (int s2 = 0; s2 < s; ++s2) dst += cnt[s2 * NL + j];
    int src = 0;
    for (int j2 = 0; j2 < j; ++j2) src += cnt[s * NL + j2];
    const int n = cnt[s * NL + j];
    for (int t = lane; t < n; t += 32) perm2[dst + t] = (int32_t)(s * cap + src + t);
  }
}

// Regroup the received rows into the grouped order (row count read on device).
__global__ void ep_regroup_kernel(const uint4* __restrict__ recv, const int32_t* __restrict__ perm2,
                                  const int32_t* __restrict__ meta, int d8, uint4* __restrict__ out) {
  DALI_PDL_ENTRY();
  const int64_t items = (int64_t)meta[0] * d8;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = it / d8;
    const int c = (int)(it - r * d8);
    out[r * d8 + c] = recv[(int64_t)perm2[r] * d8 + c];
  }
}

// Return: grouped row i (local expert j, source s, t) -> peer ret_s[rank][idx]
// with idx = sum_{j'<j} cnt[s][j'] + t; value = sum of the split-K planes for
// GPU experts, the host worker's row for CPU experts.
__global__ void ep_return_kernel(const float* __restrict__ yp, int splits, int64_t plane,
                                 const float* __restrict__ cpu_rows,
                                 const int8_t* __restrict__ gmask,
                                 const int32_t* __restrict__ offs_l,
                                 const int32_t* __restrict__ cnt, int G, int NL, int rank,
                                 int64_t cap, int d, const uint64_t* __restrict__ peer_ret,
                                 const uint64_t* __restrict__ peer_flag, unsigned int* done) {
  DALI_PDL_ENTRY();
  const int rows = offs_l[NL];
  const int d4 = d >> 2;
  const int64_t items = (int64_t)rows * d4;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(it / d4), c = (int)(it - (int64_t)i * d4);
    const int j = find_bucket(offs_l, NL, i);
    int t = i - offs_l[j], s = 0;
    while (t >= cnt[s * NL + j]) t -= cnt[s++ * NL + j];
    int idx = t;
    for (int j2 = 0; j2 < j; ++j2) idx += cnt[s * NL + j2];
    float4 v;
    if (!gmask || gmask[j]) {
      v = reinterpret_cast<const float4*>(yp + (int64_t)i * d)[c];
      for (int p = 1; p < splits; ++p) {       // planes in order, as the combine kernel
        const float4 w = reinterpret_cast<const float4*>(yp + p * plane + (int64_t)i * d)[c];
        v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
      }
    } else {
      v = reinterpret_cast<const float4*>(cpu_rows + (int64_t)i * d)[c];
    }
    reinterpret_cast<float4*>(peer_ret[s])[((int64_t)rank * cap + idx) * d4 + c] = v;
  }
  signal_peers(done, peer_flag, G);
}

// Source side: back[r] = ret[q][r - offsets[q*NL]] (q = owner of row r's expert).
__global__ void ep_gather_back_kernel(const float4* __restrict__ ret,
                                      const int32_t* __restrict__ offsets, int N, int NL,
                                      int64_t cap, int d4, float4* __restrict__ back) {
  DALI_PDL_ENTRY();
  const int rows = offsets[N];
  const int64_t items = (int64_t)rows * d4;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(it / d4), c = (int)(it - (int64_t)r * d4);
    const int q = find_bucket(offsets, N, r) / NL;
    back[(int64_t)r * d4 + c] = ret[((int64_t)q * cap + (r - offsets[q * NL])) * d4 + c];
  }
}

static unsigned int* done_counter(int which) {
  static unsigned int* p[kMaxDevices] = {};
  const int dev = current_device();
  if (!p[dev]) {
    cudaMalloc(&p[dev], 2 * sizeof(unsigned int));
    cudaMemset(p[dev], 0, 2 * sizeof(unsigned int));
  }
  return p[dev] + which;
}

static int ep_sm_count() { return device_sm_count(); }

static unsigned grid_for(int64_t items) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256,
                                                          (int64_t)ep_sm_count() * 4));
}

}  // namespace dali

using namespace dali;

extern "C" int dali_ipc_alloc(size_t bytes, void** ptr, void* handle) {
  DALI_REQUIRE(ptr && handle && bytes > 0, DALI_ECUDA, "bad ipc allocation request");
  cudaError_t e = cudaMalloc(ptr, bytes);
  DALI_REQUIRE(e == cudaSuccess, DALI_ECUDA, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
  cudaMemset(*ptr, 0, bytes);
  e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle), *ptr);
  DALI_REQUIRE(e == cudaSuccess, DALI_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  cudaDeviceSynchronize();
  return DALI_OK;
}

extern "C" int dali_ipc_open(const void* handle, void** ptr) {
  DALI_REQUIRE(ptr && handle, DALI_ECUDA, "bad ipc open request");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  DALI_REQUIRE(e == cudaSuccess, DALI_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  return DALI_OK;
}

extern "C" int dali_ipc_close(void* ptr) {
  if (ptr) cudaIpcCloseMemHandle(ptr);
  return DALI_OK;
}

extern "C" int dali_ipc_free(void* ptr) {
  if (ptr) cudaFree(ptr);
  return DALI_OK;
}

extern "C" int dali_ep_layout(int32_t G, int32_t NL, int64_t cap, int32_t d, int64_t* out) {
  DALI_REQUIRE(G >= 1 && NL >= 1 && cap >= 1 && d % 8 == 0, DALI_ESIM, "bad EP layout");
  const int64_t recv = (int64_t)G * cap * d * 2;
  const int64_t ret = (int64_t)G * cap * d * 4;
  const int64_t cnt = ((int64_t)G * NL * 4 + 255) / 256 * 256;
  out[0] = 0;                          // recv offset
  out[1] = recv;                       // ret offset
  out[2] = recv + ret;                 // cnt offset
  out[3] = recv + ret + cnt;           // flags offset (2 x u64)
  out[4] = out[3] + 256;               // total bytes
  return DALI_OK;
}

extern "C" int dali_ep_dispatch(const uint16_t* x, const int32_t* perm_token,
                                const int32_t* offsets, int32_t N, int32_t NL, int32_t G,
                                int32_t rank, int64_t cap, int32_t d, int64_t max_rows,
                                const uint64_t* peer_recv, const uint64_t* peer_cnt,
                                const uint64_t* peer_flag, void* stream) {
  DALI_REQUIRE(N == NL * G && d % 8 == 0, DALI_ESIM, "bad EP dispatch geometry");
  launch_pdl(ep_dispatch_kernel, dim3(grid_for(max_rows * (d / 8))), dim3(256), 0,
             as_stream(stream), reinterpret_cast<const uint4*>(x), perm_token, offsets, N, NL,
             G, rank, cap, d / 8, peer_recv, peer_cnt, peer_flag, done_counter(0));
  DALI_LAUNCH_CHECK("ep_dispatch_kernel");
  return DALI_OK;
}

extern "C" int dali_ep_wait(const uint64_t* flag, uint64_t target, int64_t max_spins,
                            int32_t* err, void* stream) {
  launch_pdl(ep_wait_kernel, dim3(1), dim3(32), 0, as_stream(stream),
             reinterpret_cast<const unsigned long long*>(flag), (unsigned long long)target,
             (long long)max_spins, err);
  DALI_LAUNCH_CHECK("ep_wait_kernel");
  return DALI_OK;
}

extern "C" int dali_ep_recv(const int32_t* cnt, int32_t G, int32_t NL, int64_t cap,
                            const uint16_t* recv, int32_t d, int64_t max_rows, int32_t* perm2,
                            int32_t* offs_l, int64_t* workloads, int32_t* meta, uint16_t* out,
                            void* stream) {
  DALI_REQUIRE(NL >= 1 && NL <= DALI_MAX_EXPERTS && d % 8 == 0, DALI_ESIM, "bad EP recv");
  cudaStream_t st = as_stream(stream);
  launch_pdl(ep_recv_plan_kernel, dim3(1), dim3(256), 0, st, cnt, G, NL, cap, perm2, offs_l,
             workloads, meta);
  DALI_LAUNCH_CHECK("ep_recv_plan_kernel");
  launch_pdl(ep_regroup_kernel, dim3(grid_for(max_rows * (d / 8))), dim3(256), 0, st,
             reinterpret_cast<const uint4*>(recv), perm2, meta, d / 8,
             reinterpret_cast<uint4*>(out));
  DALI_LAUNCH_CHECK("ep_regroup_kernel");
  return DALI_OK;
}

extern "C" int dali_ep_return(const float* yp, int32_t splits, int64_t plane,
                              const float* cpu_rows, const int8_t* gmask, const int32_t* offs_l,
                              const int32_t* cnt, int32_t G, int32_t NL, int32_t rank, int64_t cap,
                              int32_t d, int64_t max_rows, const uint64_t* peer_ret,
                              const uint64_t* peer_flag, void* stream) {
  DALI_REQUIRE(d % 4 == 0 && splits >= 1, DALI_ESIM, "bad EP return geometry");
  launch_pdl(ep_return_kernel, dim3(grid_for(max_rows * (d / 4))), dim3(256), 0,
             as_stream(stream), yp, splits, plane, cpu_rows, gmask, offs_l, cnt, G, NL, rank,
             cap, d, peer_ret, peer_flag, done_counter(1));
  DALI_LAUNCH_CHECK("ep_return_kernel");
  return DALI_OK;
}

extern "C" int dali_ep_gather_back(const float* ret, const int32_t* offsets, int32_t N,
                                   int32_t NL, int64_t cap, int32_t d, int64_t max_rows,
                                   float* back, void* stream) {
  DALI_REQUIRE(d % 4 == 0, DALI_ESIM, "bad EP gather geometry");
  launch_pdl(ep_gather_back_kernel, dim3(grid_for(max_rows * (d / 4))), dim3(256), 0,
             as_stream(stream), reinterpret_cast<const float4*>(ret), offsets, N, NL, cap, d / 4,
             reinterpret_cast<float4*>(back));
  DALI_LAUNCH_CHECK("ep_gather_back_kernel");
  return DALI_OK;
}
