// Host-side microbenchmark for the CPU expert worker (diagnostic, not part of
// libdali): streaming-read bandwidth vs thread count, and GEMV variants of the
// decode-regime expert (W13 then W2, bf16, AVX-512 BF16) over distinct blocks.
//
//   g++ -O3 -march=native -mavx512bf16 -pthread tools/cpu_expert_bench.cpp -o /tmp/ceb && /tmp/ceb
#include <immintrin.h>
#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

static void* alloc_touch(size_t bytes, int nth) {
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(p, bytes, MADV_HUGEPAGE);
  std::vector<std::thread> th;
  size_t chunk = (bytes + nth - 1) / nth;
  for (int t = 0; t < nth; ++t)
    th.emplace_back([=] {
      size_t a = t * chunk, b = std::min(bytes, a + chunk);
      for (size_t i = a; i < b; i += 64) ((uint8_t*)p)[i] = (uint8_t)(i * 7);
    });
  for (auto& x : th) x.join();
  return p;
}

template <class F>
static void par(int nth, F f) {
  std::vector<std::thread> th;
  for (int t = 1; t < nth; ++t) th.emplace_back([&, t] { f(t); });
  f(0);
  for (auto& x : th) x.join();
}

// variant 0: one accumulator chain per row (current libdali kernel)
static inline float dot0(const uint16_t* w, const uint16_t* x, int K) {
  __m512 a = _mm512_setzero_ps();
  for (int k = 0; k < K; k += 32)
    a = _mm512_dpbf16_ps(a, (__m512bh)_mm512_loadu_si512(w + k), (__m512bh)_mm512_loadu_si512(x + k));
  return _mm512_reduce_add_ps(a);
}
// variant 1: four independent chains
static inline float dot1(const uint16_t* w, const uint16_t* x, int K) {
  __m512 a0 = _mm512_setzero_ps(), a1 = a0, a2 = a0, a3 = a0;
  for (int k = 0; k < K; k += 128) {
    a0 = _mm512_dpbf16_ps(a0, (__m512bh)_mm512_loadu_si512(w + k), (__m512bh)_mm512_loadu_si512(x + k));
    a1 = _mm512_dpbf16_ps(a1, (__m512bh)_mm512_loadu_si512(w + k + 32), (__m512bh)_mm512_loadu_si512(x + k + 32));
    a2 = _mm512_dpbf16_ps(a2, (__m512bh)_mm512_loadu_si512(w + k + 64), (__m512bh)_mm512_loadu_si512(x + k + 64));
    a3 = _mm512_dpbf16_ps(a3, (__m512bh)_mm512_loadu_si512(w + k + 96), (__m512bh)_mm512_loadu_si512(x + k + 96));
  }
  return _mm512_reduce_add_ps(_mm512_add_ps(_mm512_add_ps(a0, a1), _mm512_add_ps(a2, a3)));
}
// variant 2: four chains + software prefetch PF bytes ahead
static int PF = 4096;
static int HINT = 0;
static inline float dot2(const uint16_t* w, const uint16_t* x, int K) {
  __m512 a0 = _mm512_setzero_ps(), a1 = a0, a2 = a0, a3 = a0;
  const int pf = PF;
  for (int k = 0; k < K; k += 128) {
    const char* q = (const char*)(w + k) + pf;
    if (HINT == 0) {
      _mm_prefetch(q, _MM_HINT_T0); _mm_prefetch(q + 64, _MM_HINT_T0);
      _mm_prefetch(q + 128, _MM_HINT_T0); _mm_prefetch(q + 192, _MM_HINT_T0);
    } else if (HINT == 1) {
      _mm_prefetch(q, _MM_HINT_NTA); _mm_prefetch(q + 64, _MM_HINT_NTA);
      _mm_prefetch(q + 128, _MM_HINT_NTA); _mm_prefetch(q + 192, _MM_HINT_NTA);
    } else {
      _mm_prefetch(q, _MM_HINT_T1); _mm_prefetch(q + 64, _MM_HINT_T1);
      _mm_prefetch(q + 128, _MM_HINT_T1); _mm_prefetch(q + 192, _MM_HINT_T1);
    }
    a0 = _mm512_dpbf16_ps(a0, (__m512bh)_mm512_loadu_si512(w + k), (__m512bh)_mm512_loadu_si512(x + k));
    a1 = _mm512_dpbf16_ps(a1, (__m512bh)_mm512_loadu_si512(w + k + 32), (__m512bh)_mm512_loadu_si512(x + k + 32));
    a2 = _mm512_dpbf16_ps(a2, (__m512bh)_mm512_loadu_si512(w + k + 64), (__m512bh)_mm512_loadu_si512(x + k + 64));
    a3 = _mm512_dpbf16_ps(a3, (__m512bh)_mm512_loadu_si512(w + k + 96), (__m512bh)_mm512_loadu_si512(x + k + 96));
  }
  return _mm512_reduce_add_ps(_mm512_add_ps(_mm512_add_ps(a0, a1), _mm512_add_ps(a2, a3)));
}

int main(int argc, char** argv) {
  const int d = 4096, f = 14336;
  const size_t blk = (size_t)3 * d * f * 2;
  const int nblk = 8;
  int hw = std::thread::hardware_concurrency();
  printf("hardware_concurrency %d\n", hw);
  int nth_max = hw;
  uint16_t* store = (uint16_t*)alloc_touch(blk * nblk, nth_max);
  // streaming read bandwidth
  for (int nth : {1, 2, 4, 8, 12, 16, 24, 32}) {
    if (nth > nth_max) break;
    double best = 1e9;
    for (int it = 0; it < 4; ++it) {
      const uint8_t* base = (const uint8_t*)store + (size_t)(it % nblk) * blk;
      std::vector<double> sink(nth * 8);
      double t0 = now();
      par(nth, [&](int t) {
        size_t a = blk * t / nth, b = blk * (t + 1) / nth;
        __m512i acc = _mm512_setzero_si512();
        for (size_t i = a; i < b; i += 64) acc = _mm512_xor_si512(acc, _mm512_load_si512(base + i));
        sink[t * 8] = (double)_mm512_reduce_add_epi64(acc);
      });
      best = std::min(best, now() - t0);
    }
    printf("read  nth=%2d  %.1f GB/s\n", nth, blk / best / 1e9);
  }
  std::vector<uint16_t> x(d, 0x3f80), h(f, 0x3f80);
  std::vector<float> y(d);
  struct Cfg { int var, pf, hint; };
  std::vector<Cfg> cfgs = {{0, 0, 0}, {1, 0, 0}, {2, 1024, 0}, {2, 2048, 0}, {2, 4096, 0},
                           {2, 8192, 0}, {2, 16384, 0}, {2, 4096, 1}, {2, 8192, 1},
                           {2, 4096, 2}, {2, 8192, 2}};
  for (auto c : cfgs) {
    const int var = c.var;
    PF = c.pf;
    HINT = c.hint;
    for (int nth : {16}) {
      if (nth > nth_max) break;
      std::vector<double> ts;
      for (int it = 0; it < 2 * nblk; ++it) {
        const uint16_t* b = store + (size_t)(it % nblk) * (blk / 2);
        const uint16_t* w13 = b;
        const uint16_t* w2 = b + (size_t)2 * f * d;
        double t0 = now();
        par(nth, [&](int t) {
          int r0 = (int)((int64_t)2 * f * t / nth), r1 = (int)((int64_t)2 * f * (t + 1) / nth);
          for (int r = r0; r < r1; ++r) {
            float v = var == 0 ? dot0(w13 + (size_t)r * d, x.data(), d)
                    : var == 1 ? dot1(w13 + (size_t)r * d, x.data(), d)
                               : dot2(w13 + (size_t)r * d, x.data(), d);
            if (r < f) h[r] = (uint16_t)(((uint32_t&)v) >> 16);
          }
        });
        par(nth, [&](int t) {
          int m0 = d * t / nth, m1 = d * (t + 1) / nth;
          for (int m = m0; m < m1; ++m)
            y[m] = var == 0 ? dot0(w2 + (size_t)m * f, h.data(), f)
                 : var == 1 ? dot1(w2 + (size_t)m * f, h.data(), f)
                            : dot2(w2 + (size_t)m * f, h.data(), f);
        });
        ts.push_back(now() - t0);
      }
      std::sort(ts.begin(), ts.end());
      printf("pf=%5d hint=%d ", PF, HINT);
      printf("expert var=%d nth=%2d  min %.3f ms  med %.3f ms  (%.1f GB/s at min)\n", var, nth,
             ts[0] * 1e3, ts[ts.size() / 2] * 1e3, blk / ts[0] / 1e9);
    }
  }
  return 0;
}
