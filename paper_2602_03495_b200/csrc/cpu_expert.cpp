// CPU expert worker (DALI hybrid execution: experts the greedy assignment
// puts on the CPU run on the host).  Native AVX-512 BF16 kernel for the
// decode regime (few tokens per expert), where the work is a weight-streaming
// GEMV bound by host DRAM bandwidth: one pass over the expert block
// [W13 (2f, d) | W2 (d, f)] bf16 per call, all rows of the token batch
// multiplied against each 64-byte weight chunk while it is in registers.
//
// Threads: a persistent pool partitions weight rows; phase 1 (W13, SwiGLU
// into a bf16 intermediate -- the same rounding point as the GPU kernel),
// barrier, phase 2 (W2 -> fp32 outputs).
#include <cpuid.h>
#include <immintrin.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/dali.h"

namespace dali {
void set_error(const char* fmt, ...);
}

namespace {

constexpr int kMaxRows = 16;

// The kernels below use AVX-512 BF16 (vdpbf16ps).  On a host without it the
// entry points return an error instead of dying on SIGILL.
bool cpu_ok() {
  static const bool ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                         __builtin_cpu_supports("avx512bf16");
  if (!ok) dali::set_error("CPU expert worker needs AVX-512 BF16 (avx512bf16) on this host");
  return ok;
}

inline float bf2f(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
inline uint16_t f2bf(float f) {  // round to nearest even
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

class Pool {
 public:
  explicit Pool(int n) : n_(n) {
    for (int i = 1; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_.store(true, std::memory_order_release);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return n_; }
  // run fn(tid) on every thread (caller is tid 0), return when all finished.
  // Workers spin briefly on the generation counter before sleeping, so the
  // two phases of an expert and back-to-back experts of a layer start without
  // a futex wake-up; the caller spins on the completion count.
  void run(const std::function<void(int)>& fn) {
    start(fn);
    join(fn);
  }
  // start: workers 1..n-1 begin fn(tid) and the caller returns at once;
  // join: the caller runs fn(0), then waits for the workers.  fn must stay
  // alive until join returns.
  void start(const std::function<void(int)>& fn) {
    fn_ = &fn;
    pending_.store(n_ - 1, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> g(m_);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
  }
  void join(const std::function<void(int)>& fn) {
    fn(0);
    while (pending_.load(std::memory_order_acquire) != 0) _mm_pause();
  }

 private:
  void loop(int tid) {
    uint64_t seen = 0;           // generation at construction (a run may precede this thread)
    for (;;) {
      uint64_t g = gen_.load(std::memory_order_acquire);
      for (int spin = 0; g == seen && spin < kSpin; ++spin) {
        _mm_pause();
        g = gen_.load(std::memory_order_acquire);
      }
      if (g == seen) {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
        g = gen_.load(std::memory_order_acquire);
      }
      seen = g;
      if (stop_.load(std::memory_order_acquire)) return;
      (*fn_)(tid);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  // pause iterations before a worker sleeps (DALI_POOL_SPIN, default 20000)
  const int kSpin = [] {
    const char* v = getenv("DALI_POOL_SPIN");
    return v ? atoi(v) : 20000;
  }();
  int n_;
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_;
  const std::function<void(int)>* fn_ = nullptr;
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> pending_{0};
  std::atomic<bool> stop_{false};
};

Pool* pool_for(int n) {
  static Pool* p = nullptr;
  static std::mutex m;
  std::lock_guard<std::mutex> g(m);
  if (!p || p->size() != n) {
    delete p;
    p = new Pool(n);
  }
  return p;
}

// Software prefetch distance for the weight stream: measured on the GPU
// box's host (tools/cpu_expert_bench.cpp) the hardware streamers alone leave
// ~10-15% of host DRAM bandwidth unused at 16 threads.
constexpr int kPrefetchBytes = 4096;

// dot of one weight row (K bf16) with R token rows (K bf16 each) -> R floats
inline void row_dot(const uint16_t* w, const uint16_t* x, int64_t ldx, int K, int R,
                    float* out) {
  if (R == 1) {
    // single token: four independent dpbf16 chains (one chain is latency-bound)
    __m512 a0 = _mm512_setzero_ps(), a1 = a0, a2 = a0, a3 = a0;
    int k = 0;
    for (; k + 128 <= K; k += 128) {
      const char* q = reinterpret_cast<const char*>(w + k) + kPrefetchBytes;
      _mm_prefetch(q, _MM_HINT_T0);
      _mm_prefetch(q + 64, _MM_HINT_T0);
      _mm_prefetch(q + 128, _MM_HINT_T0);
      _mm_prefetch(q + 192, _MM_HINT_T0);
      a0 = _mm512_dpbf16_ps(a0, (__m512bh)_mm512_loadu_si512(w + k),
                            (__m512bh)_mm512_loadu_si512(x + k));
      a1 = _mm512_dpbf16_ps(a1, (__m512bh)_mm512_loadu_si512(w + k + 32),
                            (__m512bh)_mm512_loadu_si512(x + k + 32));
      a2 = _mm512_dpbf16_ps(a2, (__m512bh)_mm512_loadu_si512(w + k + 64),
                            (__m512bh)_mm512_loadu_si512(x + k + 64));
      a3 = _mm512_dpbf16_ps(a3, (__m512bh)_mm512_loadu_si512(w + k + 96),
                            (__m512bh)_mm512_loadu_si512(x + k + 96));
    }
    for (; k < K; k += 32)
      a0 = _mm512_dpbf16_ps(a0, (__m512bh)_mm512_loadu_si512(w + k),
                            (__m512bh)_mm512_loadu_si512(x + k));
    out[0] = _mm512_reduce_add_ps(_mm512_add_ps(_mm512_add_ps(a0, a1), _mm512_add_ps(a2, a3)));
    return;
  }
  __m512 acc[kMaxRows];
  for (int r = 0; r < R; ++r) acc[r] = _mm512_setzero_ps();
  for (int k = 0; k < K; k += 32) {
    _mm_prefetch(reinterpret_cast<const char*>(w + k) + kPrefetchBytes, _MM_HINT_T0);
    const __m512bh wv = (__m512bh)_mm512_loadu_si512(w + k);
    for (int r = 0; r < R; ++r) {
      const __m512bh xv = (__m512bh)_mm512_loadu_si512(x + r * ldx + k);
      acc[r] = _mm512_dpbf16_ps(acc[r], wv, xv);
    }
  }
  for (int r = 0; r < R; ++r) out[r] = _mm512_reduce_add_ps(acc[r]);
}

// DALI_CPU_DYNAMIC=0 selects the static per-thread partition (A/B switch)
bool dynamic_chunks() {
  static const bool v = [] {
    const char* e = getenv("DALI_CPU_DYNAMIC");
    return !(e && e[0] == '0');
  }();
  return v;
}

bool async_job_busy();

// ---------------------------------------------------------------------------
// AMX-BF16 path for prefill-sized token batches (R > kMaxRows rows): the same
// SwiGLU with fp32 accumulators and fp32 outputs, rounding only the SwiGLU
// intermediate to bf16 -- the rounding points of the GPU tcgen05 kernel and
// of the AVX-512 decode kernel above, so a prefill row's numerics no longer
// depend on whether the policy placed its expert on the CPU or the GPU.
// Weights are the A operand straight from the block (16 rows x 32 k per
// tile, row stride d or f); tokens are the B operand, packed once per call
// into the VNNI layout xp[k/2][Tpad][2].  2 A x 2 B -> 4 accumulator tiles
// (gate/up rows x 32 tokens in phase 1, 32 W2 rows x 32 tokens in phase 2).
// The SwiGLU intermediate is written straight into the VNNI layout the down
// projection's B operand needs.  Work units (one per 32 weight rows) are
// handed out by an atomic counter like the decode kernel's.
// ---------------------------------------------------------------------------
struct alignas(64) TileCfg {
  uint8_t palette = 1, start_row = 0, reserved[14] = {};
  uint16_t colsb[16] = {};
  uint8_t rows[16] = {};
};

bool amx_ok() {
  static const bool ok = [] {
    const char* e = getenv("DALI_CPU_AMX");           // A/B switch: 0 = 16-row AVX passes
    if (e && e[0] == '0') return false;
    unsigned a, b, c, dx;
    if (!__get_cpuid_count(7, 0, &a, &b, &c, &dx)) return false;
    if (!((dx >> 22) & 1u) || !((dx >> 24) & 1u)) return false;     // AMX-BF16, AMX-TILE
    // Linux: the tile data state must be requested once per process
    return syscall(SYS_arch_prctl, 0x1023 /* ARCH_REQ_XCOMP_PERM */,
                   18 /* XFEATURE_XTILEDATA */) == 0;
  }();
  return ok;
}

void tile_config() {
  TileCfg c;
  for (int i = 0; i < 8; ++i) {
    c.colsb[i] = 64;
    c.rows[i] = 16;
  }
  _tile_loadconfig(&c);
}

// Same as amx_block over k in [k0, k1) with the accumulators carried in
// memory: loaded from c (or zeroed when first), stored back to c.  Splitting
// the k loop this way changes nothing numerically (tile store / load of fp32
// is exact, the dpbf16 sequence is the same).  pf: software-prefetch the
// weight rows kPfK elements ahead (the first pass over a weight chunk streams
// from DRAM as 32 interleaved row streams, more than the hardware prefetchers
// track).
inline int pf_k() {
  static const int v = getenv("DALI_AMX_PFK") ? atoi(getenv("DALI_AMX_PFK")) : 256;
  return v;
}
struct BgPf {
  const char* base[2] = {nullptr, nullptr};   // first rows of the two 16-row tiles
  int64_t ld = 0;                              // row stride, bytes
  int lines_per_row = 0, pos = 0, total = 0, per_step = 0;
  void set(const uint16_t* a0, const uint16_t* a1, int64_t lda, int k0, int k1, int steps) {
    base[0] = reinterpret_cast<const char*>(a0 + k0);
    base[1] = reinterpret_cast<const char*>(a1 + k0);
    ld = lda * 2;
    lines_per_row = (k1 - k0) * 2 / 64;
    pos = 0;
    total = 32 * lines_per_row;
    per_step = steps > 0 ? (total + steps - 1) / steps : 0;
  }
  void clear() { total = pos = per_step = 0; }
  inline void step() {
    for (int i = 0; i < per_step && pos < total; ++i, ++pos) {
      const int line = pos >> 5, row = pos & 31;     // k-major, as the next item reads them
      _mm_prefetch(base[row >> 4] + (row & 15) * ld + line * 64, _MM_HINT_T1);
    }
  }
};

inline void amx_block_acc(const uint16_t* a0, const uint16_t* a1, int64_t lda, const uint16_t* b,
                          int64_t tpad, int k0, int k1, float* c, bool first, bool pf,
                          BgPf* bg = nullptr) {
  if (first) {
    _tile_zero(0);
    _tile_zero(1);
    _tile_zero(2);
    _tile_zero(3);
  } else {
    _tile_loadd(0, c, 64);
    _tile_loadd(1, c + 256, 64);
    _tile_loadd(2, c + 512, 64);
    _tile_loadd(3, c + 768, 64);
  }
  const int pfk = pf_k();
  pf = pf && pfk > 0;
  for (int k = k0; k < k1; k += 32) {
    if (pf && k + pfk < k1) {
      for (int r = 0; r < 16; ++r) {
        _mm_prefetch(reinterpret_cast<const char*>(a0 + r * lda + k + pfk), _MM_HINT_T0);
        _mm_prefetch(reinterpret_cast<const char*>(a1 + r * lda + k + pfk), _MM_HINT_T0);
      }
    }
    _tile_loadd(4, a0 + k, (int)(lda * 2));
    _tile_loadd(5, a1 + k, (int)(lda * 2));
    const uint16_t* bk = b + (int64_t)(k / 2) * tpad * 2;
    _tile_loadd(6, bk, (int)(tpad * 4));
    _tile_loadd(7, bk + 32, (int)(tpad * 4));
    _tile_dpbf16ps(0, 4, 6);
    _tile_dpbf16ps(1, 4, 7);
    _tile_dpbf16ps(2, 5, 6);
    _tile_dpbf16ps(3, 5, 7);
    if (bg) bg->step();
  }
  _tile_stored(0, c, 64);
  _tile_stored(1, c + 256, 64);
  _tile_stored(2, c + 512, 64);
  _tile_stored(3, c + 768, 64);
}

// exp(x) for 16 lanes: 2^n * p(r), n = round(x log2 e), r = x - n ln 2 split
// in two parts, degree-6 polynomial (Cephes expf coefficients, ~1 ulp); x
// clamped to [-87.3, 88.3] (results 0 / ~2e38 at the ends, as silu needs)
inline __m512 exp16(__m512 x) {
  x = _mm512_max_ps(_mm512_min_ps(x, _mm512_set1_ps(88.3f)), _mm512_set1_ps(-87.3f));
  const __m512 n = _mm512_roundscale_ps(_mm512_mul_ps(x, _mm512_set1_ps(1.44269504088896341f)),
                                        _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
  __m512 r = _mm512_fnmadd_ps(n, _mm512_set1_ps(0.693359375f), x);
  r = _mm512_fnmadd_ps(n, _mm512_set1_ps(-2.12194440e-4f), r);
  __m512 p = _mm512_set1_ps(1.9875691500e-4f);
  p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(1.3981999507e-3f));
  p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(8.3334519073e-3f));
  p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(4.1665795894e-2f));
  p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(1.6666665459e-1f));
  p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(5.0000001201e-1f));
  p = _mm512_fmadd_ps(p, _mm512_mul_ps(r, r), _mm512_add_ps(r, _mm512_set1_ps(1.0f)));
  return _mm512_scalef_ps(p, n);
}
// silu(g) * u, fp32 (rounded to bf16 once by the caller)
inline __m512 swiglu16(__m512 g, __m512 u) {
  const __m512 den = _mm512_add_ps(_mm512_set1_ps(1.0f), exp16(_mm512_sub_ps(_mm512_setzero_ps(), g)));
  return _mm512_mul_ps(_mm512_div_ps(g, den), u);
}

// k chunk of the down projection: the fewest elements (multiple of 32,
// dividing f) per chunk such that the chunk of the SwiGLU intermediate for
// all tokens stays in a core's L2 (~1 MB budget of 2 MB)
inline int down_kchunk(int f, int64_t tpad) {
  int best = 32;
  for (int kc = 32; kc <= f; kc += 32)
    if (f % kc == 0 && (int64_t)kc * tpad * 2 <= (1 << 20)) best = kc;
  return best;
}

void amx_expert(const uint16_t* block, int d, int f, const uint16_t* x, int R, float* y,
                Pool* pool) {
  const int64_t tpad = (R + 31) / 32 * 32;
  const uint16_t* w13 = block;
  const uint16_t* w2 = block + (int64_t)2 * f * d;
  std::vector<uint16_t> xp((size_t)d * tpad), hp((size_t)f * tpad);
  // phase 0: pack tokens to VNNI (k-pair major), zero padding tokens
  std::atomic<int> next{0};
  constexpr int kPackK = 64;
  pool->run([&](int) {
    for (int c = next.fetch_add(1); c * kPackK < d; c = next.fetch_add(1)) {
      const int k0 = c * kPackK, k1 = std::min(d, k0 + kPackK);
      for (int k = k0; k < k1; k += 2) {
        uint32_t* row = reinterpret_cast<uint32_t*>(xp.data() + (int64_t)(k / 2) * tpad * 2);
        for (int t = 0; t < R; ++t)
          row[t] = *reinterpret_cast<const uint32_t*>(x + (int64_t)t * d + k);
        for (int64_t t = R; t < tpad; ++t) row[t] = 0;
      }
    }
  });
  // phase 1: gate/up (rows 128b + 16i and 128b + 64 + 16i) -> SwiGLU -> hp
  const int units1 = (f / 64) * 4;
  next.store(0);
  pool->run([&](int) {
    tile_config();
    alignas(64) float c[4 * 256];
    BgPf bg;
    auto rows1 = [&](int uu, const uint16_t*& g_, const uint16_t*& u_) {
      const int b = uu / 4, i = uu % 4;
      g_ = w13 + (int64_t)(128 * b + 16 * i) * d;
      u_ = w13 + (int64_t)(128 * b + 64 + 16 * i) * d;
    };
    int u = next.fetch_add(1);
    int un = u < units1 ? next.fetch_add(1) : units1;      // this thread's next unit
    for (; u < units1; u = un, un = u < units1 ? next.fetch_add(1) : units1) {
      const int b = u / 4, i = u % 4;
      const uint16_t *gr, *ur;
      rows1(u, gr, ur);
      if (un < units1 && tpad > 32) {
        const uint16_t *gn, *unx;
        rows1(un, gn, unx);
        bg.set(gn, unx, d, 0, d, (int)(tpad / 32 - 1) * (d / 32));
      } else {
        bg.clear();
      }
      for (int64_t t0 = 0; t0 < tpad; t0 += 32) {
        // the first token block streams this unit's 32 weight rows from DRAM
        // (L2 if the previous unit prefetched them); the later ones re-read
        // them from L2 and prefetch the next unit's rows meanwhile
        amx_block_acc(gr, ur, d, xp.data() + t0 * 2, tpad, 0, d, c, true, t0 == 0,
                      t0 == 0 ? nullptr : &bg);
        // SwiGLU of 16 tokens per vector, two adjacent columns interleaved
        // into one 64-byte row of the down projection's VNNI operand
        for (int r = 0; r < 16; r += 2) {
          const int col = 64 * b + 16 * i + r;
          uint32_t* hrow = reinterpret_cast<uint32_t*>(hp.data()) + (int64_t)(col / 2) * tpad;
          for (int jb = 0; jb < 32; jb += 16) {
            const int cg = jb ? 256 : 0, cu = jb ? 768 : 512;
            const __m512 h0 = swiglu16(_mm512_load_ps(c + cg + r * 16), _mm512_load_ps(c + cu + r * 16));
            const __m512 h1 =
                swiglu16(_mm512_load_ps(c + cg + (r + 1) * 16), _mm512_load_ps(c + cu + (r + 1) * 16));
            const __m512i lo = _mm512_cvtepu16_epi32((__m256i)_mm512_cvtneps_pbh(h0));
            const __m512i hi = _mm512_cvtepu16_epi32((__m256i)_mm512_cvtneps_pbh(h1));
            _mm512_storeu_si512(hrow + t0 + jb, _mm512_or_si512(lo, _mm512_slli_epi32(hi, 16)));
          }
        }
      }
    }
  });
  // phase 2: y[t, m] = h_t . W2_m, 32 W2 rows per unit, fp32 out.  The k loop
  // is cut into chunks whose slice of the SwiGLU intermediate (all tokens)
  // fits a core's L2, and work items run chunk-major, so each core reuses one
  // hp chunk across the units it takes instead of streaming the whole
  // intermediate (f x tokens, 3.7 MB at 128 tokens) once per 32 W2 rows.
  // Accumulators of unfinished units live in `part`; a unit's next chunk
  // waits (rarely: a full chunk of other items lies in between) until its
  // previous chunk is done.
  const int units2 = d / 32;
  const int kc = down_kchunk(f, tpad), nch = f / kc;
  const int64_t tblocks = tpad / 32;
  std::vector<float> part(nch > 1 ? (size_t)units2 * tblocks * 1024 : 0);
  std::unique_ptr<std::atomic<int>[]> chunks_done(new std::atomic<int>[units2]);
  for (int u = 0; u < units2; ++u) chunks_done[u].store(0, std::memory_order_relaxed);
  next.store(0);
  pool->run([&](int) {
    tile_config();
    alignas(64) float c[4 * 256];
    BgPf bg;
    const int items = units2 * nch;
    int it = next.fetch_add(1);
    int itn = it < items ? next.fetch_add(1) : items;
    for (; it < items; it = itn, itn = it < items ? next.fetch_add(1) : items) {
      const int ch = it / units2, u = it - ch * units2;
      const int m0 = 32 * u;
      if (itn < items && tpad > 32) {
        const int chn = itn / units2, mn = 32 * (itn - chn * units2);
        bg.set(w2 + (int64_t)mn * f, w2 + (int64_t)(mn + 16) * f, f, chn * kc, (chn + 1) * kc,
               (int)(tblocks - 1) * (kc / 32));
      } else {
        bg.clear();
      }
      while (chunks_done[u].load(std::memory_order_acquire) < ch) _mm_pause();
      for (int64_t t0 = 0; t0 < tpad; t0 += 32) {
        float* acc = nch > 1 ? part.data() + ((size_t)u * tblocks + t0 / 32) * 1024 : c;
        amx_block_acc(w2 + (int64_t)m0 * f, w2 + (int64_t)(m0 + 16) * f, f, hp.data() + t0 * 2,
                      tpad, ch * kc, (ch + 1) * kc, acc, ch == 0, t0 == 0,
                      t0 == 0 ? nullptr : &bg);
        if (ch + 1 < nch) continue;
        if (acc != c) std::copy(acc, acc + 1024, c);
        for (int j = 0; j < 32 && t0 + j < R; ++j) {
          float* yr = y + (t0 + j) * (int64_t)d + m0;
          for (int r = 0; r < 16; ++r) {
            yr[r] = c[(j < 16 ? 0 : 256) + r * 16 + (j & 15)];
            yr[16 + r] = c[(j < 16 ? 512 : 768) + r * 16 + (j & 15)];
          }
        }
      }
      chunks_done[u].store(ch + 1, std::memory_order_release);
    }
  });
}

}  // namespace

extern "C" int dali_cpu_expert_amx_available(void) { return amx_ok() ? 1 : 0; }

extern "C" int dali_cpu_expert(const uint16_t* block, int32_t d, int32_t f, const uint16_t* x,
                               int32_t R, float* y, int32_t nthreads) {
  if (!block || !x || !y || d % 32 || f % 64 || R < 0) return DALI_ETRACE;
  if (R == 0) return DALI_OK;
  if (!cpu_ok()) return DALI_ESIM;
  if (async_job_busy()) return DALI_ESIM;           // the pool is running a submitted job
  if (R > kMaxRows && amx_ok()) {
    amx_expert(block, d, f, x, R, y, pool_for(nthreads < 1 ? 1 : nthreads));
    return DALI_OK;
  }
  if (R > kMaxRows) {
    for (int r0 = 0; r0 < R; r0 += kMaxRows) {
      const int n = R - r0 < kMaxRows ? R - r0 : kMaxRows;
      int rc = dali_cpu_expert(block, d, f, x + (int64_t)r0 * d, n, y + (int64_t)r0 * d, nthreads);
      if (rc) return rc;
    }
    return DALI_OK;
  }
  if (nthreads < 1) nthreads = 1;
  Pool* pool = pool_for(nthreads);
  const uint16_t* w13 = block;
  const uint16_t* w2 = block + (int64_t)2 * f * d;
  std::vector<uint16_t> hbuf((size_t)R * f);           // SwiGLU intermediate, bf16
  const int groups = f / 64;
  auto group = [&](int b) {
    float gv[kMaxRows], uv[kMaxRows];
    for (int i = 0; i < 64; ++i) {
      row_dot(w13 + (int64_t)(128 * b + i) * d, x, d, d, R, gv);
      row_dot(w13 + (int64_t)(128 * b + 64 + i) * d, x, d, d, R, uv);
      for (int r = 0; r < R; ++r) {
        const float g = gv[r];
        hbuf[(size_t)r * f + 64 * b + i] = f2bf(g / (1.0f + std::exp(-g)) * uv[r]);
      }
    }
  };
  auto down_rows = [&](int m0, int m1) {
    float acc[kMaxRows];
    for (int m = m0; m < m1; ++m) {
      row_dot(w2 + (int64_t)m * f, hbuf.data(), f, f, R, acc);
      for (int r = 0; r < R; ++r) y[(int64_t)r * d + m] = acc[r];
    }
  };
  if (dynamic_chunks()) {
    // ~1 MB units handed out by an atomic counter: a vCPU the hypervisor
    // preempts (or the caller's own thread) delays only the units it holds
    constexpr int kDownRows = 32;
    std::atomic<int> next_g{0}, next_m{0};
    pool->run([&](int) {
      for (int b = next_g.fetch_add(1, std::memory_order_relaxed); b < groups;
           b = next_g.fetch_add(1, std::memory_order_relaxed))
        group(b);
    });
    pool->run([&](int) {
      for (int c = next_m.fetch_add(1, std::memory_order_relaxed); c * kDownRows < d;
           c = next_m.fetch_add(1, std::memory_order_relaxed))
        down_rows(c * kDownRows, std::min(d, (c + 1) * kDownRows));
    });
    return DALI_OK;
  }
  // static partition: phase 1 group b = rows [128b, 128b+64) gate +
  // [128b+64, 128b+128) up; phase 2 y[r, m] = h_r . W2_m
  pool->run([&](int tid) {
    const int g0 = (int)((int64_t)groups * tid / nthreads);
    const int g1 = (int)((int64_t)groups * (tid + 1) / nthreads);
    for (int b = g0; b < g1; ++b) group(b);
  });
  pool->run([&](int tid) {
    down_rows((int)((int64_t)d * tid / nthreads), (int)((int64_t)d * (tid + 1) / nthreads));
  });
  return DALI_OK;
}

// ---------------------------------------------------------------------------
// Asynchronous submission.  dali_cpu_expert_submit starts a layer's CPU
// experts on the pool's worker threads and returns; the caller (the engine's
// Python thread) dispatches the GPU side of the layer meanwhile and then
// joins in dali_cpu_expert_wait, taking whatever work units are left.  The
// job is a queue of stages -- every expert's gate/up stage first, then every
// expert's down stage -- each split into ~1 MB units handed out by an
// atomic counter.  A down stage waits only for its own expert's gate/up
// stage, so the only barrier a layer pays is at the last expert's gate/up
// tail, and a thread that joins late simply starts at the current stage.
// One job in flight.
// ---------------------------------------------------------------------------
namespace {
constexpr int kDownRows = 32;
constexpr int kUpCols = 64;                         // SwiGLU columns per gate/up unit

struct Stage {
  int expert = 0, down = 0, units = 0, dep = -1;   // dep: stage that must finish first
  std::atomic<int> next{0}, done{0};
};

struct StageJob {
  int d = 0, f = 0, n_stages = 0;
  std::vector<const uint16_t*> blocks, xs;
  std::vector<int32_t> rows;
  std::vector<float*> ys;
  std::vector<std::vector<uint16_t>> hbuf;     // per expert: SwiGLU intermediate
  std::unique_ptr<Stage[]> stages;
  std::function<void(int)> fn;
  Pool* pool = nullptr;
  bool busy = false;
  // completion word: the thread that finishes the job's last unit stores
  // flag_value there (release), for a device kernel polling it over UVA (the
  // decode layer's combine, launched before the join)
  std::atomic<int> left{0};
  uint64_t* flag = nullptr;
  uint64_t flag_value = 0;

  void unit(const Stage& st, int u) {
    const int e = st.expert, R = rows[e];
    const uint16_t* w13 = blocks[e];
    const uint16_t* w2 = blocks[e] + (int64_t)2 * f * d;
    uint16_t* h = hbuf[e].data();
    float a[kMaxRows], b[kMaxRows];
    if (!st.down) {                                 // SwiGLU columns [64u, 64u+64)
      const int g = u / (64 / kUpCols), c0 = (u % (64 / kUpCols)) * kUpCols;
      for (int i = c0; i < c0 + kUpCols; ++i) {
        row_dot(w13 + (int64_t)(128 * g + i) * d, xs[e], d, d, R, a);
        row_dot(w13 + (int64_t)(128 * g + 64 + i) * d, xs[e], d, d, R, b);
        for (int r = 0; r < R; ++r)
          h[(size_t)r * f + 64 * g + i] = f2bf(a[r] / (1.0f + std::exp(-a[r])) * b[r]);
      }
    } else {                                        // down rows [32u, 32u+32)
      const int m1 = std::min(d, (u + 1) * kDownRows);
      for (int m = u * kDownRows; m < m1; ++m) {
        row_dot(w2 + (int64_t)m * f, h, f, f, R, a);
        for (int r = 0; r < R; ++r) ys[e][(int64_t)r * d + m] = a[r];
      }
    }
  }
  void work() {
    for (int s = 0; s < n_stages; ++s) {
      Stage& st = stages[s];
      if (st.dep >= 0) {
        const Stage& pv = stages[st.dep];
        while (pv.done.load(std::memory_order_acquire) < pv.units) _mm_pause();
      }
      for (int u = st.next.fetch_add(1, std::memory_order_relaxed); u < st.units;
           u = st.next.fetch_add(1, std::memory_order_relaxed)) {
        unit(st, u);
        st.done.fetch_add(1, std::memory_order_release);
        if (left.fetch_sub(1, std::memory_order_acq_rel) == 1 && flag)
          __atomic_store_n(flag, flag_value, __ATOMIC_RELEASE);
      }
    }
  }
};

StageJob& stage_job() {
  static StageJob j;
  return j;
}
bool async_job_busy() { return stage_job().busy; }
}  // namespace

static int submit_job(int32_t n, const uint64_t* blocks, const uint64_t* xs, const int32_t* rows,
                      const uint64_t* ys, int32_t d, int32_t f, int32_t nthreads, uint64_t* flag,
                      uint64_t flag_value);

extern "C" int dali_cpu_expert_submit(int32_t n, const uint64_t* blocks, const uint64_t* xs,
                                      const int32_t* rows, const uint64_t* ys, int32_t d,
                                      int32_t f, int32_t nthreads) {
  return submit_job(n, blocks, xs, rows, ys, d, f, nthreads, nullptr, 0);
}

extern "C" int dali_cpu_submit_layer(const int8_t* C, const int32_t* offsets, int32_t N,
                                     const uint64_t* blocks, const uint16_t* xp, float* out,
                                     int32_t d, int32_t f, int32_t nthreads, uint64_t* done_flag,
                                     uint64_t done_value, int32_t* n_experts) {
  if (!C || !offsets || !blocks || !xp || !out || !n_experts || N < 1 || N > 4096)
    return DALI_ETRACE;
  uint64_t bl[256], xs[256], ys[256];
  int32_t rows[256];
  int n = 0;
  for (int e = 0; e < N; ++e) {
    const int r0 = offsets[e], r1 = offsets[e + 1];
    if (!C[e] || r1 <= r0) continue;
    if (r1 - r0 > kMaxRows || n == 256) {           // prefill-sized: the caller's AMX path
      *n_experts = -1;
      return DALI_OK;
    }
    bl[n] = blocks[e];
    xs[n] = reinterpret_cast<uint64_t>(xp + (int64_t)r0 * d);
    ys[n] = reinterpret_cast<uint64_t>(out + (int64_t)r0 * d);
    rows[n] = r1 - r0;
    ++n;
  }
  *n_experts = n;
  return submit_job(n, bl, xs, rows, ys, d, f, nthreads, done_flag, done_value);
}

static int submit_job(int32_t n, const uint64_t* blocks, const uint64_t* xs, const int32_t* rows,
                      const uint64_t* ys, int32_t d, int32_t f, int32_t nthreads, uint64_t* flag,
                      uint64_t flag_value) {
  if (n < 0 || (n > 0 && (!blocks || !xs || !rows || !ys)) || d % 32 || f % 64)
    return DALI_ETRACE;
  if (n > 0 && !cpu_ok()) return DALI_ESIM;
  StageJob& j = stage_job();
  if (j.busy) return DALI_ESIM;                     // previous job not joined
  for (int i = 0; i < n; ++i)
    if (rows[i] < 0 || rows[i] > kMaxRows) return DALI_ETRACE;
  j.d = d;
  j.f = f;
  j.blocks.assign(n, nullptr);
  j.xs.assign(n, nullptr);
  j.ys.assign(n, nullptr);
  j.rows.assign(rows, rows + n);
  j.hbuf.resize(n);
  j.n_stages = 2 * n;
  j.stages.reset(new Stage[std::max(1, 2 * n)]);
  for (int i = 0; i < n; ++i) {
    j.blocks[i] = reinterpret_cast<const uint16_t*>(blocks[i]);
    j.xs[i] = reinterpret_cast<const uint16_t*>(xs[i]);
    j.ys[i] = reinterpret_cast<float*>(ys[i]);
    j.hbuf[i].resize((size_t)std::max(rows[i], 1) * f);
    Stage& up = j.stages[i];
    up.expert = i;
    up.down = 0;
    up.units = rows[i] > 0 ? f / kUpCols : 0;
    Stage& dn = j.stages[n + i];
    dn.expert = i;
    dn.down = 1;
    dn.dep = i;
    dn.units = rows[i] > 0 ? (d + kDownRows - 1) / kDownRows : 0;
  }
  int total = 0;
  for (int i = 0; i < 2 * n; ++i) total += j.stages[i].units;
  j.flag = flag;
  j.flag_value = flag_value;
  j.left.store(total, std::memory_order_relaxed);
  if (total == 0) {                                 // nothing to run, nothing to join
    if (flag) __atomic_store_n(flag, flag_value, __ATOMIC_RELEASE);
    return DALI_OK;
  }
  j.pool = pool_for(nthreads < 1 ? 1 : nthreads);
  j.fn = [&j](int) { j.work(); };
  j.busy = true;
  j.pool->start(j.fn);
  return DALI_OK;
}

extern "C" int dali_cpu_expert_wait(void) {
  StageJob& j = stage_job();
  if (!j.busy) return DALI_OK;
  j.pool->join(j.fn);
  j.busy = false;
  return DALI_OK;
}
