// (5) Grouped SwiGLU expert FFN on the 5th-gen tensor cores (sm_100a).
//
// Two grouped GEMMs per launch set, both "swap-AB": the expert weights are
// the UMMA A operand (M = weight rows, 128 per tile), the permuted tokens of
// that expert are B (N = BN token columns, padded), K is contiguous in both
// (K-major, 128-byte swizzle).  Operands are staged by TMA into a
// STAGES-deep shared-memory ring (full/empty mbarriers); one elected thread
// issues tcgen05.mma (kind::f16, bf16 in, fp32 accumulate in TMEM); the
// accumulator is read back with tcgen05.ld for a fused epilogue:
//
//   up   : D = W13_tile . Xp^T     -> rows 0-63 gate, 64-127 up of the same
//          64 SwiGLU columns (block layout, see moe.cu) -> H = silu(g) * u
//   down : D = W2_tile . H^T       -> Y (fp32), optionally split-K into
//          `splits` partial planes summed in fixed order by the combine.
//
// Per-expert weight tensor maps live in global memory (built once per HBM
// slot by dali_expert_maps); the activation maps are built per launch.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace dali {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;                      // 64 bf16 = 128 B = one swizzle row
constexpr int kThreads = 128;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int x,
                                            int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(su32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
// K-major, 128-byte swizzle UMMA shared-memory descriptor (tile base 1024-B aligned):
// start>>4 | LBO=1 | SBO=1024 B (8 rows x 128 B) | version 1 | SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: F32 accumulate, BF16 A/B, K-major A/B.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                     uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <int BN>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  // BN <= 32 (decode weight streaming): 5 stages = 90-100 KB, so two CTAs
  // still share an SM (measured: 4 -> 5 stages +2% at every decode shape, 6
  // stages drops to one CTA per SM and loses 12%); BN 64: 4 stages; BN 128:
  // one CTA per SM with a deeper ring; BN 256: 4 x 48 KB.
#ifndef DALI_FFN_STAGES_SMALL
#define DALI_FFN_STAGES_SMALL 5
#endif
  static constexpr int STAGES = BN == 128 ? 6 : BN <= 32 ? DALI_FFN_STAGES_SMALL : 4;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr size_t BYTES =
      (size_t)STAGES * (A_BYTES + B_BYTES) + 64 * 17 * 4 + 1024 /*align*/ + 256 /*bars*/;
};

struct Tile {
  int e, m_tile, row0, n_valid, split;
};

// Locate this CTA's (expert, m-tile, n-tile, split) from the per-expert row
// offsets; experts whose map is 0 (not on the GPU) contribute no tiles.
// Order within an expert: split, then token tile, then weight tile, so the
// token tiles that share one weight tile run on neighbouring CTAs at the same
// time and the weight tile comes from DRAM once (L2 serves the others).
template <int BN>
__device__ bool find_tile(const int32_t* offs, const uint64_t* maps, int N, int m_tiles,
                          int splits, Tile& t, int idx) {
  for (int e = 0; e < N; ++e) {
    if (!maps[e]) continue;
    const int ne = offs[e + 1] - offs[e];
    if (ne <= 0) continue;
    const int n_tiles_e = (ne + BN - 1) / BN;
    const int cnt = n_tiles_e * m_tiles * splits;
    if (idx < cnt) {
      t.e = e;
      t.split = idx % splits;
      idx /= splits;
      const int nt = idx % n_tiles_e;
      t.m_tile = idx / n_tiles_e;
      t.row0 = offs[e] + nt * BN;
      t.n_valid = min(BN, ne - nt * BN);
      return true;
    }
    idx -= cnt;
  }
  return false;
}

// MODE 0 = up (SwiGLU epilogue into H), MODE 1 = down (fp32 into Y planes).
template <int BN, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
ffn_tc_kernel(const __grid_constant__ CUtensorMap b_map, const int32_t* __restrict__ offs,
              const uint64_t* __restrict__ a_maps, int N, int K, int m_tiles, int splits,
              int out_ld, uint16_t* __restrict__ H, float* __restrict__ Y, int64_t y_plane) {
  using S = Smem<BN>;
  // the up projection is PDL-launched behind the routing / plan kernels: its
  // tile list (offsets, expert maps) is only valid after the wait
  if (MODE == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
  Tile t;
  if (!find_tile<BN>(offs, a_maps, N, m_tiles, splits, t, blockIdx.x)) return;
  const void* a_map = reinterpret_cast<const void*>(a_maps[t.e] + (MODE == 0 ? 0 : 128));
  // Early PDL trigger: the tile list is final once the wait above returned, so
  // the down projection may launch now; its CTAs take the SM slots this
  // grid's CTAs leave and start streaming W2 (which does not depend on H)
  // while the last up tiles drain.  The down kernel's own griddepcontrol.wait
  // still orders every read of H after this grid completes.
  if (MODE == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + S::STAGES * S::A_BYTES;
  float* sU = reinterpret_cast<float*>(sB + S::STAGES * S::B_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(sU + 64 * 17);
  uint64_t* empty = full + S::STAGES;
  uint64_t* tfull = empty + S::STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb_total = K / BK;
  const int nk = kb_total / splits;
  const int kb0 = t.split * nk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S::STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tma_prefetch_desc(a_map);
    tma_prefetch_desc(&b_map);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tslot)),
                 "r"(S::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  // down: the first ring's worth of weight tiles (A) is independent of the up
  // projection, so it is requested before the PDL wait
  const int pre = MODE == 1 ? min(nk, S::STAGES) : 0;
  if (MODE == 1 && warp == 0 && lane == 0) {
    for (int i = 0; i < pre; ++i) {
      mbar_expect_tx(full + i, S::A_BYTES + S::B_BYTES);
      tma_load_2d(sA + i * S::A_BYTES, a_map, full + i, (kb0 + i) * BK, t.m_tile * BM);
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");     // PDL (no-op without it)

  if (warp == 0 && lane == 0) {
    // ---- TMA producer
    for (int i = 0; i < nk; ++i) {
      const int s = i % S::STAGES;
      const uint32_t ph = (i / S::STAGES) & 1;
      const int kx = (kb0 + i) * BK;
      if (i >= pre) {
        mbar_wait(empty + s, ph ^ 1);
        mbar_expect_tx(full + s, S::A_BYTES + S::B_BYTES);
        tma_load_2d(sA + s * S::A_BYTES, a_map, full + s, kx, t.m_tile * BM);
      }
      tma_load_2d(sB + s * S::B_BYTES, &b_map, full + s, kx, t.row0);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer
    constexpr uint32_t idesc = idesc_bf16(BM, BN < 16 ? 16 : BN);
    for (int i = 0; i < nk; ++i) {
      const int s = i % S::STAGES;
      const uint32_t ph = (i / S::STAGES) & 1;
      mbar_wait(full + s, ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t da = sw128_desc(su32(sA + s * S::A_BYTES));
      const uint64_t db = sw128_desc(su32(sB + s * S::B_BYTES));
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk)   // UMMA_K = 16 bf16 = 32 B -> +2 in desc units
        umma(tmem, da + 2 * kk, db + 2 * kk, idesc, (i | kk) != 0);
      umma_commit(empty + s);
    }
    umma_commit(tfull);
  }
  __syncwarp();

  // ---- epilogue: all 4 warps; warp w owns TMEM lanes [32w, 32w+32)
  mbar_wait(tfull, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int r = threadIdx.x;                       // accumulator row (TMEM lane)
  const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
  for (int c0 = 0; c0 < BN; c0 += 16) {
    float v[16];
    tmem_ld16(lane_addr + c0, v);
    if (MODE == 0) {
      if (r >= 64) {
#pragma unroll
        for (int i = 0; i < 16; ++i) sU[(r - 64) * 17 + i] = v[i];
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (r < 64) {
        const int j = t.m_tile * 64 + r;           // SwiGLU column
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int c = c0 + i;
          if (c < t.n_valid) {
            const float g = v[i], u = sU[r * 17 + i];
            const float hval = g / (1.0f + __expf(-g)) * u;
            H[(int64_t)(t.row0 + c) * out_ld + j] = f32_to_bf16_bits(hval);
          }
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    } else {
      const int m = t.m_tile * BM + r;
      float* y = Y + (int64_t)t.split * y_plane;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int c = c0 + i;
        if (c < t.n_valid) y[(int64_t)(t.row0 + c) * out_ld + m] = v[i];
      }
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(S::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// Persistent warp-specialized variant for wide token tiles (prefill): one CTA
// per SM loops over tiles; warp 0 = TMA producer, warp 1 = MMA issuer (owns
// TMEM), warps 2-5 = epilogue.  Two TMEM accumulator stages (tfull/tempty
// mbarriers) let the epilogue of tile i drain while tile i+1 accumulates.
// ---------------------------------------------------------------------------
constexpr int kPThreads = 192;

template <int BN>
struct PSmem {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGES = BN >= 256 ? 4 : 6;
  static constexpr int ACC_COLS = BN < 32 ? 32 : BN;      // one accumulator stage
  static constexpr int TMEM_COLS = 2 * ACC_COLS;          // <= 512
  static constexpr size_t BYTES =
      (size_t)STAGES * (A_BYTES + B_BYTES) + 2 * 64 * 17 * 4 + 1024 + 512;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}

// SwiGLU epilogue of one 16-column accumulator chunk for wide token tiles:
// rows 0-63 of the 128-row tile are gate, 64-127 up (block layout).  Both
// halves go through shared memory so that all 128 epilogue threads finish 8
// (SwiGLU column, token) outputs each -- half the per-thread exp/mul work of
// letting the 64 gate-row threads do it alone.  r = this thread's accumulator
// row (0..127, a permutation of the epilogue threads).
__device__ __forceinline__ void swiglu_chunk(const float (&v)[16], int r, float* sG, float* sU,
                                             int c0, int n_valid, int m_tile, int row0,
                                             int out_ld, uint16_t* __restrict__ H) {
  float* dst = r < 64 ? sG + r * 17 : sU + (r - 64) * 17;
#pragma unroll
  for (int i = 0; i < 16; ++i) dst[i] = v[i];
  asm volatile("bar.sync 1, 128;" ::: "memory");
  const int j = r & 63, h = r >> 6;
  const int col = m_tile * 64 + j;
#pragma unroll
  for (int i = 8 * h; i < 8 * h + 8; ++i) {
    const int c = c0 + i;
    if (c < n_valid) {
      const float g = sG[j * 17 + i], u = sU[j * 17 + i];
      H[(int64_t)(row0 + c) * out_ld + col] = f32_to_bf16_bits(g / (1.0f + __expf(-g)) * u);
    }
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

template <int BN>
__device__ int count_tiles(const int32_t* offs, const uint64_t* maps, int N, int m_tiles,
                           int splits) {
  int n = 0;
  for (int e = 0; e < N; ++e) {
    if (!maps[e]) continue;
    const int ne = offs[e + 1] - offs[e];
    if (ne > 0) n += ((ne + BN - 1) / BN) * m_tiles * splits;
  }
  return n;
}

template <int BN, int MODE>
__global__ void __launch_bounds__(kPThreads, 1)
ffn_tc_persistent(const __grid_constant__ CUtensorMap b_map, const int32_t* __restrict__ offs,
                  const uint64_t* __restrict__ a_maps, int N, int K, int m_tiles, int splits,
                  int out_ld, uint16_t* __restrict__ H, float* __restrict__ Y, int64_t y_plane) {
  using S = PSmem<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + S::STAGES * S::A_BYTES;
  float* sU = reinterpret_cast<float*>(sB + S::STAGES * S::B_BYTES);
  float* sG = sU + 64 * 17;
  uint64_t* full = reinterpret_cast<uint64_t*>(sG + 64 * 17);
  uint64_t* empty = full + S::STAGES;
  uint64_t* tfull = empty + S::STAGES;      // [2]
  uint64_t* tempty = tfull + 2;             // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (K / BK) / splits;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S::STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tma_prefetch_desc(&b_map);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tslot)),
                 "r"(S::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  // PDL: everything above overlapped the previous kernel's tail
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int n_tiles = count_tiles<BN>(offs, a_maps, N, m_tiles, splits);

  if (warp == 0) {
    if (lane == 0) {                                  // ---- TMA producer
      uint32_t it = 0;
      for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
        Tile t;
        find_tile<BN>(offs, a_maps, N, m_tiles, splits, t, ti);
        const void* a_map = reinterpret_cast<const void*>(a_maps[t.e] + (MODE == 0 ? 0 : 128));
        const int kb0 = t.split * nk;
        for (int i = 0; i < nk; ++i, ++it) {
          const int s = it % S::STAGES;
          const uint32_t ph = (it / S::STAGES) & 1;
          mbar_wait(empty + s, ph ^ 1);
          mbar_expect_tx(full + s, S::A_BYTES + S::B_BYTES);
          const int kx = (kb0 + i) * BK;
          tma_load_2d(sA + s * S::A_BYTES, a_map, full + s, kx, t.m_tile * BM);
          tma_load_2d(sB + s * S::B_BYTES, &b_map, full + s, kx, t.row0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {                                  // ---- MMA issuer
      constexpr uint32_t idesc = idesc_bf16(BM, BN < 16 ? 16 : BN);
      uint32_t it = 0, tc = 0;
      for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x, ++tc) {
        const int acc = tc & 1;
        const uint32_t aph = (tc >> 1) & 1;
        mbar_wait(tempty + acc, aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * S::ACC_COLS;
        for (int i = 0; i < nk; ++i, ++it) {
          const int s = it % S::STAGES;
          const uint32_t ph = (it / S::STAGES) & 1;
          mbar_wait(full + s, ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = sw128_desc(su32(sA + s * S::A_BYTES));
          const uint64_t db = sw128_desc(su32(sB + s * S::B_BYTES));
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma(d, da + 2 * kk, db + 2 * kk, idesc, (i | kk) != 0);
          umma_commit(empty + s);
        }
        umma_commit(tfull + acc);
      }
    }
  } else {                                            // ---- epilogue (warps 2-5)
    const int q = warp & 3;                           // TMEM lane quarter of this warp
    const int r = q * 32 + lane;                      // accumulator row
    uint32_t tc = 0;
    for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x, ++tc) {
      Tile t;
      find_tile<BN>(offs, a_maps, N, m_tiles, splits, t, ti);
      const int acc = tc & 1;
      const uint32_t aph = (tc >> 1) & 1;
      mbar_wait(tfull + acc, aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t lane_addr = tmem + acc * S::ACC_COLS + ((uint32_t)(q * 32) << 16);
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(lane_addr + c0, v);
        if (MODE == 0) {
          swiglu_chunk(v, r, sG, sU, c0, t.n_valid, t.m_tile, t.row0, out_ld, H);
        } else {
          const int m = t.m_tile * BM + r;
          float* y = Y + (int64_t)t.split * y_plane;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int c = c0 + i;
            if (c < t.n_valid) y[(int64_t)(t.row0 + c) * out_ld + m] = v[i];
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(tempty + acc);
    }
  }
  // let a dependent (PDL) grid start its prologue while we drain
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(S::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// CTA-pair variant for wide token tiles (tensor-bound prefill): a cluster of
// two CTAs on one TPC issues tcgen05.mma.cta_group::2 with M = 256.  Each CTA
// stages its own 128 weight rows (A) and HALF of the BN token columns (B) per
// k-block, so every SM moves 32 KB instead of 48 KB of operands per k-block
// for the same MMA work; each CTA's TMEM holds its 128 rows x all BN columns,
// so the epilogue is the single-CTA one.  Protocol (rank 0 = leader):
//   * both CTAs' TMA loads complete_tx on the LEADER's full[s] (2-SM TMA form);
//     only the leader arrives (expect_tx = both CTAs' bytes);
//   * the leader's single thread issues the MMAs; tcgen05.commit multicasts
//     to empty[s] / tfull[acc] of both CTAs;
//   * both CTAs' epilogue warps arrive on the leader's tempty[acc] (8
//     arrivals: 4 local + 4 remote) before the leader reuses the accumulator.
// ---------------------------------------------------------------------------
template <int BN>
struct PairSmem {
  static constexpr int A_BYTES = BM * BK * 2;            // this CTA's 128 weight rows
  static constexpr int B_BYTES = (BN / 2) * BK * 2;      // this CTA's half of the tokens
  static constexpr int STAGES = 6;
  static constexpr int TMEM_COLS = 2 * BN;               // two accumulator stages
  static constexpr size_t BYTES =
      (size_t)STAGES * (A_BYTES + B_BYTES) + 2 * 64 * 17 * 4 + 1024 + 512;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* tmap, uint64_t* bar, int x,
                                                 int y) {
  // barrier address with the peer bit cleared: the transaction bytes land on
  // the leader CTA's mbarrier
  const uint32_t b = su32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(b), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void umma_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  const uint16_t mask = 0x3;
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(su32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(su32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}

template <int BN>
__device__ bool find_pair_tile(const int32_t* offs, const uint64_t* maps, int N, int m_pairs,
                               int splits, Tile& t, int idx, int rank) {
  for (int e = 0; e < N; ++e) {
    if (!maps[e]) continue;
    const int ne = offs[e + 1] - offs[e];
    if (ne <= 0) continue;
    const int n_tiles_e = (ne + BN - 1) / BN;
    const int cnt = n_tiles_e * m_pairs * splits;
    if (idx < cnt) {
      t.e = e;
      t.split = idx % splits;
      idx /= splits;
      const int nt = idx % n_tiles_e;
      t.m_tile = 2 * (idx / n_tiles_e) + rank;
      t.row0 = offs[e] + nt * BN;
      t.n_valid = min(BN, ne - nt * BN);
      return true;
    }
    idx -= cnt;
  }
  return false;
}

template <int BN, int MODE>
__global__ void __launch_bounds__(kPThreads, 1)
ffn_tc_pair(const __grid_constant__ CUtensorMap b_map, const int32_t* __restrict__ offs,
            const uint64_t* __restrict__ a_maps, int N, int K, int m_tiles, int splits,
            int out_ld, uint16_t* __restrict__ H, float* __restrict__ Y, int64_t y_plane) {
  using S = PairSmem<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + S::STAGES * S::A_BYTES;
  float* sU = reinterpret_cast<float*>(sB + S::STAGES * S::B_BYTES);
  float* sG = sU + 64 * 17;
  uint64_t* full = reinterpret_cast<uint64_t*>(sG + 64 * 17);
  uint64_t* empty = full + S::STAGES;
  uint64_t* tfull = empty + S::STAGES;      // [2]
  uint64_t* tempty = tfull + 2;             // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int nk = (K / BK) / splits;
  const int m_pairs = m_tiles / 2;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S::STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tma_prefetch_desc(&b_map);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tslot)),
                 "r"(S::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int n_tiles = 0;
  for (int e = 0; e < N; ++e) {
    if (!a_maps[e]) continue;
    const int ne = offs[e + 1] - offs[e];
    if (ne > 0) n_tiles += ((ne + BN - 1) / BN) * m_pairs * splits;
  }

  if (warp == 0) {
    if (lane == 0) {                                  // ---- TMA producer (both CTAs)
      uint32_t it = 0;
      for (int ti = pair; ti < n_tiles; ti += n_pairs) {
        Tile t;
        find_pair_tile<BN>(offs, a_maps, N, m_pairs, splits, t, ti, (int)rank);
        const void* a_map = reinterpret_cast<const void*>(a_maps[t.e] + (MODE == 0 ? 0 : 128));
        const int kb0 = t.split * nk;
        for (int i = 0; i < nk; ++i, ++it) {
          const int s = it % S::STAGES;
          const uint32_t ph = (it / S::STAGES) & 1;
          mbar_wait(empty + s, ph ^ 1);
          if (rank == 0) mbar_expect_tx(full + s, 2 * (S::A_BYTES + S::B_BYTES));
          const int kx = (kb0 + i) * BK;
          tma_load_2d_pair(sA + s * S::A_BYTES, a_map, full + s, kx, t.m_tile * BM);
          tma_load_2d_pair(sB + s * S::B_BYTES, &b_map, full + s, kx,
                           t.row0 + (int)rank * (BN / 2));
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {                     // ---- MMA issuer (leader only)
      constexpr uint32_t idesc = idesc_bf16(2 * BM, BN);
      uint32_t it = 0, tc = 0;
      for (int ti = pair; ti < n_tiles; ti += n_pairs, ++tc) {
        const int acc = tc & 1;
        const uint32_t aph = (tc >> 1) & 1;
        mbar_wait(tempty + acc, aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * BN;
        for (int i = 0; i < nk; ++i, ++it) {
          const int s = it % S::STAGES;
          const uint32_t ph = (it / S::STAGES) & 1;
          mbar_wait(full + s, ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = sw128_desc(su32(sA + s * S::A_BYTES));
          const uint64_t db = sw128_desc(su32(sB + s * S::B_BYTES));
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_pair(d, da + 2 * kk, db + 2 * kk, idesc, (i | kk) != 0);
          umma_commit_pair(empty + s);
        }
        umma_commit_pair(tfull + acc);
      }
    }
  } else {                                            // ---- epilogue (warps 2-5)
    const int q = warp & 3;
    const int r = q * 32 + lane;
    uint32_t tc = 0;
    for (int ti = pair; ti < n_tiles; ti += n_pairs, ++tc) {
      Tile t;
      find_pair_tile<BN>(offs, a_maps, N, m_pairs, splits, t, ti, (int)rank);
      const int acc = tc & 1;
      const uint32_t aph = (tc >> 1) & 1;
      mbar_wait(tfull + acc, aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t lane_addr = tmem + acc * BN + ((uint32_t)(q * 32) << 16);
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(lane_addr + c0, v);
        if (MODE == 0) {
          swiglu_chunk(v, r, sG, sU, c0, t.n_valid, t.m_tile, t.row0, out_ld, H);
        } else {
          const int m = t.m_tile * BM + r;
          float* y = Y + (int64_t)t.split * y_plane;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int c = c0 + i;
            if (c < t.n_valid) y[(int64_t)(t.row0 + c) * out_ld + m] = v[i];
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(tempty + acc);
        else mbar_arrive_leader(tempty + acc);
      }
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();                                 // both CTAs done with TMEM / barriers
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(S::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 row-major (rows, cols) map with a (box_rows x 64) box, 128-B swizzle.
static int make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols,
                    uint32_t box_rows) {
  auto fn = encode_fn();
  DALI_REQUIRE(fn != nullptr, DALI_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DALI_REQUIRE(r == CUDA_SUCCESS, DALI_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DALI_OK;
}

template <int BN>
static int launch_bn(const int32_t* offs, const uint64_t* maps, int N, int d, int f,
                     int64_t rows, int n_gpu, uint16_t* hbuf, float* yp, int splits,
                     const uint16_t* xp, cudaStream_t st) {
  using S = Smem<BN>;
  CUtensorMap xmap, hmap;
  const uint64_t cap_rows = (uint64_t)std::max<int64_t>(rows, 1);
  int rc = make_map(&xmap, xp, cap_rows, d, BN);
  if (rc) return rc;
  rc = make_map(&hmap, hbuf, cap_rows, f, BN);
  if (rc) return rc;
  DALI_ONCE_PER_DEVICE({
    cudaFuncSetAttribute(ffn_tc_kernel<BN, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)S::BYTES);
    cudaFuncSetAttribute(ffn_tc_kernel<BN, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)S::BYTES);
  });
  // sum_e ceil(n_e / BN) <= n + (rows - n) / BN for n >= the experts with rows
  const int64_t ntile_bound = n_gpu + std::max<int64_t>(rows - n_gpu, 0) / BN;
  const int m_up = (2 * f) / BM, m_dn = d / BM;
  const int64_t g_up = ntile_bound * m_up;
  launch_pdl(ffn_tc_kernel<BN, 0>, dim3((unsigned)g_up), dim3(kThreads), S::BYTES, st, xmap, offs,
             maps, N, d, m_up, 1, f, hbuf, (float*)nullptr, (int64_t)0);
  DALI_LAUNCH_CHECK("ffn_tc_kernel<up>");
  const int64_t g_dn = ntile_bound * m_dn * splits;
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)g_dn);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = S::BYTES;
  cfg.stream = st;
  cfg.attrs = pdl;                // down prologue overlaps the up kernel's last wave
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, ffn_tc_kernel<BN, 1>, hmap, offs, maps, N, f, m_dn, splits, d,
                     (uint16_t*)nullptr, yp, rows * (int64_t)d);
  DALI_LAUNCH_CHECK("ffn_tc_kernel<down>");
  return DALI_OK;
}

template <int BN>
static int launch_persistent(const int32_t* offs, const uint64_t* maps, int N, int d, int f,
                             int64_t rows, int n_gpu, uint16_t* hbuf, float* yp, int splits,
                             const uint16_t* xp, cudaStream_t st, int n_sm) {
  using S = PSmem<BN>;
  CUtensorMap xmap, hmap;
  const uint64_t cap_rows = (uint64_t)std::max<int64_t>(rows, 1);
  int rc = make_map(&xmap, xp, cap_rows, d, BN);
  if (rc) return rc;
  rc = make_map(&hmap, hbuf, cap_rows, f, BN);
  if (rc) return rc;
  DALI_ONCE_PER_DEVICE({
    cudaFuncSetAttribute(ffn_tc_persistent<BN, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)S::BYTES);
    cudaFuncSetAttribute(ffn_tc_persistent<BN, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)S::BYTES);
  });
  const int64_t ntile_bound = n_gpu + std::max<int64_t>(rows - n_gpu, 0) / BN;
  const int m_up = (2 * f) / BM, m_dn = d / BM;
  const unsigned g_up = (unsigned)std::min<int64_t>(ntile_bound * m_up, n_sm);
  const unsigned g_dn = (unsigned)std::min<int64_t>(ntile_bound * m_dn * splits, n_sm);
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = S::BYTES;
  cfg.stream = st;
  cfg.gridDim = dim3(g_up);
  cfg.attrs = nullptr;
  cfg.numAttrs = 0;
  cudaLaunchKernelEx(&cfg, ffn_tc_persistent<BN, 0>, xmap, offs, maps, N, d, m_up, 1, f, hbuf,
                     (float*)nullptr, (int64_t)0);
  DALI_LAUNCH_CHECK("ffn_tc_persistent<up>");
  cfg.gridDim = dim3(g_dn);
  cfg.attrs = attr_pdl;           // down projection prologue overlaps the up tail
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, ffn_tc_persistent<BN, 1>, hmap, offs, maps, N, f, m_dn, splits, d,
                     (uint16_t*)nullptr, yp, rows * (int64_t)d);
  DALI_LAUNCH_CHECK("ffn_tc_persistent<down>");
  return DALI_OK;
}

template <int BN>
static int launch_pair(const int32_t* offs, const uint64_t* maps, int N, int d, int f,
                       int64_t rows, int n_gpu, uint16_t* hbuf, float* yp, int splits,
                       const uint16_t* xp, cudaStream_t st, int n_sm) {
  using S = PairSmem<BN>;
  CUtensorMap xmap, hmap;                          // token boxes of BN/2 rows per CTA
  const uint64_t cap_rows = (uint64_t)std::max<int64_t>(rows, 1);
  int rc = make_map(&xmap, xp, cap_rows, d, BN / 2);
  if (rc) return rc;
  rc = make_map(&hmap, hbuf, cap_rows, f, BN / 2);
  if (rc) return rc;
  DALI_ONCE_PER_DEVICE({
    cudaFuncSetAttribute(ffn_tc_pair<BN, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)S::BYTES);
    cudaFuncSetAttribute(ffn_tc_pair<BN, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)S::BYTES);
  });
  const int64_t ntile_bound = n_gpu + std::max<int64_t>(rows - n_gpu, 0) / BN;
  const int m_up = (2 * f) / BM, m_dn = d / BM;
  const int max_ctas = (n_sm / 2) * 2;
  const unsigned g_up = (unsigned)std::min<int64_t>(2 * ntile_bound * (m_up / 2), max_ctas);
  const unsigned g_dn = (unsigned)std::min<int64_t>(2 * ntile_bound * (m_dn / 2) * splits, max_ctas);
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = S::BYTES;
  cfg.stream = st;
  cfg.gridDim = dim3(g_up);
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, ffn_tc_pair<BN, 0>, xmap, offs, maps, N, d, m_up, 1, f, hbuf,
                     (float*)nullptr, (int64_t)0);
  DALI_LAUNCH_CHECK("ffn_tc_pair<up>");
  cfg.gridDim = dim3(g_dn);
  cfg.numAttrs = 2;                                // down prologue overlaps the up tail
  cudaLaunchKernelEx(&cfg, ffn_tc_pair<BN, 1>, hmap, offs, maps, N, f, m_dn, splits, d,
                     (uint16_t*)nullptr, yp, rows * (int64_t)d);
  DALI_LAUNCH_CHECK("ffn_tc_pair<down>");
  return DALI_OK;
}

// Token tiles of 256 go through the CTA-pair kernel (measured +3-4% at 256-512
// tokens per expert, equal at 1024; at 128-token tiles, which are HBM-bound,
// the pair kernel was 1.5% slower and is not used).  DALI_FFN_PAIR=0 selects
// the single-CTA persistent kernel (A/B switch).
static bool use_pair() {
  static const bool v = [] {
    const char* e = getenv("DALI_FFN_PAIR");
    return !(e && e[0] == '0');
  }();
  return v;
}

static int sm_count_tc() { return device_sm_count(); }

}  // namespace tc
}  // namespace dali

using namespace dali;

extern "C" int dali_expert_maps(const void* block, int32_t d, int32_t f, void* out) {
  DALI_REQUIRE(block && out, DALI_ECUDA, "null argument");
  DALI_REQUIRE(d % 128 == 0 && f % 64 == 0 && (2 * f) % 128 == 0, DALI_ETRACE,
               "tensor-core FFN needs d %% 128 == 0 and f %% 64 == 0 (d=%d f=%d)", d, f);
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(out);
  const uint16_t* w13 = reinterpret_cast<const uint16_t*>(block);
  const uint16_t* w2 = w13 + (int64_t)2 * f * d;
  int rc = tc::make_map(&m[0], w13, 2 * (uint64_t)f, d, tc::BM);
  if (rc) return rc;
  return tc::make_map(&m[1], w2, (uint64_t)d, f, tc::BM);
}

extern "C" int dali_expert_ffn_tc(const uint16_t* xp, const int32_t* offsets, int32_t N,
                                  const uint64_t* expert_maps, int32_t d, int32_t f, int64_t rows,
                                  int32_t max_rows_per_expert, int32_t n_gpu_experts,
                                  uint16_t* hbuf, float* yp, int32_t splits, void* stream) {
  DALI_REQUIRE(d % 128 == 0 && f % 64 == 0, DALI_ETRACE, "need d %% 128 == 0, f %% 64 == 0");
  DALI_REQUIRE(splits >= 1 && (f / tc::BK) % splits == 0, DALI_ETRACE,
               "splits %d must divide f/64 = %d", splits, f / tc::BK);
  if (rows <= 0 || n_gpu_experts <= 0) return DALI_OK;
  cudaStream_t st = as_stream(stream);
  const int mr = max_rows_per_expert;
  if (mr <= 16)
    return tc::launch_bn<16>(offsets, expert_maps, N, d, f, rows, n_gpu_experts, hbuf, yp, splits,
                             xp, st);
  if (mr <= 32)
    return tc::launch_bn<32>(offsets, expert_maps, N, d, f, rows, n_gpu_experts, hbuf, yp, splits,
                             xp, st);
  const int nsm = tc::sm_count_tc();
  if (mr <= 64)
    return tc::launch_persistent<64>(offsets, expert_maps, N, d, f, rows, n_gpu_experts, hbuf,
                                     yp, splits, xp, st, nsm);
  if (mr <= 128)
    return tc::launch_persistent<128>(offsets, expert_maps, N, d, f, rows, n_gpu_experts, hbuf,
                                      yp, splits, xp, st, nsm);
  // CTA pairs tile M in 256-row pairs: both projections need an even count
  // of 128-row weight tiles (true for every shipped config)
  if (tc::use_pair() && ((2 * f) / tc::BM) % 2 == 0 && (d / tc::BM) % 2 == 0)
    return tc::launch_pair<256>(offsets, expert_maps, N, d, f, rows, n_gpu_experts, hbuf, yp,
                                splits, xp, st, nsm);
  return tc::launch_persistent<256>(offsets, expert_maps, N, d, f, rows, n_gpu_experts, hbuf, yp,
                                    splits, xp, st, nsm);
}
