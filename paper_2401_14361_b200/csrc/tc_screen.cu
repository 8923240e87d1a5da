// tc_screen.cu -- tensor-core (tcgen05) screen pass of the EAMC matcher for
// large probe batches (batch regime: SW Q=4096, SC Q=65,536).
//
// Every probe row and collection row is stored a second time, normalised
// (c * RN32(1/sqrt(sum c^2))) and rounded to fp16, K-major, K = L*E padded to
// a multiple of 64.  One GEMM D[q][p] = sum_k A'[q][k] * B'[p][k] then gives
// the summed per-layer cosine similarities of every (probe, entry) pair
// directly -- the per-layer epilogue of the SIMT screen disappears.  The
// both-zero-row convention (eam.cpp:84) is added exactly as
// popc(zmask_q & zmask_p).  fp16 rounding of the operands and the fp32
// tensor-core accumulation give a screen distance within tc_eps of the
// reference distance ("tensor-core screen bound"); the argmin
// threshold / candidate-bucket logic and the exact fp64 refine are shared
// with the SIMT path, so results stay bit-exact.
//
// Kernel anatomy (one CTA per SM, persistent over 128x256 output tiles):
//   warp 0      TMA producer: A' 128x64 and B' 256x64 fp16 tiles, 128B swizzle,
//               4-stage mbarrier ring (48 KB per stage)
//   warp 1      TMEM allocator + single-thread tcgen05.mma.cta_group::1.kind::f16
//               issuer (M=128, N=256, K=16), double-buffered fp32 accumulators
//               (2 x 256 TMEM columns), tcgen05.commit -> mbarriers
//   warps 2-17  epilogue (EPI_WARPS = 16: four warps per TMEM lane quarter,
//               64 accumulator columns each): tcgen05.ld 32x32b.x32 (thread =
//               probe row), screen distance, row min -> global per-probe
//               threshold (atomicMin), candidate push into the per-probe bucket
#ifndef TC_GROUP_M
#define TC_GROUP_M 64
#endif
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace moe {

namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr uint32_t A_BYTES = BM * BK * 2;  // 16 KB
constexpr uint32_t B_BYTES = BN * BK * 2;  // 32 KB
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
constexpr uint32_t TMEM_COLS = 512;  // 2 accumulators x 256 fp32 columns
#ifndef MOE_EPI_WARPS
#define MOE_EPI_WARPS 16
#endif
constexpr int EPI_WARPS = MOE_EPI_WARPS;  // 16: 64 columns per warp (measured best; 8: 128, 4: 256)
constexpr int THREADS = 64 + 32 * EPI_WARPS;  // warp 0 TMA, warp 1 MMA, then the epilogue
constexpr uint32_t EPI_THREADS = 32 * EPI_WARPS;
// epilogue column split: EPI_PARTS warps per TMEM lane quarter, EPI_CH
// 32-column chunks per warp and call
constexpr uint32_t EPI_PARTS = EPI_WARPS >= 8 ? EPI_WARPS / 4 : 2;
constexpr uint32_t EPI_CH = 8 / EPI_PARTS;

struct TcArgs {
  float invL;          // 1/L (fp32)
  const uint64_t* zq;  // [Q] zero-row masks of the probes
  const uint64_t* zp;  // [cap] zero-row masks of the entries
  uint32_t Q, P, L;
  uint32_t n_m, n_n, n_k;
  float eps2;
  uint32_t* T;
  uint32_t* bcnt;
  uint2* bucket;
  uint32_t bcap;
  float* dmat;    // matrix mode: every screen distance -> dmat[q * ldd + p]
  uint32_t ldd;
  // refine inputs prefetched into L2 during the screen: the collection's
  // packed rows, fp64 row norms and seqs (pf[i] = bytes [0, pf_bytes[i]))
  const uint8_t* pf[3];
  uint64_t pf_bytes[3];
};

// The exact refine pass after the screen reads its candidates' packed u8 rows,
// which the screen itself never touches (it streams the fp16 copies).  Each
// CTA's producer thread prefetches its 1/grid slice of them into L2 with a
// few bulk prefetches, issued after the CTA's first tile of operand loads.
__device__ __forceinline__ void prefetch_slice_l2(const TcArgs& a, uint32_t part, uint32_t parts) {
#pragma unroll 1
  for (int i = 0; i < 3; ++i) {
    if (!a.pf[i]) continue;
    const uint64_t per = ((a.pf_bytes[i] + parts - 1) / parts + 15) & ~15ull;
    const uint64_t b0 = per * part;
    const uint64_t end = a.pf_bytes[i] & ~15ull;
    const uint64_t b1 = b0 + per < end ? b0 + per : end;
    for (uint64_t o = b0; o < b1; o += 32768) {
      const uint32_t n = b1 - o < 32768 ? (uint32_t)(b1 - o) : 32768u;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.pf[i] + o), "r"(n)
                   : "memory");
    }
  }
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Output tile t -> (probe tile m, entry tile n), grouped: GM consecutive
// probe tiles sweep all entry tiles together, so the clusters running side by
// side share entry tiles (each read once from HBM per group) while the group's
// probe tiles stay in L2.  With m fastest over all probe tiles (the previous
// order) a large probe batch cycled more probe-tile bytes than L2 holds and
// re-read them from HBM for every entry tile: 391 GB of DRAM reads per SC
// batch launch for 1.7 GB of algorithmic bytes.  Small batches (n_m <= GM) keep
// the plain order.
constexpr uint32_t kTileGroupM = TC_GROUP_M;
__device__ __forceinline__ void tile_mn(uint32_t t, uint32_t n_m, uint32_t n_n, uint32_t* m,
                                        uint32_t* n) {
  if (n_m <= kTileGroupM) {
    *m = t % n_m;
    *n = t / n_m;
    return;
  }
  const uint32_t per = kTileGroupM * n_n;
  const uint32_t g = t / per, first = g * kTileGroupM;
  const uint32_t gsz = min(kTileGroupM, n_m - first);
  const uint32_t r = t - g * per;
  *m = first + r % gsz;
  *n = r / gsz;
}

// K-major operand tile, 128-byte swizzle: 8-row atoms of 128 B, atoms 1024 B
// apart (SBO), LBO unused for swizzled K-major; version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

// kind::f16 instruction descriptor: A,B = F16 K-major, D = F32, M=128, N=256.
constexpr uint32_t kIdesc = (1u << 4) | (0u << 7) | (0u << 10) | (0u << 15) | (0u << 16) |
                            ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Epilogue of one accumulator tile for one probe row and 128 of its 256
// columns (two warps of the same TMEM lane quarter split the columns).
// Pass 1 (branch-free): screen distances -> row minimum (and runner-up) ->
// global per-probe threshold -> the single-candidate push.  Pass 2 re-reads
// TMEM only for rows with several candidates in the tile.
__device__ __forceinline__ void epilogue_half(uint32_t tcol, uint32_t col0, uint64_t zq,
                                              const uint64_t* zt, uint32_t q, bool qvalid,
                                              uint32_t p0, const TcArgs& a, float invL) {
  uint32_t r[32];
  const bool full_tile = p0 + col0 + 32 * EPI_CH <= a.P;
  if (a.dmat) {  // matrix mode (blocked construction replay): store, no threshold
#pragma unroll 1
    for (uint32_t c = 0; c < EPI_CH; ++c) {
      tmem_ld32(tcol + c * 32, r);
      if (!qvalid) continue;
      float* o = a.dmat + (uint64_t)q * a.ldd + p0 + col0 + c * 32;
      float dv[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const uint32_t col = col0 + c * 32 + j;
        const float sim = __uint_as_float(r[j]) + (float)__popcll(zq & zt[col]);
        dv[j] = fmaxf(fmaf(-sim, invL, 1.0f), 0.0f);
      }
      if (full_tile) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(o + j) = make_float4(dv[j], dv[j + 1], dv[j + 2], dv[j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (p0 + col0 + c * 32 + j < a.P) o[j] = dv[j];
      }
    }
    return;
  }
  // Pass 1 (branch-free): the row's smallest screen distance d1 (first
  // column c1 attaining it) and the second smallest d2.  Most rows that can
  // produce a candidate produce exactly one (d1 <= thr < d2): it is pushed
  // straight from registers, and the TMEM re-read of pass 2 is needed only by
  // rows with two or more candidates in this tile (incl. exact ties).
  // (tcgen05.ld is warp-collective: the loads stay outside the per-row branch)
  const bool fast = zq == 0 && full_tile;  // no zero rows: minimise d via max sim
  float s1 = -__uint_as_float(kFInf), s2 = s1;
  float d1 = __uint_as_float(kFInf), d2 = d1;
  uint32_t c1 = 0;
#pragma unroll 1
  for (uint32_t c = 0; c < EPI_CH; ++c) {
    tmem_ld32(tcol + c * 32, r);
    if (fast) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float x = __uint_as_float(r[j]);
        s2 = fmaxf(s2, fminf(s1, x));
        c1 = x > s1 ? col0 + c * 32 + j : c1;
        s1 = fmaxf(s1, x);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const uint32_t col = col0 + c * 32 + j;
        const float sim = __uint_as_float(r[j]) + (float)__popcll(zq & zt[col]);
        float d = fmaf(-sim, invL, 1.0f);
        d = (p0 + col < a.P) ? d : __uint_as_float(kFInf);
        d2 = fminf(d2, fmaxf(d1, d));
        c1 = d < d1 ? col : c1;
        d1 = fminf(d1, d);
      }
    }
  }
  if (fast) {  // rounding is monotone: min_j d_j = d(max_j sim_j)
    d1 = fmaf(-s1, invL, 1.0f);
    d2 = fmaf(-s2, invL, 1.0f);
  }
  d1 = fmaxf(d1, 0.0f);
  d2 = fmaxf(d2, 0.0f);
  float thr = -1.0f;  // invalid rows never qualify
  if (qvalid) {
    const uint32_t mb = __float_as_uint(d1);
    uint32_t tv = *reinterpret_cast<volatile uint32_t*>(&a.T[q]);
    if (mb < tv) tv = min(atomicMin(&a.T[q], mb), mb);
    thr = __uint_as_float(tv) + a.eps2;
  }
  const bool multi = d2 <= thr;  // implies d1 <= thr
  if (d1 <= thr && !multi) {
    const uint32_t pos = atomicAdd(&a.bcnt[q], 1u);
    if (pos < a.bcap) a.bucket[(uint64_t)q * a.bcap + pos] = make_uint2(p0 + c1, __float_as_uint(d1));
  }
  // tcgen05.ld is warp-collective: the (rarer) full pass is taken by the
  // whole warp whenever any of its rows has two or more candidates
  if (!__any_sync(0xffffffffu, multi)) return;
#pragma unroll 1
  for (uint32_t c = 0; c < EPI_CH; ++c) {
    tmem_ld32(tcol + c * 32, r);
#pragma unroll
    for (int j = 0; j < 32; ++j) {  // rare pass: a branch per column is fine here
      const uint32_t col = col0 + c * 32 + j;
      const float sim = __uint_as_float(r[j]) + (float)__popcll(zq & zt[col]);
      const float d = fmaxf(fmaf(-sim, invL, 1.0f), 0.0f);
      if (multi && d <= thr && p0 + col < a.P) {
        const uint32_t pos = atomicAdd(&a.bcnt[q], 1u);
        if (pos < a.bcap)
          a.bucket[(uint64_t)q * a.bcap + pos] = make_uint2(p0 + col, __float_as_uint(d));
      }
    }
  }
}

__global__ void __launch_bounds__(THREADS, 1)
    k_tc_screen(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                const TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* zp_s = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);  // [2][BN]
  uint64_t* full = zp_s + 2 * BN;
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n_tiles = a.n_m * a.n_n;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&ta);
    prefetch_tmap(&tb);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], EPI_THREADS);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // set-up above overlaps the previous grid's tail
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      uint32_t s = 0, ph = 0;
      for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        uint32_t m, n;
        tile_mn(t, a.n_m, a.n_n, &m, &n);
        for (uint32_t kb = 0; kb < a.n_k; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
          tma_load_2d(sA + s * A_BYTES, &ta, &full[s], (int)(kb * BK), (int)(m * BM));
          tma_load_2d(sB + s * B_BYTES, &tb, &full[s], (int)(kb * BK), (int)(n * BN));
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if (t == blockIdx.x) prefetch_slice_l2(a, blockIdx.x, gridDim.x);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t s = 0, ph = 0, i = 0;
      for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
        const uint32_t acc = i & 1;
        mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (uint32_t kb = 0; kb < a.n_k; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint8_t* pa = sA + s * A_BYTES;
          const uint8_t* pb = sB + s * B_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_f16(d, smem_desc_sw128(pa + 32 * k), smem_desc_sw128(pb + 32 * k),
                    (kb | k) != 0 ? 1u : 0u);
          mma_commit(&empty[s]);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else {
    // epilogue: 8 warps; warp w serves TMEM lane quarter w%4 (probe rows) and
    // column half (w-2)/4 of the 256-column accumulator
    const uint32_t quarter = warp & 3;
    const uint32_t half0 = EPI_WARPS >= 8 ? (warp - 2) >> 2 : 0;
    const uint32_t row = quarter * 32 + lane;
    const uint32_t et = threadIdx.x - 64;  // 0..255
    uint32_t i = 0;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      const uint32_t acc = i & 1;
      uint32_t m, n;
        tile_mn(t, a.n_m, a.n_n, &m, &n);
      uint64_t* zt = zp_s + acc * BN;
      {
        for (uint32_t j = et; j < BN; j += EPI_THREADS) {
          const uint32_t p = n * BN + j;
          zt[j] = p < a.P ? a.zp[p] : 0ull;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
      const uint32_t q = m * BM + row;
      const bool qvalid = q < a.Q;
      const uint64_t zq = qvalid ? a.zq[q] : 0ull;
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      tc_fence_after();
      for (uint32_t half = half0; half < half0 + (EPI_WARPS >= 8 ? 1u : 2u); ++half) {
        const uint32_t col0 = half * 32 * EPI_CH;
        const uint32_t tcol = tmem + ((quarter * 32) << 16) + acc * BN + col0;
        epilogue_half(tcol, col0, zq, zt, q, qvalid, n * BN, a, a.invL);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// 2-CTA variant (cta_group::2, cluster of 2): one MMA covers a 256x256 tile.
// CTA r of the pair loads A rows [256m + 128r, +128) and B rows
// [256n + 128r, +128) (half the N tile); the leader (r=0) issues
// tcgen05.mma.cta_group::2 over both CTAs' shared memory, accumulating the
// pair's 256x256 tile as 128 TMEM lanes x 256 columns in each CTA.  Per SM
// this halves the B bytes staged per FLOP relative to the 1-CTA kernel.
constexpr int S2 = 6;                         // pipeline stages
constexpr uint32_t A2_BYTES = 128 * BK * 2;   // 16 KB
constexpr uint32_t B2_BYTES = 128 * BK * 2;   // 16 KB (half of the N tile)
constexpr uint32_t STAGE2 = A2_BYTES + B2_BYTES;
constexpr uint32_t kIdesc2 = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // leader-CTA address of a pair barrier

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                 int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc2), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, 0;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_tc2_screen(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                 const TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + S2 * A2_BYTES;
  uint64_t* zp_s = reinterpret_cast<uint64_t*>(sB + S2 * B2_BYTES);  // [2][BN]
  uint64_t* full = zp_s + 2 * BN;
  uint64_t* empty = full + S2;
  uint64_t* tfull = empty + S2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const uint32_t cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const uint32_t n_tiles = a.n_m * a.n_n;  // n_m counts 256-row M tiles here

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&ta);
    prefetch_tmap(&tb);
    for (int s = 0; s < S2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * EPI_THREADS);  // both CTAs' epilogue threads (leader's copy)
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // set-up above overlaps the previous grid's tail
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      uint32_t s = 0, ph = 0;
      for (uint32_t t = cluster; t < n_tiles; t += n_clusters) {
        uint32_t m, n;
        tile_mn(t, a.n_m, a.n_n, &m, &n);
        for (uint32_t kb = 0; kb < a.n_k; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * STAGE2);
          tma_load_2d_pair(sA + s * A2_BYTES, &ta, &full[s], (int)(kb * BK),
                           (int)(m * 256 + rank * 128));
          tma_load_2d_pair(sB + s * B2_BYTES, &tb, &full[s], (int)(kb * BK),
                           (int)(n * BN + rank * 128));
          if (++s == S2) {
            s = 0;
            ph ^= 1;
          }
        }
        if (t == cluster) prefetch_slice_l2(a, blockIdx.x, gridDim.x);
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      uint32_t s = 0, ph = 0, i = 0;
      for (uint32_t t = cluster; t < n_tiles; t += n_clusters, ++i) {
        const uint32_t acc = i & 1;
        mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (uint32_t kb = 0; kb < a.n_k; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint8_t* pa = sA + s * A2_BYTES;
          const uint8_t* pb = sB + s * B2_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_f16_pair(d, smem_desc_sw128(pa + 32 * k), smem_desc_sw128(pb + 32 * k),
                         (kb | k) != 0 ? 1u : 0u);
          mma_commit_pair(&empty[s]);
          if (++s == S2) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit_pair(&tfull[acc]);
      }
    }
  } else {
    // epilogue: 8 warps; warp w serves TMEM lane quarter w%4 (probe rows) and
    // column half (w-2)/4 of the 256-column accumulator
    const uint32_t quarter = warp & 3;
    const uint32_t half0 = EPI_WARPS >= 8 ? (warp - 2) >> 2 : 0;
    const uint32_t row = quarter * 32 + lane;
    const uint32_t et = threadIdx.x - 64;  // 0..255
    uint32_t i = 0;
    for (uint32_t t = cluster; t < n_tiles; t += n_clusters, ++i) {
      const uint32_t acc = i & 1;
      uint32_t m, n;
        tile_mn(t, a.n_m, a.n_n, &m, &n);
      uint64_t* zt = zp_s + acc * BN;
      {
        for (uint32_t j = et; j < BN; j += EPI_THREADS) {
          const uint32_t p = n * BN + j;
          zt[j] = p < a.P ? a.zp[p] : 0ull;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
      const uint32_t q = m * 256 + rank * 128 + row;
      const bool qvalid = q < a.Q;
      const uint64_t zq = qvalid ? a.zq[q] : 0ull;
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      tc_fence_after();
      for (uint32_t half = half0; half < half0 + (EPI_WARPS >= 8 ? 1u : 2u); ++half) {
        const uint32_t col0 = half * 32 * EPI_CH;
        const uint32_t tcol = tmem + ((quarter * 32) << 16) + acc * BN + col0;
        epilogue_half(tcol, col0, zq, zt, q, qvalid, n * BN, a, a.invL);
      }
      tc_fence_before();
      mbar_arrive_leader(&tempty[acc]);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

cudaError_t encode_2d_f16(const void* base, uint64_t rows, uint64_t Kp, uint32_t box_rows,
                          CUtensorMap* map) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult qr;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
    if (e != cudaSuccess || qr != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {Kp, rows};
  const cuuint64_t strides[1] = {Kp * 2};
  const cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace

float tc_eps2(uint32_t L, uint32_t E, uint32_t Kp) {
  // |d16 - d_ref| <= 2.2*2^-11 (fp16 operand rounding, relative, per term;
  // cos <= 1 per layer) + 2*E*2^-25 (subnormal floor) + Kp*2^-22 (fp32
  // accumulation with truncation, partial sums <= L) -- DESIGN.md.
  (void)L;
  const double eps = 2.2 / 2048.0 + 2.0 * E / 33554432.0 + (double)Kp / 4194304.0 + 1e-6;
  return (float)(2.0 * 1.25 * eps);
}

bool tc_supported(const DevColl& c) { return c.L <= 64 && c.nrm != nullptr && c.Kp > 0; }

cudaError_t launch_tc_screen(const DevColl& c, const DevProbes& pr, const MatchWork& w, int n_sm,
                             cudaStream_t st, float* dmat, uint32_t ldd) {
  if (c.size == 0 || pr.Q == 0) return cudaSuccess;
  // tensor maps are re-encoded only when the operand buffers change
  struct MapCache {
    const void* base = nullptr;
    uint64_t rows = 0, Kp = 0;
    uint32_t box = 0;
    CUtensorMap map;
  };
  static thread_local MapCache ca, cb;
  cudaError_t e = cudaSuccess;
  if (ca.base != pr.nrm || ca.rows != pr.Q || ca.Kp != c.Kp) {
    e = encode_2d_f16(pr.nrm, pr.Q, c.Kp, BM, &ca.map);
    if (e != cudaSuccess) return e;
    ca.base = pr.nrm;
    ca.rows = pr.Q;
    ca.Kp = c.Kp;
  }
  if (cb.base != c.nrm || cb.rows != c.cap || cb.Kp != c.Kp) {
    e = encode_2d_f16(c.nrm, c.cap, c.Kp, BN, &cb.map);
    if (e != cudaSuccess) return e;
    cb.base = c.nrm;
    cb.rows = c.cap;
    cb.Kp = c.Kp;
    cb.box = BN;
  }
  const CUtensorMap& ta = ca.map;
  const CUtensorMap& tb = cb.map;
  TcArgs a{};
  a.invL = 1.0f / (float)c.L;
  a.zq = pr.zmask;
  a.zp = c.zmask;
  a.Q = pr.Q;
  a.P = c.size;
  a.L = c.L;
  a.n_m = (pr.Q + BM - 1) / BM;
  a.n_n = (c.size + BN - 1) / BN;
  a.n_k = c.Kp / BK;
  a.eps2 = w.eps2;
  a.T = w.T;
  a.bcnt = w.bcnt;
  a.bucket = w.bucket;
  a.bcap = w.bcap;
  a.dmat = dmat;
  a.ldd = ldd;
  if (!dmat) {  // screen pass (the refine follows): its inputs into L2
    a.pf[0] = c.counts;
    a.pf_bytes[0] = (uint64_t)c.size * c.L * c.RB;
    a.pf[1] = reinterpret_cast<const uint8_t*>(c.sqb);
    a.pf_bytes[1] = (uint64_t)c.size * c.L * sizeof(double);
    a.pf[2] = reinterpret_cast<const uint8_t*>(c.seq);
    a.pf_bytes[2] = (uint64_t)c.size * sizeof(uint64_t);
  }
  const char* e2 = getenv("MOE_TC2");
  const bool pair = (e2 ? e2[0] != '0' : true) && pr.Q > 128;
  if (pair) {  // 2-CTA pairs: 256-row M tiles, half the B tile per CTA
    if (cb.rows != c.cap || cb.base != c.nrm || cb.Kp != c.Kp || cb.box != 128) {
      e = encode_2d_f16(c.nrm, c.cap, c.Kp, 128, &cb.map);
      if (e != cudaSuccess) return e;
      cb.base = c.nrm;
      cb.rows = c.cap;
      cb.Kp = c.Kp;
      cb.box = 128;
    }
    a.n_m = (pr.Q + 255) / 256;
    const size_t smem2 = (size_t)S2 * STAGE2 + 2 * BN * 8 + (2 * S2 + 4) * 8 + 16;
    static bool attr2 = false;
    if (!attr2) {
      e = cudaFuncSetAttribute(k_tc2_screen, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem2);
      if (e != cudaSuccess) return e;
      attr2 = true;
    }
    const uint32_t tiles = a.n_m * a.n_n;
    const uint32_t clusters = std::min<uint32_t>(tiles, (uint32_t)n_sm / 2);
    return launch_pdl(k_tc2_screen, dim3(clusters * 2), dim3(THREADS), smem2, st, ta, cb.map, a);
  }
  if (cb.box != BN) {
    e = encode_2d_f16(c.nrm, c.cap, c.Kp, BN, &cb.map);
    if (e != cudaSuccess) return e;
    cb.box = BN;
  }
  const size_t smem = (size_t)STAGES * STAGE_BYTES + 2 * BN * 8 + (2 * STAGES + 4) * 8 + 16;
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(k_tc_screen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const uint32_t tiles = a.n_m * a.n_n;
  const uint32_t grid = std::min<uint32_t>(tiles, (uint32_t)n_sm);
  return launch_pdl(k_tc_screen, dim3(grid), dim3(THREADS), smem, st, ta, tb, a);
}

}  // namespace moe
