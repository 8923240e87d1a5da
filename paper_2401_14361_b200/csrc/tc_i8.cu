// tc_i8.cu -- exact-integer tensor-core (tcgen05 kind::i8) screen for SMALL
// probe batches (streaming regime: Q < 128, e.g. SC P=2^20, Q=8).
//
// B operand = the u8 collection itself: entry p's L rows of RB bytes are one
// contiguous K-major row of K = L*RB bytes (the AoS layout of DevColl.counts).
// A operand = the probes laid out BLOCK-DIAGONALLY: row (q, l) of A (R rows
// per probe, R = next power of two >= L) holds probe q's layer-l counts at
// K offset l*RB and zeros elsewhere.  One u8 x u8 -> s32 GEMM then leaves the
// EXACT per-layer dot dot_l(q, p) in TMEM lane (q, l), column p.  Most of the
// MMA work multiplies zeros, which is irrelevant: the kernel is HBM-bound
// (1 byte per count) and the i8 tensor pipe has >3x headroom even so.
//
// Epilogue (8 warps, thread = TMEM lane = (probe, layer)): fp32 screen terms
// float(dot) * ia[q][l] * ib[p][l] are summed over the R lanes of each probe
// with a register-transpose butterfly (30 shuffles per 32 columns instead of
// 128), the both-zero-row term popc(zq & zp) is added, and the per-probe
// minimum / global threshold / candidate push reuse the SIMT screen's error
// bound (same fp32 formula on the same exact integer dots) and its refine.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace moe {

namespace {

constexpr int BM = 128, BN = 256, BKB = 128;  // BKB = K bytes per stage (one SW128 atom row)
#ifndef I8_IB_STAGE
#define I8_IB_STAGE 1
#endif
// With the entry norms of a tile staged in shared memory (I8_IB_STAGE), three
// operand stages leave room for them.
constexpr int STAGES = I8_IB_STAGE ? 3 : 4;
constexpr uint32_t IBS = 257;  // staged norm row stride (odd: 16 rows -> 16 banks)
constexpr uint32_t A_BYTES = BM * BKB;  // 16 KB
constexpr uint32_t B_BYTES = BN * BKB;  // 32 KB
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
constexpr uint32_t TMEM_COLS = 512;
constexpr int THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
constexpr uint32_t EPI_THREADS = 256;

// kind::i8: A,B unsigned 8-bit K-major, D = S32, M=128, N=256.
constexpr uint32_t kIdescI8 = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(BN >> 3) << 17) |
                              ((uint32_t)(BM >> 4) << 24);

struct I8Args {
  const float* ia;     // [Q][L] probe inverse norms
  const float* ibT;    // [L][cap] entry inverse norms
  const uint64_t* zq;  // [Q] probe zero-row masks (L <= 32 here)
  const uint64_t* zp;  // [cap]
  uint64_t cap;
  uint32_t Q, P, L, R, n_m, n_n, n_k;
  float invL, eps2;
  uint32_t* T;
  uint32_t* bcnt;
  uint2* bucket;
  uint32_t bcap;
};

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
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ uint64_t desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  return ((addr >> 4) & 0x3FFFull) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(kIdescI8), "r"(acc)
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

// Sum 32 per-lane values over groups of 2^LOGR consecutive lanes with a
// register-transpose butterfly; afterwards lane holds 32>>LOGR group sums for
// columns (lane & (R-1)) * (32>>LOGR) + [0, 32>>LOGR).
template <int LOGR>
__device__ __forceinline__ void group_sum_transpose(float (&v)[32], uint32_t lane) {
  int n = 32;
#pragma unroll
  for (int s = LOGR - 1; s >= 0; --s) {
    const uint32_t o = 1u << s;
    const bool up = (lane & o) != 0;
    n >>= 1;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < n) {
        const float send = up ? v[i] : v[i + n];
        const float keep = up ? v[i + n] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
  }
}

template <int LOGR>
__global__ void __launch_bounds__(THREADS, 1)
    k_tci8_screen(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                  const I8Args a) {
  constexpr uint32_t R = 1u << LOGR;
  constexpr int VPL = 32 >> LOGR;  // group sums a lane holds per 32-column chunk
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* zp_s = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);  // [2][BN]
  float* ib_s = reinterpret_cast<float*>(zp_s + 2 * BN);                 // [2][R][IBS]
  uint64_t* full = reinterpret_cast<uint64_t*>(ib_s + (I8_IB_STAGE ? 2 * (1u << LOGR) * IBS : 0));
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
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // set-up above overlaps the previous grid's tail
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      uint32_t s = 0, ph = 0;
      for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const uint32_t m = t % a.n_m, n = t / a.n_m;
        for (uint32_t kb = 0; kb < a.n_k; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
          tma_load_2d(sA + s * A_BYTES, &ta, &full[s], (int)(kb * BKB), (int)(m * BM));
          tma_load_2d(sB + s * B_BYTES, &tb, &full[s], (int)(kb * BKB), (int)(n * BN));
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t s = 0, ph = 0, i = 0;
      for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
        const uint32_t acc = i & 1;
        mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
        fence_after();
        const uint32_t d = tmem + acc * BN;
        for (uint32_t kb = 0; kb < a.n_k; ++kb) {
          mbar_wait(&full[s], ph);
          fence_after();
          const uint8_t* pa = sA + s * A_BYTES;
          const uint8_t* pb = sB + s * B_BYTES;
#pragma unroll
          for (int k = 0; k < BKB / 32; ++k)  // K = 32 bytes per kind::i8 instruction
            mma_i8(d, desc_sw128(pa + 32 * k), desc_sw128(pb + 32 * k), (kb | k) != 0 ? 1u : 0u);
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
    const uint32_t quarter = warp & 3;
    const uint32_t half = (warp - 2) >> 2;
    const uint32_t row = quarter * 32 + lane;  // A row = (probe, layer)
    const uint32_t et = threadIdx.x - 64;
    const uint32_t qg = row >> LOGR, l = row & (R - 1);
    const uint32_t gl = lane & (R - 1);  // lane within the probe group
    uint32_t i = 0;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      const uint32_t acc = i & 1;
      const uint32_t m = t % a.n_m, n = t / a.n_m;
      uint64_t* zt = zp_s + acc * BN;
      {
        const uint32_t p = n * BN + et;
        zt[et] = p < a.P ? a.zp[p] : 0ull;
      }
#if I8_IB_STAGE
      // the tile's entry norms ibT[l][n*BN .. +BN) -> shared (coalesced rows),
      // read back per (lane = layer, column) without bank conflicts
      float* ibs = ib_s + acc * R * IBS;
      for (uint32_t k = et; k < R * BN; k += EPI_THREADS) {
        const uint32_t r = k / BN, c = k - r * BN;
        const uint32_t p = n * BN + c;
        ibs[r * IBS + c] = (r < a.L && p < a.P) ? __ldg(a.ibT + (uint64_t)r * a.cap + p) : 0.f;
      }
#endif
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const uint32_t q = m * (BM >> LOGR) + qg;
      const bool qvalid = q < a.Q;
      const bool rvalid = qvalid && l < a.L;
      const float ia = rvalid ? a.ia[(uint64_t)q * a.L + l] : 0.f;
      const uint64_t zq = qvalid ? a.zq[q] : 0ull;
      const float* ibl = a.ibT + (uint64_t)(rvalid ? l : 0) * a.cap;
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      fence_after();
      const uint32_t tbase = tmem + ((quarter * 32) << 16) + acc * BN + half * 128;
      const uint32_t p0 = n * BN + half * 128;
      float dv[4 * VPL];
      float rmin = __uint_as_float(kFInf);
#pragma unroll
      for (uint32_t c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(tbase + c * 32, r);
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const uint32_t p = p0 + c * 32 + j;
#if I8_IB_STAGE
          const float ib = ibs[l * IBS + half * 128 + c * 32 + j];
          (void)ibl;
          (void)p;
#else
          const float ib = (rvalid && p < a.P) ? __ldg(ibl + p) : 0.f;
#endif
          v[j] = __uint2float_rn(r[j]) * ia * ib;
        }
        group_sum_transpose<LOGR>(v, lane);
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          const uint32_t col = c * 32 + gl * VPL + k;  // within this half
          const uint32_t p = p0 + col;
          const float sim = v[k] + (float)__popcll(zq & zt[half * 128 + col]);
          const float d = fmaxf(fmaf(-sim, a.invL, 1.0f), 0.0f);
          dv[c * VPL + k] = (qvalid && p < a.P) ? d : __uint_as_float(kFInf);
          rmin = fminf(rmin, dv[c * VPL + k]);
        }
      }
      fence_before();
      mbar_arrive(&tempty[acc]);  // accumulator drained: the MMA may reuse it
      // per-probe minimum over the group's lanes -> global threshold
#pragma unroll
      for (int o = 1; o < (int)R; o <<= 1) rmin = fminf(rmin, __shfl_xor_sync(0xffffffffu, rmin, o));
      uint32_t tv = 0;
      if (qvalid && gl == 0) {
        const uint32_t mb = __float_as_uint(rmin);
        tv = *reinterpret_cast<volatile uint32_t*>(&a.T[q]);
        if (mb < tv) tv = min(atomicMin(&a.T[q], mb), mb);
      }
      tv = __shfl_sync(0xffffffffu, tv, lane & ~(R - 1));  // all lanes: warp-collective
      const float thr = qvalid ? __uint_as_float(tv) + a.eps2 : -1.f;
#pragma unroll
      for (uint32_t c = 0; c < 4; ++c)
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          const float d = dv[c * VPL + k];
          if (d <= thr) {
            const uint32_t p = p0 + c * 32 + gl * VPL + k;
            const uint32_t pos = atomicAdd(&a.bcnt[q], 1u);
            if (pos < a.bcap) a.bucket[(uint64_t)q * a.bcap + pos] = make_uint2(p, __float_as_uint(d));
          }
        }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

// Block-diagonal A: row (q, l) <- probe q's layer-l packed row at K offset l*RB.
__global__ void k_blockdiag(const uint8_t* packed, uint32_t Q, uint32_t L, uint32_t RB,
                            uint32_t logR, uint32_t Kp, uint32_t rows, uint8_t* A) {
  pdl_wait();
  pdl_trigger();
  const uint32_t R = 1u << logR;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)rows * Kp / 16;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t row = (uint32_t)(i / (Kp / 16));
    const uint32_t kc = (uint32_t)(i % (Kp / 16)) * 16;
    const uint32_t q = row >> logR, l = row & (R - 1);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (q < Q && l < L && kc >= l * RB && kc < (l + 1) * RB)
      v = *reinterpret_cast<const uint4*>(packed + ((uint64_t)q * L + l) * RB + (kc - l * RB));
    *reinterpret_cast<uint4*>(A + (uint64_t)row * Kp + kc) = v;
  }
}

cudaError_t encode_2d_u8(const void* base, uint64_t rows, uint64_t cols, uint64_t pitch,
                         uint32_t box_rows, CUtensorMap* map) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult qr;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
    if (e != cudaSuccess || qr != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {pitch};
  const cuuint32_t box[2] = {(cuuint32_t)BKB, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int LOGR>
cudaError_t launch_t(const CUtensorMap& ta, const CUtensorMap& tb, const I8Args& a, uint32_t grid,
                     size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_tci8_screen<LOGR>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(k_tci8_screen<LOGR>, dim3(grid), dim3(THREADS), smem, st, ta, tb, a);
}

}  // namespace

bool i8_supported(const DevColl& c) { return c.cb == 1 && c.L <= 32; }

size_t i8_blockdiag_bytes(const DevColl& c, uint32_t Q) {
  uint32_t logR = 0;
  while ((1u << logR) < c.L) ++logR;
  const uint32_t per_tile = BM >> logR;
  const uint32_t n_m = (Q + per_tile - 1) / per_tile;
  const uint64_t Kp = ((uint64_t)c.L * c.RB + BKB - 1) / BKB * BKB;
  return (size_t)n_m * BM * Kp;
}

cudaError_t launch_tci8_screen(const DevColl& c, const DevProbes& pr, const MatchWork& w,
                               uint8_t* blockdiag, int n_sm, cudaStream_t st) {
  if (c.size == 0 || pr.Q == 0) return cudaSuccess;
  uint32_t logR = 0;
  while ((1u << logR) < c.L) ++logR;
  const uint32_t per_tile = BM >> logR;
  const uint32_t n_m = (pr.Q + per_tile - 1) / per_tile;
  const uint32_t K = c.L * c.RB;
  const uint32_t Kp = (K + BKB - 1) / BKB * BKB;
  const uint32_t rows = n_m * BM;
  cudaError_t e = launch_pdl(
      k_blockdiag, dim3(std::min<uint32_t>((uint32_t)((uint64_t)rows * Kp / 16 / 256) + 1, 1024)),
      dim3(256), 0, st, (const uint8_t*)pr.packed, (uint32_t)pr.Q, c.L, c.RB, logR, Kp, rows,
      blockdiag);
  if (e != cudaSuccess) return e;
  struct MapCache {
    const void* base = nullptr;
    uint64_t rows = 0, cols = 0;
    CUtensorMap map;
  };
  static thread_local MapCache ca, cb;
  if (ca.base != blockdiag || ca.rows != rows || ca.cols != Kp) {
    e = encode_2d_u8(blockdiag, rows, Kp, Kp, BM, &ca.map);
    if (e != cudaSuccess) return e;
    ca.base = blockdiag;
    ca.rows = rows;
    ca.cols = Kp;
  }
  if (cb.base != c.counts || cb.rows != c.cap || cb.cols != K) {
    e = encode_2d_u8(c.counts, c.cap, K, K, BN, &cb.map);
    if (e != cudaSuccess) return e;
    cb.base = c.counts;
    cb.rows = c.cap;
    cb.cols = K;
  }
  I8Args a{};
  a.ia = pr.ia;
  a.ibT = c.ibT;
  a.zq = pr.zmask;
  a.zp = c.zmask;
  a.cap = c.cap;
  a.Q = pr.Q;
  a.P = c.size;
  a.L = c.L;
  a.R = 1u << logR;
  a.n_m = n_m;
  a.n_n = (c.size + BN - 1) / BN;
  a.n_k = Kp / BKB;
  a.invL = 1.0f / (float)c.L;
  a.eps2 = w.eps2;
  a.T = w.T;
  a.bcnt = w.bcnt;
  a.bucket = w.bucket;
  a.bcap = w.bcap;
  const size_t smem = (size_t)STAGES * STAGE_BYTES + 2 * BN * 8 +
                      (I8_IB_STAGE ? (2 * (size_t)(1u << logR) * IBS) * 4 : 0) +
                      (2 * STAGES + 4) * 8 + 16;
  const uint32_t grid = std::min<uint32_t>(a.n_m * a.n_n, (uint32_t)n_sm);
  switch (logR) {
    case 0: return launch_t<0>(ca.map, cb.map, a, grid, smem, st);
    case 1: return launch_t<1>(ca.map, cb.map, a, grid, smem, st);
    case 2: return launch_t<2>(ca.map, cb.map, a, grid, smem, st);
    case 3: return launch_t<3>(ca.map, cb.map, a, grid, smem, st);
    case 4: return launch_t<4>(ca.map, cb.map, a, grid, smem, st);
    case 5: return launch_t<5>(ca.map, cb.map, a, grid, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace moe
