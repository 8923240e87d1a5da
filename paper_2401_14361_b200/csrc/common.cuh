// common.cuh -- shared device helpers for the B200 (sm_100a) EAM/EAMC path:
// mbarrier + TMA (cp.async.bulk.tensor) PTX wrappers, packed-count dot
// products and the exact fp64 row-similarity epilogue.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <utility>

namespace moe {

constexpr int kNT = 128;          // entries per collection tile == threads per block
constexpr uint32_t kFInf = 0x7f800000u;
constexpr uint64_t kNone = ~0ull;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAIT;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 4-D TMA tile load global -> shared, completion counted on `bar`.
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Programmatic dependent launch.  The kernels of one match pipeline (probe
// prep -> screen -> refine -> gated exact pass -> gated merge) are launched
// with programmatic stream serialisation: grid n+1 is scheduled while grid n
// drains, runs only its shared-memory / TMEM / barrier set-up, and then
// blocks in pdl_wait() (griddepcontrol.wait returns once the preceding grid
// has completed and its writes are visible; a no-op for a normal launch).
// Every such kernel touches global memory only after pdl_wait().
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// MOE_PDL=0 disables it (A/B measurement).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("MOE_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Dot product of one 16-byte chunk of packed counts.
//  CB=1: 16 u8 counts, 4x IDP4A (u32 accumulate; exact while E*255^2 < 2^32)
//  CB=2: 8 u16 counts, u32 products accumulated in u64 (exact)
template <int CB>
struct Dot;
template <>
struct Dot<1> {
  using Acc = uint32_t;
  __device__ __forceinline__ static Acc chunk(const uint4& a, const uint4& b, Acc acc) {
    acc = __dp4a(a.x, b.x, acc);
    acc = __dp4a(a.y, b.y, acc);
    acc = __dp4a(a.z, b.z, acc);
    acc = __dp4a(a.w, b.w, acc);
    return acc;
  }
};
template <>
struct Dot<2> {
  using Acc = uint64_t;
  __device__ __forceinline__ static uint64_t w2(uint32_t a, uint32_t b) {
    return (uint64_t)((a & 0xffffu) * (b & 0xffffu)) + (uint64_t)((a >> 16) * (b >> 16));
  }
  __device__ __forceinline__ static Acc chunk(const uint4& a, const uint4& b, Acc acc) {
    return acc + w2(a.x, b.x) + w2(a.y, b.y) + w2(a.z, b.z) + w2(a.w, b.w);
  }
};

//  CB=4: 4 u32 counts, u64 products accumulated in u64.  Exact because every
//        stored row has sum c^2 < 2^53 (the reference's own exactness bound,
//        checked when rows are packed), so by Cauchy-Schwarz each dot and each
//        partial sum is < 2^53 as well.
template <>
struct Dot<4> {
  using Acc = uint64_t;
  __device__ __forceinline__ static Acc chunk(const uint4& a, const uint4& b, Acc acc) {
    return acc + (uint64_t)a.x * b.x + (uint64_t)a.y * b.y + (uint64_t)a.z * b.z +
           (uint64_t)a.w * b.w;
  }
};

// Storage-width dispatch: f<1>, f<2> or f<4> by the collection's bytes per count.
#define MOE_CB_DISPATCH(cb, F, ...) \
  ((cb) == 1 ? F<1>(__VA_ARGS__) : (cb) == 2 ? F<2>(__VA_ARGS__) : F<4>(__VA_ARGS__))

// Reference row_similarity epilogue (eam.cpp:84-86) on exact integer sums:
// both rows zero -> 1, one zero -> 0, else dot / (sqrt(na) * sqrt(nb)),
// every operation IEEE round-to-nearest, no contraction.
__device__ __forceinline__ double row_sim_exact(uint64_t dot, double sa, double sb) {
  if (sa == 0.0 && sb == 0.0) return 1.0;
  if (sa == 0.0 || sb == 0.0) return 0.0;
  if (dot == 0) return 0.0;  // +0.0 / positive: the division's exact result
  return __ddiv_rn(__ull2double_rn(dot), __dmul_rn(sa, sb));
}
// d = 1 - sim / L, clamped to [0, 1] (eam.cpp:99-103)
__device__ __forceinline__ double finish_distance(double sim, uint32_t L) {
  double d = __dsub_rn(1.0, __ddiv_rn(sim, (double)L));
  if (d < 0.0) d = 0.0;
  if (d > 1.0) d = 1.0;
  return d;
}

// Lexicographic (distance, seq) order of EamcMatch (eam.cpp:123-124, :170).
struct Best {
  double d;
  uint64_t seq;
  uint64_t idx;
};
__device__ __forceinline__ bool better(double d, uint64_t s, double bd, uint64_t bs) {
  return d < bd || (d == bd && s < bs);
}
__device__ __forceinline__ Best warp_best(Best b) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Best x;
    x.d = __shfl_xor_sync(0xffffffffu, b.d, o);
    x.seq = __shfl_xor_sync(0xffffffffu, b.seq, o);
    x.idx = __shfl_xor_sync(0xffffffffu, b.idx, o);
    if (better(x.d, x.seq, b.d, b.seq)) b = x;
  }
  return b;
}

// Exact distance of packed probe row-set `pa` vs entry `pb`, warp-cooperative
// (lane = layer), reference operation order (eam.cpp:95-103).
template <int CB>
__device__ double warp_exact_distance(const uint8_t* pa, const double* sqa, const uint8_t* pb,
                                      const double* sqb, uint32_t L, uint32_t C, uint32_t RB) {
  const uint32_t lane = threadIdx.x & 31;
  double sim = 0.0;
  for (uint32_t l0 = 0; l0 < L; l0 += 32) {
    const uint32_t l = l0 + lane;
    double r = 0.0;
    if (l < L) {
      typename Dot<CB>::Acc acc = 0;
      const uint4* ra = reinterpret_cast<const uint4*>(pa + (uint64_t)l * RB);
      const uint4* rb = reinterpret_cast<const uint4*>(pb + (uint64_t)l * RB);
      for (uint32_t c = 0; c < C; ++c) acc = Dot<CB>::chunk(ra[c], rb[c], acc);
      r = row_sim_exact((uint64_t)acc, sqa[l], sqb[l]);
    }
    const uint32_t n = min(32u, L - l0);
    for (uint32_t i = 0; i < n; ++i) sim = __dadd_rn(sim, __shfl_sync(0xffffffffu, r, i));
  }
  return finish_distance(sim, L);
}

}  // namespace moe
