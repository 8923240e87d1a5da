// trace.cu -- K1: router top-k ids -> per-request L x E expert-activation
// counts (Eam::record, eam.cpp:41-52, driven per token as
// workload.cpp:166-181 does), accumulated straight into the caller's counts.
//
// Work items are (token chunk, layer group) pairs over the id stream
// [T][L][k]: a persistent grid walks them, and inside an item the block
// processes every request piece (request r intersected with the chunk) and
// flushes that piece's histogram into counts[r] -- plain read-modify-write
// when the chunk holds the whole request (the only writer of those cells),
// global atomics when the request spans chunks.  There is no scratch
// histogram in global memory and no commit pass: the counts are written once.
//
// All-or-nothing (eam.cpp:42-47: every index is validated before any count
// moves).  An out-of-range id is skipped and raises *bad; a second, gated
// launch of the same kernel then runs only when *bad is set and subtracts
// exactly what the first added (same items, same skips; unsigned arithmetic
// is exact modulo 2^32 / 2^64), so a failed call leaves counts as it found
// them.  The gated launch costs one empty grid on the success path.
//
// k_trace_own (u8 ids, E <= 256, 16-byte aligned stream, L x E histogram in
// shared memory; the DS case): a block owns whole requests (<= 16,384
// tokens) and adds its shared histogram straight into counts[r].  The id
// stream is read in aligned 16-byte chunks; 16*CH bytes = lcm(L*k, 16) hold a
// whole number of tokens, so the histogram row of byte j of chunk i depends
// only on (i mod CH, j): each thread keeps its 16 row addresses in registers
// and, per id, does PRMT + LEA + RED.shared.  Four chunks per thread are in
// flight (a rolling register pipeline), which is what keeps HBM busy.  The
// range check is a SWAR test per word (the byte-wise __vmaxu4 is emulated on
// sm_100).  Longer requests, other index widths and shapes whose histogram
// does not fit go through k_trace_gen.
//
// Measured alternative, not kept: per-lane private counter
// copies make the shared reductions conflict-free (1.1 instead of ~3.4
// wavefronts each), but 32 copies need layer groups of ~10 layers per block,
// which cut the loads in flight per SM and added a flush per (request,
// group): 0.28 ms vs 0.19 ms for this kernel at DS.
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.cuh"

namespace moe {

namespace {

constexpr int kGenThreads = 512;
constexpr uint64_t kOwnMax = 16384;  // tokens a k_trace_own block takes whole

template <int IB>
__device__ __forceinline__ uint32_t load_id(const void* p, uint64_t i) {
  if (IB == 1) return reinterpret_cast<const uint8_t*>(p)[i];
  if (IB == 2) return reinterpret_cast<const uint16_t*>(p)[i];
  return reinterpret_cast<const uint32_t*>(p)[i];
}

template <typename OUT>
__device__ __forceinline__ void add_out(OUT* p, uint32_t v, int sign, bool owned) {
  const OUT d = sign > 0 ? (OUT)v : (OUT)0 - (OUT)v;
  if (owned)
    *p += d;
  else
    atomicAdd(p, d);
}

// Item -> token range and the first request intersecting it.
struct Item {
  uint64_t ta, tb;
  uint32_t g;
  uint64_t r0;
};

__device__ __forceinline__ Item item_of(uint64_t i, uint32_t NG, uint64_t TS, uint64_t T,
                                        const uint64_t* offsets, uint64_t R) {
  Item it;
  const uint64_t ch = i / NG;
  it.g = (uint32_t)(i - ch * NG);
  it.ta = ch * TS;
  it.tb = min(T, it.ta + TS);
  uint64_t lo = 0, hi = R;  // first request whose range ends after ta
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (offsets[mid + 1] <= it.ta) lo = mid + 1; else hi = mid;
  }
  it.r0 = lo;
  return it;
}

// Every byte of the word is a valid id (< E).  SWAR, 3 ops: with
// K = 0x01 * (128 - E) per byte (E <= 128), byte b >= E iff bit 7 of
// (b & 0x7f) + (128 - E) or of b is set; with K = 0x01 * (256 - E) (E > 128),
// iff bit 7 of b and of (b & 0x7f) + (256 - E) are both set.  No carries
// cross bytes: (b & 0x7f) + K_byte <= 255.
template <bool SMALL_E>
__device__ __forceinline__ bool word_ok(uint32_t x, uint32_t K) {
  const uint32_t t = (x & 0x7f7f7f7fu) + K;
  return ((SMALL_E ? (t | x) : (t & x)) & 0x80808080u) == 0;
}

// Launch gating through the caller's flag word: bit 0 = an out-of-range id
// was seen (the rollback launches run), bit 1 = some request is longer than
// kOwnMax (set by k_trace_own; the generic kernel's long-request pass runs).
// The last launch of a call clears bit 1.  Every kernel is PDL-launched and
// touches global memory only after pdl_wait().
enum : int { kRun = 0, kIfLong = 1, kIfBad = 2 };

__device__ __forceinline__ bool gate_open(const int* flag, int mode) {
  if (mode == kRun) return true;
  const int f = *reinterpret_cast<const volatile int*>(flag);
  return mode == kIfLong ? (f & 2) != 0 : (f & 1) != 0;
}

template <typename OUT, bool SMALL_E>
__global__ void __launch_bounds__(512)
    k_trace_own(const uint8_t* __restrict__ topk, uint32_t L, uint32_t E, uint32_t k, uint32_t CH,
                uint32_t K, const uint64_t* __restrict__ offsets, uint64_t R,
                OUT* __restrict__ counts, int* bad, int mode, int sign) {
  extern __shared__ __align__(16) uint32_t hist[];  // [L][ES]
  const uint32_t ES = E | 1;  // odd row stride
  const uint32_t Lk = L * k;
  const uint32_t stride = blockDim.x;  // a multiple of CH: thread t keeps chunk phase t mod CH
  const uint32_t t = threadIdx.x;
  const uint32_t hb = (uint32_t)__cvta_generic_to_shared(hist);
  uint32_t rowb[16];  // shared address of the histogram row of each byte of the chunk
  {
    const uint32_t pos = (16u * (t % CH)) % Lk;
    uint32_t row = pos / k, rk = pos - row * k;  // advanced without divisions
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      rowb[j] = hb + 4u * row * ES;
      if (++rk == k) {
        rk = 0;
        if (++row == L) row = 0;
      }
    }
  }
  const uint4* src = reinterpret_cast<const uint4*>(topk);
  if (mode == kRun)  // zeroing overlaps the previous grid's tail
    for (uint32_t i = t; i < L * ES; i += blockDim.x) hist[i] = 0;
  pdl_wait();
  if (!gate_open(bad, mode)) return;  // rollback launch on a clean call
  if (mode != kRun) {
    for (uint32_t i = t; i < L * ES; i += blockDim.x) hist[i] = 0;
    __syncthreads();
  }
  for (uint64_t r = blockIdx.x; r < R; r += gridDim.x) {
    const uint64_t s0 = offsets[r], s1 = offsets[r + 1];
    if (s1 - s0 > kOwnMax) {  // long: k_trace_gen's pass
      if (t == 0 && sign > 0) atomicOr(bad, 2);
      continue;
    }
    if (s1 == s0) continue;  // empty: += 0
    __syncthreads();  // the previous request's flush has re-zeroed the histogram
    const uint64_t b0 = s0 * Lk, b1 = s1 * Lk;
    const uint64_t first = b0 / 16, last = (b1 - 1) / 16;
    const uint64_t base = first - first % CH;  // whole-token aligned
    const uint4* sp = src + base;
    const uint32_t rf = (uint32_t)(first - base), rl = (uint32_t)(last - base);
    uint32_t c = t < rf ? t + stride : t;  // chunks before the request: first stride only
    constexpr int U = 4;  // rolling pipeline: chunk i + U is loaded while chunk i is counted
    uint4 w[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      w[u] = c + u * stride <= rl ? __ldg(sp + c + u * stride) : make_uint4(0, 0, 0, 0);
    for (; c <= rl; c += U * stride) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint4 cur = w[u];
        const uint32_t cu = c + u * stride, cn = cu + U * stride;
        w[u] = cn <= rl ? __ldg(sp + cn) : make_uint4(0, 0, 0, 0);
        if (cu > rl) break;
        const uint32_t v[4] = {cur.x, cur.y, cur.z, cur.w};
        const bool ok = word_ok<SMALL_E>(v[0], K) && word_ok<SMALL_E>(v[1], K) &&
                        word_ok<SMALL_E>(v[2], K) && word_ok<SMALL_E>(v[3], K);
        if (ok && cu != rf && cu != rl) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {  // hot path: PRMT + LEA + RED per id
            const uint32_t e = __byte_perm(v[j >> 2], 0u, 0x4440u | (j & 3));
            asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(rowb[j] + 4u * e));
          }
        } else {  // request-boundary chunk or an out-of-range id: per-byte tests
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const uint64_t B = (base + cu) * 16 + j;
            if (B < b0 || B >= b1) continue;
            const uint32_t e = __byte_perm(v[j >> 2], 0u, 0x4440u | (j & 3));
            if (e < E)
              asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(rowb[j] + 4u * e));
            else if (sign > 0)
              *bad = 1;
          }
        }
      }
    }
    __syncthreads();
    OUT* dst = counts + r * (uint64_t)L * E;  // this block is the only writer of counts[r]
    for (uint32_t i = t; i < L * E; i += blockDim.x) {
      const uint32_t l = i / E;
      const uint32_t v = hist[l * ES + (i - l * E)];
      if (v) {
        hist[l * ES + (i - l * E)] = 0;
        add_out(dst + i, v, sign, true);
      }
    }
  }
  pdl_trigger();
}

// Generic kernel (u8/u16/u32 ids, any alignment, any E up to ~51k): work
// items are (token chunk, layer group) pairs; per item the block processes
// every request piece (request r intersected with the chunk) into one shared
// histogram over the group's layers (odd row stride), then adds it into
// counts[r] -- plain read-modify-write when the chunk holds the whole request
// (the only writer), global atomics when the request spans chunks -- and
// re-zeroes it.  Thread = (id position in the window, token phase).  With
// min_len > 0 it takes only the requests longer than min_len (the rest
// belong to k_trace_own).
template <int IB, typename OUT>
__global__ void __launch_bounds__(kGenThreads)
    k_trace_gen(const void* __restrict__ topk, uint64_t T, uint32_t L, uint32_t E, uint32_t k,
                uint32_t G, uint32_t NG, uint64_t TS, const uint64_t* __restrict__ offsets, uint64_t R,
                OUT* __restrict__ counts, uint64_t min_len, int* bad, int mode, int clear_long, int sign) {
  extern __shared__ __align__(16) uint32_t hist[];  // [G][ES]
  const uint32_t ES = E | 1;
  const uint32_t t = threadIdx.x;
  const uint32_t Lk = L * k;
  pdl_wait();
  // the call's last launch (a kIfBad gate: bit 1 is no longer read) clears bit 1
  if (clear_long && blockIdx.x == 0 && t == 0) atomicAnd(bad, ~2);
  if (!gate_open(bad, mode)) return;
  for (uint32_t i = t; i < G * ES; i += blockDim.x) hist[i] = 0;
  const uint64_t n_items = ((T + TS - 1) / TS) * NG;
  for (uint64_t ii = blockIdx.x; ii < n_items; ii += gridDim.x) {
    const Item it = item_of(ii, NG, TS, T, offsets, R);
    const uint32_t g0 = it.g * G, g1 = min(L, g0 + G);
    const uint32_t W = (g1 - g0) * k;  // window positions per token
    const uint32_t phases = W <= blockDim.x ? blockDim.x / W : 1u;
    for (uint64_t r = it.r0; r < R; ++r) {
      const uint64_t o0 = offsets[r], o1 = offsets[r + 1];
      if (o0 >= it.tb) break;
      const uint64_t s0 = max(o0, it.ta), s1 = min(o1, it.tb);
      if (s0 >= s1 || o1 - o0 <= min_len) continue;  // empty / owned by k_trace_own
      __syncthreads();  // the previous flush has re-zeroed the histogram
      if (W > blockDim.x || t < phases * W) {
        const uint32_t phase = W <= blockDim.x ? t / W : 0u;
        for (uint32_t wi = W <= blockDim.x ? t - phase * W : t; wi < W;
             wi += W <= blockDim.x ? W : blockDim.x) {
          const uint32_t pos = g0 * k + wi;
          const uint32_t hrow = (pos / k - g0) * ES;
          constexpr int kU = 8;
          uint64_t tt = s0 + phase;
          for (; tt + (kU - 1) * (uint64_t)phases < s1; tt += kU * (uint64_t)phases) {
            uint32_t e[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) e[u] = load_id<IB>(topk, (tt + u * (uint64_t)phases) * Lk + pos);
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              if (e[u] < E) atomicAdd(&hist[hrow + e[u]], 1u);
              else if (sign > 0) *bad = 1;
            }
          }
          for (; tt < s1; tt += phases) {
            const uint32_t e = load_id<IB>(topk, tt * Lk + pos);
            if (e < E) atomicAdd(&hist[hrow + e], 1u);
            else if (sign > 0) *bad = 1;
          }
        }
      }
      __syncthreads();
      const bool owned = o0 >= it.ta && o1 <= it.tb;
      OUT* dst = counts + r * (uint64_t)L * E + (uint64_t)g0 * E;
      for (uint32_t i = t; i < (g1 - g0) * E; i += blockDim.x) {
        const uint32_t l = i / E, e = i - l * E;
        const uint32_t v = hist[l * ES + e];
        if (v) {
          hist[l * ES + e] = 0;
          add_out(dst + i, v, sign, owned);
        }
      }
    }
  }
  pdl_trigger();
}

template <typename K>
cudaError_t raise_smem(K kern, size_t smem, size_t* set) {
  if (smem <= *set) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) *set = smem;
  return e;
}

// Token chunk size: at most the piece bound of the lane-copy kernel, and small
// enough that the persistent grid gets ~8 items per block.
uint64_t chunk_tokens(uint64_t T, uint32_t NG, uint64_t slots, uint64_t cap) {
  const uint64_t want_chunks = std::max<uint64_t>(1, (slots * 8 + NG - 1) / NG);
  uint64_t ts = (T + want_chunks - 1) / want_chunks;
  ts = std::max<uint64_t>(ts, 64);
  return std::max<uint64_t>(1, std::min<uint64_t>(ts, cap));
}

template <typename OUT>
cudaError_t launch_trace_t(const void* topk, int idx_bytes, uint64_t T, uint32_t L, uint32_t E,
                           uint32_t k, const uint64_t* offsets, uint64_t R, OUT* counts, int* bad,
                           int n_sm, cudaStream_t st) {
  if (T == 0 || R == 0) return cudaSuccess;
  const uint32_t Lk = L * k;
  uint64_t min_len = 0;  // requests the generic kernel leaves to k_trace_own
  void (*own)(const uint8_t*, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t, const uint64_t*,
              uint64_t, OUT*, int*, int, int) = nullptr;
  struct { unsigned g, threads; size_t smem; uint32_t CH, K; } own_cfg = {};
  {
    uint32_t g16 = 16;
    while (Lk % g16) g16 >>= 1;
    const uint32_t CH = Lk / g16;
    const size_t smem = (size_t)L * (E | 1) * 4;
    if (idx_bytes == 1 && E <= 256 && CH <= 512 && smem <= 200u * 1024u &&
        (reinterpret_cast<uintptr_t>(topk) & 15) == 0) {
      auto kern = E <= 128 ? k_trace_own<OUT, true> : k_trace_own<OUT, false>;
      static size_t set[2] = {0, 0};
      cudaError_t e = raise_smem(kern, smem, &set[E <= 128]);
      if (e != cudaSuccess) return e;
      const uint32_t threads = (512 / CH) * CH;
      const uint32_t per_sm = std::max<uint32_t>(
          1, std::min<uint32_t>((uint32_t)((220u * 1024u) / smem), 2048u / threads));
      const unsigned g = (unsigned)std::min<uint64_t>(R, (uint64_t)n_sm * per_sm);
      const uint32_t K = 0x01010101u * (E <= 128 ? 128u - E : 256u - E);
      const uint8_t* ids = static_cast<const uint8_t*>(topk);
      e = launch_pdl(kern, dim3(g), dim3(threads), smem, st, ids, L, E, k, CH, K, offsets, R,
                     counts, bad, (int)kRun, 1);
      if (e != cudaSuccess) return e;
      own = kern;
      own_cfg = {g, threads, smem, CH, K};
      min_len = kOwnMax;
    }
  }
  // generic kernel
  const uint32_t ES = E | 1;
  const size_t budget = 100u * 1024u;
  if ((size_t)ES * 4 > 200u * 1024u) return cudaErrorInvalidValue;  // E > ~51k
  uint32_t G = (uint32_t)std::max<size_t>(1, std::min<size_t>(L, budget / ((size_t)ES * 4)));
  uint32_t NG = (L + G - 1) / G;
  G = (L + NG - 1) / NG;
  const size_t smem = (size_t)G * ES * 4;
  const uint64_t slots = (uint64_t)n_sm * std::max<uint64_t>(1, std::min<uint64_t>(4, (200u * 1024u) / smem));
  // long-requests-only mode: chunks of kOwnMax tokens (a long request spans
  // at least two, and a call without long requests costs T / kOwnMax items)
  const uint64_t TS = min_len ? kOwnMax : chunk_tokens(T, NG, slots, UINT32_MAX / std::max<uint32_t>(k, 1));
  const uint64_t n_items = ((T + TS - 1) / TS) * NG;
  const unsigned grid = (unsigned)std::min<uint64_t>(n_items, slots);
  // forward (the long-request pass only when k_trace_own flagged one), then the
  // rollback of both kernels, gated on an out-of-range id (on small grids: the
  // subtracted sums do not depend on which block takes which request)
#define MOE_TRACE_GEN(IB)                                                                       \
  {                                                                                             \
    static size_t set = 0;                                                                      \
    cudaError_t e = raise_smem(k_trace_gen<IB, OUT>, smem, &set);                               \
    if (e != cudaSuccess) return e;                                                             \
    e = launch_pdl(k_trace_gen<IB, OUT>, dim3(grid), dim3(kGenThreads), smem, st, topk, T, L, E, \
                   k, G, NG, TS, offsets, R, counts, min_len, bad, min_len ? (int)kIfLong : (int)kRun, 0, 1); \
    if (e == cudaSuccess && own)                                                                \
      e = launch_pdl(own, dim3(std::min<unsigned>(own_cfg.g, n_sm)), dim3(own_cfg.threads),     \
                     own_cfg.smem, st,                                                          \
                     static_cast<const uint8_t*>(topk), L, E, k, own_cfg.CH, own_cfg.K, offsets, R, \
                     counts, bad, (int)kIfBad, -1);                                             \
    if (e == cudaSuccess)                                                                       \
      e = launch_pdl(k_trace_gen<IB, OUT>, dim3(std::min<unsigned>(grid, n_sm)), dim3(kGenThreads), \
                     smem, st, topk, T, L, E, k, G, NG, TS, offsets, R, counts, min_len, bad,   \
                     (int)kIfBad, 1, -1);                                                       \
    if (e != cudaSuccess) return e;                                                             \
  }
  switch (idx_bytes) {
    case 1: MOE_TRACE_GEN(1) break;
    case 2: MOE_TRACE_GEN(2) break;
    case 4: MOE_TRACE_GEN(4) break;
    default: return cudaErrorInvalidValue;
  }
#undef MOE_TRACE_GEN
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_trace(const void* topk, int idx_bytes, uint64_t T, uint32_t L, uint32_t E,
                         uint32_t k, const uint64_t* offsets, uint64_t R, void* counts,
                         int count_bytes, int* bad, int n_sm, cudaStream_t st) {
  if (count_bytes == 4)
    return launch_trace_t(topk, idx_bytes, T, L, E, k, offsets, R, static_cast<uint32_t*>(counts),
                          bad, n_sm, st);
  if (count_bytes == 8)
    return launch_trace_t(topk, idx_bytes, T, L, E, k, offsets, R,
                          static_cast<unsigned long long*>(counts), bad, n_sm, st);
  return cudaErrorInvalidValue;
}

}  // namespace moe
