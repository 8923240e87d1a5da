// trace.cu -- K1: router top-k ids -> per-request L x E expert-activation
// counts (Eam::record, eam.cpp:41-52, driven per token as
// workload.cpp:166-181 does), accumulated straight into the caller's counts.
//
// Three kernels share one contract.  All-or-nothing (eam.cpp:42-47: every
// index is validated before any count moves): an out-of-range id is skipped
// and raises *bad; a second, gated launch of the same kernel then runs only
// when *bad is set and subtracts exactly what the first added (same items,
// same skips; unsigned arithmetic is exact modulo 2^32 / 2^64), so a failed
// call leaves counts as it found them.  The gated launch costs one empty grid
// on the success path.  No kernel keeps a global scratch histogram: each adds
// its shared-memory partial straight into the caller's counts once.
//
// k_trace_lane (u8 ids, L*k even, E <= 256, requests of >= 16 tokens on
// average; the DS case): bank-locked private counters fed by a bulk-copy
// ring -- see its comment below.  Any request length.
//
// k_trace_own (other u8 shapes whose L x E histogram fits): a block owns whole
// requests (<= 16,384 tokens) and adds its shared histogram straight into
// counts[r].  The id stream is read in aligned 16-byte chunks; 16*CH bytes =
// lcm(L*k, 16) hold a whole number of tokens, so the histogram row of byte j
// of chunk i depends only on (i mod CH, j): each thread keeps its 16 row
// addresses in registers and, per id, does PRMT + LEA + RED.shared (~3.3
// wavefronts each: random banks).  The range check is a SWAR test per word.
//
// k_trace_gen (u16/u32 ids, any alignment, wide shapes, and k_trace_own's long
// requests): work items are (token chunk, layer group) pairs; per item the
// block processes every request piece (request r intersected with the chunk)
// and flushes that piece's histogram into counts[r] -- plain read-modify-write
// when the chunk holds the whole request, global atomics when it spans chunks.
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

// ---- k_trace_lane: bank-locked private counters fed by a bulk-copy ring ----
//
// The id stream is cut into items of TS tokens (one per block), an item into
// pieces (request r intersected with the item) and a piece into stages of at
// most TW whole tokens; the last G stages of a piece are of equal size.  One
// producer thread streams the stages through shared-memory ring slots
// (cp.async.bulk of the 16-byte aligned window, completion on an mbarrier), so
// the loads in flight do not depend on registers.
//
// Consumer warps form G groups; group g takes every G-th stage of the item and
// owns the ring slots g, g + G, ... (one consumer group per slot: a group's
// wait for the n-th use of a slot cannot alias an earlier use by mbarrier
// parity, however far the groups drift apart).  Inside a group, thread
// tg = tp * H + q (H = L*k / 2 position pairs) owns the id positions 2q, 2q+1
// of the stage's tokens j = tp (mod TPg): it reads them as one u16 and adds 1
// (position 2q) or 0x10000 (position 2q+1) into the counter word of its column
// for expert e, cnt[e][col].  A column belongs to one lane position of one
// warp in every group (col = tg mod C), so the 32 lanes of a warp always hit
// 32 distinct banks -- one wavefront per RED.shared, where a shared L x E
// histogram takes ~3.3 (k_trace_own).  Ids >= E are clamped into a trash row
// (nonzero -> the call's flag), masked tail slots into a null row.  A 16-bit
// half counts at most one id per token of a piece and pieces are at most
// TS <= 65,535 tokens, so halves never carry.
//
// At a piece's end (every group has counted its stages of it: a named barrier
// over all consumers) the consumers reduce the counters into counts[r]: per
// (layer, expert) cell the halves of the layer's positions (and the token
// phases' columns) are summed into a padded staging row, the counters are
// zeroed, and the staged cells are added into counts[r] with coalesced
// reductions (RED: no thread waits on the counts' latency; a read-modify-write
// pass cost ~2 us per piece).  The rollback launch subtracts the same sums
// (see gate_open).
//
// Measured (DS, 1M tokens, scripts/trace_probe.py): ~0.15 ms at 1,000
// requests (k_trace_own: 0.190 ms), ~0.12 ms at 50 requests of 20k tokens
// (k_trace_own + k_trace_gen: 1.95 ms).  The remaining gap to HBM is issue
// (~10 instructions per u16 of ids) and the per-piece reduction.
constexpr int kLaneU = 16;  // tokens per thread and unrolled round
constexpr uint32_t kLaneMaxGroups = 19;  // consumer warps at most (one per group when H <= 32)

struct LaneArgs {
  const uint8_t* topk;
  uint64_t T, TS;
  const uint64_t* offsets;
  uint64_t R;
  uint32_t L, E, k, H;
  uint32_t TPg, NWg, G;  // token phases per group, warps per group, groups
  uint32_t C, NCOL;      // counter columns (thread tg uses column tg mod C), padded to 32
  uint32_t TW, NSTG, SB; // tokens per stage, ring slots, slot bytes
  int* bad;
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumers_sync(uint32_t n) {
  asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory");
}

// Effective token range of item ii: tokens outside [offsets[0], offsets[R])
// belong to no request and are neither streamed nor counted.
__device__ __forceinline__ bool lane_item(const LaneArgs& a, uint64_t ii, uint64_t lo, uint64_t hi,
                                          uint64_t* ta, uint64_t* tb) {
  *ta = max(ii * a.TS, lo);
  *tb = min(min(a.T, ii * a.TS + a.TS), hi);
  return *ta < *tb;
}

// The request holding token ta (the first one whose end lies beyond it).
__device__ __forceinline__ uint64_t lane_first_request(const LaneArgs& a, uint64_t ta) {
  uint64_t l0 = 0, h0 = a.R;
  while (l0 < h0) {
    const uint64_t mid = (l0 + h0) / 2;
    if (a.offsets[mid + 1] <= ta) l0 = mid + 1; else h0 = mid;
  }
  return l0;
}
// The next non-empty request after r, which ended at token pe.
__device__ __forceinline__ uint64_t lane_next_request(const LaneArgs& a, uint64_t r, uint64_t pe) {
  while (r + 1 < a.R && a.offsets[r + 2] <= pe) ++r;
  return r + 1;
}

// Stages of a piece of n tokens: full stages of TW tokens, then the last G of
// equal size (all of them, G at most, when the piece holds <= G*TW tokens), so
// that the G groups, which take every G-th stage, reach the piece's end
// together.
__device__ __forceinline__ uint32_t piece_stages(uint32_t n, uint32_t TW, uint32_t G) {
  const uint32_t full = (n + TW - 1) / TW;
  return full <= G ? min(G, n) : full;
}
__device__ __forceinline__ void piece_stage(uint32_t n, uint32_t TW, uint32_t G, uint32_t j,
                                            uint32_t* st, uint32_t* en) {
  const uint32_t full = (n + TW - 1) / TW;
  if (full <= G) {
    const uint32_t m = min(G, n);
    *st = n * j / m;
    *en = n * (j + 1) / m;
    return;
  }
  const uint32_t head = full - G, t0 = head * TW, tail = n - t0;
  if (j < head) {
    *st = j * TW;
    *en = *st + TW;
  } else {
    *st = t0 + tail * (j - head) / G;
    *en = t0 + tail * (j - head + 1) / G;
  }
}

// The consumers' reduction of one request piece into counts[r].
template <typename OUT>
__device__ __forceinline__ void lane_flush(const LaneArgs& a, uint32_t* cnt, uint32_t* stage_out,
                                           uint32_t NC, OUT* dst, int sign) {
  const uint32_t t = threadIdx.x, L = a.L, E = a.E, k = a.k, ES = E | 1, NCOL = a.NCOL;
  consumers_sync(NC);
  const uint32_t CM = a.C / a.H;  // columns per position pair
  // whole words per layer, one column each: a cell's words belong to it alone,
  // so the reader zeroes them (no separate zeroing pass, one barrier less)
  const bool own = CM == 1 && (k & 1) == 0 && k <= 8;
  {  // cell (l, e), layer fastest: conflict-free reads
    const uint32_t de = NC / L, dl = NC - de * L;
    uint32_t e = t / L, l = t - e * L;
    if (own) {
      const uint32_t kh = k >> 1;
      for (; e < E;) {
        uint32_t* cw = cnt + e * NCOL + l * kh;
        uint32_t c[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) c[w] = w < (int)kh ? cw[w] : 0u;
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (w < (int)kh) cw[w] = 0u;
        uint32_t sum = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) sum += (c[w] & 0xffffu) + (c[w] >> 16);
        stage_out[l * ES + e] = sum;
        l += dl;
        e += de;
        if (l >= L) l -= L, ++e;
      }
    } else {
      for (; e < E;) {
        const uint32_t p0 = l * k, p1 = p0 + k;
        uint32_t sum = 0;
        for (uint32_t w = p0 >> 1; w < (p1 + 1) >> 1; ++w) {
          const bool lo_in = 2 * w >= p0, hi_in = 2 * w + 1 < p1;
          for (uint32_t m = 0; m < CM; ++m) {
            const uint32_t c = cnt[e * NCOL + m * a.H + w];
            sum += (lo_in ? (c & 0xffffu) : 0u) + (hi_in ? (c >> 16) : 0u);
          }
        }
        stage_out[l * ES + e] = sum;
        l += dl;
        e += de;
        if (l >= L) l -= L, ++e;
      }
    }
  }
  if (own) {  // the trash row (ids >= E) and the null row (masked slots)
    for (uint32_t i = t; i < 2 * NCOL; i += NC) {
      if (i < NCOL && cnt[E * NCOL + i] != 0 && sign > 0) *a.bad = 1;
      cnt[E * NCOL + i] = 0u;
    }
    consumers_sync(NC);
  } else {
    for (uint32_t i = t; i < NCOL; i += NC)  // the trash row: ids >= E
      if (cnt[E * NCOL + i] != 0 && sign > 0) *a.bad = 1;
    consumers_sync(NC);
    for (uint32_t i = t; i < (E + 2) * NCOL / 4; i += NC)
      reinterpret_cast<uint4*>(cnt)[i] = make_uint4(0, 0, 0, 0);
  }
  // reductions without a return value: no thread waits on the counts' latency
  {
    const uint32_t dl = NC / E, de = NC - dl * E;
    uint32_t l = t / E, e = t - l * E;
    for (uint32_t i = t; i < L * E; i += NC) {
      const uint32_t v = stage_out[l * ES + e];
      if (v) add_out(dst + i, v, sign, false);
      l += dl;
      e += de;
      if (e >= E) e -= E, ++l;
    }
  }
  // with own: the counters are zero since the barrier above, and the staging
  // row is rewritten only after the next flush's first barrier
  if (!own) consumers_sync(NC);
}

template <typename OUT>
__global__ void __launch_bounds__(640, 1) k_trace_lane(LaneArgs a, OUT* __restrict__ counts, int mode, int sign) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t NC = a.G * a.NWg * 32;  // consumer threads (whole warps)
  const uint32_t t = threadIdx.x;
  const uint32_t L = a.L, E = a.E, Lk = L * a.k, ES = E | 1, NCOL = a.NCOL;
  uint8_t* ring = sm;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sm + (size_t)a.NSTG * a.SB);  // [E + 2][NCOL]
  uint32_t* stage_out = cnt + (size_t)(E + 2) * NCOL;                       // [L][ES]
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_out + (((size_t)L * ES + 1) & ~(size_t)1));
  uint64_t* empty = full + a.NSTG;
  if (t == 0) {
    for (uint32_t s = 0; s < a.NSTG; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], a.NWg);  // the stage's group
    }
    fence_mbar_init();
  }
  if (mode == kRun)  // zeroing overlaps the previous grid's tail
    for (uint32_t i = t; i < (E + 2) * NCOL / 4; i += blockDim.x)
      reinterpret_cast<uint4*>(cnt)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  pdl_wait();
  if (!gate_open(a.bad, mode)) return;  // rollback launch on a clean call
  if (mode != kRun) {
    for (uint32_t i = t; i < (E + 2) * NCOL / 4; i += blockDim.x)
      reinterpret_cast<uint4*>(cnt)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
  }
  const uint64_t lo = a.offsets[0], hi = a.offsets[a.R];
  const uint64_t n_items = (a.T + a.TS - 1) / a.TS;
  const uintptr_t base = reinterpret_cast<uintptr_t>(a.topk);
  if (t >= NC) {  // producer warp: one thread streams the stages in order
    if (t == NC) {
      // group g owns slots g, g + G, ...: each slot has one consumer group, so
      // a group's wait for the n-th use of its slot cannot alias an earlier,
      // still incomplete use (mbarrier parity) however far other groups lag
      uint32_t used[kLaneMaxGroups];  // stages issued per group so far
      for (uint32_t i = 0; i < a.G; ++i) used[i] = 0;
      const uint32_t D = a.NSTG / a.G;  // slots per group
      for (uint64_t ii = blockIdx.x; ii < n_items; ii += gridDim.x) {
        uint64_t ta, tb;
        if (!lane_item(a, ii, lo, hi, &ta, &tb)) continue;
        uint64_t r = lane_first_request(a, ta), ps = ta;
        uint32_t k = 0;
        while (ps < tb) {  // pieces: request r intersected with the item
          const uint64_t rend = a.offsets[r + 1], pe = min(rend, tb);
          const uint32_t n = (uint32_t)(pe - ps), m = piece_stages(n, a.TW, a.G);
          for (uint32_t j = 0; j < m; ++j, ++k) {
            uint32_t st, en;
            piece_stage(n, a.TW, a.G, j, &st, &en);
            const uintptr_t g0 = (base + (ps + st) * Lk) & ~(uintptr_t)15;
            const uintptr_t g1 = (base + (ps + en) * Lk + 15) & ~(uintptr_t)15;
            const uint32_t gg = k % a.G, u = used[gg]++;
            const uint32_t s = gg + a.G * (u % D), ph = (u / D) & 1u;
            mbar_wait(&empty[s], ph ^ 1u);
            mbar_arrive_expect_tx(&full[s], (uint32_t)(g1 - g0));
            bulk_g2s(ring + (size_t)s * a.SB, reinterpret_cast<const void*>(g0),
                     (uint32_t)(g1 - g0), &full[s]);
          }
          ps = pe;
          if (pe == rend) r = lane_next_request(a, r, pe);
        }
      }
    }
    return;
  }
  const uint32_t lane = t & 31, g = (t >> 5) / a.NWg, tg = t - g * a.NWg * 32;
  const bool act = tg < a.H * a.TPg;
  const uint32_t tp = act ? tg / a.H : 0, q = act ? tg - tp * a.H : 0;
  const uint32_t my = smem_u32(cnt) + 4u * (tg % a.C), rowE = 4u * NCOL;  // expert e: my + e * rowE
  const uint32_t Eh = E, dj = a.TPg * Lk;
  const uint32_t D = a.NSTG / a.G;  // this group's slots: g, g + G, ... (see the producer)
  uint32_t used = 0;                // stages this group has taken so far
  for (uint64_t ii = blockIdx.x; ii < n_items; ii += gridDim.x) {
    uint64_t ta, tb;
    if (!lane_item(a, ii, lo, hi, &ta, &tb)) continue;
    uint64_t r = lane_first_request(a, ta), ps = ta;
    uint32_t k = 0;  // stages of the item so far; group g takes k = g (mod G)
    while (ps < tb) {
      const uint64_t rend = a.offsets[r + 1], pe = min(rend, tb);
      const uint32_t n = (uint32_t)(pe - ps), m = piece_stages(n, a.TW, a.G);
      for (uint32_t j = (g + a.G - k % a.G) % a.G; j < m; j += a.G) {
        const uint32_t s = g + a.G * (used % D), ph = (used / D) & 1u;
        ++used;
        uint32_t st, en;
        piece_stage(n, a.TW, a.G, j, &st, &en);
        mbar_wait(&full[s], ph);
        if (act) {  // the stage's tokens jj in [0, en - st), phase tp takes jj = tp (mod TPg)
          const uint32_t jy = en - st;
          const uint8_t* pj = ring + s * a.SB + ((uint32_t)(base + (ps + st) * Lk) & 15u) + 2u * q +
                              tp * Lk;
          uint32_t jj = tp;
          constexpr int U = kLaneU;
          for (; jj + (U - 1) * a.TPg < jy; jj += U * a.TPg, pj += U * dj) {
            uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = *reinterpret_cast<const uint16_t*>(pj + u * dj);
#pragma unroll
            for (int u = 0; u < U; ++u) {  // ids >= E land in the trash row E
              const uint32_t e0 = min(v[u] & 0xffu, Eh), e1 = min(v[u] >> 8, Eh);
              asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(my + e0 * rowE));
              asm volatile("red.shared.add.u32 [%0], 65536;" ::"r"(my + e1 * rowE));
            }
          }
          if (jj < jy) {  // tail: one masked round, the masked slots count into the null row
            uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u)  // masked slots re-read the first slot (inside the stage)
              v[u] = *reinterpret_cast<const uint16_t*>(jj + u * a.TPg < jy ? pj + u * dj : pj);
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const bool in = jj + u * a.TPg < jy;
              const uint32_t e0 = in ? min(v[u] & 0xffu, Eh) : Eh + 1;
              const uint32_t e1 = in ? min(v[u] >> 8, Eh) : Eh + 1;
              asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(my + e0 * rowE));
              asm volatile("red.shared.add.u32 [%0], 65536;" ::"r"(my + e1 * rowE));
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      k += m;
      // the piece's end: every group has counted its stages of it
      lane_flush<OUT>(a, cnt, stage_out, NC, counts + r * (uint64_t)L * E, sign);
      ps = pe;
      if (pe == rend) r = lane_next_request(a, r, pe);
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

// k_trace_lane's shape: u8 ids, an even number of ids per token, E <= 256 and
// the private counters in shared memory; requests of at least 16 tokens on
// average (each piece costs one L x E reduction).  MOE_TRACE_LANE=0 disables
// it (A/B runs).
bool lane_config(uint64_t T, uint32_t L, uint32_t E, uint32_t k, uint64_t R, int n_sm, LaneArgs* a,
                 size_t* smem, unsigned* grid) {
  static const bool off = [] {
    const char* e = getenv("MOE_TRACE_LANE");
    return e && e[0] == '0';
  }();
  const uint32_t Lk = L * k;
  if (off || Lk == 0 || Lk % 2 || E == 0 || E > 256 || T < 16 * R) return false;
  const size_t kMax = 227u * 1024u;
  constexpr uint32_t kMaxWarps = kLaneMaxGroups;  // consumer warps (+ the producer warp: <= 640 threads)
  const uint32_t H = Lk / 2, ES = E | 1;
  if (H > kMaxWarps * 32) return false;
  // a group: the warps holding every position pair once (several token phases
  // when a warp holds more than H lanes); columns are shared by the groups
  const uint32_t NWg = (H + 31) / 32, TPg = NWg * 32 / H;
  const uint32_t C = H >= 32 ? H : H * TPg;
  const uint32_t NCOL = (C + 31) / 32 * 32;
  const size_t cnt_b = (size_t)(E + 2) * NCOL * 4;  // + the trash and null rows
  const size_t out_b = (((size_t)L * ES + 1) & ~(size_t)1) * 4;
  const size_t fixed = cnt_b + out_b;
  const uint32_t UT = kLaneU * TPg;  // tokens of one unrolled round of every phase
  const size_t sb_min = (((size_t)UT * Lk + 32) + 127) & ~(size_t)127;
  if (fixed + 2 * (sb_min + 16) + 256 > kMax) return false;
  const size_t ring = kMax - fixed - 256;
  // groups: as many as the warp budget allows with two ring slots each
  uint32_t G = std::max<uint32_t>(1, kMaxWarps / NWg);
  while (G > 1 && (size_t)(2 * G) * (sb_min + 16) > ring) --G;
  // tokens per stage: <= 24 KB, two slots per group (slots belong to groups;
  // one group of 18 warps with 3 token phases per stage instead of 3 groups
  // measured 0.177 vs 0.153 ms at DS)
  const size_t sb_max = std::min<size_t>(24576 + 160, ring / (2 * G) - 16);
  uint32_t TW = (uint32_t)std::max<size_t>(UT, (sb_max - 160) / Lk / UT * UT);
  const uint32_t SB = (uint32_t)((((size_t)TW * Lk + 32) + 127) & ~(size_t)127);
  const uint32_t D = (uint32_t)std::min<size_t>(64 / G, ring / (SB + 16) / G);  // slots per group
  if (D < 2) return false;
  const uint32_t NSTG = D * G;
  *smem = (size_t)NSTG * SB + fixed + 16 * (size_t)NSTG;
  *grid = (unsigned)n_sm;  // one block per SM
  // one item per block (equal token counts; each piece costs one reduction)
  uint64_t TS = (T + *grid - 1) / *grid;
  TS = std::min<uint64_t>(std::max<uint64_t>(TS, TW), 65535);
  *grid = (unsigned)std::min<uint64_t>(*grid, (T + TS - 1) / TS);
  a->T = T;
  a->TS = TS;
  a->R = R;
  a->L = L;
  a->E = E;
  a->k = k;
  a->H = H;
  a->TPg = TPg;
  a->NWg = NWg;
  a->G = G;
  a->C = C;
  a->NCOL = NCOL;
  a->TW = TW;
  a->NSTG = NSTG;
  a->SB = SB;
  return true;
}

template <typename OUT>
cudaError_t launch_trace_t(const void* topk, int idx_bytes, uint64_t T, uint32_t L, uint32_t E,
                           uint32_t k, const uint64_t* offsets, uint64_t R, OUT* counts, int* bad,
                           int n_sm, cudaStream_t st) {
  if (T == 0 || R == 0) return cudaSuccess;
  if (idx_bytes == 1) {
    LaneArgs a;
    size_t smem;
    unsigned grid;
    if (lane_config(T, L, E, k, R, n_sm, &a, &smem, &grid) &&
        (reinterpret_cast<uintptr_t>(topk) & 1) == 0) {
      a.topk = static_cast<const uint8_t*>(topk);
      a.offsets = offsets;
      a.bad = bad;
      static size_t set = 0;
      cudaError_t e = raise_smem(k_trace_lane<OUT>, smem, &set);
      if (e != cudaSuccess) return e;
      const unsigned threads = a.G * a.NWg * 32 + 32;
      e = launch_pdl(k_trace_lane<OUT>, dim3(grid), dim3(threads), smem, st, a, counts, (int)kRun, 1);
      if (e == cudaSuccess)  // rollback: any grid subtracts the same sums
        e = launch_pdl(k_trace_lane<OUT>, dim3(std::min<unsigned>(grid, 16)), dim3(threads), smem,
                       st, a, counts, (int)kIfBad, -1);
      if (e != cudaSuccess) return e;
      return cudaGetLastError();
    }
  }
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
