// decide.cu -- the fused single-probe decision kernel (K4 + K5, optional K6).
//
// One cooperative launch per engine decision (prefetch_priorities,
// policy.cpp:88-126, + the engine's floor filter, engine.cpp:663-668; with
// slot views also select_eviction_victim, policy.cpp:143-159):
//
//  phase A  distances of the probe to every entry (eam.cpp:91-104), thread
//           per entry.  The per-entry in-order layer sum over the probe rows
//           shared with the previous call is reused from pref[] (the engine
//           calls once per layer with the iteration EAM growing by one row,
//           engine.cpp:546, :587); only the probe's new nonzero rows need
//           integer dots, every other row adds 1.0 or 0.0 from the entry's
//           zero-row flag.  Block min -> atomicMin(d_min).
//  -- grid barrier --
//  phase B  window membership d <= d_min + window (the fp64 add of
//           eam.cpp:143, window = kMatchWindow, policy.hpp:30) and the u64
//           aggregation of the members' rows above the current layer
//           (policy.cpp:97-104): members compacted per CTA, their row words
//           spread over the CTA, one atomic per nonzero cell.
//  -- grid barrier --
//  phase C1 per layer i > l (CTA per layer): row sum, priorities in the
//           reference operation order (policy.cpp:108-120), floor filter,
//           survivors appended to a compact (key = ~bits(priority), flat
//           ExpertId) list.  K6: cache priorities of the slot views.
//  -- grid barrier --
//  phase C2 every survivor's output position = the number of (key, id)
//           pairs below it (ascending key = descending priority, ties by
//           ExpertId: the reference's std::sort order, policy.cpp:121-124,
//           since the pairs are unique); survivors are split over the CTAs,
//           the list is streamed through shared memory in tiles.  K6: the
//           victim argmin.
//
// Scratch state is self-cleaning: the running minimum and the survivor
// counter are double-buffered by call parity and the kernel resets the other
// half for the next call, so a decision is exactly one launch.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace moe {

namespace {

constexpr uint32_t kDecThreads = 256;

constexpr uint32_t kDecWarpsPerCta = kDecThreads / 32;

__device__ __forceinline__ bool pair_lt(unsigned long long ka, uint32_t ia, unsigned long long kb,
                                        uint32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Entry row zero?  zm (L <= 64) holds one bit per row; otherwise the row norm.
__device__ __forceinline__ bool entry_row_zero(const DecisionArgs& a, uint64_t zv, uint32_t p,
                                               uint32_t l) {
  return a.zm ? ((zv >> l) & 1ull) != 0 : a.sqb[(uint64_t)p * a.L + l] == 0.0;
}

// Grid barrier without a cooperative launch: every CTA of the (co-resident,
// one CTA per SM) grid adds 1 to a monotonically increasing counter and waits
// until it reaches base + k*G for the k-th barrier of this launch.  The host
// passes `base` (the arrivals of all earlier launches, unsigned wrap-around
// arithmetic), so the counter is never reset and an aborted launch cannot
// leave a half-reset state behind.  acq_rel/acquire at gpu scope order the
// phases' global writes and reads (and invalidate stale L1 lines).
__device__ __forceinline__ void grid_barrier(const DecisionArgs& a, uint32_t k) {
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(old) : "l"(a.bar) : "memory");
    const uint32_t target = a.bar_base + k * gridDim.x;
    uint32_t v = old + 1;
    while ((int32_t)(v - target) < 0) {
      __nanosleep(20);
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
    }
  }
  __syncthreads();
}

// Arrival without the wait: a barrier index every CTA passes but whose
// condition (no listed window members) needs no rendezvous; the arrival keeps
// the counter's targets base + k*G of the later barriers.
__device__ __forceinline__ void grid_arrive(const DecisionArgs& a) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar) : "memory");
}

__device__ __forceinline__ void stamp(const DecisionArgs& a, int i) {
  if (a.tprobe && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.tprobe[i] = t;
  }
}

// Read-only collection loads: the non-coherent path in a launch; L2 (ld.cg)
// in the persistent server, whose lifetime spans collection updates.
template <bool PS, typename T>
__device__ __forceinline__ T ld_ro(const T* p) {
  if constexpr (PS) return __ldcg(p);
  else return __ldg(p);
}
// The one-CTA server's collection reads: L1-cached plain loads.  Collection
// updates complete before a request is posted (the host drains the handle's
// stream), and the request's system-scope acquire fence (thread 0, then
// bar.sync) orders every later load of the CTA after them.
template <int MODE, typename T>
__device__ __forceinline__ T ld_col(const T* p) {
  if constexpr (MODE == 2) return *p;
  else return ld_ro<MODE == 1>(p);
}

// Column-split window aggregation over the listed members: CTA b owns the
// 16-byte chunks [q0, q1) of every member's rows above the current layer;
// thread (chunk j, member group g) accumulates its group's members (u8 counts
// in 16-bit SWAR lanes, widened every 256 members; wider counts in u64), the
// groups are reduced in shared memory (>= 16 KB of dsm) and each nonzero cell
// is added into agg with one atomic.
template <int CB, bool PS>
__device__ __forceinline__ void list_sum(const DecisionArgs& a, uint8_t* red, uint32_t NL,
                                         uint32_t rows_above) {
  const uint32_t tid = threadIdx.x, b = blockIdx.x, G = gridDim.x;
  const uint32_t E = a.E, RB = a.RB;
  const uint64_t LR = (uint64_t)a.L * RB;
  const uint32_t W4 = rows_above * (RB / 16);  // 16-byte chunks per member
  const uint32_t q0 = (uint32_t)((uint64_t)W4 * b / G), q1 = (uint32_t)((uint64_t)W4 * (b + 1) / G);
  const uint32_t nq = q1 - q0;
  if (nq == 0) return;
  constexpr uint32_t NPC = 16 / CB;  // counts per chunk
  const uint32_t ngr = kDecThreads / nq >= 1 ? kDecThreads / nq : 1;
  const uint32_t j = tid % nq, g = tid / nq;
  const bool act = nq <= kDecThreads ? g < ngr : tid < nq;
  uint64_t tot[NPC];
#pragma unroll
  for (uint32_t c = 0; c < NPC; ++c) tot[c] = 0;
  const uint8_t* rbase = a.counts + (uint64_t)(a.cur + 1) * RB;
  if (act) {
    for (uint32_t jj = j; jj < nq; jj += (nq <= kDecThreads ? nq : kDecThreads)) {
      const uint32_t q = q0 + jj;
      if (CB == 1) {
        for (uint32_t m0 = g; m0 < NL; m0 += 256 * ngr) {  // <= 256 members per widening
          uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          const uint32_t m1 = min(NL, m0 + 256 * ngr);
          uint32_t m = m0;
          constexpr int U = 8;  // loads in flight per thread
          for (; m + (U - 1) * ngr < m1; m += U * ngr) {
            uint32_t mi[U];
#pragma unroll
            for (int u = 0; u < U; ++u) mi[u] = __ldcg(a.mlist + m + u * ngr);
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
              v[u] = ld_ro<PS>(reinterpret_cast<const uint4*>(rbase + (uint64_t)mi[u] * LR) + q);
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                acc[2 * k] += w[k] & 0x00ff00ffu;
                acc[2 * k + 1] += (w[k] >> 8) & 0x00ff00ffu;
              }
            }
          }
          for (; m < m1; m += ngr) {
            const uint4 v = ld_ro<PS>(reinterpret_cast<const uint4*>(rbase + (uint64_t)__ldcg(a.mlist + m) * LR) + q);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              acc[2 * k] += w[k] & 0x00ff00ffu;
              acc[2 * k + 1] += (w[k] >> 8) & 0x00ff00ffu;
            }
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // byte 4k+i of the chunk: lane (i&1) of acc[2k + (i>>1)]
            tot[4 * k + 0] += acc[2 * k] & 0xffffu;
            tot[4 * k + 2] += acc[2 * k] >> 16;
            tot[4 * k + 1] += acc[2 * k + 1] & 0xffffu;
            tot[4 * k + 3] += acc[2 * k + 1] >> 16;
          }
        }
      } else {
        for (uint32_t m = g; m < NL; m += ngr) {
          const uint4 v = ld_ro<PS>(reinterpret_cast<const uint4*>(rbase + (uint64_t)__ldcg(a.mlist + m) * LR) + q);
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (uint32_t c = 0; c < NPC; ++c)
            tot[c] += CB == 2 ? (w[c >> 1] >> (16 * (c & 1))) & 0xffffu : w[c];
        }
      }
      if (nq > kDecThreads) {  // one thread per chunk: add directly
#pragma unroll
        for (uint32_t c = 0; c < NPC; ++c) {
          const uint32_t off = q * 16 + c * CB, r = off / RB, e = (off - r * RB) / CB;
          if (tot[c] && e < E) atomicAdd(&a.agg[(uint64_t)(a.cur + 1 + r) * E + e], (unsigned long long)tot[c]);
          tot[c] = 0;
        }
      }
    }
  }
  if (nq > kDecThreads) return;
  // reduce the member groups: red[g][j][c] (u64), then one thread per cell
  unsigned long long* rs = reinterpret_cast<unsigned long long*>(red);
  __syncthreads();
  if (act)
#pragma unroll
    for (uint32_t c = 0; c < NPC; ++c) rs[((uint64_t)g * nq + j) * NPC + c] = tot[c];
  __syncthreads();
  for (uint32_t cell = tid; cell < nq * NPC; cell += kDecThreads) {
    unsigned long long sum = 0;
    for (uint32_t gg = 0; gg < ngr; ++gg) sum += rs[(uint64_t)gg * nq * NPC + cell];
    const uint32_t jj = cell / NPC, c = cell - jj * NPC;
    const uint32_t off = (q0 + jj) * 16 + c * CB, r = off / RB, e = (off - r * RB) / CB;
    if (sum && e < E) atomicAdd(&a.agg[(uint64_t)(a.cur + 1 + r) * E + e], sum);
  }
}

// The staged survivors' flat ExpertIds (C2 with many survivors): u16 when
// L*E <= 65,536 (10 bytes per survivor with the u64 key), else u32.
struct StagedIds {
  void* p;
  bool h;
  __device__ __forceinline__ uint32_t operator[](uint32_t i) const {
    return h ? static_cast<const uint16_t*>(p)[i] : static_cast<const uint32_t*>(p)[i];
  }
  __device__ __forceinline__ void set(uint32_t i, uint32_t v) const {
    if (h) static_cast<uint16_t*>(p)[i] = (uint16_t)v;
    else static_cast<uint32_t*>(p)[i] = v;
  }
};

template <int CB, bool PS>
__device__ __forceinline__ void decision_body(const DecisionArgs& a) {
  using Acc = typename Dot<CB>::Acc;
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ uint16_t nz_s[kDecMaxNz];
  __shared__ double sqa_s[kDecMaxNz];
  __shared__ unsigned long long wmin[kDecWarpsPerCta];
  __shared__ uint32_t mem_s[kDecThreads];
  __shared__ uint32_t n_mem;
  __shared__ unsigned long long red_s[kDecWarpsPerCta];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t b = blockIdx.x, G = gridDim.x;
  const uint32_t L = a.L, E = a.E, RB = a.RB, C = RB / 16;
  const uint64_t LR = (uint64_t)L * RB;
  const uint32_t par = a.parity & 1u;
  const uint32_t rows_above = a.cur + 1 < L ? L - a.cur - 1 : 0;
  const uint64_t n_cells = (uint64_t)rows_above * E;

  // ---- phase A: distances -------------------------------------------------
  stamp(a, 0);
  if (b == 0 && tid == 0) a.dmin2[par ^ 1u] = ~0ull;  // the next call's running minimum
  if (a.do_agg)
    for (uint64_t i = (uint64_t)b * kDecThreads + tid; i < n_cells; i += (uint64_t)G * kDecThreads)
      a.agg[(uint64_t)(a.cur + 1) * E + i] = 0ull;  // used after the first barrier
  if (a.do_dist) {
  // explicit probe rows -> shared memory (from the launch parameters when
  // they fit there, else from the host-narrowed buffer), their norms
  const uint32_t n_nz = a.n_nz;
  const uint8_t* rows_src = a.rows_inline ? a.inline_rows : a.rows;
  const uint16_t* nz_src = a.rows_inline ? a.inline_nz : a.nz;
  for (uint32_t i = tid; i < n_nz; i += kDecThreads) nz_s[i] = nz_src[i];
  uint4* prow_s = reinterpret_cast<uint4*>(dsm);
  for (uint32_t i = tid; i < n_nz * C; i += kDecThreads)
    prow_s[i] = reinterpret_cast<const uint4*>(rows_src)[i];
  __syncthreads();
  for (uint32_t r = wid; r < n_nz; r += kDecWarpsPerCta) {
    uint64_t ss = 0;
    const uint8_t* row = reinterpret_cast<const uint8_t*>(prow_s) + (size_t)r * RB;
    for (uint32_t e = lane; e < E; e += 32) {
      const uint64_t c = CB == 1 ? row[e]
                         : CB == 2 ? reinterpret_cast<const uint16_t*>(row)[e]
                                   : reinterpret_cast<const uint32_t*>(row)[e];
      ss += c * c;  // exact: the host checked sum c^2 < 2^53 for every probe row
    }
    ss = warp_sum_u64(ss);
    if (lane == 0) sqa_s[r] = __dsqrt_rn(__ull2double_rn(ss));  // as k_prep
  }
  __syncthreads();
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  double dloc = kInf;
  const uint32_t chunk = (a.size + G - 1) / G;  // entries [b*chunk, (b+1)*chunk) per CTA
  const uint32_t p0 = min(a.size, b * chunk), p1 = min(a.size, p0 + chunk);
  for (uint32_t p = p0 + tid; p < p1; p += kDecThreads) {
    const uint64_t zv = a.zm ? a.zm[p] : 0ull;
    const double* sb = a.sqb + (uint64_t)p * L;
    const uint4* eb = reinterpret_cast<const uint4*>(a.counts + (uint64_t)p * LR);
    double sm = a.j0 ? a.pref[p] : 0.0;
    uint32_t k = 0;
    for (uint32_t l = a.j0; l <= a.hi && l < L; ++l) {
      double r;
      if (k < n_nz && nz_s[k] == l) {
        Acc acc = 0;
        const uint4* pr = prow_s + (size_t)k * C;
        const uint4* er = eb + (size_t)l * C;
        for (uint32_t c = 0; c < C; ++c) acc = Dot<CB>::chunk(pr[c], ld_ro<PS>(er + c), acc);
        r = row_sim_exact((uint64_t)acc, sqa_s[k], sb[l]);
        ++k;
      } else {
        r = entry_row_zero(a, zv, p, l) ? 1.0 : 0.0;
      }
      sm = __dadd_rn(sm, r);  // layer order (eam.cpp:95-98)
      if (l == a.keep) a.pref[p] = sm;
    }
    // rows above hi: zero probe rows, +1.0 per zero entry row (adding 0.0 is exact)
    if (a.zm) {
      uint64_t bits = a.hi + 1 < 64 ? zv & ~((2ull << a.hi) - 1ull) : 0ull;
      if (L < 64) bits &= (1ull << L) - 1ull;
      for (; bits; bits &= bits - 1) sm = __dadd_rn(sm, 1.0);
    } else {
      for (uint32_t l = a.hi + 1; l < L; ++l)
        if (sb[l] == 0.0) sm = __dadd_rn(sm, 1.0);
    }
    const double d = finish_distance(sm, L);
    a.dist[p] = d;
    dloc = d < dloc ? d : dloc;
  }
  {
    unsigned long long m = (unsigned long long)__double_as_longlong(dloc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, o);
      m = x < m ? x : m;
    }
    if (lane == 0) wmin[wid] = m;
    __syncthreads();
    if (tid == 0) {
      for (uint32_t w = 1; w < kDecWarpsPerCta; ++w) m = wmin[w] < m ? wmin[w] : m;
      m = wmin[0] < m ? wmin[0] : m;
      if (m != 0x7ff0000000000000ull) atomicMin(&a.dmin2[par], m);  // non-negative doubles
    }
  }
  }  // do_dist
  stamp(a, 1);
  grid_barrier(a, 1);
  stamp(a, 2);

  // ---- phase B: window members, u64 aggregation of their rows > cur --------
  if (a.do_agg && rows_above) {
    const unsigned long long dmb = a.do_dist ? a.dmin2[par] : *a.dmin_ext;
    const double thr = __dadd_rn(__longlong_as_double((long long)dmb), a.window);
    const uint32_t wpr = RB / 4;
    const uint32_t per = 4 / CB;
    const uint32_t chunk = (a.size + G - 1) / G;
    const uint32_t p0 = min(a.size, b * chunk), p1 = min(a.size, p0 + chunk);
    for (uint32_t base = p0; base < p1; base += kDecThreads) {
      if (tid == 0) n_mem = 0;
      __syncthreads();
      const uint32_t p = base + tid;
      if (p < p1 && a.dist[p] <= thr) mem_s[atomicAdd(&n_mem, 1u)] = p;
      __syncthreads();
      const uint32_t nm = n_mem;
      // many members x rows: listed, summed column-split below (one atomic per
      // nonzero count is cheaper only for a few members)
      if (a.mcount && (uint64_t)nm * rows_above * wpr > kDecListWords) {
        __shared__ uint32_t moff;
        if (tid == 0) moff = atomicAdd(a.mcount, nm);
        __syncthreads();
        for (uint32_t i = tid; i < nm; i += kDecThreads) a.mlist[moff + i] = mem_s[i];
        __syncthreads();
        continue;
      }
      const uint32_t per_mem = rows_above * wpr;
      for (uint32_t it = tid; it < nm * per_mem; it += kDecThreads) {
        const uint32_t mi = it / per_mem, rem = it - mi * per_mem;
        const uint32_t r = rem / wpr, w = rem - r * wpr;
        const uint32_t l = a.cur + 1 + r;
        const uint32_t word = ld_ro<PS>(reinterpret_cast<const uint32_t*>(
            a.counts + (uint64_t)mem_s[mi] * LR + (uint64_t)l * RB + 4ull * w));
        if (!word) continue;
#pragma unroll
        for (uint32_t j = 0; j < per; ++j) {
          const uint32_t e = w * per + j;
          const uint32_t c = CB == 1 ? (word >> (8 * j)) & 0xffu
                             : CB == 2 ? (word >> (16 * j)) & 0xffffu
                                       : word;
          if (c && e < E) atomicAdd(&a.agg[(uint64_t)l * E + e], (unsigned long long)c);
        }
      }
      __syncthreads();
    }
  }
  grid_barrier(a, 2);
  stamp(a, 3);
  // listed members (wide windows, e.g. the first layers of a decode step): CTA
  // b sums a slice of the rows-above region over every listed member -- its
  // own cells, coalesced 16-byte loads, no per-count atomics -- and adds its
  // nonzero cells into agg once
  const uint32_t NL = (a.do_agg && rows_above && a.mcount) ? __ldcg(a.mcount) : 0u;
  if (NL) {
    list_sum<CB, PS>(a, reinterpret_cast<uint8_t*>(dsm), NL, rows_above);
    grid_barrier(a, 3);
  } else {
    grid_arrive(a);
  }
  stamp(a, 4);

  // ---- phase C1: per layer i > l: priorities, floor filter, sorted segment --
  // One CTA per layer: keys (~bits(priority): ascending = priority desc) of the
  // layer's survivors, bitonic-sorted with their flat ExpertId as tie-break,
  // written to the layer's segment seg[li*E ...) with its length nseg[li].
  // Within a layer the order is the reference order restricted to that layer.
  const double kEps = 1e-4;  // policy.hpp:22
  {
    uint32_t np = 1;
    while (np < E) np <<= 1;
    unsigned long long* sk = reinterpret_cast<unsigned long long*>(dsm);
    uint32_t* si = reinterpret_cast<uint32_t*>(sk + np);
    __shared__ uint32_t n_pass;
    for (uint32_t li = b; li < rows_above; li += G) {
      const uint32_t l = a.cur + 1 + li;
      const unsigned long long* ag = a.agg + (uint64_t)l * E;
      unsigned long long sacc = 0;
      for (uint32_t e = tid; e < E; e += kDecThreads) sacc += ag[e];
      sacc = warp_sum_u64(sacc);
      if (lane == 0) red_s[wid] = sacc;
      if (tid == 0) n_pass = 0;
      __syncthreads();
      unsigned long long rsum = 0;
      for (uint32_t w = 0; w < kDecWarpsPerCta; ++w) rsum += red_s[w];
      const double prox = __dsub_rn(1.0, __ddiv_rn((double)(l - a.cur), (double)L));  // policy.cpp:110
      const double floor_p = __dmul_rn(__dmul_rn(kEps, prox), __dadd_rn(1.0, 1e-9));   // engine.cpp:666
      for (uint32_t e0 = 0; e0 < np; e0 += kDecThreads) {  // warp-uniform trip count (ballot)
        const uint32_t e = e0 + tid;
        unsigned long long key = ~0ull;
        uint32_t id = 0xffffffffu;
        if (e < E) {
          const unsigned long long av = ag[e];
          // a zero count gives priority kEps*prox, which never clears the floor
          if (!(a.filter && av == 0)) {
            const double ratio =
                rsum == 0 ? 0.0 : __ddiv_rn(__ull2double_rn(av), __ull2double_rn(rsum));
            const double pri = __dmul_rn(__dadd_rn(ratio, kEps), prox);
            if (!(a.filter && pri <= floor_p)) {
              key = ~(unsigned long long)__double_as_longlong(pri);
              id = l * E + e;
            }
          }
        }
        if (e < np) {
          sk[e] = key;
          si[e] = id;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, key != ~0ull);
        if (lane == 0 && m) atomicAdd(&n_pass, (uint32_t)__popc(m));
      }
      __syncthreads();
      const uint32_t np_l = n_pass;
      if (np <= 512) {
        // small layers: survivors compacted (ballot prefix, in expert order),
        // then each survivor's in-layer position = the number of survivor
        // (key, id) pairs below it (broadcast reads), one scatter
        unsigned long long* ck = sk + 2 * np;  // compact copies behind the slots
        uint32_t* ci = reinterpret_cast<uint32_t*>(ck + np);
        __shared__ uint32_t wofs[kDecWarpsPerCta + 1];
        for (uint32_t e0 = 0; e0 < np; e0 += kDecThreads) {
          const uint32_t e = e0 + tid;
          const bool sv = e < np && sk[e] != ~0ull;
          const uint32_t m = __ballot_sync(0xffffffffu, sv);
          if (lane == 0) wofs[wid] = __popc(m);
          __syncthreads();
          if (tid == 0) {
            uint32_t o = e0 == 0 ? 0u : wofs[kDecWarpsPerCta];
            for (uint32_t w = 0; w < kDecWarpsPerCta; ++w) {
              const uint32_t c = wofs[w];
              wofs[w] = o;
              o += c;
            }
            wofs[kDecWarpsPerCta] = o;
          }
          __syncthreads();
          if (sv) {
            const uint32_t q = wofs[wid] + __popc(m & ((1u << lane) - 1u));
            ck[q] = sk[e];
            ci[q] = si[e];
          }
          __syncthreads();
        }
        for (uint32_t i = tid; i < np_l; i += kDecThreads) {
          const unsigned long long ki = ck[i];
          const uint32_t ii = ci[i];
          uint32_t pos = 0;
          for (uint32_t j = 0; j < np_l; ++j) pos += pair_lt(ck[j], ci[j], ki, ii);
          a.ckey[(uint64_t)li * E + pos] = ki;
          a.cid[(uint64_t)li * E + pos] = ii;
          a.crank[(uint64_t)li * E + pos] = pos;
        }
        if (tid == 0) a.nseg[li] = np_l;
        __syncthreads();
        continue;
      }
      for (uint32_t k = 2; k <= np; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
          for (uint32_t i = tid; i < np; i += kDecThreads) {
            const uint32_t ixj = i ^ j;
            if (ixj > i) {
              const unsigned long long ki = sk[i], kj = sk[ixj];
              const uint32_t vi = si[i], vj = si[ixj];
              if (pair_lt(kj, vj, ki, vi) == ((i & k) == 0)) {
                sk[i] = kj;
                sk[ixj] = ki;
                si[i] = vj;
                si[ixj] = vi;
              }
            }
          }
          __syncthreads();
        }
      for (uint32_t i = tid; i < np_l; i += kDecThreads) {
        a.ckey[(uint64_t)li * E + i] = sk[i];
        a.cid[(uint64_t)li * E + i] = si[i];
        a.crank[(uint64_t)li * E + i] = i;  // its position inside its own layer
      }
      if (tid == 0) a.nseg[li] = np_l;
      __syncthreads();
    }
  }
  if (a.n_slots) {  // cache_priority of every slot view (policy.cpp:128-141)
    for (uint32_t s = b * kDecWarpsPerCta + wid; s < a.n_slots; s += G * kDecWarpsPerCta) {
      const moe_slot_view v = a.slots[s];
      unsigned long long rq = 0;
      for (uint32_t e = lane; e < E; e += 32) rq += a.req[(uint64_t)v.layer_idx * E + e];
      rq = warp_sum_u64(rq);
      if (lane == 0) {
        const double ratio =
            rq == 0 ? 0.0
                    : __ddiv_rn(__ull2double_rn(a.req[(uint64_t)v.layer_idx * E + v.expert_idx]),
                                __ull2double_rn(rq));
        const double w = __dsub_rn(1.0, __ddiv_rn((double)v.layer_idx, (double)L));
        a.slot_pri[s] = __dmul_rn(__dadd_rn(ratio, kEps), w);
      }
    }
  }
  stamp(a, 5);
  grid_barrier(a, 4);
  stamp(a, 6);

  // ---- phase C2: cross-layer ranks -----------------------------------------
  // A survivor's output position = its position in its own layer + for every
  // other layer j the number of j's (key, id) pairs below it (ascending key =
  // descending priority, ties by ExpertId: the reference's std::sort order,
  // policy.cpp:121-124; the pairs are unique).  The CTA holding layer j in
  // shared memory binary-searches every other survivor in it and adds the
  // count to that survivor's rank.
  __shared__ uint32_t offs[kDecMaxLayers + 1];
  if (rows_above > kDecMaxLayers) __trap();  // host checks the bound
  // segment offsets: all lengths loaded at once, then a serial prefix over
  // shared memory (a serial loop over global loads costs a latency per layer)
  for (uint32_t i = tid; i < rows_above; i += kDecThreads) offs[i + 1] = a.nseg[i];
  __syncthreads();
  if (tid == 0) {
    uint32_t o = 0;
    offs[0] = 0;
    for (uint32_t i = 0; i < rows_above; ++i) {
      o += offs[i + 1];
      offs[i + 1] = o;
    }
  }
  __syncthreads();
  const uint32_t S = offs[rows_above];
  if (b == 0 && tid == 0) *a.n_out = S;
  // many survivors (wide windows: every expert scores): every CTA stages the
  // whole sorted list and ranks its own share of the survivors against every
  // layer, (survivor, layer) pairs spread over the threads, then writes them
  // out -- no per-pair global atomics, no C3 pass
  uint32_t dsm_bytes;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsm_bytes));
  // flat ExpertIds as u16 when L*E <= 65,536: 10 bytes per staged survivor
  const bool id16 = (uint64_t)L * E <= 65536u;
  const bool staged = S > kDecStagedMin && (size_t)S * (id16 ? 10 : 12) <= dsm_bytes;
  if (staged) {
    unsigned long long* tk = reinterpret_cast<unsigned long long*>(dsm);
    StagedIds ti{tk + S, id16};
    __shared__ uint32_t rk[kDecThreads];
    // 12 survivors' loads in flight per thread; CTA b starts at its own offset
    // so the CTAs do not all request the same lines at once
    const uint32_t rot = (uint32_t)((uint64_t)S * b / G);
    for (uint32_t i0 = tid; i0 < S; i0 += 12 * kDecThreads) {
      unsigned long long kk[12];
      uint32_t ii[12];
#pragma unroll
      for (int u = 0; u < 12; ++u) {
        const uint32_t j = i0 + u * kDecThreads;
        if (j >= S) break;
        const uint32_t i = j + rot < S ? j + rot : j + rot - S;
        uint32_t li = 0, hi2 = rows_above;  // segment of i
        while (hi2 - li > 1) {
          const uint32_t mid = (li + hi2) >> 1;
          if (offs[mid] <= i) li = mid; else hi2 = mid;
        }
        const uint64_t slot = (uint64_t)li * E + (i - offs[li]);
        kk[u] = __ldcg(a.ckey + slot);
        ii[u] = __ldcg(a.cid + slot);
      }
#pragma unroll
      for (int u = 0; u < 12; ++u) {
        const uint32_t j = i0 + u * kDecThreads;
        if (j >= S) break;
        const uint32_t i = j + rot < S ? j + rot : j + rot - S;
        tk[i] = kk[u];
        ti.set(i, ii[u]);
      }
    }
    __syncthreads();
    const uint32_t s0 = (uint32_t)((uint64_t)S * b / G), s1 = (uint32_t)((uint64_t)S * (b + 1) / G);
    for (uint32_t c0 = s0; c0 < s1; c0 += kDecThreads) {  // chunks of <= kDecThreads survivors
      const uint32_t nc = min(kDecThreads, s1 - c0);
      if (tid < nc) {  // own position in its layer
        const uint32_t t = c0 + tid;
        uint32_t li = 0, hi2 = rows_above;
        while (hi2 - li > 1) {
          const uint32_t mid = (li + hi2) >> 1;
          if (offs[mid] <= t) li = mid; else hi2 = mid;
        }
        rk[tid] = t - offs[li];
      }
      __syncthreads();
      // layer-major pairs: the lanes of a warp search one segment (broadcast
      // reads) for different survivors (distinct rank counters)
      for (uint32_t pr = tid; pr < nc * rows_above; pr += kDecThreads) {
        const uint32_t lj = pr / nc, u = pr - lj * nc;
        const uint32_t t = c0 + u;
        if (t >= offs[lj] && t < offs[lj + 1]) continue;  // its own layer
        const unsigned long long kx = tk[t];
        const uint32_t ix = ti[t];
        uint32_t lo = offs[lj], hb = offs[lj + 1];  // count of (tk, ti) < (kx, ix)
        while (lo < hb) {
          const uint32_t mid = (lo + hb) >> 1;
          if (pair_lt(tk[mid], ti[mid], kx, ix)) lo = mid + 1; else hb = mid;
        }
        if (lo > offs[lj]) atomicAdd(&rk[u], lo - offs[lj]);
      }
      __syncthreads();
      if (tid < nc) a.crank[rk[tid]] = c0 + tid;  // the inverse: output position -> survivor
      __syncthreads();
    }
  } else {
    unsigned long long* tk = reinterpret_cast<unsigned long long*>(dsm);
    uint32_t* ti = reinterpret_cast<uint32_t*>(tk + E);
    for (uint32_t lj = b; lj < rows_above; lj += G) {
      const uint32_t nj = a.nseg[lj];
      __syncthreads();
      for (uint32_t i = tid; i < nj; i += kDecThreads) {
        tk[i] = a.ckey[(uint64_t)lj * E + i];
        ti[i] = a.cid[(uint64_t)lj * E + i];
      }
      __syncthreads();
      if (nj == 0) continue;
      // flat survivors t = offs[li] + pos, four per thread per round with their
      // loads issued together
      for (uint32_t t0 = 0; t0 < S; t0 += 4 * kDecThreads) {
        uint64_t slot[4];
        unsigned long long kx[4];
        uint32_t ix[4];
        bool act[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t t = t0 + u * kDecThreads + tid;
          uint32_t li = 0, hi2 = rows_above;  // segment of t: offs[li] <= t < offs[li+1]
          while (hi2 - li > 1) {
            const uint32_t mid = (li + hi2) >> 1;
            if (offs[mid] <= t) li = mid; else hi2 = mid;
          }
          act[u] = t < S && li != lj;
          slot[u] = (uint64_t)li * E + (t - offs[li]);
          if (act[u]) {
            kx[u] = a.ckey[slot[u]];
            ix[u] = a.cid[slot[u]];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (!act[u]) continue;
          uint32_t lo = 0, hb = nj;  // count of (tk, ti) < (kx, ix)
          while (lo < hb) {
            const uint32_t mid = (lo + hb) >> 1;
            if (pair_lt(tk[mid], ti[mid], kx[u], ix[u])) lo = mid + 1; else hb = mid;
          }
          if (lo) atomicAdd(&a.crank[slot[u]], lo);
        }
      }
    }
  }
  stamp(a, 7);
  grid_barrier(a, 5);
  // every CTA has read the listed-member count (barrier 3 < 5): clean it for
  // the next call, whatever path that takes
  if (b == 0 && tid == 0 && a.mcount) *a.mcount = 0u;

  // ---- phase C3: the output ------------------------------------------------
  // staged: CTA b writes output positions [b*S/G, (b+1)*S/G) in order from its
  // staged copy (contiguous stores: whole bursts to host-mapped memory)
  if (staged) {
    unsigned long long* tk = reinterpret_cast<unsigned long long*>(dsm);
    const StagedIds ti{tk + S, id16};
    const uint32_t r0 = (uint32_t)((uint64_t)S * b / G), r1 = (uint32_t)((uint64_t)S * (b + 1) / G);
    for (uint32_t r = r0 + tid; r < r1; r += kDecThreads) {
      const uint32_t t = __ldcg(a.crank + r), id = ti[t];
      moe_candidate o;
      o.layer_idx = id / E;
      o.expert_idx = id - o.layer_idx * E;
      o.priority = __longlong_as_double((long long)~tk[t]);
      a.out[r] = o;
    }
  } else
  for (uint32_t li = b; li < rows_above; li += G)
  for (uint32_t pos = tid; pos < offs[li + 1] - offs[li]; pos += kDecThreads) {
    const uint64_t slot = (uint64_t)li * E + pos;
    const unsigned long long key = a.ckey[slot];
    const uint32_t id = a.cid[slot];
    moe_candidate o;
    o.layer_idx = id / E;
    o.expert_idx = id - o.layer_idx * E;
    o.priority = __longlong_as_double((long long)~key);
    a.out[a.crank[slot]] = o;
  }

  if (a.n_slots && a.victim && b == G - 1) {
    // select_eviction_victim: argmin (cache_priority, ExpertId) over slots
    // neither prefetch-protected nor pinned (policy.cpp:143-159)
    double bp = 0.0;
    uint64_t bk = ~0ull;
    long long bs = -1;
    for (uint32_t i = tid; i < a.n_slots; i += kDecThreads) {
      const moe_slot_view v = a.slots[i];
      if (v.prefetch_protected || v.pinned) continue;
      const double p = a.slot_pri[i];
      const uint64_t k = ((uint64_t)v.layer_idx << 32) | v.expert_idx;
      if (bs < 0 || p < bp || (p == bp && k < bk)) {
        bp = p;
        bk = k;
        bs = (long long)v.slot;
      }
    }
    __shared__ double vp[kDecWarpsPerCta];
    __shared__ uint64_t vk[kDecWarpsPerCta];
    __shared__ long long vs[kDecWarpsPerCta];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double op = __shfl_xor_sync(0xffffffffu, bp, o);
      const uint64_t ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const long long os = __shfl_xor_sync(0xffffffffu, bs, o);
      if (os >= 0 && (bs < 0 || op < bp || (op == bp && ok < bk))) {
        bp = op;
        bk = ok;
        bs = os;
      }
    }
    if (lane == 0) {
      vp[wid] = bp;
      vk[wid] = bk;
      vs[wid] = bs;
    }
    __syncthreads();
    if (tid == 0) {
      for (uint32_t w = 1; w < kDecWarpsPerCta; ++w)
        if (vs[w] >= 0 && (bs < 0 || vp[w] < bp || (vp[w] == bp && vk[w] < bk))) {
          bp = vp[w];
          bk = vk[w];
          bs = vs[w];
        }
      *a.victim = bs;
    }
  }
}

// Small collections (size <= kSmallMaxP, (L-l-1)*E <= kSmallMaxCells): the
// whole decision in one CTA -- the same per-entry distance code, the window
// aggregation with shared-memory u64 atomics, and the order as one bitonic
// sort of all (~bits(priority), flat ExpertId) pairs in shared memory -- with
// no grid barriers and no global atomics.  (MIX: P=300, 31 x 8 candidates.)
#ifndef SMALL_ROWS_U
#define SMALL_ROWS_U 4
#endif
constexpr int kSmallRowsU = SMALL_ROWS_U;
constexpr uint32_t kSmallMaxCluster = 16;

// Byte offset of the staged row similarities r[entries][n_nz] of the cluster
// launch (after the members list; the layout of small_body's shared memory,
// see decision_small_smem).
__host__ __device__ __forceinline__ size_t small_rsim_offset(uint32_t n_nz, uint32_t RB, uint32_t size,
                                                             uint32_t N, uint32_t rows, uint32_t N2) {
  const size_t b = (((size_t)n_nz * RB + 15) & ~(size_t)15) + (size_t)size * 8 + (size_t)N * 8 +
                   (size_t)rows * 8 + (size_t)N2 * 12 + (size_t)size * 4;
  return (b + 15) & ~(size_t)15;
}  // rows per round of the per-entry loop (A/B builds)
constexpr uint32_t kSmallThreads = 512;
constexpr uint32_t kSmallWarps = kSmallThreads / 32;

template <int CB, int MODE>
__device__ __forceinline__ void small_body(const DecisionArgs& a) {
  using Acc = typename Dot<CB>::Acc;
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ uint16_t nz_s[kDecMaxNz];
  __shared__ double sqa_s[kDecMaxNz];
  __shared__ unsigned long long red_s[kSmallWarps];
  __shared__ uint32_t cnt_s[kSmallWarps + 1];
  __shared__ unsigned long long dmin_s, exm_s;
  __shared__ unsigned long long cmin_s[kSmallMaxCluster];  // per-CTA minima (cluster launch)
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t L = a.L, E = a.E, RB = a.RB, C = RB / 16;
  const uint64_t LR = (uint64_t)L * RB;
  const uint32_t rows_above = a.cur + 1 < L ? L - a.cur - 1 : 0;
  const uint32_t N = rows_above * E;
  uint32_t N2 = 1;
  while (N2 < N) N2 <<= 1;
  // shared layout: probe rows | dist[size] | agg[N] | rowsum[rows] | key[N2] | id[N2] | members
  const uint32_t n_nz = a.n_nz;
  uint4* prow_s = reinterpret_cast<uint4*>(dsm);
  double* dist_s = reinterpret_cast<double*>(dsm + ((n_nz * RB + 15) & ~15u));
  unsigned long long* agg_s = reinterpret_cast<unsigned long long*>(dist_s + a.size);
  unsigned long long* rsum_s = agg_s + N;
  unsigned long long* key_s = rsum_s + rows_above;
  uint32_t* id_s = reinterpret_cast<uint32_t*>(key_s + N2);
  uint32_t* mem_s = id_s + N2;
  stamp(a, 0);
  // ---- A: distances (the probe rows the prefix cache does not cover)
  const uint8_t* rows_src = a.rows_inline ? a.inline_rows : a.rows;
  const uint16_t* nz_src = a.rows_inline ? a.inline_nz : a.nz;
  for (uint32_t i = tid; i < n_nz; i += kSmallThreads) nz_s[i] = nz_src[i];
  for (uint32_t i = tid; i < n_nz * C; i += kSmallThreads)
    prow_s[i] = reinterpret_cast<const uint4*>(rows_src)[i];
  for (uint32_t i = tid; i < N; i += kSmallThreads) agg_s[i] = 0;
  if (tid == 0) dmin_s = ~0ull;
  __syncthreads();
  for (uint32_t r = wid; r < n_nz; r += kSmallWarps) {
    uint64_t ss = 0;
    const uint8_t* row = reinterpret_cast<const uint8_t*>(prow_s) + (size_t)r * RB;
    for (uint32_t e = lane; e < E; e += 32) {
      const uint64_t c = CB == 1 ? row[e]
                         : CB == 2 ? reinterpret_cast<const uint16_t*>(row)[e]
                                   : reinterpret_cast<const uint32_t*>(row)[e];
      ss += c * c;
    }
    ss = warp_sum_u64(ss);
    if (lane == 0) sqa_s[r] = __dsqrt_rn(__ull2double_rn(ss));
  }
  if (wid == 0 && L <= 64) {  // the explicit rows as a bit mask (no smem chain in the loop)
    unsigned long long m = 0;
    for (uint32_t i = lane; i < n_nz; i += 32) m |= 1ull << nz_s[i];
    const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)m);
    const uint32_t hi2 = __reduce_or_sync(0xffffffffu, (uint32_t)(m >> 32));
    if (lane == 0) exm_s = (unsigned long long)lo | ((unsigned long long)hi2 << 32);
  }
  __syncthreads();
  stamp(a, 4);
  // the arguments this loop reads, in registers (the server passes them in
  // shared memory)
  const uint64_t* const zm = a.zm;
  const double* const sqb = a.sqb;
  const uint8_t* const counts = a.counts;
  double* const pref = a.pref;
  const uint32_t j0 = a.j0, hi = a.hi, keep = a.keep, size = a.size;
  const auto row_zero = [&](uint64_t zv, uint32_t p, uint32_t l) {
    return zm ? ((zv >> l) & 1ull) != 0 : ld_col<MODE>(sqb + (uint64_t)p * L + l) == 0.0;
  };
  unsigned long long mloc = ~0ull;
  uint32_t crank = 0, csize = 1;  // a plain launch is a cluster of one
  if (MODE == 0) {
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  }
  if (csize > 1) {
    // Cluster launch: the fp64 row similarities (a correctly rounded division
    // each; one SM's FP64 pipe bounded the one-CTA loop) are spread over the
    // cluster.  CTA c takes the entries p = c (mod csize); its (entry,
    // explicit row) items are independent, staged as r[j][k] in its shared
    // memory, then summed per entry in layer order (eam.cpp:95-98).  The
    // distances and per-CTA minima go to CTA 0's shared memory (DSMEM), which
    // runs phases B and C alone after the cluster barrier.
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t nloc = size > crank ? (size - crank + csize - 1) / csize : 0;
    const uint32_t items = nloc * n_nz;
    double* r_s = reinterpret_cast<double*>(
        dsm + small_rsim_offset(n_nz, RB, size, N, rows_above, N2));
    if (C == 1) {  // two items per thread and round: both rows' loads in flight
      for (uint32_t i0 = tid; i0 < items; i0 += 2 * kSmallThreads) {
        uint4 ev[2];
        double sv[2];
        uint32_t kk[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t i = i0 + u * kSmallThreads;
          kk[u] = 0;
          if (i < items) {
            const uint32_t j = i / n_nz, k = i - j * n_nz, p = crank + csize * j, l = nz_s[k];
            kk[u] = k;
            ev[u] = ld_col<MODE>(reinterpret_cast<const uint4*>(counts + (uint64_t)p * LR + (uint64_t)l * RB));
            sv[u] = ld_col<MODE>(sqb + (uint64_t)p * L + l);
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t i = i0 + u * kSmallThreads;
          if (i < items) {
            const Acc acc = Dot<CB>::chunk(prow_s[kk[u]], ev[u], (Acc)0);
            r_s[i] = row_sim_exact((uint64_t)acc, sqa_s[kk[u]], sv[u]);
          }
        }
      }
    } else {
      for (uint32_t i = tid; i < items; i += kSmallThreads) {
        const uint32_t j = i / n_nz, k = i - j * n_nz, p = crank + csize * j, l = nz_s[k];
        const uint4* er = reinterpret_cast<const uint4*>(counts + (uint64_t)p * LR + (uint64_t)l * RB);
        const uint4* pr = prow_s + (size_t)k * C;
        Acc acc = 0;
        for (uint32_t c = 0; c < C; ++c) acc = Dot<CB>::chunk(pr[c], ld_col<MODE>(er + c), acc);
        r_s[i] = row_sim_exact((uint64_t)acc, sqa_s[k], ld_col<MODE>(sqb + (uint64_t)p * L + l));
      }
    }
    __syncthreads();
    double* dist0 = cl.map_shared_rank(dist_s, 0);
    for (uint32_t j = tid; j < nloc; j += kSmallThreads) {
      const uint32_t p = crank + csize * j;
      const uint64_t zv = zm ? ld_col<MODE>(zm + p) : 0ull;
      double sm = j0 ? pref[p] : 0.0;
      const double* rp = r_s + (size_t)j * n_nz;
      if (L <= 64) {  // explicit rows from the mask: the loads do not wait on a chain
        const uint64_t exm = exm_s;
        for (uint32_t l = j0; l <= hi && l < L; ++l) {
          const double r = (exm >> l) & 1ull ? rp[__popcll(exm & ((1ull << l) - 1ull))]
                           : row_zero(zv, p, l) ? 1.0 : 0.0;
          sm = __dadd_rn(sm, r);  // layer order (eam.cpp:95-98)
          if (l == keep) pref[p] = sm;
        }
      } else {
        uint32_t k = 0;
        for (uint32_t l = j0; l <= hi && l < L; ++l) {
          double r;
          if (k < n_nz && nz_s[k] == l) r = rp[k++];
          else r = row_zero(zv, p, l) ? 1.0 : 0.0;
          sm = __dadd_rn(sm, r);  // layer order (eam.cpp:95-98)
          if (l == keep) pref[p] = sm;
        }
      }
      if (zm) {
        uint64_t bits = hi + 1 < 64 ? zv & ~((2ull << hi) - 1ull) : 0ull;
        if (L < 64) bits &= (1ull << L) - 1ull;
        for (; bits; bits &= bits - 1) sm = __dadd_rn(sm, 1.0);
      } else {
        for (uint32_t l = hi + 1; l < L; ++l)
          if (ld_col<MODE>(sqb + (uint64_t)p * L + l) == 0.0) sm = __dadd_rn(sm, 1.0);
      }
      const double d = finish_distance(sm, L);
      dist0[p] = d;
      const unsigned long long db = (unsigned long long)__double_as_longlong(d);
      mloc = db < mloc ? db : mloc;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, mloc, o);
      mloc = x < mloc ? x : mloc;
    }
    if (lane == 0) red_s[wid] = mloc;
    __syncthreads();
    if (tid == 0) {
      unsigned long long m = ~0ull;
      for (uint32_t w = 0; w < kSmallWarps; ++w) m = red_s[w] < m ? red_s[w] : m;
      cl.map_shared_rank(cmin_s, 0)[crank] = m;
    }
    cl.sync();  // release/acquire: CTA 0 sees every distance and minimum
    if (crank != 0) return;
    if (tid == 0) {
      unsigned long long m = ~0ull;
      for (uint32_t c = 0; c < csize; ++c) m = cmin_s[c] < m ? cmin_s[c] : m;
      dmin_s = m;
    }
    __syncthreads();
  }
  for (uint32_t p = tid; p < size && csize == 1; p += kSmallThreads) {
    const uint64_t zv = zm ? ld_col<MODE>(zm + p) : 0ull;
    const double* sb = sqb + (uint64_t)p * L;
    const uint4* eb = reinterpret_cast<const uint4*>(counts + (uint64_t)p * LR);
    double sm = j0 ? (MODE == 1 ? __ldcg(pref + p) : pref[p]) : 0.0;
    uint32_t k = 0;
    uint32_t l = j0;
    if (C == 1 && L <= 64) {
      // one 16-byte chunk per row; the explicit rows and their probe-row index
      // come from the mask, so a round's loads issue without waiting on
      // shared memory
      constexpr int U = kSmallRowsU;
      const uint64_t exm = exm_s;
      const uint32_t lend = min(hi + 1, L);
      for (; l + U <= lend; l += U) {
        uint4 ev[U];
        double sv[U];
        bool ex[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          ex[u] = (exm >> (l + u)) & 1ull;
          if (ex[u]) {
            ev[u] = ld_col<MODE>(eb + l + u);
            sv[u] = ld_col<MODE>(sb + l + u);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          double r;
          if (ex[u]) {
            const uint32_t kq = __popcll(exm & ((1ull << (l + u)) - 1ull));
            const Acc acc = Dot<CB>::chunk(prow_s[kq], ev[u], (Acc)0);
            r = row_sim_exact((uint64_t)acc, sqa_s[kq], sv[u]);
          } else {
            r = row_zero(zv, p, l + u) ? 1.0 : 0.0;
          }
          sm = __dadd_rn(sm, r);  // layer order (eam.cpp:95-98)
          if (l + u == keep) pref[p] = sm;
        }
      }
      k = l >= 64 ? (uint32_t)__popcll(exm) : (uint32_t)__popcll(exm & ((1ull << l) - 1ull));
    } else if (C == 1) {  // one 16-byte chunk per row: kSmallRowsU rows' loads in flight per round
      constexpr int U = kSmallRowsU;
      const uint32_t lend = min(hi + 1, L);
      for (; l + U <= lend; l += U) {
        uint4 ev[U];
        double sv[U];
        uint32_t kk[U];
        bool ex[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          ex[u] = k < n_nz && nz_s[k] == l + u;
          kk[u] = k;
          if (ex[u]) {
            ev[u] = ld_col<MODE>(eb + l + u);
            sv[u] = ld_col<MODE>(sb + l + u);
            ++k;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          double r;
          if (ex[u]) {
            const Acc acc = Dot<CB>::chunk(prow_s[kk[u]], ev[u], (Acc)0);
            r = row_sim_exact((uint64_t)acc, sqa_s[kk[u]], sv[u]);
          } else {
            r = row_zero(zv, p, l + u) ? 1.0 : 0.0;
          }
          sm = __dadd_rn(sm, r);  // layer order (eam.cpp:95-98)
          if (l + u == keep) pref[p] = sm;
        }
      }
    }
    for (; l <= hi && l < L; ++l) {
      double r;
      if (k < n_nz && nz_s[k] == l) {
        Acc acc = 0;
        const uint4* pr = prow_s + (size_t)k * C;
        const uint4* er = eb + (size_t)l * C;
        for (uint32_t c = 0; c < C; ++c) acc = Dot<CB>::chunk(pr[c], ld_col<MODE>(er + c), acc);
        r = row_sim_exact((uint64_t)acc, sqa_s[k], ld_col<MODE>(sb + l));
        ++k;
      } else {
        r = row_zero(zv, p, l) ? 1.0 : 0.0;
      }
      sm = __dadd_rn(sm, r);  // layer order (eam.cpp:95-98)
      if (l == keep) pref[p] = sm;
    }
    if (zm) {
      uint64_t bits = hi + 1 < 64 ? zv & ~((2ull << hi) - 1ull) : 0ull;
      if (L < 64) bits &= (1ull << L) - 1ull;
      for (; bits; bits &= bits - 1) sm = __dadd_rn(sm, 1.0);
    } else {
      for (uint32_t l = hi + 1; l < L; ++l)
        if (ld_col<MODE>(sb + l) == 0.0) sm = __dadd_rn(sm, 1.0);
    }
    const double d = finish_distance(sm, L);
    dist_s[p] = d;
    const unsigned long long db = (unsigned long long)__double_as_longlong(d);
    mloc = db < mloc ? db : mloc;
  }
  stamp(a, 5);
  if (csize == 1) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, mloc, o);
      mloc = x < mloc ? x : mloc;
    }
    if (lane == 0) atomicMin(&dmin_s, mloc);
    __syncthreads();
  }
  stamp(a, 1);
  // ---- B: window members (eam.cpp:143) and their rows above cur
  const double thr = __dadd_rn(__longlong_as_double((long long)dmin_s), a.window);
  if (tid == 0) cnt_s[kSmallWarps] = 0;
  __syncthreads();
  for (uint32_t p = tid; p < a.size; p += kSmallThreads)
    if (dist_s[p] <= thr) mem_s[atomicAdd(&cnt_s[kSmallWarps], 1u)] = p;
  __syncthreads();
  const uint32_t nm = cnt_s[kSmallWarps];
  if (rows_above) {
    const uint32_t wpr = RB / 4, per = 4 / CB, per_mem = rows_above * wpr;
    for (uint32_t it = tid; it < nm * per_mem; it += kSmallThreads) {
      const uint32_t mi = it / per_mem, rem = it - mi * per_mem;
      const uint32_t r = rem / wpr, w = rem - r * wpr;
      const uint32_t l = a.cur + 1 + r;
      const uint32_t word = ld_col<MODE>(reinterpret_cast<const uint32_t*>(
          a.counts + (uint64_t)mem_s[mi] * LR + (uint64_t)l * RB + 4ull * w));
      if (!word) continue;
#pragma unroll
      for (uint32_t j = 0; j < per; ++j) {
        const uint32_t e = w * per + j;
        const uint32_t c = CB == 1 ? (word >> (8 * j)) & 0xffu
                           : CB == 2 ? (word >> (16 * j)) & 0xffffu
                                     : word;
        if (c && e < E) atomicAdd(&agg_s[r * E + e], (unsigned long long)c);
      }
    }
  }
  __syncthreads();
  stamp(a, 2);
  // ---- C: priorities (policy.cpp:106-120), floor filter (engine.cpp:663-668), order
  for (uint32_t r = wid; r < rows_above; r += kSmallWarps) {
    unsigned long long s = 0;
    for (uint32_t e = lane; e < E; e += 32) s += agg_s[r * E + e];
    s = warp_sum_u64(s);
    if (lane == 0) rsum_s[r] = s;
  }
  __syncthreads();
  stamp(a, 6);
  // survivors compacted in flat ExpertId order (ballot prefix), then each
  // survivor's output position = the number of survivor pairs below it
  const double kEps = 1e-4;
  uint32_t base = 0;
  for (uint32_t i0 = 0; i0 < N; i0 += kSmallThreads) {
    const uint32_t i = i0 + tid;
    unsigned long long key = ~0ull;
    uint32_t id = 0;
    if (i < N) {
      const uint32_t r = i / E, e = i - r * E, l = a.cur + 1 + r;
      const unsigned long long av = agg_s[i], rs = rsum_s[r];
      if (!(a.filter && av == 0)) {
        const double prox = __dsub_rn(1.0, __ddiv_rn((double)(l - a.cur), (double)L));
        const double ratio = rs == 0 ? 0.0 : __ddiv_rn(__ull2double_rn(av), __ull2double_rn(rs));
        const double pri = __dmul_rn(__dadd_rn(ratio, kEps), prox);
        const double floor_p = __dmul_rn(__dmul_rn(kEps, prox), __dadd_rn(1.0, 1e-9));
        if (!(a.filter && pri <= floor_p)) {
          key = ~(unsigned long long)__double_as_longlong(pri);
          id = l * E + e;
        }
      }
    }
    const bool sv = key != ~0ull;
    const uint32_t m = __ballot_sync(0xffffffffu, sv);
    if (lane == 0) cnt_s[wid] = __popc(m);
    __syncthreads();
    uint32_t off = base;
    for (uint32_t w = 0; w < wid; ++w) off += cnt_s[w];
    if (sv) {
      const uint32_t q = off + __popc(m & ((1u << lane) - 1u));
      key_s[q] = key;
      id_s[q] = id;
    }
    uint32_t tot = 0;
    for (uint32_t w = 0; w < kSmallWarps; ++w) tot += cnt_s[w];
    base += tot;
    __syncthreads();
  }
  const uint32_t S = base;
  stamp(a, 7);
  for (uint32_t i = tid; i < S; i += kSmallThreads) {
    const unsigned long long ki = key_s[i];
    const uint32_t ii = id_s[i];
    uint32_t pos = 0;
    for (uint32_t j = 0; j < S; ++j) pos += pair_lt(key_s[j], id_s[j], ki, ii);
    moe_candidate o;
    o.layer_idx = ii / E;
    o.expert_idx = ii - o.layer_idx * E;
    o.priority = __longlong_as_double((long long)~ki);
    a.out[pos] = o;
  }
  if (tid == 0) *a.n_out = S;
  stamp(a, 3);
}

template <int CB>
__global__ void __launch_bounds__(kSmallThreads, 1)
    k_decision_small(const __grid_constant__ DecisionArgs a) {
  small_body<CB, 0>(a);
}

// One-CTA persistent server for small collections (the k_decision_small
// phases; moe_eamc_set_decision_server): thread 0 polls the pinned mailbox,
// the CTA copies the arguments from host memory into shared memory, runs the
// decision (results straight into pinned host memory, as launched) and
// publishes seq_done.  Collection reads are L1-cached plain loads ordered by
// the request's acquire fence (ld_col).  Idle for idle_ns or asked to stop,
// it exits.
template <int CB>
__global__ void __launch_bounds__(kSmallThreads, 1)
    k_decision_small_server(DecServerCtl* ctl, uint64_t seq0, uint64_t idle_ns) {
  __shared__ DecisionArgs sa;
  __shared__ uint64_t sh_seq;
  const uint32_t tid = threadIdx.x;
  uint64_t last = seq0;
  for (;;) {
    if (tid == 0) {
      uint64_t t0, t, sq = 0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      for (;;) {
        asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(sq) : "l"(&ctl->seq_req));
        if (sq != last) break;
        int stop;
        asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(stop) : "l"(&ctl->stop));
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (stop || t - t0 > idle_ns) {
          sq = ~0ull;
          break;
        }
        __nanosleep(32);
      }
      sh_seq = sq;
      asm volatile("fence.acq_rel.sys;" ::: "memory");
    }
    __syncthreads();
    if (sh_seq == ~0ull) return;
    {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(&ctl->args);
      uint32_t* dst = reinterpret_cast<uint32_t*>(&sa);
      for (uint32_t i = tid; i < sizeof(DecisionArgs) / 4; i += kSmallThreads)
        dst[i] = *reinterpret_cast<const volatile uint32_t*>(src + i);
    }
    __syncthreads();
    small_body<CB, 2>(sa);
    __syncthreads();
    if (tid == 0) {
      __threadfence_system();
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&ctl->seq_done), "l"(sh_seq) : "memory");
    }
    last = sh_seq;
    __syncthreads();  // sh_seq is rewritten by the next poll
  }
}

template <int CB>
__global__ void __launch_bounds__(kDecThreads, 1) k_decision(const __grid_constant__ DecisionArgs a) {
  decision_body<CB, false>(a);
}

// Persistent decision server (moe_eamc_set_decision_server): the same phases,
// resident on `gridDim.x` SMs, fed through a pinned-memory mailbox instead of
// a launch per decision.  CTA 0's thread 0 polls the host mailbox; on a new
// request CTA 0 copies the arguments (and the probe's explicit rows, when they
// do not ride inline) from pinned host memory to the device, then releases the
// request to the other CTAs through a device word (every CTA follows CTA 0's
// decision, so all of them run a request or all exit).  After the phases each
// CTA makes its writes visible system-wide and counts itself done; the last one
// publishes seq_done to the host.  Idle for idle_ns (or asked to stop), the
// server exits; the host relaunches it on the next request.
template <int CB>
__global__ void __launch_bounds__(kDecThreads, 1)
    k_decision_server(DecServerCtl* ctl, DecisionArgs* dargs, uint8_t* drows, uint32_t* go,
                      uint32_t* done, uint32_t* bar, uint64_t seq0, uint32_t k0, uint64_t idle_ns,
                      uint32_t gen) {
  __shared__ DecisionArgs sa;
  __shared__ uint64_t sh_seq;
  const uint32_t tid = threadIdx.x, b = blockIdx.x, G = gridDim.x;
  // exit word of THIS launch (an earlier server's exit word carries its own
  // generation, so a relaunch does not see it as its own)
  const uint32_t kExit = 0x80000000u | (gen & 0x7fffffffu);
  uint64_t last = seq0;
  uint32_t k = k0;  // requests served by earlier servers on this state
  for (;;) {
    if (b == 0) {
      if (tid == 0) {
        uint64_t t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        uint64_t sq = 0;
        for (;;) {
          asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(sq) : "l"(&ctl->seq_req));
          if (sq != last) break;
          int stop;
          asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(stop) : "l"(&ctl->stop));
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          if (stop || t - t0 > idle_ns) {
            sq = ~0ull;
            break;
          }
          __nanosleep(100);
        }
        sh_seq = sq;
        asm volatile("fence.acq_rel.sys;" ::: "memory");
      }
      __syncthreads();
      if (sh_seq != ~0ull) {
        // arguments and explicit probe rows: pinned host memory -> device
        const uint32_t* src = reinterpret_cast<const uint32_t*>(&ctl->args);
        uint32_t* dst = reinterpret_cast<uint32_t*>(dargs);
        for (uint32_t i = tid; i < sizeof(DecisionArgs) / 4; i += kDecThreads)
          dst[i] = *reinterpret_cast<const volatile uint32_t*>(src + i);
        __syncthreads();
        if (!dargs->rows_inline && dargs->n_nz) {
          const uint32_t rows_b = dargs->n_nz * dargs->RB;
          const uint32_t nz_b = (dargs->n_nz * 2 + 15) & ~15u;
          const uint4* rs = reinterpret_cast<const uint4*>(dargs->rows);
          for (uint32_t i = tid; i < (rows_b + nz_b) / 16; i += kDecThreads)
            reinterpret_cast<uint4*>(drows)[i] = rs[i];  // rows then the row list (host layout)
          __syncthreads();
          if (tid == 0) {
            dargs->rows = drows;
            dargs->nz = reinterpret_cast<const uint16_t*>(drows + rows_b);
          }
        }
        if (tid == 0) {
          dargs->bar = bar;
          dargs->bar_base = k * kDecBarriers * G;
          dargs->out = ctl->args.out;
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(go), "r"(k + 1) : "memory");
      } else if (tid == 0) {
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(go), "r"(kExit) : "memory");
      }
    }
    // every CTA (CTA 0 included): wait for the release, acquire (fresh L1)
    __shared__ uint32_t sh_go;
    if (tid == 0) {
      uint32_t v;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(go) : "memory");
        if (v == k + 1 || v == kExit) break;
        __nanosleep(64);
      }
      sh_go = v;
    }
    __syncthreads();
    if (sh_go == kExit) return;
    {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(dargs);
      uint32_t* dst = reinterpret_cast<uint32_t*>(&sa);
      for (uint32_t i = tid; i < sizeof(DecisionArgs) / 4; i += kDecThreads) dst[i] = __ldcg(src + i);
    }
    __syncthreads();
    decision_body<CB, true>(sa);
    __syncthreads();
    if (tid == 0) {
      __threadfence_system();
      const uint32_t old = atomicAdd(done, 1u);
      if (old + 1 == (k + 1) * G) {  // the last CTA of this request
        __threadfence_system();
        uint64_t sq;
        asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(sq) : "l"(&ctl->seq_req));
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&ctl->seq_done), "l"(sq) : "memory");
      }
    }
    ++k;
    if (b == 0) last = sh_seq;
    __syncthreads();  // sh_seq is rewritten by the next poll
  }
}

}  // namespace

size_t decision_small_smem_max(uint32_t L, uint32_t RB) {
  return (((size_t)L * RB + 15) & ~(size_t)15) + (size_t)kSmallMaxP * 8 + (size_t)kSmallMaxCells * 8 +
         (size_t)L * 8 + (size_t)kSmallMaxCells * 12 + (size_t)kSmallMaxP * 4;
}

cudaError_t launch_decision_small_server(DecServerCtl* ctl, uint64_t seq0, uint64_t idle_ns, int cb,
                                        size_t smem, cudaStream_t st) {
  void (*kern)(DecServerCtl*, uint64_t, uint64_t) =
      cb == 1 ? k_decision_small_server<1> : cb == 2 ? k_decision_small_server<2> : k_decision_small_server<4>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<1, kSmallThreads, smem, st>>>(ctl, seq0, idle_ns);
  return cudaGetLastError();
}

size_t decision_small_smem(uint32_t size, uint32_t L, uint32_t E, uint32_t RB, uint32_t n_nz,
                           uint32_t cur) {
  const uint32_t rows = cur + 1 < L ? L - cur - 1 : 0, N = rows * E;
  uint32_t N2 = 1;
  while (N2 < N) N2 <<= 1;
  return (((size_t)n_nz * RB + 15) & ~(size_t)15) + (size_t)size * 8 + (size_t)N * 8 +
         (size_t)rows * 8 + (size_t)N2 * 12 + (size_t)size * 4;
}

// Cluster size of a small-path launch: the row similarities of enough
// (entry, explicit row) pairs are spread over a cluster (MOE_DEC_CLUSTER=<n>
// overrides, 1 = the one-CTA kernel; A/B runs).
static uint32_t small_cluster(uint32_t size, uint32_t n_nz) {
  static const int env = [] {
    const char* e = getenv("MOE_DEC_CLUSTER");
    return e ? atoi(e) : -1;
  }();
  uint32_t n = env >= 1 ? (uint32_t)std::min<int>(env, (int)kSmallMaxCluster) : 8u;
  if (env < 1 && (uint64_t)size * n_nz < 1024) n = 1;
  return n;
}

cudaError_t launch_decision_small(const DecisionArgs& a, int cb, size_t smem, cudaStream_t st) {
  void (*kern)(DecisionArgs) =
      cb == 1 ? k_decision_small<1> : cb == 2 ? k_decision_small<2> : k_decision_small<4>;
  static size_t set[3] = {0, 0, 0};
  const int slot = cb == 1 ? 0 : cb == 2 ? 1 : 2;
  if (smem > set[slot]) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set[slot] = smem;
  }
  static const bool prof = getenv("MOE_LAUNCH_PROF") != nullptr;
  const uint32_t ncl = small_cluster(a.size, a.n_nz);
  if (ncl > 1) {
    // the cluster's CTAs also stage their entries' row similarities
    const uint32_t rows = a.cur + 1 < a.L ? a.L - a.cur - 1 : 0, N = rows * a.E;
    uint32_t N2 = 1;
    while (N2 < N) N2 <<= 1;
    const size_t need = small_rsim_offset(a.n_nz, a.RB, a.size, N, rows, N2) +
                        (size_t)((a.size + ncl - 1) / ncl) * a.n_nz * 8;
    smem = std::max(smem, need);
    if (smem > set[slot]) {
      cudaError_t e =
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      set[slot] = smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncl);
    cfg.blockDim = dim3(kSmallThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ncl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    static bool nonportable[3] = {false, false, false};
    if (ncl > 8 && !nonportable[slot]) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
      nonportable[slot] = true;
    }
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
    if (e == cudaSuccess) return cudaGetLastError();
    // a cluster the device cannot place (shared memory, partitioned GPU):
    // the one-CTA launch computes the same result
    (void)cudaGetLastError();
  }
  if (!prof) {
    kern<<<1, kSmallThreads, smem, st>>>(a);
    return cudaGetLastError();
  }
  // launch-path instrumentation (MOE_LAUNCH_PROF=1)
  static double acc[4] = {0, 0, 0, 0};
  static uint64_t cnt = 0;
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t q = cudaStreamQuery(st);
  const auto t1 = std::chrono::steady_clock::now();
  void* args[] = {const_cast<DecisionArgs*>(&a)};
  cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void*>(kern), dim3(1), dim3(kSmallThreads),
                                   args, smem, st);
  const auto t2 = std::chrono::steady_clock::now();
  cudaError_t g = cudaGetLastError();
  const auto t3 = std::chrono::steady_clock::now();
  acc[0] += std::chrono::duration<double, std::micro>(t1 - t0).count();
  acc[1] += std::chrono::duration<double, std::micro>(t2 - t1).count();
  acc[2] += std::chrono::duration<double, std::micro>(t3 - t2).count();
  if (++cnt % 100 == 0)
    fprintf(stderr, "launch path (avg of %llu): streamQuery %.2f us, cudaLaunchKernel %.2f us, getLastError %.2f us (q=%d)\n",
            (unsigned long long)cnt, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, (int)q);
  return e != cudaSuccess ? e : g;
}

size_t decision_smem(uint32_t L, uint32_t E, uint32_t RB, uint32_t n_nz, uint32_t cur,
                     uint32_t grid) {
  (void)grid;
  uint32_t np = 1;
  while (np < E) np <<= 1;
  // staged probe rows | a layer's slots + its compacted survivors | the listed
  // members' group reduction (one u64 per count of a 16-byte chunk per thread)
  // | the staged survivor list (12 bytes per candidate, C2 with many survivors),
  // capped so that two decision CTAs still fit one SM: two launches in flight
  // on different streams (two handles, two host threads) must stay co-resident
  // for their software grid barriers
  const size_t rows = cur + 1 < L ? L - cur - 1 : 0;
  return std::max({(size_t)n_nz * RB, (size_t)np * 28, (size_t)kDecThreads * 16 * 8,
                   std::min<size_t>(rows * E * ((uint64_t)L * E <= 65536u ? 10 : 12), kDecStageCap)});
}

int decision_grid(int n_sm, uint32_t size, uint32_t L, uint32_t cur) {
  const uint32_t rows = cur + 1 < L ? L - cur - 1 : 0;
  uint32_t g = std::max<uint32_t>({(size + 63) / 64, rows, 8u});
  return (int)std::min<uint32_t>(g, (uint32_t)n_sm);
}

cudaError_t launch_decision_server(DecServerCtl* ctl, DecisionArgs* dargs, uint8_t* drows,
                                   uint32_t* go, uint32_t* done, uint32_t* bar, uint64_t seq0,
                                   uint32_t k0, uint64_t idle_ns, uint32_t gen, int cb, int grid,
                                   size_t smem, cudaStream_t st) {
  void (*kern)(DecServerCtl*, DecisionArgs*, uint8_t*, uint32_t*, uint32_t*, uint32_t*, uint64_t,
               uint32_t, uint64_t, uint32_t) =
      cb == 1 ? k_decision_server<1> : cb == 2 ? k_decision_server<2> : k_decision_server<4>;
  static size_t set[3] = {0, 0, 0};
  const int slot = cb == 1 ? 0 : cb == 2 ? 1 : 2;
  if (smem > set[slot]) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set[slot] = smem;
  }
  kern<<<(unsigned)grid, kDecThreads, smem, st>>>(ctl, dargs, drows, go, done, bar, seq0, k0,
                                                  idle_ns, gen);
  return cudaGetLastError();
}

cudaError_t launch_decision(const DecisionArgs& a, int cb, int grid, size_t smem,
                            cudaStream_t st) {
  void (*kern)(DecisionArgs) = cb == 1 ? k_decision<1> : cb == 2 ? k_decision<2> : k_decision<4>;
  // opt in once to the largest dynamic size the callers use (static + dynamic
  // shared memory above 48 KB needs it, and the co-residency check of a
  // cooperative launch counts both)
  static size_t max_dyn[3] = {0, 0, 0};
  const int slot = cb == 1 ? 0 : cb == 2 ? 1 : 2;
  if (!max_dyn[slot]) {
    int dev = 0, optin = 0;
    cudaFuncAttributes fa;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess)
      e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, kern);
    const size_t lim = (size_t)optin - fa.sharedSizeBytes;
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim);
    if (e != cudaSuccess) return e;
    max_dyn[slot] = lim;
  }
  if (smem > max_dyn[slot]) return cudaErrorInvalidValue;
  // grid <= SMs and one CTA per SM (launch bounds, shared memory): all CTAs
  // are co-resident once scheduled, which the software barrier relies on
  static const bool prof = getenv("MOE_LAUNCH_PROF") != nullptr;
  if (!prof) {
    kern<<<(unsigned)grid, kDecThreads, smem, st>>>(a);
    return cudaGetLastError();
  }
  // launch-path instrumentation (MOE_LAUNCH_PROF=1)
  static double acc[3] = {0, 0, 0};
  static uint64_t cnt = 0;
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t q = cudaStreamQuery(st);
  const auto t1 = std::chrono::steady_clock::now();
  kern<<<(unsigned)grid, kDecThreads, smem, st>>>(a);
  const auto t2 = std::chrono::steady_clock::now();
  cudaError_t e = cudaGetLastError();
  const auto t3 = std::chrono::steady_clock::now();
  acc[0] += std::chrono::duration<double, std::micro>(t1 - t0).count();
  acc[1] += std::chrono::duration<double, std::micro>(t2 - t1).count();
  acc[2] += std::chrono::duration<double, std::micro>(t3 - t2).count();
  if (++cnt % 58 == 0)
    fprintf(stderr, "k_decision launch (avg of %llu, grid %d, smem %zu, params %zu B): query %.1f us "
                    "(%d), <<<>>> %.1f us, getlasterror %.1f us\n",
            (unsigned long long)cnt, grid, smem, sizeof(DecisionArgs), acc[0] / cnt, (int)q,
            acc[1] / cnt, acc[2] / cnt);
  return e;
}

}  // namespace moe
