// kernels.cu -- hand-written sm_100a kernels of the EAM/EAMC decision path.
//
//  K3  k_match<CB,QT,0>   EAMC matcher, screen pass.  Collection tiles of
//                         128 entries x G layers stream HBM->SMEM through TMA
//                         (cp.async.bulk.tensor.4d, mbarrier ring of S stages);
//                         one thread per entry computes exact integer dots
//                         (IDP4A for u8 counts) against QT probes held in
//                         SMEM, an fp32 cosine screen with a proven error
//                         bound, and the argmin threshold / candidate
//                         buckets (warp REDUX min -> block -> global atomics).
//      k_refine           one warp per probe: exact fp64 re-evaluation, in the
//                         reference operation order, of the few candidates
//                         whose screened distance is within 2*eps of the min;
//                         lexicographic (distance, seq) argmin (eam.cpp:118-129).
//      k_match<CB,1,1>    exact argmin for probes whose bucket overflowed
//                         (mass near-ties), same TMA pipeline.
//  K4  k_match<CB,1,2>    window membership d <= d_min + window (eam.cpp:131-150)
//      k_aggregate        u64 aggregation of the matched rows (policy.cpp:97-104)
//  K5+K6 k_decide         prefetch priorities + floor filter + order
//                         (policy.cpp:106-125, engine.cpp:663-668) and the
//                         eviction victim (policy.cpp:128-159), one block.
//  (K1 tracing lives in trace.cu.)
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <tuple>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace moe {

namespace {

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

struct SmemLayout {
  uint32_t stage_bytes, off_probe, off_ia, off_sqa, off_dots, off_red, off_tnow, off_wbest,
      off_bars, total;
};

__host__ __device__ inline SmemLayout smem_layout(uint32_t L, uint32_t RB, uint32_t G, uint32_t S,
                                                  uint32_t QT, int mode, uint32_t acc_bytes) {
  SmemLayout s;
  uint32_t o = 0;
  s.stage_bytes = kNT * G * RB;
  o = S * s.stage_bytes;
  s.off_probe = o;
  o = align_up(o + QT * L * RB, 16);
  s.off_ia = o;
  o = align_up(o + QT * L * 4, 16);
  s.off_sqa = o;
  o = align_up(o + (mode ? L * 8 : 0), 16);
  s.off_dots = o;
  o = align_up(o + (mode ? L * kNT * acc_bytes : 0), 16);
  s.off_red = o;
  o = align_up(o + 4 * QT * 4, 16);
  s.off_tnow = o;
  o = align_up(o + QT * 4, 16);
  s.off_wbest = o;
  o = align_up(o + 4 * (uint32_t)sizeof(Best), 16);
  s.off_bars = o;
  o += S * 8;
  s.total = align_up(o, 128);
  return s;
}

struct MatchArgs {
  // collection
  const float* ibT;
  const double* sqb;
  const uint64_t* seq;
  uint64_t cap;
  uint32_t size;
  // probes
  const uint8_t* probes;
  const float* ia;
  const double* sqa;
  uint32_t Q;
  // geometry
  uint32_t L, RB, C, G, S, n_groups, n_pt;
  float eps2;
  // mode 0
  uint32_t* T;
  uint32_t* bcnt;
  uint2* bucket;
  uint32_t bcap;
  // mode 1 / 2
  const uint32_t* qlist;   // null: the single probe q_single
  uint32_t q_single;
  uint32_t nq_list;
  const uint32_t* nq_dev;  // mode 1: list length read on the device (minus q_off, capped)
  uint32_t q_off;
  const uint32_t* Tfinal;  // mode 1 candidate threshold (null: all)
  moe_match* partials;     // mode 1 [nq_list][grid]
};

template <typename Acc>
__device__ __forceinline__ float acc_to_float(Acc a);
template <>
__device__ __forceinline__ float acc_to_float<uint32_t>(uint32_t a) {
  return __uint2float_rn(a);
}
template <>
__device__ __forceinline__ float acc_to_float<uint64_t>(uint64_t a) {
  return __ull2float_rn(a);
}

template <int CB, int QT, int MODE>
__global__ void __launch_bounds__(kNT, 1)
    k_match(const __grid_constant__ CUtensorMap tmap, const MatchArgs a) {
  using D = Dot<CB>;
  using Acc = typename D::Acc;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const SmemLayout lay = smem_layout(a.L, a.RB, a.G, a.S, QT, MODE, sizeof(Acc));
  uint8_t* stages = smem;
  uint8_t* probe_s = smem + lay.off_probe;
  float* ia_s = reinterpret_cast<float*>(smem + lay.off_ia);
  double* sqa_s = reinterpret_cast<double*>(smem + lay.off_sqa);
  Acc* dots_s = reinterpret_cast<Acc*>(smem + lay.off_dots);
  uint32_t* red = reinterpret_cast<uint32_t*>(smem + lay.off_red);
  float* tnow = reinterpret_cast<float*>(smem + lay.off_tnow);
  Best* wbest = reinterpret_cast<Best*>(smem + lay.off_wbest);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lay.off_bars);

  pdl_wait();
  pdl_trigger();
  uint32_t nq = MODE == 0 ? (a.Q + QT - 1) / QT : a.nq_list;
  if (MODE == 1 && a.nq_dev) {  // device-gated exact pass: no work unless buckets overflowed
    const uint32_t tot = *a.nq_dev;
    nq = tot > a.q_off ? min(tot - a.q_off, a.nq_list) : 0u;
  }
  const uint64_t n_items = (uint64_t)nq * a.n_pt;
  const uint64_t it0 = n_items * blockIdx.x / gridDim.x;
  const uint64_t it1 = n_items * (blockIdx.x + 1) / gridDim.x;
  if (it0 >= it1) return;
  const uint64_t total = (it1 - it0) * a.n_groups;

  if (tid == 0) {
    prefetch_tmap(&tmap);
    for (uint32_t s = 0; s < a.S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](uint64_t j) {
    const uint64_t item = it0 + j / a.n_groups;
    const uint32_t g = (uint32_t)(j % a.n_groups);
    const uint32_t pt = (uint32_t)(item % a.n_pt);
    const uint32_t s = (uint32_t)(j % a.S);
    mbar_arrive_expect_tx(&bars[s], lay.stage_bytes);
    tma_load_4d(stages + (size_t)s * lay.stage_bytes, &tmap, &bars[s], 0, 0, (int)(g * a.G),
                (int)(pt * kNT));
  };
  if (tid == 0) {
    const uint64_t pre = total < a.S ? total : a.S;
    for (uint64_t j = 0; j < pre; ++j) issue(j);
  }

  float sim[QT];
#pragma unroll
  for (int q = 0; q < QT; ++q) sim[q] = 0.f;
  int64_t cur_qi = -1;
  Best tb{__longlong_as_double(0x7ff0000000000000ll), kNone, kNone};
  const uint32_t LR = a.L * a.RB;

  auto flush_best = [&](uint32_t qi) {  // MODE 1: block argmin -> partial
    Best b = warp_best(tb);
    if (lane == 0) wbest[warp] = b;
    __syncthreads();
    if (tid == 0) {
      Best x = wbest[0];
      for (int w = 1; w < kNT / 32; ++w)
        if (better(wbest[w].d, wbest[w].seq, x.d, x.seq)) x = wbest[w];
      moe_match m;
      m.index = x.idx;
      m.seq = x.seq;
      m.distance = x.d;
      a.partials[(uint64_t)qi * gridDim.x + blockIdx.x] = m;
    }
    __syncthreads();
    tb = Best{__longlong_as_double(0x7ff0000000000000ll), kNone, kNone};
  };

  for (uint64_t j = 0; j < total; ++j) {
    const uint64_t item = it0 + j / a.n_groups;
    const uint32_t g = (uint32_t)(j % a.n_groups);
    const uint32_t qi = (uint32_t)(item / a.n_pt);
    const uint32_t pt = (uint32_t)(item % a.n_pt);
    if (g == 0 && (int64_t)qi != cur_qi) {
      if (MODE == 1 && cur_qi >= 0) flush_best((uint32_t)cur_qi);
      __syncthreads();
      // Stage the probe tile: QT probes starting at q0 (mode 0) or qlist[qi].
      const uint32_t q0 = MODE == 0 ? qi * QT : (a.qlist ? a.qlist[qi] : a.q_single);
      const uint32_t nbytes = QT * LR;
      for (uint32_t o = tid * 16; o < nbytes; o += kNT * 16) {
        const uint32_t q = q0 + o / LR;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (q < a.Q) v = *reinterpret_cast<const uint4*>(a.probes + (uint64_t)q0 * LR + o);
        *reinterpret_cast<uint4*>(probe_s + o) = v;
      }
      for (uint32_t o = tid; o < QT * a.L; o += kNT) {
        const uint32_t q = q0 + o / a.L;
        ia_s[o] = q < a.Q ? a.ia[(uint64_t)q0 * a.L + o] : 0.f;
      }
      if (MODE != 0)
        for (uint32_t o = tid; o < a.L; o += kNT) sqa_s[o] = a.sqa[(uint64_t)q0 * a.L + o];
      __syncthreads();
      cur_qi = qi;
    }

    const uint32_t s = (uint32_t)(j % a.S);
    mbar_wait(&bars[s], (uint32_t)((j / a.S) & 1));

    const uint32_t p = pt * kNT + tid;
    const bool valid = p < a.size;
    const uint8_t* ebase = stages + (size_t)s * lay.stage_bytes + (size_t)tid * a.G * a.RB;
    for (uint32_t gg = 0; gg < a.G; ++gg) {
      const uint32_t l = g * a.G + gg;
      if (l >= a.L) break;
      Acc acc[QT];
#pragma unroll
      for (int q = 0; q < QT; ++q) acc[q] = 0;
      const uint8_t* erow = ebase + gg * a.RB;
      const uint8_t* prow = probe_s + l * a.RB;
      // Per-lane chunk rotation keeps the 32 entry-row reads of a warp on
      // distinct shared-memory bank groups (rows are RB-strided).
      uint32_t k = lane % a.C;
      for (uint32_t c = 0; c < a.C; ++c) {
        const uint4 ev = *reinterpret_cast<const uint4*>(erow + 16 * k);
#pragma unroll
        for (int q = 0; q < QT; ++q) {
          const uint4 pv = *reinterpret_cast<const uint4*>(prow + q * LR + 16 * k);
          acc[q] = D::chunk(ev, pv, acc[q]);
        }
        if (++k == a.C) k = 0;
      }
      const float ib = valid ? __ldg(&a.ibT[(uint64_t)l * a.cap + p]) : 0.f;
#pragma unroll
      for (int q = 0; q < QT; ++q) {
        const float ia = ia_s[q * a.L + l];
        if (ia == 0.f && ib == 0.f)
          sim[q] += 1.f;
        else
          sim[q] = fmaf(acc_to_float<Acc>(acc[q]) * ia, ib, sim[q]);
      }
      if (MODE != 0) dots_s[l * kNT + tid] = acc[0];
    }

    if (g == a.n_groups - 1) {
      if (MODE == 0) {
        float dq[QT];
#pragma unroll
        for (int q = 0; q < QT; ++q) {
          float d = 1.f - sim[q] / (float)a.L;
          d = fmaxf(d, 0.f);
          if (!valid || qi * QT + q >= a.Q) d = __uint_as_float(kFInf);
          dq[q] = d;
          const uint32_t m = __reduce_min_sync(0xffffffffu, __float_as_uint(d));
          if (lane == 0) red[warp * QT + q] = m;
        }
        __syncthreads();
        if (tid < QT) {
          const uint32_t qg = qi * QT + tid;
          float tv = __uint_as_float(kFInf);
          if (qg < a.Q) {
            uint32_t m = red[tid];
            for (int w = 1; w < kNT / 32; ++w) m = min(m, red[w * QT + tid]);
            uint32_t t = *reinterpret_cast<volatile uint32_t*>(&a.T[qg]);
            if (m < t) t = min(atomicMin(&a.T[qg], m), m);
            tv = __uint_as_float(t);
          }
          tnow[tid] = tv;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < QT; ++q) {
          const uint32_t qg = qi * QT + q;
          if (valid && qg < a.Q && dq[q] <= tnow[q] + a.eps2) {
            const uint32_t pos = atomicAdd(&a.bcnt[qg], 1u);
            if (pos < a.bcap)
              a.bucket[(uint64_t)qg * a.bcap + pos] = make_uint2(p, __float_as_uint(dq[q]));
          }
        }
      } else {
        // MODE 1: exact evaluation of the candidates below the final threshold
        const uint32_t q = a.qlist ? a.qlist[qi] : a.q_single;
        const float d32 = fmaxf(1.f - sim[0] / (float)a.L, 0.f);
        bool cand = valid;
        if (a.Tfinal) cand = cand && d32 <= __uint_as_float(a.Tfinal[q]) + a.eps2;
        if (cand) {
          double sm = 0.0;
          const double* sb = a.sqb + (uint64_t)p * a.L;
          for (uint32_t l = 0; l < a.L; ++l)
            sm = __dadd_rn(sm, row_sim_exact((uint64_t)dots_s[l * kNT + tid], sqa_s[l], sb[l]));
          const double d = finish_distance(sm, a.L);
          const uint64_t sq = a.seq[p];
          if (better(d, sq, tb.d, tb.seq)) tb = Best{d, sq, p};
        }
      }
#pragma unroll
      for (int q = 0; q < QT; ++q) sim[q] = 0.f;
    }
    __syncthreads();
    if (tid == 0 && j + a.S < total) issue(j + a.S);
  }
  if (MODE == 1 && cur_qi >= 0) flush_best((uint32_t)cur_qi);
}


struct RefineArgs {
  const uint8_t* counts;
  const double* sqb;
  const uint64_t* seq;
  uint32_t size;
  const uint8_t* probes;
  const double* sqa;
  uint32_t Q, L, C, RB;
  float eps2;
  const uint32_t* T;
  const uint32_t* bcnt;
  const uint2* bucket;
  uint32_t bcap;
  uint32_t* over_list;
  uint32_t* over_n;
  const uint8_t* wide;  // probes whose counts exceed the storage width
  moe_match* out;
  const int* halt;
  int* halt_set;
  uint32_t halt_value;
  uint64_t index_base;
};

// One warp per probe.  The bucket's candidates that survive the final
// threshold are evaluated exactly: (candidate, layer) pairs are spread over
// the 32 lanes (integer row dots + the fp64 row similarity), the per-layer
// values land in shared memory, and one lane per candidate then sums them in
// layer order (eam.cpp:95-98) -- so the critical path grows with
// candidates*L/32 instead of with the candidate count.
constexpr int kRefineWarps = 4;
constexpr int kRefineBuf = 256;  // doubles of per-warp scratch
constexpr int kRefinePartBytes = 4096;  // per-warp scratch of per-chunk partial dots

// Lane-per-row exact evaluation (the general path of k_refine for EAMs too
// long for the chunk-parallel scratch): (candidate, layer) pairs over the
// lanes, each lane walking its row's 16-byte chunks.
template <int CB>
__device__ __forceinline__ void refine_rows_per_lane(const RefineArgs& r, const uint8_t* pa,
                                                     const double* sqa, const uint32_t* cand,
                                                     uint32_t nc, double* rbuf, uint32_t lane,
                                                     Best& b) {
  const uint64_t LR = (uint64_t)r.L * r.RB;
  const uint32_t G = max(1u, min(32u, (uint32_t)kRefineBuf / r.L));
  for (uint32_t g0 = 0; g0 < nc; g0 += G) {
    const uint32_t gn = min(G, nc - g0);
    const uint32_t pairs = gn * r.L;
    const uint64_t my_seq = lane < gn ? r.seq[cand[g0 + lane]] : 0;
    for (uint32_t id = lane; id < pairs; id += 32) {
      const uint32_t ci = id / r.L, l = id - ci * r.L;
      const uint32_t p = cand[g0 + ci];
      typename Dot<CB>::Acc acc = 0;
      const uint4* ra = reinterpret_cast<const uint4*>(pa + (uint64_t)l * r.RB);
      const uint4* rb = reinterpret_cast<const uint4*>(r.counts + p * LR + (uint64_t)l * r.RB);
      for (uint32_t c = 0; c < r.C; ++c) acc = Dot<CB>::chunk(__ldg(ra + c), __ldg(rb + c), acc);
      rbuf[ci * r.L + l] = row_sim_exact((uint64_t)acc, sqa[l], r.sqb[(uint64_t)p * r.L + l]);
    }
    __syncwarp();
    if (lane < gn) {
      const uint32_t p = cand[g0 + lane];
      double sm = 0.0;
      for (uint32_t l = 0; l < r.L; ++l) sm = __dadd_rn(sm, rbuf[lane * r.L + l]);
      const double d = finish_distance(sm, r.L);
      if (better(d, my_seq, b.d, b.seq)) b = Best{d, my_seq, p};
    }
    __syncwarp();
  }
}

template <int CB>
__global__ void __launch_bounds__(kRefineWarps * 32, 7) k_refine(const RefineArgs r) {
  __shared__ double rbuf[kRefineWarps][kRefineBuf];
  __shared__ uint32_t cand[kRefineWarps][256];
  __shared__ uint64_t parts[kRefineWarps][kRefinePartBytes / 8];
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t q = blockIdx.x * kRefineWarps + wib;
  const uint32_t lane = threadIdx.x & 31;
  pdl_wait();
  pdl_trigger();
  if (q >= r.Q) return;
  // Every load that does not depend on another is issued up front (one
  // memory round trip instead of a chain): flags, bucket count, threshold,
  // the first 32 bucket slots (the bucket always spans bcap slots per probe)
  // and an L1 prefetch of the probe's packed rows.
  const uint64_t LR = (uint64_t)r.L * r.RB;
  const uint8_t* pa = r.probes + q * LR;
  const int halted = r.halt ? *r.halt : 0;
  const uint8_t is_wide = r.wide ? r.wide[q] : (uint8_t)0;
  const uint32_t n = r.bcnt[q];
  const float thr = __uint_as_float(r.T[q]) + r.eps2;
  uint2 e0 = make_uint2(0u, 0x7f800000u);
  if (lane < r.bcap) e0 = r.bucket[(uint64_t)q * r.bcap + lane];
  for (uint64_t o = (uint64_t)lane * 128; o < LR; o += 32 * 128)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(pa + o));
  if (halted) return;
  const moe_match none{kNone, kNone, __longlong_as_double(0x7ff0000000000000ll)};
  if (r.size == 0) {
    if (lane == 0) r.out[q] = none;
    return;
  }
  if (is_wide) {  // cannot be matched at this width: explicit sentinel
    if (lane == 0) r.out[q] = moe_match{kNone - 1, kNone, __longlong_as_double(0x7ff8000000000000ll)};
    return;
  }
  if (n > r.bcap) {
    if (lane == 0) {
      if (r.over_list) r.over_list[atomicAdd(r.over_n, 1u)] = q;
      if (r.halt_set) *r.halt_set = (int)r.halt_value;
    }
    return;
  }
  // compact the candidates that pass the final threshold
  uint32_t nc = 0;
  for (uint32_t base = 0; base < n; base += 32) {
    const uint32_t i = base + lane;
    bool pass = false;
    uint32_t p = 0;
    if (i < n) {
      const uint2 e = base == 0 ? e0 : r.bucket[(uint64_t)q * r.bcap + i];
      p = e.x;
      pass = __uint_as_float(e.y) <= thr;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, pass);
    if (pass) cand[wib][nc + __popc(m & ((1u << lane) - 1))] = p;
    nc += __popc(m);
  }
  __syncwarp();
  const double* sqa = r.sqa + (uint64_t)q * r.L;
  Best b{__longlong_as_double(0x7ff0000000000000ll), kNone, kNone};
  // Candidates are taken in groups; a group's (candidate, layer, 16-byte
  // chunk) items are spread over the lanes so that consecutive lanes read
  // consecutive chunks of the same row (coalesced 128-bit loads), the
  // per-chunk partial dots go to shared memory, one lane per (candidate,
  // layer) sums its row's chunks and applies the fp64 row similarity, and one
  // lane per candidate sums the layers in order (eam.cpp:95-98).
  using Acc = typename Dot<CB>::Acc;
  constexpr uint32_t kParts = kRefinePartBytes / sizeof(Acc);
  const uint32_t C = r.C;
  if ((uint64_t)r.L * C > kParts) {  // very long EAMs: one lane per (candidate, layer) row
    refine_rows_per_lane<CB>(r, pa, sqa, cand[wib], nc, rbuf[wib], lane, b);
    b = warp_best(b);
    if (lane == 0)
      r.out[q] = moe_match{b.idx == kNone ? kNone : b.idx + r.index_base, b.seq, b.d};
    return;
  }
  const uint32_t G = max(1u, min(min(32u, (uint32_t)kRefineBuf / r.L), kParts / (r.L * C)));
  const uint4* pa4 = reinterpret_cast<const uint4*>(pa);
  const uint4* cb4 = reinterpret_cast<const uint4*>(r.counts);
  const uint64_t LC = (uint64_t)r.L * C;
  Acc* part = reinterpret_cast<Acc*>(parts[wib]);
  const uint32_t L = r.L;
  for (uint32_t g0 = 0; g0 < nc; g0 += G) {
    const uint32_t gn = min(G, nc - g0);
    const uint32_t pairs = gn * L;
    const uint32_t items = pairs * C;
    const uint32_t* cg = cand[wib] + g0;
    // Everything the later phases load is issued together with the row loads
    // (one memory round trip): the summing lane's seq, and the norms of this
    // lane's first (candidate, layer) pair.
    const uint64_t my_seq = lane < gn ? r.seq[cg[lane]] : 0;
    const uint32_t pci0 = lane / L, pl0 = lane - pci0 * L;
    double sqa0 = 0.0, sqb0 = 0.0;
    if (lane < pairs) {
      sqa0 = sqa[pl0];
      sqb0 = r.sqb[(uint64_t)cg[pci0] * L + pl0];
    }
    // Items in batches of 2 per lane: the (candidate, chunk) coordinates are
    // computed first and the 4 loads of a batch are in flight together.
    for (uint32_t it0 = lane; it0 < items; it0 += 2 * 32) {
      uint4 va[2], vb[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t it = it0 + 32u * u;
        if (it < items) {
          const uint32_t ci = it / (uint32_t)LC, lc = it - ci * (uint32_t)LC;
          va[u] = __ldg(pa4 + lc);
          vb[u] = __ldg(cb4 + (uint64_t)cg[ci] * LC + lc);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t it = it0 + 32u * u;
        if (it < items) part[it] = Dot<CB>::chunk(va[u], vb[u], (Acc)0);
      }
    }
    __syncwarp();
    uint32_t pci = pci0, pl = pl0;
    for (uint32_t pr = lane; pr < pairs; pr += 32) {
      uint64_t dot = 0;
      for (uint32_t c = 0; c < C; ++c) dot += (uint64_t)part[pr * C + c];
      const bool first = pr == lane;
      const double sa = first ? sqa0 : sqa[pl];
      const double sb = first ? sqb0 : r.sqb[(uint64_t)cg[pci] * L + pl];
      rbuf[wib][pr] = row_sim_exact(dot, sa, sb);
      pl += 32;
      while (pl >= L) {
        pl -= L;
        ++pci;
      }
    }
    __syncwarp();
    if (lane < gn) {
      // in-order layer sum (eam.cpp:95-98); shared-memory reads batched ahead
      const double* rs = rbuf[wib] + lane * L;
      double sm = 0.0;
      uint32_t l = 0;
      for (; l + 4 <= L; l += 4) {
        const double x0 = rs[l], x1 = rs[l + 1], x2 = rs[l + 2], x3 = rs[l + 3];
        sm = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(sm, x0), x1), x2), x3);
      }
      for (; l < L; ++l) sm = __dadd_rn(sm, rs[l]);
      const double d = finish_distance(sm, L);
      if (better(d, my_seq, b.d, b.seq)) b = Best{d, my_seq, cg[lane]};
    }
    __syncwarp();
  }
  if (nc <= 1) {  // a single candidate sits on lane 0: no warp reduction
    if (lane == 0)
      r.out[q] = moe_match{b.idx == kNone ? kNone : b.idx + r.index_base, b.seq, b.d};
    return;
  }
  b = warp_best(b);
  if (lane == 0)
    r.out[q] = moe_match{b.idx == kNone ? kNone : b.idx + r.index_base, b.seq, b.d};
}

// Partial merge for mode 1: for list position qi, the blocks whose item
// range intersects [qi*n_pt, (qi+1)*n_pt).
__global__ void k_merge_partials(const moe_match* parts, uint32_t grid, uint32_t nq,
                                 uint32_t n_pt, const uint32_t* qlist, moe_match* out,
                                 uint64_t index_base, const uint32_t* nq_dev, uint32_t q_off) {
  pdl_wait();
  pdl_trigger();
  if (nq_dev) {
    const uint32_t tot = *nq_dev;
    nq = tot > q_off ? min(tot - q_off, nq) : 0u;
  }
  const uint32_t qi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (qi >= nq) return;
  const uint64_t n_items = (uint64_t)nq * n_pt;
  Best b{__longlong_as_double(0x7ff0000000000000ll), kNone, kNone};
  for (uint32_t blk = lane; blk < grid; blk += 32) {
    const uint64_t i0 = n_items * blk / grid, i1 = n_items * (blk + 1) / grid;
    const uint64_t q0 = (uint64_t)qi * n_pt, q1 = q0 + n_pt;
    if (i0 < i1 && i0 < q1 && i1 > q0) {
      const moe_match m = parts[(uint64_t)qi * grid + blk];
      if (better(m.distance, m.seq, b.d, b.seq)) b = Best{m.distance, m.seq, m.index};
    }
  }
  b = warp_best(b);
  if (lane == 0)
    out[qlist[qi]] = moe_match{b.idx == kNone ? kNone : b.idx + index_base, b.seq, b.d};
}

// Exact argmin without the TMA pipeline (shapes whose rows do not fit the
// matcher's shared-memory tiles, e.g. wide u32 rows): warp per (listed probe,
// entry), warp_exact_distance in the reference operation order, block argmin
// -> parts[qi][blockIdx.x]; k_merge_blocks folds the blocks.
template <int CB>
__global__ void __launch_bounds__(256)
    k_exact_warp(const uint8_t* counts, const double* sqb, const uint64_t* seq, uint32_t size,
                 uint32_t L, uint32_t C, uint32_t RB, const uint8_t* probes, const double* sqa,
                 const uint32_t* qlist, uint32_t nq_list, const uint32_t* nq_dev, uint32_t q_off,
                 moe_match* parts) {
  pdl_wait();
  pdl_trigger();
  uint32_t nq = nq_list;
  if (nq_dev) {
    const uint32_t tot = *nq_dev;
    nq = tot > q_off ? min(tot - q_off, nq_list) : 0u;
  }
  const uint32_t qi = blockIdx.y;
  if (qi >= nq) return;
  const uint32_t q = qlist[qi];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint64_t LR = (uint64_t)L * RB;
  Best b{__longlong_as_double(0x7ff0000000000000ll), kNone, kNone};
  for (uint32_t p = blockIdx.x * nw + wib; p < size; p += gridDim.x * nw) {
    const double d = warp_exact_distance<CB>(probes + (uint64_t)q * LR, sqa + (uint64_t)q * L,
                                             counts + (uint64_t)p * LR, sqb + (uint64_t)p * L, L,
                                             C, RB);
    const uint64_t sq = seq[p];
    if (better(d, sq, b.d, b.seq)) b = Best{d, sq, p};
  }
  __shared__ Best wb[8];
  if (lane == 0) wb[wib] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t w = 1; w < nw; ++w)
      if (better(wb[w].d, wb[w].seq, b.d, b.seq)) b = wb[w];
    parts[(uint64_t)qi * gridDim.x + blockIdx.x] = moe_match{b.idx, b.seq, b.d};
  }
}

__global__ void k_merge_blocks(const moe_match* parts, uint32_t nb, const uint32_t* qlist,
                               uint32_t nq_list, const uint32_t* nq_dev, uint32_t q_off,
                               moe_match* out, uint64_t index_base) {
  pdl_wait();
  pdl_trigger();
  uint32_t nq = nq_list;
  if (nq_dev) {
    const uint32_t tot = *nq_dev;
    nq = tot > q_off ? min(tot - q_off, nq_list) : 0u;
  }
  const uint32_t qi = blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= nq) return;
  moe_match b = parts[(uint64_t)qi * nb];
  for (uint32_t k = 1; k < nb; ++k) {
    const moe_match m = parts[(uint64_t)qi * nb + k];
    if (better(m.distance, m.seq, b.distance, b.seq)) b = m;
  }
  out[qlist[qi]] = moe_match{b.index == kNone ? kNone : b.index + index_base, b.seq, b.distance};
}

__global__ void k_merge(const moe_match* parts, uint64_t n_parts, uint64_t n, moe_match* out) {
  const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (q >= n) return;
  // A part holding the width sentinel {UINT64_MAX-1, UINT64_MAX, NaN} (a
  // probe whose counts exceed that shard's storage width, match_all async
  // mode) poisons the merged answer: the caller must redo the probe through
  // the synchronous path, so the sentinel is never hidden by another shard.
  moe_match b = parts[q];
  bool poisoned = b.index == kNone - 1;
  for (uint64_t k = 1; k < n_parts; ++k) {
    const moe_match m = parts[k * n + q];
    poisoned |= m.index == kNone - 1;
    if (better(m.distance, m.seq, b.distance, b.seq)) b = m;
  }
  if (poisoned) b = moe_match{kNone - 1, kNone, __longlong_as_double(0x7ff8000000000000ll)};
  out[q] = b;
}

template <int CB>
__global__ void k_pair_distance(const uint8_t* a, const double* sqa, const uint8_t* b,
                                const double* sqb, uint32_t L, uint32_t C, uint32_t RB,
                                double* out) {
  const double d = warp_exact_distance<CB>(a, sqa, b, sqb, L, C, RB);
  if (threadIdx.x == 0) *out = d;
}

// u64 / u16 / u8 counts -> packed rows of cb-byte counts + sqrt(sum c^2)
// and fp32 1/sqrt(sum c^2); one warp per row.  Rows with sum c^2 >= 2^53
// (where the reference's own fp64 sums stop being exact, eam.cpp:75-87)
// report ~0 as their max count: MOE_ERR_OVERFLOW on the host.
constexpr uint64_t kNormLimit = 1ull << 53;
template <int SRC>
__device__ __forceinline__ uint64_t load_count(const void* src, uint64_t i) {
  if (SRC == 8) return reinterpret_cast<const uint64_t*>(src)[i];
  if (SRC == 4) return reinterpret_cast<const uint32_t*>(src)[i];
  if (SRC == 2) return reinterpret_cast<const uint16_t*>(src)[i];
  return reinterpret_cast<const uint8_t*>(src)[i];
}

template <int SRC>
__global__ void __launch_bounds__(256)
    k_prep(const void* src, uint64_t rows, uint32_t E, uint32_t L, uint32_t RB, int cb,
           uint8_t* dst, float* ia, double* sq, float* ibT, uint64_t ib_cap, uint64_t ib_base,
           unsigned long long* max_count, uint64_t width_limit, __half* nrm, uint32_t Kp,
           uint64_t* zmask, uint8_t* wide, MatchInit init) {
  // One warp per row (max parallelism, short latency chain).  The host only
  // needs to know whether some count exceeds the storage width, so the global
  // max is touched only by rows that actually do (no atomics in the common
  // case).  Zero rows set their bit in the (pre-zeroed) per-EAM mask; the last
  // row of an EAM also writes the operand's K padding.
  pdl_wait();
  pdl_trigger();
  const uint64_t row = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (row == 0 && lane == 0) {
    if (init.over_n) *init.over_n = 0;
    if (init.dmin) *init.dmin = ~0ull;
  }
  if (row >= rows) return;
  const uint64_t it = row / L;
  const uint32_t l = (uint32_t)(row - it * L);
  if (l == 0 && lane == 0 && init.T) {
    init.T[it] = 0x7f7f7f7fu;  // 3.4e38f > any distance
    init.bcnt[it] = 0;
  }
  const uint64_t sbase = row * E;
  uint32_t* drow = reinterpret_cast<uint32_t*>(dst + row * RB);
  const uint32_t per_word = 4 / cb;
  const uint32_t nwords = RB / 4;
  constexpr int kWords = 4;
  uint32_t words[kWords] = {0, 0, 0, 0};
  uint64_t ss = 0, mx = 0;
  for (uint32_t w = lane, k = 0; w < nwords; w += 32, ++k) {
    uint32_t word = 0;
    if (SRC == 1 && cb == 1 && (E & 3) == 0 && 4 * w + 3 < E) {
      word = reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(src) + sbase)[w];
      for (int j = 0; j < 4; ++j) {
        const uint64_t c = (word >> (8 * j)) & 0xffu;
        mx = c > mx ? c : mx;
        ss += c * c;
      }
    } else {
      for (uint32_t j = 0; j < per_word; ++j) {
        const uint32_t e = w * per_word + j;
        if (e < E) {
          const uint64_t c = load_count<SRC>(src, sbase + e);
          mx = c > mx ? c : mx;
          // saturating at 2^53: a row at or above it is outside the range the
          // reference's fp64 sums are exact in (flagged below)
          ss = c >= (1ull << 27) ? kNormLimit : min(ss + c * c, kNormLimit);
          const uint64_t cc = cb == 1 ? (c & 0xffu) : cb == 2 ? (c & 0xffffu) : (c & 0xffffffffu);
          word |= (uint32_t)cc << (8 * cb * j);
        }
      }
    }
    drow[w] = word;
    if (k < kWords) words[k] = word;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);  // < 2^58
  if (ss >= kNormLimit) mx = ~0ull;  // sum c^2 >= 2^53: no storage width represents it exactly
  if (mx > width_limit) {
    if (max_count) atomicMax(max_count, (unsigned long long)mx);
    if (wide) wide[it] = 1;  // this EAM does not fit the storage width
  }
  const double s = __dsqrt_rn(__ull2double_rn(ss));
  const float inv = ss ? __double2float_rn(__drcp_rn(s)) : 0.f;
  if (lane == 0) {
    sq[row] = s;
    if (ia) ia[row] = inv;
    if (ibT) ibT[(uint64_t)l * ib_cap + ib_base + it] = inv;
    if (zmask && ss == 0)
      atomicOr(reinterpret_cast<unsigned long long*>(&zmask[it]), 1ull << (l & 63));
  }
  if (nrm) {  // unit-normalised fp16 row of the tensor-core screen operand
    __half* o = nrm + it * (uint64_t)Kp + (uint64_t)l * E;
    if (nwords <= 32 * kWords) {
      for (uint32_t w = lane, k = 0; w < nwords; w += 32, ++k) {
        const uint32_t word = k < kWords ? words[k] : 0u;
        for (uint32_t j = 0; j < per_word; ++j) {
          const uint32_t e = w * per_word + j;
          if (e < E) {
            const uint32_t c = cb == 1 ? (word >> (8 * j)) & 0xffu
                               : cb == 2 ? (word >> (16 * j)) & 0xffffu
                                         : word;
            o[e] = __float2half_rn(__uint2float_rn(c) * inv);
          }
        }
      }
    } else {
      for (uint32_t e = lane; e < E; e += 32)
        o[e] = __float2half_rn(__uint2float_rn((uint32_t)load_count<SRC>(src, sbase + e)) * inv);
    }
    if (l == L - 1) {
      __half* orow = nrm + it * (uint64_t)Kp;
      for (uint32_t k = L * E + lane; k < Kp; k += 32) orow[k] = __float2half_rn(0.f);
    }
  }
}

// Fast path of k_prep for u8 counts into u8 storage (every probe batch that
// arrives narrowed, and u8 collections): one warp per EAM, its rows loaded
// 8 at a time before any is used (one memory round trip per 8 rows), Σc² by
// IDP4A + REDUX (exact: E <= 256 so Σc² < 2^24), fp16 operand written 8 B per
// lane, and the zero-row mask / width flag stored directly (no pre-zeroing
// launches).  Same outputs as k_prep<1> with cb = 1.
template <int WPL>
__global__ void __launch_bounds__(512)
    k_prep_u8(const uint8_t* src, uint64_t n, uint32_t E, uint32_t L, uint32_t RB, uint8_t* dst,
              float* ia, double* sq, float* ibT, uint64_t ib_cap, uint64_t ib_base, __half* nrm,
              uint32_t Kp, uint64_t* zmask, uint8_t* wide, uint32_t wpe,
              unsigned long long* max_count, MatchInit init) {
  // wpe warps per EAM (1 for large batches; up to 16 for a handful of probes,
  // where one warp walking all L rows would be a long latency chain); the
  // EAMs of a block never straddle blocks (wpe divides 16).
  __shared__ unsigned long long zsh[16];
  pdl_wait();
  pdl_trigger();
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t it = gw / wpe;
  const uint32_t sub = (uint32_t)(gw - it * wpe);
  const uint32_t slot = wib / wpe;
  if (sub == 0) zsh[slot] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // u8 counts always fit: nothing exceeds the width
    if (max_count) *max_count = 0;
    if (init.over_n) *init.over_n = 0;
    if (init.dmin) *init.dmin = ~0ull;
  }
  __syncthreads();
  const bool live = it < n;
  if (live && sub == 0 && lane == 0 && init.T) {
    init.T[it] = 0x7f7f7f7fu;
    init.bcnt[it] = 0;
  }
  const uint32_t ew = E >> 2, nwords = RB >> 2;
  // Row pointers advance by a fixed stride per row of this warp (64-bit adds
  // instead of per-row 64-bit multiplies).  dst == null: the caller reads
  // the packed rows from `src` itself (u8 source already in the storage
  // layout, RB == E), so no copy is written.
  const uint32_t* sp = reinterpret_cast<const uint32_t*>(src) + (it * L + sub) * ew + lane;
  uint32_t* dp = dst ? reinterpret_cast<uint32_t*>(dst) + (it * L + sub) * nwords + lane : nullptr;
  uint2* np = nrm ? reinterpret_cast<uint2*>(nrm + it * (uint64_t)Kp + (uint64_t)sub * E) + lane
                  : nullptr;
  const uint32_t s_stride = wpe * ew, d_stride = wpe * nwords, n_stride = wpe * (E >> 2);
  uint64_t zbits = 0;
  for (uint32_t l0 = sub; live && l0 < L; l0 += 8 * wpe) {
    uint32_t wv[8][WPL];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int k = 0; k < WPL; ++k)
        wv[r][k] = (l0 + r * wpe < L && lane + 32 * k < ew) ? __ldg(sp + r * s_stride + 32 * k) : 0u;
    sp += 8 * s_stride;
    // Σc² of the 8 rows (exact integers), then the fp64 scalars of row r on
    // lane r: one dsqrt/drcp sequence per 8 rows instead of one per row.
    uint32_t my_ss = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      uint32_t ss = 0;
#pragma unroll
      for (int k = 0; k < WPL; ++k) ss = __dp4a(wv[r][k], wv[r][k], ss);
      ss = __reduce_add_sync(0xffffffffu, ss);
      my_ss = (lane & 7) == (uint32_t)r ? ss : my_ss;
    }
    {  // zero rows of this group (lane r <-> row l0 + r * wpe)
      uint32_t zb = __ballot_sync(0xffffffffu, lane < 8 && l0 + lane * wpe < L && my_ss == 0);
      while (zb) {
        const uint32_t r = __ffs(zb) - 1;
        zb &= zb - 1;
        zbits |= 1ull << ((l0 + r * wpe) & 63);
      }
    }
    const double my_sd = __dsqrt_rn((double)my_ss);
    const float my_inv = my_ss ? __double2float_rn(__drcp_rn(my_sd)) : 0.f;
    {
      const uint32_t l = l0 + lane * wpe;
      if (lane < 8 && l < L) {
        const uint64_t row = it * L + l;
        sq[row] = my_sd;
        if (ia) ia[row] = my_inv;
        if (ibT) ibT[(uint64_t)l * ib_cap + ib_base + it] = my_inv;
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (l0 + r * wpe >= L) break;
      const float inv = __shfl_sync(0xffffffffu, my_inv, r);
      if (dp) {
#pragma unroll
        for (int k = 0; k < WPL; ++k)
          if (lane + 32 * k < nwords) dp[r * d_stride + 32 * k] = wv[r][k];
      }
      if (np) {
#pragma unroll
        for (int k = 0; k < WPL; ++k) {
          if (lane + 32 * k < ew) {
            const uint32_t x = wv[r][k];
            const __half2 lo = __floats2half2_rn(__uint2float_rn(x & 0xffu) * inv,
                                                 __uint2float_rn((x >> 8) & 0xffu) * inv);
            const __half2 hi = __floats2half2_rn(__uint2float_rn((x >> 16) & 0xffu) * inv,
                                                 __uint2float_rn(x >> 24) * inv);
            uint2 v;
            v.x = *reinterpret_cast<const uint32_t*>(&lo);
            v.y = *reinterpret_cast<const uint32_t*>(&hi);
            np[r * n_stride + 32 * k] = v;
          }
        }
      }
    }
    if (dp) dp += 8 * d_stride;
    if (np) np += 8 * n_stride;
  }
  if (live && lane == 0 && zbits) atomicOr(&zsh[slot], (unsigned long long)zbits);
  __syncthreads();
  if (!live || sub != 0) return;
  if (nrm) {
    __half* orow = nrm + it * (uint64_t)Kp;
    for (uint32_t k = L * E + lane; k < Kp; k += 32) orow[k] = __float2half_rn(0.f);
  }
  if (lane == 0) {
    if (zmask) zmask[it] = zsh[slot];
    if (wide) wide[it] = 0;
  }
}

__global__ void k_replace(uint8_t* counts, float* ibT, double* sqb, uint64_t* seq, uint64_t cap,
                          uint32_t L, uint32_t RB, const uint8_t* sp, const float* sia,
                          const double* ssq, uint32_t i, const moe_match* victim,
                          uint64_t append_slot, uint64_t seq_value, const int* halt,
                          uint64_t index_base, __half* nrm, const __half* snrm, uint32_t Kp,
                          uint64_t* zmask, const uint64_t* szmask) {
  if (halt && *halt) return;
  const uint64_t slot = victim ? victim->index - index_base : append_slot;
  if (nrm) {
    const uint4* s4 = reinterpret_cast<const uint4*>(snrm + (uint64_t)i * Kp);
    uint4* d4 = reinterpret_cast<uint4*>(nrm + slot * Kp);
    for (uint32_t o = threadIdx.x; o < Kp / 8; o += blockDim.x) d4[o] = s4[o];
    if (threadIdx.x == 0) zmask[slot] = szmask[i];
  }
  const uint64_t LR = (uint64_t)L * RB;
  const uint4* src = reinterpret_cast<const uint4*>(sp + (uint64_t)i * LR);
  uint4* dst = reinterpret_cast<uint4*>(counts + slot * LR);
  for (uint32_t o = threadIdx.x; o < LR / 16; o += blockDim.x) dst[o] = src[o];
  for (uint32_t l = threadIdx.x; l < L; l += blockDim.x) {
    ibT[(uint64_t)l * cap + slot] = sia[(uint64_t)i * L + l];
    sqb[slot * L + l] = ssq[(uint64_t)i * L + l];
  }
  if (threadIdx.x == 0) seq[slot] = seq_value;
}

// Blocked construction replay (K7, Eamc::insert at capacity, eam.cpp:164-177).
// For a block of nb incoming EAMs x_0..x_{nb-1} the screen distances to the
// collection as it stood before the block (dc [nb][P]) and to each other
// (dx [nb][nb]) come from one tensor-core GEMM each; this ONE-CTA kernel then
// replays the nb sequential decisions: at step t the occupant of slot p is
// the original entry (occ[p] < 0) or x_occ[p], with screen distance
// dc[t][p] or dx[t][occ[p]]; every slot within the screen band
// (<= min + eps2, the same proof as the matcher's) is re-evaluated exactly
// in the reference operation order and the lexicographic (distance, seq)
// minimum is the victim.  k_apply_block then writes each replaced slot's
// final occupant into the collection.
constexpr uint32_t kReplayThreads = 512;
constexpr uint32_t kReplayCand = 512;  // >= kReplayThreads (the slice walk relies on it)

struct ReplayArgs {
  const uint8_t* counts;
  const double* sqb;
  const uint64_t* seq;
  uint32_t P, L, C, RB;
  uint64_t index_base;
  const uint8_t* xp;    // [nb][L][RB] packed incoming EAMs of the block
  const double* xsq;    // [nb][L] their row norms
  uint32_t nb;
  const float* dc;      // [nb][ldc]
  const float* dx;      // [nb][ldx]
  uint32_t ldc, ldx;
  float eps2;
  int* occ;             // [P], -1 = original entry (all -1 on entry and exit of a block)
  unsigned long long* prof;  // optional [4] phase cycle totals (thread 0's view)
  uint64_t seq0;        // seq given to step 0 of the block
  moe_match* vic;       // [nb] victims
};

__device__ __forceinline__ float block_min_f(float v, float* sbuf) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sbuf[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < (blockDim.x >> 5) ? sbuf[lane] : __uint_as_float(0x7f800000u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) sbuf[32] = v;
  }
  __syncthreads();
  return sbuf[32];
}

constexpr uint32_t kReplayMaxP = 16384;  // slots held in registers / shared memory per step
constexpr uint32_t kRW = 8;              // refine warps (each stages one candidate's rows)
constexpr uint32_t kReplayBlockMax = 1024;  // steps per replay block (dx row capacity)
constexpr int kXsPer = 2;                // 16-byte chunks of x_t per thread (L*RB <= 16 KB)
constexpr int kReplayRT = kReplayMaxP / (4 * kReplayThreads);  // float4 groups per thread

template <int CB>
__global__ void __launch_bounds__(kReplayThreads, 1) k_replay_block(const ReplayArgs a) {
  // dynamic: occ_s [P4*4] int16 | xs [L*RB] (x_t) | es [kRW][L*RB] | esq [kRW][64] f64
  //          | drow [2][P4*4] f32 (screen rows t, t+1, filled by bulk copies)
  extern __shared__ __align__(16) uint8_t rsm[];
  int16_t* occ_s = reinterpret_cast<int16_t*>(rsm);
  __shared__ __align__(8) uint64_t rbar[2];
  __shared__ float sbuf[33];
  __shared__ uint32_t cand[kReplayCand];
  __shared__ uint32_t ncand;
  __shared__ double rbuf[kReplayThreads / 32][64];
  __shared__ double xsq_s[64];
  __shared__ double bd[kReplayThreads / 32];
  __shared__ unsigned long long bs[kReplayThreads / 32];
  __shared__ uint32_t bp[kReplayThreads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  const uint64_t LR = (uint64_t)a.L * a.RB;
  const uint32_t P4 = (a.P + 3) >> 2;  // float4 groups of a dc row (ldc % 4 == 0)
  const uint32_t LR16 = (uint32_t)(LR / 16);
  uint4* xs = reinterpret_cast<uint4*>(rsm + (((size_t)P4 * 8 + 15) & ~(size_t)15));
  uint4* es = xs + LR16;
  double* esq = reinterpret_cast<double*>(es + (size_t)kRW * LR16);
  float* drow = reinterpret_cast<float*>(esq + (size_t)kRW * 64);
  const uint32_t row_bytes = P4 * 16;
  for (uint32_t p = tid; p < ((a.P + 3) & ~3u); p += blockDim.x) occ_s[p] = -1;
  if (tid == 0) {
    mbar_init(&rbar[0], 1);
    mbar_init(&rbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  float* dxrow = drow + (size_t)2 * P4 * 4;  // [2][ldx]
  const uint32_t dx_bytes = a.ldx * 4;
  auto fetch_row = [&](uint32_t t) {  // one thread: screen rows t of dc and dx -> buffer t & 1
    uint64_t* bar = &rbar[t & 1];
    mbar_arrive_expect_tx(bar, row_bytes + dx_bytes);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(drow + (size_t)(t & 1) * P4 * 4)),
        "l"(a.dc + (uint64_t)t * a.ldc), "r"(row_bytes), "r"(smem_u32(bar))
        : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dxrow + (size_t)(t & 1) * a.ldx)),
        "l"(a.dx + (uint64_t)t * a.ldx), "r"(dx_bytes), "r"(smem_u32(bar))
        : "memory");
  };
  if (tid == 0 && a.nb) fetch_row(0);
  if (a.nb) {  // x_0 -> shared memory
    const uint4* src = reinterpret_cast<const uint4*>(a.xp);
    for (uint32_t k = tid; k < LR16; k += blockDim.x) xs[k] = src[k];
    if (tid < a.L) xsq_s[tid] = a.xsq[tid];
  }
  __syncthreads();
  unsigned long long c0 = 0, c1 = 0, c2 = 0, c3 = 0, acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0,
                     acc4 = 0;
  for (uint32_t t = 0; t < a.nb; ++t) {
    if (a.prof) c0 = clock64();
    const float* dxt = a.dx + (uint64_t)t * a.ldx;
    // the next step's incoming EAM and row norms: loads issued now, stored to
    // shared memory at the end of this step (their latency hides behind it)
    uint4 nx[kXsPer];
    double nsq = 0.0;
    if (t + 1 < a.nb) {
      const uint4* src = reinterpret_cast<const uint4*>(a.xp + (uint64_t)(t + 1) * LR);
#pragma unroll
      for (int u = 0; u < kXsPer; ++u) {
        const uint32_t k = tid + u * blockDim.x;
        if (k < LR16) nx[u] = __ldg(src + k);
      }
      if (tid < a.L) nsq = a.xsq[(uint64_t)(t + 1) * a.L + tid];
    }
    // pass 1: the step's screen row (prefetched into shared memory during the
    // previous step by a bulk copy), kept in registers for pass 2; slots
    // replaced earlier in the block take their occupant's row of dx instead
    mbar_wait(&rbar[t & 1], (t >> 1) & 1);
    if (a.prof && tid == 0) acc4 += clock64() - c0;
    const float4* srow4 = reinterpret_cast<const float4*>(drow + (size_t)(t & 1) * P4 * 4);
    const float* sdx = dxrow + (size_t)(t & 1) * a.ldx;
    float v[kReplayRT][4];
#pragma unroll
    for (int r = 0; r < kReplayRT; ++r) {
      const uint32_t g = tid + r * kReplayThreads;
      const float4 x = g < P4 ? srow4[g] : make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
      v[r][0] = x.x;
      v[r][1] = x.y;
      v[r][2] = x.z;
      v[r][3] = x.w;
    }
    float m = __uint_as_float(0x7f800000u);
#pragma unroll
    for (int r = 0; r < kReplayRT; ++r) {
      const uint32_t g = tid + r * kReplayThreads;
      if (g >= P4) break;
      const uint2 oc = *reinterpret_cast<const uint2*>(occ_s + 4 * g);  // 4 x int16
      const int o4[4] = {(int)(int16_t)(oc.x & 0xffffu), (int)(int16_t)(oc.x >> 16),
                         (int)(int16_t)(oc.y & 0xffffu), (int)(int16_t)(oc.y >> 16)};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (4 * g + j >= a.P) v[r][j] = INFINITY;
        else if (o4[j] >= 0) v[r][j] = sdx[o4[j]];
        m = fminf(m, v[r][j]);
      }
    }
    if (tid == 0) ncand = 0;
    const float thr = block_min_f(m, sbuf) + a.eps2;
    // every thread has its screen values in registers now: buffer (t+1)&1 was
    // last read in step t-1, so the next row can land in it
    if (tid == 0 && t + 1 < a.nb) {
      fence_proxy_async();  // generic reads of that buffer before the async-proxy write
      fetch_row(t + 1);
    }
    if (a.prof) c1 = clock64();
    // pass 2: candidates inside the band
#pragma unroll
    for (int r = 0; r < kReplayRT; ++r) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (v[r][j] <= thr) {
          const uint32_t pos = atomicAdd(&ncand, 1u);
          if (pos < kReplayCand) cand[pos] = 4 * (tid + r * kReplayThreads) + j;
        }
    }
    __syncthreads();
    if (a.prof) c2 = clock64();
    const uint32_t nc = ncand;
    double best_d = __longlong_as_double(0x7ff0000000000000ll);
    unsigned long long best_s = ~0ull;
    uint32_t best_p = 0xffffffffu;
    const double* sqt = xsq_s;
    // exact re-evaluation, one candidate per refine warp: the candidate's
    // rows and row norms are first copied to shared memory with every load
    // of the warp in flight (one memory round trip), then each row's dot is
    // taken over C lanes (consecutive chunks) and reduced by shuffles when C
    // is a power of two, or by one lane per layer otherwise.
    const bool seg = (a.C & (a.C - 1)) == 0 && a.C <= 32;
    const uint32_t lpi = seg ? 32 / a.C : 0;  // layers per warp iteration
    auto refine = [&](uint32_t n_list) {
      if (w >= kRW) return;
      uint4* er = es + (size_t)w * LR16;
      double* eq = esq + (size_t)w * 64;
      const uint8_t* xb = reinterpret_cast<const uint8_t*>(xs);
      for (uint32_t ci = w; ci < n_list; ci += kRW) {
        const uint32_t p = cand[ci];
        const int o = occ_s[p];
        const unsigned long long sq = o < 0 ? a.seq[p] : a.seq0 + (uint64_t)o;  // early
        const uint4* eg = reinterpret_cast<const uint4*>(o < 0 ? a.counts + (uint64_t)p * LR
                                                                : a.xp + (uint64_t)o * LR);
        const double* sg = o < 0 ? a.sqb + (uint64_t)p * a.L : a.xsq + (uint64_t)o * a.L;
        // all loads first (up to 8 per lane in flight), then the stores
        for (uint32_t k0 = 0; k0 < LR16; k0 += 8 * 32) {
          uint4 tmp[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint32_t k = k0 + u * 32 + lane;
            if (k < LR16) tmp[u] = __ldg(eg + k);
          }
          const double q0 = lane < a.L && k0 == 0 ? sg[lane] : 0.0;
          const double q1 = lane + 32 < a.L && k0 == 0 ? sg[lane + 32] : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint32_t k = k0 + u * 32 + lane;
            if (k < LR16) er[k] = tmp[u];
          }
          if (k0 == 0) {
            if (lane < a.L) eq[lane] = q0;
            if (lane + 32 < a.L) eq[lane + 32] = q1;
          }
        }
        __syncwarp();
        const uint8_t* ebb = reinterpret_cast<const uint8_t*>(er);
        if (true) {  // lane per layer from shared memory, chunk order rotated by layer
          for (uint32_t l = lane; l < a.L; l += 32) {
            const uint4* ra = reinterpret_cast<const uint4*>(xb + (uint64_t)l * a.RB);
            const uint4* rb = reinterpret_cast<const uint4*>(ebb + (uint64_t)l * a.RB);
            typename Dot<CB>::Acc acc = 0;
            uint32_t cc = l % a.C;
            for (uint32_t k = 0; k < a.C; ++k) {
              acc = Dot<CB>::chunk(ra[cc], rb[cc], acc);
              cc = cc + 1 == a.C ? 0 : cc + 1;
            }
            rbuf[w][l] = row_sim_exact((uint64_t)acc, sqt[l], eq[l]);
          }
        } else if (seg) {
          const uint32_t c = lane & (a.C - 1);
          for (uint32_t l0 = 0; l0 < a.L; l0 += lpi) {
            const uint32_t l = l0 + lane / a.C;
            typename Dot<CB>::Acc acc = 0;
            if (l < a.L)
              acc = Dot<CB>::chunk(reinterpret_cast<const uint4*>(xb + (uint64_t)l * a.RB)[c],
                                   reinterpret_cast<const uint4*>(ebb + (uint64_t)l * a.RB)[c], acc);
            for (uint32_t off = 1; off < a.C; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (c == 0 && l < a.L) rbuf[w][l] = __longlong_as_double((long long)(uint64_t)acc);
          }
          __syncwarp();
          // the fp64 row similarities of all layers in parallel (one ddiv latency)
          for (uint32_t l = lane; l < a.L; l += 32)
            rbuf[w][l] = row_sim_exact((uint64_t)__double_as_longlong(rbuf[w][l]), sqt[l], eq[l]);
        } else {
          for (uint32_t l = lane; l < a.L; l += 32) {
            const uint4* ra = reinterpret_cast<const uint4*>(xb + (uint64_t)l * a.RB);
            const uint4* rb = reinterpret_cast<const uint4*>(ebb + (uint64_t)l * a.RB);
            typename Dot<CB>::Acc acc = 0;
            for (uint32_t cc = 0; cc < a.C; ++cc) acc = Dot<CB>::chunk(ra[cc], rb[cc], acc);
            rbuf[w][l] = row_sim_exact((uint64_t)acc, sqt[l], eq[l]);
          }
        }
        __syncwarp();
        if (lane == 0) {
          double sm = 0.0;
          uint32_t l = 0;
          for (; l + 8 <= a.L; l += 8) {
            double x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = rbuf[w][l + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) sm = __dadd_rn(sm, x[u]);
          }
          for (; l < a.L; ++l) sm = __dadd_rn(sm, rbuf[w][l]);
          const double d = finish_distance(sm, a.L);
          if (better(d, sq, best_d, best_s)) {
            best_d = d;
            best_s = sq;
            best_p = p;
          }
        }
        __syncwarp();
      }
    };
    if (nc <= kReplayCand) {
      refine(nc);
    } else {
      // mass near-ties: walk the band in slot order, one slice of
      // kReplayThreads slots at a time (each slice has at most kReplayCand members)
      for (uint32_t r0 = 0; r0 < a.P; r0 += blockDim.x) {
        __syncthreads();
        if (tid == 0) ncand = 0;
        __syncthreads();
        const uint32_t p = r0 + tid;
        if (p < a.P) {
          const int o = occ_s[p];
          if ((o < 0 ? a.dc[(uint64_t)t * a.ldc + p] : dxt[o]) <= thr)
            cand[atomicAdd(&ncand, 1u)] = p;
        }
        __syncthreads();
        refine(ncand);
      }
    }
    if (a.prof) {
      c3 = clock64();
      acc0 += c1 - c0;
      acc1 += c2 - c1;
      acc2 += c3 - c2;
    }
    if (lane == 0) {
      bd[w] = best_d;
      bs[w] = best_s;
      bp[w] = best_p;
    }
    __syncthreads();
    if (w == 0) {  // lexicographic (distance, seq) minimum over the warps
      Best b{__longlong_as_double(0x7ff0000000000000ll), ~0ull, 0xffffffffull};
      if (lane < nw) b = Best{bd[lane], bs[lane], bp[lane]};
      b = warp_best(b);
      if (lane == 0) {
        const uint32_t pp = (uint32_t)b.idx;
        a.vic[t] = moe_match{pp + a.index_base, b.seq, b.d};
        a.occ[pp] = (int)t;
        occ_s[pp] = (int16_t)t;
      }
    }
    __syncthreads();
    if (t + 1 < a.nb) {  // x_{t+1} -> shared memory (this step's readers are done)
#pragma unroll
      for (int u = 0; u < kXsPer; ++u) {
        const uint32_t k = tid + u * blockDim.x;
        if (k < LR16) xs[k] = nx[u];
      }
      if (tid < a.L) xsq_s[tid] = nsq;
    }
    if (a.prof) acc3 += clock64() - c3;
  }
  if (a.prof && tid == 0) {
    atomicAdd(a.prof + 0, acc0);
    atomicAdd(a.prof + 1, acc1);
    atomicAdd(a.prof + 2, acc2);
    atomicAdd(a.prof + 3, acc3);
  }
  if (a.prof && tid == 32) atomicAdd(a.prof + 4, acc2);  // a refine warp's view
  if (a.prof && tid == 0) atomicAdd(a.prof + 5, acc4);   // waiting for the screen row
}

// Final occupants of the slots replaced in a block -> the collection (the
// data k_replace writes for a single step); resets occ for the next block.
__global__ void k_apply_block(uint8_t* counts, float* ibT, double* sqb, uint64_t* seq,
                              uint64_t cap, uint32_t L, uint32_t RB, const uint8_t* sp,
                              const float* sia, const double* ssq, const moe_match* vic,
                              int* occ, uint64_t seq0, uint64_t index_base, __half* nrm,
                              const __half* snrm, uint32_t Kp, uint64_t* zmask,
                              const uint64_t* szmask) {
  const uint32_t t = blockIdx.x;
  const uint64_t slot = vic[t].index - index_base;
  if (occ[slot] != (int)t) return;  // a later step of the block replaced it again
  __syncthreads();
  if (nrm) {
    const uint4* s4 = reinterpret_cast<const uint4*>(snrm + (uint64_t)t * Kp);
    uint4* d4 = reinterpret_cast<uint4*>(nrm + slot * Kp);
    for (uint32_t o = threadIdx.x; o < Kp / 8; o += blockDim.x) d4[o] = s4[o];
    if (threadIdx.x == 0) zmask[slot] = szmask[t];
  }
  const uint64_t LR = (uint64_t)L * RB;
  const uint4* src = reinterpret_cast<const uint4*>(sp + (uint64_t)t * LR);
  uint4* dst = reinterpret_cast<uint4*>(counts + slot * LR);
  for (uint32_t o = threadIdx.x; o < LR / 16; o += blockDim.x) dst[o] = src[o];
  for (uint32_t l = threadIdx.x; l < L; l += blockDim.x) {
    ibT[(uint64_t)l * cap + slot] = sia[(uint64_t)t * L + l];
    sqb[slot * L + l] = ssq[(uint64_t)t * L + l];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    seq[slot] = seq0 + t;
    occ[slot] = -1;
  }
}

__global__ void k_append_staged(uint8_t* counts, float* ibT, double* sqb, uint64_t cap, uint32_t L,
                                uint32_t RB, const uint8_t* sp, const float* sia,
                                const double* ssq, uint32_t first, uint32_t n, uint64_t base,
                                __half* nrm, const __half* snrm, uint32_t Kp, uint64_t* zmask,
                                const uint64_t* szmask) {
  if (nrm) {
    const uint64_t w16 = (uint64_t)n * Kp / 8;
    const uint4* s4 = reinterpret_cast<const uint4*>(snrm + (uint64_t)first * Kp);
    uint4* d4 = reinterpret_cast<uint4*>(nrm + base * Kp);
    for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < w16;
         o += (uint64_t)gridDim.x * blockDim.x)
      d4[o] = s4[o];
    for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < n;
         o += (uint64_t)gridDim.x * blockDim.x)
      zmask[base + o] = szmask[first + o];
  }
  const uint64_t LR = (uint64_t)L * RB;
  const uint64_t words = (uint64_t)n * LR / 16;
  const uint4* src = reinterpret_cast<const uint4*>(sp + (uint64_t)first * LR);
  uint4* dst = reinterpret_cast<uint4*>(counts + base * LR);
  for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < words;
       o += (uint64_t)gridDim.x * blockDim.x)
    dst[o] = src[o];
  for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < (uint64_t)n * L;
       o += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = o / L;
    const uint32_t l = (uint32_t)(o % L);
    ibT[(uint64_t)l * cap + base + e] = sia[((uint64_t)first + e) * L + l];
    sqb[(base + e) * L + l] = ssq[((uint64_t)first + e) * L + l];
  }
}

// Re-encode rows of cb_old-byte counts as cb_new-byte counts (padding zero).
__global__ void k_widen(const uint8_t* src, uint8_t* dst, uint64_t rows, uint32_t RB_old,
                        uint32_t RB_new, int cb_old, int cb_new) {
  const uint32_t n_old = RB_old / cb_old, n_new = RB_new / cb_new;
  for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < rows * n_new;
       o += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = o / n_new;
    const uint32_t e = (uint32_t)(o % n_new);
    uint32_t v = 0;
    if (e < n_old) {
      const uint8_t* so = src + r * RB_old;
      v = cb_old == 1 ? so[e] : cb_old == 2 ? reinterpret_cast<const uint16_t*>(so)[e]
                                            : reinterpret_cast<const uint32_t*>(so)[e];
    }
    uint8_t* d = dst + r * RB_new;
    if (cb_new == 2) reinterpret_cast<uint16_t*>(d)[e] = (uint16_t)v;
    else reinterpret_cast<uint32_t*>(d)[e] = v;
  }
}

__global__ void k_window_list(const double* dist, const unsigned long long* dmin, double window,
                              const uint64_t* seq, uint32_t size, WinEntry* wl, uint32_t* wl_n) {
  const double thr = __dadd_rn(__longlong_as_double((long long)*dmin), window);
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < size; p += gridDim.x * blockDim.x) {
    const double d = dist[p];
    if (d <= thr) wl[atomicAdd(wl_n, 1u)] = WinEntry{p, seq[p], d};
  }
}

// ---- single-probe decision path (match_within / prefetch_priorities) ------
// Row-parallel exact similarities: thread per (entry, layer) row, reading the
// row (RB bytes, warp-contiguous in the AoS layout) and the probe row; the
// per-row fp64 similarity goes to r[p*L + l].
template <int CB>
__global__ void __launch_bounds__(256)
    k_rowsim(const uint8_t* counts, const double* sqb, uint32_t size, uint32_t L, uint32_t C,
             uint32_t RB, const uint8_t* probe, const double* sqa, uint32_t l0, uint32_t l1,
             double* r) {
  const uint32_t nl = l1 - l0;
  const uint64_t n = (uint64_t)size * nl;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = i / nl;
    const uint32_t l = l0 + (uint32_t)(i - p * nl);
    const uint4* ra = reinterpret_cast<const uint4*>(probe + (uint64_t)l * RB);
    const uint4* rb = reinterpret_cast<const uint4*>(counts + (p * L + l) * RB);
    typename Dot<CB>::Acc acc = 0;
    for (uint32_t c = 0; c < C; ++c) acc = Dot<CB>::chunk(ra[c], __ldg(&rb[c]), acc);
    r[p * L + l] = row_sim_exact((uint64_t)acc, sqa[l], sqb[p * L + l]);
  }
}

// In-order layer sum (eam.cpp:95-103) -> dist[p]; warp min -> atomicMin(*dmin).
__global__ void __launch_bounds__(256)
    k_rowsum(const double* r, uint32_t size, uint32_t L, double* dist, unsigned long long* dmin) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  double d = __longlong_as_double(0x7ff0000000000000ll);
  if (p < size) {
    double sm = 0.0;
    const double* rr = r + (uint64_t)p * L;
    for (uint32_t l = 0; l < L; ++l) sm = __dadd_rn(sm, rr[l]);
    d = finish_distance(sm, L);
    dist[p] = d;
  }
  unsigned long long b = (unsigned long long)__double_as_longlong(d);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, b, o);
    b = x < b ? x : b;
  }
  if ((threadIdx.x & 31) == 0 && b != 0x7ff0000000000000ull) atomicMin(dmin, b);
}

// Window members (dist <= d_min + window, eam.cpp:143) -> compact list.
__global__ void k_members(const double* dist, const unsigned long long* dmin, double window,
                          uint32_t size, uint32_t* mem, uint32_t* n_mem) {
  pdl_wait();
  pdl_trigger();
  const double thr = __dadd_rn(__longlong_as_double((long long)*dmin), window);
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < size; p += gridDim.x * blockDim.x)
    if (dist[p] <= thr) mem[atomicAdd(n_mem, 1u)] = p;
}

// u64 aggregation of the members' rows > cur (policy.cpp:97-104): thread per
// 4-byte word of the row region, a chunk of members per blockIdx.y, loads
// unrolled for memory-level parallelism, one atomic per nonzero cell.
template <int CB>
__global__ void __launch_bounds__(256)
    k_member_agg(const uint8_t* counts, uint32_t L, uint32_t E, uint32_t RB, uint32_t cur,
                 const uint32_t* mem, const uint32_t* n_mem, uint32_t chunk,
                 unsigned long long* agg) {
  pdl_wait();
  pdl_trigger();
  const uint32_t rows = L - cur - 1;
  const uint32_t wpr = RB / 4;  // words per row
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t n = *n_mem;
  const uint32_t m0 = blockIdx.y * chunk;
  if (w >= rows * wpr || m0 >= n) return;
  const uint32_t m1 = min(n, m0 + chunk);
  const uint32_t r = w / wpr, wi = w - r * wpr;
  const uint64_t off = (uint64_t)(cur + 1 + r) * RB + 4ull * wi;
  const uint64_t LR = (uint64_t)L * RB;
  // per-cell partial sums (u32 for 1-2 byte counts: <= chunk * 65535; u64 for u32 counts)
  using Sum = typename std::conditional<CB == 4, uint64_t, uint32_t>::type;
  Sum s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  uint32_t m = m0;
  for (; m + 4 <= m1; m += 4) {
    uint32_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      v[k] = __ldg(reinterpret_cast<const uint32_t*>(counts + mem[m + k] * LR + off));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (CB == 1) {
        s0 += v[k] & 0xffu;
        s1 += (v[k] >> 8) & 0xffu;
        s2 += (v[k] >> 16) & 0xffu;
        s3 += v[k] >> 24;
      } else if (CB == 2) {
        s0 += v[k] & 0xffffu;
        s1 += v[k] >> 16;
      } else {
        s0 += v[k];
      }
    }
  }
  for (; m < m1; ++m) {
    const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(counts + mem[m] * LR + off));
    if (CB == 1) {
      s0 += v & 0xffu;
      s1 += (v >> 8) & 0xffu;
      s2 += (v >> 16) & 0xffu;
      s3 += v >> 24;
    } else if (CB == 2) {
      s0 += v & 0xffffu;
      s1 += v >> 16;
    } else {
      s0 += v;
    }
  }
  const uint32_t per = 4 / CB;
  const uint32_t e0 = wi * per;
  const uint64_t base = (uint64_t)(cur + 1 + r) * E;
  const Sum sums[4] = {s0, s1, s2, s3};
  for (uint32_t k = 0; k < per; ++k)
    if (e0 + k < E && sums[k]) atomicAdd(&agg[base + e0 + k], (unsigned long long)sums[k]);
}

// K5+K6 fused decision kernel (one block).
__global__ void __launch_bounds__(1024)
    k_decide(const unsigned long long* agg, uint32_t L, uint32_t E, uint32_t cur, int filter,
             int do_prefetch, const unsigned long long* req, const moe_slot_view* slots,
             uint64_t n_slots, moe_candidate* out, uint32_t* n_out, long long* victim,
             double* slot_pri, uint32_t npow2) {
  extern __shared__ __align__(16) uint8_t sm[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(sm);
  uint32_t* val = reinterpret_cast<uint32_t*>(key + npow2);
  unsigned long long* rs = reinterpret_cast<unsigned long long*>(val + npow2);  // [L] agg rows
  unsigned long long* rq = rs + L;                                             // [L] req rows
  __shared__ uint32_t cnt;
  __shared__ double vbest_p[32];
  __shared__ uint64_t vbest_k[32];
  __shared__ long long vbest_s[32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const double kEps = 1e-4;  // policy.hpp:22
  if (tid == 0) cnt = 0;
  for (uint32_t l = wid; l < L; l += nw) {
    unsigned long long a = 0, b = 0;
    for (uint32_t e = lane; e < E; e += 32) {
      if (do_prefetch && l > cur) a += agg[(uint64_t)l * E + e];
      if (req) b += req[(uint64_t)l * E + e];
    }
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (lane == 0) {
      rs[l] = a;
      rq[l] = b;
    }
  }
  __syncthreads();
  if (do_prefetch) {
    const uint32_t first = (cur + 1) * E;
    const uint32_t n = L * E - first;
    for (uint32_t i = tid; i < n; i += blockDim.x) {
      const uint32_t flat = first + i;
      const uint32_t l = flat / E;
      const unsigned long long rsum = rs[l];
      const double ratio =
          rsum == 0 ? 0.0 : __ddiv_rn(__ull2double_rn(agg[flat]), __ull2double_rn(rsum));
      const double prox = __dsub_rn(1.0, __ddiv_rn((double)(l - cur), (double)L));
      const double pri = __dmul_rn(__dadd_rn(ratio, kEps), prox);
      if (filter && pri <= __dmul_rn(__dmul_rn(kEps, prox), __dadd_rn(1.0, 1e-9))) continue;
      const uint32_t pos = atomicAdd(&cnt, 1u);
      key[pos] = ~(unsigned long long)__double_as_longlong(pri);  // descending priority
      val[pos] = flat;
    }
    __syncthreads();
    const uint32_t m = cnt;
    uint32_t np = 1;
    while (np < m) np <<= 1;
    for (uint32_t i = m + tid; i < np; i += blockDim.x) {
      key[i] = ~0ull;
      val[i] = 0xffffffffu;
    }
    __syncthreads();
    // bitonic sort on (key asc, val asc)
    for (uint32_t k = 2; k <= np; k <<= 1) {
      for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
        for (uint32_t i = tid; i < np; i += blockDim.x) {
          const uint32_t ixj = i ^ jj;
          if (ixj > i) {
            const bool up = (i & k) == 0;
            const unsigned long long ki = key[i], kj = key[ixj];
            const uint32_t vi = val[i], vj = val[ixj];
            const bool gt = ki > kj || (ki == kj && vi > vj);
            if (gt == up) {
              key[i] = kj;
              key[ixj] = ki;
              val[i] = vj;
              val[ixj] = vi;
            }
          }
        }
        __syncthreads();
      }
    }
    for (uint32_t i = tid; i < m; i += blockDim.x) {
      const uint32_t flat = val[i];
      moe_candidate c;
      c.layer_idx = flat / E;
      c.expert_idx = flat - c.layer_idx * E;
      c.priority = __longlong_as_double((long long)~key[i]);
      out[i] = c;
    }
    if (tid == 0) *n_out = m;
  }
  if (victim || slot_pri) {
    // select_eviction_victim: argmin (cache_priority, ExpertId) over
    // unprotected, unpinned slots (policy.cpp:143-159).
    double bp = 0.0;
    uint64_t bk = ~0ull;
    long long bs = -1;
    for (uint64_t i = tid; i < n_slots; i += blockDim.x) {
      const moe_slot_view v = slots[i];
      if (!slot_pri && (v.prefetch_protected || v.pinned)) continue;
      const unsigned long long rsum = rq[v.layer_idx];
      const double ratio =
          rsum == 0 ? 0.0
                    : __ddiv_rn(__ull2double_rn(req[(uint64_t)v.layer_idx * E + v.expert_idx]),
                                __ull2double_rn(rsum));
      const double w = __dsub_rn(1.0, __ddiv_rn((double)v.layer_idx, (double)L));
      const double p = __dmul_rn(__dadd_rn(ratio, kEps), w);
      if (slot_pri) slot_pri[i] = p;
      if (v.prefetch_protected || v.pinned) continue;
      const uint64_t k = ((uint64_t)v.layer_idx << 32) | v.expert_idx;
      if (bs < 0 || p < bp || (p == bp && k < bk)) {
        bp = p;
        bk = k;
        bs = (long long)v.slot;
      }
    }
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
      vbest_p[wid] = bp;
      vbest_k[wid] = bk;
      vbest_s[wid] = bs;
    }
    __syncthreads();
    if (tid == 0 && victim) {
      for (uint32_t w = 1; w < nw; ++w) {
        if (vbest_s[w] >= 0 &&
            (bs < 0 || vbest_p[w] < bp || (vbest_p[w] == bp && vbest_k[w] < bk))) {
          bp = vbest_p[w];
          bk = vbest_k[w];
          bs = vbest_s[w];
        }
      }
      *victim = bs;
    }
  }
}

template <int CB, int QT, int MODE>
cudaError_t set_smem_attr(size_t smem) {
  static size_t set = 0;  // cudaFuncSetAttribute only when the requirement grows
  if (smem <= set) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_match<CB, QT, MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) set = smem;
  return e;
}

template <int CB, int QT, int MODE>
cudaError_t launch_match_t(const CUtensorMap& map, const MatchArgs& a, const MatchGeom& g,
                           cudaStream_t st) {
  cudaError_t e = set_smem_attr<CB, QT, MODE>(g.smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(k_match<CB, QT, MODE>, dim3(g.grid), dim3(kNT), g.smem, st, map, a);
}

template <int MODE>
cudaError_t dispatch_match(int cb, uint32_t QT, const CUtensorMap& map, const MatchArgs& a,
                           const MatchGeom& g, cudaStream_t st) {
  if (MODE != 0) {
    return cb == 1   ? launch_match_t<1, 1, MODE>(map, a, g, st)
           : cb == 2 ? launch_match_t<2, 1, MODE>(map, a, g, st)
                     : launch_match_t<4, 1, MODE>(map, a, g, st);
  }
#define MOE_QT_CASE(q)                                                      \
  case q:                                                                   \
    return cb == 1   ? launch_match_t<1, q, 0>(map, a, g, st)               \
           : cb == 2 ? launch_match_t<2, q, 0>(map, a, g, st)               \
                     : launch_match_t<4, q, 0>(map, a, g, st);
  switch (QT) {
    MOE_QT_CASE(1)
    MOE_QT_CASE(2)
    MOE_QT_CASE(4)
    MOE_QT_CASE(8)
    MOE_QT_CASE(16)
    default:
      return cudaErrorInvalidValue;
  }
#undef MOE_QT_CASE
}

MatchArgs base_args(const DevColl& c, const DevProbes& pr, const MatchGeom& g) {
  MatchArgs a{};
  a.ibT = c.ibT;
  a.sqb = c.sqb;
  a.seq = c.seq;
  a.cap = c.cap;
  a.size = c.size;
  a.probes = pr.packed;
  a.ia = pr.ia;
  a.sqa = pr.sqa;
  a.Q = pr.Q;
  a.L = c.L;
  a.RB = c.RB;
  a.C = c.C;
  a.G = g.G;
  a.S = g.S;
  a.n_groups = g.n_groups;
  a.n_pt = g.n_pt;
  a.eps2 = screen_eps2(c.L);
  return a;
}

}  // namespace

float screen_eps2(uint32_t L) {
  // |d32 - d_ref| <= u * (6 + (L+1)/2) with u = 2^-24 (see DESIGN.md
  // "screen bound"); 1.5x safety margin plus an absolute floor.
  const double u = 1.0 / 16777216.0;
  const double eps = 1.5 * u * (6.0 + 0.5 * (L + 1.0)) + 1e-9;
  return (float)(2.0 * eps);
}

namespace {
template <int CB, int QT, int MODE>
int occ_blocks_t(size_t smem) {
  if (set_smem_attr<CB, QT, MODE>(smem) != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_match<CB, QT, MODE>, kNT, smem) !=
      cudaSuccess)
    return 0;
  return n;
}
int occ_blocks(int cb, uint32_t QT, int mode, size_t smem) {
#define MOE_OCC(q, md) \
  (cb == 1 ? occ_blocks_t<1, q, md>(smem) \
           : cb == 2 ? occ_blocks_t<2, q, md>(smem) : occ_blocks_t<4, q, md>(smem))
  if (mode == 1) return MOE_OCC(1, 1);
  switch (QT) {
    case 1: return MOE_OCC(1, 0);
    case 2: return MOE_OCC(2, 0);
    case 4: return MOE_OCC(4, 0);
    case 8: return MOE_OCC(8, 0);
    case 16: return MOE_OCC(16, 0);
  }
  return 0;
}
}  // namespace

// Launch geometry of the matcher: the layer-group depth G (rows per TMA box),
// pipeline depth S and resident blocks per SM are chosen together to maximize
//   (resident warps, capped at 16/SM) x (shared-memory bank efficiency of the
//   per-lane rotated row reads) / (TMA bytes wasted on out-of-range layers)
// subject to keeping >= ~32 KB of TMA traffic in flight per SM.
bool plan_match(const DevColl& c, int n_sm, int mode, uint32_t QT, MatchGeom* g) {
  static std::map<std::tuple<uint32_t, uint32_t, int, int, uint32_t>, MatchGeom> cache;
  const auto key = std::make_tuple(c.L, c.RB, c.cb, mode, QT);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *g = it->second;
    g->n_pt = (c.size + kNT - 1) / kNT;
    g->grid = (uint32_t)n_sm * g->blocks_per_sm;
    return true;
  }
  const size_t kMaxSmem = 227 * 1024;
  const uint32_t acc_bytes = c.cb == 1 ? 4 : 8;
  double best_score = -1.0;
  MatchGeom best;
  for (uint32_t S = 2; S <= 4; ++S) {
    for (uint32_t G = 1; G <= std::min<uint32_t>(c.L, 16); ++G) {
      const SmemLayout lay = smem_layout(c.L, c.RB, G, S, QT, mode, acc_bytes);
      if (lay.total > kMaxSmem) continue;
      const int blocks = occ_blocks(c.cb, QT, mode, lay.total);
      if (blocks < 1) continue;
      double wf = 0.0;  // bank-group wavefronts of one warp-wide 16-byte row read
      for (uint32_t cc = 0; cc < c.C; ++cc) {
        int cnt[8] = {0};
        for (uint32_t ln = 0; ln < 32; ++ln) {
          const uint32_t k = (cc + ln) % c.C;
          const uint64_t chunk = (uint64_t)ln * G * c.C + k;
          cnt[chunk % 8]++;
        }
        int m = 4;
        for (int b = 0; b < 8; ++b) m = std::max(m, cnt[b]);
        wf += m;
      }
      wf /= c.C;
      const uint32_t ng = (c.L + G - 1) / G;
      const double waste = (double)(ng * G) / c.L;
      const double warps = std::min(16.0, 4.0 * blocks) / 16.0;
      const double inflight = (double)(S - 1) * lay.stage_bytes * blocks;
      const double score = warps * (4.0 / wf) / waste * std::min(1.0, inflight / 32768.0) +
                           1e-3 * G + 1e-4 * S;
      if (score > best_score) {
        best_score = score;
        best.G = G;
        best.S = S;
        best.smem = lay.total;
        best.blocks_per_sm = (uint32_t)blocks;
      }
    }
  }
  if (best_score < 0) return false;
  best.QT = QT;
  best.n_groups = (c.L + best.G - 1) / best.G;
  cache[key] = best;
  best.n_pt = (c.size + kNT - 1) / kNT;
  best.grid = (uint32_t)n_sm * best.blocks_per_sm;
  *g = best;
  return true;
}

cudaError_t encode_tmap(const DevColl& c, uint32_t G, CUtensorMap* map) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[4] = {16, c.C, c.L, c.cap};
  const cuuint64_t strides[3] = {16, c.RB, (cuuint64_t)c.L * c.RB};
  const cuuint32_t box[4] = {16, c.C, G, (cuuint32_t)kNT};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, c.counts, dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_prep(const void* src, int src_bytes, uint64_t n, uint32_t L, uint32_t E,
                        uint32_t RB, int cb, uint8_t* dst, float* ia, double* sq, float* ibT,
                        uint64_t ib_cap, uint64_t ib_base, unsigned long long* max_count,
                        __half* nrm, uint32_t Kp, uint64_t* zmask, uint8_t* wide,
                        cudaStream_t st, MatchInit init) {
  if (n == 0) return cudaSuccess;
  const uint32_t threads = 256;
  // u8 -> u8 fast path (8-byte aligned fp16 rows need E % 4 == 0)
  if (src_bytes == 1 && cb == 1 && (E & 3) == 0 && E <= 256 &&
      (reinterpret_cast<uintptr_t>(src) & 3) == 0) {
    // warps per EAM: enough warps in flight for small batches
    uint32_t wpe = 1;
    while (wpe < 16 && n * wpe < 2048 && wpe * 8 < L) wpe <<= 1;
    // small blocks (4 warps, or one EAM's warps) spread evenly over the SMs
    const uint32_t pt = 32 * std::max<uint32_t>(4, wpe);
    const uint64_t wblocks = (n * wpe * 32 + pt - 1) / pt;
    return launch_pdl(E <= 128 ? k_prep_u8<1> : k_prep_u8<2>, dim3((unsigned)wblocks), dim3(pt),
                      0, st, static_cast<const uint8_t*>(src), n, E, L, RB, dst, ia, sq, ibT,
                      ib_cap, ib_base, nrm, Kp, zmask, wide, wpe, max_count, init);
  }
  const uint64_t rows = n * L;
  const uint64_t blocks = (rows * 32 + threads - 1) / threads;
  const uint64_t limit = cb == 1 ? 255ull : cb == 2 ? 65535ull : 0xffffffffull;
  if (max_count) {
    cudaError_t e = cudaMemsetAsync(max_count, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
  }
  if (zmask) {
    cudaError_t e = cudaMemsetAsync(zmask, 0, n * sizeof(uint64_t), st);
    if (e != cudaSuccess) return e;
  }
  if (wide) {
    cudaError_t e = cudaMemsetAsync(wide, 0, n, st);
    if (e != cudaSuccess) return e;
  }
#define MOE_PREP(S)                                                                          \
  return launch_pdl(k_prep<S>, dim3((unsigned)blocks), dim3(threads), 0, st, src, rows, E, L, RB, \
                    cb, dst, ia, sq, ibT, ib_cap, ib_base, max_count, limit, nrm, Kp, zmask,     \
                    wide, init)
  switch (src_bytes) {
    case 8: MOE_PREP(8);
    case 4: MOE_PREP(4);
    case 2: MOE_PREP(2);
    case 1: MOE_PREP(1);
    default: return cudaErrorInvalidValue;
  }
#undef MOE_PREP
}

cudaError_t launch_screen(const CUtensorMap& map, const DevColl& c, const DevProbes& pr,
                          const MatchGeom& g, const MatchWork& w, cudaStream_t st) {
  if (c.size == 0 || pr.Q == 0) return cudaSuccess;
  MatchArgs a = base_args(c, pr, g);
  a.T = w.T;
  a.bcnt = w.bcnt;
  a.bucket = w.bucket;
  a.bcap = w.bcap;
  return dispatch_match<0>(c.cb, g.QT, map, a, g, st);
}

cudaError_t launch_refine(const DevColl& c, const DevProbes& pr, const MatchWork& w,
                          moe_match* out, const int* halt, int* halt_set, uint32_t halt_value,
                          cudaStream_t st) {
  if (pr.Q == 0) return cudaSuccess;
  RefineArgs r{};
  r.counts = c.counts;
  r.sqb = c.sqb;
  r.seq = c.seq;
  r.size = c.size;
  r.probes = pr.packed;
  r.sqa = pr.sqa;
  r.Q = pr.Q;
  r.L = c.L;
  r.C = c.C;
  r.RB = c.RB;
  r.eps2 = w.eps2 > 0.f ? w.eps2 : screen_eps2(c.L);
  r.T = w.T;
  r.bcnt = w.bcnt;
  r.bucket = w.bucket;
  r.bcap = w.bcap;
  r.over_list = w.over_list;
  r.over_n = w.over_n;
  r.wide = pr.wide;
  r.out = out;
  r.halt = halt;
  r.halt_set = halt_set;
  r.halt_value = halt_value;
  r.index_base = c.index_base;
  const uint32_t blocks = (pr.Q + kRefineWarps - 1) / kRefineWarps;
  return c.cb == 1   ? launch_pdl(k_refine<1>, dim3(blocks), dim3(kRefineWarps * 32), 0, st, r)
         : c.cb == 2 ? launch_pdl(k_refine<2>, dim3(blocks), dim3(kRefineWarps * 32), 0, st, r)
                     : launch_pdl(k_refine<4>, dim3(blocks), dim3(kRefineWarps * 32), 0, st, r);
}

cudaError_t launch_exact(const CUtensorMap& map, const DevColl& c, const DevProbes& pr,
                         const MatchGeom& g, const MatchWork& w, const uint32_t* qlist,
                         uint32_t qlist_n, const uint32_t* T, moe_match* out, cudaStream_t st,
                         const uint32_t* nq_dev) {
  if (qlist_n == 0) return cudaSuccess;
  for (uint32_t off = 0; off < qlist_n; off += w.part_chunk) {
    const uint32_t n = std::min(w.part_chunk, qlist_n - off);
    MatchArgs a = base_args(c, pr, g);
    a.eps2 = std::max(a.eps2, w.eps2);  // band of whichever screen produced T
    a.qlist = qlist + off;
    a.nq_list = n;
    a.nq_dev = nq_dev;
    a.q_off = off;
    a.Tfinal = T;
    a.partials = w.partials;
    cudaError_t e = dispatch_match<1>(c.cb, 1, map, a, g, st);
    if (e != cudaSuccess) return e;
    const uint32_t threads = 256;
    const uint32_t blocks = (uint32_t)(((uint64_t)n * 32 + threads - 1) / threads);
    e = launch_pdl(k_merge_partials, dim3(blocks), dim3(threads), 0, st,
                   (const moe_match*)w.partials, (uint32_t)g.grid, n, (uint32_t)g.n_pt,
                   qlist + off, out, (uint64_t)c.index_base, nq_dev, off);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

uint32_t exact_warp_blocks(int n_sm) { return (uint32_t)n_sm * 2; }

cudaError_t launch_exact_warp(const DevColl& c, const DevProbes& pr, const uint32_t* qlist,
                              uint32_t qlist_n, moe_match* out, moe_match* parts,
                              uint32_t chunk, int n_sm, cudaStream_t st, const uint32_t* nq_dev) {
  const uint32_t nb = exact_warp_blocks(n_sm);
  for (uint32_t off = 0; off < qlist_n; off += chunk) {
    const uint32_t n = std::min(chunk, qlist_n - off);
    auto kern = c.cb == 1 ? k_exact_warp<1> : c.cb == 2 ? k_exact_warp<2> : k_exact_warp<4>;
    cudaError_t e = launch_pdl(kern, dim3(nb, n), dim3(256), 0, st, (const uint8_t*)c.counts,
                               (const double*)c.sqb, (const uint64_t*)c.seq, c.size, c.L, c.C,
                               c.RB, (const uint8_t*)pr.packed, (const double*)pr.sqa,
                               qlist + off, n, nq_dev, off, parts);
    if (e != cudaSuccess) return e;
    e = launch_pdl(k_merge_blocks, dim3((n + 255) / 256), dim3(256), 0, st,
                   (const moe_match*)parts, nb, qlist + off, n, nq_dev, off, out,
                   (uint64_t)c.index_base);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_merge(const moe_match* parts, uint64_t n_parts, uint64_t n, moe_match* out,
                         cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_merge<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(parts, n_parts, n, out);
  return cudaGetLastError();
}

cudaError_t launch_pair_distance(const uint8_t* a, const double* sqa, const uint8_t* b,
                                 const double* sqb, uint32_t L, uint32_t C, uint32_t RB, int cb,
                                 double* out, cudaStream_t st) {
  if (cb == 1)
    k_pair_distance<1><<<1, 32, 0, st>>>(a, sqa, b, sqb, L, C, RB, out);
  else if (cb == 2)
    k_pair_distance<2><<<1, 32, 0, st>>>(a, sqa, b, sqb, L, C, RB, out);
  else
    k_pair_distance<4><<<1, 32, 0, st>>>(a, sqa, b, sqb, L, C, RB, out);
  return cudaGetLastError();
}

cudaError_t launch_replace(const DevColl& c, const DevProbes& staged, uint32_t i,
                           const moe_match* victim, uint64_t seq_value, const int* halt,
                           cudaStream_t st) {
  k_replace<<<1, 256, 0, st>>>(c.counts, c.ibT, c.sqb, c.seq, c.cap, c.L, c.RB, staged.packed,
                               staged.ia, staged.sqa, i, victim, c.size, seq_value, halt,
                               c.index_base, c.nrm, staged.nrm, c.Kp, c.zmask, staged.zmask);
  return cudaGetLastError();
}

size_t replay_block_smem(const DevColl& c) {
  const size_t P4 = (c.size + 3) / 4;
  const size_t LR = (size_t)c.L * c.RB;
  return ((P4 * 8 + 15) & ~(size_t)15) + LR + kRW * LR + kRW * 64 * 8 + 2 * P4 * 16 +
         2 * (size_t)4 * ((kReplayBlockMax + 3) & ~3u);
}

cudaError_t launch_replay_block(const DevColl& c, const DevProbes& staged, uint32_t first,
                                uint32_t nb, const float* dc, uint32_t ldc, const float* dx,
                                uint32_t ldx, float eps2, int* occ, uint64_t seq0,
                                moe_match* vic, cudaStream_t st, unsigned long long* prof) {
  if (nb == 0) return cudaSuccess;
  if (c.L > 64 || c.size > kReplayMaxP || nb > kReplayBlockMax || ldx > kReplayBlockMax ||
      (ldc & 3) ||
      (uint64_t)c.L * c.RB > 16ull * kXsPer * kReplayThreads)
    return cudaErrorInvalidValue;
  ReplayArgs a;
  a.counts = c.counts;
  a.sqb = c.sqb;
  a.seq = c.seq;
  a.P = c.size;
  a.L = c.L;
  a.C = c.C;
  a.RB = c.RB;
  a.index_base = c.index_base;
  const uint64_t LR = (uint64_t)c.L * c.RB;
  a.xp = staged.packed + (uint64_t)first * LR;
  a.xsq = staged.sqa + (uint64_t)first * c.L;
  a.nb = nb;
  a.dc = dc;
  a.dx = dx;
  a.ldc = ldc;
  a.ldx = ldx;
  a.eps2 = eps2;
  a.occ = occ;
  a.seq0 = seq0;
  a.vic = vic;
  a.prof = prof;
  const size_t smem = replay_block_smem(c);
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  static size_t set = 0;
  if (smem > set) {
    cudaError_t e1 = cudaFuncSetAttribute(k_replay_block<1>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e1 == cudaSuccess)
      e1 = cudaFuncSetAttribute(k_replay_block<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem);
    if (e1 == cudaSuccess)
      e1 = cudaFuncSetAttribute(k_replay_block<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem);
    if (e1 != cudaSuccess) return e1;
    set = smem;
  }
  if (c.cb == 1)
    k_replay_block<1><<<1, kReplayThreads, smem, st>>>(a);
  else if (c.cb == 2)
    k_replay_block<2><<<1, kReplayThreads, smem, st>>>(a);
  else
    k_replay_block<4><<<1, kReplayThreads, smem, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_apply_block<<<nb, 256, 0, st>>>(c.counts, c.ibT, c.sqb, c.seq, c.cap, c.L, c.RB,
                                    a.xp, staged.ia + (uint64_t)first * c.L, a.xsq, vic, occ,
                                    seq0, c.index_base, c.nrm,
                                    staged.nrm ? staged.nrm + (uint64_t)first * c.Kp : nullptr,
                                    c.Kp, c.zmask, staged.zmask ? staged.zmask + first : nullptr);
  return cudaGetLastError();
}

cudaError_t launch_append_staged(const DevColl& c, const DevProbes& staged, uint32_t first,
                                 uint32_t n, uint64_t base, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_append_staged<<<256, 256, 0, st>>>(c.counts, c.ibT, c.sqb, c.cap, c.L, c.RB, staged.packed,
                                       staged.ia, staged.sqa, first, n, base, c.nrm, staged.nrm,
                                       c.Kp, c.zmask, staged.zmask);
  return cudaGetLastError();
}

cudaError_t launch_widen(const uint8_t* src, uint8_t* dst, uint64_t rows, uint32_t RB_old,
                         uint32_t RB_new, int cb_old, int cb_new, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  k_widen<<<1024, 256, 0, st>>>(src, dst, rows, RB_old, RB_new, cb_old, cb_new);
  return cudaGetLastError();
}

cudaError_t launch_decide(const unsigned long long* agg, uint32_t L, uint32_t E, uint32_t cur,
                          int filter, int do_prefetch, const unsigned long long* req,
                          const moe_slot_view* slots, uint64_t n_slots, moe_candidate* out,
                          uint32_t* n_out, long long* victim, double* slot_pri,
                          cudaStream_t st) {
  uint32_t n = do_prefetch && cur + 1 < L ? (L - cur - 1) * E : 1;
  uint32_t np = 2;
  while (np < n) np <<= 1;
  const size_t smem = (size_t)np * 12 + (size_t)L * 16 + 16;
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  static size_t set = 0;
  if (smem > set) {
    cudaError_t e =
        cudaFuncSetAttribute(k_decide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set = smem;
  }
  k_decide<<<1, 1024, smem, st>>>(agg, L, E, cur, filter, do_prefetch && cur + 1 < L, req, slots,
                                  n_slots, out, n_out, victim, slot_pri, np);
  return cudaGetLastError();
}

cudaError_t launch_window_list(const DevColl& c, const double* dist,
                               const unsigned long long* dmin, double window, WinEntry* wl,
                               uint32_t* wl_n, cudaStream_t st) {
  if (c.size == 0) return cudaSuccess;
  k_window_list<<<(c.size + 255) / 256, 256, 0, st>>>(dist, dmin, window, c.seq, c.size, wl, wl_n);
  return cudaGetLastError();
}

cudaError_t launch_exact_rows(const DevColl& c, const DevProbes& pr, uint32_t q0, uint32_t l0,
                              uint32_t l1, double* r, double* dist, unsigned long long* dmin,
                              int n_sm, cudaStream_t st) {
  if (c.size == 0) return cudaSuccess;
  const uint64_t LR = (uint64_t)c.L * c.RB;
  const uint64_t n = (uint64_t)c.size * (l1 - l0);
  if (n) {
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)n_sm * 16);
    auto kern = c.cb == 1 ? k_rowsim<1> : c.cb == 2 ? k_rowsim<2> : k_rowsim<4>;
    kern<<<grid, 256, 0, st>>>(c.counts, c.sqb, c.size, c.L, c.C, c.RB, pr.packed + q0 * LR,
                               pr.sqa + (uint64_t)q0 * c.L, l0, l1, r);
  }
  k_rowsum<<<(c.size + 255) / 256, 256, 0, st>>>(r, c.size, c.L, dist, dmin);
  return cudaGetLastError();
}

cudaError_t launch_member_agg(const DevColl& c, const double* dist,
                              const unsigned long long* dmin, double window, uint32_t cur,
                              uint32_t* mem, uint32_t* n_mem, unsigned long long* agg, int n_sm,
                              cudaStream_t st, bool n_mem_zeroed) {
  if (c.size == 0) return cudaSuccess;
  if (!n_mem_zeroed) {
    cudaError_t e = cudaMemsetAsync(n_mem, 0, 4, st);
    if (e != cudaSuccess) return e;
  }
  launch_pdl(k_members, dim3(std::min<uint32_t>((c.size + 255) / 256, (uint32_t)n_sm * 4)), dim3(256), 0, st, 
      dist, dmin, window, c.size, mem, n_mem);
  if (cur + 1 >= c.L) return cudaGetLastError();
  const uint32_t words = (c.L - cur - 1) * (c.RB / 4);
  const uint32_t bx = (words + 255) / 256;
  const uint32_t by = std::max<uint32_t>(1, std::min<uint32_t>((uint32_t)n_sm * 8 / bx + 1,
                                                               (c.size + 31) / 32));
  const uint32_t chunk = (c.size + by - 1) / by;
  dim3 grid(bx, by);
  auto kern = c.cb == 1 ? k_member_agg<1> : c.cb == 2 ? k_member_agg<2> : k_member_agg<4>;
  launch_pdl(kern, dim3(grid), dim3(256), 0, st, c.counts, c.L, c.E, c.RB, cur, mem, n_mem, chunk,
             agg);
  return cudaGetLastError();
}

}  // namespace moe
