// cluster.cu -- kernels of the clustering EAMC construction
// (moe_eamc_build_clustered; north-star item 3: "pairwise distance plus
// clustering step that picks P representatives from N traces").
//
// The reference constructs its EAMC by nearest-replacement inserts
// (eam.cpp:152-178) and defers clustering, so this
// mode has no reference to be pinned to; it starts FROM the reference
// construction and improves it by k-medoids-style iterations, each of which
// keeps representatives as real request EAMs and never increases the
// objective sum_i min_p d(trace_i, rep_p):
//   assign   every trace to its nearest representative (the exact batch
//            matcher: tensor-core screen + exact refine, (d, seq) argmin)
//   centroid per cluster, the u64 sum of its members' counts
//   propose  per cluster, the member closest to the centroid (fp64 cosine
//            per layer on exact integer dots; ties to the lowest trace index)
//   accept   a proposal replaces the representative only when the cluster's
//            total exact distance to it is strictly lower (fixed-point u64
//            sums of the exact distances: order-independent, deterministic)
#include "common.cuh"
#include "kernels.cuh"

namespace moe {

namespace {

constexpr double kFix = 1099511627776.0;  // 2^40: distances in [0, 1] as u64 fixed point

template <int CB>
__device__ __forceinline__ uint32_t count_at(const uint8_t* row, uint32_t e) {
  if (CB == 1) return row[e];
  if (CB == 2) return reinterpret_cast<const uint16_t*>(row)[e];
  return reinterpret_cast<const uint32_t*>(row)[e];
}

// Warp per trace: its counts added into its cluster's centroid.
template <int CB>
__global__ void k_centroid_add(const uint8_t* packed, uint64_t n, uint32_t L, uint32_t E,
                               uint32_t RB, const moe_match* m, uint64_t base,
                               unsigned long long* cent) {
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (w >= n) return;
  const uint64_t slot = m[w].index - base;
  const uint8_t* tr = packed + w * (uint64_t)L * RB;
  unsigned long long* cr = cent + slot * (uint64_t)L * E;
  for (uint32_t i = lane; i < L * E; i += 32) {
    const uint32_t l = i / E, e = i - l * E;
    const uint32_t c = count_at<CB>(tr + (uint64_t)l * RB, e);
    if (c) atomicAdd(&cr[i], (unsigned long long)c);
  }
}

// Warp per trace: fp64 distance to its cluster's centroid (row_similarity
// conventions: both rows zero -> 1, one zero -> 0), cluster minimum.
template <int CB>
__global__ void k_centroid_dist(const uint8_t* packed, uint64_t n, uint32_t L, uint32_t E,
                                uint32_t RB, const moe_match* m, uint64_t base,
                                const unsigned long long* cent, double* dc,
                                unsigned long long* cmin) {
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (w >= n) return;
  const uint64_t slot = m[w].index - base;
  const uint8_t* tr = packed + w * (uint64_t)L * RB;
  const unsigned long long* cr = cent + slot * (uint64_t)L * E;
  double sim = 0.0;
  for (uint32_t l = 0; l < L; ++l) {
    unsigned long long dot = 0, na = 0;
    double nb = 0.0;
    for (uint32_t e = lane; e < E; e += 32) {
      const unsigned long long a = count_at<CB>(tr + (uint64_t)l * RB, e);
      const unsigned long long b = cr[(uint64_t)l * E + e];
      dot += a * b;
      na += a * a;
      nb += (double)b * (double)b;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dot += __shfl_xor_sync(0xffffffffu, dot, o);
      na += __shfl_xor_sync(0xffffffffu, na, o);
      nb += __shfl_xor_sync(0xffffffffu, nb, o);
    }
    double r;
    if (na == 0 && nb == 0.0) r = 1.0;
    else if (na == 0 || nb == 0.0) r = 0.0;
    else r = (double)dot / (sqrt((double)na) * sqrt(nb));
    sim += r;
  }
  double d = 1.0 - sim / (double)L;
  d = d < 0.0 ? 0.0 : d > 1.0 ? 1.0 : d;
  if (lane == 0) {
    dc[w] = d;
    atomicMin(&cmin[slot], (unsigned long long)__double_as_longlong(d));
  }
}

// Thread per trace: the lowest trace index attaining its cluster's minimum.
__global__ void k_centroid_pick(uint64_t n, const moe_match* m, uint64_t base, const double* dc,
                                const unsigned long long* cmin, unsigned long long* cidx) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t slot = m[i].index - base;
  if ((unsigned long long)__double_as_longlong(dc[i]) == cmin[slot]) atomicMin(&cidx[slot], i);
}

// Warp per trace: fixed-point cluster totals of the current representative's
// exact distance (from the matcher) and of the proposal's (exact, reference
// operation order).
template <int CB>
__global__ void k_cluster_totals(const uint8_t* packed, const double* sq, uint64_t n, uint32_t L,
                                 uint32_t C, uint32_t RB, const moe_match* m, uint64_t base,
                                 const unsigned long long* cidx, unsigned long long* tot_cur,
                                 unsigned long long* tot_cand) {
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (w >= n) return;
  const uint64_t slot = m[w].index - base;
  const uint64_t cand = cidx[slot];
  const uint64_t LR = (uint64_t)L * RB;
  const double d = warp_exact_distance<CB>(packed + w * LR, sq + w * L, packed + cand * LR,
                                               sq + cand * L, L, C, RB);
  if (lane == 0) {
    atomicAdd(&tot_cur[slot], (unsigned long long)__double2ull_rn(m[w].distance * kFix));
    atomicAdd(&tot_cand[slot], (unsigned long long)__double2ull_rn(d * kFix));
  }
}

}  // namespace

cudaError_t launch_cluster_step(const uint8_t* packed, const double* sq, uint64_t n, uint32_t L,
                                uint32_t E, uint32_t RB, int cb, const moe_match* m,
                                uint64_t base, uint64_t P, unsigned long long* cent, double* dc,
                                unsigned long long* cmin, unsigned long long* cidx,
                                unsigned long long* tot_cur, unsigned long long* tot_cand,
                                cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(cent, 0, P * (uint64_t)L * E * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(cmin, 0xff, P * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(cidx, 0xff, P * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(tot_cur, 0, P * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(tot_cand, 0, P * 8, st);
  if (e != cudaSuccess) return e;
  const unsigned wb = (unsigned)((n * 32 + 255) / 256), tb = (unsigned)((n + 255) / 256);
  const uint32_t C = RB / 16;
#define MOE_CLUSTER(CB)                                                                          \
  k_centroid_add<CB><<<wb, 256, 0, st>>>(packed, n, L, E, RB, m, base, cent);                    \
  k_centroid_dist<CB><<<wb, 256, 0, st>>>(packed, n, L, E, RB, m, base, cent, dc, cmin);         \
  k_centroid_pick<<<tb, 256, 0, st>>>(n, m, base, dc, cmin, cidx);                               \
  k_cluster_totals<CB><<<wb, 256, 0, st>>>(packed, sq, n, L, C, RB, m, base, cidx, tot_cur,      \
                                           tot_cand);
  if (cb == 1) {
    MOE_CLUSTER(1)
  } else if (cb == 2) {
    MOE_CLUSTER(2)
  } else {
    MOE_CLUSTER(4)
  }
#undef MOE_CLUSTER
  return cudaGetLastError();
}

}  // namespace moe
