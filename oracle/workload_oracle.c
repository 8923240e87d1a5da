/*
 * workload_oracle.c -- CPU ORACLE: restatement of the reference synthetic
 * routing-trace generator (proj/core/src/workload.cpp:64-197).
 *
 * TEST INFRASTRUCTURE ONLY (see eamc_oracle.c header).  It produces the
 * "F2" workload family (request-level EAMs, as moesim_main.cpp:192-201
 * builds them) and the "F3" raw router traces (the per-token top-k picks
 * that workload.cpp:166-181 aggregates into RoutingEvents), so the tracer's
 * input and the matcher's realistic inputs are bit-identical to what the
 * reference library generates.  Pinned against oracle/_ref in tests/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct orc_rng { uint64_t state; } orc_rng;
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_next_double(orc_rng* r);
uint64_t orc_rng_bounded(orc_rng* r, uint64_t n);
int orc_rng_bernoulli(orc_rng* r, double p);
orc_rng orc_rng_stream(uint64_t seed, uint64_t tag);

/* WeightedSampler: workload.cpp:15-34 */
typedef struct { double* cdf; uint32_t n; } orc_sampler;
static orc_sampler sampler_make(const double* w, uint32_t n) {
  orc_sampler s = {(double*)malloc(n * sizeof(double)), n};
  double acc = 0.0;
  for (uint32_t i = 0; i < n; ++i) {
    acc += w[i];
    s.cdf[i] = acc;
  }
  for (uint32_t i = 0; i < n; ++i) s.cdf[i] /= acc;
  s.cdf[n - 1] = 1.0;
  return s;
}
static uint32_t sampler_sample(const orc_sampler* s, orc_rng* r) {
  const double u = orc_rng_next_double(r);
  /* std::upper_bound: first element > u */
  uint32_t lo = 0, hi = s->n;
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (s->cdf[mid] > u) hi = mid; else lo = mid + 1;
  }
  return lo < s->n - 1 ? lo : s->n - 1;
}

/* random_permutation: workload.cpp:36-43 */
static void random_permutation(uint32_t n, orc_rng* r, uint32_t* p) {
  for (uint32_t i = 0; i < n; ++i) p[i] = i;
  for (uint32_t i = n; i > 1; --i) {
    const uint32_t j = (uint32_t)orc_rng_bounded(r, i);
    const uint32_t t = p[i - 1];
    p[i - 1] = p[j];
    p[j] = t;
  }
}

static int contains(const uint32_t* v, uint32_t n, uint32_t x) {
  for (uint32_t i = 0; i < n; ++i)
    if (v[i] == x) return 1;
  return 0;
}
static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y);
}

/* draw_zipf_topk: workload.cpp:98-117 */
static void draw_zipf_topk(const orc_sampler* s, const uint32_t* perm, uint32_t E, uint32_t k,
                           orc_rng* r, uint32_t* out) {
  uint32_t n = 0;
  int attempts = 0;
  while (n < k) {
    const uint32_t rank = sampler_sample(s, r);
    const uint32_t expert = perm[rank];
    if (!contains(out, n, expert)) {
      out[n++] = expert;
    } else if (++attempts > 64) {
      for (uint32_t q = 0; q < E && n < k; ++q)
        if (!contains(out, n, perm[q])) out[n++] = perm[q];
    }
  }
}

/* WorkloadSpec (workload.hpp:33-45) with DiscreteDist pmfs as arrays. */
typedef struct orc_workload {
  uint32_t L, E, top_k;
  uint32_t n_groups;
  double group_fidelity;
  double reuse_skew;
  const uint32_t* prompt_vals; const double* prompt_w; uint32_t prompt_n;
  const uint32_t* decode_vals; const double* decode_w; uint32_t decode_n;
  uint32_t batch_size;
  uint64_t seed;
} orc_workload;

/* sample_dist: workload.cpp:68-74 (builds a sampler, consumes one draw) */
static uint32_t sample_dist(const uint32_t* vals, const double* w, uint32_t n, orc_rng* r) {
  orc_sampler s = sampler_make(w, n);
  const uint32_t v = vals[sampler_sample(&s, r)];
  free(s.cdf);
  return v;
}

/* build_groups: workload.cpp:79-96 -> groups[g][l][k] */
static uint32_t* build_groups(const orc_workload* w) {
  orc_rng r = orc_rng_stream(w->seed, 0xFFFFFFFFFFFF0001ull);
  uint32_t* g = (uint32_t*)malloc((size_t)w->n_groups * w->L * w->top_k * sizeof(uint32_t));
  for (uint32_t gi = 0; gi < w->n_groups; ++gi)
    for (uint32_t l = 0; l < w->L; ++l) {
      uint32_t* d = g + ((size_t)gi * w->L + l) * w->top_k;
      uint32_t n = 0;
      while (n < w->top_k) {
        const uint32_t cand = (uint32_t)orc_rng_bounded(&r, w->E);
        if (!contains(d, n, cand)) d[n++] = cand;
      }
      qsort(d, n, sizeof(uint32_t), cmp_u32);
    }
  return g;
}

/* generate_trace: workload.cpp:121-190.
 *
 * Emits, for the request, (a) per-iteration L x E counts into `iter_counts`
 * ([n_iter][L][E], may be NULL) and (b) the per-token top-k picks into
 * `picks` ([n_tokens][L][k], may be NULL), token order = iteration, then
 * sequence s, then token t (the order workload.cpp:166-181 visits them).
 * Returns the number of iterations; *n_tokens_out gets the token count.
 * Call once with NULL buffers to size them (max_iters/max_tokens unused). */
uint32_t orc_generate_trace(const orc_workload* w, uint64_t request_index, uint64_t* iter_counts,
                            uint32_t* picks, uint64_t* n_tokens_out, uint64_t* prompt_tokens_out) {
  const uint32_t L = w->L, E = w->E, k = w->top_k;
  uint32_t* groups = build_groups(w);
  orc_rng r = orc_rng_stream(w->seed, request_index);

  double* zipf = (double*)malloc(E * sizeof(double));
  for (uint32_t q = 0; q < E; ++q) zipf[q] = pow((double)(q + 1), -w->reuse_skew);
  orc_sampler zs = sampler_make(zipf, E);

  uint32_t* perm = (uint32_t*)malloc((size_t)L * E * sizeof(uint32_t));
  for (uint32_t l = 0; l < L; ++l) random_permutation(E, &r, perm + (size_t)l * E);

  double* gw = (double*)malloc(w->n_groups * sizeof(double));
  for (uint32_t g = 0; g < w->n_groups; ++g) gw[g] = pow((double)(g + 1), -w->reuse_skew);
  orc_sampler gs = sampler_make(gw, w->n_groups);

  uint32_t* seq_group = (uint32_t*)malloc(w->batch_size * sizeof(uint32_t));
  for (uint32_t s = 0; s < w->batch_size; ++s) seq_group[s] = sampler_sample(&gs, &r);

  const uint32_t prompt_len = sample_dist(w->prompt_vals, w->prompt_w, w->prompt_n, &r);
  const uint32_t decode_len = sample_dist(w->decode_vals, w->decode_w, w->decode_n, &r);
  const uint32_t n_iter = 1 + decode_len;
  const uint64_t n_tokens = (uint64_t)w->batch_size * prompt_len + (uint64_t)w->batch_size * decode_len;
  if (n_tokens_out) *n_tokens_out = n_tokens;
  if (prompt_tokens_out) *prompt_tokens_out = (uint64_t)prompt_len * w->batch_size;

  if (iter_counts || picks) {
    uint32_t* pk = (uint32_t*)malloc(k * sizeof(uint32_t));
    uint64_t tok_base = 0;
    for (uint32_t it = 0; it < n_iter; ++it) {
      const uint32_t tps = it == 0 ? prompt_len : 1;
      for (uint32_t l = 0; l < L; ++l) {
        uint64_t* c = iter_counts ? iter_counts + ((uint64_t)it * L + l) * E : NULL;
        if (c) memset(c, 0, E * sizeof(uint64_t));
        for (uint32_t s = 0; s < w->batch_size; ++s)
          for (uint32_t t = 0; t < tps; ++t) {
            const uint64_t tok = tok_base + (uint64_t)s * tps + t;
            const uint32_t* src;
            if (orc_rng_bernoulli(&r, w->group_fidelity)) {
              src = groups + ((size_t)seq_group[s] * L + l) * k;
            } else {
              draw_zipf_topk(&zs, perm + (size_t)l * E, E, k, &r, pk);
              src = pk;
            }
            for (uint32_t j = 0; j < k; ++j) {
              if (c) c[src[j]] += 1;
              if (picks) picks[(tok * L + l) * k + j] = src[j];
            }
          }
      }
      tok_base += (uint64_t)w->batch_size * tps;
    }
    free(pk);
  }
  free(seq_group);
  free(gs.cdf);
  free(gw);
  free(perm);
  free(zs.cdf);
  free(zipf);
  free(groups);
  return n_iter;
}

/* request_level_eam: proj/tools/moesim_main.cpp:192-201 (prefill =
 * iteration 0, decode = iterations 1..end).  phase: 0 prefill, 1 decode.
 * Returns the number of iterations folded in. */
uint32_t orc_request_eam(const orc_workload* w, uint64_t request_index, int phase, uint64_t* out) {
  uint64_t nt = 0, pt = 0;
  const uint32_t n_iter = orc_generate_trace(w, request_index, NULL, NULL, &nt, &pt);
  uint64_t* it = (uint64_t*)malloc((size_t)n_iter * w->L * w->E * sizeof(uint64_t));
  orc_generate_trace(w, request_index, it, NULL, &nt, &pt);
  const uint64_t cells = (uint64_t)w->L * w->E;
  memset(out, 0, cells * sizeof(uint64_t));
  const uint32_t begin = phase == 0 ? 0 : 1;
  const uint32_t end = phase == 0 ? 1 : n_iter;
  for (uint32_t i = begin; i < end && i < n_iter; ++i)
    for (uint64_t c = 0; c < cells; ++c) out[c] += it[i * cells + c];
  free(it);
  return end > begin ? end - begin : 0;
}

/* Iteration-level EAM of iteration `iteration` truncated after layer
 * `layer` (rows > layer zero), as the engine's cur_iter_eam_ looks when
 * prefetch_priorities is called for `layer` (engine.cpp:546, :587, :660). */
int orc_iteration_probe(const orc_workload* w, uint64_t request_index, uint32_t iteration,
                        uint32_t layer, uint64_t* out) {
  uint64_t nt = 0, pt = 0;
  const uint32_t n_iter = orc_generate_trace(w, request_index, NULL, NULL, &nt, &pt);
  if (iteration >= n_iter || layer >= w->L) return -1;
  uint64_t* it = (uint64_t*)malloc((size_t)n_iter * w->L * w->E * sizeof(uint64_t));
  orc_generate_trace(w, request_index, it, NULL, &nt, &pt);
  const uint64_t cells = (uint64_t)w->L * w->E;
  for (uint64_t c = 0; c < cells; ++c) out[c] = (c / w->E) <= layer ? it[iteration * cells + c] : 0;
  free(it);
  return 0;
}
