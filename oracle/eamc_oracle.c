/*
 * eamc_oracle.c -- CPU ORACLE for the EAM/EAMC decision path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is a plain-C restatement of the
 * reference algorithm (MoE-Infinity / moesim, /root/reference/proj) used as
 * the parity checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg.  The product (paper_2401_14361_b200/) never links,
 * loads or calls it.
 *
 * Parity pinning: every function below is checked in tests/ against
 *   (1) golden vectors produced by the real reference library compiled from
 *       /root/reference sources (oracle/_ref, see oracle/Makefile and
 *       oracle/make_golden.py), committed under tests/golden/, and
 *   (2) the live oracle/_ref library when it is present.
 *
 * Arithmetic follows the reference literally: fp64 accumulation of
 * integer-valued operands in element order, no FMA contraction (build with
 * -ffp-contract=off), sqrt/div in IEEE double.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng */
/* splitmix64 stream: proj/core/include/moesim/rng.hpp:19-24 */
typedef struct orc_rng { uint64_t state; } orc_rng;

uint64_t orc_rng_next_u64(orc_rng* r) {
  uint64_t z = (r->state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
/* rng.hpp:27 */
double orc_rng_next_double(orc_rng* r) {
  return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53;
}
/* rng.hpp:30-36 (unbiased rejection) */
uint64_t orc_rng_bounded(orc_rng* r, uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const uint64_t x = orc_rng_next_u64(r);
    if (x >= threshold) return x % n;
  }
}
/* rng.hpp:38 */
int orc_rng_bernoulli(orc_rng* r, double p) { return orc_rng_next_double(r) < p; }
/* rng.hpp:42-45 */
orc_rng orc_rng_stream(uint64_t seed, uint64_t tag) {
  orc_rng mix = {seed ^ (0xA0761D6478BD642Full + tag * 0xE7037ED1A0B428DBull)};
  orc_rng out = {orc_rng_next_u64(&mix)};
  return out;
}

/* --------------------------------------------------------- input families */
/* F1 "bench family": proj/core/src/bench.cpp:44-54 (random_request_eam),
 * drawn from Rng::stream(seed, 0x6265636E) in bench_match order
 * (bench.cpp:60-66: P collection entries first, then the probes).  Fills
 * n consecutive EAMs, continuing the stream `r`. */
void orc_bench_family_next(orc_rng* r, uint32_t L, uint32_t E, uint64_t n, uint64_t* out) {
  const uint32_t active = E < 4 ? E : 4;
  const uint64_t cells = (uint64_t)L * E;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t* c = out + i * cells;
    memset(c, 0, cells * sizeof(uint64_t));
    for (uint32_t l = 0; l < L; ++l) {
      for (uint32_t k = 0; k < active; ++k) {
        const uint32_t e = (uint32_t)orc_rng_bounded(r, E);
        c[(uint64_t)l * E + e] = orc_rng_bounded(r, 32) + 1; /* Eam::set: last write wins */
      }
    }
  }
}
void orc_bench_family(uint64_t seed, uint32_t L, uint32_t E, uint64_t n, uint64_t* out) {
  orc_rng r = orc_rng_stream(seed, 0x6265636Eull);
  orc_bench_family_next(&r, L, E, n, out);
}

/* "random_eam" test family: proj/tests/test_eam.cpp:58-66 and
 * acceptance_main.cpp:63-69 (Bernoulli(0.4) cells, counts U[1,16]). */
void orc_random_eam(orc_rng* r, uint32_t L, uint32_t E, uint64_t* out) {
  for (uint32_t l = 0; l < L; ++l)
    for (uint32_t e = 0; e < E; ++e) {
      out[(uint64_t)l * E + e] = 0;
      if (orc_rng_bernoulli(r, 0.4)) out[(uint64_t)l * E + e] = orc_rng_bounded(r, 16) + 1;
    }
}

/* --------------------------------------------------------------- distance */
/* row_similarity: proj/core/src/eam.cpp:75-87 */
static double orc_row_similarity(const uint64_t* a, const uint64_t* b, uint32_t E) {
  double dot = 0.0, na = 0.0, nb = 0.0;
  for (uint32_t i = 0; i < E; ++i) {
    const double x = (double)a[i];
    const double y = (double)b[i];
    dot += x * y;
    na += x * x;
    nb += y * y;
  }
  if (na == 0.0 && nb == 0.0) return 1.0;
  if (na == 0.0 || nb == 0.0) return 0.0;
  return dot / (sqrt(na) * sqrt(nb));
}

/* eam_distance: proj/core/src/eam.cpp:91-104 */
double orc_eam_distance(uint32_t L, uint32_t E, const uint64_t* a, const uint64_t* b) {
  double sim = 0.0;
  for (uint32_t l = 0; l < L; ++l) sim += orc_row_similarity(a + (uint64_t)l * E, b + (uint64_t)l * E, E);
  double d = 1.0 - sim / L;
  if (d < 0.0) d = 0.0;
  if (d > 1.0) d = 1.0;
  return d;
}

/* ---------------------------------------------------------------- match */
/* Eamc::match: proj/core/src/eam.cpp:118-129.  entries are slot-ordered
 * [P][L][E]; seqs[P] the insertion numbers.  Returns 0 when P == 0. */
int orc_match(uint32_t L, uint32_t E, const uint64_t* entries, const uint64_t* seqs, uint64_t P,
              const uint64_t* probe, uint64_t* idx, uint64_t* seq, double* dist) {
  int found = 0;
  uint64_t bi = 0, bs = 0;
  double bd = 0.0;
  const uint64_t cells = (uint64_t)L * E;
  for (uint64_t i = 0; i < P; ++i) {
    const double d = orc_eam_distance(L, E, entries + i * cells, probe);
    if (!found || d < bd || (d == bd && seqs[i] < bs)) {
      found = 1;
      bi = i;
      bs = seqs[i];
      bd = d;
    }
  }
  if (found) {
    *idx = bi;
    *seq = bs;
    *dist = bd;
  }
  return found;
}

void orc_match_batch(uint32_t L, uint32_t E, const uint64_t* entries, const uint64_t* seqs,
                     uint64_t P, const uint64_t* probes, uint64_t Q, uint64_t* idx, uint64_t* seq,
                     double* dist, uint8_t* found) {
  const uint64_t cells = (uint64_t)L * E;
  for (uint64_t q = 0; q < Q; ++q)
    found[q] = (uint8_t)orc_match(L, E, entries, seqs, P, probes + q * cells, idx + q, seq + q, dist + q);
}

/* Eamc::match_within: proj/core/src/eam.cpp:131-150.  Writes all matches
 * (sorted by (distance, seq)) into out_*; returns their number. */
typedef struct orc_m { uint64_t idx, seq; double d; } orc_m;
static int orc_m_cmp(const void* pa, const void* pb) {
  const orc_m* a = (const orc_m*)pa;
  const orc_m* b = (const orc_m*)pb;
  if (a->d != b->d) return a->d < b->d ? -1 : 1;
  return a->seq < b->seq ? -1 : (a->seq > b->seq ? 1 : 0);
}
uint64_t orc_match_within(uint32_t L, uint32_t E, const uint64_t* entries, const uint64_t* seqs,
                          uint64_t P, const uint64_t* probe, double window, uint64_t* out_idx,
                          uint64_t* out_seq, double* out_d) {
  const uint64_t cells = (uint64_t)L * E;
  orc_m* all = (orc_m*)malloc((P ? P : 1) * sizeof(orc_m));
  double best = INFINITY;
  for (uint64_t i = 0; i < P; ++i) {
    const double d = orc_eam_distance(L, E, entries + i * cells, probe);
    if (d < best) best = d; /* std::min(best, d) */
    all[i].idx = i;
    all[i].seq = seqs[i];
    all[i].d = d;
  }
  uint64_t n = 0;
  for (uint64_t i = 0; i < P; ++i)
    if (all[i].d <= best + window) all[n++] = all[i];
  qsort(all, n, sizeof(orc_m), orc_m_cmp);
  for (uint64_t i = 0; i < n; ++i) {
    out_idx[i] = all[i].idx;
    out_seq[i] = all[i].seq;
    out_d[i] = all[i].d;
  }
  free(all);
  return n;
}

/* --------------------------------------------------------------- insert */
/* Eamc::insert: proj/core/src/eam.cpp:152-178 (capacity check, append with
 * seq = next_seq++, or nearest-entry replacement with oldest-seq tie-break,
 * in place).  State is caller-owned: entries [cap][L][E], seqs [cap].
 * Returns the victim slot or -1 for an append. */
int64_t orc_insert(uint32_t L, uint32_t E, uint64_t capacity, uint64_t* entries, uint64_t* seqs,
                   uint64_t* size, uint64_t* next_seq, const uint64_t* eam) {
  const uint64_t cells = (uint64_t)L * E;
  if (*size < capacity) {
    memcpy(entries + *size * cells, eam, cells * sizeof(uint64_t));
    seqs[*size] = (*next_seq)++;
    ++*size;
    return -1;
  }
  uint64_t victim = 0;
  double victim_d = INFINITY;
  for (uint64_t i = 0; i < *size; ++i) {
    const double d = orc_eam_distance(L, E, entries + i * cells, eam);
    if (d < victim_d || (d == victim_d && seqs[i] < seqs[victim])) {
      victim = i;
      victim_d = d;
    }
  }
  memcpy(entries + victim * cells, eam, cells * sizeof(uint64_t));
  seqs[victim] = (*next_seq)++;
  return (int64_t)victim;
}

/* ------------------------------------------------------------- policy */
/* prefetch_priorities: proj/core/src/policy.cpp:88-126, plus the engine's
 * floor filter proj/core/src/engine.cpp:663-668 when apply_filter != 0.
 * Output in the reference order (priority desc, ExpertId asc). */
typedef struct orc_c { uint32_t layer, expert; double pri; } orc_c;
static int orc_c_cmp(const void* pa, const void* pb) {
  const orc_c* a = (const orc_c*)pa;
  const orc_c* b = (const orc_c*)pb;
  if (a->pri != b->pri) return a->pri > b->pri ? -1 : 1;
  if (a->layer != b->layer) return a->layer < b->layer ? -1 : 1;
  return a->expert < b->expert ? -1 : (a->expert > b->expert ? 1 : 0);
}
uint64_t orc_prefetch_priorities(uint32_t L, uint32_t E, const uint64_t* entries,
                                 const uint64_t* seqs, uint64_t P, const uint64_t* cur,
                                 uint32_t current_layer, int apply_filter, uint32_t* out_layer,
                                 uint32_t* out_expert, double* out_pri) {
  const double kEpsilon = 1e-4;     /* policy.hpp:22 */
  const double kMatchWindow = 0.01; /* policy.hpp:30 */
  if (current_layer >= L || P == 0) return 0;
  const uint64_t cells = (uint64_t)L * E;
  uint64_t* midx = (uint64_t*)malloc(P * sizeof(uint64_t));
  uint64_t* mseq = (uint64_t*)malloc(P * sizeof(uint64_t));
  double* md = (double*)malloc(P * sizeof(double));
  const uint64_t nm = orc_match_within(L, E, entries, seqs, P, cur, kMatchWindow, midx, mseq, md);
  uint64_t* agg = (uint64_t*)calloc(cells, sizeof(uint64_t));
  for (uint64_t m = 0; m < nm; ++m) {
    const uint64_t* c = entries + midx[m] * cells;
    for (uint64_t i = 0; i < cells; ++i) agg[i] += c[i];
  }
  const uint64_t n_all = (uint64_t)(L - current_layer - 1) * E;
  orc_c* out = (orc_c*)malloc((n_all ? n_all : 1) * sizeof(orc_c));
  uint64_t n = 0;
  for (uint32_t i = current_layer + 1; i < L; ++i) {
    uint64_t row_sum = 0;
    const uint64_t base = (uint64_t)i * E;
    for (uint32_t j = 0; j < E; ++j) row_sum += agg[base + j];
    const double proximity = 1.0 - (double)(i - current_layer) / (double)L;
    for (uint32_t j = 0; j < E; ++j) {
      const double ratio = row_sum == 0 ? 0.0 : (double)agg[base + j] / (double)row_sum;
      out[n].layer = i;
      out[n].expert = j;
      out[n].pri = (ratio + kEpsilon) * proximity;
      ++n;
    }
  }
  qsort(out, n, sizeof(orc_c), orc_c_cmp);
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (apply_filter) {
      const double proximity = 1.0 - (double)(out[i].layer - current_layer) / (double)L;
      if (out[i].pri <= kEpsilon * proximity * (1.0 + 1e-9)) continue;
    }
    out_layer[k] = out[i].layer;
    out_expert[k] = out[i].expert;
    out_pri[k] = out[i].pri;
    ++k;
  }
  free(out);
  free(agg);
  free(md);
  free(mseq);
  free(midx);
  return k;
}

/* cache_priority: proj/core/src/policy.cpp:128-141.  Returns NAN on an
 * out-of-range expert (the reference throws std::out_of_range). */
double orc_cache_priority(uint32_t L, uint32_t E, const uint64_t* req, uint32_t layer,
                          uint32_t expert) {
  if (layer >= L || expert >= E) return NAN;
  uint64_t row_sum = 0;
  for (uint32_t j = 0; j < E; ++j) row_sum += req[(uint64_t)layer * E + j];
  const double ratio =
      row_sum == 0 ? 0.0 : (double)req[(uint64_t)layer * E + expert] / (double)row_sum;
  const double layer_weight = 1.0 - (double)layer / (double)L;
  return (ratio + 1e-4) * layer_weight;
}

/* select_eviction_victim: proj/core/src/policy.cpp:143-159.  Slot views as
 * parallel arrays (policy.hpp:96-101).  Returns -1 when every slot is
 * protected or pinned. */
int64_t orc_select_victim(uint32_t L, uint32_t E, const uint64_t* req, const uint64_t* slot,
                          const uint32_t* layer, const uint32_t* expert,
                          const uint8_t* prot, const uint8_t* pinned, uint64_t n) {
  int64_t victim = -1;
  double vp = 0.0;
  uint32_t vl = 0, ve = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (prot[i] || pinned[i]) continue;
    const double p = orc_cache_priority(L, E, req, layer[i], expert[i]);
    if (victim < 0 || p < vp ||
        (p == vp && (layer[i] < vl || (layer[i] == vl && expert[i] < ve)))) {
      victim = (int64_t)slot[i];
      vp = p;
      vl = layer[i];
      ve = expert[i];
    }
  }
  return victim;
}

/* ------------------------------------------------------------- tracing */
/* Eam::record: proj/core/src/eam.cpp:41-52 (validate every index, then
 * add).  Returns 0 on success, -1 (no mutation) on an out-of-range index. */
int orc_record(uint32_t L, uint32_t E, uint64_t* counts, uint32_t layer, const uint32_t* experts,
               const uint64_t* tokens, uint64_t n) {
  if (layer >= L) return -1;
  for (uint64_t i = 0; i < n; ++i)
    if (experts[i] >= E) return -1;
  for (uint64_t i = 0; i < n; ++i) counts[(uint64_t)layer * E + experts[i]] += tokens[i];
  return 0;
}

/* Router top-k trace -> per-request L x E counts: the per-token
 * `counts[e] += 1` loop of proj/core/src/workload.cpp:166-181 followed by
 * Eam::record of the aggregated events (eam.cpp:41-52).  topk is
 * [T][L][k] (uint32), offsets[R+1] token ranges per request.  All-or-
 * nothing: returns -1 and leaves `counts` untouched on a bad index. */
int orc_trace(uint32_t L, uint32_t E, uint32_t k, const uint32_t* topk, uint64_t T,
              const uint64_t* offsets, uint64_t R, uint64_t* counts) {
  for (uint64_t i = 0; i < T * L * k; ++i)
    if (topk[i] >= E) return -1;
  if (R && offsets[R] > T) return -1;
  for (uint64_t r = 0; r < R; ++r) {
    uint64_t* c = counts + r * (uint64_t)L * E;
    for (uint64_t t = offsets[r]; t < offsets[r + 1]; ++t)
      for (uint32_t l = 0; l < L; ++l)
        for (uint32_t j = 0; j < k; ++j) c[(uint64_t)l * E + topk[(t * L + l) * k + j]] += 1;
  }
  return 0;
}

/* eamc_capacity_bound: proj/core/src/eam.cpp:258-268.  0 = unsupported. */
uint64_t orc_capacity_bound(uint32_t L, uint32_t E, double similarity) {
  const uint64_t total = (uint64_t)L * E;
  const double le = (double)total;
  if (similarity == 0.75) return 2 * total;
  if (similarity == 0.98) return (uint64_t)ceil(0.5 * le * log(le));
  return 0;
}
