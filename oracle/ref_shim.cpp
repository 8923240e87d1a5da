// ref_shim.cpp -- TEST INFRASTRUCTURE: an extern "C" face over the UNMODIFIED
// reference library (moesim, compiled from /root/reference/proj/core/src by
// oracle/Makefile into oracle/_ref/libmoesim_ref.so).  It lets tests/ and
// bench.py's reference/cpu_baseline arm drive the reference's own code path
// (Eam, Eamc::insert/match/match_within, prefetch_priorities, cache_priority,
// select_eviction_victim, bench_match, generate_trace) from Python via
// ctypes.  Nothing here re-implements reference arithmetic: every number it
// returns is computed by the reference library itself.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <thread>
#include <vector>

#include "moesim/bench.hpp"
#include "moesim/eam.hpp"
#include "moesim/model.hpp"
#include "moesim/policy.hpp"
#include "moesim/rng.hpp"
#include "moesim/workload.hpp"

using namespace moesim;

namespace {

Eam make_eam(const ModelShape& s, const uint64_t* c, EamKind kind, Phase phase) {
  Eam eam(s, kind, phase);
  for (uint32_t l = 0; l < s.n_layers; ++l)
    for (uint32_t e = 0; e < s.n_experts_per_layer; ++e) {
      const uint64_t v = c[uint64_t{l} * s.n_experts_per_layer + e];
      if (v) eam.set(l, e, v);
    }
  return eam;
}

struct RefEamc {
  Eamc eamc;
  std::vector<uint64_t> seq_of_slot;  // mirrors entry_seq for slot lookup
};

// Error convention of the shim: 0 ok, 1 invalid_argument, 2 out_of_range,
// 3 snapshot, 4 logic_error, 9 other.
int code_of(const std::exception_ptr& p) {
  try {
    std::rethrow_exception(p);
  } catch (const EamcSnapshotError&) {
    return 3;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::out_of_range&) {
    return 2;
  } catch (const std::logic_error&) {
    return 4;
  } catch (...) {
    return 9;
  }
}

}  // namespace

extern "C" {

double ref_eam_distance(uint32_t L, uint32_t E, const uint64_t* a, const uint64_t* b) {
  const ModelShape s{L, E, 1};
  return eam_distance(make_eam(s, a, EamKind::request, Phase::decode),
                      make_eam(s, b, EamKind::request, Phase::decode));
}

void* ref_eamc_new(uint32_t L, uint32_t E, uint32_t top_k, int phase, uint64_t capacity) {
  try {
    return new RefEamc{Eamc(ModelShape{L, E, top_k}, phase == 0 ? Phase::prefill : Phase::decode,
                            capacity),
                       {}};
  } catch (...) {
    return nullptr;
  }
}

void ref_eamc_free(void* h) { delete static_cast<RefEamc*>(h); }

uint64_t ref_eamc_size(void* h) { return static_cast<RefEamc*>(h)->eamc.size(); }

// Inserts one request-level EAM; *slot = replaced slot or -1.
int ref_eamc_insert(void* h, const uint64_t* counts, int kind, int phase, int64_t* slot) {
  auto* r = static_cast<RefEamc*>(h);
  try {
    const Eamc& e = r->eamc;
    const bool full = e.size() == e.capacity();
    auto evicted = r->eamc.insert(make_eam(e.shape(), counts,
                                           kind == 0 ? EamKind::iteration : EamKind::request,
                                           phase == 0 ? Phase::prefill : Phase::decode));
    if (!full) {
      *slot = -1;
    } else {
      // The newcomer holds the largest seq; find its slot.
      uint64_t best = 0;
      for (size_t i = 0; i < e.size(); ++i)
        if (e.entry_seq(i) > e.entry_seq(best)) best = i;
      *slot = static_cast<int64_t>(best);
    }
    (void)evicted;
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

void ref_eamc_entry(void* h, uint64_t i, uint64_t* counts, uint64_t* seq) {
  const Eamc& e = static_cast<RefEamc*>(h)->eamc;
  auto c = e.entry(i).counts();
  std::copy(c.begin(), c.end(), counts);
  *seq = e.entry_seq(i);
}

int ref_eamc_match(void* h, const uint64_t* probes, uint64_t Q, uint64_t* idx, uint64_t* seq,
                   double* dist, uint8_t* found) {
  const Eamc& e = static_cast<RefEamc*>(h)->eamc;
  try {
    const uint64_t cells = e.shape().total_experts();
    for (uint64_t q = 0; q < Q; ++q) {
      auto m = e.match(make_eam(e.shape(), probes + q * cells, EamKind::request, e.phase()));
      found[q] = m.has_value();
      if (m) {
        idx[q] = m->index;
        seq[q] = m->seq;
        dist[q] = m->distance;
      }
    }
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// Multi-threaded probe split over the const Eamc::match (SPEC.md:198 allows
// concurrent readers).  Returns wall seconds spent inside match calls.
double ref_eamc_match_mt(void* h, const uint64_t* probes, uint64_t Q, uint64_t* idx,
                         uint64_t* seq, double* dist, uint8_t* found, int n_threads) {
  const Eamc& e = static_cast<RefEamc*>(h)->eamc;
  const uint64_t cells = e.shape().total_experts();
  std::vector<Eam> eams;
  eams.reserve(Q);
  for (uint64_t q = 0; q < Q; ++q)
    eams.push_back(make_eam(e.shape(), probes + q * cells, EamKind::request, e.phase()));
  if (n_threads < 1) n_threads = 1;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < n_threads; ++t)
    pool.emplace_back([&, t] {
      for (uint64_t q = t; q < Q; q += n_threads) {
        auto m = e.match(eams[q]);
        found[q] = m.has_value();
        if (m) {
          idx[q] = m->index;
          seq[q] = m->seq;
          dist[q] = m->distance;
        }
      }
    });
  for (auto& th : pool) th.join();
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

int64_t ref_eamc_match_within(void* h, const uint64_t* probe, double window, uint64_t* idx,
                              uint64_t* seq, double* dist, uint64_t cap) {
  const Eamc& e = static_cast<RefEamc*>(h)->eamc;
  try {
    auto ms = e.match_within(make_eam(e.shape(), probe, EamKind::iteration, e.phase()), window);
    for (size_t i = 0; i < ms.size() && i < cap; ++i) {
      idx[i] = ms[i].index;
      seq[i] = ms[i].seq;
      dist[i] = ms[i].distance;
    }
    return static_cast<int64_t>(ms.size());
  } catch (...) {
    return -code_of(std::current_exception());
  }
}

// prefetch_priorities (+ optional engine.cpp:663-668 floor filter).
int64_t ref_prefetch_priorities(void* h, const uint64_t* cur, uint32_t current_layer,
                                int apply_filter, uint32_t* out_layer, uint32_t* out_expert,
                                double* out_pri, uint64_t cap) {
  const Eamc& e = static_cast<RefEamc*>(h)->eamc;
  try {
    auto cands = prefetch_priorities(make_eam(e.shape(), cur, EamKind::iteration, e.phase()), e,
                                     current_layer);
    if (apply_filter) {
      const uint32_t L = e.shape().n_layers;
      std::erase_if(cands, [&](const PrefetchCandidate& c) {
        const double proximity =
            1.0 - static_cast<double>(c.expert.layer_idx - current_layer) / static_cast<double>(L);
        return c.priority <= kEpsilon * proximity * (1.0 + 1e-9);
      });
    }
    for (size_t i = 0; i < cands.size() && i < cap; ++i) {
      out_layer[i] = cands[i].expert.layer_idx;
      out_expert[i] = cands[i].expert.expert_idx;
      out_pri[i] = cands[i].priority;
    }
    return static_cast<int64_t>(cands.size());
  } catch (...) {
    return -code_of(std::current_exception());
  }
}

int ref_cache_priority(uint32_t L, uint32_t E, const uint64_t* req, uint32_t layer,
                       uint32_t expert, double* out) {
  try {
    *out = cache_priority(make_eam(ModelShape{L, E, 1}, req, EamKind::request, Phase::decode),
                          ExpertId{layer, expert});
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int64_t ref_select_victim(uint32_t L, uint32_t E, const uint64_t* req, const uint64_t* slot,
                          const uint32_t* layer, const uint32_t* expert, const uint8_t* prot,
                          const uint8_t* pinned, uint64_t n) {
  std::vector<SlotView> views;
  for (uint64_t i = 0; i < n; ++i)
    views.push_back({slot[i], ExpertId{layer[i], expert[i]}, prot[i] != 0, pinned[i] != 0});
  auto v = select_eviction_victim(
      views, make_eam(ModelShape{L, E, 1}, req, EamKind::request, Phase::decode));
  return v ? static_cast<int64_t>(*v) : -1;
}

// Eam::record of one event on a caller-owned count matrix; all-or-nothing.
int ref_eam_record(uint32_t L, uint32_t E, uint64_t* counts, uint32_t layer,
                   const uint32_t* experts, const uint64_t* tokens, uint64_t n) {
  try {
    Eam eam = make_eam(ModelShape{L, E, 1}, counts, EamKind::iteration, Phase::decode);
    RoutingEvent ev;
    ev.layer_idx = layer;
    for (uint64_t i = 0; i < n; ++i) ev.assignments.push_back({experts[i], tokens[i]});
    eam.record(ev);
    auto c = eam.counts();
    std::copy(c.begin(), c.end(), counts);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// Router top-k ids [T][L][k] (u8) -> per-request request-level EAMs with the
// reference's own types: per request and layer, the per-expert token counts
// are gathered as workload.cpp:166-181 does and handed to Eam::record as one
// RoutingEvent per layer.  Requests are split over n_threads std::threads
// (independent Eams).  Returns wall seconds, or -1 on a record error.
double ref_trace_mt(uint32_t L, uint32_t E, uint32_t k, const uint8_t* topk,
                    const uint64_t* offsets, uint64_t R, uint64_t* out, int n_threads) {
  if (n_threads < 1) n_threads = 1;
  const ModelShape shape{L, E, k};
  std::vector<int> err(n_threads, 0);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int th = 0; th < n_threads; ++th)
    pool.emplace_back([&, th] {
      std::vector<uint64_t> c(E);
      try {
        for (uint64_t r = th; r < R; r += n_threads) {
          Eam eam(shape, EamKind::request, Phase::decode);
          for (uint32_t l = 0; l < L; ++l) {
            std::fill(c.begin(), c.end(), 0);
            for (uint64_t t = offsets[r]; t < offsets[r + 1]; ++t)
              for (uint32_t j = 0; j < k; ++j) {
                const uint32_t e = topk[(t * L + l) * k + j];
                if (e < E) ++c[e]; else throw std::out_of_range("expert");
              }
            RoutingEvent ev;
            ev.layer_idx = l;
            for (uint32_t e = 0; e < E; ++e)
              if (c[e]) ev.assignments.push_back({e, c[e]});
            if (!ev.assignments.empty()) eam.record(ev);
          }
          auto cnt = eam.counts();
          std::copy(cnt.begin(), cnt.end(), out + r * uint64_t{L} * E);
        }
      } catch (...) {
        err[th] = 1;
      }
    });
  for (auto& t : pool) t.join();
  const auto t1 = std::chrono::steady_clock::now();
  for (int e : err)
    if (e) return -1.0;
  return std::chrono::duration<double>(t1 - t0).count();
}

uint64_t ref_capacity_bound(uint32_t L, uint32_t E, double similarity) {
  try {
    return eamc_capacity_bound(ModelShape{L, E, 1}, similarity);
  } catch (...) {
    return 0;
  }
}

// The bench family of bench_match (bench.cpp:44-54, :60-66) drawn from the
// reference's own Rng: Rng::stream(seed, 0x6265636E), <= 4 set()s per row,
// counts U[1,32] (random_request_eam is file-local in bench.cpp, so its four
// lines of generator logic are restated here; every draw is the reference
// Rng's).  ref_gen_bench skips `skip` EAMs and writes n as u64 [n][L][E];
// ref_eamc_fill_bench inserts the first n of the stream into an Eamc through
// Eamc::insert exactly as bench_match's fill loop does (no host copy of the
// collection is materialised: P = 2^20 at 12x128 is 12.9 GB as Eams).
namespace {
Eam bench_eam(const ModelShape& shape, Rng& rng) {
  Eam eam(shape, EamKind::request, Phase::decode);
  const uint32_t active = std::min<uint32_t>(4, shape.n_experts_per_layer);
  for (uint32_t l = 0; l < shape.n_layers; ++l)
    for (uint32_t k = 0; k < active; ++k) {
      const auto e = static_cast<uint32_t>(rng.bounded(shape.n_experts_per_layer));
      eam.set(l, e, rng.bounded(32) + 1);
    }
  return eam;
}
}  // namespace

void ref_gen_bench(uint64_t seed, uint32_t L, uint32_t E, uint64_t skip, uint64_t n,
                   uint64_t* out) {
  const ModelShape s{L, E, 1};
  Rng rng = Rng::stream(seed, 0x6265636Eull);
  for (uint64_t i = 0; i < skip; ++i) (void)bench_eam(s, rng);
  const uint64_t cells = uint64_t{L} * E;
  for (uint64_t i = 0; i < n; ++i) {
    const Eam eam = bench_eam(s, rng);
    const auto c = eam.counts();
    std::copy(c.begin(), c.end(), out + i * cells);
  }
}

int ref_eamc_fill_bench(void* h, uint64_t seed, uint64_t n) {
  auto* r = static_cast<RefEamc*>(h);
  try {
    Rng rng = Rng::stream(seed, 0x6265636Eull);
    const ModelShape s = r->eamc.shape();
    for (uint64_t i = 0; i < n; ++i) r->eamc.insert(bench_eam(s, rng));
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// bench_match (bench.cpp:58-88): returns the checksum, mean/median us.
uint64_t ref_bench_match(uint64_t n_entries, uint32_t L, uint32_t E, uint64_t n_queries,
                         uint64_t seed, double* mean_us, double* median_us) {
  auto r = bench_match(n_entries, ModelShape{L, E, 1}, n_queries, seed);
  if (mean_us) *mean_us = r.mean_us;
  if (median_us) *median_us = r.median_us;
  return r.checksum;
}

// Reference-generated request trace (workload.cpp generate_trace) folded
// into per-iteration L x E counts by Eam::record, for pinning the oracle's
// workload restatement.  Returns the iteration count; writes up to
// max_iter iterations.
uint32_t ref_generate_trace_counts(uint32_t L, uint32_t E, uint32_t top_k, uint32_t n_groups,
                                   double fidelity, double skew, uint32_t prompt_len,
                                   uint32_t decode_len, uint32_t batch, uint64_t seed,
                                   uint64_t request_index, uint64_t* iter_counts,
                                   uint32_t max_iter) {
  WorkloadSpec w;
  w.shape = ModelShape{L, E, top_k};
  w.n_groups = n_groups;
  w.group_fidelity = fidelity;
  w.reuse_skew = skew;
  w.prompt_len = DiscreteDist::constant(prompt_len);
  w.decode_len = DiscreteDist::constant(decode_len);
  w.batch_size = batch;
  w.seed = seed;
  const RequestTrace t = generate_trace(w, request_index);
  const uint64_t cells = uint64_t{L} * E;
  for (uint32_t it = 0; it < t.iterations.size() && it < max_iter; ++it) {
    Eam eam(w.shape, EamKind::iteration, it == 0 ? Phase::prefill : Phase::decode);
    for (const RoutingEvent& ev : t.iterations[it]) eam.record(ev);
    auto c = eam.counts();
    std::copy(c.begin(), c.end(), iter_counts + it * cells);
  }
  return static_cast<uint32_t>(t.iterations.size());
}

// The reference's own JSONL writer over its own corpus generator
// (workload.cpp generate_corpus, model.cpp write_traces_jsonl): trace fixtures.
int ref_write_corpus_jsonl(const char* path, uint32_t L, uint32_t E, uint32_t top_k,
                           uint32_t n_groups, double fidelity, double skew, uint32_t prompt_len,
                           uint32_t decode_len, uint32_t batch, uint64_t seed, uint64_t n) {
  try {
    WorkloadSpec w;
    w.shape = ModelShape{L, E, top_k};
    w.n_groups = n_groups;
    w.group_fidelity = fidelity;
    w.reuse_skew = skew;
    w.prompt_len = DiscreteDist::constant(prompt_len);
    w.decode_len = DiscreteDist::constant(decode_len);
    w.batch_size = batch;
    w.seed = seed;
    const auto traces = generate_corpus(w, n);
    write_traces_jsonl(path, traces);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// `moesim eamc save` (tools/moesim_main.cpp:203-221) on the reference
// library: ingest_traces (validated), request_level_eam (restated verbatim
// from moesim_main.cpp:192-201, which lives in that file's anonymous
// namespace), Eamc::insert in file order, Eamc::save.  Returns 0, or 9 with
// the TraceIngestError text in err.
int ref_eamc_save_from_traces(const char* trace_path, uint32_t L, uint32_t E, uint32_t top_k,
                              int phase, uint64_t capacity, const char* out_path, char* err,
                              uint64_t err_len) {
  try {
    const ModelShape shape{L, E, top_k};
    const Phase ph = phase == 0 ? Phase::prefill : Phase::decode;
    const auto traces = ingest_traces(trace_path, shape);
    Eamc eamc(shape, ph, capacity);
    for (const auto& trace : traces) {
      if (ph == Phase::decode && trace.iterations.size() < 2) continue;
      Eam eam(shape, EamKind::request, ph);
      const std::size_t begin = ph == Phase::prefill ? 0 : 1;
      const std::size_t end = ph == Phase::prefill ? 1 : trace.iterations.size();
      for (std::size_t it = begin; it < end && it < trace.iterations.size(); ++it)
        for (const RoutingEvent& ev : trace.iterations[it]) eam.record(ev);
      eamc.insert(std::move(eam));
    }
    eamc.save(out_path);
    return 0;
  } catch (const TraceIngestError& e) {
    std::snprintf(err, err_len, "%s", e.what());
    return 9;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

}  // extern "C"
