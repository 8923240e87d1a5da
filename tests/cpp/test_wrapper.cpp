// test_wrapper.cpp -- the reference's own EAM/EAMC/policy test cases
// (proj/tests/test_eam.cpp, test_policy.cpp), re-expressed against the
// GPU-backed C++ mirror (include/moesim_b200/eamc.hpp).  Built and run by
// tests/test_cpp_wrapper.py.  Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <map>
#include <set>
#include <vector>

#include "moesim_b200/eamc.hpp"

using namespace moesim_b200;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                        \
  do {                                                                  \
    if (c) {                                                            \
      ++g_pass;                                                         \
    } else {                                                            \
      ++g_fail;                                                         \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
    }                                                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, T) \
  do {                           \
    bool ok_ = false;            \
    try {                        \
      (void)(expr);              \
    } catch (const T&) {         \
      ok_ = true;                \
    } catch (...) {              \
    }                            \
    CHECK(ok_);                  \
  } while (0)

static bool approx(double a, double b, double eps = 1e-12) {
  return std::fabs(a - b) <= eps * std::max(1.0, std::max(std::fabs(a), std::fabs(b)));
}

// splitmix64 (rng.hpp:19-36)
struct Rng {
  std::uint64_t s;
  std::uint64_t next() {
    std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  std::uint64_t bounded(std::uint64_t n) {
    const std::uint64_t t = (0 - n) % n;
    for (;;) {
      const std::uint64_t r = next();
      if (r >= t) return r % n;
    }
  }
  bool bernoulli(double p) { return next_double() < p; }
};

static Eam make_eam(const ModelShape& s, std::vector<std::vector<std::uint64_t>> rows,
                    EamKind kind = EamKind::request, Phase phase = Phase::decode) {
  Eam e(s, kind, phase);
  for (std::uint32_t l = 0; l < rows.size(); ++l)
    for (std::uint32_t x = 0; x < rows[l].size(); ++x) e.set(l, x, rows[l][x]);
  return e;
}

static Eam random_eam(const ModelShape& s, Rng& rng) {  // test_eam.cpp:58-66
  Eam e(s, EamKind::request, Phase::decode);
  for (std::uint32_t l = 0; l < s.n_layers; ++l)
    for (std::uint32_t x = 0; x < s.n_experts_per_layer; ++x)
      if (rng.bernoulli(0.4)) e.set(l, x, rng.bounded(16) + 1);
  return e;
}

// test_eam.cpp:22-47: independent scalar oracle with explicit normalisation
static double oracle_distance(const Eam& a, const Eam& b) {
  const ModelShape& s = a.shape();
  double sim = 0.0;
  for (std::uint32_t l = 0; l < s.n_layers; ++l) {
    double sa = 0, sb = 0;
    for (std::uint32_t e = 0; e < s.n_experts_per_layer; ++e) {
      sa += double(a.at(l, e));
      sb += double(b.at(l, e));
    }
    if (sa == 0 && sb == 0) {
      sim += 1;
      continue;
    }
    if (sa == 0 || sb == 0) continue;
    double dot = 0, na = 0, nb = 0;
    for (std::uint32_t e = 0; e < s.n_experts_per_layer; ++e) {
      const double x = double(a.at(l, e)) / sa, y = double(b.at(l, e)) / sb;
      dot += x * y;
      na += x * x;
      nb += y * y;
    }
    sim += dot / (std::sqrt(na) * std::sqrt(nb));
  }
  return 1.0 - sim / s.n_layers;
}

static double scalar_prefetch_priority(std::uint64_t c, std::uint64_t row, std::uint32_t i,
                                       std::uint32_t l, std::uint32_t L) {
  double p = row ? double(c) / double(row) : 0.0;
  return (p + 1e-4) * (1.0 - double(i - l) / double(L));
}
static double scalar_cache_priority(std::uint64_t c, std::uint64_t row, std::uint32_t l,
                                    std::uint32_t L) {
  double p = row ? double(c) / double(row) : 0.0;
  return (p + 1e-4) * (1.0 - double(l) / double(L));
}

int main() {
  // ---- distance (test_eam.cpp:170-225)
  {
    const ModelShape s{2, 2, 1};
    CHECK(approx(eam_distance(make_eam(s, {{1, 0}, {0, 1}}), make_eam(s, {{1, 0}, {1, 0}})), 0.5));
    const ModelShape s1{1, 2, 1};
    CHECK(approx(eam_distance(make_eam(s1, {{1, 0}}), make_eam(s1, {{2, 0}})), 0.0));
    CHECK_THROWS_AS(eam_distance(Eam({1, 2, 1}, EamKind::request, Phase::decode),
                                 Eam({2, 2, 1}, EamKind::request, Phase::decode)),
                    std::invalid_argument);
    const Eam zero = make_eam(s, {{0, 0}, {0, 0}});
    const Eam one = make_eam(s, {{1, 0}, {0, 0}});
    CHECK(approx(eam_distance(zero, zero), 0.0));
    CHECK(approx(eam_distance(one, zero), 0.5));
    const ModelShape s3{3, 5, 1};
    Rng rng{17};
    for (int t = 0; t < 200; ++t) {
      const Eam a = random_eam(s3, rng), b = random_eam(s3, rng);
      const double d = eam_distance(a, b);
      CHECK(d == eam_distance(b, a));
      CHECK(d >= 0.0 && d <= 1.0);
      CHECK(approx(d, oracle_distance(a, b)));
    }
  }
  // ---- match (test_eam.cpp:227-261)
  {
    const ModelShape s{2, 4, 1};
    Eamc eamc(s, Phase::decode, 200);
    Rng rng{23};
    const Eam probe = random_eam(s, rng);
    CHECK(!eamc.match(probe).has_value());
    std::vector<Eam> entries;
    for (int i = 0; i < 100; ++i) {
      entries.push_back(random_eam(s, rng));
      eamc.insert(entries.back());
    }
    for (int q = 0; q < 20; ++q) {
      const Eam p = random_eam(s, rng);
      std::size_t best = 0;
      double best_d = oracle_distance(entries[0], p);
      for (std::size_t i = 1; i < entries.size(); ++i) {
        const double d = oracle_distance(entries[i], p);
        if (d < best_d) {
          best = i;
          best_d = d;
        }
      }
      const auto m = eamc.match(p);
      CHECK(m.has_value() && m->index == best && approx(m->distance, best_d));
    }
    const auto self = eamc.match(entries[42]);
    CHECK(self && self->index == 42 && approx(self->distance, 0.0));
  }
  // ---- insert (test_eam.cpp:263-342)
  {
    const ModelShape s{1, 4, 1};
    Eamc eamc(s, Phase::decode, 3);
    const Eam e1 = make_eam(s, {{10, 0, 0, 0}}), e2 = make_eam(s, {{0, 10, 0, 0}}),
              e3 = make_eam(s, {{0, 0, 10, 0}}), e4 = make_eam(s, {{0, 0, 9, 1}});
    CHECK(!eamc.insert(e1).has_value());
    eamc.insert(e2);
    eamc.insert(e3);
    const auto ev = eamc.insert(e4);
    CHECK(ev.has_value() && *ev == e3);
    CHECK(eamc.size() == 3);
    CHECK(approx(eamc.match(e1)->distance, 0.0));

    const ModelShape s2{2, 4, 1};
    Eamc c(s2, Phase::decode, 10);
    std::vector<std::pair<Eam, std::uint64_t>> model;
    Rng rng{31};
    std::uint64_t next_seq = 0;
    for (int step = 0; step < 50; ++step) {
      const Eam in = random_eam(s2, rng);
      std::optional<std::size_t> expect;
      if (model.size() == 10) {
        double best = 1e9;
        std::uint64_t bs = 0;
        for (std::size_t i = 0; i < model.size(); ++i) {
          const double d = oracle_distance(model[i].first, in);
          if (d < best || (d == best && model[i].second < bs)) {
            best = d;
            bs = model[i].second;
            expect = i;
          }
        }
      }
      const auto got = c.insert(in);
      if (expect) {
        CHECK(got.has_value() && *got == model[*expect].first);
        model[*expect] = {in, next_seq++};
      } else {
        CHECK(!got.has_value());
        model.emplace_back(in, next_seq++);
      }
    }
    const ModelShape s3{1, 2, 1};
    Eamc v(s3, Phase::decode, 2);
    CHECK_THROWS_AS(v.insert(Eam(s3, EamKind::iteration, Phase::decode)), std::invalid_argument);
    CHECK_THROWS_AS(v.insert(Eam(s3, EamKind::request, Phase::prefill)), std::invalid_argument);
    CHECK_THROWS_AS(v.insert(Eam({2, 2, 1}, EamKind::request, Phase::decode)),
                    std::invalid_argument);
  }
  // ---- capacity bounds (test_eam.cpp:344-349)
  CHECK(eamc_capacity_bound({12, 128, 1}, 0.75) == 3072);
  CHECK(eamc_capacity_bound({12, 128, 1}, 0.98) == 5635);
  CHECK_THROWS_AS(eamc_capacity_bound({2, 2, 1}, 0.9), std::invalid_argument);
  // ---- snapshot (test_eam.cpp:351-395)
  {
    const auto path = std::filesystem::temp_directory_path() / "moesim_b200_snap.json";
    const ModelShape s{3, 6, 1};
    Eamc full(s, Phase::decode, 64);
    Rng rng{41};
    for (int i = 0; i < 100; ++i) full.insert(random_eam(s, rng));
    full.save(path);
    const Eamc back = Eamc::load(path, s);
    CHECK(back.size() == full.size());
    for (std::size_t i = 0; i < back.size(); ++i) {
      CHECK(back.entry(i) == full.entry(i));
      CHECK(back.entry_seq(i) == full.entry_seq(i));
    }
    Eamc f2 = Eamc::load(path, s), f3 = Eamc::load(path, s);
    const Eam next = random_eam(s, rng);
    CHECK(f2.insert(next) == f3.insert(next));
    CHECK_THROWS_AS(Eamc::load(path, ModelShape{4, 6, 1}), EamcSnapshotError);
    {
      std::ofstream o(path);
      o << "not json\n";
    }
    CHECK_THROWS_AS(Eamc::load(path), EamcSnapshotError);
    std::filesystem::remove(path);
  }
  // ---- prefetch priorities (test_policy.cpp:46-148)
  {
    const ModelShape s{4, 2, 1};
    Eamc eamc(s, Phase::decode, 4);
    eamc.insert(make_eam(s, {{1, 0}, {1, 0}, {2, 1}, {0, 3}}));
    const Eam cur = make_eam(s, {{1, 0}, {1, 0}, {0, 0}, {0, 0}}, EamKind::iteration);
    const auto out = prefetch_priorities(cur, eamc, 1);
    CHECK(out.size() == 4);
    CHECK((out[0].expert == ExpertId{2, 0}) && approx(out[0].priority, 0.500075));
    for (std::size_t i = 1; i < out.size(); ++i) CHECK(out[i - 1].priority >= out[i].priority);
    CHECK_THROWS_AS(prefetch_priorities(cur, eamc, 4), std::out_of_range);
    const Eamc empty(s, Phase::decode, 2);
    CHECK(prefetch_priorities(cur, empty, 0).empty());

    Rng rng{71};
    for (int t = 0; t < 100; ++t) {
      const std::uint32_t L = 2 + rng.bounded(6), E = 1 + rng.bounded(6);
      const ModelShape sh{L, E, 1};
      Eam entry(sh, EamKind::request, Phase::decode);
      for (std::uint32_t l = 0; l < L; ++l)
        for (std::uint32_t e = 0; e < E; ++e)
          if (rng.bernoulli(0.5)) entry.set(l, e, rng.bounded(20) + 1);
      Eamc c(sh, Phase::decode, 1);
      c.insert(entry);
      Eam cu(sh, EamKind::iteration, Phase::decode);
      cu.set(0, 0, 1);
      const std::uint32_t l0 = rng.bounded(L);
      const auto o = prefetch_priorities(cu, c, l0);
      CHECK(o.size() == std::size_t{L - l0 - 1} * E);
      for (const auto& pc : o)
        CHECK(approx(pc.priority,
                     scalar_prefetch_priority(entry.at(pc.expert.layer_idx, pc.expert.expert_idx),
                                              entry.row_sum(pc.expert.layer_idx),
                                              pc.expert.layer_idx, l0, L)));
    }
  }
  // ---- cache priority + victims (test_policy.cpp:164-193, 330-377)
  {
    const ModelShape s{3, 2, 1};
    const Eam req = make_eam(s, {{1, 3}, {0, 0}, {2, 2}});
    CHECK(approx(cache_priority(req, {0, 1}), 0.7501));
    CHECK(approx(cache_priority(req, {1, 0}), 1e-4 * (1.0 - 1.0 / 3.0)));
    CHECK_THROWS_AS(cache_priority(req, {3, 0}), std::out_of_range);
    const ModelShape s2{2, 4, 1};
    const Eam r2 = make_eam(s2, {{4, 3, 2, 1}, {1, 1, 1, 1}});
    std::vector<SlotView> one{{0, {0, 2}, false, false}};
    CHECK(select_eviction_victim(one, r2) == std::optional<std::size_t>(0));
    std::vector<SlotView> prot{{0, {0, 2}, true, false}, {1, {0, 3}, false, true}};
    CHECK(!select_eviction_victim(prot, r2).has_value());

    Rng rng{83};
    const ModelShape s4{4, 8, 1};
    for (int t = 0; t < 200; ++t) {
      Eam rq(s4, EamKind::request, Phase::decode);
      for (std::uint32_t l = 0; l < 4; ++l)
        for (std::uint32_t e = 0; e < 8; ++e)
          if (rng.bernoulli(0.6)) rq.set(l, e, rng.bounded(20));
      std::vector<SlotView> views;
      std::set<std::pair<std::uint32_t, std::uint32_t>> used;
      for (std::size_t slot = 0; slot < 8; ++slot) {
        ExpertId id;
        do {
          id = {static_cast<std::uint32_t>(rng.bounded(4)), static_cast<std::uint32_t>(rng.bounded(8))};
        } while (!used.insert({id.layer_idx, id.expert_idx}).second);
        const bool pr = rng.bernoulli(0.2);
        const bool pn = rng.bernoulli(0.2);
        views.push_back({slot, id, pr, pn});
      }
      std::optional<std::size_t> expect;
      double best = 0;
      ExpertId bid;
      for (const SlotView& v : views) {
        if (v.prefetch_protected || v.pinned) continue;
        const double p = scalar_cache_priority(rq.at(v.occupant.layer_idx, v.occupant.expert_idx),
                                               rq.row_sum(v.occupant.layer_idx),
                                               v.occupant.layer_idx, 4);
        if (!expect || p < best || (p == best && v.occupant < bid)) {
          expect = v.slot;
          best = p;
          bid = v.occupant;
        }
      }
      CHECK(select_eviction_victim(views, rq) == expect);
    }
  }
  std::printf("wrapper parity: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
