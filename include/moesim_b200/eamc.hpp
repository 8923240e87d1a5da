// moesim_b200/eamc.hpp -- header-only C++ mirror of the reference's EAM/EAMC/policy
// API (moesim: core/include/moesim/{model,eam,policy}.hpp) over the C ABI of
// libmoe_eamc.so (include/moe_eamc.h).  Same type and function names, same
// argument meaning, and the same exceptions (status codes are mapped back:
// std::invalid_argument, std::out_of_range, EamcSnapshotError), so reference
// callers switch by changing the include and the namespace.
//
// Deviation: Eamc::entry(i) returns the Eam by value (the entries live in
// device memory), where the reference returns `const Eam&`.
#pragma once

#include <compare>
#include <cstdint>
#include <filesystem>
#include <limits>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../moe_eamc.h"

namespace moesim_b200 {

// ------------------------------------------------------------- model.hpp
struct ModelShape {
  std::uint32_t n_layers = 0;
  std::uint32_t n_experts_per_layer = 0;
  std::uint32_t top_k = 1;
  std::uint64_t total_experts() const { return std::uint64_t{n_layers} * n_experts_per_layer; }
  bool operator==(const ModelShape&) const = default;
  moe_shape c() const { return moe_shape{n_layers, n_experts_per_layer, top_k}; }
  void validate() const {  // model.cpp:13-19
    if (n_layers < 1) throw std::invalid_argument("ModelShape: n_layers must be >= 1");
    if (n_experts_per_layer < 1)
      throw std::invalid_argument("ModelShape: n_experts_per_layer must be >= 1");
    if (top_k < 1 || top_k > n_experts_per_layer)
      throw std::invalid_argument("ModelShape: top_k must be in [1, n_experts_per_layer]");
  }
};

struct ExpertId {
  std::uint32_t layer_idx = 0;
  std::uint32_t expert_idx = 0;
  auto operator<=>(const ExpertId&) const = default;
  std::uint64_t flat(const ModelShape& s) const {
    return std::uint64_t{layer_idx} * s.n_experts_per_layer + expert_idx;
  }
};

struct ExpertAssignment {
  std::uint32_t expert_idx = 0;
  std::uint64_t token_count = 0;
  bool operator==(const ExpertAssignment&) const = default;
};

struct RoutingEvent {
  std::uint32_t layer_idx = 0;
  std::vector<ExpertAssignment> assignments;
  bool operator==(const RoutingEvent&) const = default;
};

// --------------------------------------------------------------- errors
struct EamcSnapshotError : std::runtime_error {
  explicit EamcSnapshotError(const std::string& w) : std::runtime_error(w) {}
};
struct DeviceError : std::runtime_error {
  explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

inline void throw_on(moe_status s) {
  if (s == MOE_OK) return;
  const std::string msg = moe_last_error();
  switch (s) {
    case MOE_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case MOE_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case MOE_ERR_SNAPSHOT: throw EamcSnapshotError(msg);
    case MOE_ERR_LOGIC: throw std::logic_error(msg);
    case MOE_ERR_OVERFLOW: throw std::overflow_error(msg);
    default: throw DeviceError(msg);
  }
}

// ---------------------------------------------------------------- eam.hpp
enum class EamKind : std::uint8_t { iteration, request };
enum class Phase : std::uint8_t { prefill, decode };

class Eam {
 public:
  Eam(ModelShape shape, EamKind kind, Phase phase) : shape_(shape), kind_(kind), phase_(phase) {
    shape_.validate();
    counts_.assign(shape_.total_experts(), 0);
  }
  const ModelShape& shape() const { return shape_; }
  EamKind kind() const { return kind_; }
  Phase phase() const { return phase_; }
  std::uint64_t at(std::uint32_t l, std::uint32_t e) const {
    return counts_[std::uint64_t{l} * shape_.n_experts_per_layer + e];
  }
  std::uint64_t row_sum(std::uint32_t l) const {
    std::uint64_t s = 0;
    for (std::uint64_t c : row(l)) s += c;
    return s;
  }
  std::span<const std::uint64_t> row(std::uint32_t l) const {
    const std::size_t e = shape_.n_experts_per_layer;
    return {counts_.data() + std::size_t{l} * e, e};
  }
  std::span<const std::uint64_t> counts() const { return counts_; }
  std::uint64_t* data() { return counts_.data(); }
  const std::uint64_t* data() const { return counts_.data(); }

  // eam.cpp:41-52 (single-event bookkeeping; batched tracing from router ids
  // is trace_requests(), the GPU kernel)
  void record(const RoutingEvent& ev) {
    if (ev.layer_idx >= shape_.n_layers)
      throw std::out_of_range("Eam::record: layer index out of range");
    for (const ExpertAssignment& a : ev.assignments)
      if (a.expert_idx >= shape_.n_experts_per_layer)
        throw std::out_of_range("Eam::record: expert index out of range");
    const std::uint64_t base = std::uint64_t{ev.layer_idx} * shape_.n_experts_per_layer;
    for (const ExpertAssignment& a : ev.assignments) counts_[base + a.expert_idx] += a.token_count;
  }
  void accumulate(const Eam& o) {  // eam.cpp:54-60
    if (!(shape_ == o.shape_)) throw std::invalid_argument("Eam::accumulate: shape mismatch");
    if (phase_ != o.phase_) throw std::invalid_argument("Eam::accumulate: phase mismatch");
    for (std::size_t i = 0; i < counts_.size(); ++i) counts_[i] += o.counts_[i];
  }
  void reset() { counts_.assign(counts_.size(), 0); }
  void set(std::uint32_t l, std::uint32_t e, std::uint64_t c) {
    if (l >= shape_.n_layers || e >= shape_.n_experts_per_layer)
      throw std::out_of_range("Eam::set: index out of range");
    counts_[std::uint64_t{l} * shape_.n_experts_per_layer + e] = c;
  }
  bool operator==(const Eam&) const = default;

 private:
  ModelShape shape_;
  EamKind kind_;
  Phase phase_;
  std::vector<std::uint64_t> counts_;
};

inline double eam_distance(const Eam& a, const Eam& b) {  // eam.cpp:91-104 (GPU)
  if (!(a.shape() == b.shape())) throw std::invalid_argument("eam_distance: shape mismatch");
  const moe_shape s = a.shape().c();
  double d = 0.0;
  throw_on(moe_eam_distance(&s, a.data(), b.data(), &d));
  return d;
}

struct EamcMatch {
  std::size_t index = 0;
  std::uint64_t seq = 0;
  double distance = 0.0;
};

class Eamc {
 public:
  Eamc(ModelShape shape, Phase phase, std::size_t capacity, int device = 0) : shape_(shape) {
    const moe_shape s = shape.c();
    throw_on(moe_eamc_create(&s, static_cast<moe_phase>(phase), capacity, 0, device, &h_));
  }
  Eamc(Eamc&& o) noexcept : shape_(o.shape_), h_(std::exchange(o.h_, nullptr)) {}
  Eamc& operator=(Eamc&& o) noexcept {
    std::swap(h_, o.h_);
    shape_ = o.shape_;
    return *this;
  }
  Eamc(const Eamc&) = delete;
  Eamc& operator=(const Eamc&) = delete;
  ~Eamc() {
    if (h_) moe_eamc_destroy(h_);
  }

  const ModelShape& shape() const { return shape_; }
  Phase phase() const { return static_cast<Phase>(info().phase); }
  std::size_t capacity() const { return info().capacity; }
  std::size_t size() const { return info().size; }
  bool empty() const { return size() == 0; }
  Eam entry(std::size_t i) const {
    Eam e(shape_, EamKind::request, phase());
    throw_on(moe_eamc_entry(h_, i, e.data(), nullptr));
    return e;
  }
  std::uint64_t entry_seq(std::size_t i) const {
    std::uint64_t s = 0;
    throw_on(moe_eamc_entry(h_, i, nullptr, &s));
    return s;
  }

  std::optional<EamcMatch> match(const Eam& probe) const {  // eam.cpp:118-129
    check_probe(probe);
    moe_match m{};
    std::uint8_t found = 0;
    throw_on(moe_eamc_match(h_, probe.data(), 1, &m, &found));
    if (!found) return std::nullopt;
    return EamcMatch{static_cast<std::size_t>(m.index), m.seq, m.distance};
  }
  // Batched Eamc::match over [n][L][E] probes.
  std::vector<moe_match> match_batch(const std::uint64_t* probes, std::size_t n) const {
    std::vector<moe_match> out(n);
    throw_on(moe_eamc_match(h_, probes, n, out.data(), nullptr));
    return out;
  }
  std::vector<EamcMatch> match_within(const Eam& probe, double window) const {
    check_probe(probe);
    std::vector<moe_match> buf(std::max<std::size_t>(size(), 1));
    std::uint64_t n = 0;
    throw_on(moe_eamc_match_within(h_, probe.data(), window, buf.data(), buf.size(), &n));
    std::vector<EamcMatch> out;
    out.reserve(n);
    for (std::uint64_t i = 0; i < n; ++i)
      out.push_back({static_cast<std::size_t>(buf[i].index), buf[i].seq, buf[i].distance});
    return out;
  }
  std::optional<Eam> insert(Eam eam) {  // eam.cpp:152-178
    if (!(eam.shape() == shape_)) throw std::invalid_argument("Eamc::insert: shape mismatch");
    Eam evicted(shape_, EamKind::request, phase());
    std::int64_t slot = -1;
    throw_on(moe_eamc_insert(h_, eam.data(), static_cast<moe_eam_kind>(eam.kind()),
                             static_cast<moe_phase>(eam.phase()), &slot, evicted.data()));
    if (slot < 0) return std::nullopt;
    return evicted;
  }
  void save(const std::filesystem::path& p) const { throw_on(moe_eamc_save(h_, p.c_str())); }
  static Eamc load(const std::filesystem::path& p, int device = 0) {
    moe_eamc* h = nullptr;
    throw_on(moe_eamc_load(p.c_str(), nullptr, device, &h));
    return Eamc(h);
  }
  static Eamc load(const std::filesystem::path& p, const ModelShape& expected, int device = 0) {
    moe_eamc* h = nullptr;
    const moe_shape s = expected.c();
    throw_on(moe_eamc_load(p.c_str(), &s, device, &h));
    return Eamc(h);
  }
  moe_eamc* handle() const { return h_; }

 private:
  struct Info {
    moe_shape shape;
    int phase;
    std::uint64_t capacity, size, next_seq;
    int cb;
  };
  explicit Eamc(moe_eamc* h) : h_(h) {
    const Info i = info();
    shape_ = ModelShape{i.shape.n_layers, i.shape.n_experts_per_layer, i.shape.top_k};
  }
  Info info() const {
    Info i{};
    throw_on(moe_eamc_info(h_, &i.shape, &i.phase, &i.capacity, &i.size, &i.next_seq, &i.cb));
    return i;
  }
  void check_probe(const Eam& p) const {  // eam.cpp:113-116
    if (!(p.shape() == shape_)) throw std::invalid_argument("Eamc: probe shape mismatch");
  }
  ModelShape shape_;
  moe_eamc* h_ = nullptr;
};

inline std::uint64_t eamc_capacity_bound(const ModelShape& s, double similarity) {
  const moe_shape c = s.c();
  std::uint64_t v = 0;
  throw_on(moe_eamc_capacity_bound(&c, similarity, &v));
  return v;
}

// ------------------------------------------------------------- policy.hpp
inline constexpr double kEpsilon = 1e-4;
inline constexpr double kMaxPriority = std::numeric_limits<double>::infinity();
inline constexpr double kMatchWindow = 0.01;

struct PrefetchCandidate {
  ExpertId expert;
  double priority = 0.0;
  bool operator==(const PrefetchCandidate&) const = default;
};

inline std::vector<PrefetchCandidate> prefetch_priorities(const Eam& cur, const Eamc& eamc,
                                                          std::uint32_t current_layer,
                                                          bool apply_floor_filter = false) {
  std::vector<moe_candidate> buf(std::max<std::uint64_t>(cur.shape().total_experts(), 1));
  std::uint64_t n = 0;
  throw_on(moe_prefetch_priorities(eamc.handle(), cur.data(), current_layer,
                                   apply_floor_filter ? 1 : 0, buf.data(), buf.size(), &n));
  std::vector<PrefetchCandidate> out;
  out.reserve(n);
  for (std::uint64_t i = 0; i < n; ++i)
    out.push_back({ExpertId{buf[i].layer_idx, buf[i].expert_idx}, buf[i].priority});
  return out;
}

inline double cache_priority(const Eam& request_eam, const ExpertId& e) {
  const moe_shape s = request_eam.shape().c();
  double p = 0.0;
  throw_on(moe_cache_priority(&s, request_eam.data(), e.layer_idx, e.expert_idx, &p));
  return p;
}

struct SlotView {
  std::size_t slot = 0;
  ExpertId occupant;
  bool prefetch_protected = false;
  bool pinned = false;
};

inline std::optional<std::size_t> select_eviction_victim(std::span<const SlotView> slots,
                                                         const Eam& request_eam) {
  std::vector<moe_slot_view> v(slots.size());
  for (std::size_t i = 0; i < slots.size(); ++i)
    v[i] = moe_slot_view{slots[i].slot, slots[i].occupant.layer_idx, slots[i].occupant.expert_idx,
                         static_cast<std::uint8_t>(slots[i].prefetch_protected),
                         static_cast<std::uint8_t>(slots[i].pinned), {}};
  const moe_shape s = request_eam.shape().c();
  std::int64_t victim = -1;
  throw_on(moe_select_eviction_victim(&s, request_eam.data(), v.data(), v.size(), &victim));
  if (victim < 0) return std::nullopt;
  return static_cast<std::size_t>(victim);
}

}  // namespace moesim_b200
