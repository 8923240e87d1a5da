// Definitions behind include/moesim_dropin/moesim/eam.hpp: the reference's
// Eam / Eamc / eam_distance surface (eam.hpp:14-121) over the C ABI of
// libmoe_eamc.so. Replaces core/src/eam.cpp at link time.
#include "moesim/eam.hpp"

#include <cmath>
#include <cstdlib>
#include <utility>

#include "dropin_common.hpp"
#include "moe_eamc.h"

namespace {
// Device bring-up at program start (as an integrating engine would do when it
// loads its policy library), so the first decision does not pay for CUDA
// context creation.  Failure is ignored here: every later call reports it.
const bool g_warm = [] {
  (void)moe_device_warmup(moesim::dropin::device());
  return true;
}();
}  // namespace

namespace moesim {

using dropin::check;
using dropin::to_c;

const char* to_string(EamKind k) { return k == EamKind::iteration ? "iteration" : "request"; }
const char* to_string(Phase p) { return p == Phase::prefill ? "prefill" : "decode"; }

// ------------------------------------------------------------------- Eam
// eam.cpp:20-68. Host value type; semantics (validation order, messages,
// no mutation on a rejected record) as the reference.
Eam::Eam(ModelShape shape, EamKind kind, Phase phase) : shape_(shape), kind_(kind), phase_(phase) {
  shape_.validate();
  counts_.assign(shape_.total_experts(), 0);
}

std::uint64_t Eam::at(std::uint32_t layer, std::uint32_t expert) const {
  return counts_[std::uint64_t{layer} * shape_.n_experts_per_layer + expert];
}

std::uint64_t Eam::row_sum(std::uint32_t layer) const {
  std::uint64_t total = 0;
  for (const std::uint64_t c : row(layer)) total += c;
  return total;
}

std::span<const std::uint64_t> Eam::row(std::uint32_t layer) const {
  return {counts_.data() + std::size_t{layer} * shape_.n_experts_per_layer,
          shape_.n_experts_per_layer};
}

void Eam::record(const RoutingEvent& event) {
  if (event.layer_idx >= shape_.n_layers)
    throw std::out_of_range("Eam::record: layer index out of range");
  for (const ExpertAssignment& a : event.assignments)
    if (a.expert_idx >= shape_.n_experts_per_layer)
      throw std::out_of_range("Eam::record: expert index out of range");
  std::uint64_t* row_base = counts_.data() + std::size_t{event.layer_idx} * shape_.n_experts_per_layer;
  for (const ExpertAssignment& a : event.assignments) row_base[a.expert_idx] += a.token_count;
}

void Eam::accumulate(const Eam& other) {
  if (!(shape_ == other.shape_)) throw std::invalid_argument("Eam::accumulate: shape mismatch");
  if (phase_ != other.phase_) throw std::invalid_argument("Eam::accumulate: phase mismatch");
  for (std::size_t i = 0; i < counts_.size(); ++i) counts_[i] += other.counts_[i];
}

void Eam::reset() { std::fill(counts_.begin(), counts_.end(), 0); }

void Eam::set(std::uint32_t layer, std::uint32_t expert, std::uint64_t count) {
  if (layer >= shape_.n_layers || expert >= shape_.n_experts_per_layer)
    throw std::out_of_range("Eam::set: index out of range");
  counts_[std::size_t{layer} * shape_.n_experts_per_layer + expert] = count;
}

double eam_distance(const Eam& a, const Eam& b) {
  if (!(a.shape() == b.shape())) throw std::invalid_argument("eam_distance: shape mismatch");
  const moe_shape s = to_c(a.shape());
  double d = 0.0;
  check(moe_eam_distance(&s, a.counts().data(), b.counts().data(), &d));
  return d;
}

// ------------------------------------------------------------------ Eamc
Eamc::Eamc(ModelShape shape, Phase phase, std::size_t capacity)
    : shape_(shape), phase_(phase), capacity_(capacity) {
  shape_.validate();
  if (capacity_ < 1) throw std::invalid_argument("Eamc: capacity must be >= 1");
  const moe_shape s = to_c(shape_);
  const moe_phase ph = phase == Phase::prefill ? MOE_PHASE_PREFILL : MOE_PHASE_DECODE;
  const std::vector<int> shards = dropin::shard_devices();
  if (shards.size() > 1 && capacity_ >= shards.size())
    check(moe_eamc_create_sharded(&s, ph, capacity_, 0, (int)shards.size(), shards.data(), &h_));
  else
    check(moe_eamc_create(&s, ph, capacity_, 0, dropin::device(), &h_));
}

Eamc::Eamc(moe_eamc* h) : h_(h) {
  moe_shape s{};
  int phase = 0, cb = 0;
  uint64_t cap = 0, size = 0, next = 0;
  check(moe_eamc_info(h_, &s, &phase, &cap, &size, &next, &cb));
  shape_ = ModelShape{s.n_layers, s.n_experts_per_layer, s.top_k};
  phase_ = phase == MOE_PHASE_PREFILL ? Phase::prefill : Phase::decode;
  capacity_ = cap;
  size_ = size;
}

Eamc::Eamc(const Eamc& other)
    : shape_(other.shape_), phase_(other.phase_), capacity_(other.capacity_),
      size_(other.size_), host_(other.host_) {
  check(moe_eamc_clone(other.h_, &h_));
}

Eamc::Eamc(Eamc&& other) noexcept
    : shape_(other.shape_), phase_(other.phase_), capacity_(other.capacity_),
      size_(other.size_), h_(std::exchange(other.h_, nullptr)), host_(std::move(other.host_)) {
  other.size_ = 0;
}

Eamc& Eamc::operator=(const Eamc& other) {
  if (this != &other) *this = Eamc(other);
  return *this;
}

Eamc& Eamc::operator=(Eamc&& other) noexcept {
  if (this != &other) {
    if (h_) moe_eamc_destroy(h_);
    shape_ = other.shape_;
    phase_ = other.phase_;
    capacity_ = other.capacity_;
    size_ = std::exchange(other.size_, 0);
    h_ = std::exchange(other.h_, nullptr);
    host_ = std::move(other.host_);
  }
  return *this;
}

Eamc::~Eamc() {
  if (h_) moe_eamc_destroy(h_);
}

void Eamc::check_probe(const Eam& probe) const {
  if (!(probe.shape() == shape_)) throw std::invalid_argument("Eamc: probe shape mismatch");
}

const Eam& Eamc::entry(std::size_t index) const {
  if (index >= size_) throw std::out_of_range("Eamc::entry: index out of range");
  if (host_.size() < capacity_) host_.resize(capacity_);
  std::optional<Eam>& slot = host_[index];
  if (!slot) {
    Eam e(shape_, EamKind::request, phase_);
    check(moe_eamc_entry(h_, index, e.counts_.data(), nullptr));
    slot.emplace(std::move(e));
  }
  return *slot;
}

std::uint64_t Eamc::entry_seq(std::size_t index) const {
  std::uint64_t seq = 0;
  check(moe_eamc_entry(h_, index, nullptr, &seq));
  return seq;
}

std::optional<EamcMatch> Eamc::match(const Eam& probe) const {
  check_probe(probe);
  moe_match m{};
  std::uint8_t found = 0;
  check(moe_eamc_match(h_, probe.counts().data(), 1, &m, &found));
  if (!found) return std::nullopt;
  return EamcMatch{static_cast<std::size_t>(m.index), m.seq, m.distance};
}

std::vector<EamcMatch> Eamc::match_within(const Eam& probe, double window) const {
  check_probe(probe);
  std::vector<moe_match> buf(size_);
  std::uint64_t n = 0;
  check(moe_eamc_match_within(h_, probe.counts().data(), window, buf.data(), buf.size(), &n));
  std::vector<EamcMatch> out;
  out.reserve(n);
  for (std::uint64_t i = 0; i < n; ++i)
    out.push_back({static_cast<std::size_t>(buf[i].index), buf[i].seq, buf[i].distance});
  return out;
}

std::optional<Eam> Eamc::insert(Eam eam) {
  // eam.cpp:153-158 validation order: shape, then kind and phase (in the ABI)
  if (!(eam.shape() == shape_)) throw std::invalid_argument("Eamc::insert: shape mismatch");
  std::int64_t slot = -1;
  Eam evicted(shape_, EamKind::request, phase_);
  check(moe_eamc_insert(h_, eam.counts().data(),
                        eam.kind() == EamKind::request ? MOE_KIND_REQUEST : MOE_KIND_ITERATION,
                        eam.phase() == Phase::prefill ? MOE_PHASE_PREFILL : MOE_PHASE_DECODE,
                        &slot, evicted.counts_.data()));
  if (slot < 0) {
    ++size_;
    return std::nullopt;
  }
  if (static_cast<std::size_t>(slot) < host_.size()) host_[slot].reset();
  return evicted;
}

void Eamc::save(const std::filesystem::path& path) const {
  check(moe_eamc_save(h_, path.string().c_str()));
}

namespace {
moe_eamc* load_handle(const std::filesystem::path& path, const moe_shape* expected) {
  moe_eamc* h = nullptr;
  const std::vector<int> shards = dropin::shard_devices();
  if (shards.size() > 1)
    check(moe_eamc_load_sharded(path.string().c_str(), expected, (int)shards.size(),
                                shards.data(), &h));
  else
    check(moe_eamc_load(path.string().c_str(), expected, dropin::device(), &h));
  return h;
}
}  // namespace

Eamc Eamc::load(const std::filesystem::path& path) { return Eamc(load_handle(path, nullptr)); }

Eamc Eamc::load(const std::filesystem::path& path, const ModelShape& expected) {
  const moe_shape s = to_c(expected);
  return Eamc(load_handle(path, &s));
}

std::uint64_t eamc_capacity_bound(const ModelShape& shape, double similarity) {
  shape.validate();
  const moe_shape s = to_c(shape);
  std::uint64_t out = 0;
  check(moe_eamc_capacity_bound(&s, similarity, &out));
  return out;
}

}  // namespace moesim
