// The three hot-path functions of the reference's policy.hpp (policy.hpp:82-106)
// over the C ABI of libmoe_eamc.so.  Everything else policy.hpp declares
// (TransferQueue, baselines, priority_reset_on_event, ...) stays the
// integrator's host code: the reference's policy.o is linked with these three
// symbols weakened (objcopy --weaken-symbol, oracle/Makefile `dropin`), so the
// linker binds the definitions below.
#include "moesim/policy.hpp"

#include <vector>

#include "dropin_common.hpp"
#include "moe_eamc.h"

namespace moesim {

using dropin::check;
using dropin::to_c;

// policy.cpp:88-126: match_within(cur, 0.01) -> aggregate -> per-row ratios
// x proximity, sorted (priority desc, ExpertId asc); one device pipeline
// (moe_prefetch_priorities), no floor filter (the engine applies its own,
// engine.cpp:663-668).
std::vector<PrefetchCandidate> prefetch_priorities(const Eam& cur_eam, const Eamc& eamc,
                                                   std::uint32_t current_layer) {
  const ModelShape& shape = cur_eam.shape();
  if (current_layer >= shape.n_layers)
    throw std::out_of_range("prefetch_priorities: current_layer out of range");
  if (eamc.empty()) return {};
  if (!(shape == eamc.shape())) throw std::invalid_argument("Eamc: probe shape mismatch");
  const std::uint64_t cap =
      std::uint64_t{shape.n_layers - current_layer - 1} * shape.n_experts_per_layer;
  std::vector<moe_candidate> buf(cap);
  std::uint64_t n = 0;
  check(moe_prefetch_priorities(eamc.handle(), cur_eam.counts().data(), current_layer, 0,
                                buf.data(), cap, &n));
  std::vector<PrefetchCandidate> out;
  out.reserve(n);
  for (std::uint64_t i = 0; i < n; ++i)
    out.push_back({ExpertId{buf[i].layer_idx, buf[i].expert_idx}, buf[i].priority});
  return out;
}

// policy.cpp:128-141
double cache_priority(const Eam& request_eam, const ExpertId& expert) {
  const moe_shape s = to_c(request_eam.shape());
  double p = 0.0;
  check(moe_cache_priority(&s, request_eam.counts().data(), expert.layer_idx, expert.expert_idx,
                           &p));
  return p;
}

// policy.cpp:143-159
std::optional<std::size_t> select_eviction_victim(std::span<const SlotView> slots,
                                                  const Eam& request_eam) {
  std::vector<moe_slot_view> views(slots.size());
  for (std::size_t i = 0; i < slots.size(); ++i) {
    views[i].slot = slots[i].slot;
    views[i].layer_idx = slots[i].occupant.layer_idx;
    views[i].expert_idx = slots[i].occupant.expert_idx;
    views[i].prefetch_protected = slots[i].prefetch_protected ? 1 : 0;
    views[i].pinned = slots[i].pinned ? 1 : 0;
  }
  const moe_shape s = to_c(request_eam.shape());
  std::int64_t victim = -1;
  check(moe_select_eviction_victim(&s, request_eam.counts().data(), views.data(), views.size(),
                                   &victim));
  if (victim < 0) return std::nullopt;
  return static_cast<std::size_t>(victim);
}

}  // namespace moesim
