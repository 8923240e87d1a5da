// abi.cu -- the C ABI of include/moe_eamc.h on top of the sm_100a kernels.
//
// Host code here only marshals buffers, validates arguments the way the
// reference does (and returns the status its exception maps to), sizes the
// launch geometry and sequences kernels.  Every number the path produces
// (counts, norms, distances, argmins, windows, aggregates, priorities,
// orders, victims, histograms) is computed on the GPU.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <atomic>
#include <chrono>

#include "abi_internal.hpp"

namespace moe::abi {

namespace {
thread_local std::string g_err;
}

moe_status fail(moe_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

const char* last_error() { return g_err.c_str(); }

}  // namespace moe::abi

using namespace moe::abi;

moe::abi::HandleLock::HandleLock(const moe_eamc* h) {
  if (h) {
    m = &const_cast<moe_eamc*>(h)->mu;
    m->lock();
  }
}

namespace {

constexpr uint32_t kBucketCap = 256;  // early tiles push before the shared threshold tightens

// Grow the device collection to hold `need` entries (<= capacity).
moe_status ensure_alloc(moe_eamc* h, uint64_t need) {
  DevColl& c = h->c;
  if (need <= c.cap) return MOE_OK;
  uint64_t nc = std::max<uint64_t>(need, std::min<uint64_t>(h->capacity, std::max<uint64_t>(c.cap * 2, 1024)));
  nc = std::min<uint64_t>(std::max(nc, need), h->capacity);
  const uint64_t LR = (uint64_t)c.L * c.RB;
  uint8_t* counts = nullptr;
  float* ibT = nullptr;
  double* sqb = nullptr;
  uint64_t* seq = nullptr;
  __half* nrm = nullptr;
  uint64_t* zmask = nullptr;
  if (c.Kp) {
    CK(cudaMalloc(&nrm, (size_t)nc * c.Kp * sizeof(__half)));
    CK(cudaMalloc(&zmask, (size_t)nc * sizeof(uint64_t)));
    if (c.size) {
      CK(cudaMemcpyAsync(nrm, c.nrm, (size_t)c.size * c.Kp * sizeof(__half),
                         cudaMemcpyDeviceToDevice, h->st));
      CK(cudaMemcpyAsync(zmask, c.zmask, (size_t)c.size * 8, cudaMemcpyDeviceToDevice, h->st));
    }
  }
  // +kNT entries of slack so TMA boxes of the last tile stay in-bounds
  CK(cudaMalloc(&counts, (nc + moe::kNT) * LR));
  CK(cudaMalloc(&ibT, (size_t)c.L * nc * sizeof(float)));
  CK(cudaMalloc(&sqb, (size_t)nc * c.L * sizeof(double)));
  CK(cudaMalloc(&seq, (size_t)nc * sizeof(uint64_t)));
  CK(cudaMemsetAsync(counts, 0, (nc + moe::kNT) * LR, h->st));
  if (c.size) {
    CK(cudaMemcpyAsync(counts, c.counts, (size_t)c.size * LR, cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpy2DAsync(ibT, nc * sizeof(float), c.ibT, c.cap * sizeof(float),
                         (size_t)c.size * sizeof(float), c.L, cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpyAsync(sqb, c.sqb, (size_t)c.size * c.L * sizeof(double),
                       cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpyAsync(seq, c.seq, (size_t)c.size * sizeof(uint64_t), cudaMemcpyDeviceToDevice,
                       h->st));
  }
  CK(cudaStreamSynchronize(h->st));
  if (c.counts) cudaFree(c.counts);
  if (c.ibT) cudaFree(c.ibT);
  if (c.sqb) cudaFree(c.sqb);
  if (c.seq) cudaFree(c.seq);
  if (c.nrm) cudaFree(c.nrm);
  if (c.zmask) cudaFree(c.zmask);
  c.counts = counts;
  c.ibT = ibT;
  c.sqb = sqb;
  c.seq = seq;
  c.nrm = nrm;
  c.zmask = zmask;
  c.cap = nc;
  return MOE_OK;
}

uint64_t width_max(int cb) { return cb == 1 ? 255ull : cb == 2 ? 65535ull : 0xffffffffull; }

// Re-encode the collection with cb_new-byte counts (2 or 4).
moe_status widen(moe_eamc* h, int cb_new) {
  DevColl& c = h->c;
  ++h->version;
  if (cb_new <= c.cb) return MOE_OK;
  const uint32_t RB2 = row_bytes(c.E, cb_new);
  const uint64_t rows = c.cap ? (c.cap + moe::kNT) * c.L : 0;
  if (c.counts) {
    uint8_t* nc = nullptr;
    CK(cudaMalloc(&nc, rows * RB2));
    CK(moe::launch_widen(c.counts, nc, rows, c.RB, RB2, c.cb, cb_new, h->st));
    CK(cudaStreamSynchronize(h->st));
    cudaFree(c.counts);
    c.counts = nc;
  }
  c.cb = cb_new;
  c.RB = RB2;
  c.C = RB2 / 16;
  return MOE_OK;
}

// The outcome of a packing pass whose largest unrepresentable count (or ~0 for
// a row with sum c^2 >= 2^53, see k_prep) is mx: widen the collection to the
// width mx needs, or MOE_ERR_OVERFLOW when no width represents it exactly --
// the reference's fp64 sums are exact only while every row's sum of squares
// is below 2^53 (eam.cpp:75-87), and past that bound this library refuses
// rather than answer differently.
moe_status widen_for(moe_eamc* h, uint64_t mx) {
  if (mx > 0xffffffffull)
    return fail(MOE_ERR_OVERFLOW,
                "count %s: a row's sum of squared counts reaches 2^53, beyond the range where "
                "the reference's fp64 arithmetic (eam.cpp:75-87) is exact",
                mx == ~0ull ? "too large" : "exceeds 2^32-1");
  return widen(h, mx <= 65535ull ? 2 : 4);
}

// Exact-integer tensor-core screen for small batches (MOE_I8=0 disables,
// MOE_I8=1 forces it for any batch size it supports).
bool use_i8(const moe_eamc* h, uint64_t Q) {
  if (!moe::i8_supported(h->c)) return false;
  if (const char* e = getenv("MOE_I8")) {
    if (e[0] == '0') return false;
    if (e[0] == '1') return true;
  }
  // one 128-row block-diagonal M tile holds 128/R probes; up to three M
  // tiles the i8 screen still beats the fp16 one (its M tiles share each
  // entry tile through L2; measured at P=2^20, L=12: Q=16 0.38 vs 0.73 ms,
  // Q=24 0.51 vs 0.65 ms, Q=32 0.70 vs 0.63 ms)
  uint32_t R = 1;
  while (R < h->c.L) R <<= 1;
  return Q <= 3 * (128 / R);
}

// Tensor-core screen for probe batches that fill its 128-row M tile
// (MOE_TC=0 disables it, MOE_TC=1 forces it for any batch size).
bool use_tc(const moe_eamc* h, uint64_t Q) {
  if (!h->c.Kp) return false;
  if (const char* e = getenv("MOE_TC")) {
    if (e[0] == '0') return false;
    if (e[0] == '1') return true;
  }
  if (use_i8(h, Q)) return false;
  if (Q >= 8) return true;
  // small batches take the SIMT screen unless its tiles do not fit the shape
  MatchGeom g;
  return !moe::plan_match(h->c, h->n_sm, 0, 1, &g);
}

// Fold a completed event set into the per-kernel totals.
moe_status prof_collect(moe_eamc* h, moe_eamc::EvSet& es) {
  if (!es.pending) return MOE_OK;
  CK(cudaEventSynchronize(es.ev[4]));
  float t0 = 0.f, t1 = 0.f, t2 = 0.f;
  CK(cudaEventElapsedTime(&t0, es.ev[0], es.ev[1]));
  CK(cudaEventElapsedTime(&t1, es.ev[2], es.ev[3]));
  CK(cudaEventElapsedTime(&t2, es.ev[3], es.ev[4]));
  h->ms[0] += t0;
  h->ms[1] += t1;
  h->ms[2] += t2;
  h->calls[0]++;
  h->calls[1]++;
  h->calls[2]++;
  es.pending = false;
  return MOE_OK;
}

// Pick the event set for the next matching call (collecting whatever it held).
moe_status prof_begin(moe_eamc* h) {
  if (!h->prof) return MOE_OK;
  moe_eamc::EvSet& es = h->ring[h->ring_i];
  h->ring_i = (h->ring_i + 1) % h->ring.size();
  CKS(prof_collect(h, es));
  es.pending = true;
  h->ev = es.ev;
  return MOE_OK;
}

// Launch the packing of n probes (device source) at the collection's current
// width; *dmax (device) receives the largest count.  No synchronisation.
moe_status launch_probe_prep(moe_eamc* h, const void* dsrc, int src_bytes, uint64_t n,
                             cudaStream_t st, DevProbes* pr,
                             moe::MatchInit init = moe::MatchInit{}, bool alias_ok = false) {
  DevColl& c = h->c;
  const uint64_t LR = (uint64_t)c.L * c.RB;
  // A u8 device source already in the storage layout (RB == E) is used as the
  // packed probe rows directly (no copy) when the caller keeps it alive for
  // the whole pipeline; the condition implies launch_prep's u8 fast path.
  const bool alias = alias_ok && src_bytes == 1 && c.cb == 1 && c.RB == c.E && (c.E & 3) == 0 &&
                     c.E <= 256 && (reinterpret_cast<uintptr_t>(dsrc) & 15) == 0;
  CK(h->packed.ensure(n * LR + 16));
  CK(h->ia.ensure(n * c.L * sizeof(float)));
  CK(h->sqa.ensure(n * c.L * sizeof(double)));
  CK(h->small.ensure(256));
  CK(h->pin.ensure(256));
  unsigned long long* dmax = h->small.as<unsigned long long>();
  __half* nrm = nullptr;
  uint64_t* zq = nullptr;
  const bool tc = c.Kp && use_tc(h, n);
  if (tc) {
    CK(h->nrm.ensure(n * c.Kp * sizeof(__half)));
    nrm = h->nrm.as<__half>();
  }
  if (tc || (c.Kp && use_i8(h, n))) {
    CK(h->zq.ensure(n * 8));
    zq = h->zq.as<uint64_t>();
  }
  CK(h->wide.ensure(n));
  if (h->prof) CK(cudaEventRecord(h->ev[0], st));
  CK(moe::launch_prep(dsrc, src_bytes, n, c.L, c.E, c.RB, c.cb,
                      alias ? nullptr : h->packed.as<uint8_t>(), h->ia.as<float>(),
                      h->sqa.as<double>(), nullptr, 0, 0, dmax, nrm, c.Kp, zq,
                      h->wide.as<uint8_t>(), st, init));
  if (h->prof) CK(cudaEventRecord(h->ev[1], st));
  pr->Q = (uint32_t)n;
  pr->packed = alias ? static_cast<uint8_t*>(const_cast<void*>(dsrc)) : h->packed.as<uint8_t>();
  pr->ia = h->ia.as<float>();
  pr->sqa = h->sqa.as<double>();
  pr->nrm = nrm;
  pr->zmask = zq;
  pr->wide = h->wide.as<uint8_t>();
  return MOE_OK;
}

// Width check after the caller's synchronisation: widen if needed.  Returns
// true when the packed probes are exact (nothing to redo).
moe_status check_width(moe_eamc* h, uint64_t mx, bool* ok) {
  *ok = mx <= width_max(h->c.cb);
  if (*ok) return MOE_OK;
  return widen_for(h, mx);
}

const void* stage_source(moe_eamc* h, const void* src, int src_bytes, uint64_t n, bool src_device,
                         cudaStream_t st, moe_status* status) {
  *status = MOE_OK;
  if (src_device) return src;
  const uint64_t bytes = n * (uint64_t)h->c.L * h->c.E * src_bytes;
  cudaError_t e = h->raw.ensure(bytes);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h->raw.p, src, bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) *status = fail(MOE_ERR_CUDA, "probe upload: %s", cudaGetErrorString(e));
  return h->raw.p;
}

// H2D (or D2D) + pack probes, synchronously width-checked.
moe_status prep_probes(moe_eamc* h, const void* src, int src_bytes, uint64_t n, bool src_device,
                       cudaStream_t st, DevProbes* pr) {
  moe_status ss;
  const void* dsrc = stage_source(h, src, src_bytes, n, src_device, st, &ss);
  CKS(ss);
  for (;;) {
    const bool prof = h->prof;
    h->prof = false;  // standalone packing is not part of the matcher's timing
    const moe_status ps = launch_probe_prep(h, dsrc, src_bytes, n, st, pr);
    h->prof = prof;
    CKS(ps);
    CK(cudaMemcpyAsync(h->pin.p, h->small.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    bool ok = false;
    CKS(check_width(h, *h->pin.as<unsigned long long>(), &ok));
    if (ok) return MOE_OK;
  }
}

uint32_t pick_qt(uint64_t Q) {
  if (const char* e = getenv("MOE_QT")) {
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) return (uint32_t)v;
  }
  if (Q <= 1) return 1;
  if (Q <= 2) return 2;
  if (Q <= 4) return 4;
  if (Q <= 64) return 8;
  return 16;
}

struct Plan {
  MatchGeom g;
  CUtensorMap map;
};

moe_status make_plan(moe_eamc* h, int mode, uint32_t QT, Plan* p) {
  if (!moe::plan_match(h->c, h->n_sm, mode, QT, &p->g))
    return fail(MOE_ERR_INVALID_ARGUMENT, "shape %ux%u does not fit the matcher's shared memory",
                h->c.L, h->c.E);
  CK(moe::encode_tmap(h->c, p->g.G, &p->map));
  return MOE_OK;
}

// Scratch of one match pipeline for Q probes (allocated before the probe prep
// that initialises it).
moe_status match_work(moe_eamc* h, uint64_t Q, MatchWork* wout) {
  CK(h->T.ensure(Q * 4));
  CK(h->bcnt.ensure(Q * 4));
  CK(h->bucket.ensure(Q * kBucketCap * sizeof(uint2)));
  CK(h->over_list.ensure(Q * 4));
  CK(h->small.ensure(256));
  CK(h->pin.ensure(256));
  MatchWork w;
  w.T = h->T.as<uint32_t>();
  w.bcnt = h->bcnt.as<uint32_t>();
  w.bucket = h->bucket.as<uint2>();
  w.bcap = kBucketCap;
  w.over_list = h->over_list.as<uint32_t>();
  w.over_n = h->small.as<uint32_t>() + 4;
  *wout = w;
  return MOE_OK;
}

// Exact argmin for the probes in qlist[0..n) (or *nq_dev of them): the TMA
// matcher in exact mode where the shape fits its shared-memory tiles, else the
// warp-per-entry kernel.  chunk = probes per partials pass.
moe_status exact_pass(moe_eamc* h, const DevProbes& pr, const MatchWork& w0, const uint32_t* qlist,
                      uint32_t n, const uint32_t* T, moe_match* out, cudaStream_t st,
                      uint32_t chunk, const uint32_t* nq_dev = nullptr) {
  MatchWork w = w0;
  Plan pe;
  if (moe::plan_match(h->c, h->n_sm, 1, 1, &pe.g)) {
    CK(moe::encode_tmap(h->c, pe.g.G, &pe.map));
    w.part_chunk = chunk;
    CK(h->partials.ensure((size_t)chunk * pe.g.grid * sizeof(moe_match)));
    w.partials = h->partials.as<moe_match>();
    CK(moe::launch_exact(pe.map, h->c, pr, pe.g, w, qlist, n, T, out, st, nq_dev));
    return MOE_OK;
  }
  CK(h->partials.ensure((size_t)chunk * moe::exact_warp_blocks(h->n_sm) * sizeof(moe_match)));
  CK(moe::launch_exact_warp(h->c, pr, qlist, n, out, h->partials.as<moe_match>(), chunk, h->n_sm,
                            st, nq_dev));
  return MOE_OK;
}

// Screen + refine launches for packed probes (no synchronisation).  `inited`:
// the probe prep already initialised w's threshold / bucket counters
// (MatchInit); otherwise they are reset here.
moe_status launch_match(moe_eamc* h, const DevProbes& pr, moe_match* out, cudaStream_t st,
                        MatchWork* wout, bool inited = false) {
  const uint64_t Q = pr.Q;
  DevColl& c = h->c;
  MatchWork w;
  if (inited) {
    w = *wout;
  } else {
    CKS(match_work(h, Q, &w));
    CK(cudaMemsetAsync(w.T, 0x7f, Q * 4, st));  // 0x7f7f7f7f = 3.4e38f > any distance
    CK(cudaMemsetAsync(w.bcnt, 0, Q * 4, st));
    CK(cudaMemsetAsync(w.over_n, 0, 4, st));
  }
  const bool tc = pr.nrm != nullptr && moe::tc_supported(c);
  const bool i8 = !tc && pr.zmask != nullptr && use_i8(h, Q);
  w.eps2 = tc ? moe::tc_eps2(c.L, c.E, c.Kp) : moe::screen_eps2(c.L);
  if (h->prof) CK(cudaEventRecord(h->ev[2], st));
  if (c.size > 0) {
    if (tc) {
      CK(moe::launch_tc_screen(c, pr, w, h->n_sm, st));
    } else if (i8) {
      CK(h->bdiag.ensure(moe::i8_blockdiag_bytes(c, (uint32_t)Q)));
      CK(moe::launch_tci8_screen(c, pr, w, h->bdiag.as<uint8_t>(), h->n_sm, st));
    } else {
      // the largest probe tile whose shared-memory layout fits this shape
      uint32_t qt = pick_qt(Q);
      MatchGeom g;
      while (qt > 1 && !moe::plan_match(c, h->n_sm, 0, qt, &g)) qt >>= 1;
      Plan p;
      CKS(make_plan(h, 0, qt, &p));
      CK(moe::launch_screen(p.map, c, pr, p.g, w, st));
    }
  }
  if (h->prof) CK(cudaEventRecord(h->ev[3], st));
  CK(moe::launch_refine(c, pr, w, out, nullptr, nullptr, 0, st));
  if (h->prof) CK(cudaEventRecord(h->ev[4], st));
  *wout = w;
  return MOE_OK;
}

// Full matching pipeline.  Probe packing, screen and refine are launched back
// to back.  Synchronous mode (host API): ONE synchronisation then checks the
// probe count width (rare widening -> redo) and candidate-bucket overflow
// (rare -> exact pass).  Asynchronous mode (device API): nothing waits on the
// host -- the exact pass is launched device-gated on the overflow count, and
// probes whose counts exceed the storage width get the sentinel result
// {UINT64_MAX-1, UINT64_MAX, NaN}.  `out` is a device array; `pr` receives
// the packed probes for follow-up passes.
moe_status match_all(moe_eamc* h, const void* src, int src_bytes, uint64_t n, bool src_device,
                     moe_match* out, cudaStream_t st, DevProbes* pr, bool async = false,
                     cudaEvent_t after_prep = nullptr) {
  if (n == 0) return MOE_OK;
  moe_status ss;
  const void* dsrc = stage_source(h, src, src_bytes, n, src_device, st, &ss);
  CKS(ss);
  for (;;) {
    CKS(prof_begin(h));
    MatchWork w;
    CKS(match_work(h, n, &w));
    CKS(launch_probe_prep(h, dsrc, src_bytes, n, st, pr, moe::MatchInit{w.T, w.bcnt, w.over_n},
                          /*alias_ok=*/after_prep == nullptr));
    if (after_prep) CK(cudaEventRecord(after_prep, st));  // the source buffer may be reused
    CKS(launch_match(h, *pr, out, st, &w, /*inited=*/true));
    if (async) {
      if (h->c.size)
        CKS(exact_pass(h, *pr, w, w.over_list, (uint32_t)n, w.T, out, st,
                       (uint32_t)std::min<uint64_t>(n, 8192), w.over_n));
      return MOE_OK;
    }
    CK(cudaMemcpyAsync(h->pin.p, h->small.p, 32, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h->prof) CKS(prof_collect(h, h->ring[(h->ring_i + h->ring.size() - 1) % h->ring.size()]));
    bool ok = false;
    CKS(check_width(h, *h->pin.as<unsigned long long>(), &ok));
    if (!ok) continue;  // collection widened: redo with the wider packing
    const uint32_t n_over = h->pin.as<uint32_t>()[4];  // w.over_n = small + 16 B
    if (n_over) CKS(exact_pass(h, *pr, w, w.over_list, n_over, w.T, out, st, 1024));
    return MOE_OK;
  }
}

// Exact distance of one host probe to every entry (dist[p] in h->dist) and
// the minimum (*h->small @224) -- the single collection pass behind
// match_within and prefetch_priorities.  Asynchronous; the caller checks the
// probe width (dmax @0) after its synchronisation.
moe_status launch_exact_distances(moe_eamc* h, const uint64_t* probe, cudaStream_t st,
                                  DevProbes* pr) {
  moe_status ss;
  const void* dsrc = stage_source(h, probe, 8, 1, false, st, &ss);
  CKS(ss);
  const bool prof = h->prof;
  h->prof = false;
  ss = launch_probe_prep(h, dsrc, 8, 1, st, pr);
  h->prof = prof;
  CKS(ss);
  CK(h->dist.ensure((size_t)std::max<uint32_t>(h->c.size, 1) * sizeof(double)));
  CK(h->rsim.ensure((size_t)std::max<uint32_t>(h->c.size, 1) * h->c.L * sizeof(double)));
  unsigned long long* dmin = reinterpret_cast<unsigned long long*>(h->small.as<uint8_t>() + 224);
  CK(cudaMemsetAsync(dmin, 0xff, 8, st));  // > every distance bit pattern
  CK(moe::launch_exact_rows(h->c, *pr, 0, 0, h->c.L, h->rsim.as<double>(), h->dist.as<double>(),
                            dmin, h->n_sm, st));
  return MOE_OK;
}

// Compatibility wrapper used by the insert path: packed probes in hand.
moe_status match_packed(moe_eamc* h, const DevProbes& pr, moe_match* out, cudaStream_t st) {
  if (pr.Q == 0) return MOE_OK;
  MatchWork w;
  const bool prof = h->prof;
  h->prof = false;
  const moe_status ls = launch_match(h, pr, out, st, &w);
  h->prof = prof;
  CKS(ls);
  CK(cudaMemcpyAsync(h->pin.p, h->small.p, 32, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const uint32_t n_over = h->pin.as<uint32_t>()[4];  // w.over_n = small + 16 B
  if (n_over) CKS(exact_pass(h, pr, w, w.over_list, n_over, w.T, out, st, 1024));
  return MOE_OK;
}

inline uint64_t unpack_count(const uint8_t* row, uint32_t e, int cb) {
  return cb == 1 ? row[e]
         : cb == 2 ? reinterpret_cast<const uint16_t*>(row)[e]
                   : reinterpret_cast<const uint32_t*>(row)[e];
}

// Unpack one device entry to host u64 counts.
moe_status read_entry(moe_eamc* h, uint64_t slot, uint64_t* counts, uint64_t* seq) {
  DevColl& c = h->c;
  const uint64_t LR = (uint64_t)c.L * c.RB;
  std::vector<uint8_t> row(LR);
  if (counts) {
    CK(cudaMemcpy(row.data(), c.counts + slot * LR, LR, cudaMemcpyDeviceToHost));
    for (uint32_t l = 0; l < c.L; ++l)
      for (uint32_t e = 0; e < c.E; ++e)
        counts[(uint64_t)l * c.E + e] = unpack_count(row.data() + (size_t)l * c.RB, e, c.cb);
  }
  if (seq) CK(cudaMemcpy(seq, c.seq + slot, 8, cudaMemcpyDeviceToHost));
  return MOE_OK;
}

// Stage n EAMs (device raw) as packed rows in a private staging set.
struct Staged {
  DevBuf packed, ia, sqa, nrm, zmask;
  DevProbes pr;
};

moe_status stage_entries(moe_eamc* h, const void* dsrc, int src_bytes, uint64_t n, Staged* s) {
  DevColl& c = h->c;
  for (;;) {
    const uint64_t LR = (uint64_t)c.L * c.RB;
    CK(s->packed.ensure(n * LR + 16));
    CK(s->ia.ensure(n * c.L * 4));
    CK(s->sqa.ensure(n * c.L * 8));
    CK(h->small.ensure(256));
    CK(h->pin.ensure(256));
    unsigned long long* dmax = h->small.as<unsigned long long>();  // reset by launch_prep
    if (c.Kp) {
      CK(s->nrm.ensure(n * c.Kp * sizeof(__half)));
      CK(s->zmask.ensure(n * 8));
    }
    CK(moe::launch_prep(dsrc, src_bytes, n, c.L, c.E, c.RB, c.cb, s->packed.as<uint8_t>(),
                        s->ia.as<float>(), s->sqa.as<double>(), nullptr, 0, 0, dmax,
                        c.Kp ? s->nrm.as<__half>() : nullptr, c.Kp,
                        c.Kp ? s->zmask.as<uint64_t>() : nullptr, nullptr, h->st));
    CK(cudaMemcpyAsync(h->pin.p, dmax, 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    const uint64_t mx = *h->pin.as<unsigned long long>();
    if (mx <= width_max(c.cb)) break;
    CKS(widen_for(h, mx));
  }
  s->pr.Q = (uint32_t)n;
  s->pr.packed = s->packed.as<uint8_t>();
  s->pr.ia = s->ia.as<float>();
  s->pr.sqa = s->sqa.as<double>();
  s->pr.nrm = c.Kp ? s->nrm.as<__half>() : nullptr;
  s->pr.zmask = c.Kp ? s->zmask.as<uint64_t>() : nullptr;
  return MOE_OK;
}

// Sequential Eamc::insert semantics for a staged batch (K7 replay).
moe_status replay_staged(moe_eamc* h, Staged& s, int64_t* evicted_slots) {
  DevColl& c = h->c;
  ++h->version;
  const uint32_t n = s.pr.Q;
  uint32_t i = 0;
  // appends below capacity (eam.cpp:160-162)
  const uint64_t room = h->capacity - c.size;
  const uint32_t n_app = (uint32_t)std::min<uint64_t>(room, n);
  if (n_app) {
    CKS(ensure_alloc(h, c.size + n_app));
    CK(moe::launch_append_staged(c, s.pr, 0, n_app, c.size, h->st));
    std::vector<uint64_t> seqs(n_app);
    for (uint32_t k = 0; k < n_app; ++k) seqs[k] = h->next_seq + k;
    CK(cudaMemcpyAsync(c.seq + c.size, seqs.data(), n_app * 8, cudaMemcpyHostToDevice, h->st));
    CK(cudaStreamSynchronize(h->st));
    c.size += n_app;
    h->next_seq += n_app;
    if (evicted_slots)
      for (uint32_t k = 0; k < n_app; ++k) evicted_slots[k] = -1;
    i = n_app;
  }
  if (i == n) return MOE_OK;
  const uint32_t n_rep = n - i;
  CK(h->out.ensure((size_t)n * sizeof(moe_match)));
  moe_match* vic = h->out.as<moe_match>();
  const char* rs_env = getenv("MOE_REPLAY_STEPWISE");
  if (c.nrm && c.Kp && moe::tc_supported(c) && c.L <= 64 && c.size <= 16384 && n_rep >= 16 &&
      moe::replay_block_smem(c) <= 220 * 1024 && (uint64_t)c.L * c.RB <= 16384 &&
      !(rs_env && rs_env[0] == '1')) {
    // blocked replay: screen matrices on the tensor cores, the sequential
    // decisions in one CTA per block of steps (launch_replay_block)
    uint32_t B = 512;
    if (const char* e = getenv("MOE_REPLAY_BLOCK")) B = std::min(1024, std::max(16, atoi(e)));
    const uint32_t ldc = (c.size + 3) & ~3u, ldx = (B + 3) & ~3u;
    CK(h->rdc.ensure((size_t)B * ldc * 4));
    CK(h->rdx.ensure((size_t)B * ldx * 4));
    if (h->rocc.n < (size_t)c.size * 4) {
      CK(h->rocc.ensure((size_t)c.cap * 4));
      CK(cudaMemsetAsync(h->rocc.p, 0xff, h->rocc.n, h->st));
    }
    const float eps2 = moe::tc_eps2(c.L, c.E, c.Kp);
    unsigned long long* rprof = nullptr;
    if (getenv("MOE_REPLAY_PROF")) {
      CK(h->partials.ensure(64));
      rprof = h->partials.as<unsigned long long>();
      CK(cudaMemsetAsync(rprof, 0, 64, h->st));
    }
    MatchWork w;
    for (uint32_t b0 = i; b0 < n; b0 += B) {
      const uint32_t nb = std::min(B, n - b0);
      DevProbes xb;
      xb.Q = nb;
      xb.nrm = s.pr.nrm + (uint64_t)b0 * c.Kp;
      xb.zmask = s.pr.zmask + b0;
      CK(moe::launch_tc_screen(c, xb, w, h->n_sm, h->st, h->rdc.as<float>(), ldc));
      DevColl cx = c;
      cx.nrm = xb.nrm;
      cx.zmask = xb.zmask;
      cx.size = nb;
      cx.cap = nb;
      CK(moe::launch_tc_screen(cx, xb, w, h->n_sm, h->st, h->rdx.as<float>(), ldx));
      CK(moe::launch_replay_block(c, s.pr, b0, nb, h->rdc.as<float>(), ldc, h->rdx.as<float>(),
                                  ldx, eps2, h->rocc.as<int>(), h->next_seq + (b0 - i), vic + b0,
                                  h->st, rprof));
    }
    if (rprof) {  // MOE_REPLAY_PROF: phase cycles of the sequential kernel
      unsigned long long pc[6];
      CK(cudaMemcpy(pc, rprof, sizeof pc, cudaMemcpyDeviceToHost));
      fprintf(stderr, "replay phases (cycles/step): screen-min %.0f (row wait %.0f) band %.0f refine %.0f (warp1 %.0f) pick %.0f\n",
              pc[0] / (double)n_rep, pc[5] / (double)n_rep, pc[1] / (double)n_rep,
              pc[2] / (double)n_rep, pc[4] / (double)n_rep, pc[3] / (double)n_rep);
    }
    h->next_seq += n_rep;
    std::vector<moe_match> v(n_rep);
    CK(cudaMemcpyAsync(v.data(), vic + i, n_rep * sizeof(moe_match), cudaMemcpyDeviceToHost,
                       h->st));
    CK(cudaStreamSynchronize(h->st));
    if (evicted_slots)
      for (uint32_t j = 0; j < n_rep; ++j)
        evicted_slots[i + j] = (int64_t)(v[j].index - h->c.index_base);
    return MOE_OK;
  }
  // stepwise: at-capacity replacement steps, stream-ordered on the device; a
  // bucket overflow halts the remaining launched steps and is resolved exactly.
  CK(h->T.ensure(4));
  CK(h->bcnt.ensure(4));
  CK(h->bucket.ensure(kBucketCap * sizeof(uint2)));
  CK(h->small.ensure(256));
  CK(h->pin.ensure(256));
  int* halt = h->small.as<int>() + 16;
  CK(cudaMemsetAsync(halt, 0, 4, h->st));
  Plan p;
  CKS(make_plan(h, 0, 1, &p));
  MatchWork w;
  w.T = h->T.as<uint32_t>();
  w.bcnt = h->bcnt.as<uint32_t>();
  w.bucket = h->bucket.as<uint2>();
  w.bcap = kBucketCap;
  const uint64_t LR = (uint64_t)c.L * c.RB;
  const uint32_t kBatch = 256;
  uint32_t k = i;
  while (k < n) {
    const uint32_t kend = std::min(n, k + kBatch);
    for (uint32_t j = k; j < kend; ++j) {
      DevProbes one;
      one.Q = 1;
      one.packed = s.pr.packed + (uint64_t)j * LR;
      one.ia = s.pr.ia + (uint64_t)j * c.L;
      one.sqa = s.pr.sqa + (uint64_t)j * c.L;
      CK(cudaMemsetAsync(w.T, 0x7f, 4, h->st));
      CK(cudaMemsetAsync(w.bcnt, 0, 4, h->st));
      CK(moe::launch_screen(p.map, c, one, p.g, w, h->st));
      CK(moe::launch_refine(c, one, w, vic + j, halt, halt, j + 1, h->st));
      CK(moe::launch_replace(c, s.pr, j, vic + j, h->next_seq + (j - i), halt, h->st));
    }
    CK(cudaMemcpyAsync(h->pin.p, halt, 4, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    const int hv = *h->pin.as<int>();
    if (hv == 0) {
      k = kend;
      continue;
    }
    // step j0 overflowed its candidate bucket: resolve it with the exact
    // pass, apply the replacement, and resume after it.
    const uint32_t j0 = (uint32_t)hv - 1;
    CK(cudaMemsetAsync(halt, 0, 4, h->st));
    DevProbes one;
    one.Q = 1;
    one.packed = s.pr.packed + (uint64_t)j0 * LR;
    one.ia = s.pr.ia + (uint64_t)j0 * c.L;
    one.sqa = s.pr.sqa + (uint64_t)j0 * c.L;
    CK(cudaMemsetAsync(w.T, 0x7f, 4, h->st));
    CK(cudaMemsetAsync(w.bcnt, 0, 4, h->st));
    CK(moe::launch_screen(p.map, c, one, p.g, w, h->st));
    uint32_t* q0 = h->small.as<uint32_t>() + 32;
    CK(cudaMemsetAsync(q0, 0, 4, h->st));
    // exact argmin for probe 0 of `one`, written to vic[j0]
    CKS(exact_pass(h, one, w, q0, 1, w.T, vic + j0 - 0, h->st, 1));
    CK(moe::launch_replace(c, s.pr, j0, vic + j0, h->next_seq + (j0 - i), halt, h->st));
    CK(cudaStreamSynchronize(h->st));
    k = j0 + 1;
  }
  h->next_seq += n_rep;
  if (evicted_slots) {
    std::vector<moe_match> v(n_rep);
    CK(cudaMemcpy(v.data(), vic + i, n_rep * sizeof(moe_match), cudaMemcpyDeviceToHost));
    for (uint32_t j = 0; j < n_rep; ++j)
      evicted_slots[i + j] = (int64_t)(v[j].index - h->c.index_base);
  }
  return MOE_OK;
}

}  // namespace

// ---- shard-level internals used by the sharded facade (sharded.cu) --------
namespace moe::abi {

moe_status replace_slot(moe_eamc* h, const uint64_t* counts, uint64_t slot, uint64_t seq) {
  HandleLock hl_(h);
  DeviceGuard dg(h->device);
  if (slot >= h->c.size) return fail(MOE_ERR_OUT_OF_RANGE, "replace_slot: slot out of range");
  const uint64_t cells = (uint64_t)h->c.L * h->c.E;
  Staged s;
  CK(h->raw.ensure(cells * 8));
  CK(cudaMemcpyAsync(h->raw.p, counts, cells * 8, cudaMemcpyHostToDevice, h->st));
  CKS(stage_entries(h, h->raw.p, 8, 1, &s));
  CK(h->pin.ensure(256));
  moe_match* v = reinterpret_cast<moe_match*>(h->pin.as<uint8_t>() + 128);
  *v = moe_match{h->c.index_base + slot, 0, 0.0};
  CK(h->out.ensure(sizeof(moe_match)));
  CK(cudaMemcpyAsync(h->out.p, v, sizeof(moe_match), cudaMemcpyHostToDevice, h->st));
  ++h->version;
  CK(moe::launch_replace(h->c, s.pr, 0, h->out.as<moe_match>(), seq, nullptr, h->st));
  CK(cudaStreamSynchronize(h->st));
  return MOE_OK;
}

moe_status ensure_width(moe_eamc* h, uint64_t mx) {
  HandleLock hl_(h);
  DeviceGuard dg(h->device);
  if (mx <= width_max(h->c.cb)) return MOE_OK;
  return widen_for(h, mx);
}

moe_status window_list(moe_eamc* h, uint64_t dmin_bits, double window,
                       std::vector<moe::WinEntry>* v) {
  HandleLock hl_(h);
  DeviceGuard dg(h->device);
  v->clear();
  if (h->c.size == 0) return MOE_OK;
  CK(h->pin.ensure(256));
  CK(h->small.ensure(256));
  CK(h->wl.ensure((size_t)h->c.size * sizeof(moe::WinEntry)));
  uint64_t* hp = h->pin.as<uint64_t>();
  hp[0] = dmin_bits;
  hp[1] = 0;
  unsigned long long* dm = reinterpret_cast<unsigned long long*>(h->small.as<uint8_t>() + 232);
  uint32_t* wl_n = h->small.as<uint32_t>() + 60;
  CK(cudaMemcpyAsync(dm, hp, 16, cudaMemcpyHostToDevice, h->st));  // dmin and wl_n = 0
  CK(moe::launch_window_list(h->c, h->dist.as<double>(), dm, window, h->wl.as<moe::WinEntry>(),
                             wl_n, h->st));
  CK(cudaMemcpyAsync(hp + 4, wl_n, 4, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  const uint32_t n = *reinterpret_cast<uint32_t*>(hp + 4);
  v->resize(n);
  if (n) CK(cudaMemcpy(v->data(), h->wl.p, n * sizeof(moe::WinEntry), cudaMemcpyDeviceToHost));
  for (auto& w : *v) w.p += h->c.index_base;
  return MOE_OK;
}

}  // namespace moe::abi

// SMs held by resident decision servers per device (see server_run).
static std::atomic<int> g_srv_sms[64];

extern "C" {

static moe_status server_stop(moe_eamc* h);

int moe_abi_version(void) { return MOE_EAMC_ABI_VERSION; }

const char* moe_last_error(void) { return last_error(); }

int moe_host_threads(void) { return moe::host::pool_threads(); }

moe_status moe_device_info(int device, int* sm_count, int* cc_major, int* cc_minor,
                           size_t* l2_bytes) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    return fail(MOE_ERR_CUDA, "no CUDA device visible");
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  if (l2_bytes) *l2_bytes = (size_t)prop.l2CacheSize;
  return MOE_OK;
}

moe_status moe_device_warmup(int device) {
  int n_sm = 0;
  CKS(device_ok(device, &n_sm));
  DeviceGuard dg(device);
  CK(cudaFree(nullptr));
  return MOE_OK;
}

moe_status moe_eamc_create(const moe_shape* shape, moe_phase phase, uint64_t capacity,
                           int count_bytes, int device, moe_eamc** out) {
  if (!out) return fail(MOE_ERR_INVALID_ARGUMENT, "null out");
  *out = nullptr;
  CKS(check_shape(shape));
  if (capacity < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "Eamc: capacity must be >= 1");
  if (phase != MOE_PHASE_PREFILL && phase != MOE_PHASE_DECODE)
    return fail(MOE_ERR_INVALID_ARGUMENT, "bad phase");
  if (count_bytes == 0) count_bytes = 1;
  if (count_bytes != 1 && count_bytes != 2 && count_bytes != 4)
    return fail(MOE_ERR_INVALID_ARGUMENT, "count_bytes must be 0, 1, 2 or 4");
  int n_sm = 0;
  CKS(device_ok(device, &n_sm));
  DeviceGuard dg(device);
  auto* h = new moe_eamc();
  h->device = device;
  h->n_sm = n_sm;
  h->shape = *shape;
  h->phase = phase;
  h->capacity = capacity;
  h->c.L = shape->n_layers;
  h->c.E = shape->n_experts_per_layer;
  h->c.cb = count_bytes;
  h->c.RB = row_bytes(h->c.E, count_bytes);
  h->c.C = h->c.RB / 16;
  if (h->c.L <= 64) h->c.Kp = (h->c.L * h->c.E + 63) / 64 * 64;
  if (cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking) != cudaSuccess) {
    delete h;
    return fail(MOE_ERR_CUDA, "stream create failed");
  }
  *out = h;
  return MOE_OK;
}

moe_status moe_eamc_create_sharded(const moe_shape* shape, moe_phase phase, uint64_t capacity,
                                   int count_bytes, int n_shards, const int* device_ids,
                                   moe_eamc** out) {
  if (phase != MOE_PHASE_PREFILL && phase != MOE_PHASE_DECODE)
    return fail(MOE_ERR_INVALID_ARGUMENT, "bad phase");
  if (count_bytes != 0 && count_bytes != 1 && count_bytes != 2 && count_bytes != 4)
    return fail(MOE_ERR_INVALID_ARGUMENT, "count_bytes must be 0, 1, 2 or 4");
  return moe::abi::sh_create(shape, phase, capacity, count_bytes, n_shards, device_ids, out);
}

moe_status moe_eamc_load_sharded(const char* path, const moe_shape* expected, int n_shards,
                                 const int* device_ids, moe_eamc** out) {
  if (!out || !device_ids || n_shards < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "bad argument");
  moe_eamc* one = nullptr;
  CKS(moe_eamc_load(path, expected, device_ids[0], &one));
  if (one->capacity < (uint64_t)n_shards || n_shards == 1) {
    *out = one;
    return MOE_OK;
  }
  moe_eamc* h = nullptr;
  moe_status st = moe::abi::sh_create(&one->shape, (moe_phase)one->phase, one->capacity,
                                      one->c.cb, n_shards, device_ids, &h);
  const uint64_t cells = (uint64_t)one->c.L * one->c.E, n = one->c.size;
  std::vector<uint64_t> counts(n * cells), seqs(n);
  for (uint64_t i = 0; i < n && st == MOE_OK; ++i)
    st = moe_eamc_entry(one, i, counts.data() + i * cells, &seqs[i]);
  if (st == MOE_OK && n) st = moe_eamc_append(h, counts.data(), seqs.data(), n);
  if (st == MOE_OK) h->next_seq = one->next_seq;
  moe_eamc_destroy(one);
  if (st != MOE_OK) {
    moe_eamc_destroy(h);
    return st;
  }
  *out = h;
  return MOE_OK;
}

moe_status moe_eamc_shard_layout(const moe_eamc* h, int* n_shards, int* uses_nccl) {
  if (!h) return fail(MOE_ERR_INVALID_ARGUMENT, "null handle");
  if (!h->sh) {
    if (n_shards) *n_shards = 1;
    if (uses_nccl) *uses_nccl = 0;
    return MOE_OK;
  }
  return moe::abi::sh_layout(h, n_shards, uses_nccl);
}

moe_status moe_eamc_destroy(moe_eamc* h) {
  if (!h) return MOE_OK;
  if (h->sh) return moe::abi::sh_destroy(h);
  DeviceGuard dg(h->device);
  cudaStreamSynchronize(h->st);
  if (h->srv.G) g_srv_sms[h->device & 63] -= h->srv.G;
  delete h;
  return MOE_OK;
}

moe_status moe_eamc_info(const moe_eamc* h, moe_shape* shape, int* phase, uint64_t* capacity,
                         uint64_t* size, uint64_t* next_seq, int* count_bytes) {
  if (!h) return fail(MOE_ERR_INVALID_ARGUMENT, "null handle");
  if (shape) *shape = h->shape;
  if (phase) *phase = h->phase;
  if (capacity) *capacity = h->capacity;
  if (size) *size = h->c.size;
  if (next_seq) *next_seq = h->next_seq;
  if (count_bytes) *count_bytes = h->c.cb;
  if (h->sh) return moe::abi::sh_info(h, size, count_bytes);
  return MOE_OK;
}

moe_status moe_eamc_entry(const moe_eamc* hc, uint64_t index, uint64_t* counts, uint64_t* seq) {
  HandleLock hl_(hc);
  moe_eamc* h = const_cast<moe_eamc*>(hc);
  if (!h) return fail(MOE_ERR_INVALID_ARGUMENT, "null handle");
  if (h->sh) return moe::abi::sh_entry(h, index, counts, seq);
  if (index >= h->c.size) return fail(MOE_ERR_OUT_OF_RANGE, "entry index out of range");
  DeviceGuard dg(h->device);
  return read_entry(h, index, counts, seq);
}

moe_status moe_eamc_insert(moe_eamc* h, const uint64_t* counts, moe_eam_kind kind,
                           moe_phase phase, int64_t* evicted_slot, uint64_t* evicted_counts) {
  HandleLock hl_(h);
  if (!h || !counts) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  // Eamc::insert validation order (eam.cpp:153-158)
  if (kind != MOE_KIND_REQUEST)
    return fail(MOE_ERR_INVALID_ARGUMENT, "Eamc::insert: only request-level EAMs are stored");
  if ((int)phase != h->phase) return fail(MOE_ERR_INVALID_ARGUMENT, "Eamc::insert: phase mismatch");
  if (h->sh) return moe::abi::sh_insert(h, counts, evicted_slot, evicted_counts);
  DeviceGuard dg(h->device);
  const uint64_t cells = (uint64_t)h->c.L * h->c.E;
  Staged s;
  CK(h->raw.ensure(cells * 8));
  CK(cudaMemcpyAsync(h->raw.p, counts, cells * 8, cudaMemcpyHostToDevice, h->st));
  CKS(stage_entries(h, h->raw.p, 8, 1, &s));
  if (h->c.size < h->capacity) {
    int64_t slot = -1;
    CKS(replay_staged(h, s, &slot));
    if (evicted_slot) *evicted_slot = -1;
    return MOE_OK;
  }
  // at capacity: find the victim first so the evicted Eam can be returned
  CK(h->out.ensure(sizeof(moe_match)));
  moe_match* dv = h->out.as<moe_match>();
  CKS(match_packed(h, s.pr, dv, h->st));
  moe_match v;
  CK(cudaMemcpyAsync(&v, dv, sizeof v, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (evicted_counts) CKS(read_entry(h, v.index - h->c.index_base, evicted_counts, nullptr));
  ++h->version;
  CK(moe::launch_replace(h->c, s.pr, 0, dv, h->next_seq, nullptr, h->st));
  CK(cudaStreamSynchronize(h->st));
  h->next_seq++;
  if (evicted_slot) *evicted_slot = (int64_t)(v.index - h->c.index_base);
  return MOE_OK;
}

// Upload m host u64 EAMs for staging: narrowed to the storage width on the
// host pool into pinned memory (1-2 B per count over PCIe instead of 8),
// or, when some count does not fit that width, as u64 (stage_entries then
// widens the collection).  *src_bytes = the width now in h->raw.
static moe_status upload_host_counts(moe_eamc* h, const uint64_t* src, uint64_t m,
                                     int* src_bytes) {
  const uint64_t cells = (uint64_t)h->c.L * h->c.E;
  const int cb = h->c.cb;
  CK(h->hpack.ensure(m * cells * cb));
  const uint64_t o = moe::host::pack_counts(src, m * cells, cb, h->hpack.p);
  if (o <= width_max(cb)) {
    CK(h->raw.ensure(m * cells * cb));
    CK(cudaMemcpyAsync(h->raw.p, h->hpack.p, m * cells * cb, cudaMemcpyHostToDevice, h->st));
    // the pinned staging buffer is reused by the next chunk
    CK(cudaStreamSynchronize(h->st));
    *src_bytes = cb;
    return MOE_OK;
  }
  CK(h->raw.ensure(m * cells * 8));
  CK(cudaMemcpyAsync(h->raw.p, src, m * cells * 8, cudaMemcpyHostToDevice, h->st));
  *src_bytes = 8;
  return MOE_OK;
}

moe_status moe_eamc_build(moe_eamc* h, const uint64_t* counts, uint64_t n,
                          int64_t* evicted_slots) {
  HandleLock hl_(h);
  if (!h || (!counts && n)) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (h->sh) return moe::abi::sh_build(h, counts, n, evicted_slots);
  DeviceGuard dg(h->device);
  const uint64_t cells = (uint64_t)h->c.L * h->c.E;
  const uint64_t chunk = std::max<uint64_t>(1, (256ull << 20) / (cells * 8));
  Staged s;
  for (uint64_t off = 0; off < n; off += chunk) {
    const uint64_t m = std::min(chunk, n - off);
    int sb = 8;
    CKS(upload_host_counts(h, counts + off * cells, m, &sb));
    CKS(stage_entries(h, h->raw.p, sb, m, &s));
    CKS(replay_staged(h, s, evicted_slots ? evicted_slots + off : nullptr));
  }
  return MOE_OK;
}

static moe_status append_impl(moe_eamc* h, const void* counts, int cbytes, const uint64_t* seqs,
                              uint64_t n) {
  if (h->c.size + n > h->capacity)
    return fail(MOE_ERR_SNAPSHOT, "snapshot holds more entries than its capacity");
  ++h->version;
  const uint64_t cells = (uint64_t)h->c.L * h->c.E;
  const uint64_t chunk = std::max<uint64_t>(1, (256ull << 20) / (cells * cbytes));
  Staged s;
  for (uint64_t off = 0; off < n; off += chunk) {
    const uint64_t m = std::min(chunk, n - off);
    int sb = cbytes;
    if (cbytes == 8) {
      CKS(upload_host_counts(h, static_cast<const uint64_t*>(counts) + off * cells, m, &sb));
    } else {
      CK(h->raw.ensure(m * cells * cbytes));
      CK(cudaMemcpyAsync(h->raw.p, static_cast<const uint8_t*>(counts) + off * cells * cbytes,
                         m * cells * cbytes, cudaMemcpyHostToDevice, h->st));
    }
    CKS(stage_entries(h, h->raw.p, sb, m, &s));
    CKS(ensure_alloc(h, h->c.size + m));
    CK(moe::launch_append_staged(h->c, s.pr, 0, (uint32_t)m, h->c.size, h->st));
    CK(cudaMemcpyAsync(h->c.seq + h->c.size, seqs + off, m * 8, cudaMemcpyHostToDevice, h->st));
    CK(cudaStreamSynchronize(h->st));
    h->c.size += (uint32_t)m;
    for (uint64_t k = 0; k < m; ++k) h->next_seq = std::max(h->next_seq, seqs[off + k] + 1);
  }
  return MOE_OK;
}

// Clustering construction (cluster.cu has the kernels and the method).
moe_status moe_eamc_build_clustered(moe_eamc* h, const uint64_t* counts, uint64_t n,
                                    uint32_t iterations, double* objective, uint64_t* rep_index,
                                    uint32_t* iterations_run) {
  HandleLock hl_(h);
  if (!h || (!counts && n)) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (h->sh) return fail(MOE_ERR_INVALID_ARGUMENT, "clustering builds a single-device collection");
  if (h->c.size != 0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "build_clustered: the collection must start empty");
  if (iterations_run) *iterations_run = 0;
  if (n == 0) return MOE_OK;
  DeviceGuard dg(h->device);
  // iteration 0: the reference construction (n ordered Eamc::insert calls)
  std::vector<int64_t> ev(n);
  CKS(moe_eamc_build(h, counts, n, ev.data()));
  DevColl& c = h->c;
  const uint64_t P = c.size, cells = (uint64_t)c.L * c.E;
  std::vector<uint64_t> rep(P);  // input index of each slot's trace (= its seq here)
  {
    uint64_t appended = 0;
    for (uint64_t k = 0; k < n; ++k) rep[ev[k] < 0 ? appended++ : (uint64_t)ev[k]] = k;
  }
  // every trace once on the device: narrow rows for the matcher, staged rows
  // (packed, norms) for the exact distances and the replacements
  DevBuf tr;
  Staged S;
  {
    int sb = 8;
    CKS(upload_host_counts(h, counts, n, &sb));
    CK(tr.ensure(n * cells * sb + 16));
    CK(cudaMemcpyAsync(tr.p, h->raw.p, n * cells * sb, cudaMemcpyDeviceToDevice, h->st));
    CKS(stage_entries(h, tr.p, sb, n, &S));
    if (sb != c.cb) {  // the staging widened the collection: matcher probes at its width
      std::vector<uint8_t> hp(n * cells * c.cb);
      moe::host::pack_counts(counts, n * cells, c.cb, hp.data());
      CK(tr.ensure(hp.size() + 16));
      CK(cudaMemcpy(tr.p, hp.data(), hp.size(), cudaMemcpyHostToDevice));
    }
  }
  DevBuf dm, cent, dc, cmin, cidx, tcur, tcand, vic;
  CK(dm.ensure(n * sizeof(moe_match)));
  CK(cent.ensure(P * cells * 8));
  CK(dc.ensure(n * 8));
  CK(cmin.ensure(P * 8));
  CK(cidx.ensure(P * 8));
  CK(tcur.ensure(P * 8));
  CK(tcand.ensure(P * 8));
  CK(vic.ensure(P * sizeof(moe_match)));
  std::vector<moe_match> hm(n);
  std::vector<uint64_t> hidx(P), hcur(P), hcand(P);
  uint32_t t = 0;
  for (;; ++t) {
    CKS(moe_eamc_match_device(h, tr.p, c.cb, n, dm.as<moe_match>(), h->st));
    CK(cudaMemcpyAsync(hm.data(), dm.p, n * sizeof(moe_match), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    double obj = 0.0;
    for (uint64_t i = 0; i < n; ++i) obj += hm[i].distance;  // input order: deterministic
    if (objective) objective[t] = obj;
    if (t == iterations) break;
    CK(moe::launch_cluster_step(S.pr.packed, S.pr.sqa, n, c.L, c.E, c.RB, c.cb, dm.as<moe_match>(),
                                c.index_base, P, cent.as<unsigned long long>(), dc.as<double>(),
                                cmin.as<unsigned long long>(), cidx.as<unsigned long long>(),
                                tcur.as<unsigned long long>(), tcand.as<unsigned long long>(),
                                h->st));
    CK(cudaMemcpyAsync(hidx.data(), cidx.p, P * 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaMemcpyAsync(hcur.data(), tcur.p, P * 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaMemcpyAsync(hcand.data(), tcand.p, P * 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    std::vector<moe_match> acc;
    std::vector<uint64_t> acc_i;
    for (uint64_t p = 0; p < P; ++p)
      if (hidx[p] != ~0ull && hidx[p] != rep[p] && hcand[p] < hcur[p]) {
        acc.push_back(moe_match{c.index_base + p, 0, 0.0});
        acc_i.push_back(hidx[p]);
        rep[p] = hidx[p];
      }
    if (acc.empty()) {  // converged: later iterations would repeat this one
      for (uint32_t u = t + 1; objective && u <= iterations; ++u) objective[u] = obj;
      break;
    }
    ++h->version;
    CK(cudaMemcpyAsync(vic.p, acc.data(), acc.size() * sizeof(moe_match), cudaMemcpyHostToDevice,
                       h->st));
    for (size_t k = 0; k < acc.size(); ++k)  // seq = the trace's input index (unique)
      CK(moe::launch_replace(c, S.pr, (uint32_t)acc_i[k], vic.as<moe_match>() + k, acc_i[k],
                             nullptr, h->st));
    CK(cudaStreamSynchronize(h->st));
  }
  h->next_seq = std::max<uint64_t>(h->next_seq, n);
  if (rep_index) std::copy(rep.begin(), rep.end(), rep_index);
  if (iterations_run) *iterations_run = t;
  return MOE_OK;
}

moe_status moe_eamc_append(moe_eamc* h, const uint64_t* counts, const uint64_t* seqs, uint64_t n) {
  HandleLock hl_(h);
  if (!h || ((!counts || !seqs) && n)) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (h->sh) return moe::abi::sh_append(h, counts, 8, seqs, n);
  DeviceGuard dg(h->device);
  return append_impl(h, counts, 8, seqs, n);
}

moe_status moe_eamc_append_packed(moe_eamc* h, const void* counts, int count_bytes,
                                  const uint64_t* seqs, uint64_t n) {
  HandleLock hl_(h);
  if (!h || ((!counts || !seqs) && n)) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (count_bytes != 1 && count_bytes != 2 && count_bytes != 4 && count_bytes != 8)
    return fail(MOE_ERR_INVALID_ARGUMENT, "count_bytes must be 1, 2, 4 or 8");
  if (h->sh) return moe::abi::sh_append(h, counts, count_bytes, seqs, n);
  DeviceGuard dg(h->device);
  return append_impl(h, counts, count_bytes, seqs, n);
}

// Host-narrowed matching for large host batches.  The reference API hands over
// u64 counts (eam.hpp:55); shipping them as is makes the call PCIe-bound
// (8 B/count).  Each host-pool task narrows one chunk to the storage width
// into a pinned buffer (the OR of the chunk is the exact width check) and
// enqueues that chunk's DMA on the copy stream itself, so transfers start
// while other chunks are still being narrowed (MOE_MATCH_GROUPS > 1 also
// splits the batch into groups matched as they arrive).
// *done = false (nothing usable written) when some count exceeds the storage
// width: the caller then takes the u64 path, which widens the collection.
struct PackJob {
  const uint64_t* src;
  uint8_t *hp, *dp;
  uint64_t cells, row_b, g0, g1, chunk;
  int cb, device;
  cudaStream_t st;
  std::atomic<int> bad{0};
  std::atomic<int> err{0};
};

static void pack_chunk_task(void* vj, int t) {
  PackJob* j = static_cast<PackJob*>(vj);
  const uint64_t off = j->g0 + (uint64_t)t * j->chunk;
  const uint64_t m = std::min(j->chunk, j->g1 - off);
  if (j->bad.load(std::memory_order_relaxed)) return;
  const uint64_t o = moe::host::pack_counts_serial(j->src + off * j->cells, m * j->cells, j->cb,
                                                   j->hp + off * j->row_b);
  if (o > width_max(j->cb)) {
    j->bad.store(1);
    return;
  }
  if (cudaSetDevice(j->device) != cudaSuccess ||
      cudaMemcpyAsync(j->dp + off * j->row_b, j->hp + off * j->row_b, m * j->row_b,
                      cudaMemcpyHostToDevice, j->st) != cudaSuccess)
    j->err.store(1);
}

static moe_status match_host_packed(moe_eamc* h, const uint64_t* probes, uint64_t n,
                                    moe_match* out, bool* done) {
  *done = false;
  const int cb = h->c.cb;
  const uint64_t cells = (uint64_t)h->c.L * h->c.E;
  const uint64_t row_b = cells * cb;
  if (!h->st2) {
    CK(cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&h->ev_copy[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_free[i], cudaEventDisableTiming));
    }
  }
  CK(h->hpack.ensure(n * row_b));
  CK(h->raw.ensure(n * row_b));
  CK(h->outall.ensure(n * sizeof(moe_match)));
  moe_match* dout = h->outall.as<moe_match>();
  // one group measured fastest at SW (0.53 vs 0.55 ms for two: host narrowing
  // is bound by host memory bandwidth, the GPU tail is short)
  uint64_t groups = 1;
  if (const char* e = getenv("MOE_MATCH_GROUPS")) groups = std::max(1, atoi(e));
  groups = std::min<uint64_t>(groups, n);
  const uint64_t threads = (uint64_t)moe::host::pool_threads();
  // group g is narrowed by the pool workers while this thread launches the
  // matching of group g-1 (its DMAs were issued by the tasks themselves)
  PackJob jobs[2];
  for (int k = 0; k < 2; ++k) {
    PackJob& j = jobs[k];
    j.src = probes;
    j.hp = h->hpack.as<uint8_t>();
    j.dp = h->raw.as<uint8_t>();
    j.cells = cells;
    j.row_b = row_b;
    j.cb = cb;
    j.device = h->device;
    j.st = h->st2;
  }
  auto submit = [&](uint64_t g) {
    PackJob& j = jobs[g & 1];
    j.bad.store(0);
    j.err.store(0);
    j.g0 = n * g / groups;
    j.g1 = n * (g + 1) / groups;
    // one chunk per pool thread (>= 64 KiB of input each)
    j.chunk = std::max<uint64_t>((j.g1 - j.g0 + threads - 1) / threads,
                                 std::max<uint64_t>(1, 8192 / cells));
    if (const char* e = getenv("MOE_PACK_CHUNK")) j.chunk = std::max(1, atoi(e));
    const int tasks = (int)((j.g1 - j.g0 + j.chunk - 1) / j.chunk);
    if (groups == 1) moe::host::pool_run(tasks, pack_chunk_task, &j);
    else moe::host::pool_submit(tasks, pack_chunk_task, &j);
  };
  auto finish = [&](uint64_t g) -> moe_status {  // after the group's tasks are done
    PackJob& j = jobs[g & 1];
    if (j.err.load()) return fail(MOE_ERR_CUDA, "probe upload failed");
    if (j.bad.load()) return MOE_ERR_OVERFLOW;  // sentinel for the caller below
    CK(cudaEventRecord(h->ev_copy[g & 1], h->st2));
    return MOE_OK;
  };
  auto launch = [&](uint64_t g) -> moe_status {
    PackJob& j = jobs[g & 1];
    CK(cudaStreamWaitEvent(h->st, h->ev_copy[g & 1], 0));
    DevProbes pr;
    CKS(match_all(h, j.dp + j.g0 * row_b, cb, j.g1 - j.g0, true, dout + j.g0, h->st, &pr,
                  /*async=*/true));
    return MOE_OK;
  };
  moe_status fs = MOE_OK;
  submit(0);
  if (groups > 1) moe::host::pool_wait();
  fs = finish(0);
  for (uint64_t g = 1; g <= groups && fs == MOE_OK; ++g) {
    if (g < groups) submit(g);
    const moe_status ls = launch(g - 1);
    if (g < groups) moe::host::pool_wait();
    if (ls != MOE_OK) return ls;
    if (g < groups) fs = finish(g);
  }
  if (fs == MOE_ERR_OVERFLOW) {  // rare: widen through the u64 path
    CK(cudaStreamSynchronize(h->st2));
    CK(cudaStreamSynchronize(h->st));
    return MOE_OK;
  }
  CKS(fs);
  CK(cudaMemcpyAsync(out, dout, n * sizeof(moe_match), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  *done = true;
  return MOE_OK;
}

moe_status moe_eamc_match(const moe_eamc* hc, const uint64_t* probes, uint64_t n_probes,
                          moe_match* out, uint8_t* found) {
  HandleLock hl_(hc);
  moe_eamc* h = const_cast<moe_eamc*>(hc);
  if (!h || ((!probes || !out) && n_probes)) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (n_probes == 0) return MOE_OK;
  if (h->sh) {
    CKS(moe::abi::sh_match(h, probes, n_probes, out));
    if (found)
      for (uint64_t q = 0; q < n_probes; ++q) found[q] = out[q].index != ~0ull;
    return MOE_OK;
  }
  DeviceGuard dg(h->device);
  const uint64_t cells = (uint64_t)h->c.L * h->c.E;
  const uint64_t bytes = n_probes * cells * 8;
  const char* hp_env = getenv("MOE_HOST_PACK");
  if (bytes >= (4ull << 20) && !(hp_env && hp_env[0] == '0')) {
    bool done = false;
    CKS(match_host_packed(h, probes, n_probes, out, &done));
    if (done) {
      // probes the device pass could not represent (a row's sum of squares
      // past 2^53) come back as width sentinels: the synchronous path below
      // reports them (MOE_ERR_OVERFLOW)
      for (uint64_t q = 0; q < n_probes; ++q)
        if (out[q].index == ~0ull - 1) {
          DevProbes pr;
          CK(h->out.ensure(sizeof(moe_match)));
          CKS(match_all(h, probes + q * cells, 8, 1, false, h->out.as<moe_match>(), h->st, &pr));
          CK(cudaMemcpy(out + q, h->out.p, sizeof(moe_match), cudaMemcpyDeviceToHost));
        }
      if (found)
        for (uint64_t q = 0; q < n_probes; ++q) found[q] = out[q].index != ~0ull;
      return MOE_OK;
    }
  }
  uint64_t pipe_chunk = 0;  // probes per pipelined chunk (0 = one shot)
  if (const char* pc = getenv("MOE_PIPE_CHUNK")) pipe_chunk = strtoull(pc, nullptr, 10);
  else if (bytes >= (16ull << 20)) pipe_chunk = std::max<uint64_t>(1024, (n_probes + 3) / 4);
  if (pipe_chunk == 0 || pipe_chunk >= n_probes) {  // one shot
    DevProbes pr;
    CK(h->out.ensure(n_probes * sizeof(moe_match)));
    CKS(match_all(h, probes, 8, n_probes, false, h->out.as<moe_match>(), h->st, &pr));
    CK(cudaMemcpyAsync(out, h->out.p, n_probes * sizeof(moe_match), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
  } else {
    // Pipelined: the H2D copy of chunk k+1 (copy stream) overlaps the matching
    // of chunk k (compute stream); two staging buffers, event-ordered reuse.
    // Probes that do not fit the storage width come back as sentinels and
    // are redone below (the collection widens then).
    if (!h->st2) {
      CK(cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        CK(cudaEventCreateWithFlags(&h->ev_copy[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->ev_free[i], cudaEventDisableTiming));
      }
    }
    const uint64_t chunk = std::max<uint64_t>(
        128, std::min<uint64_t>(pipe_chunk, (128ull << 20) / (cells * 8)));
    CK(h->raw2[0].ensure(chunk * cells * 8));
    CK(h->raw2[1].ensure(chunk * cells * 8));
    CK(h->outall.ensure(n_probes * sizeof(moe_match)));
    moe_match* dout = h->outall.as<moe_match>();
    uint64_t k = 0;
    for (uint64_t off = 0; off < n_probes; off += chunk, ++k) {
      const uint64_t m = std::min(chunk, n_probes - off);
      const int b = (int)(k & 1);
      if (k >= 2) CK(cudaStreamWaitEvent(h->st2, h->ev_free[b], 0));
      CK(cudaMemcpyAsync(h->raw2[b].p, probes + off * cells, m * cells * 8, cudaMemcpyHostToDevice,
                         h->st2));
      CK(cudaEventRecord(h->ev_copy[b], h->st2));
      CK(cudaStreamWaitEvent(h->st, h->ev_copy[b], 0));
      DevProbes pr;
      CKS(match_all(h, h->raw2[b].p, 8, m, true, dout + off, h->st, &pr, /*async=*/true,
                    h->ev_free[b]));
    }
    CK(cudaMemcpyAsync(out, dout, n_probes * sizeof(moe_match), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    std::vector<uint64_t> redo;
    for (uint64_t q = 0; q < n_probes; ++q)
      if (out[q].index == ~0ull - 1) redo.push_back(q);
    if (!redo.empty()) {
      std::vector<uint64_t> sub(redo.size() * cells);
      for (size_t i = 0; i < redo.size(); ++i)
        std::copy(probes + redo[i] * cells, probes + (redo[i] + 1) * cells, sub.begin() + i * cells);
      // synchronous path: widens the collection, then matches exactly
      const uint64_t step = std::max<uint64_t>(1, (8ull << 20) / (cells * 8));
      for (uint64_t o = 0; o < redo.size(); o += step) {
        const uint64_t m = std::min<uint64_t>(step, redo.size() - o);
        DevProbes pr;
        CK(h->out.ensure(m * sizeof(moe_match)));
        CKS(match_all(h, sub.data() + o * cells, 8, m, false, h->out.as<moe_match>(), h->st, &pr));
        std::vector<moe_match> res(m);
        CK(cudaMemcpyAsync(res.data(), h->out.p, m * sizeof(moe_match), cudaMemcpyDeviceToHost,
                           h->st));
        CK(cudaStreamSynchronize(h->st));
        for (uint64_t i = 0; i < m; ++i) out[redo[o + i]] = res[i];
      }
    }
  }
  if (found)
    for (uint64_t q = 0; q < n_probes; ++q) found[q] = out[q].index != ~0ull;
  return MOE_OK;
}

moe_status moe_eamc_match_device(const moe_eamc* hc, const void* probes, int probe_bytes,
                                 uint64_t n_probes, moe_match* out, void* stream) {
  HandleLock hl_(hc);
  moe_eamc* h = const_cast<moe_eamc*>(hc);
  if (!h || ((!probes || !out) && n_probes)) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (probe_bytes != 1 && probe_bytes != 2 && probe_bytes != 4 && probe_bytes != 8)
    return fail(MOE_ERR_INVALID_ARGUMENT, "probe_bytes must be 1, 2, 4 or 8");
  if (n_probes == 0) return MOE_OK;
  if (n_probes > 0xffffffffull) return fail(MOE_ERR_INVALID_ARGUMENT, "too many probes");
  if (h->sh)
    return fail(MOE_ERR_INVALID_ARGUMENT,
                "moe_eamc_match_device: a sharded collection spans devices; use moe_eamc_match");
  DeviceGuard dg(h->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->st;
  DevProbes pr;
  CKS(match_all(h, probes, probe_bytes, n_probes, true, out, st, &pr, /*async=*/true));
  return MOE_OK;
}

// Host probes already narrow ([n][L][E] of 1 or 2 bytes, e.g. traced
// counts): one H2D of the narrow batch (a true DMA when the buffer is pinned),
// the matching pipeline in synchronous mode (width check; widening redo), D2H.
moe_status moe_eamc_match_packed(const moe_eamc* hc, const void* probes, int probe_bytes,
                                 uint64_t n_probes, moe_match* out, uint8_t* found) {
  HandleLock hl_(hc);
  moe_eamc* h = const_cast<moe_eamc*>(hc);
  if (!h || ((!probes || !out) && n_probes)) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (probe_bytes == 8)
    return moe_eamc_match(hc, static_cast<const uint64_t*>(probes), n_probes, out, found);
  if (probe_bytes != 1 && probe_bytes != 2 && probe_bytes != 4)
    return fail(MOE_ERR_INVALID_ARGUMENT, "probe_bytes must be 1, 2, 4 or 8");
  if (n_probes == 0) return MOE_OK;
  if (n_probes > 0xffffffffull) return fail(MOE_ERR_INVALID_ARGUMENT, "too many probes");
  if (h->sh) {  // the sharded matcher packs u64 probes itself
    const uint64_t m = n_probes * (uint64_t)h->c.L * h->c.E;
    std::vector<uint64_t> wide(m);
    for (uint64_t i = 0; i < m; ++i)
      wide[i] = probe_bytes == 1 ? static_cast<const uint8_t*>(probes)[i]
                : probe_bytes == 2 ? static_cast<const uint16_t*>(probes)[i]
                                   : static_cast<const uint32_t*>(probes)[i];
    return moe_eamc_match(hc, wide.data(), n_probes, out, found);
  }
  DeviceGuard dg(h->device);
  const uint64_t bytes = n_probes * (uint64_t)h->c.L * h->c.E * probe_bytes;
  CK(h->raw.ensure(bytes + 16));
  CK(h->outall.ensure(n_probes * sizeof(moe_match)));
  CK(cudaMemcpyAsync(h->raw.p, probes, bytes, cudaMemcpyHostToDevice, h->st));
  DevProbes pr;
  CKS(match_all(h, h->raw.p, probe_bytes, n_probes, true, h->outall.as<moe_match>(), h->st, &pr));
  CK(cudaMemcpyAsync(out, h->outall.p, n_probes * sizeof(moe_match), cudaMemcpyDeviceToHost,
                     h->st));
  CK(cudaStreamSynchronize(h->st));
  if (found)
    for (uint64_t q = 0; q < n_probes; ++q) found[q] = out[q].index != ~0ull;
  return MOE_OK;
}

moe_status moe_eamc_match_within(const moe_eamc* hc, const uint64_t* probe, double window,
                                 moe_match* out, uint64_t cap, uint64_t* n_out) {
  HandleLock hl_(hc);
  moe_eamc* h = const_cast<moe_eamc*>(hc);
  if (!h || !probe || !n_out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  *n_out = 0;
  if (h->sh) return moe::abi::sh_match_within(h, probe, window, out, cap, n_out);
  if (h->c.size == 0) return MOE_OK;
  DeviceGuard dg(h->device);
  cudaStream_t st = h->st;
  for (;;) {
    DevProbes pr;
    CKS(launch_exact_distances(h, probe, st, &pr));
    CK(h->wl.ensure((size_t)h->c.size * sizeof(moe::WinEntry)));
    uint32_t* wl_n = h->small.as<uint32_t>() + 8;
    CK(cudaMemsetAsync(wl_n, 0, 4, st));
    CK(moe::launch_window_list(
        h->c, h->dist.as<double>(),
        reinterpret_cast<unsigned long long*>(h->small.as<uint8_t>() + 224), window,
        h->wl.as<moe::WinEntry>(), wl_n, st));
    CK(cudaMemcpyAsync(h->pin.p, h->small.p, 64, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    bool ok = false;
    CKS(check_width(h, *h->pin.as<unsigned long long>(), &ok));
    if (!ok) continue;
    const uint32_t n = h->pin.as<uint32_t>()[8];
    std::vector<moe::WinEntry> v(n);
    CK(cudaMemcpy(v.data(), h->wl.p, n * sizeof(moe::WinEntry), cudaMemcpyDeviceToHost));
    // (distance, seq) order of the result list (eam.cpp:145-148)
    std::sort(v.begin(), v.end(), [](const moe::WinEntry& a, const moe::WinEntry& b) {
      return a.d != b.d ? a.d < b.d : a.seq < b.seq;
    });
    for (uint64_t i = 0; i < n && i < cap; ++i)
      out[i] = moe_match{v[i].p + h->c.index_base, v[i].seq, v[i].d};
    *n_out = n;
    return MOE_OK;
  }
}

moe_status moe_match_merge(const moe_match* parts, uint64_t n_parts, uint64_t n, moe_match* out) {
  if ((!parts || !out) && n) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (n == 0 || n_parts == 0) return MOE_OK;
  int n_sm = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  CKS(device_ok(dev, &n_sm));
  moe_match* d = nullptr;
  CK(cudaMalloc(&d, (n_parts + 1) * n * sizeof(moe_match)));
  cudaError_t e = cudaMemcpy(d, parts, n_parts * n * sizeof(moe_match), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = moe::launch_merge(d, n_parts, n, d + n_parts * n, nullptr);
  if (e == cudaSuccess)
    e = cudaMemcpy(out, d + n_parts * n, n * sizeof(moe_match), cudaMemcpyDeviceToHost);
  cudaFree(d);
  CK(e);
  return MOE_OK;
}

moe_status moe_match_merge_device(const moe_match* parts, uint64_t n_parts, uint64_t n,
                                  moe_match* out, void* stream) {
  if ((!parts || !out) && n) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (n == 0 || n_parts == 0) return MOE_OK;
  CK(moe::launch_merge(parts, n_parts, n, out, static_cast<cudaStream_t>(stream)));
  return MOE_OK;
}

moe_status moe_eamc_clone(const moe_eamc* hc, moe_eamc** out) {
  HandleLock hl_(hc);
  moe_eamc* src = const_cast<moe_eamc*>(hc);
  if (!src || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (src->sh) return moe::abi::sh_clone(src, out);
  DeviceGuard dg(src->device);
  const uint64_t cells = (uint64_t)src->c.L * src->c.E, n = src->c.size;
  std::vector<uint64_t> counts(n * cells), seqs(n);
  for (uint64_t i = 0; i < n; ++i) CKS(read_entry(src, i, counts.data() + i * cells, &seqs[i]));
  moe_eamc* h = nullptr;
  CKS(moe_eamc_create(&src->shape, (moe_phase)src->phase, src->capacity, src->c.cb, src->device,
                      &h));
  if (n) {
    const moe_status s = moe_eamc_append(h, counts.data(), seqs.data(), n);
    if (s != MOE_OK) {
      moe_eamc_destroy(h);
      return s;
    }
  }
  h->next_seq = src->next_seq;
  h->c.index_base = src->c.index_base;
  *out = h;
  return MOE_OK;
}

moe_status moe_eamc_set_index_base(moe_eamc* h, uint64_t base) {
  if (h && h->sh)
    return fail(MOE_ERR_INVALID_ARGUMENT, "a sharded collection sets its shards' index bases");
  HandleLock hl_(h);
  if (!h) return fail(MOE_ERR_INVALID_ARGUMENT, "null handle");
  h->c.index_base = base;
  return MOE_OK;
}

moe_status moe_eamc_set_decision_server(moe_eamc* h, int n_ctas) {
  HandleLock hl_(h);
  if (!h) return fail(MOE_ERR_INVALID_ARGUMENT, "null handle");
  if (h->sh) return fail(MOE_ERR_INVALID_ARGUMENT, "the decision server is per shard handle");
  if (n_ctas < 0) return fail(MOE_ERR_INVALID_ARGUMENT, "n_ctas must be >= 0");
  DeviceGuard dg(h->device);
  const int want = std::min(n_ctas, h->n_sm / 2);
  if (want == h->srv.G) return MOE_OK;
  CKS(server_stop(h));
  g_srv_sms[h->device & 63] += want - h->srv.G;
  h->srv.G = want;
  return MOE_OK;
}

moe_status moe_eamc_set_profiling(moe_eamc* h, int enable) {
  HandleLock hl_(h);
  if (!h) return fail(MOE_ERR_INVALID_ARGUMENT, "null handle");
  if (h->sh) return fail(MOE_ERR_INVALID_ARGUMENT, "profiling is per shard handle");
  DeviceGuard dg(h->device);
  if (h->ring.empty()) {
    h->ring.resize(256);
    for (auto& es : h->ring)
      for (cudaEvent_t& e : es.ev) CK(cudaEventCreate(&e));
  }
  for (auto& es : h->ring) es.pending = false;
  h->prof = enable != 0;
  for (int i = 0; i < 3; ++i) {
    h->ms[i] = 0.0;
    h->calls[i] = 0;
  }
  return MOE_OK;
}

moe_status moe_eamc_kernel_times(const moe_eamc* hc, double* ms, uint64_t* calls) {
  HandleLock hl_(hc);
  moe_eamc* h = const_cast<moe_eamc*>(hc);
  if (!h) return fail(MOE_ERR_INVALID_ARGUMENT, "null handle");
  DeviceGuard dg(h->device);
  for (auto& es : h->ring) CKS(prof_collect(h, es));
  for (int i = 0; i < 3; ++i) {
    if (ms) ms[i] = h->ms[i];
    if (calls) calls[i] = h->calls[i];
  }
  return MOE_OK;
}

// Scalar entry points (eam_distance, cache_priority, select_eviction_victim)
// run on a persistent per-(device, shape) scratch collection: creating a
// handle costs device allocations and streams, which would dominate a call
// the engine makes per slot (engine.cpp:443,:472,:644).  The lease holds the
// cache lock, so concurrent scalar calls serialise on it.
struct ScratchLease {
  std::unique_lock<std::mutex> lock;
  moe_eamc* h = nullptr;
};

static moe_status scratch_handle(const moe_shape* shape, ScratchLease* lease) {
  struct Slot {
    int dev;
    uint32_t L, E;
    moe_eamc* h;
  };
  static std::mutex mu;
  static std::vector<Slot> cache;  // never destroyed: lives until process exit
  int dev = 0, n_sm = 0;
  cudaGetDevice(&dev);
  CKS(device_ok(dev, &n_sm));
  std::unique_lock<std::mutex> lk(mu);
  for (const Slot& c : cache)
    if (c.dev == dev && c.L == shape->n_layers && c.E == shape->n_experts_per_layer) {
      lease->h = c.h;
      lease->lock = std::move(lk);
      return MOE_OK;
    }
  moe_eamc* h = nullptr;
  CKS(moe_eamc_create(shape, MOE_PHASE_DECODE, 1, 1, dev, &h));
  if (cache.size() >= 8) {
    moe_eamc_destroy(cache.front().h);
    cache.erase(cache.begin());
  }
  cache.push_back({dev, shape->n_layers, shape->n_experts_per_layer, h});
  lease->h = h;
  lease->lock = std::move(lk);
  return MOE_OK;
}

moe_status moe_eam_distance(const moe_shape* shape, const uint64_t* a, const uint64_t* b,
                            double* out) {
  CKS(check_shape(shape));
  if (!a || !b || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  ScratchLease lease;
  CKS(scratch_handle(shape, &lease));
  moe_eamc* h = lease.h;
  const uint64_t cells = (uint64_t)shape->n_layers * shape->n_experts_per_layer;
  std::vector<uint64_t> both(2 * cells);
  std::copy(a, a + cells, both.begin());
  std::copy(b, b + cells, both.begin() + cells);
  DevProbes pr;
  CKS(prep_probes(h, both.data(), 8, 2, false, h->st, &pr));
  cudaError_t e = h->dist.ensure(8);
  const uint64_t LR = (uint64_t)h->c.L * h->c.RB;
  if (e == cudaSuccess)
    e = moe::launch_pair_distance(pr.packed, pr.sqa, pr.packed + LR, pr.sqa + h->c.L, h->c.L,
                                  h->c.C, h->c.RB, h->c.cb, h->dist.as<double>(), h->st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, h->dist.p, 8, cudaMemcpyDeviceToHost, h->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->st);
  if (e != cudaSuccess) return fail(MOE_ERR_CUDA, "eam_distance: %s", cudaGetErrorString(e));
  return MOE_OK;
}

// ---- decision path (K4 + K5 [+ K6]): one cooperative launch (decide.cu) ---
// MOE_DEC_TIMING=1: host-side launch / completion latency of the decision
// kernel on stderr (diagnostics).
static bool dec_timing() {
  static const bool on = [] {
    const char* e = getenv("MOE_DEC_TIMING");
    return e && e[0] == '1';
  }();
  return on;
}

// Device scratch of the fused decision kernel, grown on demand.
static moe_status dec_scratch(moe_eamc* h, uint64_t n_slots) {
  const DevColl& c = h->c;
  const uint64_t cells = (uint64_t)c.L * c.E;
  const size_t n = std::max<uint32_t>(c.size, 1);
  if (h->pref.n < n * 8) {
    CK(h->pref.ensure(n * 8));
    h->dec_keep = -1;  // the layer-prefix sums did not survive the reallocation
  }
  CK(h->dist.ensure(n * 8));
  CK(h->agg.ensure(cells * 8));
  CK(h->dkey.ensure(cells * 8));
  CK(h->did.ensure(cells * 4));
  CK(h->drank.ensure(cells * 4));
  CK(h->dseg.ensure((size_t)c.L * 4));
  CK(h->dmlist.ensure(n * 4));
  if (!h->dstate.p) {  // dmin2[2] = ~0 (then self-cleaning by call parity), barriers and
                       // listed-member counts = 0
    CK(h->dstate.ensure(64));  // synchronous: device-step calls run on the caller's stream
    CK(cudaMemset(h->dstate.p, 0xff, 16));
    CK(cudaMemset(h->dstate.as<uint8_t>() + 16, 0, 48));
    h->bar_base = h->bar_base2 = 0;
  }
  CK(h->cpin.ensure(std::max<uint64_t>(cells, 1) * sizeof(moe_candidate)));
  CK(h->fpin.ensure(64));
  if (n_slots) {
    CK(h->req.ensure(cells * 8));
    CK(h->slots.ensure(n_slots * (sizeof(moe_slot_view) + 8)));
  }
  return MOE_OK;
}

// ---- persistent decision server --------------------------------------------
// SMs held by resident decision servers per device: other software-grid-
// barrier launches (k_decision) must stay co-resident, so they size their grid
// to the SMs that remain.
static int decision_sms(const moe_eamc* h) {
  return std::max(8, h->n_sm - g_srv_sms[h->device & 63].load());
}

static bool small_off() {  // MOE_DEC_SMALL=0: always the multi-CTA kernel (A/B runs)
  static const bool off = [] {
    const char* e = getenv("MOE_DEC_SMALL");
    return e && e[0] == '0';
  }();
  return off;
}

static bool server_takes(const moe_eamc* h, uint64_t n_slots) {
  return h->srv.G > 0 && n_slots == 0 && !dec_timing();
}

static moe_status server_stop(moe_eamc* h) {
  auto& v = h->srv;
  if (!v.st) return MOE_OK;
  reinterpret_cast<volatile int*>(&v.ctl.as<moe::DecServerCtl>()->stop)[0] = 1;
  CK(cudaStreamSynchronize(v.st));
  reinterpret_cast<volatile int*>(&v.ctl.as<moe::DecServerCtl>()->stop)[0] = 0;
  v.launched = false;
  return MOE_OK;
}

static moe_status server_launch(moe_eamc* h, bool small) {
  auto& v = h->srv;
  const DevColl& c = h->c;
  if (small) {  // one CTA, shared memory for the largest small-path request
    auto* ctl = v.ctl.as<moe::DecServerCtl>();
    v.cb = c.cb;
    v.small = true;
    CK(moe::launch_decision_small_server(
        ctl, reinterpret_cast<volatile uint64_t*>(&ctl->seq_done)[0], 50'000'000ull, c.cb,
        moe::decision_small_smem_max(c.L, c.RB), v.st));
    v.launched = true;
    return MOE_OK;
  }
  v.small = false;
  uint32_t np = 1;
  while (np < c.E) np <<= 1;
  v.smem = std::max({(size_t)c.L * c.RB, (size_t)np * 28, moe::decision_smem(c.L, c.E, c.RB, 0, 0, 1)});
  CK(v.drows.ensure((size_t)c.L * c.RB + 2 * c.L + 32));
  v.cb = c.cb;
  auto* ctl = v.ctl.as<moe::DecServerCtl>();
  // seq0 = the last request completed: a pending request (seq_req > seq0) is served
  CK(moe::launch_decision_server(ctl, v.dargs.as<moe::DecisionArgs>(), v.drows.as<uint8_t>(),
                                 v.state.as<uint32_t>(), v.state.as<uint32_t>() + 1,
                                 v.state.as<uint32_t>() + 2,
                                 reinterpret_cast<volatile uint64_t*>(&ctl->seq_done)[0], v.k,
                                 50'000'000ull, ++v.gen, c.cb, v.G, v.smem, v.st));
  v.launched = true;
  return MOE_OK;
}

// One request through the server: post the arguments in the pinned mailbox,
// wait for seq_done (relaunching an idled-out server).
static moe_status server_run(moe_eamc* h, const moe::DecisionArgs& a, bool small) {
  auto& v = h->srv;
  if (!v.st) {
    CK(cudaStreamCreateWithFlags(&v.st, cudaStreamNonBlocking));
    CK(v.ctl.ensure(sizeof(moe::DecServerCtl)));
    std::memset(v.ctl.p, 0, sizeof(moe::DecServerCtl));
    CK(v.dargs.ensure(sizeof(moe::DecisionArgs)));
    CK(v.state.ensure(64));
    CK(cudaMemset(v.state.p, 0, 64));
    v.seq = 0;
    v.k = 0;
  }
  // widened, or the other server kind: relaunch
  if (v.launched && (v.cb != h->c.cb || v.small != small)) CKS(server_stop(h));
  // collection updates queued on the handle's stream complete before the
  // resident kernel reads the collection
  const cudaError_t q = cudaStreamQuery(h->st);
  if (q == cudaErrorNotReady) CK(cudaStreamSynchronize(h->st));
  else CK(q);
  auto* ctl = v.ctl.as<moe::DecServerCtl>();
  std::memcpy(&ctl->args, &a, sizeof a);
  std::atomic_thread_fence(std::memory_order_seq_cst);
  const uint64_t seq = ++v.seq;
  reinterpret_cast<volatile uint64_t*>(&ctl->seq_req)[0] = seq;
  if (!v.launched) CKS(server_launch(h, small));
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t spin = 1;; ++spin) {
    if (reinterpret_cast<volatile uint64_t*>(&ctl->seq_done)[0] == seq) break;
    if ((spin & 1023) == 0) {
      const cudaError_t q = cudaStreamQuery(v.st);
      if (q == cudaSuccess) {  // the server idled out before seeing the request
        if (reinterpret_cast<volatile uint64_t*>(&ctl->seq_done)[0] == seq) break;
        v.launched = false;
        CKS(server_launch(h, small));
      } else if (q != cudaErrorNotReady) {
        CK(q);
      }
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(10)) {
        reinterpret_cast<volatile int*>(&ctl->stop)[0] = 1;
        return fail(MOE_ERR_CUDA, "decision server: request %llu not served within 10 s",
                    (unsigned long long)seq);
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_seq_cst);
  if (!small) ++v.k;  // the multi-CTA server's barrier and completion counters
  return MOE_OK;
}

// Common launch + result copy of a DecisionArgs set up by the callers below.
static moe_status run_decision(moe_eamc* h, moe::DecisionArgs& a, size_t stage_rows,
                               const uint64_t* request_eam, const moe_slot_view* slots,
                               uint64_t n_slots, moe_candidate* out, uint64_t cap, uint64_t* n_out,
                               int64_t* victim) {
  const DevColl& c = h->c;
  cudaStream_t st = h->st;
  const uint64_t cells = (uint64_t)c.L * c.E;
  a.counts = c.counts;
  a.sqb = c.sqb;
  a.zm = c.L <= 64 ? c.zmask : nullptr;
  a.size = c.size;
  a.L = c.L;
  a.E = c.E;
  a.RB = c.RB;
  a.pref = h->pref.as<double>();
  a.dist = h->dist.as<double>();
  a.window = 0.01;  // kMatchWindow (policy.hpp:30)
  a.dmin2 = h->dstate.as<unsigned long long>();
  a.agg = h->agg.as<unsigned long long>();
  a.mcount = reinterpret_cast<uint32_t*>(h->dstate.as<uint8_t>() + 24);
  a.mlist = h->dmlist.as<uint32_t>();
  a.ckey = h->dkey.as<unsigned long long>();
  a.cid = h->did.as<uint32_t>();
  a.crank = h->drank.as<uint32_t>();
  a.nseg = h->dseg.as<uint32_t>();
  a.parity = (uint32_t)(h->dec_calls++ & 1);
  // results straight into pinned host memory (device-visible under UVA)
  a.out = h->cpin.as<moe_candidate>();
  a.n_out = h->fpin.as<uint32_t>();
  long long* vpin = reinterpret_cast<long long*>(h->fpin.as<uint8_t>() + 8);
  if (n_slots && request_eam) {
    CK(cudaMemcpyAsync(h->req.p, request_eam, cells * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(h->slots.p, slots, n_slots * sizeof(moe_slot_view), cudaMemcpyHostToDevice,
                       st));
    a.req = h->req.as<unsigned long long>();
    a.slots = h->slots.as<moe_slot_view>();
    a.n_slots = (uint32_t)n_slots;
    a.slot_pri = reinterpret_cast<double*>(h->slots.as<moe_slot_view>() + n_slots);
    a.victim = vpin;
    *vpin = -1;
  }
  if (c.L - a.cur > moe::kDecMaxLayers || c.E > moe::kDecMaxExperts)
    return fail(MOE_ERR_INVALID_ARGUMENT, "decision: shape %ux%u exceeds the order phases' limits",
                c.L, c.E);
  const uint32_t rows_above = a.cur + 1 < c.L ? c.L - a.cur - 1 : 0;
  const bool small_ok = !n_slots && a.do_dist && a.do_agg && c.size <= moe::kSmallMaxP &&
                        (uint64_t)rows_above * c.E <= moe::kSmallMaxCells && !small_off() &&
                        moe::decision_small_smem_max(c.L, c.RB) <= 200 * 1024;
  if (server_takes(h, n_slots)) {
    a.tprobe = nullptr;
    CKS(server_run(h, a, small_ok));
    const uint32_t n = *reinterpret_cast<volatile uint32_t*>(a.n_out);
    if (n_out) *n_out = n;
    if (n && out && cap) std::memcpy(out, a.out, std::min<uint64_t>(n, cap) * sizeof(moe_candidate));
    if (victim) *victim = -1;
    return MOE_OK;
  }
  if (small_ok) {
    // small collection: one CTA, no grid barriers
    const size_t smem = moe::decision_small_smem(c.size, c.L, c.E, c.RB, a.n_nz, a.cur);
    if (smem <= 200 * 1024) {
      a.tprobe = nullptr;
      if (dec_timing()) {
        CK(h->tprobe.ensure(64));
        a.tprobe = h->tprobe.as<unsigned long long>();
      }
      const auto t0 = std::chrono::steady_clock::now();
      CK(moe::launch_decision_small(a, c.cb, smem, st));
      const auto t1 = std::chrono::steady_clock::now();
      CK(cudaStreamSynchronize(st));
      if (dec_timing()) {
        const auto t2 = std::chrono::steady_clock::now();
        static double acc[11] = {0};
        static uint64_t cnt = 0;
        unsigned long long ts[8];
        CK(cudaMemcpy(ts, h->tprobe.p, sizeof ts, cudaMemcpyDeviceToHost));
        acc[0] += std::chrono::duration<double, std::micro>(t1 - t0).count();
        acc[1] += std::chrono::duration<double, std::micro>(t2 - t1).count();
        for (int i = 1; i < 4; ++i) acc[1 + i] += (ts[i] - ts[i - 1]) * 1e-3;
        // phase A split: rows + norms (0..4), the entry loop (4..5), the minimum (5..1)
        acc[5] += (ts[4] - ts[0]) * 1e-3;
        acc[6] += (ts[5] - ts[4]) * 1e-3;
        acc[7] += (ts[1] - ts[5]) * 1e-3;
        // phase C split: row sums (2..6), priorities + compaction (6..7), rank + output (7..3)
        acc[8] += (ts[6] - ts[2]) * 1e-3;
        acc[9] += (ts[7] - ts[6]) * 1e-3;
        acc[10] += (ts[3] - ts[7]) * 1e-3;
        if (++cnt % 58 == 0)
          fprintf(stderr, "small decision (avg of %llu): launch %.1f us, launch->done %.1f us | "
                          "A %.1f (rows %.1f, entries %.1f, min %.1f) B %.1f C %.1f (rowsum %.1f, "
                          "priorities %.1f, rank %.1f)\n",
                  (unsigned long long)cnt, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[5] / cnt,
                  acc[6] / cnt, acc[7] / cnt, acc[3] / cnt, acc[4] / cnt, acc[8] / cnt,
                  acc[9] / cnt, acc[10] / cnt);
      }
      const uint32_t n = *reinterpret_cast<volatile uint32_t*>(a.n_out);
      if (n_out) *n_out = n;
      if (n && out && cap)
        std::memcpy(out, a.out, std::min<uint64_t>(n, cap) * sizeof(moe_candidate));
      if (victim) *victim = -1;
      return MOE_OK;
    }
  }
  const int grid = moe::decision_grid(decision_sms(h), c.size, c.L, a.cur);
  const size_t smem = std::max(stage_rows, moe::decision_smem(c.L, c.E, c.RB, 0, a.cur, grid));
  if (smem > 220 * 1024)
    return fail(MOE_ERR_INVALID_ARGUMENT, "decision: shape %ux%u needs %zu B of shared memory",
                c.L, c.E, smem);
  a.tprobe = nullptr;
  if (dec_timing()) {
    CK(h->tprobe.ensure(64));
    a.tprobe = h->tprobe.as<unsigned long long>();
  }
  const auto t0 = std::chrono::steady_clock::now();
  a.bar = reinterpret_cast<uint32_t*>(h->dstate.as<uint8_t>() + 16);
  a.bar_base = h->bar_base;
  CK(moe::launch_decision(a, c.cb, grid, smem, st));
  h->bar_base += moe::kDecBarriers * (uint32_t)grid;
  const auto t1 = std::chrono::steady_clock::now();
  CK(cudaStreamSynchronize(st));
  const auto t2 = std::chrono::steady_clock::now();
  if (dec_timing()) {
    static double acc[9] = {0};
    static uint64_t cnt = 0;
    unsigned long long ts[8];
    CK(cudaMemcpy(ts, h->tprobe.p, sizeof ts, cudaMemcpyDeviceToHost));
    acc[0] += std::chrono::duration<double, std::micro>(t1 - t0).count();
    acc[1] += std::chrono::duration<double, std::micro>(t2 - t1).count();
    for (int i = 1; i < 8; ++i) acc[1 + i] += (ts[i] - ts[i - 1]) * 1e-3;
    if (++cnt % 58 == 0)
      fprintf(stderr,
              "decision (avg of %llu): launch %.1f us, launch->done %.1f us | A %.1f sync %.1f "
              "B %.1f sync %.1f C1 %.1f sync %.1f C2 %.1f\n",
              (unsigned long long)cnt, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt,
              acc[4] / cnt, acc[5] / cnt, acc[6] / cnt, acc[7] / cnt, acc[8] / cnt);
  }
  const uint32_t n = *reinterpret_cast<volatile uint32_t*>(a.n_out);
  if (n_out) *n_out = n;
  if (n && out && cap) std::memcpy(out, a.out, std::min<uint64_t>(n, cap) * sizeof(moe_candidate));
  if (victim) *victim = n_slots ? *reinterpret_cast<volatile long long*>(vpin) : -1;
  return MOE_OK;
}

// The engine's decision on a host probe.  The probe is narrowed to the
// storage width on the host (padded rows, so the explicit rows ship inside
// the launch parameters), and the per-entry layer sums over the rows it
// shares with the previous call's probe are reused from pref (k_decision
// phase A).  *handled = false: the probe has more explicit rows than the
// kernel stages; decide_impl then takes the row-parallel distance pass.
static moe_status decide_fused(moe_eamc* h, const uint64_t* probe, uint32_t cur, int filter,
                               const uint64_t* request_eam, const moe_slot_view* slots,
                               uint64_t n_slots, moe_candidate* out, uint64_t cap,
                               uint64_t* n_out, int64_t* victim, bool* handled) {
  *handled = false;
  const auto th0 = std::chrono::steady_clock::now();
  DevColl& c = h->c;
  const uint32_t L = c.L, E = c.E;
  const uint64_t cells = (uint64_t)L * E;
  uint8_t* hb = nullptr;
  for (;;) {  // narrow at the storage width; widen and redo when a count needs it
    CK(h->dpin.ensure((size_t)L * c.RB + 64));
    hb = h->dpin.as<uint8_t>();
    uint64_t o = 0;
    const uint64_t row_b = (uint64_t)E * c.cb;
    for (uint32_t l = 0; l < L; ++l) {
      o |= moe::host::pack_counts_serial(probe + (uint64_t)l * E, E, c.cb, hb + (size_t)l * c.RB);
      std::memset(hb + (size_t)l * c.RB + row_b, 0, c.RB - row_b);
    }
    if (o > width_max(c.cb)) {
      const uint64_t mx = *std::max_element(probe, probe + cells);
      if (mx > width_max(c.cb)) {
        CKS(widen_for(h, mx));
        continue;
      }
    }
    // the reference's fp64 sums are exact only while sum c^2 < 2^53 per row
    if ((double)o * (double)o * (double)E >= 9007199254740992.0)
      for (uint32_t l = 0; l < L; ++l) {
        uint64_t ss = 0;
        for (uint32_t e = 0; e < E; ++e) {
          const uint64_t v = probe[(uint64_t)l * E + e];
          ss = v >= (1ull << 27) ? (1ull << 53) : std::min<uint64_t>(ss + v * v, 1ull << 53);
        }
        if (ss >= (1ull << 53)) CKS(widen_for(h, ~0ull));  // MOE_ERR_OVERFLOW
      }
    break;
  }
  CKS(dec_scratch(h, n_slots));
  const uint32_t RB = c.RB;
  // layer-prefix reuse: rows [0, dec_keep] unchanged, same collection contents
  uint32_t j0 = 0;
  if (h->dec_keep >= 0 && h->dec_version == h->version && h->dec_cb == c.cb &&
      std::memcmp(hb, h->dec_rows.data(), (size_t)(h->dec_keep + 1) * RB) == 0)
    j0 = (uint32_t)h->dec_keep + 1;
  const bool store = (int64_t)cur > h->dec_keep || j0 == 0;
  const uint32_t keep = store ? cur : L;  // L: leave pref as it is
  std::vector<uint16_t>& nz = h->dec_nz;
  nz.clear();
  for (uint32_t l = j0; l < L; ++l) {
    const uint64_t* r = reinterpret_cast<const uint64_t*>(hb + (size_t)l * RB);
    bool any = false;
    for (uint32_t w = 0; w < RB / 8 && !any; ++w) any = r[w] != 0;
    if (any) nz.push_back((uint16_t)l);
  }
  const uint32_t n_nz = (uint32_t)nz.size();
  if (n_nz > moe::kDecMaxNz || L > 65535) return MOE_OK;  // decide_impl's general path
  // explicit rows: through the last nonzero probe row and the stored row
  uint32_t hi = n_nz ? nz.back() : 0;
  if (keep < L) hi = std::max(hi, keep);
  if (!n_nz && keep >= L) hi = j0 ? j0 - 1 : 0;  // nothing explicit beyond the cached prefix
  moe::DecisionArgs& a = h->dargs;
  a.do_dist = 1;
  a.do_agg = 1;
  a.dmin_ext = nullptr;
  a.n_nz = n_nz;
  a.j0 = j0;
  a.hi = hi;
  a.keep = keep;
  a.cur = cur;
  a.filter = filter;
  a.req = nullptr;
  a.slots = nullptr;
  a.n_slots = 0;
  a.slot_pri = nullptr;
  a.victim = nullptr;
  a.rows_inline = n_nz <= moe::kDecInlineNz && (size_t)n_nz * RB <= moe::kDecInlineBytes;
  if (a.rows_inline) {
    for (uint32_t i = 0; i < n_nz; ++i) {
      a.inline_nz[i] = nz[i];
      std::memcpy(a.inline_rows + (size_t)i * RB, hb + (size_t)nz[i] * RB, RB);
    }
    a.rows = nullptr;
    a.nz = nullptr;
  } else {  // one DMA of the explicit rows and their list
    const size_t rows_b = (size_t)n_nz * RB, nz_b = ((size_t)n_nz * 2 + 15) & ~(size_t)15;
    CK(h->xpin.ensure(rows_b + nz_b));
    CK(h->xdev.ensure(rows_b + nz_b));
    for (uint32_t i = 0; i < n_nz; ++i)
      std::memcpy(h->xpin.as<uint8_t>() + (size_t)i * RB, hb + (size_t)nz[i] * RB, RB);
    std::memcpy(h->xpin.as<uint8_t>() + rows_b, nz.data(), (size_t)n_nz * 2);
    if (server_takes(h, n_slots)) {  // the server copies them from pinned memory itself
      a.rows = h->xpin.as<uint8_t>();
      a.nz = reinterpret_cast<const uint16_t*>(h->xpin.as<uint8_t>() + rows_b);
    } else {
      CK(cudaMemcpyAsync(h->xdev.p, h->xpin.p, rows_b + nz_b, cudaMemcpyHostToDevice, h->st));
      a.rows = h->xdev.as<uint8_t>();
      a.nz = reinterpret_cast<const uint16_t*>(h->xdev.as<uint8_t>() + rows_b);
    }
  }
  const auto th1 = std::chrono::steady_clock::now();
  CKS(run_decision(h, a, (size_t)n_nz * RB, request_eam, slots, n_slots, out, cap, n_out, victim));
  if (dec_timing()) {
    static double acc = 0;
    static uint64_t cnt = 0;
    acc += std::chrono::duration<double, std::micro>(th1 - th0).count();
    if (++cnt % 58 == 0)
      fprintf(stderr, "decision host prep (avg of %llu): %.1f us\n", (unsigned long long)cnt, acc / cnt);
  }
  if (store) {
    h->dec_rows.assign(hb, hb + (size_t)(cur + 1) * RB);
    h->dec_keep = cur;
    h->dec_version = h->version;
    h->dec_cb = c.cb;
  }
  *handled = true;
  return MOE_OK;
}

static moe_status decide_impl(moe_eamc* h, const moe_shape* shape, const uint64_t* cur_eam,
                              uint32_t current_layer, int filter, int do_prefetch,
                              const uint64_t* request_eam, const moe_slot_view* slots,
                              uint64_t n_slots, moe_candidate* out, uint64_t cap, uint64_t* n_out,
                              int64_t* victim, double* slot_pri) {
  const uint32_t L = shape->n_layers, E = shape->n_experts_per_layer;
  const uint64_t cells = (uint64_t)L * E;
  cudaStream_t st = h->st;
  CK(h->small.ensure(256));
  CK(h->pin.ensure(256));
  if (do_prefetch && h->c.size > 0 && !slot_pri) {
    bool handled = false;
    CKS(decide_fused(h, cur_eam, current_layer, filter, request_eam, slots, n_slots, out, cap,
                     n_out, victim, &handled));
    if (handled) return MOE_OK;
    // more explicit probe rows than the fused kernel stages: row-parallel
    // exact distances + minimum, then the fused kernel's aggregation + order
    for (;;) {
      DevProbes pr;
      CKS(launch_exact_distances(h, cur_eam, st, &pr));
      CK(cudaMemcpyAsync(h->pin.p, h->small.p, 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      bool ok = false;
      CKS(check_width(h, *h->pin.as<unsigned long long>(), &ok));
      if (ok) break;
    }
    CKS(dec_scratch(h, n_slots));
    moe::DecisionArgs& a = h->dargs;
    a.do_dist = 0;
    a.do_agg = 1;
    a.dmin_ext = reinterpret_cast<const unsigned long long*>(h->small.as<uint8_t>() + 224);
    a.n_nz = 0;
    a.rows_inline = 1;
    a.j0 = 0;
    a.hi = 0;
    a.keep = L;
    a.cur = current_layer;
    a.filter = filter;
    a.req = nullptr;
    a.slots = nullptr;
    a.n_slots = 0;
    a.slot_pri = nullptr;
    a.victim = nullptr;
    return run_decision(h, a, 0, request_eam, slots, n_slots, out, cap, n_out, victim);
  }
  // eviction scoring only (cache_priority / select_eviction_victim), or an
  // empty collection: k_decide over the slot views
  if (n_out) *n_out = 0;
  unsigned long long* req = nullptr;
  if (request_eam) {
    CK(h->req.ensure(cells * 8));
    CK(cudaMemcpyAsync(h->req.p, request_eam, cells * 8, cudaMemcpyHostToDevice, st));
    req = h->req.as<unsigned long long>();
  }
  moe_slot_view* dslots = nullptr;
  double* dpri = nullptr;
  if (n_slots) {
    CK(h->slots.ensure(n_slots * (sizeof(moe_slot_view) + 8)));
    CK(cudaMemcpyAsync(h->slots.p, slots, n_slots * sizeof(moe_slot_view), cudaMemcpyHostToDevice,
                       st));
    dslots = h->slots.as<moe_slot_view>();
    if (slot_pri) dpri = reinterpret_cast<double*>(dslots + n_slots);
  }
  long long* dv = reinterpret_cast<long long*>(h->small.as<uint8_t>() + 192);
  if (victim || slot_pri)
    CK(moe::launch_decide(h->agg.as<unsigned long long>(), L, E, current_layer, filter, 0, req,
                          dslots, n_slots, nullptr, nullptr, victim ? dv : nullptr, dpri, st));
  CK(cudaMemcpyAsync(h->pin.p, h->small.p, 256, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (victim) *victim = *reinterpret_cast<const long long*>(h->pin.as<uint8_t>() + 192);
  if (slot_pri && n_slots) CK(cudaMemcpy(slot_pri, dpri, n_slots * 8, cudaMemcpyDeviceToHost));
  return MOE_OK;
}

moe_status moe_prefetch_priorities(const moe_eamc* hc, const uint64_t* cur_eam,
                                   uint32_t current_layer, int apply_floor_filter,
                                   moe_candidate* out, uint64_t cap, uint64_t* n_out) {
  HandleLock hl_(hc);
  moe_eamc* h = const_cast<moe_eamc*>(hc);
  if (!h || !cur_eam || !n_out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  // policy.cpp:91-93
  if (current_layer >= h->shape.n_layers)
    return fail(MOE_ERR_OUT_OF_RANGE, "prefetch_priorities: current_layer out of range");
  *n_out = 0;
  if (h->sh)
    return moe::abi::sh_prefetch(h, cur_eam, current_layer, apply_floor_filter, out, cap, n_out);
  if (h->c.size == 0) return MOE_OK;
  DeviceGuard dg(h->device);
  return decide_impl(h, &h->shape, cur_eam, current_layer, apply_floor_filter, 1, nullptr, nullptr,
                     0, out, cap, n_out, nullptr, nullptr);
}

// ---- P-sharded decision (K4 window aggregate + K5) -------------
// prefetch_priorities (policy.cpp:88-126) over a collection sharded by P:
// (1) every rank's exact distances and local minimum, (2) MIN all-reduce of
// the minimum's bits, (3) every rank's window members (d <= d_min + window,
// the fp64 add of eam.cpp:143) aggregated into u64 [L][E] rows > current
// layer, (4) SUM all-reduce, (5) priorities / floor filter / order from the
// summed rows.  Integer sums and a min are order-independent, so the result is
// bit-identical to the unsharded call.

moe_status moe_eamc_window_min_device(const moe_eamc* hc, const uint64_t* cur_eam,
                                      uint64_t* d_min_bits, void* stream) {
  HandleLock hl_(hc);
  moe_eamc* h = const_cast<moe_eamc*>(hc);
  if (!h || !cur_eam || !d_min_bits) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (h->sh) return fail(MOE_ERR_INVALID_ARGUMENT, "device decision steps are per shard handle");
  DeviceGuard dg(h->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->st;
  CK(h->small.ensure(256));
  CK(h->pin.ensure(256));
  if (h->c.size == 0) {  // an empty shard contributes +inf
    *h->pin.as<uint64_t>() = 0x7ff0000000000000ull;
    CK(cudaMemcpyAsync(d_min_bits, h->pin.p, 8, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    return MOE_OK;
  }
  for (;;) {  // the width check needs the host: one synchronisation
    DevProbes pr;
    CKS(launch_exact_distances(h, cur_eam, st, &pr));
    CK(cudaMemcpyAsync(h->pin.p, h->small.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    bool ok = false;
    CKS(check_width(h, *h->pin.as<unsigned long long>(), &ok));
    if (ok) break;
  }
  CK(cudaMemcpyAsync(d_min_bits, h->small.as<uint8_t>() + 224, 8, cudaMemcpyDeviceToDevice, st));
  return MOE_OK;
}

moe_status moe_eamc_window_aggregate_device(const moe_eamc* hc, uint32_t current_layer,
                                            double window, const uint64_t* d_min_bits,
                                            uint64_t* agg, void* stream) {
  HandleLock hl_(hc);
  moe_eamc* h = const_cast<moe_eamc*>(hc);
  if (!h || !d_min_bits || !agg) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (h->sh) return fail(MOE_ERR_INVALID_ARGUMENT, "device decision steps are per shard handle");
  if (current_layer >= h->shape.n_layers)
    return fail(MOE_ERR_OUT_OF_RANGE, "prefetch_priorities: current_layer out of range");
  DeviceGuard dg(h->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->st;
  const uint64_t cells = (uint64_t)h->shape.n_layers * h->shape.n_experts_per_layer;
  CK(cudaMemsetAsync(agg, 0, cells * 8, st));
  if (h->c.size == 0) return MOE_OK;
  CK(h->small.ensure(256));
  CK(h->mem.ensure((size_t)h->c.size * 4));
  CK(moe::launch_member_agg(h->c, h->dist.as<double>(),
                            reinterpret_cast<const unsigned long long*>(d_min_bits), window,
                            current_layer, h->mem.as<uint32_t>(), h->small.as<uint32_t>() + 10,
                            reinterpret_cast<unsigned long long*>(agg), h->n_sm, st));
  return MOE_OK;
}

moe_status moe_eamc_prefetch_order_device(const moe_eamc* hc, const uint64_t* agg,
                                          uint32_t current_layer, int apply_floor_filter,
                                          moe_candidate* out, uint32_t* n_out, void* stream) {
  HandleLock hl_(hc);
  moe_eamc* h = const_cast<moe_eamc*>(hc);
  if (!h || !agg || !out || !n_out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (h->sh) return fail(MOE_ERR_INVALID_ARGUMENT, "device decision steps are per shard handle");
  const uint32_t L = h->shape.n_layers, E = h->shape.n_experts_per_layer;
  if (current_layer >= L)
    return fail(MOE_ERR_OUT_OF_RANGE, "prefetch_priorities: current_layer out of range");
  DeviceGuard dg(h->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->st;
  CKS(dec_scratch(h, 0));
  // the fused decision kernel's order phases on the caller's aggregate
  moe::DecisionArgs& a = h->dargs;
  a = moe::DecisionArgs{};
  a.do_dist = 0;
  a.do_agg = 0;
  a.rows_inline = 1;
  a.keep = L;
  a.cur = current_layer;
  a.filter = apply_floor_filter;
  a.L = L;
  a.E = E;
  a.RB = h->c.RB;
  a.size = 0;
  a.agg = const_cast<unsigned long long*>(reinterpret_cast<const unsigned long long*>(agg));
  a.dmin2 = h->dstate.as<unsigned long long>();
  a.ckey = h->dkey.as<unsigned long long>();
  a.cid = h->did.as<uint32_t>();
  a.crank = h->drank.as<uint32_t>();
  a.nseg = h->dseg.as<uint32_t>();
  a.parity = (uint32_t)(h->dec_calls++ & 1);
  a.out = out;
  a.n_out = n_out;
  if (L - current_layer > moe::kDecMaxLayers || E > moe::kDecMaxExperts)
    return fail(MOE_ERR_INVALID_ARGUMENT, "decision: shape %ux%u exceeds the order phases' limits",
                L, E);
  const int grid = moe::decision_grid(decision_sms(h), 0, L, current_layer);
  const size_t smem = moe::decision_smem(L, E, h->c.RB, 0, current_layer, grid);
  if (smem > 220 * 1024)
    return fail(MOE_ERR_INVALID_ARGUMENT, "decision: shape %ux%u needs %zu B of shared memory", L,
                E, smem);
  // its own barrier counter: this launch runs on the caller's stream
  a.bar = reinterpret_cast<uint32_t*>(h->dstate.as<uint8_t>() + 20);
  a.bar_base = h->bar_base2;
  CK(moe::launch_decision(a, h->c.cb, grid, smem, st));
  h->bar_base2 += moe::kDecBarriers * (uint32_t)grid;
  return MOE_OK;
}

moe_status moe_decide(const moe_eamc* hc, const uint64_t* cur_eam, uint32_t current_layer,
                      const uint64_t* request_eam, const moe_slot_view* slots, uint64_t n_slots,
                      moe_candidate* out, uint64_t cap, uint64_t* n_out, int64_t* victim) {
  HandleLock hl_(hc);
  moe_eamc* h = const_cast<moe_eamc*>(hc);
  if (!h || !cur_eam || !request_eam || (!slots && n_slots))
    return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (current_layer >= h->shape.n_layers)
    return fail(MOE_ERR_OUT_OF_RANGE, "prefetch_priorities: current_layer out of range");
  for (uint64_t i = 0; i < n_slots; ++i)
    if (slots[i].layer_idx >= h->shape.n_layers ||
        slots[i].expert_idx >= h->shape.n_experts_per_layer)
      return fail(MOE_ERR_OUT_OF_RANGE, "cache_priority: expert out of range");
  if (h->sh) {  // the sharded prefetch order, then the (unsharded) eviction scoring
    uint64_t n = 0;
    CKS(moe::abi::sh_prefetch(h, cur_eam, current_layer, 1, out, cap, &n));
    if (n_out) *n_out = n;
    if (victim) CKS(moe_select_eviction_victim(&h->shape, request_eam, slots, n_slots, victim));
    return MOE_OK;
  }
  DeviceGuard dg(h->device);
  return decide_impl(h, &h->shape, cur_eam, current_layer, 1, 1, request_eam, slots, n_slots, out,
                     cap, n_out, victim, nullptr);
}

moe_status moe_cache_priority(const moe_shape* shape, const uint64_t* request_eam,
                              uint32_t layer, uint32_t expert, double* out) {
  CKS(check_shape(shape));
  if (!request_eam || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  // policy.cpp:130-131
  if (layer >= shape->n_layers || expert >= shape->n_experts_per_layer)
    return fail(MOE_ERR_OUT_OF_RANGE, "cache_priority: expert out of range");
  ScratchLease lease;
  CKS(scratch_handle(shape, &lease));
  moe_eamc* h = lease.h;
  moe_slot_view v{};
  v.slot = 0;
  v.layer_idx = layer;
  v.expert_idx = expert;
  return decide_impl(h, shape, nullptr, 0, 0, 0, request_eam, &v, 1, nullptr, 0, nullptr, nullptr,
                     out);
}

moe_status moe_select_eviction_victim(const moe_shape* shape, const uint64_t* request_eam,
                                      const moe_slot_view* slots, uint64_t n_slots,
                                      int64_t* victim) {
  CKS(check_shape(shape));
  if (!request_eam || !victim || (!slots && n_slots))
    return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  for (uint64_t i = 0; i < n_slots; ++i) {
    if (slots[i].prefetch_protected || slots[i].pinned) continue;  // never priced
    if (slots[i].layer_idx >= shape->n_layers || slots[i].expert_idx >= shape->n_experts_per_layer)
      return fail(MOE_ERR_OUT_OF_RANGE, "cache_priority: expert out of range");
  }
  *victim = -1;
  if (n_slots == 0) return MOE_OK;
  ScratchLease lease;
  CKS(scratch_handle(shape, &lease));
  return decide_impl(lease.h, shape, nullptr, 0, 0, 0, request_eam, slots, n_slots, nullptr, 0,
                     nullptr, victim, nullptr);
}

moe_status moe_eam_trace_device(const moe_shape* shape, const void* topk_idx, int idx_bytes,
                                uint64_t n_tokens, const uint64_t* offsets, uint64_t n_requests,
                                uint32_t* counts_u32, int* bad_index_flag, void* stream) {
  CKS(check_shape(shape));
  if (idx_bytes != 1 && idx_bytes != 2 && idx_bytes != 4)
    return fail(MOE_ERR_INVALID_ARGUMENT, "idx_bytes must be 1, 2 or 4");
  if (!bad_index_flag || ((!topk_idx || !offsets || !counts_u32) && n_requests))
    return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  int dev = 0, n_sm = 0;
  cudaGetDevice(&dev);
  CKS(device_ok(dev, &n_sm));
  // no scratch: the kernels accumulate into counts_u32 directly and roll their
  // additions back on an out-of-range id (trace.cu)
  CK(moe::launch_trace(topk_idx, idx_bytes, n_tokens, shape->n_layers, shape->n_experts_per_layer,
                       shape->top_k, offsets, n_requests, counts_u32, 4, bad_index_flag, n_sm,
                       static_cast<cudaStream_t>(stream)));
  return MOE_OK;
}

// Pageable host <-> device transfers through a ring of pinned staging
// buffers: the host pool copies chunk k into its slot while the DMA of chunk
// k-1 runs (a pageable cudaMemcpy moves ~3-5 GB/s; this runs at PCIe rate).
struct StagingRing {
  static constexpr int kSlots = 4;
  static constexpr size_t kChunk = 16u << 20;
  PinBuf slot[kSlots];
  cudaEvent_t ev[kSlots] = {};
  bool init = false;
  moe_status setup() {
    if (init) return MOE_OK;
    for (int i = 0; i < kSlots; ++i) {
      CK(slot[i].ensure(kChunk));
      CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    init = true;
    return MOE_OK;
  }
};

struct CopyJob {
  uint8_t* dst;
  const uint8_t* src;
  size_t n;
  int parts;
};

static void copy_task(void* vj, int t) {
  CopyJob* j = static_cast<CopyJob*>(vj);
  const size_t a = j->n * t / j->parts, b = j->n * (t + 1) / j->parts;
  std::memcpy(j->dst + a, j->src + a, b - a);
}

static void pool_memcpy(void* dst, const void* src, size_t n) {
  CopyJob j{static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), n,
            (int)std::max<size_t>(1, std::min<size_t>((size_t)moe::host::pool_threads(),
                                                      n / (1u << 20)))};
  moe::host::pool_run(j.parts, copy_task, &j);
}

static moe_status h2d_staged(StagingRing& r, void* dst, const void* src, size_t n,
                             cudaStream_t st) {
  CKS(r.setup());
  size_t k = 0;
  for (size_t off = 0; off < n; off += StagingRing::kChunk, ++k) {
    const int sl = (int)(k % StagingRing::kSlots);
    const size_t m = std::min(StagingRing::kChunk, n - off);
    CK(cudaEventSynchronize(r.ev[sl]));  // the slot's previous DMA (this or an earlier call)
    pool_memcpy(r.slot[sl].p, static_cast<const uint8_t*>(src) + off, m);
    CK(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + off, r.slot[sl].p, m, cudaMemcpyHostToDevice,
                       st));
    CK(cudaEventRecord(r.ev[sl], st));
  }
  return MOE_OK;
}

static moe_status d2h_staged(StagingRing& r, void* dst, const void* src, size_t n,
                             cudaStream_t st) {
  CKS(r.setup());
  const size_t nchunks = (n + StagingRing::kChunk - 1) / StagingRing::kChunk;
  // keep kSlots DMAs in flight; drain chunk k - kSlots + 1 once its slot is needed
  for (size_t k = 0; k < nchunks + StagingRing::kSlots - 1; ++k) {
    if (k < nchunks) {
      const int sl = (int)(k % StagingRing::kSlots);
      if (k >= StagingRing::kSlots) {  // slot busy with chunk k - kSlots: drain it first
        const size_t kd = k - StagingRing::kSlots;
        CK(cudaEventSynchronize(r.ev[sl]));
        const size_t off = kd * StagingRing::kChunk;
        pool_memcpy(static_cast<uint8_t*>(dst) + off, r.slot[sl].p,
                    std::min(StagingRing::kChunk, n - off));
      }
      const size_t off = k * StagingRing::kChunk;
      CK(cudaMemcpyAsync(r.slot[sl].p, static_cast<const uint8_t*>(src) + off,
                         std::min(StagingRing::kChunk, n - off), cudaMemcpyDeviceToHost, st));
      CK(cudaEventRecord(r.ev[sl], st));
    }
  }
  // drain the last min(nchunks, kSlots) chunks
  const size_t first = nchunks > (size_t)StagingRing::kSlots ? nchunks - StagingRing::kSlots : 0;
  for (size_t kd = first; kd < nchunks; ++kd) {
    const int sl = (int)(kd % StagingRing::kSlots);
    CK(cudaEventSynchronize(r.ev[sl]));
    const size_t off = kd * StagingRing::kChunk;
    pool_memcpy(static_cast<uint8_t*>(dst) + off, r.slot[sl].p,
                std::min(StagingRing::kChunk, n - off));
  }
  return MOE_OK;
}

moe_status moe_eam_trace(const moe_shape* shape, const void* topk_idx, int idx_bytes,
                         uint64_t n_tokens, const uint64_t* offsets, uint64_t n_requests,
                         uint64_t* counts) {
  CKS(check_shape(shape));
  if (idx_bytes != 1 && idx_bytes != 2 && idx_bytes != 4)
    return fail(MOE_ERR_INVALID_ARGUMENT, "idx_bytes must be 1, 2 or 4");
  if (n_requests == 0) return MOE_OK;
  if (!topk_idx || !offsets || !counts) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  for (uint64_t r = 0; r < n_requests; ++r)
    if (offsets[r] > offsets[r + 1])
      return fail(MOE_ERR_INVALID_ARGUMENT, "request offsets must be non-decreasing");
  if (offsets[n_requests] > n_tokens)
    return fail(MOE_ERR_INVALID_ARGUMENT, "request offsets exceed n_tokens");
  int dev = 0, n_sm = 0;
  cudaGetDevice(&dev);
  CKS(device_ok(dev, &n_sm));
  const uint64_t cells = (uint64_t)shape->n_layers * shape->n_experts_per_layer;
  const uint64_t in_bytes = n_tokens * shape->n_layers * shape->top_k * idx_bytes;
  // persistent per-device state: stream, buffers, pinned staging ring
  struct TraceState {
    cudaStream_t st = nullptr;
    DevBuf din, doff, dcnt, dbad;
    PinBuf hbad;
    StagingRing ring;
  };
  static std::mutex mu;
  static TraceState states[64];
  std::lock_guard<std::mutex> lock(mu);
  TraceState& S = states[dev & 63];
  if (!S.st) CK(cudaStreamCreateWithFlags(&S.st, cudaStreamNonBlocking));
  cudaStream_t st = S.st;
  CK(S.din.ensure(std::max<uint64_t>(in_bytes, 16)));
  CK(S.doff.ensure((n_requests + 1) * 8));
  CK(S.dcnt.ensure(n_requests * cells * 8));
  CK(S.dbad.ensure(4));
  CK(S.hbad.ensure(4));
  CKS(h2d_staged(S.ring, S.din.p, topk_idx, in_bytes, st));
  CK(cudaMemcpyAsync(S.doff.p, offsets, (n_requests + 1) * 8, cudaMemcpyHostToDevice, st));
  CKS(h2d_staged(S.ring, S.dcnt.p, counts, n_requests * cells * 8, st));
  CK(cudaMemsetAsync(S.dbad.p, 0, 4, st));
  CK(moe::launch_trace(S.din.p, idx_bytes, n_tokens, shape->n_layers,
                       shape->n_experts_per_layer, shape->top_k, S.doff.as<uint64_t>(),
                       n_requests, S.dcnt.p, 8, S.dbad.as<int>(), n_sm, st));
  CK(cudaMemcpyAsync(S.hbad.p, S.dbad.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (*S.hbad.as<int>())  // all-or-nothing (eam.cpp:42-47): the caller's counts untouched
    return fail(MOE_ERR_OUT_OF_RANGE, "Eam::record: expert index out of range");
  CKS(d2h_staged(S.ring, counts, S.dcnt.p, n_requests * cells * 8, st));
  return MOE_OK;
}

moe_status moe_traces_request_eams(const char* path, const moe_shape* shape, moe_phase phase,
                                   uint64_t* counts, uint64_t cap, uint64_t* n_eams) {
  if (!path || !shape || !n_eams || (cap && !counts))
    return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  CKS(check_shape(shape));
  std::vector<uint64_t> c;
  uint64_t n = 0;
  std::string err;
  if (!moe::host::ingest_request_eams(path, shape->n_layers, shape->n_experts_per_layer,
                                      phase == MOE_PHASE_PREFILL ? 0 : 1, &c, &n, &err))
    return fail(MOE_ERR_TRACE, "%s", err.c_str());
  *n_eams = n;
  if (cap) std::copy(c.begin(), c.begin() + std::min(n, cap) * shape->n_layers *
                                               shape->n_experts_per_layer, counts);
  return MOE_OK;
}

moe_status moe_eamc_build_from_traces(moe_eamc* h, const char* path, uint64_t* n_inserted) {
  HandleLock hl_(h);
  if (!h || !path) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  std::vector<uint64_t> c;
  uint64_t n = 0;
  std::string err;
  if (!moe::host::ingest_request_eams(path, h->c.L, h->c.E, h->phase, &c, &n, &err))
    return fail(MOE_ERR_TRACE, "%s", err.c_str());
  CKS(moe_eamc_build(h, c.data(), n, nullptr));
  if (n_inserted) *n_inserted = n;
  return MOE_OK;
}

moe_status moe_eamc_capacity_bound(const moe_shape* shape, double similarity, uint64_t* out) {
  CKS(check_shape(shape));
  if (!out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  const uint64_t v = moe::host::capacity_bound(shape->n_layers, shape->n_experts_per_layer, similarity);
  if (!v)
    return fail(MOE_ERR_INVALID_ARGUMENT,
                "eamc_capacity_bound: supported similarity levels are 0.75 and 0.98");
  *out = v;
  return MOE_OK;
}

moe_status moe_eamc_save(const moe_eamc* hc, const char* path) {
  HandleLock hl_(hc);
  moe_eamc* h = const_cast<moe_eamc*>(hc);
  if (!h || !path) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (h->sh) return moe::abi::sh_save(h, path, false);
  DeviceGuard dg(h->device);
  const DevColl& c = h->c;
  const uint64_t LR = (uint64_t)c.L * c.RB;
  std::vector<uint8_t> rows((size_t)c.size * LR);
  std::vector<uint64_t> seqs(c.size);
  if (c.size) {
    CK(cudaMemcpy(rows.data(), c.counts, rows.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(seqs.data(), c.seq, c.size * 8, cudaMemcpyDeviceToHost));
  }
  moe::host::Snapshot snap;
  snap.L = c.L;
  snap.E = c.E;
  snap.top_k = h->shape.top_k;
  snap.phase = h->phase;
  snap.capacity = h->capacity;
  snap.next_seq = h->next_seq;
  snap.seqs = std::move(seqs);
  snap.counts.resize((size_t)c.size * c.L * c.E);
  for (uint64_t i = 0; i < c.size; ++i)
    for (uint32_t l = 0; l < c.L; ++l)
      for (uint32_t e = 0; e < c.E; ++e) {
        const uint8_t* r = rows.data() + i * LR + (uint64_t)l * c.RB;
        snap.counts[(i * c.L + l) * c.E + e] = unpack_count(r, e, c.cb);
      }
  std::string err;
  if (!moe::host::save_snapshot(path, snap, &err)) return fail(MOE_ERR_SNAPSHOT, "%s", err.c_str());
  return MOE_OK;
}

// ---- binary snapshots: the fast path next to JSON v1 ----------------------
// Layout (little-endian): 64-byte header {char magic[8] = "MOEEAMCB"; u32
// version = 1; u32 n_layers, n_experts_per_layer, top_k, phase (0 prefill,
// 1 decode), count_bytes (1, 2, 4); u64 capacity, size, next_seq; 8 bytes
// zero}, then seq[size] u64, then counts [size][L][E] of count_bytes each
// (the device storage width, unpadded).  Slot order, seqs and next_seq are
// those of Eamc::save (eam.cpp:184-205); the counts move as one D2H / H2D of
// the storage-width rows instead of a decimal JSON text.
namespace {
struct BinHeader {
  char magic[8];
  uint32_t version, L, E, top_k, phase, cb;
  uint64_t capacity, size, next_seq, zero;
};
static_assert(sizeof(BinHeader) == 64, "binary snapshot header");
constexpr char kBinMagic[8] = {'M', 'O', 'E', 'E', 'A', 'M', 'C', 'B'};

struct StripJob {
  const uint8_t* rows;  // [n][L][RB]
  uint8_t* dst;         // [n][L][E*cb]
  uint64_t n;
  uint32_t L, RB, rb;
  int parts;
};
void strip_task(void* vj, int t) {
  StripJob* j = static_cast<StripJob*>(vj);
  const uint64_t a = j->n * t / j->parts, b = j->n * (t + 1) / j->parts;
  for (uint64_t i = a; i < b; ++i)
    for (uint32_t l = 0; l < j->L; ++l)
      std::memcpy(j->dst + (i * j->L + l) * j->rb, j->rows + (i * j->L + l) * j->RB, j->rb);
}
}  // namespace

moe_status moe_eamc_save_binary(const moe_eamc* hc, const char* path) {
  HandleLock hl_(hc);
  moe_eamc* h = const_cast<moe_eamc*>(hc);
  if (!h || !path) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (h->sh) return moe::abi::sh_save(h, path, true);
  DeviceGuard dg(h->device);
  const DevColl& c = h->c;
  const uint32_t rb = c.E * (uint32_t)c.cb;
  BinHeader hd{};
  std::memcpy(hd.magic, kBinMagic, 8);
  hd.version = 1;
  hd.L = c.L;
  hd.E = c.E;
  hd.top_k = h->shape.top_k;
  hd.phase = (uint32_t)h->phase;
  hd.cb = (uint32_t)c.cb;
  hd.capacity = h->capacity;
  hd.size = c.size;
  hd.next_seq = h->next_seq;
  std::vector<uint8_t> buf(sizeof hd + (size_t)c.size * 8 + (size_t)c.size * c.L * rb);
  std::memcpy(buf.data(), &hd, sizeof hd);
  if (c.size) {
    CK(cudaMemcpy(buf.data() + sizeof hd, c.seq, (size_t)c.size * 8, cudaMemcpyDeviceToHost));
    const uint64_t LR = (uint64_t)c.L * c.RB;
    PinBuf rows;
    CK(rows.ensure((size_t)c.size * LR));
    CK(cudaMemcpy(rows.p, c.counts, (size_t)c.size * LR, cudaMemcpyDeviceToHost));
    StripJob j{rows.as<uint8_t>(), buf.data() + sizeof hd + (size_t)c.size * 8, c.size, c.L,
               c.RB, rb,
               (int)std::max<uint64_t>(1, std::min<uint64_t>(moe::host::pool_threads(),
                                                             c.size / 1024 + 1))};
    moe::host::pool_run(j.parts, strip_task, &j);
  }
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(MOE_ERR_SNAPSHOT, "cannot open for writing: %s", path);
  const bool ok = std::fwrite(buf.data(), 1, buf.size(), f) == buf.size();
  if (std::fclose(f) != 0 || !ok) return fail(MOE_ERR_SNAPSHOT, "write failed: %s", path);
  return MOE_OK;
}

static moe_status load_binary(const char* path, const moe_shape* expected, int device,
                              moe_eamc** out) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return fail(MOE_ERR_SNAPSHOT, "cannot open for reading: %s", path);
  std::fseek(f, 0, SEEK_END);
  const long flen = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  BinHeader hd{};
  if (flen < (long)sizeof hd || std::fread(&hd, 1, sizeof hd, f) != sizeof hd) {
    std::fclose(f);
    return fail(MOE_ERR_SNAPSHOT, "corrupt snapshot: truncated header");
  }
  const moe_shape s{hd.L, hd.E, hd.top_k};
  auto bad = [&](const char* why) {
    std::fclose(f);
    return fail(MOE_ERR_SNAPSHOT, "corrupt snapshot: %s", why);
  };
  if (hd.version != 1) {
    std::fclose(f);
    return fail(MOE_ERR_SNAPSHOT, "unsupported snapshot version");
  }
  if (check_shape(&s) != MOE_OK) return bad("bad shape");
  if (hd.phase > 1) return bad("unknown phase");
  if (hd.cb != 1 && hd.cb != 2 && hd.cb != 4) return bad("bad count width");
  if (hd.capacity < 1) return bad("capacity must be >= 1");
  if (hd.size > hd.capacity) {
    std::fclose(f);
    return fail(MOE_ERR_SNAPSHOT, "snapshot holds more entries than its capacity");
  }
  const uint64_t body = hd.size * 8 + hd.size * (uint64_t)hd.L * hd.E * hd.cb;
  if ((uint64_t)flen != sizeof hd + body) return bad("file length does not match its header");
  if (expected && (expected->n_layers != s.n_layers ||
                   expected->n_experts_per_layer != s.n_experts_per_layer ||
                   expected->top_k != s.top_k)) {
    std::fclose(f);
    return fail(MOE_ERR_SNAPSHOT, "snapshot shape does not match the configured model shape");
  }
  PinBuf data;
  CK(data.ensure(std::max<uint64_t>(body, 64)));
  const bool rd = std::fread(data.p, 1, body, f) == body;
  std::fclose(f);
  if (!rd) return fail(MOE_ERR_SNAPSHOT, "corrupt snapshot: truncated body");
  moe_eamc* h = nullptr;
  CKS(moe_eamc_create(&s, (moe_phase)hd.phase, hd.capacity, (int)hd.cb, device, &h));
  moe_status st = MOE_OK;
  if (hd.size) {
    const uint64_t* seqs = data.as<uint64_t>();
    st = moe_eamc_append_packed(h, data.as<uint8_t>() + hd.size * 8, (int)hd.cb, seqs, hd.size);
  }
  if (st != MOE_OK) {
    moe_eamc_destroy(h);
    return st;
  }
  h->next_seq = hd.next_seq;
  *out = h;
  return MOE_OK;
}

moe_status moe_eamc_load(const char* path, const moe_shape* expected, int device, moe_eamc** out) {
  if (!path || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  {  // format by magic: the binary fast path, else JSON v1
    FILE* f = std::fopen(path, "rb");
    char m[8] = {0};
    const bool bin = f && std::fread(m, 1, 8, f) == 8 && std::memcmp(m, kBinMagic, 8) == 0;
    if (f) std::fclose(f);
    if (bin) return load_binary(path, expected, device, out);
  }
  moe::host::Snapshot snap;
  std::string err;
  if (!moe::host::load_snapshot(path, &snap, &err)) return fail(MOE_ERR_SNAPSHOT, "%s", err.c_str());
  const moe_shape s{snap.L, snap.E, snap.top_k};
  if (check_shape(&s) != MOE_OK) return fail(MOE_ERR_SNAPSHOT, "corrupt snapshot: %s", std::string(last_error()).c_str());
  if (snap.capacity < 1) return fail(MOE_ERR_SNAPSHOT, "corrupt snapshot: capacity must be >= 1");
  if (snap.seqs.size() > snap.capacity)
    return fail(MOE_ERR_SNAPSHOT, "snapshot holds more entries than its capacity");
  if (expected && (expected->n_layers != s.n_layers ||
                   expected->n_experts_per_layer != s.n_experts_per_layer ||
                   expected->top_k != s.top_k))
    return fail(MOE_ERR_SNAPSHOT, "snapshot shape does not match the configured model shape");
  moe_eamc* h = nullptr;
  CKS(moe_eamc_create(&s, (moe_phase)snap.phase, snap.capacity, 1, device, &h));
  moe_status st = MOE_OK;
  if (!snap.seqs.empty())
    st = moe_eamc_append(h, snap.counts.data(), snap.seqs.data(), snap.seqs.size());
  if (st != MOE_OK) {
    moe_eamc_destroy(h);
    return st == MOE_ERR_OVERFLOW ? fail(MOE_ERR_SNAPSHOT, "snapshot counts: %s", std::string(last_error()).c_str()) : st;
  }
  h->next_seq = snap.next_seq;  // eam.cpp:244
  *out = h;
  return MOE_OK;
}

moe_status moe_gen_bench_family(uint64_t seed, uint32_t L, uint32_t E, uint64_t skip, uint64_t n,
                                int count_bytes, void* out) {
  if (!out && n) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  if (L < 1 || E < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "bad shape");
  if (count_bytes != 1 && count_bytes != 2 && count_bytes != 8)
    return fail(MOE_ERR_INVALID_ARGUMENT, "count_bytes must be 1, 2 or 8");
  moe::host::bench_family(seed, L, E, skip, n, count_bytes, out);
  return MOE_OK;
}

}  // extern "C"
