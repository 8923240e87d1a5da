// host.cpp -- snapshot codec, capacity bound and the bench-family generator.
#include "host.hpp"

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>

namespace moe {
namespace host {

// ---------------------------------------------------------------- JSON v1
// Writer: the byte layout nlohmann::json::dump() gives the reference's
// snapshot (eam.cpp:184-205): compact, object keys in sorted order.
bool save_snapshot(const char* path, const Snapshot& s, std::string* err) {
  std::ofstream out(path, std::ios::binary);
  if (!out) {
    *err = std::string("cannot open for writing: ") + path;
    return false;
  }
  std::string buf;
  buf.reserve(64 + s.counts.size() * 3);
  buf += "{\"capacity\":" + std::to_string(s.capacity) + ",\"entries\":[";
  const uint64_t cells = (uint64_t)s.L * s.E;
  for (size_t i = 0; i < s.seqs.size(); ++i) {
    if (i) buf += ',';
    buf += "{\"counts\":[";
    for (uint64_t c = 0; c < cells; ++c) {
      if (c) buf += ',';
      buf += std::to_string(s.counts[i * cells + c]);
    }
    buf += "],\"seq\":" + std::to_string(s.seqs[i]) + "}";
  }
  buf += "],\"next_seq\":" + std::to_string(s.next_seq);
  buf += ",\"phase\":\"";
  buf += s.phase == 0 ? "prefill" : "decode";
  buf += "\",\"shape\":{\"n_experts_per_layer\":" + std::to_string(s.E) +
         ",\"n_layers\":" + std::to_string(s.L) + ",\"top_k\":" + std::to_string(s.top_k) +
         "},\"version\":1}\n";
  out << buf;
  if (!out) {
    *err = std::string("write failed: ") + path;
    return false;
  }
  return true;
}

namespace {

// Minimal JSON DOM sufficient for the snapshot schema.
struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  bool is_uint = false;
  uint64_t u = 0;
  double d = 0.0;
  std::string s;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;
};

struct Parser {
  const char* p;
  const char* end;
  std::string err;
  void ws() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  bool lit(const char* w) {
    const size_t n = strlen(w);
    if ((size_t)(end - p) < n || strncmp(p, w, n) != 0) return false;
    p += n;
    return true;
  }
  bool str(std::string* o) {
    if (p >= end || *p != '"') return false;
    ++p;
    while (p < end && *p != '"') {
      if (*p == '\\') {
        ++p;
        if (p >= end) return false;
        switch (*p) {
          case 'n': o->push_back('\n'); break;
          case 't': o->push_back('\t'); break;
          case 'r': o->push_back('\r'); break;
          case 'b': o->push_back('\b'); break;
          case 'f': o->push_back('\f'); break;
          case 'u':
            if (end - p < 5) return false;
            o->push_back('?');
            p += 4;
            break;
          default: o->push_back(*p);
        }
        ++p;
      } else {
        o->push_back(*p++);
      }
    }
    if (p >= end) return false;
    ++p;
    return true;
  }
  bool value(JVal* v, int depth) {
    if (depth > 64) return false;
    ws();
    if (p >= end) return false;
    if (*p == '{') {
      ++p;
      v->kind = JVal::Obj;
      ws();
      if (p < end && *p == '}') {
        ++p;
        return true;
      }
      for (;;) {
        ws();
        std::string k;
        if (!str(&k)) return false;
        ws();
        if (p >= end || *p != ':') return false;
        ++p;
        JVal child;
        if (!value(&child, depth + 1)) return false;
        v->obj[k] = std::move(child);
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == '}') {
          ++p;
          return true;
        }
        return false;
      }
    }
    if (*p == '[') {
      ++p;
      v->kind = JVal::Arr;
      ws();
      if (p < end && *p == ']') {
        ++p;
        return true;
      }
      for (;;) {
        JVal child;
        if (!value(&child, depth + 1)) return false;
        v->arr.push_back(std::move(child));
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == ']') {
          ++p;
          return true;
        }
        return false;
      }
    }
    if (*p == '"') {
      v->kind = JVal::Str;
      return str(&v->s);
    }
    if (lit("true")) {
      v->kind = JVal::Bool;
      v->b = true;
      return true;
    }
    if (lit("false")) {
      v->kind = JVal::Bool;
      return true;
    }
    if (lit("null")) return true;
    // number
    const char* s = p;
    if (p < end && (*p == '-' || *p == '+')) ++p;
    bool digits_only = true;
    while (p < end && (isdigit((unsigned char)*p) || *p == '.' || *p == 'e' || *p == 'E' ||
                       *p == '-' || *p == '+')) {
      if (!isdigit((unsigned char)*p)) digits_only = false;
      ++p;
    }
    if (p == s) return false;
    v->kind = JVal::Num;
    const std::string tok(s, p);
    v->d = strtod(tok.c_str(), nullptr);
    if (digits_only && tok[0] != '-' && tok[0] != '+' && tok.size() <= 20) {
      errno = 0;
      char* e = nullptr;
      const unsigned long long u = strtoull(tok.c_str(), &e, 10);
      if (errno == 0 && e && *e == 0) {
        v->is_uint = true;
        v->u = u;
      }
    }
    return true;
  }
};

const JVal* at(const JVal& v, const char* key, std::string* err) {
  if (v.kind != JVal::Obj) {
    *err = "corrupt snapshot: expected an object";
    return nullptr;
  }
  auto it = v.obj.find(key);
  if (it == v.obj.end()) {
    *err = std::string("corrupt snapshot: key '") + key + "' not found";
    return nullptr;
  }
  return &it->second;
}

bool get_u64(const JVal* v, uint64_t* out, std::string* err) {
  if (!v) return false;
  if (v->kind != JVal::Num || !v->is_uint) {
    *err = "corrupt snapshot: expected an unsigned integer";
    return false;
  }
  *out = v->u;
  return true;
}

}  // namespace

// Reader with the validation of Eamc::load (eam.cpp:207-249).
bool load_snapshot(const char* path, Snapshot* s, std::string* err) {
  std::ifstream in(path, std::ios::binary);
  if (!in) {
    *err = std::string("cannot open for reading: ") + path;
    return false;
  }
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string text = ss.str();
  Parser ps{text.data(), text.data() + text.size(), {}};
  JVal root;
  if (!ps.value(&root, 0)) {
    *err = "corrupt snapshot: parse error";
    return false;
  }
  ps.ws();
  if (ps.p != ps.end) {
    *err = "corrupt snapshot: trailing characters";
    return false;
  }
  uint64_t version = 0;
  const JVal* jv = at(root, "version", err);
  if (!jv) return false;
  if (jv->kind != JVal::Num || !jv->is_uint || jv->u != 1) {
    *err = "unsupported snapshot version";
    return false;
  }
  (void)version;
  const JVal* shape = at(root, "shape", err);
  if (!shape) return false;
  uint64_t L = 0, E = 0, K = 0, cap = 0, nseq = 0;
  if (!get_u64(at(*shape, "n_layers", err), &L, err)) return false;
  if (!get_u64(at(*shape, "n_experts_per_layer", err), &E, err)) return false;
  if (!get_u64(at(*shape, "top_k", err), &K, err)) return false;
  if (L > 0xffffffffull || E > 0xffffffffull || K > 0xffffffffull) {
    *err = "corrupt snapshot: shape out of range";
    return false;
  }
  const JVal* ph = at(root, "phase", err);
  if (!ph) return false;
  if (ph->kind != JVal::Str) {
    *err = "corrupt snapshot: phase must be a string";
    return false;
  }
  int phase;
  if (ph->s == "prefill") phase = 0;
  else if (ph->s == "decode") phase = 1;
  else {
    *err = "unknown phase: " + ph->s;
    return false;
  }
  if (!get_u64(at(root, "capacity", err), &cap, err)) return false;
  const JVal* entries = at(root, "entries", err);
  if (!entries) return false;
  if (entries->kind != JVal::Arr) {
    *err = "corrupt snapshot: entries must be an array";
    return false;
  }
  const uint64_t cells = L * E;
  s->L = (uint32_t)L;
  s->E = (uint32_t)E;
  s->top_k = (uint32_t)K;
  s->phase = phase;
  s->capacity = cap;
  s->seqs.clear();
  s->counts.clear();
  s->counts.reserve(entries->arr.size() * cells);
  for (const JVal& je : entries->arr) {
    const JVal* counts = at(je, "counts", err);
    if (!counts) return false;
    if (counts->kind != JVal::Arr || counts->arr.size() != cells) {
      *err = "entry count array does not match shape";
      return false;
    }
    for (const JVal& c : counts->arr) {
      uint64_t v = 0;
      if (!get_u64(&c, &v, err)) return false;
      s->counts.push_back(v);
    }
    if (s->seqs.size() >= cap) {
      *err = "snapshot holds more entries than its capacity";
      return false;
    }
    uint64_t sq = 0;
    if (!get_u64(at(je, "seq", err), &sq, err)) return false;
    s->seqs.push_back(sq);
  }
  if (!get_u64(at(root, "next_seq", err), &nseq, err)) return false;
  s->next_seq = nseq;
  return true;
}

// eamc_capacity_bound (eam.cpp:258-268); 0 = unsupported similarity.
uint64_t capacity_bound(uint32_t L, uint32_t E, double similarity) {
  const uint64_t total = (uint64_t)L * E;
  const double le = (double)total;
  if (similarity == 0.75) return 2 * total;
  if (similarity == 0.98) return (uint64_t)std::ceil(0.5 * le * std::log(le));
  return 0;
}

// ------------------------------------------------------ bench family
// splitmix64 stream (rng.hpp:19-45) and random_request_eam
// (bench.cpp:44-54), the reference benchmark's own synthetic EAMs.
namespace {
struct Rng {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  uint64_t bounded(uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
      const uint64_t r = next();
      if (r >= threshold) return r % n;
    }
  }
  static Rng stream(uint64_t seed, uint64_t tag) {
    Rng mix{seed ^ (0xA0761D6478BD642Full + tag * 0xE7037ED1A0B428DBull)};
    return Rng{mix.next()};
  }
};
}  // namespace

void bench_family(uint64_t seed, uint32_t L, uint32_t E, uint64_t skip, uint64_t n,
                  int count_bytes, void* out) {
  Rng rng = Rng::stream(seed, 0x6265636Eull);
  const uint32_t active = E < 4 ? E : 4;
  const uint64_t cells = (uint64_t)L * E;
  for (uint64_t i = 0; i < skip; ++i)
    for (uint32_t l = 0; l < L; ++l)
      for (uint32_t k = 0; k < active; ++k) {
        rng.bounded(E);
        rng.bounded(32);
      }
  uint8_t* o = static_cast<uint8_t*>(out);
  memset(o, 0, n * cells * count_bytes);
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t l = 0; l < L; ++l)
      for (uint32_t k = 0; k < active; ++k) {
        const uint64_t e = rng.bounded(E);
        const uint64_t v = rng.bounded(32) + 1;
        const uint64_t idx = i * cells + (uint64_t)l * E + e;
        if (count_bytes == 1) o[idx] = (uint8_t)v;
        else if (count_bytes == 2) reinterpret_cast<uint16_t*>(o)[idx] = (uint16_t)v;
        else reinterpret_cast<uint64_t*>(o)[idx] = v;
      }
}

}  // namespace host
}  // namespace moe

// ---------------------------------------------------------------- traces
namespace moe {
namespace host {
namespace {

// One parsed RequestTrace (model.hpp:58-66) as flat events.
struct TraceEvent {
  uint32_t layer;
  std::vector<std::pair<uint64_t, uint64_t>> assign;  // (expert, tokens)
};

bool as_u64(const JVal& v, uint64_t* o) {
  if (v.kind != JVal::Num || !v.is_uint) return false;
  *o = v.u;
  return true;
}

// trace_from_jsonl (model.cpp:92-121): request_id string, prompt_tokens
// number, iterations [[[layer, [[expert, tokens], ...]], ...], ...]; unknown
// fields ignored.  Returns "" or the structure error.
std::string parse_trace(const JVal& j, std::string* id,
                        std::vector<std::vector<TraceEvent>>* iters) {
  if (j.kind != JVal::Obj) return "bad trace structure: not an object";
  auto rid = j.obj.find("request_id");
  auto pt = j.obj.find("prompt_tokens");
  auto it = j.obj.find("iterations");
  if (rid == j.obj.end() || rid->second.kind != JVal::Str)
    return "bad trace structure: request_id";
  uint64_t ptok = 0;
  if (pt == j.obj.end() || !as_u64(pt->second, &ptok)) return "bad trace structure: prompt_tokens";
  if (it == j.obj.end() || it->second.kind != JVal::Arr) return "bad trace structure: iterations";
  *id = rid->second.s;
  iters->clear();
  for (const JVal& ji : it->second.arr) {
    if (ji.kind != JVal::Arr) return "bad trace structure: iteration";
    std::vector<TraceEvent> evs;
    for (const JVal& je : ji.arr) {
      if (je.kind != JVal::Arr || je.arr.size() < 2 || je.arr[1].kind != JVal::Arr)
        return "bad trace structure: routing event";
      uint64_t layer = 0;
      if (!as_u64(je.arr[0], &layer) || layer > 0xffffffffull)
        return "bad trace structure: layer";
      TraceEvent ev;
      ev.layer = (uint32_t)layer;
      for (const JVal& ja : je.arr[1].arr) {
        uint64_t ex = 0, tok = 0;
        if (ja.kind != JVal::Arr || ja.arr.size() < 2 || !as_u64(ja.arr[0], &ex) ||
            ex > 0xffffffffull || !as_u64(ja.arr[1], &tok))
          return "bad trace structure: assignment";
        ev.assign.emplace_back(ex, tok);
      }
      evs.push_back(std::move(ev));
    }
    iters->push_back(std::move(evs));
  }
  return "";
}

// validate_trace (model.cpp:32-71), same order and messages.
std::string validate(const std::string& id, const std::vector<std::vector<TraceEvent>>& iters,
                     uint32_t L, uint32_t E) {
  std::ostringstream os;
  if (iters.empty()) return "EmptyIterationList: request '" + id + "' has no iterations";
  for (size_t it = 0; it < iters.size(); ++it) {
    if (iters[it].size() != L) {
      os << "LayerCountMismatch: iteration " << it << " has " << iters[it].size()
         << " routing events, expected " << L;
      return os.str();
    }
    for (uint32_t l = 0; l < L; ++l) {
      const TraceEvent& ev = iters[it][l];
      if (ev.layer != l) {
        os << "LayerCountMismatch: iteration " << it << " position " << l << " carries layer "
           << ev.layer;
        return os.str();
      }
      for (const auto& a : ev.assign) {
        if (a.first >= E) {
          os << "ExpertIndexOutOfRange: iteration " << it << " layer " << l << " routes expert "
             << a.first << " outside [0, " << E << ")";
          return os.str();
        }
        if (a.second < 1) {
          os << "InvalidTokenCount: iteration " << it << " layer " << l << " expert " << a.first
             << " has zero token count";
          return os.str();
        }
      }
    }
  }
  return "";
}

}  // namespace

bool ingest_request_eams(const char* path, uint32_t L, uint32_t E, int phase,
                         std::vector<uint64_t>* counts, uint64_t* n, std::string* err) {
  std::ifstream in(path, std::ios::binary);
  if (!in) {
    *err = std::string("cannot open for reading: ") + path;
    return false;
  }
  counts->clear();
  *n = 0;
  const uint64_t cells = (uint64_t)L * E;
  std::string line, id;
  std::vector<std::vector<TraceEvent>> iters;
  uint64_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty()) continue;
    Parser ps{line.data(), line.data() + line.size(), {}};
    JVal j;
    ps.ws();
    bool ok = ps.value(&j, 0);
    ps.ws();
    if (ok && ps.p != ps.end) ok = false;
    std::string e = ok ? parse_trace(j, &id, &iters) : "bad JSON: " + ps.err;
    if (e.empty()) e = validate(id, iters, L, E);
    if (!e.empty()) {
      *err = "line " + std::to_string(line_no) + ": " + e;
      return false;
    }
    // request_level_eam (moesim_main.cpp:192-201) + the decode skip (:212-214)
    if (phase == 1 && iters.size() < 2) continue;
    const size_t b = phase == 0 ? 0 : 1, e_it = phase == 0 ? 1 : iters.size();
    const size_t base = counts->size();
    counts->resize(base + cells, 0);
    uint64_t* c = counts->data() + base;
    for (size_t it = b; it < e_it && it < iters.size(); ++it)
      for (const TraceEvent& ev : iters[it])
        for (const auto& a : ev.assign) c[(uint64_t)ev.layer * E + a.first] += a.second;
    ++*n;
  }
  return true;
}

}  // namespace host
}  // namespace moe

// ---------------------------------------------------------------- host pool
namespace moe {
namespace host {
namespace {

class Pool {
 public:
  Pool() {
    int n = (int)std::thread::hardware_concurrency();
    if (const char* e = std::getenv("MOE_HOST_THREADS")) n = std::atoi(e);
    n_ = std::max(1, std::min(n, 64));
    for (int i = 1; i < n_; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    stop_.store(true);
    {
      std::lock_guard<std::mutex> g(mu_);
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int size() const { return n_; }

  // Asynchronous job: the workers only (the caller keeps going); wait()
  // returns when every task is done.  Jobs are serialised across callers.
  void submit(int n, void (*fn)(void*, int), void* ctx) {
    run_mu_.lock();
    async_n_ = n;
    if (n <= 0) return;
    if (n_ == 1) {  // no workers: run inline
      for (int i = 0; i < n; ++i) fn(ctx, i);
      done_.store(n, std::memory_order_release);
      return;
    }
    publish(n, fn, ctx);
  }
  void wait() {
    if (async_n_ > 0)
      while (done_.load(std::memory_order_acquire) < async_n_) std::this_thread::yield();
    async_n_ = 0;
    run_mu_.unlock();
  }

  void run(int n, void (*fn)(void*, int), void* ctx) {
    if (n <= 0) return;
    std::lock_guard<std::mutex> serial(run_mu_);  // one job at a time
    if (n_ == 1 || n == 1) {
      for (int i = 0; i < n; ++i) fn(ctx, i);
      return;
    }
    publish(n, fn, ctx);
    work();
    while (done_.load(std::memory_order_acquire) < n) std::this_thread::yield();
  }

 private:
  // A job is published by one release store of claim_ = (job << 32 | 0)
  // after fn_/ctx_/n_tasks_ are set.  Tasks are claimed by a CAS on the
  // whole word, so a worker still leaving the previous job (holding that
  // job's tag) can never take an index of the next one: its CAS fails once
  // the tag changes.  The next job is only published after every task of the
  // previous one has finished (done_ == n), so a successful claim always
  // reads the fn_/ctx_ of its own job.
  void publish(int n, void (*fn)(void*, int), void* ctx) {
    fn_.store(fn, std::memory_order_relaxed);
    ctx_.store(ctx, std::memory_order_relaxed);
    n_tasks_.store(n, std::memory_order_relaxed);
    done_.store(0, std::memory_order_relaxed);
    ++job_;
    claim_.store((uint64_t)job_ << 32, std::memory_order_release);
    {
      std::lock_guard<std::mutex> g(mu_);  // no lost wake-up for a sleeping worker
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
  }
  void work() {
    uint64_t c = claim_.load(std::memory_order_acquire);
    const uint64_t job = c >> 32;
    for (;;) {
      if ((c >> 32) != job) return;
      const uint32_t i = (uint32_t)c;
      if ((int)i >= n_tasks_.load(std::memory_order_relaxed)) return;
      if (!claim_.compare_exchange_weak(c, c + 1, std::memory_order_acq_rel,
                                        std::memory_order_acquire))
        continue;  // c reloaded: re-check the tag and the index
      fn_.load(std::memory_order_relaxed)(ctx_.load(std::memory_order_relaxed), (int)i);
      done_.fetch_add(1, std::memory_order_release);
      c = claim_.load(std::memory_order_acquire);
    }
  }
  // Workers spin for a while after each job (back-to-back jobs of one call
  // then start without a futex wake-up), and sleep on the condvar after.
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      const auto t0 = std::chrono::steady_clock::now();
      int k = 0;
      while (gen_.load(std::memory_order_acquire) == seen) {
        if ((++k & 63) == 0 &&
            std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(300)) {
          std::unique_lock<std::mutex> g(mu_);
          cv_.wait(g, [&] { return gen_.load(std::memory_order_acquire) != seen; });
          break;
        }
        std::this_thread::yield();
      }
      seen = gen_.load(std::memory_order_acquire);
      if (stop_.load()) return;
      work();
    }
  }
  int n_ = 1;
  std::vector<std::thread> workers_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_;
  std::atomic<uint64_t> gen_{0};
  std::atomic<bool> stop_{false};
  std::atomic<void (*)(void*, int)> fn_{nullptr};
  std::atomic<void*> ctx_{nullptr};
  std::atomic<int> n_tasks_{0};
  int async_n_ = 0;
  uint32_t job_ = 0;                 // written by the (serialised) publisher only
  std::atomic<uint64_t> claim_{0};   // (job << 32) | next task index
  std::atomic<int> done_{0};
};

Pool& pool() {
  static Pool* p = new Pool();  // leaked: workers outlive static destruction order
  return *p;
}

struct PackCtx {
  const uint64_t* src;
  uint64_t n;
  int cb, parts;
  void* dst;
  uint64_t ors[64];
};

// u64 -> u8 with AVX-512 (VPMOVQB) where the host has it (runtime dispatch;
// the library is built for the baseline x86-64 ISA).
__attribute__((target("avx512f,avx512bw"))) uint64_t pack_u8_avx512(const uint64_t* s,
                                                                     uint8_t* d, uint64_t n) {
  __m512i o = _mm512_setzero_si512();
  uint64_t i = 0;
  for (; i + 32 <= n; i += 32) {
    const __m512i a = _mm512_loadu_si512(s + i), b = _mm512_loadu_si512(s + i + 8);
    const __m512i c = _mm512_loadu_si512(s + i + 16), e = _mm512_loadu_si512(s + i + 24);
    o = _mm512_or_si512(o, _mm512_or_si512(_mm512_or_si512(a, b), _mm512_or_si512(c, e)));
    const __m128i lo = _mm_unpacklo_epi64(_mm512_cvtepi64_epi8(a), _mm512_cvtepi64_epi8(b));
    const __m128i hi = _mm_unpacklo_epi64(_mm512_cvtepi64_epi8(c), _mm512_cvtepi64_epi8(e));
    _mm_storeu_si128(reinterpret_cast<__m128i*>(d + i), lo);
    _mm_storeu_si128(reinterpret_cast<__m128i*>(d + i + 16), hi);
  }
  uint64_t r = (uint64_t)_mm512_reduce_or_epi64(o);
  for (; i < n; ++i) {
    r |= s[i];
    d[i] = (uint8_t)s[i];
  }
  return r;
}

const bool g_avx512 = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");

template <typename T>
uint64_t pack_range(const uint64_t* __restrict s, T* __restrict d, uint64_t n) {
  if (sizeof(T) == 1 && g_avx512) return pack_u8_avx512(s, reinterpret_cast<uint8_t*>(d), n);
  uint64_t o = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t v = s[i];
    o |= v;
    d[i] = (T)v;
  }
  return o;
}

void pack_task(void* vc, int t) {
  PackCtx* c = static_cast<PackCtx*>(vc);
  // 64-element aligned piece boundaries
  const uint64_t a = (c->n * t / c->parts) & ~63ull;
  const uint64_t b = t + 1 == c->parts ? c->n : (c->n * (t + 1) / c->parts) & ~63ull;
  c->ors[t] = c->cb == 1   ? pack_range(c->src + a, static_cast<uint8_t*>(c->dst) + a, b - a)
              : c->cb == 2 ? pack_range(c->src + a, static_cast<uint16_t*>(c->dst) + a, b - a)
                           : pack_range(c->src + a, static_cast<uint32_t*>(c->dst) + a, b - a);
}

}  // namespace

uint64_t pack_counts_serial(const uint64_t* src, uint64_t n, int cb, void* dst) {
  return cb == 1   ? pack_range(src, static_cast<uint8_t*>(dst), n)
         : cb == 2 ? pack_range(src, static_cast<uint16_t*>(dst), n)
                   : pack_range(src, static_cast<uint32_t*>(dst), n);
}

int pool_threads() { return pool().size(); }

void pool_run(int n, void (*fn)(void*, int), void* ctx) { pool().run(n, fn, ctx); }

void pool_submit(int n, void (*fn)(void*, int), void* ctx) { pool().submit(n, fn, ctx); }

void pool_wait() { pool().wait(); }

uint64_t pack_counts(const uint64_t* src, uint64_t n, int cb, void* dst) {
  PackCtx c{src, n, cb, 1, dst, {}};
  // >= 256 KiB of input per piece keeps the pool's fork/join cost negligible
  c.parts = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)pool().size(), n / 32768));
  pool().run(c.parts, pack_task, &c);
  uint64_t o = 0;
  for (int t = 0; t < c.parts; ++t) o |= c.ors[t];
  return o;
}

}  // namespace host
}  // namespace moe
