// Live PCIe mover + per-function bandwidth-share scheduler (native runtime).
//
// Every host->GPU leg of a fetch is submitted here as a *stage* of k routes
// (dataplane.py:203-250): route i moves bytes [off_i, off_i+len_i) of the host
// object either straight into dst on the copy engine of the target's own PCIe
// root, or into a chunk ring on a staging GPU followed by an NVLink forward
// (ft_copy_ex, vector engine) into dst, chained per chunk by events.
//
// Managed stages (strategy.pcie_sched; engine.py:537-646) are paced by one
// pacer thread: the stage enters the arbiter's SLO partition (ft::Arbiter, the
// restated engine logic, pcie_sched.py:80-104) and its bytes are issued batch
// by batch (batch = 5 x 2 MB, pcie_sched.py:14-15) at the stage's rate, with
// rate changes landing on batch boundaries (engine.py:628-646); the stage is
// finished in the arbiter when its last byte has landed (polled events), which
// re-partitions the link for the others (engine.py:558-564). Unmanaged stages
// are issued at once.
//
// submit() returns once every byte of the stage is enqueued on its route
// streams (for a paced stage: when its last batch is issued, a few batches
// before it lands) and makes the consumer's stream wait for the routes' last
// ops, so consumer kernels issued after fetch() are ordered after the data —
// the same stream semantics as the SM-driven movers, and the tail of the
// transfer overlaps whatever the caller issues next. No stream is ever parked
// on host progress (a parked stream would deadlock against lazy module
// loading, which synchronizes the context).
//
// Both directions are paced (engine.py:537-575 starts a managed stage for any
// host_gpu plan; engine.py:186-190 gives each direction its own arbiter):
// host->GPU legs for fetches, GPU->host legs for responses and host fetches.
//
// Pageable host objects are staged through one shared pinned ring
// (PinnedRing, pcie_sched.py:122-162) by worker threads; a slot
// is refilled once the DMA that drained it has completed.
//
// Landing is detected by polling each route's last-op event from the pacer
// thread (cudaEventQuery, every 20 us while a stage drains): a host callback
// (cudaLaunchHostFunc) in the route stream costs ~0.25 ms of stream time per
// stage on this driver (measured), 20% of a 64 MiB transfer.
//
// Locking: `mu` guards all scheduling state and is held while enqueueing
// async CUDA work only (never a synchronizing call). Workers wait on ring
// slots without holding `mu`.
#include <cuda_runtime.h>
#include <emmintrin.h>

#include "forward.h"
#include <sys/prctl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <thread>

#include "decisions.h"

namespace {

constexpr uint64_t kAlign = 256;     // route slice boundaries (tube._ALIGN)
// Copy into a pinned ring slot with non-temporal stores: the slot's next reader is
// the copy engine, and DMA out of lines the CPU still holds dirty in its caches ran
// at ~21 GB/s on the B200 hosts vs 55 GB/s from DRAM (tools/diag_calib2.py)
static void stream_copy(uint8_t* dst, const uint8_t* src, uint64_t n) {
  uint64_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
  if (head > n) head = n;
  std::memcpy(dst, src, head);
  uint64_t i = head;
  for (; i + 64 <= n; i += 64) {
    __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
  }
  std::memcpy(dst + i, src + i, n - i);
  _mm_sfence();  // the stores are globally visible before the DMA is issued
}

constexpr int kInflightBatches = 4;  // issued-but-not-landed batches per stage
constexpr double kLookahead = 2.0;   // batches issued ahead of the rate schedule (host jitter)
constexpr int kOwnerCoalesce = 2;  // batches per DMA op for a stage that holds the whole link
// smallest DMA the link estimator samples: 4 MB, or half a batch when batches are
// smaller (a direct route's DMA is a byte share of one batch, so with small chunks or
// several routes a fixed 4 MB would never be reached and the estimator would stop)
constexpr uint64_t kMinSampleBytes = 4ull << 20;
constexpr int kMaxDev = 64;
constexpr int kWorkers = 8;  // pageable staging threads (1 GiB pageable -> GPU with a 40 MB ring: 4 workers
                             // 28-37 GB/s, 8: 44-47, 12: 41-45, 16: 37-42; profiles/r01/sweep_pageable.txt)

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

struct CudaFail {
  std::string msg;
};
inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFail{std::string(what) + ": " + cudaGetErrorString(e)};
}

struct Route {
  int dev = 0;                  // GPU the PCIe leg lands on (== dst_dev for a direct route)
  uint64_t off = 0, len = 0;    // byte range of the object
  uint64_t done = 0;            // bytes handed out (issued, or queued to a worker)
  cudaStream_t ce = nullptr;    // copy-engine stream on `dev`
  cudaStream_t fw = nullptr;    // forward stream on `dev` (staged routes only)
  bool staged() const { return fw != nullptr; }
  // the route's final op: h2d staged routes end with the forward kernel, d2h
  // staged routes with the CE leg out of the staging ring
  cudaStream_t last(int dir) const { return staged() && dir == 0 ? fw : ce; }
};

struct Ev {
  cudaEvent_t e;
  int dev;
  bool timing;  // from the timing-event pool
};
struct Timing {  // a direct-route batch bracketed by timing events (link service rate)
  cudaEvent_t t0, t1;
  int dir, dev;
  uint64_t bytes;
  double issued;
  bool contended;  // another stage had bytes on the link when it was issued
};
struct Batch {
  std::vector<Ev> ev;  // last op of each route's share of the batch
  std::vector<Timing> timing;
  int batches = 1;     // 5 x 2 MB batches this entry carries (coalesced ops)
};

struct Stage {
  uint64_t ticket = 0;
  std::string key;
  bool managed = false;
  int dir = 0;              // 0 host->GPU, 1 GPU->host
  uint8_t* dst = nullptr;   // the GPU-side buffer (destination h2d, source d2h)
  int dst_dev = 0;          // its GPU
  uint8_t* host = nullptr;  // the host-side buffer (source h2d, destination d2h)
  bool pinned = true;
  uint64_t bytes = 0;
  std::vector<Route> routes;
  double next_t = NAN, last_rate = -1.0;
  std::deque<Batch> inflight;  // issued, not yet landed batches
  int jobs = 0;         // pageable chunks queued to workers, not yet issued
  bool was_full = false;  // trace: inflight cap reached (the link, not the rate, limits)
  bool inline_route = false;  // one direct route on the consumer's own stream (submit_impl)
  bool issued = false;  // every byte handed out
  bool sealed = false;  // every byte enqueued: join events recorded (or failed)
  std::vector<std::pair<cudaEvent_t, int>> join;     // last op of each route (the submitter's)
  std::vector<std::pair<cudaEvent_t, int>> landing;  // same points, polled by the pacer
  int err = FT_OK;
  std::string msg;
};

struct Job {
  uint64_t ticket;
  int route;
  uint64_t obj_off, n;  // bytes [obj_off, obj_off+n) of the object, n <= chunk
};

struct StagingRing {  // chunk ring on a staging GPU
  uint8_t* buf = nullptr;
  int slots = 0, next = 0;
  std::vector<cudaEvent_t> landed, freed;
  std::vector<char> used;
};

struct KRing {  // K2 chunk ring on a staging GPU (host->GPU staged routes, forward.h)
  uint8_t* buf = nullptr;
  int slots = 0, next = 0;
  uint64_t slot_bytes = 0;
  uint32_t *landed = nullptr, *freed = nullptr, *err = nullptr;
  std::vector<uint32_t> uses;  // per slot: chunks issued into it so far
  uint64_t alt = 0;            // CE ops issued (alternates the two CE streams)
};

struct HostSlot {
  bool busy = false;
  int last_dev = -1;  // device of the event guarding the slot's last DMA
  cudaEvent_t ev[kMaxDev] = {};
};

std::string jnum(double x) {
  if (std::isnan(x)) return "null";
  char b[40];
  snprintf(b, sizeof b, "%.17g", x);
  return b;
}

}  // namespace

struct ft_pacer {
  // ---- configuration
  int batch_chunks = 5;
  uint64_t chunk = 2000000;
  int staging_slots = 4;
  uint64_t stage_chunk = 0;        // staging ring slot (bytes): 4 chunks, or FT_STAGE_CHUNK
  bool fixed_stage_chunk = false;  // FT_STAGE_CHUNK: every piece is one full slot
  bool logging = false;
  ft::Arbiter arbs[2];  // per direction (engine.py:186-190)
  ft::Arbiter& arb_of(const Stage& st) { return arbs[st.dir]; }
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();

  // ---- state (mu)
  std::mutex mu;
  std::condition_variable cv;       // pacer thread
  std::condition_variable done_cv;  // waiters
  std::condition_variable jcv;      // workers
  std::map<uint64_t, std::shared_ptr<Stage>> active;  // ticket order == submission order
  uint64_t next_ticket = 1;
  std::map<uint64_t, std::pair<int, std::string>> errors;
  std::deque<Job> jobs;
  bool stop = false;
  std::vector<cudaEvent_t> evpool[kMaxDev];
  std::vector<cudaEvent_t> tpool[kMaxDev];  // timing-enabled events
  // link estimator: the arbiter's bw_all tracks the service rate of uncontended
  // batches (a calibration at start-up can be far off on a shared host)
  int links = 1;
  double link_gbps[2] = {0.0, 0.0};          // per-link capacity the partition assumes, per direction
  std::deque<double> samples[2][kMaxDev];
  // per link: the newest pinned DMA issue (ticket, time) and the newest by any other
  // ticket than that one — so a sample can tell whether ANOTHER stage issued onto its
  // link after it (timed or not)
  double last_issue_t[2][kMaxDev] = {}, other_issue_t[2][kMaxDev] = {};
  uint64_t last_issue_ticket[2][kMaxDev] = {};
  void note_issue(int dir, int dev, uint64_t ticket, double t) {
    if (last_issue_ticket[dir][dev] != ticket) other_issue_t[dir][dev] = last_issue_t[dir][dev];
    last_issue_ticket[dir][dev] = ticket;
    last_issue_t[dir][dev] = t;
  }
  double newest_other_issue(int dir, int dev, uint64_t ticket) const {
    return last_issue_ticket[dir][dev] != ticket ? last_issue_t[dir][dev] : other_issue_t[dir][dev];
  }
  bool adapt = true;
  bool sampling = !std::getenv("FT_PACER_NOSAMPLE");  // (diagnostic switch)
  uint64_t timed_skip = 0;
  std::map<int, StagingRing> rings;  // GPU->host staged routes
  std::map<int, KRing> krings;       // host->GPU staged routes (K2)
  std::map<cudaStream_t, cudaStream_t> ce2;  // second CE stream of each route CE stream
  // K2 (one forward kernel per batch on device flags) or the per-piece event chain:
  // measured on one link, 1 GiB staged, the chain is 1-4 % faster at every piece
  // size (a stream memory op costs the CE more than an event record/wait:
  // profiles/r02/sweep_k2.txt), so it is the default; FT_K2=1 selects K2
  bool k2 = false;
  bool ce_alt = true;                // K2: alternate two CE streams per route (FT_K2_CE2=0: one)
  std::map<std::string, double> guarded;  // last early boundary per stage key (A2 guard)
  uint64_t n_stages = 0, n_managed = 0, n_batches = 0, n_bytes = 0, n_errors = 0;
  std::vector<std::string> trace, log;

  // ---- stages that have landed (or failed), to retire (lmu)
  std::mutex lmu;
  std::vector<uint64_t> landed;

  // ---- pinned host ring (hmu only)
  std::mutex hmu;
  std::condition_variable hcv;
  uint8_t* hring = nullptr;
  uint64_t host_chunk = 0;  // pinned-ring slot = one worker memcpy + one DMA op (FT_HOST_CHUNK)
  std::vector<HostSlot> hslots;
  int hnext = 0;

  std::thread pacer;
  std::vector<std::thread> workers;

  double now() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }

  // ------------------------------------------------------------ helpers (mu held)
  cudaEvent_t get_event(int dev) {
    auto& pool = evpool[dev];
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    DevGuard g(dev);
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    return e;
  }
  void put_event(int dev, cudaEvent_t e) { evpool[dev].push_back(e); }
  cudaEvent_t get_tevent(int dev) {
    auto& pool = tpool[dev];
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    DevGuard g(dev);
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate(timing)");
    return e;
  }
  void put(const Ev& e) { (e.timing ? tpool : evpool)[e.dev].push_back(e.e); }

  // anything else of ours on `dev`'s link right now?
  bool link_busy(int dir, int dev, uint64_t self) const {
    for (auto& kv : active) {
      const Stage& o = *kv.second;
      if (o.ticket == self || o.dir != dir) continue;
      bool on = false;
      for (auto& r : o.routes) on = on || r.dev == dev;
      if (on && (!o.inflight.empty() || (o.sealed && !o.landing.empty()) || (!o.managed && !o.sealed) || o.jobs))
        return true;
    }
    return false;
  }

  void sample(int dir, int dev, double gbps, double now) {
    auto& q = samples[dir][dev];
    q.push_back(gbps);
    if (q.size() > 32) q.pop_front();
    if (!adapt || q.size() < 6) return;
    double est = *std::max_element(q.begin(), q.end());  // least-disturbed service rate
    if (est > link_gbps[dir] * 1.05 || est < link_gbps[dir] * 0.85) {
      link_gbps[dir] = est;
      arbs[dir].set_bw(now, est * links, est);
      arb_log(dir, now, "bw", jnum(est), est * links);  // key: the per-link estimate
      q.clear();
    }
  }

  void note(const Stage& st, const char* kind, double v) {
    if (!logging) return;
    trace.push_back("[" + jnum(now()) + "," + std::to_string(st.ticket) + ",\"" + kind + "\"," + jnum(v) + "]");
  }
  // log entry of an arbiter call; the GPU->host arbiter's calls carry a "d2h:" prefix
  // [t, call, key, decisions, arg]: arg = the per-branch cap of a start, the new
  // bw_all of a "bw" call, null otherwise
  void arb_log(int dir, double t, const char* call, const std::string& key, double arg = NAN) {
    if (!logging) return;
    log.push_back("[" + jnum(t) + ",\"" + (dir ? "d2h:" : "") + call + "\",\"" + key + "\"," +
                  arbs[dir].last_json + "," + jnum(arg) + "]");
  }

  StagingRing& ring(int dev) {
    auto it = rings.find(dev);
    if (it != rings.end()) return it->second;
    StagingRing r;
    DevGuard g(dev);
    void* p = nullptr;
    ck(cudaMalloc(&p, (size_t)staging_slots * stage_chunk), "staging ring cudaMalloc");
    r.buf = static_cast<uint8_t*>(p);
    r.slots = staging_slots;
    r.landed.resize(r.slots);
    r.freed.resize(r.slots);
    r.used.assign(r.slots, 0);
    for (int i = 0; i < r.slots; ++i) {
      ck(cudaEventCreateWithFlags(&r.landed[i], cudaEventDisableTiming), "cudaEventCreate");
      ck(cudaEventCreateWithFlags(&r.freed[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    return rings.emplace(dev, std::move(r)).first->second;
  }

  KRing& kring(int dev) {
    auto it = krings.find(dev);
    if (it != krings.end()) return it->second;
    KRing K;
    DevGuard g(dev);
    // staging_slots slots of one staging piece each (stage_chunk: up to 4 chunks of
    // pcie_sched.py:14's 2 MB): a copy-engine op carries one piece — the CE loses
    // ~10 % of the link to per-op cost at 2 MB ops (profiles/r02/sweep_k2.txt)
    K.slot_bytes = (stage_chunk + 255) / 256 * 256;
    K.slots = std::clamp(staging_slots, 2, ft::kFwdMaxChunks);
    void* p = nullptr;
    ck(cudaMalloc(&p, (size_t)K.slots * K.slot_bytes), "K2 ring cudaMalloc");
    K.buf = static_cast<uint8_t*>(p);
    if (ft::fwd_ring_words(dev, K.slots, &K.landed, &K.freed, &K.err) != FT_OK ||
        ft::fwd_preload(dev) != FT_OK)
      throw CudaFail{std::string("K2 ring: ") + ft_last_error()};
    K.uses.assign(K.slots, 0);
    return krings.emplace(dev, std::move(K)).first->second;
  }
  cudaStream_t ce_pair(cudaStream_t ce, int dev) {
    auto it = ce2.find(ce);
    if (it != ce2.end()) return it->second;
    DevGuard g(dev);
    cudaStream_t s2;
    ck(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking), "second CE stream");
    ce2.emplace(ce, s2);
    return s2;
  }

  // K2: the staged host->GPU leg. Chunks alternate over two CE streams (one op's
  // fixed cost hides behind the other's transfer), each followed by a device-side
  // write of the slot's landed word; one forward kernel per <= slots chunks pulls
  // them as they land and counts each slot free. Returns the CE stream of the last op.
  cudaStream_t issue_k2(Route& r, uint8_t* dptr, uint8_t* hptr, uint64_t n) {
    KRing& K = kring(r.dev);
    cudaStream_t c2 = ce_pair(r.ce, r.dev), last = r.ce;
    ft::FwdBatch b;
    b.n = 0;
    auto flush = [&] {
      if (!b.n) return;
      if (ft::fwd_launch(r.dev, r.fw, dptr, K.buf, K.slot_bytes, K.landed, K.freed, K.err, b) != FT_OK)
        throw CudaFail{std::string("forward: ") + ft_last_error()};
      b.n = 0;
    };
    // pieces: 1/32 of the route, between one chunk and a full slot (a long route
    // moves in big CE ops, a short one keeps its pipeline fill short)
    const uint64_t step = fixed_stage_chunk ? K.slot_bytes
                                            : std::clamp<uint64_t>(r.len / 32 / 65536 * 65536, chunk, K.slot_bytes);
    for (uint64_t o = 0; o < n; o += step) {
      const uint64_t c = std::min<uint64_t>(step, n - o);
      const int s = K.next;
      K.next = (s + 1) % K.slots;
      cudaStream_t cs = (ce_alt && (K.alt++ & 1)) ? c2 : r.ce;
      // the slot's previous chunk has been read by every CTA of its forward launch
      // (that launch was enqueued before: a launch holds at most one chunk per slot)
      if (K.uses[s] && ft::mem_wait_geq32(cs, K.freed + s, K.uses[s] * (uint32_t)ft::kFwdCtas) != FT_OK)
        throw CudaFail{std::string("wait slot freed: ") + ft_last_error()};
      const uint32_t gen = ++K.uses[s];
      ck(cudaMemcpyAsync(K.buf + (uint64_t)s * K.slot_bytes, hptr + o, c, cudaMemcpyHostToDevice, cs),
         "staging H2D");
      if (ft::mem_write32(cs, K.landed + s, gen) != FT_OK)
        throw CudaFail{std::string("write landed: ") + ft_last_error()};
      b.c[b.n++] = ft::FwdChunk{o, (uint32_t)s, gen, c};
      n_bytes += c;
      last = cs;
      if (b.n == K.slots) flush();
    }
    flush();
    return last;
  }

  // n bytes between the GPU buffer `dptr` and the pinned host buffer `hptr` over
  // route r: host->GPU (dir 0) or GPU->host (dir 1). Returns the stream of the
  // last copy-engine op (the one that reads / writes host memory last).
  cudaStream_t issue(Route& r, uint8_t* dptr, uint8_t* hptr, uint64_t n, int dir) {
    if (n == 0) return r.ce;
    DevGuard g(r.dev);
    if (!r.staged()) {
      if (dir == 0)
        ck(cudaMemcpyAsync(dptr, hptr, n, cudaMemcpyHostToDevice, r.ce), "H2D");
      else
        ck(cudaMemcpyAsync(hptr, dptr, n, cudaMemcpyDeviceToHost, r.ce), "D2H");
      n_bytes += n;
      return r.ce;
    }
    if (dir == 0 && k2) return issue_k2(r, dptr, hptr, n);
    StagingRing& R = ring(r.dev);
    // pieces per route: 1/32 of it, between one chunk and a full slot. Each piece is
    // a CE op + forward kernel; a 2 MB piece loses ~9 % of the link to per-op gaps
    // (1 GiB through one staged route: 49.6 GB/s at 2 MB, 52.4 at 4, 53.4 at 8,
    // 54.1 at 16, direct 54.5), a big one costs pipeline fill: 1/32 balances both
    const uint64_t step = fixed_stage_chunk ? stage_chunk
                                            : std::clamp<uint64_t>(r.len / 32 / 65536 * 65536, chunk, stage_chunk);
    for (uint64_t o = 0; o < n; o += step) {
      uint64_t c = std::min<uint64_t>(step, n - o);
      int s = R.next;
      R.next = (s + 1) % R.slots;
      uint8_t* slot = R.buf + (uint64_t)s * stage_chunk;
      if (dir == 0) {
        // CE into the staging slot, forward kernel (NVLink push) into the target
        if (R.used[s]) ck(cudaStreamWaitEvent(r.ce, R.freed[s], 0), "wait slot freed");
        ck(cudaMemcpyAsync(slot, hptr + o, c, cudaMemcpyHostToDevice, r.ce), "staging H2D");
        ck(cudaEventRecord(R.landed[s], r.ce), "record landed");
        ck(cudaStreamWaitEvent(r.fw, R.landed[s], 0), "wait landed");
        int rc = ft_copy_ex(dptr + o, slot, c, r.dev, r.fw, 2, 0);
        if (rc != FT_OK) throw CudaFail{std::string("forward: ") + ft_last_error()};
        ck(cudaEventRecord(R.freed[s], r.fw), "record freed");
      } else {
        // forward kernel (NVLink pull) into the staging slot, CE out of it to the host
        if (R.used[s]) ck(cudaStreamWaitEvent(r.fw, R.freed[s], 0), "wait slot freed");
        int rc = ft_copy_ex(slot, dptr + o, c, r.dev, r.fw, 2, 0);
        if (rc != FT_OK) throw CudaFail{std::string("forward: ") + ft_last_error()};
        ck(cudaEventRecord(R.landed[s], r.fw), "record landed");
        ck(cudaStreamWaitEvent(r.ce, R.landed[s], 0), "wait landed");
        ck(cudaMemcpyAsync(hptr + o, slot, c, cudaMemcpyDeviceToHost, r.ce), "staging D2H");
        ck(cudaEventRecord(R.freed[s], r.ce), "record freed");
      }
      R.used[s] = 1;
      n_bytes += c;
    }
    return r.ce;
  }

  // hand bytes [rel, rel+n) of route i to the movers (direct DMA or worker jobs)
  void hand_out(Stage& st, int i, uint64_t rel, uint64_t n, bool track) {
    Route& r = st.routes[i];
    uint64_t o = r.off + rel;
    if (st.pinned) {
      if (track && sampling && !r.staged() && n >= std::min<uint64_t>(kMinSampleBytes, (uint64_t)batch_chunks * chunk / 2) &&
          (samples[st.dir][r.dev].size() < 6 || ++timed_skip % 8 == 0)) {
        // direct route: bracket the DMA with timing events (service-rate sample) —
        // every batch until the estimator has its window, then every 8th (a timed
        // event between two DMAs costs copy-engine time). Small DMAs are not
        // sampled: their fixed cost says nothing about the link (a 4 KiB copy
        // "runs" at ~1 GB/s) and a window of them would drag the estimate down
        DevGuard g(r.dev);
        Timing tm{get_tevent(r.dev), nullptr, st.dir, r.dev, n, now(), link_busy(st.dir, r.dev, st.ticket)};
        ck(cudaEventRecord(tm.t0, r.ce), "record t0");
        issue(r, st.dst + o, st.host + o, n, st.dir);
        tm.t1 = get_tevent(r.dev);
        ck(cudaEventRecord(tm.t1, r.ce), "record t1");
        st.inflight.back().timing.push_back(tm);
        note_issue(st.dir, r.dev, st.ticket, tm.issued);
        return;
      }
      issue(r, st.dst + o, st.host + o, n, st.dir);
      note_issue(st.dir, r.dev, st.ticket, now());
      // (an inline stage's only batch: the landing event seal() records follows it on
      // the same stream, nothing polls a batch event for it)
      if (track && !(st.inline_route && rel + n == r.len)) {
        DevGuard g(r.dev);
        cudaEvent_t e = get_event(r.dev);
        ck(cudaEventRecord(e, r.last(st.dir)), "record batch");
        st.inflight.back().ev.push_back(Ev{e, r.dev, false});
      }
      return;
    }
    for (uint64_t k = 0; k < n; k += host_chunk) {
      jobs.push_back(Job{st.ticket, i, o + k, std::min<uint64_t>(host_chunk, n - k)});
      ++st.jobs;
    }
    jcv.notify_all();
  }

  // the link service rate of a landed batch's timed DMAs (unless another DMA of ours
  // shared the link meanwhile)
  void take_samples(const Stage& st, const Batch& b, double t) {
    for (auto& tm : b.timing) {
      float ms = 0.f;
      bool overlapped = tm.contended || newest_other_issue(tm.dir, tm.dev, st.ticket) > tm.issued;
      if (!overlapped && cudaEventElapsedTime(&ms, tm.t0, tm.t1) == cudaSuccess && ms > 0.f)
        sample(tm.dir, tm.dev, (double)tm.bytes / ((double)ms * 1e6), t);
    }
  }

  void release_batch(Batch& b) {
    for (auto& e : b.ev) put(e);
    for (auto& t : b.timing) {
      tpool[t.dev].push_back(t.t0);
      tpool[t.dev].push_back(t.t1);
    }
    b.ev.clear();
    b.timing.clear();
  }
  void release_inflight(Stage& st) {
    for (auto& b : st.inflight) release_batch(b);
    st.inflight.clear();
  }

  // every byte is on a stream: record each route's last op twice — for the
  // submitter (consumer stream waits) and for the pacer's landing poll
  void seal(Stage& st) {
    if (st.sealed) return;
    for (auto& r : st.routes) {
      DevGuard g(r.dev);
      cudaEvent_t b = get_event(r.dev);
      if (!st.inline_route) {  // (an inline route ran on the consumer's stream: nothing to join)
        cudaEvent_t a = get_event(r.dev);
        ck(cudaEventRecord(a, r.last(st.dir)), "record join");
        st.join.emplace_back(a, r.dev);
      }
      ck(cudaEventRecord(b, r.last(st.dir)), "record landing");
      st.landing.emplace_back(b, r.dev);
    }
    st.sealed = true;
    done_cv.notify_all();
  }

  // sealed stages whose every route has drained -> landed list
  bool poll_landing() {
    bool pending = false;
    for (auto& kv : active) {
      Stage& st = *kv.second;
      if (!st.sealed || st.landing.empty()) continue;
      bool all = true;
      for (auto& e : st.landing) {
        cudaError_t q = cudaEventQuery(e.first);
        if (q == cudaErrorNotReady) {
          all = false;
          break;
        }
        if (q != cudaSuccess && st.err == FT_OK) {
          st.err = FT_E_CUDA;
          st.msg = std::string("route failed: ") + cudaGetErrorString(q);
        }
      }
      if (!all) {
        pending = true;
        continue;
      }
      if (st.dir == 0 && st.err == FT_OK)
        for (auto& r : st.routes)
          if (r.staged()) {
            auto k = krings.find(r.dev);
            if (k != krings.end() && *(volatile uint32_t*)k->second.err) {
              st.err = FT_E_TIMEOUT;
              st.msg = "forward kernel: a staged chunk never landed (60 s)";
              const KRing& K = k->second;
              std::vector<uint32_t> w(2 * K.slots);
              DevGuard g(r.dev);
              if (cudaMemcpy(w.data(), K.landed, w.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess) {
                st.msg += "; slot uses/landed/freed:";
                for (int i = 0; i < K.slots; ++i)
                  st.msg += " " + std::to_string(K.uses[i]) + "/" + std::to_string(w[i]) + "/" +
                            std::to_string(w[K.slots + i]);
              }
            }
          }
      for (auto& e : st.landing) put_event(e.second, e.first);
      st.landing.clear();
      std::lock_guard<std::mutex> lk(lmu);
      landed.push_back(st.ticket);
    }
    return pending;
  }

  // a stage that cannot finish on its streams: once no worker still reads its
  // host object, release its waiters from the host
  void fail(Stage& st, const std::string& msg) {
    if (st.err == FT_OK) {
      st.err = FT_E_CUDA;
      st.msg = msg;
    }
    st.issued = true;
    if (!st.sealed && st.jobs == 0) {
      st.sealed = true;
      {
        std::lock_guard<std::mutex> lk(lmu);
        landed.push_back(st.ticket);
      }
      cv.notify_all();
      done_cv.notify_all();
    }
  }

  // one 5 x 2 MB batch (or `mult` of them as one op per route) split over the
  // routes by byte share
  void issue_batch(Stage& st, int mult = 1) {
    const double batch = (double)mult * (double)batch_chunks * (double)chunk;
    if (st.pinned) {
      st.inflight.emplace_back();
      st.inflight.back().batches = mult;
    }
    bool all = true;
    uint64_t took = 0;
    for (size_t i = 0; i < st.routes.size(); ++i) {
      Route& r = st.routes[i];
      if (r.done >= r.len) continue;
      uint64_t share = (uint64_t)(batch * (double)r.len / (double)st.bytes) / kAlign * kAlign;
      uint64_t take = std::min<uint64_t>(r.len - r.done, share ? share : r.len - r.done);
      hand_out(st, (int)i, r.done, take, true);
      r.done += take;
      took += take;
      if (r.done < r.len) all = false;
    }
    const uint64_t one = (uint64_t)batch_chunks * chunk;
    n_batches += mult == 1 ? 1 : std::max<uint64_t>(1, (took + one - 1) / one);
    note(st, "issue", (double)done_bytes(st));
    if (all) {
      st.issued = true;
      if (st.jobs == 0) seal(st);
    }
  }
  static uint64_t done_bytes(const Stage& st) {
    uint64_t s = 0;
    for (auto& r : st.routes) s += r.done;
    return s;
  }

  void deliver_due(double now) {  // engine.py:628-646, fired at their armed times
    for (int dir = 0; dir < 2; ++dir) {
      ft::Arbiter& arb = arbs[dir];
      for (;;) {
        double best = NAN;
        const std::string* bk = nullptr;
        for (auto& kv : arb.stages.items)
          if (!std::isnan(kv.second.armed) && (std::isnan(best) || kv.second.armed < best)) {
            best = kv.second.armed;
            bk = &kv.first;
          }
        if (!bk || best > now) break;
        std::string key = *bk;
        arb.boundary(best, key);
        arb_log(dir, best, "boundary", key);
      }
    }
  }

  // Live guard for reference defect A2: a stage running at a
  // near-zero rate (least rate of a loose SLO, or the 1e12 ms infeasible fallback)
  // re-arms its next boundary one batch *at that rate* away — hours — so a rate
  // increase handed to it when the link frees up would never apply and the stage
  // starves. The engine only needs rate changes to land on batch boundaries; live,
  // a pending change applies no later than two batches at the higher of the two
  // rates. Decreases are never early (their boundary is within one batch already).
  void guard_pending(double now) {
    for (int dir = 0; dir < 2; ++dir) {
      ft::Arbiter& arb = arbs[dir];
      std::vector<std::string> due;
      for (auto& kv : arb.stages.items) {
        const auto& m = kv.second;
        if (!m.started || std::isnan(m.pending) || std::isnan(m.armed)) continue;
        double allowed = 2.0 * arb.batch_bytes / (std::max(m.pending, m.rate) * 1e6);
        auto g = guarded.find(kv.first);
        if (m.armed - now > allowed && (g == guarded.end() || now - g->second >= 0.5 * allowed))
          due.push_back(kv.first);
      }
      for (auto& key : due) {
        guarded[key] = now;
        arb.boundary(now, key);
        arb_log(dir, now, "boundary", key);
        if (logging) trace.push_back("[" + jnum(now) + ",0,\"guard\",0]");
      }
    }
  }

  double next_armed() const {
    double best = NAN;
    for (int dir = 0; dir < 2; ++dir)
      for (auto& kv : arbs[dir].stages.items)
        if (!std::isnan(kv.second.armed) && (std::isnan(best) || kv.second.armed < best)) best = kv.second.armed;
    return best;
  }

  void retire_landed() {
    std::vector<uint64_t> L;
    {
      std::lock_guard<std::mutex> lk(lmu);
      L.swap(landed);
    }
    if (L.empty()) return;
    double t = now();
    for (uint64_t tk : L) {
      auto it = active.find(tk);
      if (it == active.end()) continue;
      Stage& st = *it->second;
      if (st.managed) {
        arb_of(st).finish(t, st.key);
        arb_log(st.dir, t, "finish", st.key);
        guarded.erase(st.key);
      }
      note(st, "land", (double)st.bytes);
      // the batches still listed landed with the stage: their timed DMAs are samples
      // too (a stage's last batches, and all of a one-batch stage, are never stepped
      // again — unread, the estimator's window would not fill from small stages and
      // every one of their DMAs would keep paying for timing events)
      if (st.err == FT_OK)
        for (auto& b : st.inflight) take_samples(st, b, t);
      release_inflight(st);  // join events are returned by the submitter
      if (st.err != FT_OK) {
        errors[tk] = {st.err, st.msg};
        ++n_errors;
      }
      active.erase(it);
    }
    done_cv.notify_all();
  }

  // One pacing step of a managed stage at time t: drop its landed batches (and
  // sample the link), then issue its next batch if the rate schedule (with
  // lookahead) and the in-flight cap allow. Returns when to look again.
  double step(Stage& st, double t) {
    const double batch = (double)batch_chunks * (double)chunk;
    while (!st.inflight.empty()) {  // drop landed batches (non-blocking)
      Batch& b = st.inflight.front();
      bool ok = true;
      for (auto& e : b.ev)
        if (cudaEventQuery(e.e) != cudaSuccess) ok = false;
      for (auto& tm : b.timing)
        if (cudaEventQuery(tm.t1) != cudaSuccess) ok = false;
      if (!ok) break;
      take_samples(st, b, t);
      release_batch(b);
      st.inflight.pop_front();
      note(st, "done", (double)st.inflight.size());
    }
    const auto* m = arb_of(st).stages.find(st.key);
    if (!m || !m->started || m->rate <= 0) return INFINITY;  // waiting: a boundary / finish / start wakes it
    double dur = batch / (m->rate * 1e6);                     // ms per batch at the stage rate
    if (std::isnan(st.next_t) || m->rate != st.last_rate) {
      // (re)anchor on rate changes: a stage paced slowly must not keep its far-out slot
      st.next_t = std::isnan(st.next_t) ? t : std::min(st.next_t, t + dur);
      st.last_rate = m->rate;
      note(st, "rate", m->rate);
    }
    // A stage that holds the whole link — the only managed stage of its direction,
    // at a rate no lower than 95% of what the estimator measured its links to serve —
    // is paced by the links themselves: the rate schedule is skipped and its batches
    // go out two per DMA op (each op costs the copy engine ~3.5 us of gap: 10 MB ops
    // ran a 64 MiB stage at 53.8 GB/s vs 54.7 for one op). Bytes queued on its
    // streams stay within kInflightBatches batches, so a newcomer's first batch waits
    // no longer than under pacing. Without the estimator the calibration is trusted
    // and every stage is paced.
    const ft::Arbiter& arb = arb_of(st);
    const bool owner = adapt && st.pinned && arb.stages.items.size() == 1 &&
                       m->rate >= 0.95 * link_gbps[st.dir] * (double)st.routes.size();
    const int mult = owner ? kOwnerCoalesce : 1;
    // A stage with slack (rate >= 2x its least) that shares the link with a stage
    // running at its least rate yields: no lookahead and one batch on the engines at
    // a time. The copy engines split the link evenly among streams with DMAs queued,
    // whatever the batch schedule, so a loose stage that always has a batch queued
    // takes 1/k of the link from a tight one whose least rate is more than that.
    // ("tight": held at its least rate, and that rate is a real share of the link —
    // a loose stage parked at a token least rate behind the earliest arrival is not.
    // Conservative across roots: one arbiter spans every link of a direction, so a
    // stage also yields to a tight stage on another GPU's root; that only slows it.)
    bool yield = false;
    if (!owner && arb.stages.items.size() > 1 && m->rate >= 2.0 * m->demand.least) {
      const double floor_gbps = 0.1 * link_gbps[st.dir];
      for (auto& kv : arb.stages.items) {
        const auto& o = kv.second;
        if (kv.first != st.key && o.started && o.rate < 1.2 * o.demand.least && o.demand.least >= floor_gbps) {
          yield = true;
          break;
        }
      }
    }
    const double la = yield ? 0.0 : kLookahead;
    if (!owner && t < st.next_t - la * dur) return st.next_t - la * dur;
    int queued = 0;
    for (auto& b : st.inflight) queued += b.batches;
    bool full = st.pinned ? queued + mult > (yield ? 1 : kInflightBatches)
                          : st.jobs * host_chunk >= 2 * (uint64_t)batch_chunks * chunk;
    if (full) {
      if (!st.was_full) note(st, "full", (double)st.inflight.size());
      st.was_full = true;
      return t + 0.02;
    }
    st.was_full = false;
    try {
      issue_batch(st, mult);
    } catch (const CudaFail& f) {
      fail(st, f.msg);
    } catch (const ft::Error& e) {
      fail(st, e.what());
    }
    st.next_t = owner ? t + mult * dur : st.next_t + dur;
    return t;  // re-evaluate at once (lookahead may allow another batch)
  }

  // ------------------------------------------------------------ pacer thread
  void run() {
    prctl(PR_SET_TIMERSLACK, 1000UL, 0, 0, 0);  // 1 us timer slack: batch slots are ~0.2 ms
    std::unique_lock<std::mutex> lk(mu);
    for (;;) {
      bool draining = poll_landing();
      retire_landed();
      if (stop && active.empty()) return;
      double t = now();
      deliver_due(t);
      guard_pending(t);
      double wake = INFINITY;
      bool waiting_land = false;
      for (auto& kv : active) {
        Stage& st = *kv.second;
        if (st.sealed) {
          waiting_land = true;
          continue;
        }
        if (!st.managed || st.issued) continue;
        wake = std::min(wake, step(st, t));
      }
      double armed = next_armed();
      if (!std::isnan(armed)) wake = std::min(wake, armed);
      if (waiting_land || draining) wake = std::min(wake, t + 0.02);  // landing poll
      if (wake <= t) continue;
      if (std::isinf(wake)) {
        if (active.empty())
          cv.wait(lk);
        else
          cv.wait_for(lk, std::chrono::milliseconds(5));
      } else {
        cv.wait_for(lk, std::chrono::duration<double, std::milli>(wake - t));
      }
    }
  }

  // ------------------------------------------------------------ workers (pageable)
  void work() {
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu);
        jcv.wait(lk, [&] { return stop || !jobs.empty(); });
        if (jobs.empty()) return;
        j = jobs.front();
        jobs.pop_front();
      }
      int k;
      {
        std::unique_lock<std::mutex> lk(hmu);
        k = hnext;
        hnext = (hnext + 1) % (int)hslots.size();
        hcv.wait(lk, [&] { return !hslots[k].busy; });
        hslots[k].busy = true;
      }
      HostSlot& hs = hslots[k];
      if (hs.last_dev >= 0) cudaEventSynchronize(hs.ev[hs.last_dev]);  // its previous DMA drained it
      uint8_t* slot = hring + (uint64_t)k * host_chunk;
      const uint8_t* src = nullptr;
      {
        std::lock_guard<std::mutex> lk(mu);
        auto it = active.find(j.ticket);
        if (it != active.end() && it->second->err == FT_OK) src = it->second->host + j.obj_off;
      }
      if (src) stream_copy(slot, src, j.n);  // the tube keeps the object alive until landing
      {
        std::lock_guard<std::mutex> lk(mu);
        auto it = active.find(j.ticket);
        if (it != active.end()) {
          Stage& st = *it->second;
          Route& r = st.routes[j.route];
          try {
            if (st.err == FT_OK) {
              cudaStream_t rd = issue(r, st.dst + j.obj_off, slot, j.n, 0);  // pageable: host->GPU only
              DevGuard g(r.dev);
              if (!hs.ev[r.dev]) ck(cudaEventCreateWithFlags(&hs.ev[r.dev], cudaEventDisableTiming), "event");
              ck(cudaEventRecord(hs.ev[r.dev], rd), "record slot");  // the CE read of the slot
              hs.last_dev = r.dev;
            }
            --st.jobs;
            if (st.jobs == 0 && st.issued && st.err == FT_OK) seal(st);
          } catch (const CudaFail& f) {
            if (st.jobs > 0) --st.jobs;
            fail(st, f.msg);
          }
          if (st.jobs == 0 && st.err != FT_OK) fail(st, st.msg);
        }
      }
      {
        std::lock_guard<std::mutex> lk(hmu);
        hs.busy = false;
      }
      hcv.notify_all();
      cv.notify_all();
    }
  }

  int wait_ticket(std::unique_lock<std::mutex>& lk, uint64_t ticket, double timeout_ms) {
    auto pred = [&] { return !active.count(ticket); };
    if (timeout_ms < 0) {
      done_cv.wait(lk, pred);
    } else if (!done_cv.wait_for(lk, std::chrono::duration<double, std::milli>(timeout_ms), pred)) {
      ft::set_last_error("ft_pacer_wait: timeout");
      return FT_E_TIMEOUT;
    }
    auto it = errors.find(ticket);
    if (it != errors.end()) {
      ft::set_last_error(it->second.second);
      return it->second.first;
    }
    return FT_OK;
  }
};

extern "C" {

int ft_pacer_create(double bw_all_gbps, int links, int batch_chunks, int64_t chunk_bytes, int staging_slots,
                    uint64_t host_ring_bytes, int flags, ft_pacer** out) {
  int logging = flags & 1;
  if (!out || batch_chunks <= 0 || chunk_bytes <= 0 || !(bw_all_gbps > 0)) {
    ft::set_last_error("ft_pacer_create: bad arguments");
    return FT_E_VALUE;
  }
  auto p = std::make_unique<ft_pacer>();
  p->batch_chunks = batch_chunks;
  p->chunk = (uint64_t)chunk_bytes;
  p->staging_slots = std::max(2, staging_slots);
  p->stage_chunk = 4 * (uint64_t)chunk_bytes;
  if (const char* c = std::getenv("FT_K2")) p->k2 = std::atoi(c) != 0;
  if (const char* c = std::getenv("FT_K2_CE2")) p->ce_alt = std::atoi(c) != 0;
  if (const char* c = std::getenv("FT_STAGE_CHUNK")) {
    p->stage_chunk = std::max<uint64_t>(1 << 16, std::atoll(c));
    p->fixed_stage_chunk = true;
  }
  p->logging = logging != 0;
  for (auto& a : p->arbs) a.quiet = !p->logging;  // the decision JSON is only read by the log
  p->links = std::max(1, links);
  p->link_gbps[0] = p->link_gbps[1] = bw_all_gbps / p->links;
  p->adapt = !(flags & 2);
  for (auto& a : p->arbs) {
    a.share = ft::PcieState{bw_all_gbps, batch_chunks, chunk_bytes, {}};
    a.batch_bytes = (double)(chunk_bytes * batch_chunks);
  }
  p->host_chunk = (uint64_t)chunk_bytes;
  if (const char* c = std::getenv("FT_HOST_CHUNK")) p->host_chunk = std::max<uint64_t>(1 << 16, std::atoll(c));
  uint64_t slots = std::max<uint64_t>(4, host_ring_bytes / p->host_chunk);
  void* h = nullptr;
  cudaError_t e = cudaHostAlloc(&h, slots * p->host_chunk, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    ft::set_last_error(std::string("ft_pacer_create: pinned ring: ") + cudaGetErrorString(e));
    return FT_E_CUDA;
  }
  p->hring = static_cast<uint8_t*>(h);
  p->hslots = std::vector<HostSlot>(slots);
  ft_pacer* raw = p.get();
  raw->pacer = std::thread([raw] { raw->run(); });
  int nw = kWorkers;
  if (const char* w = std::getenv("FT_PACER_WORKERS")) nw = std::max(1, std::atoi(w));
  for (int i = 0; i < nw; ++i) raw->workers.emplace_back([raw] { raw->work(); });
  *out = p.release();
  return FT_OK;
}

int ft_pacer_destroy(ft_pacer* p) {
  if (!p) return FT_OK;
  int rc = FT_OK;
  {
    std::unique_lock<std::mutex> lk(p->mu);
    bool drained = p->done_cv.wait_for(lk, std::chrono::seconds(120), [&] { return p->active.empty(); });
    if (!drained) {
      for (auto& kv : p->active) p->fail(*kv.second, "pacer destroyed with the stage in flight");
      ft::set_last_error("ft_pacer_destroy: stages still in flight after 120 s (failed)");
      rc = FT_E_TIMEOUT;
    }
    p->stop = true;
  }
  p->cv.notify_all();
  p->jcv.notify_all();
  p->pacer.join();
  for (auto& t : p->workers) t.join();
  for (auto& kv : p->krings) {
    DevGuard g(kv.first);
    cudaDeviceSynchronize();
    cudaFree(kv.second.buf);
    ft::fwd_ring_words_free(kv.first, kv.second.landed, kv.second.err);
  }
  for (auto& kv : p->ce2) {
    cudaStreamSynchronize(kv.second);
    cudaStreamDestroy(kv.second);
  }
  for (auto& kv : p->rings) {
    DevGuard g(kv.first);
    cudaDeviceSynchronize();
    for (auto e : kv.second.landed) cudaEventDestroy(e);
    for (auto e : kv.second.freed) cudaEventDestroy(e);
    cudaFree(kv.second.buf);
  }
  for (int d = 0; d < kMaxDev; ++d) {
    for (auto e : p->evpool[d]) cudaEventDestroy(e);
    for (auto e : p->tpool[d]) cudaEventDestroy(e);
  }
  for (auto& hs : p->hslots)
    for (int d = 0; d < kMaxDev; ++d)
      if (hs.ev[d]) {
        cudaEventSynchronize(hs.ev[d]);
        cudaEventDestroy(hs.ev[d]);
      }
  cudaFreeHost(p->hring);
  delete p;
  return rc;
}

static int submit_impl(ft_pacer* p, int dir, const char* key, int managed, double slo_ms, double infer_ms,
                       double per_branch_cap_gbps, void* dst, int dst_dev, void* host, uint64_t bytes,
                       int host_pinned, int k, const ft_route* routes, void* consumer_stream, uint64_t* ticket) {
  if (!p || !ticket || k <= 0 || !routes || (bytes && (!dst || !host)) || dst_dev < 0 || dst_dev >= kMaxDev) {
    ft::set_last_error("ft_pacer_submit: bad arguments");
    return FT_E_VALUE;
  }
  if (dir == 1 && !host_pinned) {
    ft::set_last_error("ft_pacer_submit_d2h: the host destination must be pinned");
    return FT_E_VALUE;
  }
  uint64_t covered = 0;
  for (int i = 0; i < k; ++i) {
    const ft_route& r = routes[i];
    if (r.stage_dev < 0 || r.stage_dev >= kMaxDev || !r.ce_stream || r.off + r.len > bytes ||
        (r.stage_dev != dst_dev && !r.fw_stream)) {
      ft::set_last_error("ft_pacer_submit: bad route (device, streams or range)");
      return FT_E_VALUE;
    }
    covered += r.len;
  }
  if (covered != bytes) {
    ft::set_last_error("ft_pacer_submit: routes do not cover the object");
    return FT_E_VALUE;
  }
  auto sp = std::make_shared<Stage>();
  Stage& st = *sp;
  st.managed = managed != 0;
  st.dir = dir;
  st.dst = static_cast<uint8_t*>(dst);
  st.dst_dev = dst_dev;
  st.host = static_cast<uint8_t*>(host);
  st.pinned = host_pinned != 0;
  st.bytes = bytes;
  for (int i = 0; i < k; ++i) {
    Route r;
    r.dev = routes[i].stage_dev;
    r.off = routes[i].off;
    r.len = routes[i].len;
    r.ce = (cudaStream_t)routes[i].ce_stream;
    r.fw = r.dev == dst_dev && !routes[i].force_staging ? nullptr : (cudaStream_t)routes[i].fw_stream;
    st.routes.push_back(r);
  }
  cudaStream_t cs = (cudaStream_t)consumer_stream;
  // A stage of one direct pinned route issues its DMAs on the consumer's own stream:
  // no cross-stream event hops (consumer -> CE stream -> consumer) around them —
  // measured at 1 MiB the hops cost ~10 us of device time over a raw copy
  // (tools/prof_h2g.py). The stage's batches still go out at its rate (the pacer
  // thread issues them onto that stream while submit() waits for the last one), and
  // tenants stay apart: each one's DMAs queue on its own stream.
  const bool inline_route = dir == 0 && st.pinned && k == 1 && !st.routes[0].staged() &&
                            st.routes[0].dev == dst_dev && bytes > 0;
  if (inline_route) st.routes[0].ce = cs;
  st.inline_route = inline_route;
  std::unique_lock<std::mutex> lk(p->mu);
  // a stage that already landed but that the pacer thread has not polled yet (it
  // looks every 20 us) must leave the arbiter before this one starts: otherwise the
  // newcomer is partitioned against a finished stage and runs at half rate until its
  // next boundary (1-2 % of back-to-back e2e steps at 1.7 vs 1.33 ms)
  if (managed) {
    p->poll_landing();
    p->retire_landed();
  }
  st.ticket = p->next_ticket++;
  // (an unnamed host->GPU stage is "h<ticket>": the tube's own names are "m<n>")
  st.key = key && *key ? std::string(key) : (dir == 0 ? "h" : "m") + std::to_string(st.ticket);
  try {
    // the routes start after the consumer stream's prior work (object ready, dst free)
    DevGuard g(dst_dev);
    if (!inline_route) {
      cudaEvent_t e = p->get_event(dst_dev);
      ck(cudaEventRecord(e, cs), "record consumer");
      for (auto& r : st.routes) {
        DevGuard gr(r.dev);
        ck(cudaStreamWaitEvent(r.ce, e, 0), "route waits consumer");
        if (r.staged()) {
          ck(cudaStreamWaitEvent(r.fw, e, 0), "forward waits consumer");
          if (dir == 0 && p->k2) ck(cudaStreamWaitEvent(p->ce_pair(r.ce, r.dev), e, 0), "CE pair waits consumer");
        }
      }
      p->put_event(dst_dev, e);
    }
    ++p->n_stages;
    p->note(st, "start", (double)bytes);
    if (st.managed) {
      ++p->n_managed;
      double t = p->now();
      // the branch cap is the plan's link rate — the same calibration the estimator
      // corrects: a link measured faster than planned caps at the measurement
      double cap = p->adapt ? std::max(per_branch_cap_gbps, p->link_gbps[dir]) : per_branch_cap_gbps;
      p->arb_of(st).start(t, st.key, (double)bytes, slo_ms, infer_ms, t, cap, k);  // engine.py:537-575
      p->arb_log(dir, t, "start", st.key, cap);
      if (bytes == 0) {
        st.issued = true;
        p->seal(st);
      } else if (st.pinned) {
        // the first batches go out from the submitting thread: no pacer wake-up latency
        for (int i = 0; i < kInflightBatches && !st.issued && p->step(st, t) <= t; ++i) {
        }
      }
    } else {
      for (int i = 0; i < k; ++i) {
        p->hand_out(st, i, 0, st.routes[i].len, false);  // one DMA op per range (pinned)
        st.routes[i].done = st.routes[i].len;
      }
      st.issued = true;
      if (st.jobs == 0) p->seal(st);
    }
  } catch (const CudaFail& f) {
    p->fail(st, f.msg);
  } catch (const ft::Error& e) {
    p->fail(st, e.what());
    st.err = e.code;
  }
  *ticket = st.ticket;
  p->active.emplace(st.ticket, sp);
  p->cv.notify_all();
  // every byte enqueued (a paced stage: its last batch issued) -> the consumer waits on the routes
  p->done_cv.wait(lk, [&] { return st.sealed; });
  int rc = st.err;
  std::string msg = st.msg;
  if (rc == FT_OK) {
    try {
      DevGuard g(dst_dev);
      for (auto& e : st.join) ck(cudaStreamWaitEvent(cs, e.first, 0), "consumer waits route");
    } catch (const CudaFail& f) {
      rc = FT_E_CUDA;
      msg = f.msg;
    }
  }
  for (auto& e : st.join) p->put_event(e.second, e.first);  // the waits captured their records
  st.join.clear();
  if (rc != FT_OK) ft::set_last_error(msg);
  return rc;
}

int ft_pacer_submit(ft_pacer* p, const char* key, int managed, double slo_ms, double infer_ms,
                    double per_branch_cap_gbps, void* dst, int dst_dev, const void* host, uint64_t bytes,
                    int host_pinned, int k, const ft_route* routes, void* consumer_stream, uint64_t* ticket) {
  return submit_impl(p, 0, key, managed, slo_ms, infer_ms, per_branch_cap_gbps, dst, dst_dev, const_cast<void*>(host),
                     bytes, host_pinned, k, routes, consumer_stream, ticket);
}

int ft_pacer_submit_d2h(ft_pacer* p, const char* key, int managed, double slo_ms, double infer_ms,
                        double per_branch_cap_gbps, void* host_dst, const void* src, int src_dev, uint64_t bytes,
                        int k, const ft_route* routes, void* producer_stream, uint64_t* ticket) {
  return submit_impl(p, 1, key, managed, slo_ms, infer_ms, per_branch_cap_gbps, const_cast<void*>(src), src_dev,
                     host_dst, bytes, 1, k, routes, producer_stream, ticket);
}

int ft_pacer_wait(ft_pacer* p, uint64_t ticket, double timeout_ms) {
  if (!p) {
    ft::set_last_error("null argument: p");
    return FT_E_VALUE;
  }
  std::unique_lock<std::mutex> lk(p->mu);
  return p->wait_ticket(lk, ticket, timeout_ms);
}

int ft_pacer_done(ft_pacer* p, uint64_t ticket, int* done) {
  if (!p || !done) {
    ft::set_last_error("ft_pacer_done: null argument");
    return FT_E_VALUE;
  }
  std::lock_guard<std::mutex> lk(p->mu);
  *done = !p->active.count(ticket);
  return FT_OK;
}

int ft_pacer_stats(ft_pacer* p, uint64_t* out, int cap) {
  if (!p || !out) {
    ft::set_last_error("ft_pacer_stats: null argument");
    return FT_E_VALUE;
  }
  std::lock_guard<std::mutex> lk(p->mu);
  uint64_t v[7] = {p->n_stages, p->n_managed, p->n_batches, p->n_bytes, (uint64_t)p->active.size(), p->n_errors,
                   0};
  for (int i = 0; i < cap && i < 7; ++i) out[i] = v[i];
  return FT_OK;
}

int ft_pacer_now_ms(ft_pacer* p, double* out) {
  if (!p || !out) {
    ft::set_last_error("ft_pacer_now_ms: null argument");
    return FT_E_VALUE;
  }
  *out = p->now();
  return FT_OK;
}

static int emit_list(const std::vector<std::string>& v, char* buf, size_t cap, size_t* need) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) s += ",";
    s += v[i];
  }
  s += "]";
  if (need) *need = s.size() + 1;
  if (!buf || cap < s.size() + 1) {
    ft::set_last_error("json output buffer too small");
    return FT_E_TRUNCATED;
  }
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return FT_OK;
}

int ft_pacer_trace_json(ft_pacer* p, char* buf, size_t cap, size_t* need) {
  if (!p) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(p->mu);
  return emit_list(p->trace, buf, cap, need);
}

int ft_pacer_log_json(ft_pacer* p, char* buf, size_t cap, size_t* need) {
  if (!p) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(p->mu);
  return emit_list(p->log, buf, cap, need);
}

int ft_pacer_state_json(ft_pacer* p, char* buf, size_t cap, size_t* need) {
  if (!p) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(p->mu);
  std::string s = p->arbs[0].state_json();
  if (need) *need = s.size() + 1;
  if (!buf || cap < s.size() + 1) {
    ft::set_last_error("json output buffer too small");
    return FT_E_TRUNCATED;
  }
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return FT_OK;
}

}  // extern "C"
