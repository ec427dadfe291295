// The daemon's native lane: function-process put/get served by a C++ worker
// thread per connection (PAPER.md:557, 568, 805 — the per-GPU daemon that
// function processes talk to over a local channel, GPU buffers handed over by
// CUDA IPC). The hot requests arrive as binary messages on the connection's
// shared-memory ring (chan.cc) and are answered without Python:
//
//   unique_id  FaaSTube.unique_id                    dataplane.py:69-70
//   commit     FaaSTube.store of a lent pool block    engine.py:342-360 (zero copy)
//              + the lend of the producer's next block (datastore.py:130-144 reuse)
//   fetch      FaaSTube.fetch, same GPU: a zero-copy view of the stored block
//              (dataplane.py:184-185), the consumer counted (engine.py:667-679)
//   done       the view's release: the block returns once the last view is gone
//
// Objects committed here live in the lane's table until their last consumer is
// done. The decisions that belong to the tube run in Python, in order, from an
// event queue the tube drains (index entries are written here at once, so a
// later store of the same id fails and a fetch after the retire misses):
//
//   COMMITTED  histogram sample + live/stored accounting + shrink timer + cap check
//   RETIRED    accounting (the index entry is already gone)
//   FREED      the block back to the pool policy, fenced on the reader's event
//   STOCK      refill a connection's stock of lendable blocks of a size class
//   UNPIN      a view's release of an object the tube has since adopted
//
// Anything else (msgpack requests, misses, responses, host payloads) is handed to
// the connection's Python thread, one request at a time: the worker waits until
// Python has replied before it reads the next message, so replies keep request
// order and only one side writes the reply ring at a time. The tube adopts lane
// objects (ft_lane_take) whenever it needs them in its own table (in-process
// fetches, migration, release, close).
#include <cuda_runtime.h>
#include <poll.h>
#include <sys/socket.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.h"
#include "forward.h"

namespace {

enum : uint8_t { OP_COMMIT = 1, OP_FETCH = 2, OP_DONE = 3, OP_UID = 4 };
enum : uint8_t { REP_KIND = 0xB1 };
enum : uint32_t { EV_COMMITTED = 1, EV_RETIRED = 2, EV_FREED = 3, EV_STOCK = 4, EV_UNPIN = 5 };
constexpr int kDtypes = 10;
const int kItem[kDtypes] = {1, 1, 2, 4, 8, 2, 2, 4, 8, 1};  // uint8 int8 int16 int32 int64 f16 bf16 f32 f64 bool
constexpr int kMaxDim = 8;
// lendable blocks kept per (GPU, size class): a steady producer takes one per commit
// while the tube refills asynchronously (a refill costs it ~0.1 ms), so one block of
// headroom was not enough (most commits missed and paid an alloc round trip)
constexpr size_t kStockDepth = 3;
constexpr uint64_t kTokenBase = 1ull << 62;

#pragma pack(push, 1)
struct CommitReq {
  uint8_t op, dtype, ndim, response;
  int32_t ev, consumers;
  uint32_t name_len;
  uint64_t token;
  int64_t did;
  uint64_t next;  // byte count of the producer's next output (0: none)
};
struct FetchReq {
  uint8_t op, pad[3];
  int32_t gpu;
  int64_t did;
  double slo_ms, infer_ms;  // NaN: None (used only when Python serves it)
};
struct DoneReq {
  uint8_t op, pad[3];
  int32_t ev;
  uint64_t token;
};
struct RepHdr {
  uint8_t kind, ok, has_fd, pad;
  uint32_t acked, n_drop, pad2;
};
struct BlockRep {
  uint64_t token, arena, off, arena_bytes, nbytes;
  int32_t ev;
  uint8_t dtype, ndim, loan, pad;
};
struct EvRec {  // == ft_lane_event (include/faastube.h)
  uint32_t kind, name_len;
  int64_t did;
  int32_t gpu, consumers;
  int64_t pbid;
  uint64_t nbytes;
  double now_ms;
  uint64_t handle;  // cudaEvent_t (FREED / UNPIN fence), ownership passes to the tube
};
#pragma pack(pop)

struct LBlock {
  int64_t pbid = -1;   // pool policy block id (the tube's PoolBlock)
  uint64_t vmm = 0;    // VMM block id (export / locate)
  uint8_t* ptr = nullptr;
  uint64_t cap = 0;    // class bytes
  uint64_t arena = 0, off = 0, arena_bytes = 0;
  int gpu = -1;
  std::vector<cudaEvent_t> fences;  // the previous holder's last users (the tube keeps them alive)
  cudaEvent_t own = nullptr;        // or: the lane's fence event of a recycled block's last users
};

struct LObj {
  int64_t did = 0;
  LBlock blk;
  uint64_t nbytes = 0;
  uint8_t dtype = 0;
  std::vector<int64_t> shape;
  std::string producer;
  int consumers = 1, remaining = 1, pins = 0;
  bool retired = false;
  bool adopted = false;  // the tube took it while views were alive (their releases go to it)
  cudaEvent_t ready = nullptr;
  double stored_at = 0.0;
  uint64_t conn = 0;        // the committing connection, and the client's mark the commit waited for
  uint32_t commit_seq = 0;  //   (a client that dies before that mark executes never wrote the bytes)
  bool has_seq = false;
};

struct Token {
  int kind = 0;  // 1 lend (blk), 2 view (did)
  LBlock blk;
  int64_t did = 0;
};

int64_t now_us() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (int64_t)ts.tv_sec * 1000000 + ts.tv_nsec / 1000;
}

}  // namespace

struct ft_lane;

struct ft_lane_conn {
  ft_lane* lane = nullptr;
  ft_chan* ch = nullptr;
  int sock = -1;
  int gpu = -1;
  cudaStream_t stream = nullptr;
  // ordering with the client: two words of pool memory both processes map; each side
  // writes its next sequence number after its work (stream memory op) and the other
  // side's stream waits for it (a cross-process CUDA event took ~110 us to resolve)
  uint32_t* c2d = nullptr;  // the client's marks
  uint32_t* d2c = nullptr;  // ours
  uint32_t seq_d = 0;       // our last mark
  uint32_t seen_c = 0;      // the client's highest mark we waited for (a dead client's waits are released)
  bool any_c = false;
  uint32_t served = 0;
  std::set<std::pair<int, uint64_t>> mapped;  // (gpu, arena) the client has mapped
  std::vector<uint64_t> drops;                // arenas to unmap, sent with the next reply
  std::set<uint64_t> tokens;                  // native tokens of this connection
  uint64_t id = 0;                            // the lane's connection id (stock refills name it)
  // lendable blocks per size class for this producer's next outputs: returned to the
  // pool when the connection goes away
  std::map<uint64_t, std::deque<LBlock>> stock;
  std::set<uint64_t> stock_asked;
  // hand-off of one request to Python
  std::mutex fmu;
  std::condition_variable fcv;
  std::string fwd;
  bool has_fwd = false, py_busy = false, dead = false, stop = false;
  bool gone = false;  // (lane->mu) the worker has released everything: no more stock
  std::thread worker;
  std::string rep;  // reply buffer (worker)
};

struct ft_lane {
  std::mutex mu;  // table, stock, tokens, conns' mapped/drops
  double t0 = 0.0;  // the tube's clock origin (CLOCK_MONOTONIC seconds)
  int node = 0;
  ft_index* index = nullptr;
  std::map<int, ft_vmm_pool*> pools;
  std::unordered_map<int64_t, LObj> objs;
  std::unordered_map<uint64_t, Token> tokens;
  uint64_t next_token = kTokenBase;
  std::vector<ft_lane_conn*> conns;
  uint64_t next_conn = 1;
  std::map<int, std::vector<cudaEvent_t>> evpool;
  // event queue to the tube. While events keep coming the service thread polls the
  // queue (every kPollUs) instead of sleeping on `ecv`: a wake-up per event put a
  // futex syscall into every request the workers answer (~5 us a request). After
  // kIdleUs without an event it sleeps on `ecv` (`sleeping`) and the next emit wakes it.
  static constexpr int64_t kPollUs = 500, kIdleUs = 20000;
  std::mutex emu;
  std::condition_variable ecv;
  std::string events;
  bool sleeping = false;
  int64_t last_emit_us = 0;
  uint64_t stats[10] = {};  // commits, fetches, dones, uids, forwarded, stock hits / misses, adopted, recycled, lost

  double now_ms() const { return ((double)now_us() * 1e-6 - t0) * 1e3; }
  cudaEvent_t get_event(int gpu) {
    auto& v = evpool[gpu];
    if (!v.empty()) {
      cudaEvent_t e = v.back();
      v.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != gpu) cudaSetDevice(gpu);
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (cur != gpu && cur >= 0) cudaSetDevice(cur);
    return e;
  }
  void put_event(int gpu, cudaEvent_t e) {
    if (e) evpool[gpu].push_back(e);
  }
  void emit(const EvRec& r, const std::string& name = std::string()) {
    std::lock_guard<std::mutex> lk(emu);
    EvRec x = r;
    x.name_len = (uint32_t)name.size();
    events.append(reinterpret_cast<const char*>(&x), sizeof x);
    events.append(name);
    last_emit_us = now_us();
    if (sleeping) ecv.notify_all();
  }
};

namespace {

uint64_t size_class_bytes(uint64_t n) {
  int64_t c = 0;
  if (ft_size_class((double)(n ? n : 1), &c) != FT_OK) return n;
  return (uint64_t)c;
}

// mark: our next sequence number, written to d2c after the connection stream's work
// (0 and ~0 are never used: 0 means "no mark" in the protocol, ~0 is -1 as int32)
int mark(ft_lane_conn* c) {
  if (!c->d2c) return 0;
  uint32_t v = c->seq_d + 1;
  if (v == 0 || v == 0xFFFFFFFFu) v = 1;
  if (ft::mem_write32(c->stream, c->d2c, v) != FT_OK) return 0;
  c->seq_d = v;
  return (int)v;
}
void wait_peer(ft_lane_conn* c, int ev) {
  if (!c->c2d || ev == 0 || ev == -1) return;
  const uint32_t v = (uint32_t)ev;
  ft::mem_wait_geq32(c->stream, c->c2d, v);
  if (!c->any_c || (int32_t)(v - c->seen_c) > 0) c->seen_c = v;
  c->any_c = true;
}
// (lane->mu held) a client that went away may never write the marks our stream waits
// for. The last mark it did write is read back: objects it committed after that mark
// were never written, so they are dropped (a later fetch misses, nobody reads garbage).
// Then the highest mark is written from the host (a separate stream: the connection
// stream is parked on it), releasing the waits.
void retire_obj(ft_lane* L, LObj& o);
void free_obj(ft_lane* L, ft_lane_conn* c, LObj& o);
void release_dead(ft_lane* L, ft_lane_conn* c) {
  if (!c->c2d || !c->any_c) return;
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return;
  uint32_t written = 0, v = c->seen_c;
  cudaMemcpyAsync(&written, c->c2d, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  std::vector<int64_t> lost;
  for (auto& kv : L->objs) {
    const LObj& o = kv.second;
    if (o.conn == c->id && o.has_seq && !o.retired && !o.adopted && (int32_t)(o.commit_seq - written) > 0)
      lost.push_back(kv.first);
  }
  cudaMemcpyAsync(c->c2d, &v, 4, cudaMemcpyHostToDevice, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  for (int64_t did : lost) {
    auto it = L->objs.find(did);
    if (it == L->objs.end()) continue;
    ++L->stats[9];
    retire_obj(L, it->second);
    if (it->second.pins <= 0) free_obj(L, c, it->second);
  }
}


// header + payload + drops; fd sent after the message when `fd >= 0`
int send_reply(ft_lane_conn* c, const std::string& payload, bool ok, int fd) {
  std::vector<uint64_t> drops;
  {
    // at most 256 notices per reply (the rest ride on the next ones): a reply fits a slot
    std::lock_guard<std::mutex> lk(c->lane->mu);
    const size_t k = std::min<size_t>(c->drops.size(), 256);
    drops.assign(c->drops.begin(), c->drops.begin() + k);
    c->drops.erase(c->drops.begin(), c->drops.begin() + k);
  }
  c->served += 1;
  RepHdr h{REP_KIND, (uint8_t)ok, (uint8_t)(fd >= 0), 0, c->served, (uint32_t)drops.size(), 0};
  std::string& b = c->rep;
  b.clear();
  b.append(reinterpret_cast<const char*>(&h), sizeof h);
  b.append(payload);
  for (uint64_t d : drops) b.append(reinterpret_cast<const char*>(&d), 8);
  int rc = ft_chan_send(c->ch, 1, b.data(), (uint32_t)b.size(), 5000000);
  if (rc == FT_OK && fd >= 0) rc = ft_fd_send(c->sock, fd, 0);
  return rc;
}

int send_error(ft_lane_conn* c, const char* name, const std::string& msg) {
  std::string p;
  uint32_t n = (uint32_t)strlen(name), m = (uint32_t)msg.size();
  p.append(reinterpret_cast<const char*>(&n), 4);
  p.append(name, n);
  p.append(reinterpret_cast<const char*>(&m), 4);
  p.append(msg);
  return send_reply(c, p, false, -1);
}

// (lane->mu held) the block's arena, exported once per connection
int arena_fd(ft_lane_conn* c, const LBlock& b, bool* need) {
  auto key = std::make_pair(b.gpu, b.arena);
  *need = !c->mapped.count(key);
  if (!*need) return -1;
  auto it = c->lane->pools.find(b.gpu);
  int fd = -1;
  if (it == c->lane->pools.end() || ft_vmm_block_export_fd(it->second, b.vmm, &fd) != FT_OK) return -2;
  c->mapped.insert(key);
  return fd;
}

// (lane->mu held) a lendable block of `n` bytes on the connection's GPU: its previous
// users are waited on by the connection stream; nullopt-like (pbid < 0) on a miss
bool take_stock(ft_lane* L, ft_lane_conn* c, uint64_t n, LBlock* out) {
  const uint64_t cls = size_class_bytes(n);
  auto& dq = c->stock[cls];
  bool hit = !dq.empty();
  if (hit) {
    *out = std::move(dq.front());
    dq.pop_front();
    for (cudaEvent_t f : out->fences) cudaStreamWaitEvent(c->stream, f, 0);
    out->fences.clear();
    if (out->own) {  // (the wait captured the record: the event can be reused)
      cudaStreamWaitEvent(c->stream, out->own, 0);
      L->put_event(out->gpu, out->own);
      out->own = nullptr;
    }
    ++L->stats[5];
  } else {
    ++L->stats[6];
  }
  if (dq.size() < kStockDepth && !c->stock_asked.count(cls)) {
    c->stock_asked.insert(cls);
    EvRec r{};
    r.kind = EV_STOCK;
    r.did = (int64_t)c->id;                             // the connection to stock
    r.gpu = c->gpu;
    r.consumers = (int32_t)(kStockDepth - dq.size());  // blocks wanted
    r.nbytes = cls;
    L->emit(r);
  }
  return hit;
}

// (lane->mu held) a connection's stocked blocks go back to the pool (a recycled one
// with its last users' fence, whose ownership passes to the tube)
void return_stock(ft_lane* L, ft_lane_conn* c) {
  for (auto& kv : c->stock)
    for (auto& b : kv.second) {
      EvRec r{};
      r.kind = EV_FREED;
      r.gpu = b.gpu;
      r.pbid = b.pbid;
      r.handle = (uint64_t)(uintptr_t)b.own;
      L->emit(r);
    }
  c->stock.clear();
  c->stock_asked.clear();
}

// (lane->mu held) a block whose last users are fenced by the lane's event `f` goes
// straight into the stock of a connection that lends its size class and is below
// depth — the pool policy's exact-class reuse (datastore.py:130-144) without the
// round trip through the tube; false: the caller returns it to the pool
bool recycle(ft_lane* L, const LBlock& blk, cudaEvent_t f) {
  for (auto* x : L->conns) {
    if (x->gone || x->gpu != blk.gpu) continue;
    auto it = x->stock.find(blk.cap);
    if (it == x->stock.end() || it->second.size() >= kStockDepth) continue;
    LBlock b = blk;
    b.fences.clear();
    b.own = f;
    it->second.push_back(std::move(b));
    ++L->stats[8];
    return true;
  }
  return false;
}

std::string block_payload(uint64_t token, const LBlock& b, uint64_t nbytes, int ev, uint8_t dtype,
                          const std::vector<int64_t>& shape, bool loan) {
  std::string p;
  BlockRep r{token, b.arena, b.off, b.arena_bytes, nbytes, ev, dtype, (uint8_t)shape.size(), (uint8_t)loan, 0};
  p.append(reinterpret_cast<const char*>(&r), sizeof r);
  for (int64_t d : shape) p.append(reinterpret_cast<const char*>(&d), 8);
  return p;
}

// (lane->mu held) a retired object with no view left: the block goes back to the pool,
// fenced on the connection stream (it waited for the reader's release)
void free_obj(ft_lane* L, ft_lane_conn* c, LObj& o) {
  cudaEvent_t f = L->get_event(c->gpu);
  cudaEventRecord(f, c->stream);
  if (recycle(L, o.blk, f)) {
    L->put_event(o.blk.gpu, o.ready);
    L->objs.erase(o.did);
    return;
  }
  EvRec r{};
  r.kind = EV_FREED;
  r.did = o.did;
  r.gpu = o.blk.gpu;
  r.pbid = o.blk.pbid;
  r.nbytes = o.nbytes;
  r.handle = (uint64_t)(uintptr_t)f;
  L->emit(r, o.producer);
  L->put_event(o.blk.gpu, o.ready);
  L->objs.erase(o.did);
}

void retire_obj(ft_lane* L, LObj& o) {  // (lane->mu held) engine.py:667-679
  o.retired = true;
  ft_index_drop(L->index, o.did);
  EvRec r{};
  r.kind = EV_RETIRED;
  r.did = o.did;
  r.gpu = o.blk.gpu;
  r.pbid = o.blk.pbid;
  r.nbytes = o.nbytes;
  L->emit(r, o.producer);
}

// ---- hot requests ------------------------------------------------------------

bool handle_uid(ft_lane_conn* c) {
  int64_t id = 0;
  ft_index_unique_id(c->lane->index, &id);
  ++c->lane->stats[3];
  std::string p(reinterpret_cast<const char*>(&id), 8);
  send_reply(c, p, true, -1);
  return true;
}

// false: hand it to Python
bool handle_commit(ft_lane_conn* c, const std::string& m) {
  ft_lane* L = c->lane;
  if (m.size() < sizeof(CommitReq)) return false;
  CommitReq q;
  memcpy(&q, m.data(), sizeof q);
  if (q.response || q.ndim > kMaxDim || q.dtype >= kDtypes || c->gpu < 0 ||
      m.size() != sizeof q + 8 * (size_t)q.ndim + q.name_len)
    return false;
  std::vector<int64_t> shape(q.ndim);
  memcpy(shape.data(), m.data() + sizeof q, 8 * (size_t)q.ndim);
  std::string name(m.data() + sizeof q + 8 * q.ndim, q.name_len);
  uint64_t nbytes = (uint64_t)kItem[q.dtype];
  for (int64_t d : shape)  // a negative or overflowing shape: Python rejects it
    if (d < 0 || __builtin_mul_overflow(nbytes, (uint64_t)d, &nbytes)) return false;
  std::unique_lock<std::mutex> lk(L->mu);
  auto tk = L->tokens.find(q.token);
  if (tk == L->tokens.end() || tk->second.kind != 1) return false;  // a Python loan (or unknown): Python
  LBlock blk = tk->second.blk;
  if (nbytes > blk.cap) {
    lk.unlock();
    return false;  // Python reports it (and returns the block)
  }
  // the client's copy into the block is done (stream-ordered), then the index entry
  wait_peer(c, q.ev);
  const double now = L->now_ms();
  double vis = 0.0;
  if (L->objs.count(q.did) ||
      ft_index_store(L->index, q.did, L->node, blk.gpu, (double)nbytes, now, name.c_str(), 0, &vis) != FT_OK) {
    // DuplicateStore: not published; the block goes back to the pool
    L->tokens.erase(tk);
    c->tokens.erase(q.token);
    cudaEvent_t f = L->get_event(c->gpu);
    cudaEventRecord(f, c->stream);
    EvRec r{};
    r.kind = EV_FREED;
    r.did = q.did;
    r.gpu = blk.gpu;
    r.pbid = blk.pbid;
    r.handle = (uint64_t)(uintptr_t)f;
    L->emit(r);
    lk.unlock();
    send_error(c, "DuplicateStore", "data id " + std::to_string(q.did) + " already stored");
    return true;
  }
  L->tokens.erase(tk);
  c->tokens.erase(q.token);
  LObj& o = L->objs[q.did];
  o.did = q.did;
  o.blk = blk;
  o.nbytes = nbytes;
  o.dtype = q.dtype;
  o.shape = shape;
  o.producer = name;
  o.consumers = o.remaining = q.consumers > 0 ? q.consumers : 1;
  o.ready = L->get_event(c->gpu);
  o.stored_at = now;
  o.conn = c->id;
  o.has_seq = q.ev != 0 && q.ev != -1;
  o.commit_seq = (uint32_t)q.ev;
  cudaEventRecord(o.ready, c->stream);
  EvRec r{};
  r.kind = EV_COMMITTED;
  r.did = q.did;
  r.gpu = blk.gpu;
  r.consumers = o.consumers;
  r.pbid = blk.pbid;
  r.nbytes = nbytes;
  r.now_ms = now;
  L->emit(r, name);
  ++L->stats[0];
  // lend the producer's next block now: its next store is one round trip
  LBlock nb;
  bool loan = q.next && take_stock(L, c, q.next, &nb);
  std::string payload;
  int fd = -1;
  if (loan) {
    uint64_t tok = L->next_token++;
    Token t;
    t.kind = 1;
    t.blk = nb;
    L->tokens[tok] = t;
    c->tokens.insert(tok);
    int ev = mark(c);
    bool need = false;
    fd = arena_fd(c, nb, &need);
    if (fd == -2) fd = -1;  // export failed: the client will fail to map and fall back
    payload = block_payload(tok, nb, q.next, ev, 0, {}, true);
  } else {
    BlockRep z{};
    payload.assign(reinterpret_cast<const char*>(&z), sizeof z);
  }
  lk.unlock();
  send_reply(c, payload, true, fd);
  if (fd >= 0) close(fd);
  return true;
}

bool handle_fetch(ft_lane_conn* c, const std::string& m) {
  ft_lane* L = c->lane;
  if (m.size() < sizeof(FetchReq)) return false;
  FetchReq q;
  memcpy(&q, m.data(), sizeof q);
  std::unique_lock<std::mutex> lk(L->mu);
  auto it = L->objs.find(q.did);
  if (it == L->objs.end() || it->second.retired || it->second.adopted || it->second.blk.gpu != q.gpu ||
      q.gpu != c->gpu)
    return false;  // elsewhere (or not ours): Python serves it
  LObj& o = it->second;
  cudaStreamWaitEvent(c->stream, o.ready, 0);  // the stored bytes are in place
  o.pins += 1;
  o.remaining -= 1;
  if (o.remaining <= 0) retire_obj(L, o);
  uint64_t tok = L->next_token++;
  Token t;
  t.kind = 2;
  t.did = o.did;
  L->tokens[tok] = t;
  c->tokens.insert(tok);
  int ev = mark(c);
  bool need = false;
  int fd = arena_fd(c, o.blk, &need);
  if (fd == -2) fd = -1;
  std::string payload = block_payload(tok, o.blk, o.nbytes, ev, o.dtype, o.shape, false);
  ++L->stats[1];
  lk.unlock();
  send_reply(c, payload, true, fd);
  if (fd >= 0) close(fd);
  return true;
}

// (lane->mu held) release one native token: a view (unpin, free when retired) or an
// unused lend (back to the pool). The connection stream has waited for the client.
void release_token(ft_lane* L, ft_lane_conn* c, uint64_t tok) {
  auto tk = L->tokens.find(tok);
  if (tk == L->tokens.end()) return;
  Token t = std::move(tk->second);
  L->tokens.erase(tk);
  c->tokens.erase(tok);
  if (t.kind == 1) {
    cudaEvent_t f = L->get_event(c->gpu);
    cudaEventRecord(f, c->stream);
    if (!c->gone && recycle(L, t.blk, f)) return;
    EvRec r{};
    r.kind = EV_FREED;
    r.gpu = t.blk.gpu;
    r.pbid = t.blk.pbid;
    r.handle = (uint64_t)(uintptr_t)f;
    L->emit(r);
    return;
  }
  auto it = L->objs.find(t.did);
  if (it == L->objs.end()) return;
  LObj& o = it->second;
  o.pins -= 1;
  if (o.adopted) {  // the tube owns it now: it unpins its own object
    cudaEvent_t f = L->get_event(c->gpu);
    cudaEventRecord(f, c->stream);
    EvRec r{};
    r.kind = EV_UNPIN;
    r.did = o.did;
    r.gpu = o.blk.gpu;
    r.handle = (uint64_t)(uintptr_t)f;
    L->emit(r);
    if (o.pins <= 0) L->objs.erase(it);
    return;
  }
  if (o.retired && o.pins <= 0) free_obj(L, c, o);
}

bool handle_done(ft_lane_conn* c, const std::string& m) {
  ft_lane* L = c->lane;
  if (m.size() < sizeof(DoneReq)) return false;
  DoneReq q;
  memcpy(&q, m.data(), sizeof q);
  std::lock_guard<std::mutex> lk(L->mu);
  if (!L->tokens.count(q.token)) return false;  // a Python token
  wait_peer(c, q.ev);  // the client's last read of the block (stream-ordered)
  release_token(L, c, q.token);
  c->served += 1;  // no reply: acknowledged by the next one
  ++L->stats[2];
  return true;
}

// ---- the worker ----------------------------------------------------------------

bool peer_gone(int sock) {
  pollfd p{sock, POLLIN, 0};
  if (poll(&p, 1, 0) <= 0) return false;
  if (p.revents & (POLLHUP | POLLERR | POLLNVAL)) return true;
  char b;
  ssize_t n = recv(sock, &b, 1, MSG_PEEK | MSG_DONTWAIT);
  return n == 0;
}

void forward(ft_lane_conn* c, std::string&& m) {
  std::unique_lock<std::mutex> lk(c->fmu);
  c->fwd = std::move(m);
  c->has_fwd = true;
  c->py_busy = true;
  ++c->lane->stats[4];
  c->fcv.notify_all();
  c->fcv.wait(lk, [&] { return !c->py_busy || c->stop; });
}

void run_worker(ft_lane_conn* c) {
  std::vector<char> buf(1 << 16);
  int spin = 2000;
  if (const char* s = std::getenv("FT_CHAN_SPIN_US")) spin = std::atoi(s);
  for (;;) {
    {
      std::lock_guard<std::mutex> lk(c->fmu);
      if (c->stop) break;
    }
    uint32_t n = 0;
    int rc = ft_chan_recv(c->ch, 0, buf.data(), (uint32_t)buf.size(), &n, spin, 50000);
    if (rc == FT_E_TIMEOUT) {
      if (peer_gone(c->sock)) break;
      continue;
    }
    if (rc != FT_OK) break;  // closed (or a message that cannot fit)
    std::string m(buf.data(), n);
    const uint8_t op = n ? (uint8_t)m[0] : 0;
    bool done = false;
    int dev = c->gpu;
    if (dev >= 0) cudaSetDevice(dev);
    switch (op) {
      case OP_UID: done = handle_uid(c); break;
      case OP_COMMIT: done = handle_commit(c, m); break;
      case OP_FETCH: done = handle_fetch(c, m); break;
      case OP_DONE: done = handle_done(c, m); break;
      default: break;
    }
    if (!done) forward(c, std::move(m));
  }
  // the client is gone (or the daemon closes): its native loans go back, its views are
  // released (the connection stream orders the frees after everything it waited on)
  {
    std::lock_guard<std::mutex> lk(c->lane->mu);
    std::vector<uint64_t> toks(c->tokens.begin(), c->tokens.end());
    if (c->gpu >= 0) cudaSetDevice(c->gpu);
    release_dead(c->lane, c);
    for (uint64_t t : toks) release_token(c->lane, c, t);
    return_stock(c->lane, c);
    c->gone = true;
  }
  std::lock_guard<std::mutex> lk(c->fmu);
  c->dead = true;
  c->fcv.notify_all();
}

}  // namespace

extern "C" {

int ft_lane_create(ft_index* index, int node, double t0_s, ft_lane** out) {
  if (!index || !out) {
    ft::set_last_error("ft_lane_create: bad arguments");
    return FT_E_VALUE;
  }
  auto* L = new ft_lane;
  L->index = index;
  L->node = node;
  L->t0 = t0_s;
  *out = L;
  return FT_OK;
}

int ft_lane_set_pool(ft_lane* L, int gpu, ft_vmm_pool* pool) {
  if (!L || !pool) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(L->mu);
  L->pools[gpu] = pool;
  return FT_OK;
}

int ft_lane_destroy(ft_lane* L) {
  if (!L) return FT_OK;
  for (auto& kv : L->evpool)
    for (cudaEvent_t e : kv.second) cudaEventDestroy(e);
  delete L;
  return FT_OK;
}

// a connection upgraded to shared-memory rings: start its worker
int ft_lane_attach(ft_lane* L, ft_chan* ch, int sock, ft_lane_conn** out) {
  if (!L || !ch || !out) return FT_E_VALUE;
  auto* c = new ft_lane_conn;
  c->lane = L;
  c->ch = ch;
  c->sock = sock;
  {
    std::lock_guard<std::mutex> lk(L->mu);
    c->id = L->next_conn++;
    L->conns.push_back(c);
  }
  c->worker = std::thread(run_worker, c);
  *out = c;
  return FT_OK;
}

int ft_lane_conn_id(ft_lane_conn* c, uint64_t* id) {
  if (!c || !id) return FT_E_VALUE;
  *id = c->id;
  return FT_OK;
}

// after hello: the client's GPU, the connection stream, the two sync words
int ft_lane_conn_set_gpu(ft_lane_conn* c, int gpu, void* stream, void* c2d, void* d2c) {
  if (!c) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(c->lane->mu);
  c->gpu = gpu;
  c->stream = (cudaStream_t)stream;
  c->c2d = static_cast<uint32_t*>(c2d);
  c->d2c = static_cast<uint32_t*>(d2c);
  return FT_OK;
}

int ft_lane_conn_wait(ft_lane_conn* c, uint32_t seq) {
  if (!c) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(c->lane->mu);
  wait_peer(c, (int)seq);
  return FT_OK;
}

// Python's side of a connection: the next request the worker handed over (FT_E_CLOSED
// once the client is gone), then exactly one of reply / finish
int ft_lane_conn_next(ft_lane_conn* c, void* buf, uint32_t cap, uint32_t* n, int64_t timeout_us) {
  if (!c || !n) return FT_E_VALUE;
  std::unique_lock<std::mutex> lk(c->fmu);
  auto pred = [&] { return c->has_fwd || c->dead; };
  if (timeout_us < 0)
    c->fcv.wait(lk, pred);
  else if (!c->fcv.wait_for(lk, std::chrono::microseconds(timeout_us), pred))
    return FT_E_TIMEOUT;
  if (!c->has_fwd) return FT_E_CLOSED;
  *n = (uint32_t)c->fwd.size();
  if (c->fwd.size() > cap) {
    ft::set_last_error("ft_lane_conn_next: buffer too small");
    return FT_E_TRUNCATED;
  }
  memcpy(buf, c->fwd.data(), c->fwd.size());
  c->has_fwd = false;
  return FT_OK;
}

// the message number a reply acknowledges (Python builds msgpack replies itself)
int ft_lane_conn_served(ft_lane_conn* c, uint32_t* out) {
  if (!c || !out) return FT_E_VALUE;
  *out = c->served + 1;
  return FT_OK;
}

// Python's reply to the handed-over request (a msgpack frame, raw on the reply ring)
int ft_lane_conn_reply(ft_lane_conn* c, const void* buf, uint32_t n) {
  if (!c) return FT_E_VALUE;
  c->served += 1;
  int rc = ft_chan_send(c->ch, 1, buf, n, 5000000);
  std::lock_guard<std::mutex> lk(c->fmu);
  c->py_busy = false;
  c->fcv.notify_all();
  return rc;
}

// a binary reply built by Python: header (acked, drops) added here
int ft_lane_conn_reply_bin(ft_lane_conn* c, const void* payload, uint32_t n, int ok, int fd) {
  if (!c) return FT_E_VALUE;
  int rc = send_reply(c, std::string(static_cast<const char*>(payload), n), ok != 0, fd);
  std::lock_guard<std::mutex> lk(c->fmu);
  c->py_busy = false;
  c->fcv.notify_all();
  return rc;
}

// the handed-over request needed no reply (done)
int ft_lane_conn_finish(ft_lane_conn* c) {
  if (!c) return FT_E_VALUE;
  c->served += 1;
  std::lock_guard<std::mutex> lk(c->fmu);
  c->py_busy = false;
  c->fcv.notify_all();
  return FT_OK;
}

// record one of the daemon's events on the connection stream (Python's slow paths)
int ft_lane_conn_mark(ft_lane_conn* c, int* ev) {
  if (!c || !ev) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(c->lane->mu);
  *ev = mark(c);
  return FT_OK;
}

// (gpu, arena) mapped by this client already? (marks it mapped)
int ft_lane_conn_known(ft_lane_conn* c, int gpu, uint64_t arena, int* known) {
  if (!c || !known) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(c->lane->mu);
  auto key = std::make_pair(gpu, arena);
  *known = c->mapped.count(key) ? 1 : 0;
  c->mapped.insert(key);
  return FT_OK;
}

// an arena was unmapped: every connection that mapped it is told with its next reply
int ft_lane_dropped(ft_lane* L, int gpu, uint64_t arena) {
  if (!L) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(L->mu);
  for (auto* c : L->conns)
    if (c->mapped.erase(std::make_pair(gpu, arena))) c->drops.push_back(arena);
  return FT_OK;
}

// pending unmap notices of one connection (for Python's msgpack replies)
int ft_lane_conn_take_drops(ft_lane_conn* c, uint64_t* out, int cap, int* n) {
  if (!c || !n) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(c->lane->mu);
  int k = std::min<int>(cap, (int)c->drops.size());
  for (int i = 0; i < k; ++i) out[i] = c->drops[i];
  c->drops.erase(c->drops.begin(), c->drops.begin() + k);
  *n = k;
  return FT_OK;
}

// a block lent through Python (alloc): the lane owns the token, so its commit is native
int ft_lane_lend(ft_lane_conn* c, int64_t pbid, uint64_t vmm, void* ptr, uint64_t cap, uint64_t arena, uint64_t off,
                 uint64_t arena_bytes, uint64_t* token) {
  if (!c || !token) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(c->lane->mu);
  Token t;
  t.kind = 1;
  t.blk = LBlock{pbid, vmm, static_cast<uint8_t*>(ptr), cap, arena, off, arena_bytes, c->gpu, {}};
  uint64_t tok = c->lane->next_token++;
  c->lane->tokens[tok] = t;
  c->tokens.insert(tok);
  *token = tok;
  return FT_OK;
}

// a lendable block for connection `conn_id`'s stock (the tube allocated it; fences: its
// previous users). FT_E_KEY if the connection is gone (the tube keeps the block).
int ft_lane_stock_put(ft_lane* L, uint64_t conn_id, int gpu, int64_t pbid, uint64_t vmm, void* ptr, uint64_t cap,
                      uint64_t arena, uint64_t off, uint64_t arena_bytes, void* const* fences, int nf) {
  if (!L) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(L->mu);
  ft_lane_conn* c = nullptr;
  for (auto* x : L->conns)
    if (x->id == conn_id && !x->gone) c = x;
  if (!c) {
    ft::set_last_error("no such connection");
    return FT_E_KEY;
  }
  LBlock b{pbid, vmm, static_cast<uint8_t*>(ptr), cap, arena, off, arena_bytes, gpu, {}};
  for (int i = 0; i < nf; ++i) b.fences.push_back(static_cast<cudaEvent_t>(fences[i]));
  c->stock[cap].push_back(std::move(b));
  c->stock_asked.erase(cap);  // (the next take below depth asks again)
  return FT_OK;
}

// the tube's event queue (binary EvRec + name records), waiting up to timeout_us
int ft_lane_events(ft_lane* L, void* buf, uint64_t cap, uint64_t* n, int64_t timeout_us) {
  if (!L || !n) return FT_E_VALUE;
  std::unique_lock<std::mutex> lk(L->emu);
  if (L->events.empty() && timeout_us != 0) {
    if (now_us() - L->last_emit_us < ft_lane::kIdleUs) {
      // busy: look again shortly, without asking the emitters for a wake-up
      lk.unlock();
      std::this_thread::sleep_for(std::chrono::microseconds(
          timeout_us < 0 ? ft_lane::kPollUs : std::min<int64_t>(timeout_us, ft_lane::kPollUs)));
      lk.lock();
    } else {
      auto pred = [&] { return !L->events.empty(); };
      L->sleeping = true;
      if (timeout_us < 0)
        L->ecv.wait(lk, pred);
      else
        L->ecv.wait_for(lk, std::chrono::microseconds(timeout_us), pred);
      L->sleeping = false;
    }
  }
  // whole records only
  uint64_t take = 0;
  while (take + sizeof(EvRec) <= L->events.size()) {
    EvRec r;
    memcpy(&r, L->events.data() + take, sizeof r);
    uint64_t len = sizeof r + r.name_len;
    if (take + len > cap) break;
    take += len;
  }
  memcpy(buf, L->events.data(), take);
  L->events.erase(0, take);
  *n = take;
  return FT_OK;
}

// adopt: the tube takes object `did` into its own table (the ready event's ownership
// passes to it). A pinned object stays listed, marked adopted, so its views' releases
// reach the tube as UNPIN events. FT_E_MISSING if the lane does not hold it.
int ft_lane_take(ft_lane* L, int64_t did, ft_lane_obj* out, int64_t* shape, char* producer, int producer_cap) {
  if (!L || !out || !shape || !producer) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(L->mu);
  auto it = L->objs.find(did);
  if (it == L->objs.end() || it->second.adopted) {
    ft::set_last_error("not in the lane");
    return FT_E_MISSING;
  }
  LObj& o = it->second;
  *out = ft_lane_obj{o.did, o.blk.pbid, o.nbytes, o.stored_at, (void*)o.ready, o.blk.gpu, o.dtype,
                     (int32_t)o.shape.size(), o.retired ? 0 : o.remaining, o.pins, o.consumers};
  memcpy(shape, o.shape.data(), 8 * o.shape.size());
  snprintf(producer, (size_t)producer_cap, "%s", o.producer.c_str());
  ++L->stats[7];
  o.ready = nullptr;
  if (o.pins > 0)
    o.adopted = true;
  else
    L->objs.erase(it);
  return FT_OK;
}

// a lend token Python takes over (a forwarded commit it serves itself): its pool block id
int ft_lane_take_lend(ft_lane_conn* c, uint64_t token, int64_t* pbid) {
  if (!c || !pbid) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(c->lane->mu);
  auto tk = c->lane->tokens.find(token);
  if (tk == c->lane->tokens.end() || tk->second.kind != 1) {
    ft::set_last_error("unknown token " + std::to_string(token));
    return FT_E_KEY;
  }
  *pbid = tk->second.blk.pbid;
  c->lane->tokens.erase(tk);
  c->tokens.erase(token);
  return FT_OK;
}

// Python releases a native token (a forwarded done; the connection stream waited)
int ft_lane_conn_release(ft_lane_conn* c, uint64_t token) {
  if (!c) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(c->lane->mu);
  if (c->gpu >= 0) cudaSetDevice(c->gpu);
  release_token(c->lane, c, token);
  return FT_OK;
}

// ids of the lane's objects (on `gpu`, or all with gpu < 0), not yet adopted
int ft_lane_ids(ft_lane* L, int gpu, int64_t* out, int cap, int* n) {
  if (!L || !n) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(L->mu);
  int k = 0;
  for (auto& kv : L->objs)
    if (!kv.second.adopted && (gpu < 0 || kv.second.blk.gpu == gpu)) {
      if (k < cap) out[k] = kv.first;
      ++k;
    }
  *n = k;
  return k > cap ? FT_E_TRUNCATED : FT_OK;
}

int ft_lane_stats(ft_lane* L, uint64_t* out, int cap) {
  if (!L) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(L->mu);
  for (int i = 0; i < cap && i < 10; ++i) out[i] = L->stats[i];
  return FT_OK;
}

// stop the worker (the client has gone or the daemon closes) and free the connection
int ft_lane_conn_close(ft_lane_conn* c) {
  if (!c) return FT_OK;
  {
    std::lock_guard<std::mutex> lk(c->fmu);
    c->stop = true;
    c->py_busy = false;
    c->fcv.notify_all();
  }
  shutdown(c->sock, SHUT_RDWR);
  if (c->worker.joinable()) c->worker.join();
  {
    std::lock_guard<std::mutex> lk(c->lane->mu);
    auto& v = c->lane->conns;
    v.erase(std::remove(v.begin(), v.end(), c), v.end());
  }
  delete c;
  return FT_OK;
}

}  // extern "C"
