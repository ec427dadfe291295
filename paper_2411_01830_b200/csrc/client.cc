// The function-process side of the native lane (lane.cc): each hot request of
// Listing 1 through the daemon is one call here —
// the request/reply on the connection's shared-memory rings (chan.cc), the copy
// into / out of the mapped pool block on the caller's stream, and the ordering
// with the daemon through the connection's two sync words (stream write / wait
// value: a cross-process CUDA event dependency takes ~110 us to resolve on B200).
// A zero-copy view is a DLPack tensor whose deleter releases the block: it marks
// the legacy default stream (ordered after the caller's work on blocking streams)
// and sends the release from whatever thread frees the tensor — every send goes
// through the client's mutex, so the rings keep one producer at a time.
#include <cuda_runtime.h>
#include <poll.h>
#include <sys/socket.h>

#include <atomic>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.h"
#include "forward.h"

namespace {

// DLPack (dlpack.h v0.8 ABI)
struct DLDevice {
  int32_t device_type;  // kDLCUDA = 2
  int32_t device_id;
};
struct DLDataType {
  uint8_t code;  // kDLInt 0, kDLUInt 1, kDLFloat 2, kDLBfloat 4, kDLBool 6
  uint8_t bits;
  uint16_t lanes;
};
struct DLTensor {
  void* data;
  DLDevice device;
  int32_t ndim;
  DLDataType dtype;
  int64_t* shape;
  int64_t* strides;
  uint64_t byte_offset;
};
struct DLManagedTensor {
  DLTensor dl_tensor;
  void* manager_ctx;
  void (*deleter)(DLManagedTensor*);
};
const DLDataType kDl[10] = {{1, 8, 1}, {0, 8, 1}, {0, 16, 1}, {0, 32, 1}, {0, 64, 1},
                            {2, 16, 1}, {4, 16, 1}, {2, 32, 1}, {2, 64, 1}, {6, 8, 1}};

#pragma pack(push, 1)
struct DoneReq {
  uint8_t op, pad[3];
  int32_t ev;
  uint64_t token;
};
#pragma pack(pop)
constexpr uint8_t OP_DONE = 3;
constexpr size_t kRepHdr = 16, kEvOff = kRepHdr + 40;  // RepHdr, then BlockRep.ev

bool sock_gone(int sock) {  // the daemon's end of the connection socket closed
  pollfd p{sock, POLLIN, 0};
  if (poll(&p, 1, 0) <= 0) return false;
  if (p.revents & (POLLHUP | POLLERR | POLLNVAL)) return true;
  char b;
  return recv(sock, &b, 1, MSG_PEEK | MSG_DONTWAIT) == 0;
}

}  // namespace

struct ft_client {
  ft_chan* ch = nullptr;
  int sock = -1;          // the connection socket (liveness of the daemon; the caller owns it)
  bool dead = false;      // the daemon went away: sends fail at once
  bool abandoned = false;
  std::atomic<uint32_t> newest_d{0};  // the newest daemon mark a stream of ours waits for
  std::atomic<bool> any_d{false};
  uint32_t* c2d = nullptr;
  uint32_t* d2c = nullptr;
  int device = 0;
  std::mutex mu;
  uint32_t seq = 0;
  uint64_t sent = 0;
  int views = 0;          // live DLPack views (mu)
  bool closed = false;    // ft_client_destroy ran; the last view frees the client

  int mark(cudaStream_t st, int32_t* ev) {  // (mu held) our next sequence number after st's work
    uint32_t v = seq + 1;
    if (v == 0 || v == 0xFFFFFFFFu) v = 1;
    int rc = ft::mem_write32(st, c2d, v);
    if (rc != FT_OK) return rc;
    seq = v;
    *ev = (int32_t)v;
    return FT_OK;
  }
  int wait(cudaStream_t st, int32_t ev) {  // st waits for the daemon's mark `ev`
    if (ev == 0 || ev == -1) return FT_OK;
    uint32_t v = (uint32_t)ev, cur = newest_d.load(std::memory_order_relaxed);
    while ((!any_d.load(std::memory_order_relaxed) || (int32_t)(v - cur) > 0) &&
           !newest_d.compare_exchange_weak(cur, v, std::memory_order_relaxed)) {
    }
    any_d.store(true, std::memory_order_relaxed);
    return ft::mem_wait_geq32(st, d2c, v);
  }
  // the daemon went away: the marks our streams wait for may never be written. The
  // newest one waited for is written from here (a non-blocking stream: the waiting
  // streams are parked), so they drain instead of hanging every later synchronise
  // (the blocks they read stay mapped: the imports hold the memory)
  void abandon() {
    if (!any_d.load() || abandoned) return;
    abandoned = true;
    uint32_t v = newest_d.load();
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != device) cudaSetDevice(device);
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess) {
      cudaMemcpyAsync(d2c, &v, 4, cudaMemcpyHostToDevice, s);
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
    if (cur >= 0 && cur != device) cudaSetDevice(cur);
  }
  // (mu held) a full ring waits for the daemon to drain it while the daemon lives: a
  // daemon that died never will (release messages get no reply, so they can fill it)
  int send(const void* b, uint32_t n) {
    if (dead) {
      ft::set_last_error("ft_client: the daemon went away");
      return FT_E_CLOSED;
    }
    for (;;) {
      int rc = ft_chan_send(ch, 0, b, n, 200000);
      if (rc == FT_OK) ++sent;
      if (rc != FT_E_TIMEOUT) return rc;
      if (sock >= 0 && sock_gone(sock)) {
        dead = true;
        abandon();
        ft::set_last_error("ft_client: the daemon went away (request ring full)");
        return FT_E_CLOSED;
      }
    }
  }
  // (mu held) FT_E_TIMEOUT after 200 ms without a reply: the caller checks the daemon
  int recv(void* b, uint32_t cap, uint32_t* n, int64_t spin_us) {
    return ft_chan_recv(ch, 1, b, cap, n, spin_us, 200000);
  }
};

namespace {

struct View {
  DLManagedTensor m;
  std::vector<int64_t> shape;
  ft_client* cl;
  uint64_t token;
};

void release_client(ft_client* cl) {  // (mu not held)
  if (cl->ch) ft_chan_close(cl->ch);
  delete cl;
}

void view_deleter(DLManagedTensor* m) {
  View* v = static_cast<View*>(m->manager_ctx);
  ft_client* cl = v->cl;
  bool free_client = false;
  {
    std::lock_guard<std::mutex> lk(cl->mu);
    if (!cl->closed) {
      // the release, ordered after the caller's work on the legacy default stream
      // (which every blocking stream synchronises with)
      int dev = -1;
      cudaGetDevice(&dev);
      if (dev != cl->device) cudaSetDevice(cl->device);
      DoneReq q{OP_DONE, {0, 0, 0}, 0, v->token};
      if (cl->mark(cudaStreamLegacy, &q.ev) != FT_OK) q.ev = 0;
      cl->send(&q, sizeof q);
      if (dev >= 0 && dev != cl->device) cudaSetDevice(dev);
    }
    cl->views -= 1;
    free_client = cl->closed && cl->views == 0;
  }
  if (free_client) release_client(cl);
  delete v;
}

}  // namespace

extern "C" {

// the function process's lane client over an upgraded connection (takes over `ch`;
// `sock`, the connection's socket, stays the caller's and only tells it the daemon
// is alive — -1: never checked)
int ft_client_create(ft_chan* ch, int sock, void* c2d, void* d2c, int device, ft_client** out) {
  if (!ch || !c2d || !d2c || !out) return FT_E_VALUE;
  auto* cl = new ft_client;
  cl->ch = ch;
  cl->sock = sock;
  cl->c2d = static_cast<uint32_t*>(c2d);
  cl->d2c = static_cast<uint32_t*>(d2c);
  cl->device = device;
  *out = cl;
  return FT_OK;
}

// closes the rings (now, or when the last view is released)
int ft_client_destroy(ft_client* cl) {
  if (!cl) return FT_OK;
  bool now;
  {
    std::lock_guard<std::mutex> lk(cl->mu);
    cl->closed = true;
    now = cl->views == 0;
  }
  if (now) release_client(cl);
  return FT_OK;
}

// the caller found the daemon gone: sends fail from now on and our streams' waits
// on its marks are released
int ft_client_abandon(ft_client* cl) {
  if (!cl) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(cl->mu);
  cl->dead = true;
  cl->abandon();
  return FT_OK;
}

int ft_client_views(ft_client* cl, int* out) {
  if (!cl || !out) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(cl->mu);
  *out = cl->views;
  return FT_OK;
}

int ft_client_sent(ft_client* cl, uint64_t* out) {
  if (!cl || !out) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(cl->mu);
  *out = cl->sent;
  return FT_OK;
}

int ft_client_send(ft_client* cl, const void* msg, uint32_t n) {
  if (!cl) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(cl->mu);
  return cl->send(msg, n);
}

// one request and its reply (FT_E_TIMEOUT after 200 ms without one: the caller
// checks the daemon and calls ft_client_recv again)
int ft_client_call(ft_client* cl, const void* req, uint32_t n, void* rep, uint32_t cap, uint32_t* rep_len,
                   int64_t spin_us) {
  if (!cl || !rep_len) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(cl->mu);
  int rc = cl->send(req, n);
  if (rc != FT_OK) return rc;
  return cl->recv(rep, cap, rep_len, spin_us);
}

int ft_client_recv(ft_client* cl, void* rep, uint32_t cap, uint32_t* rep_len, int64_t spin_us) {
  if (!cl || !rep_len) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(cl->mu);
  return cl->recv(rep, cap, rep_len, spin_us);
}

// our mark on `stream` (Python's slow paths send it in a msgpack message)
int ft_client_mark(ft_client* cl, void* stream, int32_t* ev) {
  if (!cl || !ev) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(cl->mu);
  return cl->mark((cudaStream_t)stream, ev);
}

// `stream` waits for the daemon's mark `ev`
int ft_client_wait(ft_client* cl, void* stream, int32_t ev) {
  if (!cl) return FT_E_VALUE;
  return cl->wait((cudaStream_t)stream, ev);
}

// store into a lent block in one call: `stream` waits for the loan's mark, copies the
// output into the block, marks; the commit request (its ev field at byte 4 is filled
// in here) goes out and its reply comes back into `rep`
int ft_client_store(ft_client* cl, void* stream, int32_t wait_ev, void* dst, const void* src, uint64_t n, int engine,
                    const void* req_in, uint32_t req_len, void* rep, uint32_t cap, uint32_t* rep_len,
                    int64_t spin_us) {
  uint8_t req[1024];
  if (!cl || !req_in || req_len < 8 || req_len > sizeof req || !rep_len) return FT_E_VALUE;
  memcpy(req, req_in, req_len);
  cudaStream_t st = (cudaStream_t)stream;
  int rc = cl->wait(st, wait_ev);
  if (rc == FT_OK && n) rc = ft_copy_ex(dst, src, n, cl->device, stream, engine, 0);
  if (rc != FT_OK) return rc;
  std::lock_guard<std::mutex> lk(cl->mu);
  int32_t ev = 0;
  rc = cl->mark(st, &ev);
  if (rc != FT_OK) return rc;
  memcpy(req + 4, &ev, 4);
  rc = cl->send(req, req_len);
  if (rc != FT_OK) return rc;
  return cl->recv(rep, cap, rep_len, spin_us);
}

// a fetch request and its reply; `stream` waits for the reply's mark (a block reply)
int ft_client_fetch(ft_client* cl, void* stream, const void* req, uint32_t req_len, void* rep, uint32_t cap,
                    uint32_t* rep_len, int64_t spin_us) {
  if (!cl || !rep_len) return FT_E_VALUE;
  int rc;
  {
    std::lock_guard<std::mutex> lk(cl->mu);
    rc = cl->send(req, req_len);
    if (rc == FT_OK) rc = cl->recv(rep, cap, rep_len, spin_us);
  }
  if (rc != FT_OK) return rc;
  const uint8_t* r = static_cast<const uint8_t*>(rep);
  if (*rep_len >= kEvOff + 4 && r[1] /* ok */) {
    int32_t ev;
    memcpy(&ev, r + kEvOff, 4);
    rc = cl->wait((cudaStream_t)stream, ev);
  }
  return rc;
}

// copy a fetched block into the caller's buffer on `stream`, then release it (done)
int ft_client_copy_done(ft_client* cl, void* stream, void* dst, const void* src, uint64_t n, int engine,
                        uint64_t token) {
  if (!cl) return FT_E_VALUE;
  int rc = n ? ft_copy_ex(dst, src, n, cl->device, stream, engine, 0) : FT_OK;
  if (rc != FT_OK) return rc;
  std::lock_guard<std::mutex> lk(cl->mu);
  DoneReq q{OP_DONE, {0, 0, 0}, 0, token};
  rc = cl->mark((cudaStream_t)stream, &q.ev);
  if (rc != FT_OK) return rc;
  return cl->send(&q, sizeof q);
}

// release a block after `stream`'s work (ev 0: no ordering needed)
int ft_client_done(ft_client* cl, void* stream, uint64_t token, int ordered) {
  if (!cl) return FT_E_VALUE;
  std::lock_guard<std::mutex> lk(cl->mu);
  DoneReq q{OP_DONE, {0, 0, 0}, 0, token};
  if (ordered) {
    int rc = cl->mark((cudaStream_t)stream, &q.ev);
    if (rc != FT_OK) return rc;
  }
  return cl->send(&q, sizeof q);
}

// a zero-copy view of a fetched block as a DLPack tensor (dtype code as the lane's);
// freeing the tensor releases the block (done, ordered on the legacy default stream)
int ft_client_view(ft_client* cl, void* ptr, int dtype, int ndim, const int64_t* shape, uint64_t token,
                   void** dlmanaged) {
  if (!cl || !dlmanaged || dtype < 0 || dtype >= 10 || ndim < 0 || ndim > 8) return FT_E_VALUE;
  auto* v = new View;
  v->shape.assign(shape, shape + ndim);
  v->cl = cl;
  v->token = token;
  DLTensor& t = v->m.dl_tensor;
  t.data = ptr;
  t.device = {2, cl->device};
  t.ndim = ndim;
  t.dtype = kDl[dtype];
  t.shape = v->shape.data();
  t.strides = nullptr;
  t.byte_offset = 0;
  v->m.manager_ctx = v;
  v->m.deleter = view_deleter;
  {
    std::lock_guard<std::mutex> lk(cl->mu);
    cl->views += 1;
  }
  *dlmanaged = &v->m;
  return FT_OK;
}

}  // extern "C"
