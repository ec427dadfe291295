// Function <-> daemon message channel over shared memory (the
// paper's fast local channel between a function process and the per-GPU
// daemon). Two single-producer/single-consumer rings of fixed-size slots in a
// memfd both processes map: ring 0 carries the client's requests, ring 1 the
// daemon's replies. A receiver spins on the producer's head counter for a
// bounded time (the reply to a request, or the next request of a steady
// function, arrives within tens of microseconds), then sleeps on it with a
// futex; a producer wakes it only if it announced that it sleeps. Blocking
// calls take a timeout so the Python side can check the peer for liveness
// (its AF_UNIX socket, which still carries SCM_RIGHTS descriptors).
#include <linux/futex.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <cstring>
#include <string>

#include "common.h"

namespace {

constexpr uint32_t kMagic = 0x46544348;  // "FTCH"

struct alignas(64) Word {
  std::atomic<uint32_t> v;
};

struct Ring {
  Word head;       // messages published (producer)
  Word tail;       // messages consumed (consumer)
  Word rsleep;     // consumer sleeps on head
  Word psleep;     // producer sleeps on tail (ring full)
};

struct Hdr {
  uint32_t magic, slot_bytes, slots, pad;
  Word closed;
  Ring ring[2];
};

inline int64_t now_us() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (int64_t)ts.tv_sec * 1000000 + ts.tv_nsec / 1000;
}

inline void cpu_relax() {
#if defined(__x86_64__)
  __builtin_ia32_pause();
#endif
}

inline void futex_wait(std::atomic<uint32_t>* w, uint32_t val, int64_t us) {
  timespec ts{(time_t)(us / 1000000), (long)(us % 1000000) * 1000};
  syscall(SYS_futex, reinterpret_cast<uint32_t*>(w), FUTEX_WAIT, val, &ts, nullptr, 0);
}

inline void futex_wake(std::atomic<uint32_t>* w) {
  syscall(SYS_futex, reinterpret_cast<uint32_t*>(w), FUTEX_WAKE, 0x7fffffff, nullptr, nullptr, 0);
}

// wait until pred() or the peer closed, spinning `spin_us` first, then sleeping on
// `word` (expected value from `cur()`) with `flag` raised; false on timeout
template <class Pred, class Cur>
int wait_on(Hdr* h, std::atomic<uint32_t>* word, std::atomic<uint32_t>* flag, Pred pred, Cur cur, int64_t spin_us,
            int64_t timeout_us) {
  if (pred()) return FT_OK;
  const int64_t t0 = now_us();
  const int64_t spin_end = t0 + spin_us;
  while (now_us() < spin_end) {
    for (int i = 0; i < 64; ++i) {
      if (pred()) return FT_OK;
      cpu_relax();
    }
    if (h->closed.v.load(std::memory_order_acquire)) return pred() ? FT_OK : FT_E_CLOSED;
  }
  for (;;) {
    if (h->closed.v.load(std::memory_order_acquire)) return pred() ? FT_OK : FT_E_CLOSED;
    const int64_t left = timeout_us < 0 ? 10000 : t0 + timeout_us - now_us();
    if (left <= 0) return pred() ? FT_OK : FT_E_TIMEOUT;
    const uint32_t seen = cur();
    flag->store(1, std::memory_order_seq_cst);
    if (pred()) {
      flag->store(0, std::memory_order_relaxed);
      return FT_OK;
    }
    futex_wait(word, seen, std::min<int64_t>(left, 10000));
    flag->store(0, std::memory_order_relaxed);
    if (pred()) return FT_OK;
  }
}

}  // namespace

struct ft_chan {
  Hdr* hdr = nullptr;
  uint8_t* data[2] = {nullptr, nullptr};
  size_t bytes = 0;
  // the geometry as this side mapped it: never re-read from the shared header,
  // which the peer can write (a daemon must not index its mapping by a client's word)
  uint32_t slot_bytes = 0, slots = 0;
  int fd = -1;  // the creator's memfd (closed by ft_chan_close)
};

extern "C" {

int ft_chan_create(uint32_t slot_bytes, uint32_t slots, int* memfd, ft_chan** out) {
  if (!memfd || !out || slot_bytes < 64 || slots < 2 || slot_bytes % 8) {
    ft::set_last_error("ft_chan_create: bad arguments");
    return FT_E_VALUE;
  }
  const size_t bytes = sizeof(Hdr) + 2 * (size_t)slot_bytes * slots;
  int fd = memfd_create("faastube-chan", MFD_CLOEXEC);
  if (fd < 0 || ftruncate(fd, (off_t)bytes) != 0) {
    ft::set_last_error(std::string("ft_chan_create: memfd: ") + strerror(errno));
    if (fd >= 0) close(fd);
    return FT_E_VALUE;
  }
  void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  if (m == MAP_FAILED) {
    ft::set_last_error(std::string("ft_chan_create: mmap: ") + strerror(errno));
    close(fd);
    return FT_E_VALUE;
  }
  auto* h = new (m) Hdr();
  h->slot_bytes = slot_bytes;
  h->slots = slots;
  h->closed.v.store(0);
  for (auto& r : h->ring) {
    r.head.v.store(0);
    r.tail.v.store(0);
    r.rsleep.v.store(0);
    r.psleep.v.store(0);
  }
  std::atomic_thread_fence(std::memory_order_release);
  h->magic = kMagic;
  auto* c = new ft_chan;
  c->hdr = h;
  c->bytes = bytes;
  c->slot_bytes = slot_bytes;
  c->slots = slots;
  c->fd = fd;
  c->data[0] = reinterpret_cast<uint8_t*>(m) + sizeof(Hdr);
  c->data[1] = c->data[0] + (size_t)slot_bytes * slots;
  *memfd = fd;
  *out = c;
  return FT_OK;
}

int ft_chan_attach(int memfd, ft_chan** out) {
  if (memfd < 0 || !out) {
    ft::set_last_error("ft_chan_attach: bad arguments");
    return FT_E_VALUE;
  }
  Hdr probe;
  struct stat sb;
  if (pread(memfd, &probe, sizeof probe, 0) != (ssize_t)sizeof probe || probe.magic != kMagic ||
      fstat(memfd, &sb) != 0) {
    ft::set_last_error("ft_chan_attach: not a channel");
    return FT_E_VALUE;
  }
  // the creator's geometry, checked against the file it really sized (a mapping past
  // the end of the memfd faults on first touch)
  if (probe.slot_bytes < 64 || probe.slot_bytes % 8 || probe.slot_bytes > (1u << 24) || probe.slots < 2 ||
      probe.slots > (1u << 16) ||
      sizeof(Hdr) + 2 * (size_t)probe.slot_bytes * probe.slots > (size_t)sb.st_size) {
    ft::set_last_error("ft_chan_attach: bad ring geometry");
    return FT_E_VALUE;
  }
  const size_t bytes = sizeof(Hdr) + 2 * (size_t)probe.slot_bytes * probe.slots;
  void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, memfd, 0);
  if (m == MAP_FAILED) {
    ft::set_last_error(std::string("ft_chan_attach: mmap: ") + strerror(errno));
    return FT_E_VALUE;
  }
  auto* c = new ft_chan;
  c->hdr = reinterpret_cast<Hdr*>(m);
  c->bytes = bytes;
  c->slot_bytes = probe.slot_bytes;
  c->slots = probe.slots;
  c->data[0] = reinterpret_cast<uint8_t*>(m) + sizeof(Hdr);
  c->data[1] = c->data[0] + (size_t)c->slot_bytes * c->slots;
  *out = c;
  return FT_OK;
}

int ft_chan_send(ft_chan* c, int dir, const void* buf, uint32_t n, int64_t timeout_us) {
  if (!c || (dir != 0 && dir != 1) || (n && !buf)) {
    ft::set_last_error("ft_chan_send: bad arguments");
    return FT_E_VALUE;
  }
  Hdr* h = c->hdr;
  const uint32_t slots = c->slots, slot_bytes = c->slot_bytes;
  if ((uint64_t)n + 8 > slot_bytes) {
    ft::set_last_error("ft_chan_send: message larger than a slot");
    return FT_E_VALUE;
  }
  Ring& r = h->ring[dir];
  const uint32_t head = r.head.v.load(std::memory_order_relaxed);
  int rc = wait_on(
      h, &r.tail.v, &r.psleep.v,
      [&] { return head - r.tail.v.load(std::memory_order_acquire) < slots; },
      [&] { return r.tail.v.load(std::memory_order_acquire); }, 50, timeout_us);
  if (rc != FT_OK) {
    ft::set_last_error(rc == FT_E_CLOSED ? "ft_chan_send: channel closed" : "ft_chan_send: ring full (timeout)");
    return rc;
  }
  uint8_t* slot = c->data[dir] + (size_t)(head % slots) * slot_bytes;
  std::memcpy(slot, &n, 4);
  if (n) std::memcpy(slot + 8, buf, n);
  r.head.v.store(head + 1, std::memory_order_seq_cst);
  if (r.rsleep.v.load(std::memory_order_seq_cst)) futex_wake(&r.head.v);
  return FT_OK;
}

int ft_chan_recv(ft_chan* c, int dir, void* buf, uint32_t cap, uint32_t* n, int64_t spin_us, int64_t timeout_us) {
  if (!c || (dir != 0 && dir != 1) || !n) {
    ft::set_last_error("ft_chan_recv: bad arguments");
    return FT_E_VALUE;
  }
  Hdr* h = c->hdr;
  Ring& r = h->ring[dir];
  const uint32_t tail = r.tail.v.load(std::memory_order_relaxed);
  int rc = wait_on(
      h, &r.head.v, &r.rsleep.v, [&] { return r.head.v.load(std::memory_order_acquire) != tail; },
      [&] { return r.head.v.load(std::memory_order_acquire); }, spin_us, timeout_us);
  if (rc != FT_OK) {
    ft::set_last_error(rc == FT_E_CLOSED ? "ft_chan_recv: channel closed" : "ft_chan_recv: timeout");
    return rc;
  }
  const uint8_t* slot = c->data[dir] + (size_t)(tail % c->slots) * c->slot_bytes;
  uint32_t len;
  std::memcpy(&len, slot, 4);
  if ((uint64_t)len + 8 > c->slot_bytes) {  // a length the peer could not have sent
    ft::set_last_error("ft_chan_recv: corrupt message length");
    return FT_E_VALUE;
  }
  *n = len;
  if (len > cap) {
    ft::set_last_error("ft_chan_recv: buffer too small");
    return FT_E_TRUNCATED;  // the message stays queued
  }
  if (len) std::memcpy(buf, slot + 8, len);
  r.tail.v.store(tail + 1, std::memory_order_seq_cst);
  if (r.psleep.v.load(std::memory_order_seq_cst)) futex_wake(&r.tail.v);
  return FT_OK;
}

// mark closed (both sides' waits return FT_E_CLOSED once drained), unmap
int ft_chan_close(ft_chan* c) {
  if (!c) return FT_OK;
  Hdr* h = c->hdr;
  h->closed.v.store(1, std::memory_order_seq_cst);
  for (auto& r : h->ring) {
    futex_wake(&r.head.v);
    futex_wake(&r.tail.v);
  }
  munmap(h, c->bytes);
  if (c->fd >= 0) close(c->fd);
  delete c;
  return FT_OK;
}

}  // extern "C"
