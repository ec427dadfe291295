// Device side of libfaastube (sm_100a): elastic VMM pool, SM-driven copy
// kernels (TMA bulk + vector engines), fused integrity digest, PCIe legs on
// the copy engines, and the striped host->gFunc pass with NVLink forwarding.
//
// Design notes: the probes in profiles/r01 showed that on
// B200 the copy engine is the fastest PCIe mover (55.6 GB/s H2D vs 51.5 GB/s
// for any SM-initiated read shape), while for HBM- and NVLink-side copies an
// SM-driven TMA bulk pipeline matches or beats the copy engine (6.48 TB/s
// read+write vs 6.40). So PCIe legs run on the CE, everything after the PCIe
// hop runs in our kernels.
#include <cuda.h>
#include <chrono>
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/faastube.h"
#include "forward.h"

namespace ft {
void set_last_error(const std::string& msg);
}

namespace {

int cuda_fail(cudaError_t e, const char* what) {
  ft::set_last_error(std::string(what) + ": " + cudaGetErrorString(e));
  return FT_E_CUDA;
}
#define CU_RT(x)                                  \
  do {                                            \
    cudaError_t e_ = (x);                         \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x); \
  } while (0)

// ------------------------------------------------------------ driver API
// Resolved through the runtime so libfaastube.so loads on machines without
// a driver (build container) and never links libcuda directly.
struct Drv {
  bool ok = false;
  decltype(&cuMemCreate) create;
  decltype(&cuMemRelease) release;
  decltype(&cuMemAddressReserve) reserve;
  decltype(&cuMemAddressFree) addr_free;
  decltype(&cuMemMap) map;
  decltype(&cuMemUnmap) unmap;
  decltype(&cuMemSetAccess) set_access;
  decltype(&cuMemExportToShareableHandle) export_handle;
  decltype(&cuMemImportFromShareableHandle) import_handle;
  decltype(&cuMemGetAllocationGranularity) granularity;
  decltype(&cuGetErrorString) err;
  decltype(&cuStreamWaitValue32) wait32;
  decltype(&cuStreamWriteValue32) write32;
};
Drv g_drv;
std::once_flag g_drv_once;
template <class F>
bool sym(const char* name, F* out) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return false;
  *out = reinterpret_cast<F>(p);
  return true;
}
Drv* drv() {
  std::call_once(g_drv_once, [] {
    Drv& d = g_drv;
    d.ok = sym("cuMemCreate", &d.create) && sym("cuMemRelease", &d.release) &&
           sym("cuMemAddressReserve", &d.reserve) && sym("cuMemAddressFree", &d.addr_free) &&
           sym("cuMemMap", &d.map) && sym("cuMemUnmap", &d.unmap) && sym("cuMemSetAccess", &d.set_access) &&
           sym("cuMemExportToShareableHandle", &d.export_handle) &&
           sym("cuMemImportFromShareableHandle", &d.import_handle) &&
           sym("cuMemGetAllocationGranularity", &d.granularity) && sym("cuGetErrorString", &d.err) &&
           sym("cuStreamWaitValue32", &d.wait32) && sym("cuStreamWriteValue32", &d.write32);
  });
  return g_drv.ok ? &g_drv : nullptr;
}
int cu_fail(CUresult r, const char* what) {
  const char* s = "unknown";
  if (g_drv.err) g_drv.err(r, &s);
  ft::set_last_error(std::string(what) + ": " + s);
  return r == CUDA_ERROR_OUT_OF_MEMORY ? FT_E_OOM : FT_E_CUDA;
}
#define CU_DRV(x)                              \
  do {                                         \
    CUresult r_ = (x);                         \
    if (r_ != CUDA_SUCCESS) return cu_fail(r_, #x); \
  } while (0)

CUmemAllocationProp block_prop(int device) {
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

// Grant read/write to `device` and every GPU that can reach it peer-to-peer.
int grant_access(Drv* d, CUdeviceptr va, size_t bytes, int owner, bool all_peers) {
  int n = 0;
  CU_RT(cudaGetDeviceCount(&n));
  std::vector<CUmemAccessDesc> acc;
  for (int g = 0; g < n; ++g) {
    int ok = g == owner;
    if (!ok && all_peers) cudaDeviceCanAccessPeer(&ok, g, owner);
    if (!ok) continue;
    CUmemAccessDesc a = {};
    a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a.location.id = g;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    acc.push_back(a);
  }
  CU_DRV(d->set_access(va, bytes, acc.data(), acc.size()));
  return FT_OK;
}

// ------------------------------------------------------------ kernels
constexpr int kBulkThreads = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{ .reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W%=; }" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem), "r"(smem_u32(smem)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// L2 cache-policy variants (createpolicy + .L2::cache_hint): used to keep a
// freshly stored pool block resident for the consumer's fetch that follows.
__device__ __forceinline__ uint64_t l2_policy(uint32_t kind) {
  uint64_t p;
  if (kind == 1)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else if (kind == 2)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* gmem, const void* smem, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gmem),
               "r"(smem_u32(smem)), "r"(bytes), "l"(pol)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

// K1/K3 TMA-bulk engine. One elected thread per CTA runs a STAGES-deep
// global->smem->global ring; tiles are dealt round-robin over a persistent
// grid. Requires 16-byte aligned src/dst and a multiple-of-16 byte count
// (the host wrapper peels the unaligned head/tail to the vector engine).
template <int STAGES, bool HINT>
__global__ void __launch_bounds__(kBulkThreads) k_copy_bulk(uint8_t* __restrict__ dst,
                                                            const uint8_t* __restrict__ src, uint64_t bytes,
                                                            uint32_t tile, uint32_t hints) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint64_t psrc = 0, pdst = 0;
  if (HINT) {
    psrc = l2_policy(hints & 3);
    pdst = l2_policy((hints >> 2) & 3);
  }
  auto load = [&](void* sm, const void* g, uint32_t n, uint64_t* bar) {
    if (HINT) bulk_g2s_hint(sm, g, n, bar, psrc);
    else bulk_g2s(sm, g, n, bar);
  };
  auto store = [&](void* g, const void* sm, uint32_t n) {
    if (HINT) bulk_s2g_hint(g, sm, n, pdst);
    else bulk_s2g(g, sm, n);
  };
  const uint64_t ntiles = (bytes + tile - 1) / tile;
  auto tile_len = [&](uint64_t t) -> uint32_t {
    uint64_t off = t * tile;
    return (uint32_t)((bytes - off) < tile ? (bytes - off) : tile);
  };
  uint64_t next = blockIdx.x;  // next tile to load
  for (int s = 0; s < STAGES && next < ntiles; ++s, next += gridDim.x) {
    uint32_t len = tile_len(next);
    mbar_expect_tx(&full[s], len);
    load(smem + (size_t)s * tile, src + next * tile, len, &full[s]);
  }
  uint32_t phase = 0;
  int s = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(&full[s], phase);
    store(dst + t * tile, smem + (size_t)s * tile, tile_len(t));
    if (t != blockIdx.x && next < ntiles) {
      // refill the PREVIOUS slot: its store was issued one tile ago, so waiting
      // for all but the newest store group to finish reading smem rarely
      // stalls, and the store just issued keeps streaming meanwhile.
      const int ps = s == 0 ? STAGES - 1 : s - 1;
      bulk_wait_read<1>();
      uint32_t len = tile_len(next);
      mbar_expect_tx(&full[ps], len);
      load(smem + (size_t)ps * tile, src + next * tile, len, &full[ps]);
      next += gridDim.x;
    }
    if (++s == STAGES) {
      s = 0;
      phase ^= 1;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Vector engine (also the peer-safe engine): 16-byte loads/stores, UNROLL
// independent requests in flight per thread, grid-stride. `bytes` multiple
// of 16 and both pointers 16-byte aligned.
// STREAM: .cs (evict-first) loads/stores for large copies that must not displace
// the L2; small copies use plain ones (0.3-0.6 us less per 1 MiB launch on B200,
// profiles/r02/probe_small.txt)
template <int UNROLL, bool STREAM = true>
__global__ void __launch_bounds__(512) k_copy_vec(int4* __restrict__ dst, const int4* __restrict__ src,
                                                  uint64_t n16) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (UNROLL - 1) * stride < n16; i += UNROLL * stride) {
    int4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) v[u] = STREAM ? __ldcs(src + i + u * stride) : src[i + u * stride];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (STREAM)
        __stcs(dst + i + u * stride, v[u]);
      else
        dst[i + u * stride] = v[u];
    }
  }
  for (; i < n16; i += stride) {
    if (STREAM)
      __stcs(dst + i, __ldcs(src + i));
    else
      dst[i] = src[i];
  }
}

// Many segments in one launch (batched small-message passing): the launch is
// paid once for the whole batch. Segments are cut into 32 KiB tiles dealt
// over the grid; a CTA copies a tile with 128-bit loads/stores (4 in flight per
// thread) when both ends are 16-byte aligned, bytewise otherwise and for tails.
// Peer (NVLink) pointers work like local ones.
constexpr int kMultiMax = 64;
constexpr uint32_t kMultiTile = 32768;
struct MultiArgs {
  uint8_t* dst[kMultiMax];
  const uint8_t* src[kMultiMax];
  uint64_t bytes[kMultiMax];
  uint64_t first_tile[kMultiMax + 1];  // prefix sum of tiles per segment
  int n;
};
__global__ void __launch_bounds__(512) k_copy_multi(const __grid_constant__ MultiArgs a) {
  const uint64_t tiles = a.first_tile[a.n];
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    int s = 0;
    while (a.first_tile[s + 1] <= t) ++s;  // <= 64 segments: a short scan
    const uint64_t off = (t - a.first_tile[s]) * kMultiTile;
    const uint64_t len = min((uint64_t)kMultiTile, a.bytes[s] - off);
    uint8_t* d = a.dst[s] + off;
    const uint8_t* x = a.src[s] + off;
    if ((((uintptr_t)d | (uintptr_t)x) & 15) == 0) {
      const uint64_t n16 = len / 16;
      int4* d4 = reinterpret_cast<int4*>(d);
      const int4* x4 = reinterpret_cast<const int4*>(x);
      for (uint64_t i = threadIdx.x; i < n16; i += blockDim.x * 4) {
        int4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * blockDim.x < n16) v[u] = __ldcs(x4 + i + u * blockDim.x);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * blockDim.x < n16) __stcs(d4 + i + u * blockDim.x, v[u]);
      }
      for (uint64_t i = n16 * 16 + threadIdx.x; i < len; i += blockDim.x) d[i] = x[i];
    } else {
      for (uint64_t i = threadIdx.x; i < len; i += blockDim.x) d[i] = x[i];
    }
  }
}

__global__ void k_copy_bytes(uint8_t* dst, const uint8_t* src, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// Digest: words w_i (8 bytes little-endian, tail zero-padded) mixed with
// their index; accumulators are u64 sum and xor (order independent, so any
// grid shape gives the same value). Identical to ft_fingerprint_host.
__host__ __device__ __forceinline__ uint64_t fp_mix(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}
__host__ __device__ __forceinline__ uint64_t fp_word(uint64_t w, uint64_t i) {
  return fp_mix(w ^ (i * 0x9e3779b97f4a7c15ull + 0x632be59bd9b4e019ull));
}
__global__ void __launch_bounds__(512) k_fingerprint(const uint8_t* __restrict__ src, uint64_t bytes,
                                                     unsigned long long* out) {
  const uint64_t nw = bytes / 8;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t s = 0, x = 0;
  const uint64_t* w = reinterpret_cast<const uint64_t*>(src);
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    // 16-byte loads, 4 in flight per thread: the digest is bound by bytes in flight,
    // not by the mixing (order independent, so any traversal gives the same value)
    const ulonglong2* w2 = reinterpret_cast<const ulonglong2*>(src);
    const uint64_t n2 = nw / 2;
    for (; i + 3 * stride < n2; i += 4 * stride) {
      ulonglong2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(w2 + i + u * stride);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint64_t j = 2 * (i + u * stride);
        uint64_t h0 = fp_word(v[u].x, j), h1 = fp_word(v[u].y, j + 1);
        s += h0 + h1;
        x ^= h0 ^ h1;
      }
    }
    for (; i < n2; i += stride) {
      ulonglong2 v = __ldcs(w2 + i);
      uint64_t h0 = fp_word(v.x, 2 * i), h1 = fp_word(v.y, 2 * i + 1);
      s += h0 + h1;
      x ^= h0 ^ h1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (nw & 1)) {  // odd trailing word
      uint64_t h = fp_word(__ldcs(w + nw - 1), nw - 1);
      s += h;
      x ^= h;
    }
  } else if ((reinterpret_cast<uintptr_t>(src) & 7) == 0) {
    for (; i < nw; i += stride) {
      uint64_t h = fp_word(__ldcs(w + i), i);
      s += h;
      x ^= h;
    }
  } else {  // unaligned source: assemble each little-endian word from bytes
    for (; i < nw; i += stride) {
      uint64_t t = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) t |= (uint64_t)src[i * 8 + k] << (8 * k);
      uint64_t h = fp_word(t, i);
      s += h;
      x ^= h;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (bytes & 7)) {
    uint64_t t = 0;
    for (uint64_t k = 0; k < (bytes & 7); ++k) t |= (uint64_t)src[nw * 8 + k] << (8 * k);
    uint64_t h = fp_word(t, nw);
    s += h;
    x ^= h;
  }
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    x ^= __shfl_xor_sync(0xffffffffu, x, o);
  }
  __shared__ uint64_t ws[16], wx[16];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    ws[wid] = s;
    wx[wid] = x;
  }
  __syncthreads();
  if (wid == 0) {
    int nwarp = blockDim.x / 32;
    s = lane < nwarp ? ws[lane] : 0;
    x = lane < nwarp ? wx[lane] : 0;
    for (int o = 16; o; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      x ^= __shfl_xor_sync(0xffffffffu, x, o);
    }
    if (lane == 0) {
      atomicAdd(&out[0], (unsigned long long)s);
      atomicXor(&out[1], (unsigned long long)x);
    }
  }
}

// Stream-ordered doorbells over (peer-)mapped memory: a producer publishes
// "payload k is in place" by a system-scope release store after its copy
// kernel; a consumer's stream parks on an acquire-load spin until the value
// is reached, then pulls the payload over NVLink — no host round trip.
__global__ void k_signal(unsigned int* flag, unsigned int value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}
// Bounded doorbell wait: a peer that never rings (crashed process, mismatched
// setup) must not park the stream forever — after timeout_ns the wait gives up
// and, when err is given, records the value it was waiting for there.
__global__ void k_wait(const unsigned int* flag, unsigned int value, uint64_t timeout_ns, unsigned int* err) {
  unsigned int v;
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int)(v - value) >= 0) return;
    __nanosleep(200);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < timeout_ns);
  if (err) *err = value ? value : 1u;
}

// Fixed-duration GPU occupancy (the runtime's synthetic gFunc compute,
// harness compute_latency_ms): spins on the global nanosecond timer, so the
// duration does not depend on the SM clock (an idle-clocked GPU runs a
// cycle-count sleep many times longer than asked).
__global__ void k_spin_ns(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

// K2 forward: chunks of a staging ring -> destination (over NVLink when the
// destination is a peer's memory). See forward.h for the protocol. Every CTA
// walks the batch's chunks in order: thread 0 polls the slot's landed word
// (acquire, bounded), the CTA pulls its tiles of the chunk with 16-byte loads
// (4 in flight per thread), then thread 0 counts the CTA's share read
// (release add on the slot's freed word: the CE may overwrite it once all
// kFwdCtas CTAs have counted).
__global__ void __launch_bounds__(256) k_forward(uint8_t* __restrict__ dst, const uint8_t* __restrict__ ring,
                                                 uint64_t slot_bytes, const uint32_t* landed, uint32_t* freed,
                                                 uint32_t* err, const __grid_constant__ ft::FwdBatch b) {
  constexpr uint64_t kTile = 256 * 4 * 16;  // bytes per CTA step
  __shared__ int ok;
  for (int c = 0; c < b.n; ++c) {
    const ft::FwdChunk ch = b.c[c];
    if (threadIdx.x == 0) {
      uint32_t v;
      uint64_t t0, t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      int good = 1;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(landed + ch.slot) : "memory");
        if ((int32_t)(v - ch.gen) >= 0) break;
        __nanosleep(64);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 60000000000ull) {  // 60 s: the DMA never landed; report, do not hang
          good = 0;
          if (err) atomicExch(err, 1u);
          break;
        }
      }
      ok = good;
    }
    __syncthreads();
    const uint8_t* src = ring + (uint64_t)ch.slot * slot_bytes;
    uint8_t* d = dst + ch.dst_off;
    if (ok && (reinterpret_cast<uintptr_t>(d) & 15)) {  // misaligned destination: bytewise
      for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ch.len;
           i += (uint64_t)gridDim.x * blockDim.x)
        d[i] = src[i];
    } else if (ok) {
      const uint64_t n16 = ch.len / 16;
      const int4* s4 = reinterpret_cast<const int4*>(src);
      int4* d4 = reinterpret_cast<int4*>(d);
      for (uint64_t base = (uint64_t)blockIdx.x * (kTile / 16); base < n16; base += (uint64_t)gridDim.x * (kTile / 16)) {
        int4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint64_t i = base + threadIdx.x + u * 256;
          if (i < n16) v[u] = __ldcg(s4 + i);  // L2 only: a reused slot never hits a stale L1 line
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint64_t i = base + threadIdx.x + u * 256;
          if (i < n16) __stcs(d4 + i, v[u]);
        }
      }
      if (blockIdx.x == 0)
        for (uint64_t i = n16 * 16 + threadIdx.x; i < ch.len; i += blockDim.x) d[i] = src[i];
    }
    __syncthreads();  // every load of this CTA's share has returned (its values were stored)
    if (threadIdx.x == 0) {
      __threadfence();
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(freed + ch.slot) : "memory");
    }
  }
}

// ------------------------------------------------------------ launch config
struct DevInfo {
  int sms = 0;
  bool init = false;
};
std::mutex g_dev_mu;
DevInfo g_dev[64];
int dev_sms(int device) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (!g_dev[device].init) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    g_dev[device].sms = v > 0 ? v : 148;
    g_dev[device].init = true;
  }
  return g_dev[device].sms;
}
// Bulk-engine shape: STAGES x tile bytes of smem per CTA, ctas_per_sm CTAs
// resident per SM. Defaults from the sweep in profiles/r01 (override with
// FT_BULK_STAGES / FT_BULK_TILE / FT_BULK_CTAS_PER_SM for tuning runs).
struct BulkCfg {
  int stages = 2;
  uint32_t tile = 16384;
  int ctas_per_sm = 3;
};
BulkCfg bulk_cfg() {
  static BulkCfg c = [] {
    BulkCfg b;
    if (const char* e = getenv("FT_BULK_STAGES")) b.stages = atoi(e);
    if (const char* e = getenv("FT_BULK_TILE")) b.tile = (uint32_t)atoi(e);
    if (const char* e = getenv("FT_BULK_CTAS_PER_SM")) b.ctas_per_sm = atoi(e);
    if (b.stages != 2 && b.stages != 3 && b.stages != 4 && b.stages != 6) b.stages = 2;
    if (b.tile < 1024 || b.tile % 16 || (size_t)b.tile * b.stages > 200 * 1024) b.tile = 16384;
    if (b.ctas_per_sm < 1) b.ctas_per_sm = 1;
    return b;
  }();
  return c;
}
template <int S, bool H>
int launch_bulk_s(uint8_t* dst, const uint8_t* src, uint64_t bytes, int device, cudaStream_t st, int grid,
                  uint32_t tile, int per_sm, uint32_t hints) {
  size_t smem = (size_t)S * tile;
  CU_RT(cudaFuncSetAttribute(k_copy_bulk<S, H>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  uint64_t tiles = (bytes + tile - 1) / tile;
  if (grid <= 0) grid = per_sm * dev_sms(device);
  if ((uint64_t)grid > tiles) grid = (int)tiles;
  k_copy_bulk<S, H><<<grid, kBulkThreads, smem, st>>>(dst, src, bytes, tile, hints);
  CU_RT(cudaGetLastError());
  return FT_OK;
}
template <int S>
int launch_bulk_h(uint8_t* dst, const uint8_t* src, uint64_t bytes, int device, cudaStream_t st, int grid,
                  uint32_t tile, int per_sm, uint32_t hints) {
  return hints ? launch_bulk_s<S, true>(dst, src, bytes, device, st, grid, tile, per_sm, hints)
               : launch_bulk_s<S, false>(dst, src, bytes, device, st, grid, tile, per_sm, 0);
}
int launch_bulk(uint8_t* dst, const uint8_t* src, uint64_t bytes, int device, cudaStream_t st, int grid,
                uint32_t hints) {
  BulkCfg c = bulk_cfg();
  switch (c.stages) {
    case 3: return launch_bulk_h<3>(dst, src, bytes, device, st, grid, c.tile, c.ctas_per_sm, hints);
    case 4: return launch_bulk_h<4>(dst, src, bytes, device, st, grid, c.tile, c.ctas_per_sm, hints);
    case 6: return launch_bulk_h<6>(dst, src, bytes, device, st, grid, c.tile, c.ctas_per_sm, hints);
    default: return launch_bulk_h<2>(dst, src, bytes, device, st, grid, c.tile, c.ctas_per_sm, hints);
  }
}
// Small copies (<= kVecWide): the whole payload in flight at once — 2 x 16 B per
// thread, 256-thread CTAs, one CTA per 8 KiB (1 MiB -> 128 CTAs). A peer pull is
// latency-bound at these sizes (900 GB/s x ~1.5 us of NVLink round trip is ~1.3 MB
// in flight), so every load must be issued in the first wave; the grid-stride
// shape below (4 x 16 B per thread, 2 CTAs/SM of 512) would put only 32 CTAs on
// a 1 MiB copy. Larger copies: persistent grid-stride.
constexpr uint64_t kVecWide = 4ull << 20;
int launch_vec(uint8_t* dst, const uint8_t* src, uint64_t bytes, int device, cudaStream_t st, int grid) {
  uint64_t n16 = bytes / 16;
  if (grid <= 0 && bytes <= kVecWide) {
    uint64_t ctas = (n16 + 256 * 2 - 1) / (256 * 2);
    k_copy_vec<2, false><<<(int)(ctas ? ctas : 1), 256, 0, st>>>(reinterpret_cast<int4*>(dst),
                                                                 reinterpret_cast<const int4*>(src), n16);
    CU_RT(cudaGetLastError());
    return FT_OK;
  }
  if (grid <= 0) grid = 2 * dev_sms(device);
  uint64_t need = (n16 + 512 * 4 - 1) / (512 * 4);
  if (need < (uint64_t)grid) grid = (int)(need ? need : 1);
  k_copy_vec<4><<<grid, 512, 0, st>>>(reinterpret_cast<int4*>(dst), reinterpret_cast<const int4*>(src), n16);
  CU_RT(cudaGetLastError());
  return FT_OK;
}

int copy_impl(void* dst_, const void* src_, uint64_t bytes, int device, cudaStream_t st, int engine, int grid,
              uint32_t hints = 0) {
  if (bytes == 0) return FT_OK;
  if (!dst_ || !src_) {
    ft::set_last_error("ft_copy: null pointer");
    return FT_E_VALUE;
  }
  int cur = -1;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  uint8_t* dst = static_cast<uint8_t*>(dst_);
  const uint8_t* src = static_cast<const uint8_t*>(src_);
  int rc = FT_OK;
  // Peel so the body is 16-byte aligned on both sides (only possible when the
  // two pointers share alignment mod 16; otherwise fall back to bytes).
  uintptr_t ms = (uintptr_t)src & 15, md = (uintptr_t)dst & 15;
  if (ms != md) {
    k_copy_bytes<<<2 * dev_sms(device), 256, 0, st>>>(dst, src, bytes);
    cudaError_t e = cudaGetLastError();
    if (cur != device) cudaSetDevice(cur);
    return e == cudaSuccess ? FT_OK : cuda_fail(e, "k_copy_bytes");
  }
  uint64_t head = ms ? (16 - ms) : 0;
  if (head > bytes) head = bytes;
  uint64_t body = (bytes - head) & ~(uint64_t)15;
  uint64_t tail = bytes - head - body;
  if (head) k_copy_bytes<<<1, 32, 0, st>>>(dst, src, head);
  if (body) {
    if (engine == 0) engine = 1;
    rc = engine == 1 ? launch_bulk(dst + head, src + head, body, device, st, grid, hints)
                     : launch_vec(dst + head, src + head, body, device, st, grid);
  }
  if (rc == FT_OK && tail) k_copy_bytes<<<1, 32, 0, st>>>(dst + head + body, src + head + body, tail);
  cudaError_t e = cudaGetLastError();
  if (cur != device) cudaSetDevice(cur);
  if (rc) return rc;
  return e == cudaSuccess ? FT_OK : cuda_fail(e, "ft_copy");
}

// event pool for the one-shot striped copy (ft_h2g_striped)
std::mutex g_evp_mu;
std::map<int, std::vector<cudaEvent_t>> g_evp;
std::vector<cudaEvent_t> take_events(int device, int n) {
  std::vector<cudaEvent_t> out;
  {
    std::lock_guard<std::mutex> lk(g_evp_mu);
    auto& v = g_evp[device];
    while ((int)out.size() < n && !v.empty()) {
      out.push_back(v.back());
      v.pop_back();
    }
  }
  while ((int)out.size() < n) {  // current device is `device` (the caller set it)
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) break;
    out.push_back(e);
  }
  return out;
}
void put_events(int device, const std::vector<cudaEvent_t>& evs) {
  std::lock_guard<std::mutex> lk(g_evp_mu);
  auto& v = g_evp[device];
  v.insert(v.end(), evs.begin(), evs.end());
}

// ------------------------------------------------------------ VMM pool
// A pool block is a range of an arena: one physical allocation (cuMemCreate),
// mapped once into the pool's VA range with every peer's access. Blocks are
// carved out of arenas and given back to them without any driver call; only a
// new arena maps memory (and only an idle trim unmaps). cuMemMap / cuMemUnmap
// wait for the GPU's running kernels and stall every CUDA call of the process
// meanwhile (0.3-1 s under load, profiles/r01/diag_vmm_map_unmap.txt), so they
// must not happen per block on the request path.
struct Arena {
  CUmemGenericAllocationHandle h;
  CUdeviceptr va;
  size_t bytes;
  size_t used = 0;
  bool keep = false;                 // reserved up front: never trimmed
  std::map<size_t, size_t> free;     // offset -> length (coalesced)
};
struct Block {
  uint64_t arena;
  size_t off;
  size_t bytes;
};
struct Import {
  CUmemGenericAllocationHandle h;
  CUdeviceptr va;
  size_t bytes;
};
std::mutex g_imp_mu;
std::map<uint64_t, Import> g_imports;
std::atomic<uint64_t> g_imp_next{1};

// VA ranges of the pools (reserved per GPU): a pointer inside one is device memory
// of that GPU, so ft_copy picks its engine without cudaPointerGetAttributes (two
// driver queries, ~1 us each) for pool blocks — the request path's usual operands.
struct VaRange {
  uintptr_t lo, hi;
  int device;
};
std::mutex g_va_mu;
std::vector<VaRange> g_va;
std::atomic<int> g_va_n{0};
int va_device(const void* p) {
  if (!g_va_n.load(std::memory_order_acquire)) return -1;
  uintptr_t a = (uintptr_t)p;
  std::lock_guard<std::mutex> lk(g_va_mu);
  for (const VaRange& r : g_va)
    if (a >= r.lo && a < r.hi) return r.device;
  return -1;
}
void va_add(uintptr_t lo, size_t n, int device) {
  std::lock_guard<std::mutex> lk(g_va_mu);
  g_va.push_back({lo, lo + n, device});
  g_va_n.store((int)g_va.size(), std::memory_order_release);
}
void va_remove(uintptr_t lo) {
  std::lock_guard<std::mutex> lk(g_va_mu);
  g_va.erase(std::remove_if(g_va.begin(), g_va.end(), [&](const VaRange& r) { return r.lo == lo; }), g_va.end());
  g_va_n.store((int)g_va.size(), std::memory_order_release);
}

}  // namespace

struct ft_vmm_pool {
  int device;
  size_t gran;
  CUdeviceptr base;
  size_t va_bytes;
  std::map<size_t, size_t> free_va;  // offset -> length (arena VA ranges)
  std::map<uint64_t, Arena> arenas;
  std::map<uint64_t, Block> blocks;
  uint64_t next_id = 1, next_arena = 1;
  size_t mapped = 0;
  size_t arena_bytes = 1ull << 30;   // growth unit (FT_POOL_ARENA_BYTES)
  std::mutex mu;
};

namespace {
// carve sz bytes (granule multiple) out of the first arena with a fitting free range
bool carve(ft_vmm_pool* p, size_t sz, uint64_t* arena, size_t* off) {
  for (auto& kv : p->arenas) {
    Arena& a = kv.second;
    if (a.bytes - a.used < sz) continue;
    for (auto it = a.free.begin(); it != a.free.end(); ++it) {
      if (it->second < sz) continue;
      size_t o = it->first, len = it->second;
      a.free.erase(it);
      if (len > sz) a.free[o + sz] = len - sz;
      a.used += sz;
      *arena = kv.first;
      *off = o;
      return true;
    }
  }
  return false;
}
void give_back(Arena& a, size_t off, size_t len) {
  a.used -= len;
  auto nxt = a.free.lower_bound(off);
  if (nxt != a.free.end() && nxt->first == off + len) {
    len += nxt->second;
    a.free.erase(nxt);
  }
  auto prv = a.free.lower_bound(off);
  if (prv != a.free.begin()) {
    --prv;
    if (prv->first + prv->second == off) {
      off = prv->first;
      len += prv->second;
      a.free.erase(prv);
    }
  }
  a.free[off] = len;
}
// map a new arena of `bytes` (outside the pool mutex: the driver calls are slow)
int map_arena(ft_vmm_pool* p, size_t bytes, bool keep, uint64_t* id_out) {
  Drv* d = drv();
  size_t off = SIZE_MAX;
  {
    std::lock_guard<std::mutex> lk(p->mu);
    for (auto& kv : p->free_va)
      if (kv.second >= bytes) {
        off = kv.first;
        break;
      }
    if (off == SIZE_MAX) {
      ft::set_last_error("VMM pool virtual range exhausted");
      return FT_E_OOM;
    }
    size_t len = p->free_va[off];
    p->free_va.erase(off);
    if (len > bytes) p->free_va[off + bytes] = len - bytes;
  }
  auto give_back_va = [&] {
    std::lock_guard<std::mutex> lk(p->mu);
    p->free_va[off] = bytes;
  };
  static const bool trace = std::getenv("FT_VMM_TRACE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  cudaError_t ce = cudaSetDevice(p->device);
  if (ce != cudaSuccess) {
    give_back_va();
    return cuda_fail(ce, "cudaSetDevice");
  }
  CUmemAllocationProp prop = block_prop(p->device);
  CUmemGenericAllocationHandle h;
  CUresult r = d->create(&h, bytes, &prop, 0);
  if (r != CUDA_SUCCESS) {
    give_back_va();
    return cu_fail(r, "cuMemCreate");
  }
  CUdeviceptr va = p->base + off;
  r = d->map(va, bytes, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    d->release(h);
    give_back_va();
    return cu_fail(r, "cuMemMap");
  }
  int rc = grant_access(d, va, bytes, p->device, true);
  if (rc) {
    d->unmap(va, bytes);
    d->release(h);
    give_back_va();
    return rc;
  }
  if (trace) {
    auto ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[ft_vmm] arena %zu MB mapped in %.2f ms\n", bytes >> 20, ms);
  }
  std::lock_guard<std::mutex> lk(p->mu);
  uint64_t id = p->next_arena++;
  Arena a;
  a.h = h;
  a.va = va;
  a.bytes = bytes;
  a.keep = keep;
  a.free[0] = bytes;
  p->arenas.emplace(id, std::move(a));
  p->mapped += bytes;
  if (id_out) *id_out = id;
  return FT_OK;
}
}  // namespace

namespace ft {

int fwd_ring_words(int device, int slots, uint32_t** landed, uint32_t** freed, uint32_t** err_host) {
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  void* w = nullptr;
  void* e = nullptr;
  cudaError_t r = cudaMalloc(&w, 2 * sizeof(uint32_t) * (size_t)slots);
  if (r == cudaSuccess) r = cudaMemset(w, 0, 2 * sizeof(uint32_t) * (size_t)slots);
  if (r == cudaSuccess) r = cudaHostAlloc(&e, sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable);
  if (cur != device) cudaSetDevice(cur);
  if (r != cudaSuccess) {
    if (w) cudaFree(w);
    return cuda_fail(r, "forward ring words");
  }
  *static_cast<uint32_t*>(e) = 0;
  *landed = static_cast<uint32_t*>(w);
  *freed = static_cast<uint32_t*>(w) + slots;
  *err_host = static_cast<uint32_t*>(e);
  return FT_OK;
}
void fwd_ring_words_free(int device, uint32_t* landed, uint32_t* err_host) {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(device);
  if (landed) cudaFree(landed);
  if (err_host) cudaFreeHost(err_host);
  cudaSetDevice(cur);
}
int fwd_preload(int device) {
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  cudaFuncAttributes a;
  cudaError_t r = cudaFuncGetAttributes(&a, k_forward);
  if (cur != device) cudaSetDevice(cur);
  return r == cudaSuccess ? FT_OK : cuda_fail(r, "k_forward preload");
}
int mem_write32(cudaStream_t st, uint32_t* addr, uint32_t value) {
  Drv* d = drv();
  if (!d) {
    set_last_error("CUDA driver stream memory operations unavailable");
    return FT_E_NOT_SUPPORTED;
  }
  static const unsigned flags =
      std::getenv("FT_K2_NOBAR") ? CU_STREAM_WRITE_VALUE_NO_MEMORY_BARRIER : CU_STREAM_WRITE_VALUE_DEFAULT;
  CU_DRV(d->write32((CUstream)st, (CUdeviceptr)addr, value, flags));
  return FT_OK;
}
int mem_wait_geq32(cudaStream_t st, uint32_t* addr, uint32_t value) {
  Drv* d = drv();
  if (!d) {
    set_last_error("CUDA driver stream memory operations unavailable");
    return FT_E_NOT_SUPPORTED;
  }
  CU_DRV(d->wait32((CUstream)st, (CUdeviceptr)addr, value, CU_STREAM_WAIT_VALUE_GEQ));
  return FT_OK;
}
int fwd_launch(int device, cudaStream_t st, uint8_t* dst, const uint8_t* ring, uint64_t slot_bytes,
               const uint32_t* landed, uint32_t* freed, uint32_t* err, const FwdBatch& b) {
  if (b.n <= 0) return FT_OK;
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  k_forward<<<kFwdCtas, 256, 0, st>>>(dst, ring, slot_bytes, landed, freed, err, b);
  cudaError_t e = cudaGetLastError();
  if (cur != device) cudaSetDevice(cur);
  return e == cudaSuccess ? FT_OK : cuda_fail(e, "k_forward");
}

}  // namespace ft

extern "C" {

int ft_device_count(int* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *out = 0;
    cudaGetLastError();
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  *out = n;
  return FT_OK;
}

int ft_peer_enable(int device, int peer) {
  if (device == peer) return FT_OK;
  int ok = 0;
  CU_RT(cudaDeviceCanAccessPeer(&ok, device, peer));
  if (!ok) {
    ft::set_last_error("peer access not supported between these GPUs");
    return FT_E_NOT_SUPPORTED;
  }
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  CU_RT(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(cur);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return FT_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  return FT_OK;
}

int ft_vmm_granularity(int device, uint64_t* out) {
  Drv* d = drv();
  if (!d) {
    ft::set_last_error("CUDA driver VMM entry points unavailable");
    return FT_E_NOT_SUPPORTED;
  }
  CU_RT(cudaSetDevice(device));
  CU_RT(cudaFree(0));
  CUmemAllocationProp p = block_prop(device);
  size_t g = 0;
  CU_DRV(d->granularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  *out = g;
  return FT_OK;
}

int ft_vmm_pool_create(int device, uint64_t va_bytes, ft_vmm_pool** out) {
  Drv* d = drv();
  if (!d) {
    ft::set_last_error("CUDA driver VMM entry points unavailable");
    return FT_E_NOT_SUPPORTED;
  }
  uint64_t gran = 0;
  int rc = ft_vmm_granularity(device, &gran);
  if (rc) return rc;
  va_bytes = (va_bytes + gran - 1) / gran * gran;
  CUdeviceptr base = 0;
  CU_DRV(d->reserve(&base, va_bytes, gran, 0, 0));
  auto* p = new ft_vmm_pool{};
  p->device = device;
  p->gran = gran;
  p->base = base;
  p->va_bytes = va_bytes;
  p->free_va[0] = va_bytes;
  if (const char* e = std::getenv("FT_POOL_ARENA_BYTES")) p->arena_bytes = std::max<size_t>(gran, std::atoll(e));
  p->arena_bytes = (p->arena_bytes + gran - 1) / gran * gran;
  va_add((uintptr_t)base, va_bytes, device);
  *out = p;
  return FT_OK;
}

void ft_vmm_pool_destroy(ft_vmm_pool* p) {
  if (!p) return;
  Drv* d = drv();
  if (d) {
    for (auto& kv : p->arenas) {
      d->unmap(kv.second.va, kv.second.bytes);
      d->release(kv.second.h);
    }
    va_remove((uintptr_t)p->base);
    d->addr_free(p->base, p->va_bytes);
  }
  delete p;
}

int ft_vmm_pool_reserve(ft_vmm_pool* p, uint64_t bytes) {
  if (!p || !bytes) {
    ft::set_last_error("ft_vmm_pool_reserve: bad arguments");
    return FT_E_VALUE;
  }
  size_t sz = (bytes + p->gran - 1) / p->gran * p->gran;
  return map_arena(p, sz, true, nullptr);
}

int ft_vmm_block_map(ft_vmm_pool* p, uint64_t bytes, uint64_t* block, void** dptr) {
  if (!p || !bytes) {
    ft::set_last_error("ft_vmm_block_map: bad arguments");
    return FT_E_VALUE;
  }
  size_t sz = (bytes + p->gran - 1) / p->gran * p->gran;
  for (int attempt = 0; attempt < 2; ++attempt) {
    {
      std::lock_guard<std::mutex> lk(p->mu);
      uint64_t ar = 0;
      size_t off = 0;
      if (carve(p, sz, &ar, &off)) {
        uint64_t id = p->next_id++;
        p->blocks[id] = Block{ar, off, sz};
        *block = id;
        *dptr = reinterpret_cast<void*>(p->arenas[ar].va + off);
        return FT_OK;
      }
    }
    if (attempt) break;
    // no arena has room: map a new one (the growth unit, or the block if larger)
    int rc = map_arena(p, std::max(sz, p->arena_bytes), false, nullptr);
    if (rc == FT_E_OOM && sz < p->arena_bytes) rc = map_arena(p, sz, false, nullptr);  // near the memory limit
    if (rc) return rc;
  }
  ft::set_last_error("ft_vmm_block_map: no room after growth");
  return FT_E_OOM;
}

int ft_vmm_block_unmap(ft_vmm_pool* p, uint64_t block) {
  std::lock_guard<std::mutex> lk(p->mu);
  auto it = p->blocks.find(block);
  if (it == p->blocks.end()) {
    ft::set_last_error("unknown VMM block");
    return FT_E_KEY;
  }
  Block b = it->second;
  p->blocks.erase(it);
  give_back(p->arenas[b.arena], b.off, b.bytes);  // no driver call: the arena stays mapped
  return FT_OK;
}

int ft_vmm_pool_trim(ft_vmm_pool* p, uint64_t* arenas_out, int cap, int* n_out) {
  // unmap every arena no block uses (and not reserved): physical memory back to
  // the driver. Call when the GPU is quiet (the unmap stalls the process otherwise)
  Drv* d = drv();
  std::vector<std::pair<uint64_t, Arena>> gone;
  {
    std::lock_guard<std::mutex> lk(p->mu);
    for (auto it = p->arenas.begin(); it != p->arenas.end();) {
      if (it->second.used == 0 && !it->second.keep) {
        gone.emplace_back(it->first, std::move(it->second));
        it = p->arenas.erase(it);
      } else {
        ++it;
      }
    }
  }
  int n = 0, rc = FT_OK;
  for (auto& g : gone) {
    CUresult r = d->unmap(g.second.va, g.second.bytes);
    if (r == CUDA_SUCCESS) r = d->release(g.second.h);
    if (r != CUDA_SUCCESS && rc == FT_OK) rc = cu_fail(r, "trim");
    std::lock_guard<std::mutex> lk(p->mu);
    p->mapped -= g.second.bytes;
    size_t off = g.second.va - p->base, len = g.second.bytes;
    auto nxt = p->free_va.lower_bound(off);
    if (nxt != p->free_va.end() && nxt->first == off + len) {
      len += nxt->second;
      p->free_va.erase(nxt);
    }
    auto prv = p->free_va.lower_bound(off);
    if (prv != p->free_va.begin()) {
      --prv;
      if (prv->first + prv->second == off) {
        off = prv->first;
        len += prv->second;
        p->free_va.erase(prv);
      }
    }
    p->free_va[off] = len;
    if (arenas_out && n < cap) arenas_out[n] = g.first;
    ++n;
  }
  if (n_out) *n_out = n;
  return rc;
}

int ft_vmm_block_locate(ft_vmm_pool* p, uint64_t block, uint64_t* arena, uint64_t* offset, uint64_t* arena_bytes) {
  std::lock_guard<std::mutex> lk(p->mu);
  auto it = p->blocks.find(block);
  if (it == p->blocks.end()) {
    ft::set_last_error("unknown VMM block");
    return FT_E_KEY;
  }
  if (arena) *arena = it->second.arena;
  if (offset) *offset = it->second.off;
  if (arena_bytes) *arena_bytes = p->arenas[it->second.arena].bytes;
  return FT_OK;
}

int ft_vmm_block_export_fd(ft_vmm_pool* p, uint64_t block, int* fd) {
  // the block's arena (the unit of physical memory); the importer maps the whole
  // arena once and finds the block at its offset (ft_vmm_block_locate)
  Drv* d = drv();
  std::lock_guard<std::mutex> lk(p->mu);
  auto it = p->blocks.find(block);
  if (it == p->blocks.end()) {
    ft::set_last_error("unknown VMM block");
    return FT_E_KEY;
  }
  int f = -1;
  CU_DRV(d->export_handle(&f, p->arenas[it->second.arena].h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  *fd = f;
  return FT_OK;
}

int ft_vmm_pool_stats(const ft_vmm_pool* p, uint64_t* mapped, uint64_t* reserved, int* blocks) {
  if (mapped) *mapped = p->mapped;
  if (reserved) *reserved = p->va_bytes;
  if (blocks) *blocks = (int)p->blocks.size();
  return FT_OK;
}

int ft_vmm_import_fd(int device, int fd, uint64_t bytes, void** dptr, uint64_t* handle) {
  Drv* d = drv();
  if (!d) {
    ft::set_last_error("CUDA driver VMM entry points unavailable");
    return FT_E_NOT_SUPPORTED;
  }
  CU_RT(cudaSetDevice(device));
  CU_RT(cudaFree(0));
  CUmemGenericAllocationHandle h;
  CU_DRV(d->import_handle(&h, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
  uint64_t gran = 0;
  int rc = ft_vmm_granularity(device, &gran);
  if (rc) {
    d->release(h);
    return rc;
  }
  size_t sz = (bytes + gran - 1) / gran * gran;
  CUdeviceptr va = 0;
  CUresult r = d->reserve(&va, sz, gran, 0, 0);
  if (r != CUDA_SUCCESS) {
    d->release(h);
    return cu_fail(r, "cuMemAddressReserve");
  }
  r = d->map(va, sz, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    d->addr_free(va, sz);
    d->release(h);
    return cu_fail(r, "cuMemMap(import)");
  }
  rc = grant_access(d, va, sz, device, false);
  if (rc) {
    d->unmap(va, sz);
    d->addr_free(va, sz);
    d->release(h);
    return rc;
  }
  uint64_t id = g_imp_next++;
  {
    std::lock_guard<std::mutex> lk(g_imp_mu);
    g_imports[id] = Import{h, va, sz};
  }
  *dptr = reinterpret_cast<void*>(va);
  *handle = id;
  return FT_OK;
}

int ft_vmm_unimport(uint64_t handle) {
  Drv* d = drv();
  Import im;
  {
    std::lock_guard<std::mutex> lk(g_imp_mu);
    auto it = g_imports.find(handle);
    if (it == g_imports.end()) {
      ft::set_last_error("unknown import handle");
      return FT_E_KEY;
    }
    im = it->second;
    g_imports.erase(it);
  }
  CU_DRV(d->unmap(im.va, im.bytes));
  CU_DRV(d->addr_free(im.va, im.bytes));
  CU_DRV(d->release(im.h));
  return FT_OK;
}

// ---- interprocess events: cross-process stream ordering without host syncs
int ft_ipc_event_create(int device, void** ev, void* handle64) {
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  cudaEvent_t e = nullptr;
  cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventInterprocess | cudaEventDisableTiming);
  cudaIpcEventHandle_t h;
  if (r == cudaSuccess) r = cudaIpcGetEventHandle(&h, e);
  if (cur != device) cudaSetDevice(cur);
  if (r != cudaSuccess) {
    if (e) cudaEventDestroy(e);
    return cuda_fail(r, "ft_ipc_event_create");
  }
  static_assert(sizeof(h) == 64, "cudaIpcEventHandle_t is 64 bytes");
  memcpy(handle64, &h, 64);
  *ev = e;
  return FT_OK;
}
int ft_ipc_event_open(int device, const void* handle64, void** ev) {
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  cudaIpcEventHandle_t h;
  memcpy(&h, handle64, 64);
  cudaEvent_t e = nullptr;
  cudaError_t r = cudaIpcOpenEventHandle(&e, h);
  if (cur != device) cudaSetDevice(cur);
  if (r != cudaSuccess) return cuda_fail(r, "ft_ipc_event_open");
  *ev = e;
  return FT_OK;
}

int ft_fd_send(int sock, int fd, uint64_t tag) {
  struct msghdr msg = {};
  char cbuf[CMSG_SPACE(sizeof(int))];
  memset(cbuf, 0, sizeof cbuf);
  struct iovec iov = {&tag, sizeof tag};
  msg.msg_iov = &iov;
  msg.msg_iovlen = 1;
  msg.msg_control = cbuf;
  msg.msg_controllen = sizeof cbuf;
  struct cmsghdr* c = CMSG_FIRSTHDR(&msg);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(sizeof(int));
  memcpy(CMSG_DATA(c), &fd, sizeof(int));
  if (sendmsg(sock, &msg, 0) != (ssize_t)sizeof tag) {
    ft::set_last_error(std::string("sendmsg: ") + strerror(errno));
    return FT_E_VALUE;
  }
  return FT_OK;
}

int ft_fd_recv(int sock, int* fd, uint64_t* tag) {
  struct msghdr msg = {};
  char cbuf[CMSG_SPACE(sizeof(int))];
  uint64_t t = 0;
  struct iovec iov = {&t, sizeof t};
  msg.msg_iov = &iov;
  msg.msg_iovlen = 1;
  msg.msg_control = cbuf;
  msg.msg_controllen = sizeof cbuf;
  if (recvmsg(sock, &msg, 0) != (ssize_t)sizeof t) {
    ft::set_last_error(std::string("recvmsg: ") + strerror(errno));
    return FT_E_VALUE;
  }
  struct cmsghdr* c = CMSG_FIRSTHDR(&msg);
  if (!c || c->cmsg_type != SCM_RIGHTS) {
    ft::set_last_error("recvmsg: no fd attached");
    return FT_E_VALUE;
  }
  memcpy(fd, CMSG_DATA(c), sizeof(int));
  if (tag) *tag = t;
  return FT_OK;
}

int ft_copy(void* dst, const void* src, uint64_t bytes, int device, void* stream) {
  // auto engine: TMA bulk when both sides are memory of `device`, else the
  // peer-safe vector engine. Pool blocks are recognised by their VA range.
  const int vd = va_device(dst), vs = va_device(src);
  if (vd >= 0 && vs >= 0) return copy_impl(dst, src, bytes, device, (cudaStream_t)stream,
                                           vd == device && vs == device ? 1 : 2, 0);
  cudaPointerAttributes a{}, b{};
  int engine = 1;
  if (cudaPointerGetAttributes(&a, dst) != cudaSuccess || cudaPointerGetAttributes(&b, src) != cudaSuccess) {
    cudaGetLastError();
    engine = 2;
  } else if (a.type != cudaMemoryTypeDevice || b.type != cudaMemoryTypeDevice || a.device != device ||
             b.device != device) {
    engine = 2;
  }
  return copy_impl(dst, src, bytes, device, (cudaStream_t)stream, engine, 0);
}

int ft_copy_ex(void* dst, const void* src, uint64_t bytes, int device, void* stream, int engine, int grid) {
  if (engine < 0 || engine > 2) {
    ft::set_last_error("unknown copy engine");
    return FT_E_VALUE;
  }
  if (engine == 0) return ft_copy(dst, src, bytes, device, stream);
  return copy_impl(dst, src, bytes, device, (cudaStream_t)stream, engine, grid);
}

int ft_signal(uint32_t* flag, uint32_t value, int device, void* stream) {
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  k_signal<<<1, 1, 0, (cudaStream_t)stream>>>(flag, value);
  cudaError_t e = cudaGetLastError();
  if (cur != device) cudaSetDevice(cur);
  return e == cudaSuccess ? FT_OK : cuda_fail(e, "ft_signal");
}

int ft_wait(const uint32_t* flag, uint32_t value, int device, void* stream) {
  return ft_wait_timeout(flag, value, 30000000000ull, nullptr, device, stream);
}
int ft_wait_timeout(const uint32_t* flag, uint32_t value, uint64_t timeout_ns, uint32_t* err, int device,
                    void* stream) {
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  k_wait<<<1, 1, 0, (cudaStream_t)stream>>>(flag, value, timeout_ns, err);
  cudaError_t e = cudaGetLastError();
  if (cur != device) cudaSetDevice(cur);
  return e == cudaSuccess ? FT_OK : cuda_fail(e, "ft_wait");
}

// ---- batched copies: one launch per <= 64 segments
int ft_copy_batch(const ft_segment* segs, int n, int device, void* stream) {
  if (n < 0 || (n && !segs)) {
    ft::set_last_error("ft_copy_batch: bad arguments");
    return FT_E_VALUE;
  }
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  cudaError_t e = cudaSuccess;
  for (int base = 0; base < n && e == cudaSuccess;) {
    MultiArgs a;
    a.n = 0;
    a.first_tile[0] = 0;
    for (; base < n && a.n < kMultiMax; ++base) {
      if (!segs[base].bytes) continue;
      int k = a.n++;
      a.dst[k] = static_cast<uint8_t*>(segs[base].dst);
      a.src[k] = static_cast<const uint8_t*>(segs[base].src);
      a.bytes[k] = segs[base].bytes;
      a.first_tile[k + 1] = a.first_tile[k] + (segs[base].bytes + kMultiTile - 1) / kMultiTile;
    }
    if (!a.n) break;
    uint64_t tiles = a.first_tile[a.n];
    int grid = (int)std::min<uint64_t>(tiles, (uint64_t)4 * dev_sms(device));
    k_copy_multi<<<grid, 512, 0, (cudaStream_t)stream>>>(a);
    e = cudaGetLastError();
  }
  if (cur != device) cudaSetDevice(cur);
  return e == cudaSuccess ? FT_OK : cuda_fail(e, "ft_copy_batch");
}

// ---- private streams: torch.cuda.Stream() hands out a round-robin pool of 32
// streams per device, so "new" torch streams alias each other — a CE route
// could share a FIFO with another tenant's consumer stream. Ours are unique.
int ft_stream_create(int device, void** stream) {
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  cudaStream_t st = nullptr;
  cudaError_t r = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (cur != device) cudaSetDevice(cur);
  if (r != cudaSuccess) return cuda_fail(r, "ft_stream_create");
  *stream = st;
  return FT_OK;
}
int ft_stream_destroy(void* stream) {
  CU_RT(cudaStreamDestroy((cudaStream_t)stream));
  return FT_OK;
}

// ---- raw events (the request path's ordering, without torch.cuda.Event objects)
int ft_event_create(int device, void** ev) {
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  cudaEvent_t e = nullptr;
  cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  if (cur != device) cudaSetDevice(cur);
  if (r != cudaSuccess) return cuda_fail(r, "ft_event_create");
  *ev = e;
  return FT_OK;
}
int ft_event_destroy(void* ev) {
  CU_RT(cudaEventDestroy((cudaEvent_t)ev));
  return FT_OK;
}
int ft_event_record(void* ev, void* stream) {
  CU_RT(cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)stream));
  return FT_OK;
}
int ft_event_query(void* ev, int* done) {
  cudaError_t r = cudaEventQuery((cudaEvent_t)ev);
  if (r == cudaErrorNotReady) {
    *done = 0;
    return FT_OK;
  }
  if (r != cudaSuccess) return cuda_fail(r, "ft_event_query");
  *done = 1;
  return FT_OK;
}
int ft_event_synchronize(void* ev) {
  CU_RT(cudaEventSynchronize((cudaEvent_t)ev));
  return FT_OK;
}
int ft_stream_wait_events(void* stream, void* const* evs, int n) {
  for (int i = 0; i < n; ++i)
    if (evs[i]) CU_RT(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)evs[i], 0));
  return FT_OK;
}
// one call for a request-path copy: wait on `waits`, TMA-bulk copy with L2 hints,
// record `done` (any of them may be absent)
int ft_copy_ordered(void* dst, const void* src, uint64_t bytes, int device, void* stream, uint32_t hints,
                    void* const* waits, int nwaits, void* done) {
  int rc = ft_stream_wait_events(stream, waits, nwaits);
  if (rc != FT_OK) return rc;
  rc = copy_impl(dst, src, bytes, device, (cudaStream_t)stream, 1, 0, hints & 15u);
  if (rc != FT_OK) return rc;
  if (done) CU_RT(cudaEventRecord((cudaEvent_t)done, (cudaStream_t)stream));
  return FT_OK;
}

int ft_stream_write32(void* stream, void* addr, uint32_t value) {
  return ft::mem_write32((cudaStream_t)stream, static_cast<uint32_t*>(addr), value);
}
int ft_stream_wait32(void* stream, const void* addr, uint32_t value) {
  return ft::mem_wait_geq32((cudaStream_t)stream, const_cast<uint32_t*>(static_cast<const uint32_t*>(addr)), value);
}

int ft_spin_ns(uint64_t ns, int device, void* stream) {
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  k_spin_ns<<<1, 1, 0, (cudaStream_t)stream>>>(ns);
  cudaError_t e = cudaGetLastError();
  if (cur != device) cudaSetDevice(cur);
  return e == cudaSuccess ? FT_OK : cuda_fail(e, "ft_spin_ns");
}

int ft_copy_hint(void* dst, const void* src, uint64_t bytes, int device, void* stream, uint32_t hints) {
  return copy_impl(dst, src, bytes, device, (cudaStream_t)stream, 1, 0, hints & 15u);
}

int ft_fingerprint(const void* src, uint64_t bytes, uint64_t* out_dev, int device, void* stream) {
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(out_dev, 0, 16, st);
  if (e == cudaSuccess) {
    uint64_t nw = bytes / 8;
    int grid = 2 * dev_sms(device);
    uint64_t need = (nw + 511) / 512;
    if (need < (uint64_t)grid) grid = (int)(need ? need : 1);
    k_fingerprint<<<grid, 512, 0, st>>>(static_cast<const uint8_t*>(src), bytes,
                                        reinterpret_cast<unsigned long long*>(out_dev));
    e = cudaGetLastError();
  }
  if (cur != device) cudaSetDevice(cur);
  return e == cudaSuccess ? FT_OK : cuda_fail(e, "ft_fingerprint");
}

int ft_fingerprint_host(const void* src_, uint64_t bytes, uint64_t out[2]) {
  const uint8_t* src = static_cast<const uint8_t*>(src_);
  uint64_t nw = bytes / 8, s = 0, x = 0;
  for (uint64_t i = 0; i < nw; ++i) {
    uint64_t w;
    memcpy(&w, src + 8 * i, 8);
    uint64_t h = fp_word(w, i);
    s += h;
    x ^= h;
  }
  if (bytes & 7) {
    uint64_t t = 0;
    for (uint64_t k = 0; k < (bytes & 7); ++k) t |= (uint64_t)src[nw * 8 + k] << (8 * k);
    uint64_t h = fp_word(t, nw);
    s += h;
    x ^= h;
  }
  out[0] = s;
  out[1] = x;
  return FT_OK;
}

int ft_pcie_copy(void* dst, const void* src, uint64_t bytes, int to_device, int device, void* stream,
                 uint64_t batch_bytes) {
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  if (cur != device) CU_RT(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyKind kind = to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  uint64_t step = batch_bytes ? batch_bytes : bytes;
  cudaError_t e = cudaSuccess;
  for (uint64_t off = 0; off < bytes && e == cudaSuccess; off += step) {
    uint64_t n = bytes - off < step ? bytes - off : step;
    e = cudaMemcpyAsync(static_cast<uint8_t*>(dst) + off, static_cast<const uint8_t*>(src) + off, n, kind, st);
  }
  if (cur != device) cudaSetDevice(cur);
  return e == cudaSuccess ? FT_OK : cuda_fail(e, "ft_pcie_copy");
}

int ft_h2g_striped(void* dst_, int dst_dev, const void* host_, uint64_t bytes, int k, const int32_t* stage_dev,
                   const uint64_t* off, const uint64_t* len, void* const* staging, uint64_t chunk, int ring,
                   void* const* streams) {
  if (k <= 0 || !off || !len || !streams || !stage_dev) {
    ft::set_last_error("ft_h2g_striped: bad arguments");
    return FT_E_VALUE;
  }
  uint8_t* dst = static_cast<uint8_t*>(dst_);
  const uint8_t* host = static_cast<const uint8_t*>(host_);
  int cur = 0;
  CU_RT(cudaGetDevice(&cur));
  int rc = FT_OK;
  for (int r = 0; r < k && rc == FT_OK; ++r) {
    if (off[r] + len[r] > bytes) {
      ft::set_last_error("ft_h2g_striped: route outside the payload");
      rc = FT_E_VALUE;
      break;
    }
    cudaStream_t ce = (cudaStream_t)streams[2 * r], fw = (cudaStream_t)streams[2 * r + 1];
    int sd = stage_dev[r];
    if (!staging || !staging[r]) {
      // own link: straight into the destination by CE
      rc = ft_pcie_copy(dst + off[r], host + off[r], len[r], 1, dst_dev, ce, 0);
      continue;
    }
    if (!chunk || ring <= 0) {
      ft::set_last_error("ft_h2g_striped: chunk/ring required for staging routes");
      rc = FT_E_VALUE;
      break;
    }
    cudaSetDevice(sd);
    // ring events from a per-device pool (re-recording an event is safe once every
    // wait on its previous record is enqueued, i.e. after this call): no create /
    // destroy per call
    std::vector<cudaEvent_t> landed = take_events(sd, ring), freed = take_events(sd, ring);
    if ((int)landed.size() < ring || (int)freed.size() < ring) {
      put_events(sd, landed);
      put_events(sd, freed);
      ft::set_last_error("ft_h2g_striped: cudaEventCreate failed");
      rc = FT_E_CUDA;
      break;
    }
    uint8_t* stg = static_cast<uint8_t*>(staging[r]);
    uint64_t nch = (len[r] + chunk - 1) / chunk;
    for (uint64_t j = 0; j < nch && rc == FT_OK; ++j) {
      int slot = (int)(j % ring);
      uint64_t o = j * chunk, n = len[r] - o < chunk ? len[r] - o : chunk;
      if (j >= (uint64_t)ring) cudaStreamWaitEvent(ce, freed[slot], 0);  // slot drained by the forward
      cudaError_t e = cudaMemcpyAsync(stg + (uint64_t)slot * chunk, host + off[r] + o, n, cudaMemcpyHostToDevice, ce);
      if (e != cudaSuccess) {
        rc = cuda_fail(e, "staging H2D");
        break;
      }
      cudaEventRecord(landed[slot], ce);
      cudaStreamWaitEvent(fw, landed[slot], 0);
      rc = copy_impl(dst + off[r] + o, stg + (uint64_t)slot * chunk, n, sd, fw, 2, 0);  // push over NVLink
      cudaEventRecord(freed[slot], fw);
    }
    put_events(sd, landed);
    put_events(sd, freed);
  }
  cudaSetDevice(cur);
  return rc;
}

}  // extern "C"
