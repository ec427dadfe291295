// Probe 2: SM-driven host->device pull variants (PCIe read request shaping).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ int4 ld_l2_256(const int4* p) {
  int4 r; asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)); return r;
}
__device__ __forceinline__ void ld256(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "l"(p));
}
__device__ __forceinline__ void st256(void* p, const uint32_t (&r)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}

template <int U>
__global__ void pull_l2hint(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += U * stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * stride < n16) v[u] = ld_l2_256(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * stride < n16) __stcs(dst + i + u * stride, v[u]);
  }
}
template <int U>
__global__ void pull_256(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, size_t n32) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n32; i += U * stride) {
    uint32_t v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * stride < n32) ld256(src + 32 * (i + u * stride), v[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * stride < n32) st256(dst + 32 * (i + u * stride), v[u]);
  }
}

// TMA bulk: one elected thread per CTA streams chunks host->smem->device with an mbarrier ring.
template <int STAGES>
__global__ void pull_bulk(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, size_t nbytes, uint32_t tile) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  size_t ntiles = nbytes / tile;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t phase[STAGES] = {0};
  size_t t0 = blockIdx.x;
  // prologue
  int issued = 0;
  size_t t = t0;
  for (int s = 0; s < STAGES && t < ntiles; ++s, t += gridDim.x, ++issued) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t sm = (uint32_t)__cvta_generic_to_shared(smem + s * tile);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(tile));
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sm), "l"(src + t * tile), "r"(tile), "r"(b) : "memory");
  }
  int s = 0;
  for (size_t c = t0; c < ntiles; c += gridDim.x) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t sm = (uint32_t)__cvta_generic_to_shared(smem + s * tile);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" :: "r"(b), "r"(phase[s]));
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst + c * tile), "r"(sm), "r"(tile) : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    // refill this stage once its store has read smem
    if (t < ntiles) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(tile));
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sm), "l"(src + t * tile), "r"(tile), "r"(b) : "memory");
      t += gridDim.x;
    }
    s = (s + 1) % STAGES;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t N = 1ull << 30;
  void* h; CK(cudaHostAlloc(&h, N, cudaHostAllocMapped | cudaHostAllocPortable));
  for (size_t i = 0; i < N / 8; ++i) ((uint64_t*)h)[i] = i * 0x9E3779B97F4A7C15ull;
  void* hd; CK(cudaHostGetDevicePointer(&hd, h, 0));
  void *d; CK(cudaMalloc(&d, N));
  void* chk = malloc(N);
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto best = [&](auto fn, int reps) { float bm = 1e9; for (int r = 0; r < reps; ++r) { cudaEventRecord(a, s); fn(); cudaEventRecord(b, s); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); bm = std::min(bm, ms); } return bm; };
  auto verify = [&](const char* tag) { cudaMemset(d, 0, N); return tag; };
  auto check = [&]() { cudaMemcpy(chk, d, N, cudaMemcpyDeviceToHost); return memcmp(chk, h, N) == 0; };
  float ms;
  ms = best([&] { cudaMemcpyAsync(d, h, N, cudaMemcpyHostToDevice, s); }, 5); printf("CE H2D: %.3f ms %.2f GB/s\n", ms, N / ms / 1e6);
  for (int g : {148, 296, 592}) {
    verify(""); ms = best([&] { pull_l2hint<4><<<g, 512, 0, s>>>((const int4*)hd, (int4*)d, N / 16); }, 3);
    printf("pull L2::256B g=%d: %.3f ms %.2f GB/s ok=%d\n", g, ms, N / ms / 1e6, check());
  }
  for (int g : {148, 296, 592}) {
    verify(""); ms = best([&] { pull_256<4><<<g, 256, 0, s>>>((const uint8_t*)hd, (uint8_t*)d, N / 32); }, 3);
    printf("pull v8.b32 g=%d: %.3f ms %.2f GB/s ok=%d err=%s\n", g, ms, N / ms / 1e6, check(), cudaGetErrorString(cudaGetLastError()));
  }
  for (uint32_t tile : {4096u, 16384u, 32768u}) for (int g : {148, 296}) {
    const int ST = 4; size_t sm = ST * tile; cudaFuncSetAttribute(pull_bulk<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    verify(""); ms = best([&] { pull_bulk<ST><<<g, 32, sm, s>>>((const uint8_t*)hd, (uint8_t*)d, N, tile); }, 3);
    printf("pull TMA-bulk tile=%u st=4 g=%d: %.3f ms %.2f GB/s ok=%d err=%s\n", tile, g, ms, N / ms / 1e6, check(), cudaGetErrorString(cudaGetLastError()));
  }
  for (uint32_t tile : {16384u, 49152u}) for (int g : {148, 296}) {
    const int ST = 2; size_t sm = ST * tile; cudaFuncSetAttribute(pull_bulk<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    verify(""); ms = best([&] { pull_bulk<ST><<<g, 32, sm, s>>>((const uint8_t*)hd, (uint8_t*)d, N, tile); }, 3);
    printf("pull TMA-bulk tile=%u st=2 g=%d: %.3f ms %.2f GB/s ok=%d err=%s\n", tile, g, ms, N / ms / 1e6, check(), cudaGetErrorString(cudaGetLastError()));
  }
  // D2D with TMA bulk
  void* d2; CK(cudaMalloc(&d2, N));
  for (uint32_t tile : {16384u, 32768u}) for (int g : {148, 296}) {
    const int ST = 4; size_t sm = ST * tile; cudaFuncSetAttribute(pull_bulk<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    ms = best([&] { pull_bulk<ST><<<g, 32, sm, s>>>((const uint8_t*)d, (uint8_t*)d2, N, tile); }, 5);
    printf("D2D TMA-bulk tile=%u g=%d: %.3f ms %.2f GB/s (r+w %.1f)\n", tile, g, ms, N / ms / 1e6, 2 * N / ms / 1e6);
  }
  for (int g : {296, 592, 1184}) {
    ms = best([&] { pull_256<4><<<g, 256, 0, s>>>((const uint8_t*)d, (uint8_t*)d2, N / 32); }, 5);
    printf("D2D v8 g=%d: %.3f ms %.2f GB/s (r+w %.1f)\n", g, ms, N / ms / 1e6, 2 * N / ms / 1e6);
  }
  return 0;
}
