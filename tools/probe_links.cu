// Link/bandwidth probe for the B200 box (run once per round under gpurun).
// Measures: CE pinned H2D/D2H, SM-pull from mapped pinned host memory,
// local D2D copy (CE and v4 kernel), VMM granularity / POSIX-FD support.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int UNROLL>
__global__ void pull_v4(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = tid;
  for (; i + (UNROLL - 1) * stride < n16; i += UNROLL * stride) {
    int4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) __stcs(dst + i + u * stride, v[u]);
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

// chunked: each CTA owns contiguous 64 KiB slabs (better PCIe request locality)
template <int UNROLL>
__global__ void pull_slab(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16, size_t slab16) {
  size_t nslab = (n16 + slab16 - 1) / slab16;
  for (size_t s = blockIdx.x; s < nslab; s += gridDim.x) {
    size_t base = s * slab16;
    size_t end = min(base + slab16, n16);
    for (size_t i = base + threadIdx.x; i < end; i += UNROLL * blockDim.x) {
      int4 v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) { size_t j = i + u * blockDim.x; if (j < end) v[u] = __ldcs(src + j); }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) { size_t j = i + u * blockDim.x; if (j < end) __stcs(dst + j, v[u]); }
    }
  }
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) { float ms; cudaEventElapsedTime(&ms, a, b); return ms; }

int main() {
  int ndev = 0; CK(cudaGetDeviceCount(&ndev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("devices=%d name=%s sms=%d pciBus=%d asyncEngines=%d canMapHost=%d unifiedAddr=%d\n", ndev, p.name, p.multiProcessorCount, p.pciBusID, p.asyncEngineCount, p.canMapHostMemory, p.unifiedAddressing);
  const size_t N = 1ull << 30;
  void* h; CK(cudaHostAlloc(&h, N, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 7, N);
  void* hd; CK(cudaHostGetDevicePointer(&hd, h, 0));
  void *d, *d2; CK(cudaMalloc(&d, N)); CK(cudaMalloc(&d2, N));
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto best = [&](auto fn, int reps) { float bm = 1e9; for (int r = 0; r < reps; ++r) { cudaEventRecord(a, s); fn(); cudaEventRecord(b, s); cudaEventSynchronize(b); bm = std::min(bm, time_ms(a, b)); } return bm; };
  float ms;
  ms = best([&] { cudaMemcpyAsync(d, h, N, cudaMemcpyHostToDevice, s); }, 5); printf("CE H2D 1GiB: %.3f ms %.2f GB/s\n", ms, N / ms / 1e6);
  ms = best([&] { cudaMemcpyAsync(h, d, N, cudaMemcpyDeviceToHost, s); }, 5); printf("CE D2H 1GiB: %.3f ms %.2f GB/s\n", ms, N / ms / 1e6);
  for (size_t ch : {2000000ul, 2097152ul, 8388608ul}) {
    ms = best([&] { for (size_t o = 0; o < N; o += ch) cudaMemcpyAsync((char*)d + o, (char*)h + o, std::min(ch, N - o), cudaMemcpyHostToDevice, s); }, 3);
    printf("CE H2D 1GiB in %zu-byte chunks: %.3f ms %.2f GB/s\n", ch, ms, N / ms / 1e6);
  }
  for (size_t sz : {1ul << 20, 4ul << 20, 16ul << 20, 64ul << 20, 256ul << 20}) {
    ms = best([&] { cudaMemcpyAsync(d, h, sz, cudaMemcpyHostToDevice, s); }, 10); printf("CE H2D %zu: %.4f ms %.2f GB/s\n", sz, ms, sz / ms / 1e6);
  }
  size_t n16 = N / 16;
  for (int blocks : {148, 296, 592, 1184, 2368}) for (int th : {256, 512, 1024}) {
    ms = best([&] { pull_v4<4><<<blocks, th, 0, s>>>((const int4*)hd, (int4*)d, n16); }, 3);
    printf("SM-pull v4 u4 grid=%d thr=%d: %.3f ms %.2f GB/s\n", blocks, th, ms, N / ms / 1e6);
  }
  for (int blocks : {148, 296, 592, 1184}) for (size_t slab : {65536ul, 262144ul, 2097152ul}) {
    ms = best([&] { pull_slab<4><<<blocks, 512, 0, s>>>((const int4*)hd, (int4*)d, n16, slab / 16); }, 3);
    printf("SM-pull slab=%zu grid=%d: %.3f ms %.2f GB/s\n", slab, blocks, ms, N / ms / 1e6);
  }
  // SM push: device -> mapped host
  for (int blocks : {296, 1184}) {
    ms = best([&] { pull_v4<4><<<blocks, 512, 0, s>>>((const int4*)d, (int4*)hd, n16); }, 3);
    printf("SM-push(D2H) grid=%d: %.3f ms %.2f GB/s\n", blocks, ms, N / ms / 1e6);
  }
  // concurrent CE + SM pull (two halves)
  ms = best([&] { cudaMemcpyAsync(d, h, N / 2, cudaMemcpyHostToDevice, s); }, 3); printf("CE half: %.3f\n", ms);
  // local copy
  ms = best([&] { cudaMemcpyAsync(d2, d, N, cudaMemcpyDeviceToDevice, s); }, 5); printf("CE D2D 1GiB: %.3f ms %.2f GB/s (r+w %.1f)\n", ms, N / ms / 1e6, 2 * N / ms / 1e6);
  for (int blocks : {148, 296, 592, 1184}) for (int th : {256, 512, 1024}) {
    ms = best([&] { pull_v4<4><<<blocks, th, 0, s>>>((const int4*)d, (int4*)d2, n16); }, 5);
    printf("D2D v4 u4 grid=%d thr=%d: %.3f ms %.2f GB/s (r+w %.1f)\n", blocks, th, ms, N / ms / 1e6, 2 * N / ms / 1e6);
  }
  for (int blocks : {296, 592}) {
    ms = best([&] { pull_v4<8><<<blocks, 512, 0, s>>>((const int4*)d, (int4*)d2, n16); }, 5);
    printf("D2D v4 u8 grid=%d: %.3f ms %.2f GB/s (r+w %.1f)\n", blocks, ms, N / ms / 1e6, 2 * N / ms / 1e6);
  }
  // VMM
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED; prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE; prop.location.id = 0;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuMemGetAllocationGranularity", &fn, cudaEnableDefault, &q));
  size_t gran = 0, granr = 0;
  auto getg = (CUresult(*)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags))fn;
  CUresult r1 = getg(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
  CUresult r2 = getg(&granr, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  printf("VMM granularity min=%zu rec=%zu (r=%d,%d)\n", gran, granr, (int)r1, (int)r2);
  int v = 0; cudaDeviceGetAttribute(&v, (cudaDeviceAttr)103, 0); printf("posixFD supported=%d\n", v);
  cudaDeviceGetAttribute(&v, (cudaDeviceAttr)102, 0); printf("VMM supported=%d\n", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrIpcEventSupport, 0); printf("ipc event=%d\n", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrPageableMemoryAccess, 0); printf("pageableMemoryAccess=%d\n", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrHostRegisterSupported, 0); printf("hostRegister=%d\n", v);
  return 0;
}
