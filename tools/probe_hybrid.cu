// Probe 3: does SM-pull alongside CE (or several CE streams) beat one CE stream on one PCIe link?
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)
__global__ void pull(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += 4 * stride) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * stride < n16) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * stride < n16) __stcs(dst + i + u * stride, v[u]);
  }
}
int main() {
  const size_t N = 1ull << 30;
  char* h; CK(cudaHostAlloc((void**)&h, N, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 3, N);
  char* hd; CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  char* d; CK(cudaMalloc(&d, N));
  cudaStream_t s[4]; for (auto& x : s) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
  cudaEvent_t a, b, j[4]; cudaEventCreate(&a); cudaEventCreate(&b); for (auto& x : j) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  auto run = [&](auto fn) { float bm = 1e9; for (int r = 0; r < 4; ++r) { cudaEventRecord(a, s[0]); for (int k = 1; k < 4; ++k) cudaStreamWaitEvent(s[k], a, 0); fn(); for (int k = 1; k < 4; ++k) { cudaEventRecord(j[k], s[k]); cudaStreamWaitEvent(s[0], j[k], 0); } cudaEventRecord(b, s[0]); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); bm = std::min(bm, ms); } return bm; };
  float ms = run([&] { cudaMemcpyAsync(d, h, N, cudaMemcpyHostToDevice, s[0]); }); printf("CE x1: %.2f GB/s\n", N / ms / 1e6);
  ms = run([&] { cudaMemcpyAsync(d, h, N / 2, cudaMemcpyHostToDevice, s[0]); cudaMemcpyAsync(d + N / 2, h + N / 2, N / 2, cudaMemcpyHostToDevice, s[1]); }); printf("CE x2 streams: %.2f GB/s\n", N / ms / 1e6);
  ms = run([&] { for (int k = 0; k < 4; ++k) cudaMemcpyAsync(d + k * N / 4, h + k * N / 4, N / 4, cudaMemcpyHostToDevice, s[k]); }); printf("CE x4 streams: %.2f GB/s\n", N / ms / 1e6);
  for (double f : {0.5, 0.7, 0.8, 0.9, 0.95}) for (int g : {16, 37, 74, 148}) {
    size_t nce = ((size_t)(N * f)) & ~(size_t)4095;
    ms = run([&] { cudaMemcpyAsync(d, h, nce, cudaMemcpyHostToDevice, s[0]); pull<<<g, 512, 0, s[1]>>>((const int4*)(hd + nce), (int4*)(d + nce), (N - nce) / 16); });
    printf("CE %.2f + SM(g=%d): %.2f GB/s\n", f, g, N / ms / 1e6);
  }
  // D2H
  ms = run([&] { cudaMemcpyAsync(h, d, N, cudaMemcpyDeviceToHost, s[0]); }); printf("D2H CE x1: %.2f GB/s\n", N / ms / 1e6);
  ms = run([&] { cudaMemcpyAsync(h, d, N / 2, cudaMemcpyDeviceToHost, s[0]); cudaMemcpyAsync(h + N / 2, d + N / 2, N / 2, cudaMemcpyDeviceToHost, s[1]); }); printf("D2H CE x2: %.2f GB/s\n", N / ms / 1e6);
  // bidirectional
  char* d2; CK(cudaMalloc(&d2, N)); char* h2; CK(cudaHostAlloc((void**)&h2, N, cudaHostAllocMapped));
  ms = run([&] { cudaMemcpyAsync(d, h, N, cudaMemcpyHostToDevice, s[0]); cudaMemcpyAsync(h2, d2, N, cudaMemcpyDeviceToHost, s[1]); }); printf("bidir CE: %.2f GB/s each way\n", N / ms / 1e6);
  return 0;
}
