// Probe: what bounds a 1 MiB device copy's kernel time on B200 (run under ncu
// --cache-control none; compare gpu__time_duration of each shape).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/probe_small tools/probe_small.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty() {}
template <int U>
__global__ void k_vec(int4* __restrict__ d, const int4* __restrict__ s, unsigned long long n16) {
  unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(s + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(d + i + u * stride, v[u]);
  }
  for (; i < n16; i += stride) __stcs(d + i, __ldcs(s + i));
}
template <int U>
__global__ void k_vec_plain(int4* __restrict__ d, const int4* __restrict__ s, unsigned long long n16) {
  unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = s[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) d[i + u * stride] = v[u];
  }
  for (; i < n16; i += stride) d[i] = s[i];
}

int main() {
  const size_t n = 1 << 20;
  int4 *a, *b;
  cudaMalloc(&a, n);
  cudaMalloc(&b, n);
  cudaMemset(a, 1, n);
  unsigned long long n16 = n / 16;
  for (int r = 0; r < 3; ++r) {
    k_empty<<<1, 32>>>();
    k_empty<<<128, 256>>>();
    k_empty<<<148, 1024>>>();
    k_vec<2><<<128, 256>>>(b, a, n16);         // the product's small-copy shape
    k_vec<1><<<256, 256>>>(b, a, n16);
    k_vec<4><<<64, 256>>>(b, a, n16);
    k_vec<2><<<64, 512>>>(b, a, n16);
    k_vec<8><<<32, 256>>>(b, a, n16);
    k_vec_plain<2><<<128, 256>>>(b, a, n16);
    cudaMemcpyAsync(b, a, n, cudaMemcpyDeviceToDevice);
  }
  cudaDeviceSynchronize();
  printf("ok %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
