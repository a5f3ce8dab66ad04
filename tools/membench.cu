// Micro-benchmark: cost of random 32 B / 64 B gathers and scatters on this GPU
// (informs the PoVar term layout).  nvcc -O3 -arch=sm_100a
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s\n", cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ double4 ldg4(const double* p) {
  double4 v; asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p)); return v; }
__device__ __forceinline__ void st4(double* p, double4 v) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory"); }
template <int W>  // W doubles4 per item
__global__ void gather(const double* __restrict__ src, const int* __restrict__ idx, double* __restrict__ out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
  const double* p = src + (size_t)idx[i] * 4 * W;
  double4 a = ldg4(p); double s = a.x + a.y + a.z + a.w;
  if (W == 2) { double4 b = ldg4(p + 4); s += b.x + b.y + b.z + b.w; }
  out[i] = s;
}
template <int W>
__global__ void scatter(double* __restrict__ dst, const int* __restrict__ idx, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
  double* p = dst + (size_t)idx[i] * 4 * W;
  double4 v = make_double4(i, 1, 2, 3);
  st4(p, v); if (W == 2) st4(p + 4, v);
}
__global__ void stream(const double* __restrict__ src, double* __restrict__ out, size_t n4) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; if (i >= n4) return;
  double4 a = ldg4(src + 4 * i); out[i] = a.x + a.y + a.z + a.w;
}
int main() {
  const int n = 29000000;
  std::mt19937 rng(1);
  double *big, *out; int* idx;
  const size_t nbig = 64ull << 20;  // doubles4-items capacity: 64M items x 64 B = 4 GB
  CK(cudaMalloc(&big, nbig * 64)); CK(cudaMalloc(&out, (size_t)n * 8)); CK(cudaMalloc(&idx, (size_t)n * 4));
  CK(cudaMemset(big, 0, nbig * 64));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](auto fn) { fn(); CK(cudaDeviceSynchronize()); cudaEventRecord(a); for (int r = 0; r < 5; ++r) fn(); cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5; };
  for (size_t items : {4456117ull, 2000000ull, 29000000ull}) {
    std::vector<int> h(n); for (auto& v : h) v = rng() % items;
    CK(cudaMemcpy(idx, h.data(), (size_t)n * 4, cudaMemcpyHostToDevice));
    float g1 = timeit([&] { gather<1><<<(n + 255) / 256, 256>>>(big, idx, out, n); });
    float g2 = timeit([&] { gather<2><<<(n + 255) / 256, 256>>>(big, idx, out, n); });
    printf("items %zu: gather32 %.3f ms (%.0f GB/s useful)  gather64 %.3f ms (%.0f GB/s useful)\n", items, g1, n * 32.0 / g1 / 1e6, g2, n * 64.0 / g2 / 1e6);
  }
  {  // scatter as a permutation of n slots
    std::vector<int> h(n); for (int i = 0; i < n; ++i) h[i] = i; std::shuffle(h.begin(), h.end(), rng);
    CK(cudaMemcpy(idx, h.data(), (size_t)n * 4, cudaMemcpyHostToDevice));
    float s1 = timeit([&] { scatter<1><<<(n + 255) / 256, 256>>>(big, idx, n); });
    float s2 = timeit([&] { scatter<2><<<(n + 255) / 256, 256>>>(big, idx, n); });
    float g1 = timeit([&] { gather<1><<<(n + 255) / 256, 256>>>(big, idx, out, n); });
    printf("perm: scatter32 %.3f ms (%.0f GB/s)  scatter64 %.3f ms (%.0f GB/s)  gather32 %.3f ms (%.0f GB/s)\n", s1, n * 32.0 / s1 / 1e6, s2, n * 64.0 / s2 / 1e6, g1, n*32.0/g1/1e6);
    for (int i = 0; i < n; ++i) h[i] = i;
    CK(cudaMemcpy(idx, h.data(), (size_t)n * 4, cudaMemcpyHostToDevice));
    float s3 = timeit([&] { scatter<1><<<(n + 255) / 256, 256>>>(big, idx, n); });
    float st = timeit([&] { stream<<<(n + 255) / 256, 256>>>(big, out, (size_t)n); });
    printf("sequential scatter32 %.3f ms (%.0f GB/s)  stream read %.3f ms (%.0f GB/s)\n", s3, n * 32.0 / s3 / 1e6, st, n * 32.0 / st / 1e6);
  }
  return 0;
}
