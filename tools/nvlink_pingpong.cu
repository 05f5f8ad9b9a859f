// Cross-GPU doorbell latency over NVLink (single process, GPU0 <-> GPU1):
// one thread on each GPU bounces a counter through flags that live in the
// receiver's memory (st.release.sys to the peer, ld.acquire.sys polling of
// local memory) -- the primitive the hand-off's ready/free doorbells use.
// Variants: polling with and without __nanosleep back-off.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/nvlink_pingpong tools/nvlink_pingpong.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool SLEEP>
__global__ void pinger(uint32_t* my_flag, uint32_t* peer_flag, int n, unsigned long long* t) {
  unsigned long long t0 = 0, t1 = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= n; ++i) {
    st_rel(peer_flag, i);
    while (ld_acq(my_flag) != uint32_t(i)) if (SLEEP) __nanosleep(32);
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  *t = t1 - t0;
}

template <bool SLEEP>
__global__ void ponger(uint32_t* my_flag, uint32_t* peer_flag, int n) {
  for (int i = 1; i <= n; ++i) {
    while (ld_acq(my_flag) != uint32_t(i)) if (SLEEP) __nanosleep(32);
    st_rel(peer_flag, i);
  }
}

template <bool SLEEP>
double run(uint32_t* f0, uint32_t* f1, unsigned long long* t, int n) {
  cudaSetDevice(0); cudaMemset(f0, 0, 4);
  cudaSetDevice(1); cudaMemset(f1, 0, 4);
  cudaDeviceSynchronize();
  cudaSetDevice(1); ponger<SLEEP><<<1, 1>>>(f1, f0, n);
  cudaSetDevice(0); pinger<SLEEP><<<1, 1>>>(f0, f1, n, t);
  cudaDeviceSynchronize();
  cudaSetDevice(1); cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaSetDevice(0); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  return double(h) / n / 2.0;  // ns per one-way hop
}

int main() {
  int nd = 0; cudaGetDeviceCount(&nd);
  if (nd < 2) { printf("{\"error\": \"needs 2 GPUs\"}\n"); return 0; }
  uint32_t *f0, *f1; unsigned long long* t;
  cudaSetDevice(0); cudaDeviceEnablePeerAccess(1, 0); cudaMalloc(&f0, 256); cudaMalloc(&t, 8);
  cudaSetDevice(1); cudaDeviceEnablePeerAccess(0, 0); cudaMalloc(&f1, 256);
  const int n = 20000;
  run<false>(f0, f1, t, 100);
  double a = run<false>(f0, f1, t, n);
  double b = run<true>(f0, f1, t, n);
  printf("{\"one_way_ns_spin\": %.0f, \"one_way_ns_nanosleep32\": %.0f, \"status\": \"%s\"}\n", a, b,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
