// HBM ceiling for the hand-off kernels' traffic mixes (B200, sm_100a).
// Streams N bytes in and N*ratio bytes out with 256-bit accesses and no math,
// to tell how close K1 (read 4 : write 1) and K3 (read 1 : write 4) are to
// what the memory system delivers for THAT mix (the MEASURED_PEAKS copy is
// 1 : 1).   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/membench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct __align__(32) V8 { uint32_t v[8]; };

__device__ __forceinline__ V8 ld(const V8* p) {
  V8 r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]),
                 "=r"(r.v[5]), "=r"(r.v[6]), "=r"(r.v[7]) : "l"(p));
  return r;
}
__device__ __forceinline__ void st(V8* p, const V8& r) {
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
               "r"(r.v[0]), "r"(r.v[1]), "r"(r.v[2]), "r"(r.v[3]), "r"(r.v[4]), "r"(r.v[5]),
               "r"(r.v[6]), "r"(r.v[7]) : "memory");
}

// in_per_out: how many input vectors per output vector (4 = K1-like, 1 = copy);
// out_per_in: outputs per input (4 = K3-like)
template <int IN, int OUT, int U>
__global__ void __launch_bounds__(256) mix(const V8* __restrict__ in, V8* __restrict__ out, int64_t n_units) {
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  for (int64_t u0 = tid; u0 < n_units; u0 += nth * U) {
    V8 a[U][IN];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = u0 + k * nth;
      if (u < n_units)
#pragma unroll
        for (int i = 0; i < IN; ++i) a[k][i] = ld(in + u * IN + i);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = u0 + k * nth;
      if (u < n_units) {
        V8 r = a[k][0];
#pragma unroll
        for (int i = 1; i < IN; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) r.v[j] ^= a[k][i].v[j];
#pragma unroll
        for (int o = 0; o < OUT; ++o) st(out + u * OUT + o, r);
      }
    }
  }
}

template <int IN, int OUT>
void run(const char* name, V8* in, V8* out, int64_t in_bytes) {
  const int64_t units = in_bytes / (32 * IN);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto k = mix<IN, OUT, 2>;
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, 0);
  dim3 grid(sms * per);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<<<grid, 256>>>(in, out, units);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    k<<<grid, 256>>>(in, out, units);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double bytes = double(units) * 32 * (IN + OUT);
  printf("{\"mix\": \"%s\", \"read_GB\": %.3f, \"write_GB\": %.3f, \"ms\": %.4f, \"GBps\": %.1f}\n", name,
         units * 32.0 * IN / 1e9, units * 32.0 * OUT / 1e9, best, bytes / (best * 1e-3) / 1e9);
}

int main() {
  const int64_t in_bytes = int64_t(8) << 30;  // 8 GiB read side (like K1's fp16 input)
  V8 *in, *out;
  if (cudaMalloc(&in, in_bytes) != cudaSuccess || cudaMalloc(&out, in_bytes) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(in, 1, in_bytes);
  run<1, 1>("copy 1:1", in, out, in_bytes);
  run<4, 1>("K1-like read 4 : write 1", in, out, in_bytes);
  run<1, 0>("read only", in, out, in_bytes);
  // K3-like: read 1 : write 4 (input 1/4 of the output)
  run<1, 4>("K3-like read 1 : write 4", in, out, in_bytes / 4);
  cudaError_t e = cudaGetLastError();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
