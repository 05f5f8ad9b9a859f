// HBM ceiling for the hand-off kernels' traffic mixes (B200, sm_100a).
// Streams N bytes in and N*ratio bytes out with 256-bit accesses and no math,
// to tell how close K1 (read 4 : write 1) and K3 (read 1 : write 4) are to
// what the memory system delivers for THAT mix (the MEASURED_PEAKS copy is
// 1 : 1).  Round 2 adds the store flavours K3 could use: plain 256-bit
// stores, streaming (.cs) stores, and TMA bulk stores from shared memory
// (cp.async.bulk.global.shared::cta), plus a pure-write line per flavour.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/membench.cu -o tools/membench
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
template <bool CS>
__device__ __forceinline__ void st(V8* p, const V8& r) {
  if (CS)
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r.v[0]),
                 "r"(r.v[1]), "r"(r.v[2]), "r"(r.v[3]), "r"(r.v[4]), "r"(r.v[5]), "r"(r.v[6]),
                 "r"(r.v[7]) : "memory");
  else
    asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "r"(r.v[0]), "r"(r.v[1]), "r"(r.v[2]), "r"(r.v[3]), "r"(r.v[4]), "r"(r.v[5]),
                 "r"(r.v[6]), "r"(r.v[7]) : "memory");
}

// IN input vectors -> OUT output vectors per unit; IN == 0: pure write;
// OUT == 0: pure read (the XOR is kept live by a never-true store)
template <int IN, int OUT, int U, bool CS>
__global__ void __launch_bounds__(256) mix(const V8* __restrict__ in, V8* __restrict__ out,
                                            int64_t n_units, uint32_t magic) {
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (int64_t u0 = tid; u0 < n_units; u0 += nth * U) {
    V8 a[U][IN > 0 ? IN : 1];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = u0 + k * nth;
      if (IN == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[k][0].v[j] = uint32_t(u) + j;
      } else if (u < n_units) {
#pragma unroll
        for (int i = 0; i < IN; ++i) a[k][i] = ld(in + u * IN + i);
      }
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
        if (OUT == 0) {
#pragma unroll
          for (int j = 0; j < 8; ++j) acc ^= r.v[j];
        }
#pragma unroll
        for (int o = 0; o < OUT; ++o) st<CS>(out + u * OUT + o, r);
      }
    }
  }
  if (OUT == 0 && acc == magic) out[tid].v[0] = acc;
}

// TMA bulk-store flavour: each CTA expands its input rows (ROW bytes of
// output each, IN:OUT as above) into a shared-memory ring of STAGES rows and
// one thread stores each finished row with cp.async.bulk.global.shared::cta.
template <int IN, int OUT, int ROW, int STAGES>
__global__ void __launch_bounds__(256) mix_tma(const V8* __restrict__ in, V8* __restrict__ out,
                                                int64_t n_rows) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int kOutVec = ROW / 32;             // output vectors per row
  constexpr int kInVec = kOutVec * IN / OUT;    // input vectors per row (IN may be 0)
  int slot = 0;
  for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
    V8* buf = reinterpret_cast<V8*>(smem + size_t(slot) * ROW);
    // the stage about to be overwritten must have been read by its bulk store
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
    __syncthreads();
    for (int v = threadIdx.x; v < kOutVec; v += blockDim.x) {
      V8 x;
      if (IN == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x.v[j] = uint32_t(r) + v + j;
      } else {
        x = ld(in + r * kInVec + v * IN / OUT);
      }
      buf[v] = x;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + r * kOutVec),
                   "r"(s), "n"(ROW) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    slot = slot + 1 == STAGES ? 0 : slot + 1;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename K, typename... A>
float time_best(K k, dim3 grid, int smem, A... args) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<<<grid, 256, smem>>>(args...);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    k<<<grid, 256, smem>>>(args...);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

static void report(const char* name, const char* how, double rd, double wr, float ms) {
  printf("{\"mix\": \"%s\", \"how\": \"%s\", \"read_GB\": %.3f, \"write_GB\": %.3f, \"ms\": %.4f, "
         "\"GBps\": %.1f}\n",
         name, how, rd / 1e9, wr / 1e9, ms, (rd + wr) / (ms * 1e-3) / 1e9);
  fflush(stdout);
}

static int sms() {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0);
  return n;
}

template <int IN, int OUT, bool CS>
void run(const char* name, V8* in, V8* out, int64_t units) {
  auto k = mix<IN, OUT, 2, CS>;
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, 0);
  const float ms = time_best(k, dim3(sms() * per), 0, (const V8*)in, out, units, 0x9e3779b9u);
  report(name, CS ? "st.global.cs.v8" : "st.global.v8", units * 32.0 * IN, units * 32.0 * OUT, ms);
}

template <int IN, int OUT, int ROW, int STAGES>
void run_tma(const char* name, V8* in, V8* out, int64_t out_bytes) {
  auto k = mix_tma<IN, OUT, ROW, STAGES>;
  const int smem = ROW * STAGES;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, smem);
  const int64_t rows = out_bytes / ROW;
  const float ms = time_best(k, dim3(sms() * per), smem, (const V8*)in, out, rows);
  char how[96];
  snprintf(how, sizeof how, "cp.async.bulk store, %d B rows x %d stages, %d CTA/SM", ROW, STAGES, per);
  report(name, how, double(rows) * ROW * IN / (OUT ? OUT : 1), double(rows) * ROW, ms);
}

int main() {
  const int64_t bytes = int64_t(8) << 30;  // 8 GiB: far above the 126 MB L2
  V8 *in, *out;
  if (cudaMalloc(&in, bytes) != cudaSuccess || cudaMalloc(&out, bytes) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(in, 1, bytes);
  cudaMemset(out, 0, bytes);
  const int64_t v = bytes / 32;
  run<1, 1, false>("copy 1:1", in, out, v);
  run<1, 1, true>("copy 1:1", in, out, v);
  run<4, 1, false>("K1-like read 4 : write 1", in, out, v / 4);
  run<4, 1, true>("K1-like read 4 : write 1", in, out, v / 4);
  run<1, 0, false>("read only", in, out, v);
  run<0, 1, false>("write only", in, out, v);
  run<0, 1, true>("write only", in, out, v);
  run<1, 4, false>("K3-like read 1 : write 4", in, out, v / 4);
  run<1, 4, true>("K3-like read 1 : write 4", in, out, v / 4);
  run_tma<0, 1, 8192, 4>("write only", in, out, bytes);
  run_tma<0, 1, 8192, 8>("write only", in, out, bytes);
  run_tma<0, 1, 16384, 4>("write only", in, out, bytes);
  run_tma<1, 4, 8192, 4>("K3-like read 1 : write 4", in, out, bytes);
  run_tma<1, 4, 8192, 8>("K3-like read 1 : write 4", in, out, bytes);
  run_tma<1, 4, 16384, 4>("K3-like read 1 : write 4", in, out, bytes);
  run_tma<1, 4, 4096, 8>("K3-like read 1 : write 4", in, out, bytes);
  run_tma<1, 1, 8192, 4>("copy 1:1", in, out, bytes);
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
