// NVLink 5 peer-transfer ceilings on B200 for the transport design choices
// (single process, GPU0 <-> GPU1, peer access enabled):
//   pull_ldg   GPU1 kernel: 16-B LDG from GPU0 memory -> 16-B STG local
//   pull_bulk  GPU1 kernel: cp.async.bulk GPU0 -> smem (mbarrier) -> STG local
//   push_stg   GPU0 kernel: 16-B LDG local -> 16-B STG into GPU1 memory
//   push_bulk  GPU0 kernel: LDG local -> smem -> cp.async.bulk smem -> GPU1 memory
//   ce_peer    cudaMemcpyPeerAsync (copy engines)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/nvlink_bench tools/nvlink_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void copy_ldg(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x, st = size_t(gridDim.x) * blockDim.x;
  for (; i + 3 * st < n; i += 4 * st) {
    uint4 a = src[i], b = src[i + st], c = src[i + 2 * st], d = src[i + 3 * st];
    dst[i] = a; dst[i + st] = b; dst[i + 2 * st] = c; dst[i + 3 * st] = d;
  }
  for (; i < n; i += st) dst[i] = src[i];
}

__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

// pull: one thread issues bulk loads of CH bytes into a 4-stage ring, the block stores
template <int CH>
__global__ void __launch_bounds__(256) pull_bulk(const char* src, char* dst, size_t n_chunks) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[4];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t k = 0;
  auto issue = [&](size_t c, int st) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(smem + st * CH)), "l"(src + c * CH), "r"(CH), "r"(sa(&full[st])) : "memory");
  };
  size_t c0 = blockIdx.x;
  if (threadIdx.x == 0)
    for (int j = 0; j < 3; ++j) if (c0 + j * gridDim.x < n_chunks) issue(c0 + j * gridDim.x, j);
  for (size_t c = c0; c < n_chunks; c += gridDim.x, ++k) {
    const int st = k % 4;
    const size_t nx = c + 3 * size_t(gridDim.x);
    if (threadIdx.x == 0 && nx < n_chunks) issue(nx, (k + 3) % 4);
    asm volatile("{.reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=;}"
                 ::"r"(sa(&full[st])), "r"((k / 4) & 1) : "memory");
    const uint4* s4 = reinterpret_cast<const uint4*>(smem + st * CH);
    uint4* d4 = reinterpret_cast<uint4*>(dst + c * CH);
    for (int i = threadIdx.x; i < CH / 16; i += blockDim.x) d4[i] = s4[i];
    __syncthreads();
  }
}

// push: block loads CH bytes into smem, one thread bulk-stores them to the peer
template <int CH>
__global__ void __launch_bounds__(256) push_bulk(const char* src, char* dst, size_t n_chunks) {
  extern __shared__ __align__(128) char smem[];
  uint32_t k = 0;
  for (size_t c = blockIdx.x; c < n_chunks; c += gridDim.x, ++k) {
    char* buf = smem + (k & 1) * CH;
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // buffer free
    __syncthreads();
    const uint4* s4 = reinterpret_cast<const uint4*>(src + c * CH);
    uint4* b4 = reinterpret_cast<uint4*>(buf);
    for (int i = threadIdx.x; i < CH / 16; i += blockDim.x) b4[i] = s4[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * CH),
                   "r"(sa(buf)), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename F>
float timeit(int dev, F f) {
  cudaSetDevice(dev);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const size_t bytes = size_t(1) << 30;  // 1 GiB per direction
  int n = 0; cudaGetDeviceCount(&n);
  if (n < 2) { printf("{\"error\": \"needs 2 GPUs\"}\n"); return 0; }
  char *g0a, *g0b, *g1a, *g1b;
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0)); CK(cudaMalloc(&g0a, bytes)); CK(cudaMalloc(&g0b, bytes));
  CK(cudaMemset(g0a, 1, bytes));
  CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0)); CK(cudaMalloc(&g1a, bytes)); CK(cudaMalloc(&g1b, bytes));
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  constexpr int CH = 16384;
  cudaSetDevice(1); cudaFuncSetAttribute(pull_bulk<CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * CH);
  cudaSetDevice(0); cudaFuncSetAttribute(push_bulk<CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * CH);
  const size_t n16 = bytes / 16, nch = bytes / CH;
  struct R { const char* name; float ms; } r[8];
  r[0] = {"pull_ldg (GPU1 LDG.128 from GPU0)", timeit(1, [&] { copy_ldg<<<sms * 8, 256>>>((const uint4*)g0a, (uint4*)g1a, n16); })};
  r[1] = {"pull_bulk (GPU1 cp.async.bulk from GPU0, 16 KB)", timeit(1, [&] { pull_bulk<CH><<<sms * 2, 256, 4 * CH>>>(g0a, g1a, nch); })};
  r[2] = {"push_stg (GPU0 STG.128 into GPU1)", timeit(0, [&] { copy_ldg<<<sms * 8, 256>>>((const uint4*)g0a, (uint4*)g1b, n16); })};
  r[3] = {"push_bulk (GPU0 cp.async.bulk store into GPU1, 16 KB)", timeit(0, [&] { push_bulk<CH><<<sms * 2, 256, 2 * CH>>>(g0a, g1b, nch); })};
  r[4] = {"ce_peer (cudaMemcpyPeerAsync GPU0 -> GPU1)", timeit(0, [&] { cudaMemcpyPeerAsync(g1b, 1, g0a, 0, bytes, 0); })};
  r[5] = {"ce_pull (cudaMemcpyPeerAsync issued on GPU1, GPU0 -> GPU1)", timeit(1, [&] { cudaMemcpyPeerAsync(g1b, 1, g0a, 0, bytes, 0); })};
  r[6] = {"ce_pull_default (cudaMemcpyAsync Default on GPU1, GPU0 -> GPU1)", timeit(1, [&] { cudaMemcpyAsync(g1b, g0a, bytes, cudaMemcpyDefault, 0); })};
  r[7] = {"ce_pull_samedev (cudaMemcpyPeerAsync(dst,1,src,1) on GPU1)", timeit(1, [&] { cudaMemcpyPeerAsync(g1b, 1, g0a, 1, bytes, 0); })};
  for (auto& x : r) printf("{\"path\": \"%s\", \"ms\": %.4f, \"GBps\": %.1f}\n", x.name, x.ms, bytes / (x.ms * 1e-3) / 1e9);
  cudaError_t e = cudaGetLastError();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
