// C-ABI of the B200 KV hand-off library (see include/kvx.h for the contract).
//
// Host side only: argument validation, launch geometry, dispatch on
// (bits, group), and the transport primitives (peer access, IPC mapping,
// stream-ordered doorbells).  Device code lives in kvx_kernels.cuh.
#include <cuda.h>  // driver API types only; entry points resolved at run time
#include <cuda_runtime.h>

#include <atomic>
#include <dlfcn.h>
#include <nccl.h>  // types only: the entry points are resolved at run time (dlopen)

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <map>
#include <mutex>
#include <tuple>

#include "../../include/kvx.h"
#include "kvx_kernels.cuh"
#include "kvx_kivi.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kWarpsPerBlock = kThreads / 32;
constexpr int kMaxDev = 64;

// Per-device / per-kernel launch facts, queried once and shared by every host
// thread (kvx.h promises re-entrancy): atomics for the SM counts, a mutex for
// the occupancy and shared-memory-attribute caches.
int sm_count(int dev) {
  static std::atomic<int> cache[kMaxDev];
  if (dev < 0 || dev >= kMaxDev) return 148;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (!n) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;
    }
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

std::mutex g_cache_mu;
std::map<std::tuple<int, const void*, int, int>, int> g_occupancy;  // (dev, fn, threads, smem)
std::map<std::pair<int, const void*>, int> g_smem_attr;            // (dev, fn) -> bytes set


int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

template <typename K>
int blocks_per_sm(K kernel, int threads = kThreads, int smem = 0) {
  const auto key = std::make_tuple(current_device(), reinterpret_cast<const void*>(kernel), threads, smem);
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_occupancy.find(key);
    if (it != g_occupancy.end()) return it->second;
  }
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem) != cudaSuccess || b <= 0) {
    cudaGetLastError();
    b = 1;
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_occupancy[key] = b;
  return b;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel)
// -- not a stream op, so it never lands inside a graph capture.
template <typename K>
cudaError_t ensure_smem_attr(K kernel, int bytes) {
  const auto key = std::make_pair(current_device(), reinterpret_cast<const void*>(kernel));
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_smem_attr.find(key);
  if (it != g_smem_attr.end() && it->second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) g_smem_attr[key] = bytes;
  return e;
}

// Persistent-style grid: enough warps to cover every token row once, capped at
// the number of CTAs the SMs hold concurrently (a multiple of the SM count).
template <typename K>
dim3 grid_for(K kernel, int64_t n_token_rows) {
  const int64_t full = int64_t(sm_count(current_device())) * blocks_per_sm(kernel);
  const int64_t need = (n_token_rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
  int64_t g = need < full ? need : full;
  if (g < 1) g = 1;
  return dim3(unsigned(g));
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int valid_format(int head_dim, int group, int bits) {
  if (head_dim <= 0 || head_dim % 8) return KVX_ERR_INVALID_ARG;
  if (bits == 16) return KVX_OK;
  if (bits != 2 && bits != 4 && bits != 8) return KVX_ERR_INVALID_ARG;
  if (group != 32 && group != 64 && group != 128) return KVX_ERR_INVALID_ARG;
  if (head_dim % group) return KVX_ERR_INVALID_ARG;
  return KVX_OK;
}

int make_geo(kvx::Geo& g, const void* k, const void* v, int64_t layer_stride, const int64_t* slots,
             int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim, int group, int bits,
             int64_t payload_layer_stride, int planes = 2, int plane0 = 0, int plane_heads = 0,
             int head_offset = 0) {
  if (n_layers < 0 || n_tokens < 0 || n_heads <= 0) return KVX_ERR_INVALID_ARG;
  if (plane_heads == 0) plane_heads = n_heads;
  if (head_offset < 0 || head_offset + n_heads > plane_heads) return KVX_ERR_INVALID_ARG;
  g.plane_row_b = int64_t(plane_heads) * head_dim * 2;
  g.head_off_b = int64_t(head_offset) * head_dim * 2;
#ifdef KVX_DEBUG
  g.dbg_rows = (layer_stride > 0 && g.plane_row_b > 0) ? layer_stride * 2 / g.plane_row_b : 0;
#endif
  if (g.head_off_b % 32 || g.plane_row_b % 32) {
    if (n_layers > 0 && n_tokens > 0 && (g.head_off_b % 16 || g.plane_row_b % 16))
      return KVX_ERR_INVALID_ARG;
  }
  const int64_t row_elems = int64_t(n_heads) * head_dim;
  if (row_elems > (int64_t(1) << 30)) return KVX_ERR_INVALID_ARG;
  if (n_layers > 0 && n_tokens > 0) {
    if (!k || !v || !aligned(k, 16) || !aligned(v, 16)) return KVX_ERR_INVALID_ARG;
    if ((layer_stride * 2) % 16) return KVX_ERR_INVALID_ARG;
  }
  g.k_plane = static_cast<const char*>(k);
  g.v_plane = static_cast<const char*>(v);
  g.layer_stride_b = layer_stride * 2;
  g.slots = slots;
  g.n_tokens = n_tokens;
  g.planes = planes;
  g.plane0 = plane0;
  g.n_token_rows = n_layers * planes * n_tokens;
  g.row_elems = int(row_elems);
  g.vecs = int(row_elems / 8);
  // Payload layer strides: dense per-array layout when payload_layer_stride == 0,
  // else one segment per layer holding [codes | scale | zero].
  const int64_t rows_per_layer = planes * n_tokens * n_heads;
  const int64_t ng = bits == 16 ? 0 : head_dim / group;
  if (payload_layer_stride < 0) return KVX_ERR_INVALID_ARG;
  if (payload_layer_stride == 0) {
    g.codes_ls = rows_per_layer * head_dim * bits / 8;
    g.meta_ls = rows_per_layer * ng * 2;
  } else {
    // 8-bit codes move as 32-byte vectors (st/ld.global.v8.b32): the layer
    // stride must keep every layer's codes 32-byte aligned
    if (payload_layer_stride % (bits == 8 ? 32 : 16)) return KVX_ERR_INVALID_ARG;
    g.codes_ls = payload_layer_stride;
    g.meta_ls = payload_layer_stride;
  }
  return KVX_OK;
}

constexpr int kUnroll = 4;

kvx::FastDiv make_fastdiv(uint32_t d) {
  kvx::FastDiv f;
  f.d = d ? d : 1;
  uint32_t s = 0;
  while ((uint64_t(1) << s) < f.d) ++s;
  f.s = s;
  f.m = uint32_t(((uint64_t(1) << 32) * ((uint64_t(1) << s) - f.d)) / f.d + 1);
  return f;
}

// Item geometry shared by K1 and K3: one item = one token row's block of up
// to 32 chunks of 32 elements; one warp per item at a time.
cudaError_t make_items(const kvx::Geo& g, kvx::ItemGeo& ig) {
  ig.cpr = g.row_elems / 32;
  const uint32_t ipr = uint32_t((ig.cpr + 31) / 32);
  int64_t n_items = g.n_token_rows * ipr;
  ig.rpi_shift = 0;
  ig.cpr_shift = 0;
  ig.pt = 0;
  ig.ipl = make_fastdiv(1);
  if (ig.cpr > 0 && ig.cpr < 32 && (32 % ig.cpr) == 0 && g.n_tokens > 0) {
    // short rows: pack 32 / cpr rows of one layer into each item
    while ((1 << ig.cpr_shift) < ig.cpr) ++ig.cpr_shift;
    ig.rpi_shift = 5 - ig.cpr_shift;
    const int64_t pt = int64_t(g.planes) * g.n_tokens;
    const int64_t ipl = (pt + (int64_t(1) << ig.rpi_shift) - 1) >> ig.rpi_shift;
    if (pt >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    ig.pt = uint32_t(pt);
    ig.ipl = make_fastdiv(uint32_t(ipl));
    n_items = (g.n_token_rows / pt) * ipl;
  }
  if (n_items >= (int64_t(1) << 31) || g.n_tokens >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  ig.ipr = make_fastdiv(ipr);
  ig.tokens = make_fastdiv(uint32_t(g.n_tokens));
  ig.n_items = uint32_t(n_items);
  return cudaSuccess;
}

#ifdef KVX_TRACE
// trace builds: the epoch of the pair hand-off being launched on this thread
thread_local uint32_t g_trace_epoch = 0;
#endif

// Doorbell request for kvx_quant_pack_signal (null peer_flags = plain K1).
struct SignalReq {
  uint32_t* counters = nullptr;
  uint32_t* peer_flags = nullptr;
  uint32_t ready_value = 0;
  const uint32_t* free_flag = nullptr;
  uint32_t free_value = 0;
  kvx::Ctl* ctl = nullptr;
  int layers_per_chunk = 1;
  int64_t n_layers = 0;
  bool pdl = false;  // programmatic dependent launch behind the stream's previous kernel
};

// K1 with TMA-staged source rows (quant_pack_bulk_kernel) is the default; the
// register-prefetch K1 remains for rows a stage cannot hold and as the A/B
// baseline (-DKVX_K1_BULK=0, or KVX_K1_REG=1 at run time).  Stage geometry A/B
// (N=1 config 2, K1 ms; profiles/r02_k1bulk.md): register K1 1.814; bulk
// 4 x 16 KB 2.20 (before hoisting) / 1.985, 6 x 8 KB 2.91, 4 x 24 KB 1.773,
// 3 x 32 KB 1.678, 4 x 32 KB (1 CTA/SM) 2.157, 2 x 40 KB 1.607,
// 2 x 48 KB 1.600 (2 CTAs/SM: 192 KB of source rows in flight per SM).
#ifndef KVX_K1_BULK
#define KVX_K1_BULK 1
#endif
#ifndef KVX_K1B_STAGES
#define KVX_K1B_STAGES 2
#endif
#ifndef KVX_K1B_STAGE_BYTES
#define KVX_K1B_STAGE_BYTES 49152
#endif

// K1-bulk launch (see quant_pack_bulk_kernel); *ok = false: shape not staged.
template <int BITS, int G>
cudaError_t launch_quant_bulk(const kvx::Geo& g, void* codes, void* scale, void* zero,
                              cudaStream_t s, const SignalReq& rq, bool* ok) {
  *ok = false;
  constexpr int kStages = KVX_K1B_STAGES;
  const int row_bytes = g.row_elems * 2;
  if (g.n_tokens < 1 || g.row_elems % 32 || row_bytes > KVX_K1B_STAGE_BYTES) return cudaSuccess;
  kvx::K1BulkGeo kb;
  int64_t r = KVX_K1B_STAGE_BYTES / row_bytes;
  if (r > g.n_tokens) r = g.n_tokens;
  kb.rows_per_span = int(r);
  kb.spans_per_plane = int((g.n_tokens + r - 1) / r);
  const int64_t n_layers = g.n_token_rows / (int64_t(g.planes) * g.n_tokens);
  const int64_t n_spans = n_layers * g.planes * kb.spans_per_plane;
  if (n_spans >= (int64_t(1) << 31)) return cudaSuccess;
  kb.n_spans = uint32_t(n_spans);
  kb.row_bytes = row_bytes;
  kb.stage_bytes = kb.rows_per_span * row_bytes;
  kb.cpr = g.row_elems / 32;
  kb.contiguous = (g.slots == nullptr && g.plane_row_b == row_bytes) ? 1 : 0;
  kb.spans_per_chunk = uint32_t(int64_t(rq.layers_per_chunk > 0 ? rq.layers_per_chunk : 1) *
                                g.planes * kb.spans_per_plane);
  kvx::SignalGeo sig = {};
  sig.counters = rq.counters;
  sig.peer_flags = rq.peer_flags;
  sig.ready_value = rq.ready_value;
  sig.free_flag = rq.free_flag;
  sig.free_value = rq.free_value;
  sig.ctl = rq.ctl;
#ifdef KVX_TRACE
  sig.trace_id = g_trace_epoch;
#endif
  if (rq.peer_flags && (n_spans + kb.spans_per_chunk - 1) / kb.spans_per_chunk > kvx::kMaxSignalChunks)
    return cudaErrorInvalidValue;
  const int smem = kStages * kb.stage_bytes;
  auto k = kvx::quant_pack_bulk_kernel<BITS, G, kStages>;
  cudaError_t attr = ensure_smem_attr(k, kStages * KVX_K1B_STAGE_BYTES);
  if (attr != cudaSuccess) return attr;
  constexpr int kThreadsB = 288;  // 8 consumer warps + the producer warp
  int per_sm = blocks_per_sm(k, kThreadsB, smem);
  int64_t grid = int64_t(sm_count(current_device())) * (per_sm > 0 ? per_sm : 1);
  if (grid > n_spans) grid = n_spans;
  *ok = true;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(kThreadsB);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = rq.pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, g, kb, static_cast<uint8_t*>(codes),
                            static_cast<__half*>(scale), static_cast<__half*>(zero), sig);
}

template <int BITS, int G>
cudaError_t launch_quant(const kvx::Geo& g, void* codes, void* scale, void* zero, cudaStream_t s,
                         const SignalReq& rq = SignalReq()) {
  static const bool bulk = KVX_K1_BULK ? std::getenv("KVX_K1_REG") == nullptr
                                       : std::getenv("KVX_K1_BULK") != nullptr;
  if (bulk) {
    bool ok = false;
    cudaError_t e = launch_quant_bulk<BITS, G>(g, codes, scale, zero, s, rq, &ok);
    if (e != cudaSuccess || ok) return e;
  }
  kvx::ItemGeo ig;
  cudaError_t e = make_items(g, ig);
  if (e != cudaSuccess) return e;
  kvx::SignalGeo sig;
  sig.counters = rq.counters;
  sig.peer_flags = rq.peer_flags;
  sig.items_per_chunk = 1;
  sig.ipc = make_fastdiv(1);
  sig.ready_value = rq.ready_value;
  sig.free_flag = rq.free_flag;
  sig.free_value = rq.free_value;
  sig.ctl = rq.ctl;
#ifdef KVX_TRACE
  sig.trace_id = g_trace_epoch;
#endif
  if (rq.peer_flags) {
    const int64_t per_layer = ig.n_items / (rq.n_layers > 0 ? rq.n_layers : 1);
    const int64_t ipc = per_layer * rq.layers_per_chunk;
    if (ipc <= 0 || ipc >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    sig.items_per_chunk = uint32_t(ipc);
    sig.ipc = make_fastdiv(uint32_t(ipc));
    const int64_t n_chunks = (ig.n_items + ipc - 1) / ipc;
    if (n_chunks > kvx::kMaxSignalChunks) return cudaErrorInvalidValue;
    // (the counters are zero between launches: each chunk's last arrival resets its own)
  }
  auto k = kvx::quant_pack_kernel<BITS, G>;
  if (!rq.pdl) {
    k<<<grid_for(k, ig.n_items), kThreads, 0, s>>>(g, ig, static_cast<uint8_t*>(codes),
                                                   static_cast<__half*>(scale),
                                                   static_cast<__half*>(zero), sig);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid_for(k, ig.n_items);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, g, ig, static_cast<uint8_t*>(codes),
                            static_cast<__half*>(scale), static_cast<__half*>(zero), sig);
}

template <int BITS, int G>
cudaError_t launch_dequant(const kvx::Geo& g, const void* codes, const void* scale,
                           const void* zero, cudaStream_t s) {
  kvx::ItemGeo ig;
  cudaError_t e = make_items(g, ig);
  if (e != cudaSuccess) return e;
  auto k = ig.rpi_shift ? kvx::dequant_scatter_kernel<BITS, G, true>
                        : kvx::dequant_scatter_kernel<BITS, G, false>;
  k<<<grid_for(k, ig.n_items), kThreads, 0, s>>>(g, ig, static_cast<const uint8_t*>(codes),
                                                 static_cast<const __half*>(scale),
                                                 static_cast<const __half*>(zero));
  return cudaGetLastError();
}

#ifndef KVX_BULK_STAGES
#define KVX_BULK_STAGES 4
#endif
#ifndef KVX_BULK_STAGE_BYTES
#define KVX_BULK_STAGE_BYTES 12288
#endif
constexpr int kBulkStages = KVX_BULK_STAGES;

constexpr int kBulkThreads = 288;
// code bytes per stage: 4 x 12 KB in flight per SM.  A/B at one CTA per SM
// (N=2, GB/s fp16-eq, cfg3 / cfg4 pair): 8 KB 2,833 / 2,867; 12 KB 2,945 /
// 2,903; 16 KB 2,947 / 2,865; 32 KB 2,758 / 2,629; 6 x 16 KB 2,707 / 2,604.
constexpr int kBulkStageTarget = KVX_BULK_STAGE_BYTES;
#ifndef KVX_PULL_PER_SM
#define KVX_PULL_PER_SM 1
#endif
constexpr int kPullCtasPerSm = KVX_PULL_PER_SM;  // bulk-pull CTAs per SM (A/B: -DKVX_PULL_PER_SM)
// 2-bit pulls write 8 fp16 bytes per payload byte (4 at 4-bit): at link speed
// eight consumer warps per SM cannot keep up, so they run 3 CTAs per SM
// (N=2 config-4 pair, GB/s fp16-eq: 1 CTA 3,707, 2 CTAs 4,101-4,314, 3 CTAs
// 4,336; config 3: 4,102 / 4,299-4,365 / 4,314.  4- and 8-bit lose 3 % and
// 2 % with 2 CTAs; profiles/r02_bench/pull_2bit_n2.log, val2_n2.log)
#ifndef KVX_PULL_PER_SM_2BIT
#define KVX_PULL_PER_SM_2BIT 3
#endif
template <int BITS>
constexpr int pull_ctas_per_sm() { return BITS == 2 ? KVX_PULL_PER_SM_2BIT : kPullCtasPerSm; }

// K3-bulk on a LOCAL payload (no doorbells: N=1 hand-offs, the decode side of
// push / copy): HBM feeds the stages, not the link, so the consumers' fp16
// stores bound it and it wants more CTAs per SM and larger stages than a
// pull, and its spans are whole passes of the consumer warps (a 6-row span
// leaves 2 of 8 warps idle).  N=1 sweep (r02_bench/k3_local_geo_n1.log), K3 ms
// at 1 CTA per SM, 16 / 24 / 32 KB stages: config 2 1.834 / 1.837 / 1.749,
// 2-bit 1.547 / 1.562 / 1.545, 13B 2.732 / 2.734 / 2.731; 2 CTAs per SM equal
// or slower.  KVX_LOCAL_PULL_PER_SM / _STAGE_BYTES / _ROW_ALIGN override.
int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : dflt;
}
#ifndef KVX_LOCAL_PULL_PER_SM
#define KVX_LOCAL_PULL_PER_SM 1
#endif
#ifndef KVX_LOCAL_STAGE_BYTES
#define KVX_LOCAL_STAGE_BYTES 32768
#endif
int local_pull_ctas_per_sm() {
  static const int v = env_int("KVX_LOCAL_PULL_PER_SM", KVX_LOCAL_PULL_PER_SM);
  return v < 1 ? 1 : v;
}
int local_row_align() {
  static const int v = env_int("KVX_LOCAL_ROW_ALIGN", 1);
  return v;
}
int local_stage_target() {
  static const int v = env_int("KVX_LOCAL_STAGE_BYTES", KVX_LOCAL_STAGE_BYTES);
  return v < 1024 ? 1024 : v;
}

// Smallest row count whose code and metadata bytes are both 16-byte multiples.
int64_t bulk_row_multiple(int64_t code_row_bytes, int64_t meta_row_bytes) {
  auto need = [](int64_t b) {
    int64_t k = 1;
    while ((k * b) % 16) k *= 2;
    return k;
  };
  const int64_t a = need(code_row_bytes), b = need(meta_row_bytes);
  return a > b ? a : b;  // powers of two: the max is the lcm
}

struct PullDone {  // optional in-kernel completion of a pull hand-off
  uint32_t* done_counter = nullptr;
  uint32_t* peer_free = nullptr;
  bool chained = false;  // KVX_PULL_CHAINED: consumers skip the up-front PDL wait
};

// Span geometry of a K3-bulk pull (false: not bulk-stageable).
template <int BITS, int G>
bool plan_pull(const kvx::Geo& g, const void* codes, const void* scale, const void* zero,
               const uint32_t* ready, uint32_t ready_value, int layers_per_chunk,
               const PullDone& done, kvx::Ctl* ctl, kvx::BulkGeo& bg) {
  bg = kvx::BulkGeo{};
  bg.ready = ready;
  bg.ready_value = ready_value;
  bg.done_counter = done.done_counter;
  bg.peer_free = done.peer_free;
  bg.chained = done.chained ? 1 : 0;
  bg.ctl = ctl;
#ifdef KVX_TRACE
  bg.trace_id = g_trace_epoch;
#endif
  bg.layers_per_chunk = layers_per_chunk > 0 ? layers_per_chunk : 1;
  bg.code_row_bytes = int(int64_t(g.row_elems) * BITS / 8);
  bg.meta_row_bytes = int(int64_t(g.row_elems) / G * 2);
  bg.cpr = g.row_elems / 32;
  const int64_t two_t = int64_t(g.planes) * g.n_tokens;
  // every bulk copy (a span of R rows, or the layer's last partial span) must
  // be a multiple of 16 bytes at a 16-byte aligned offset
  const int64_t m = bulk_row_multiple(bg.code_row_bytes, bg.meta_row_bytes);
  if ((two_t * bg.code_row_bytes) % 16 || (two_t * bg.meta_row_bytes) % 16 ||
      !aligned(codes, 16) || !aligned(scale, 16) || !aligned(zero, 16) || g.codes_ls % 16 ||
      g.meta_ls % 16)
    return false;  // not bulk-copyable: caller falls back to the LDG kernel
  const int target = ready ? kBulkStageTarget : local_stage_target();
  int64_t unit = m;
  if (!ready && local_row_align()) {
    // local payload: the consumers bound the pull, so a span is a whole number
    // of passes of the 8 consumer warps (rpw rows per warp for short rows)
    const int64_t rpw = (bg.cpr < 32 && 32 % bg.cpr == 0) ? 32 / bg.cpr : 1;
    const int64_t w = 8 * rpw;  // powers of two: the max is the lcm
    unit = w > m ? w : m;
  }
  int64_t r = target / bg.code_row_bytes;
  r = r / unit * unit;
  if (r < unit) r = unit;
  if (r > two_t) r = two_t;
  bg.rows_per_span = int(r);
  bg.stage_bytes = bg.rows_per_span * (bg.code_row_bytes + 2 * bg.meta_row_bytes);
  if (kBulkStages * bg.stage_bytes > 200 * 1024) return false;
  bg.spans_per_layer = int((two_t + r - 1) / r);
  const int64_t n_layers = g.n_token_rows / two_t;
  const int64_t n_spans = n_layers * bg.spans_per_layer;
  if (n_spans >= (int64_t(1) << 31)) return false;
  bg.n_spans = uint32_t(n_spans);
  return true;
}

template <int BITS, int G>
cudaError_t launch_pull(const kvx::Geo& g, const void* codes, const void* scale, const void* zero,
                        cudaStream_t s, bool* ok, const uint32_t* ready, uint32_t ready_value,
                        int layers_per_chunk, const PullDone& done = PullDone(),
                        kvx::Ctl* ctl = nullptr, bool pdl = false) {
  *ok = false;
  kvx::BulkGeo bg;
  if (!plan_pull<BITS, G>(g, codes, scale, zero, ready, ready_value, layers_per_chunk, done, ctl,
                          bg))
    return cudaSuccess;
  const int smem = kBulkStages * bg.stage_bytes;
  const int64_t n_spans = bg.n_spans;
  auto k = kvx::pull_dequant_scatter_kernel<BITS, G, kBulkStages>;
  cudaError_t attr = ensure_smem_attr(k, 200 * 1024);
  if (attr != cudaSuccess) return attr;
  int per_sm = blocks_per_sm(k, kBulkThreads, smem);
  // ONE CTA per SM (4 stages x ~12 KB in flight each, ~7 MB device-wide):
  // enough to saturate the link, and measured faster than filling every SM
  // with as many CTAs as fit (cfg3 pair 2,948 vs 2,798 GB/s fp16-eq), while
  // leaving room on each SM for the decode GPU's own kernels -- and for the
  // next hand-off's pull, which PDL schedules next to this one
  // (tools/decode_interference.py: a concurrent HBM-bound round slows 1.96x
  // instead of 2.2x).
  const int want = ready ? pull_ctas_per_sm<BITS>() : local_pull_ctas_per_sm();
  per_sm = per_sm < want ? per_sm : want;
  int64_t grid = int64_t(sm_count(current_device())) * per_sm;
#ifdef KVX_PULL_MAX_CTAS
  if (grid > KVX_PULL_MAX_CTAS) grid = KVX_PULL_MAX_CTAS;
#endif
  if (grid > n_spans) grid = n_spans;
  *ok = true;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(kBulkThreads);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, g, bg, static_cast<const uint8_t*>(codes),
                            static_cast<const __half*>(scale), static_cast<const __half*>(zero));
}

template <int BITS>
cudaError_t dispatch_pull(int group, const kvx::Geo& g, const void* c, const void* sc,
                          const void* z, cudaStream_t s, bool* ok, const uint32_t* ready,
                          uint32_t rv, int lpc, const PullDone& done, kvx::Ctl* ctl, bool pdl) {
  switch (group) {
    case 32: return launch_pull<BITS, 32>(g, c, sc, z, s, ok, ready, rv, lpc, done, ctl, pdl);
    case 64: return launch_pull<BITS, 64>(g, c, sc, z, s, ok, ready, rv, lpc, done, ctl, pdl);
    default: return launch_pull<BITS, 128>(g, c, sc, z, s, ok, ready, rv, lpc, done, ctl, pdl);
  }
}

// K3-bulk over several queued hand-offs (kvx_pair_recv_many).  parts[i]
// carries the slot payload, doorbells, slot mapping and token count; the
// span geometry is filled in here.  *ok = false: not bulk-stageable.
template <int BITS, int G>
cudaError_t launch_pull_many(const kvx::Geo& g, int64_t n_layers, kvx::PullMany& pm,
                             cudaStream_t s, bool* ok, bool pdl) {
  *ok = false;
  pm.code_row_bytes = int(int64_t(g.row_elems) * BITS / 8);
  pm.meta_row_bytes = int(int64_t(g.row_elems) / G * 2);
  pm.cpr = g.row_elems / 32;
  const int64_t m = bulk_row_multiple(pm.code_row_bytes, pm.meta_row_bytes);
  int64_t max_two_t = 0;
  for (int i = 0; i < pm.count; ++i) {
    const kvx::PullPart& P = pm.part[i];
    const int64_t two_t = 2 * P.n_tokens;
    if (two_t < 1 || (two_t * pm.code_row_bytes) % 16 || (two_t * pm.meta_row_bytes) % 16 ||
        !aligned(P.codes, 16) || !aligned(P.scale, 16) || !aligned(P.zero, 16) ||
        P.payload_ls % 16)
      return cudaSuccess;
    max_two_t = two_t > max_two_t ? two_t : max_two_t;
  }
  int64_t r = kBulkStageTarget / pm.code_row_bytes;
  r = r / m * m;
  if (r < m) r = m;
  if (r > max_two_t) r = max_two_t;
  pm.stage_rows = int(r);
  pm.stage_bytes = pm.stage_rows * (pm.code_row_bytes + 2 * pm.meta_row_bytes);
  const int smem = kBulkStages * pm.stage_bytes;
  if (smem > 200 * 1024) return cudaSuccess;
  int64_t span0 = 0;
  for (int i = 0; i < pm.count; ++i) {
    kvx::PullPart& P = pm.part[i];
    const int64_t two_t = 2 * P.n_tokens;
    P.rows_per_span = int(r < two_t ? r : two_t);
    P.spans_per_layer = int((two_t + P.rows_per_span - 1) / P.rows_per_span);
    P.span0 = uint32_t(span0);
    span0 += n_layers * P.spans_per_layer;
    if (span0 >= (int64_t(1) << 31)) return cudaSuccess;
  }
  pm.n_spans = uint32_t(span0);
  auto k = kvx::pull_many_kernel<BITS, G, kBulkStages>;
  cudaError_t attr = ensure_smem_attr(k, 200 * 1024);
  if (attr != cudaSuccess) return attr;
  int per_sm = blocks_per_sm(k, kBulkThreads, smem);
  per_sm = per_sm < pull_ctas_per_sm<BITS>() ? per_sm : pull_ctas_per_sm<BITS>();
  int64_t grid = int64_t(sm_count(current_device())) * per_sm;
  if (grid > pm.n_spans) grid = pm.n_spans;
  *ok = true;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(kBulkThreads);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, g, pm);
}

template <int BITS>
cudaError_t dispatch_quant(int group, const kvx::Geo& g, void* c, void* sc, void* z, cudaStream_t s,
                           const SignalReq& rq = SignalReq()) {
  switch (group) {
    case 32: return launch_quant<BITS, 32>(g, c, sc, z, s, rq);
    case 64: return launch_quant<BITS, 64>(g, c, sc, z, s, rq);
    default: return launch_quant<BITS, 128>(g, c, sc, z, s, rq);
  }
}

template <int BITS>
cudaError_t dispatch_dequant(int group, const kvx::Geo& g, const void* c, const void* sc,
                             const void* z, cudaStream_t s) {
  switch (group) {
    case 32: return launch_dequant<BITS, 32>(g, c, sc, z, s);
    case 64: return launch_dequant<BITS, 64>(g, c, sc, z, s);
    default: return launch_dequant<BITS, 128>(g, c, sc, z, s);
  }
}

// ---- driver entry points (resolved lazily; no link-time libcuda dependency)
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_writeValue32 g_write32 = nullptr;
PFN_waitValue32 g_wait32 = nullptr;
std::once_flag g_drv_once;
int g_drv_status = KVX_ERR_UNSUPPORTED;

void resolve_driver() {
  std::call_once(g_drv_once, [] {
    cudaDriverEntryPointQueryResult q1, q2;
    void* w = nullptr;
    void* t = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWaitValue32", &t, cudaEnableDefault, &q2) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && w && t) {
      g_write32 = reinterpret_cast<PFN_writeValue32>(w);
      g_wait32 = reinterpret_cast<PFN_waitValue32>(t);
      g_drv_status = KVX_OK;
    }
  });
}

// Sub-array offsets of a kivi payload segment: 16-byte aligned, and the V
// codes (8-bit: 32-byte vector accesses) 32-byte aligned in every layer.
bool kivi_offsets_bad(const int64_t* seg_offsets, int64_t payload_layer_stride, int bits) {
  for (int i = 0; i < 7; ++i)
    if (seg_offsets[i] < 0 || seg_offsets[i] % 16) return true;
  if (bits == 8 && (seg_offsets[4] % 32 || payload_layer_stride % 32)) return true;
  return false;
}

int kivi_check(int head_dim, int group, int bits) {
  if (bits != 4 && bits != 8) return KVX_ERR_INVALID_ARG;
  if (group != 32 && group != 64) return KVX_ERR_INVALID_ARG;
  if (head_dim <= 0 || head_dim % 32 || head_dim % group) return KVX_ERR_INVALID_ARG;
  return KVX_OK;
}

template <int BITS, int G>
cudaError_t launch_kchan_quant(const kvx::KchanGeo& kg, cudaStream_t s, uint32_t* counters = nullptr,
                               uint32_t* peer_flags = nullptr, int layers_per_chunk = 1,
                               uint32_t ready_value = 0) {
  constexpr int cta_ch = 4 * (32 / (G / 16)) * 8;  // matches quant_pack_kchan_kernel
  const int cblocks = (kg.row_elems + cta_ch - 1) / cta_ch;
  const int64_t items = kg.n_layers * kg.n_groups * cblocks;
  int64_t grid = int64_t(sm_count(current_device())) * 8;
  if (grid > items) grid = items;
  kvx::KchanSignal sig;
  sig.counters = counters;
  sig.peer_flags = peer_flags;
  sig.items_per_chunk = kg.n_groups * cblocks * int64_t(layers_per_chunk > 0 ? layers_per_chunk : 1);
  sig.ready_value = ready_value;
  kvx::quant_pack_kchan_kernel<BITS, G><<<unsigned(grid), 128, 0, s>>>(kg, sig);
  return cudaGetLastError();
}

template <int BITS, int G>
cudaError_t launch_kchan_dequant(const kvx::KchanGeo& kg, const int64_t* slots, void* kc,
                                        int64_t dst_ls_b, cudaStream_t s) {
  auto k = kvx::dequant_kchan_kernel<BITS, G>;
  const int64_t cblk = (kg.row_elems / 32 + 31) / 32;
  const int64_t items = kg.n_layers * kg.n_groups * cblk;  // one warp per item
  k<<<grid_for(k, items), kThreads, 0, s>>>(kg, slots, static_cast<char*>(kc), dst_ls_b);
  return cudaGetLastError();
}

#ifndef KVX_KCHAN_STAGE_CODES
#define KVX_KCHAN_STAGE_CODES 16384
#endif
constexpr int kKchanStageCodes = KVX_KCHAN_STAGE_CODES;  // code bytes per kchan span

// Span geometry of a bulk-staged kchan pull (false: not stageable).
template <int BITS, int G>
bool plan_kchan_pull(const kvx::KchanGeo& kg, const uint32_t* ready, uint32_t ready_value,
                     int layers_per_chunk, kvx::Ctl* ctl, kvx::KchanBulk& kb) {
  kb = kvx::KchanBulk{};
  kb.ready = ready;
  kb.ready_value = ready_value;
  kb.ctl = ctl;
  kb.layers_per_chunk = layers_per_chunk > 0 ? layers_per_chunk : 1;
  kb.slab = kKchanStageCodes / (G * BITS / 8);  // channels per span (S/32 divides 256)
  // rows that fit one span whole: the group's code rows are then a single
  // contiguous range, one bulk copy instead of G (when S/32 still divides 256)
  if (kg.row_elems <= kb.slab && 256 % (kg.row_elems / 32) == 0) kb.slab = kg.row_elems;
  if (kg.row_elems % 32 || !aligned(kg.codes, 16) || !aligned(kg.scale, 16) ||
      !aligned(kg.zero, 16) || kg.payload_ls % 16)
    return false;
  kb.slabs = (kg.row_elems + kb.slab - 1) / kb.slab;
  kb.n_spans = kg.n_layers * kg.n_groups * kb.slabs;
  kb.stage_bytes = G * kb.slab * BITS / 8 + 4 * kb.slab;
  return true;
}

// Bulk-staged kchan dequant (payload read over NVLink).  *ok = false when the
// shape cannot be staged (caller falls back to the per-lane kernel).
template <int BITS, int G>
cudaError_t launch_kchan_pull(const kvx::KchanGeo& kg, const int64_t* slots, void* kc,
                              int64_t dst_ls_b, cudaStream_t s, bool* ok,
                              const uint32_t* ready = nullptr, uint32_t ready_value = 0,
                              int layers_per_chunk = 1, kvx::Ctl* ctl = nullptr,
                              bool pdl = false) {
  *ok = false;
  constexpr int kStages = 4;
  kvx::KchanBulk kb;
  if (!plan_kchan_pull<BITS, G>(kg, ready, ready_value, layers_per_chunk, ctl, kb))
    return cudaSuccess;
  const int smem = kStages * kb.stage_bytes;
  auto k = kvx::pull_kchan_kernel<BITS, G, kStages>;
  {
    // the largest span of this instantiation (the slab shrinks for short rows)
    const int s_max = kKchanStageCodes / (G * BITS / 8);
    const int smem_max = kStages * (G * s_max * BITS / 8 + 4 * s_max);
    cudaError_t attr = ensure_smem_attr(k, smem_max);
    if (attr != cudaSuccess) return attr;
  }
  int per_sm = blocks_per_sm(k, kBulkThreads, smem);
  per_sm = per_sm < kPullCtasPerSm ? per_sm : kPullCtasPerSm;  // as launch_pull
  int64_t grid = int64_t(sm_count(current_device())) * per_sm;
  if (grid > kb.n_spans) grid = kb.n_spans;
  if (grid < 1) return cudaSuccess;
  *ok = true;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(kBulkThreads);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, kg, kb, slots, static_cast<char*>(kc), dst_ls_b);
}

// The kivi pull as ONE kernel (pull_kivi_kernel): the K groups' spans then
// the V rows' spans.  *ok = false when either part cannot be bulk-staged.
template <int BITS, int G>
cudaError_t launch_kivi_pull(const kvx::KchanGeo& kg, const kvx::Geo& gv, const void* vc,
                             const void* vs, const void* vz, const int64_t* slots, void* kc,
                             int64_t dst_ls_b, cudaStream_t s, bool* ok, const uint32_t* ready,
                             uint32_t ready_value, int layers_per_chunk, kvx::Ctl* ctl,
                             const PullDone& done, kvx::KiviResidual kr) {
  *ok = false;
  constexpr int kStages = 4;
  kvx::KchanBulk kb;
  kvx::BulkGeo bg;
  if (!plan_kchan_pull<BITS, G>(kg, ready, ready_value, layers_per_chunk, ctl, kb)) return cudaSuccess;
  if (!plan_pull<BITS, G>(gv, vc, vs, vz, ready ? ready + KVX_KIVI_V_FLAGS : nullptr, ready_value,
                          layers_per_chunk, done, ctl, bg))
    return cudaSuccess;
  const int stage = kb.stage_bytes > bg.stage_bytes ? kb.stage_bytes : bg.stage_bytes;
  const int smem = kStages * stage;
  if (smem > 200 * 1024) return cudaSuccess;
  if (kr.n_rows > 0) {  // residual spans: as many whole rows as a stage holds
    if (kr.row_bytes % 16 || kr.row_bytes > stage || !aligned(kr.rows, 16) || kr.payload_ls % 16)
      return cudaSuccess;
    kr.rows_per_span = stage / kr.row_bytes;
    kr.spans_per_layer = int((kr.n_rows + kr.rows_per_span - 1) / kr.rows_per_span);
    kr.n_spans = kg.n_layers * kr.spans_per_layer;
  } else {
    kr.n_spans = 0;
    kr.rows_per_span = 1;
    kr.spans_per_layer = 1;
  }
  auto k = kvx::pull_kivi_kernel<BITS, G, kStages>;
  cudaError_t attr = ensure_smem_attr(k, 200 * 1024);
  if (attr != cudaSuccess) return attr;
  int per_sm = blocks_per_sm(k, kBulkThreads, smem);
  per_sm = per_sm < kPullCtasPerSm ? per_sm : kPullCtasPerSm;
  int64_t grid = int64_t(sm_count(current_device())) * per_sm;
  const int64_t n_all = kb.n_spans + int64_t(bg.n_spans) + kr.n_spans;
  if (grid > n_all) grid = n_all;
  if (grid < 1) return cudaSuccess;
  *ok = true;
  kvx::pull_kivi_kernel<BITS, G, kStages><<<unsigned(grid), kBulkThreads, smem, s>>>(
      kg, kb, gv, bg, static_cast<const uint8_t*>(vc), static_cast<const __half*>(vs),
      static_cast<const __half*>(vz), slots, static_cast<char*>(kc), dst_ls_b, stage, kr);
  return cudaGetLastError();
}

}  // namespace

extern "C" {

int kvx_version(void) { return 20000; }

const char* kvx_strerror(int code) {
  switch (code) {
    case KVX_OK: return "ok";
    case KVX_ERR_INVALID_ARG: return "kvx: invalid argument";
    case KVX_ERR_NO_PATH: return "kvx: no peer path between devices";
    case KVX_ERR_UNSUPPORTED: return "kvx: operation unsupported on this device/driver";
    case KVX_ERR_NCCL: return "kvx: NCCL call failed";
    default: return cudaGetErrorString(static_cast<cudaError_t>(code));
  }
}

int kvx_device_count(int* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (count) *count = n;
  return KVX_OK;
}

int kvx_packed_sizes(int64_t n_rows, int head_dim, int group, int bits, int64_t* codes_bytes,
                     int64_t* scale_bytes, int64_t* zero_bytes) {
  int rc = valid_format(head_dim, group, bits);
  if (rc) return rc;
  if (n_rows < 0) return KVX_ERR_INVALID_ARG;
  const int64_t ng = bits == 16 ? 0 : head_dim / group;
  if (codes_bytes) *codes_bytes = n_rows * head_dim * bits / 8;
  if (scale_bytes) *scale_bytes = n_rows * ng * 2;
  if (zero_bytes) *zero_bytes = n_rows * ng * 2;
  return KVX_OK;
}

int kvx_quant_pack(const void* k_src, const void* v_src, int64_t src_layer_stride,
                   const int64_t* src_slots, int64_t n_layers, int64_t n_tokens, int n_heads,
                   int head_dim, int group, int bits, void* codes, void* scale, void* zero,
                   int64_t payload_layer_stride, int plane_heads, int head_offset, void* stream) {
  int rc = valid_format(head_dim, group, bits);
  if (rc) return rc;
  kvx::Geo g;
  rc = make_geo(g, k_src, v_src, src_layer_stride, src_slots, n_layers, n_tokens, n_heads, head_dim,
                group, bits, payload_layer_stride, 2, 0, plane_heads, head_offset);
  if (rc) return rc;
  if (g.n_token_rows == 0) return KVX_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (bits == 16) {
    if (!codes || !aligned(codes, 16)) return KVX_ERR_INVALID_ARG;
    auto k = kvx::pack16_kernel<kUnroll>;
    k<<<grid_for(k, g.n_token_rows), kThreads, 0, s>>>(g, static_cast<uint8_t*>(codes));
    return cudaGetLastError();
  }
  if (!codes || !scale || !zero || !aligned(codes, 8 * bits) || !aligned(scale, 2) ||
      !aligned(zero, 2))
    return KVX_ERR_INVALID_ARG;
  if (k_src && (!aligned(k_src, 32) || !aligned(v_src, 32) || (src_layer_stride * 2) % 32 ||
                g.plane_row_b % 32 || g.head_off_b % 32))
    return KVX_ERR_INVALID_ARG;  // 256-bit loads
  switch (bits) {
    case 2: return dispatch_quant<2>(group, g, codes, scale, zero, s);
    case 8: return dispatch_quant<8>(group, g, codes, scale, zero, s);
    default: return dispatch_quant<4>(group, g, codes, scale, zero, s);
  }
}

int kvx_quant_pack_signal(const void* k_src, const void* v_src, int64_t src_layer_stride,
                          const int64_t* src_slots, int64_t n_layers, int64_t n_tokens,
                          int n_heads, int head_dim, int group, int bits, void* codes,
                          void* scale, void* zero, int64_t payload_layer_stride,
                          int plane_heads, int head_offset, void* counters,
                          void* peer_ready_flags, int layers_per_chunk, uint32_t ready_value,
                          const void* free_flag, uint32_t free_value, void* ctl, void* stream) {
  int rc = valid_format(head_dim, group, bits);
  if (rc) return rc;
  if (bits == 16 || !counters || !peer_ready_flags || layers_per_chunk < 1 ||
      !aligned(counters, 4) || !aligned(peer_ready_flags, 4) || !aligned(free_flag, 4) ||
      !aligned(ctl, 8))
    return KVX_ERR_INVALID_ARG;
  kvx::Geo g;
  rc = make_geo(g, k_src, v_src, src_layer_stride, src_slots, n_layers, n_tokens, n_heads, head_dim,
                group, bits, payload_layer_stride, 2, 0, plane_heads, head_offset);
  if (rc) return rc;
  if (g.n_token_rows == 0) return KVX_OK;
  if (!codes || !scale || !zero || !aligned(codes, 8 * bits) || !aligned(scale, 2) ||
      !aligned(zero, 2) || !aligned(k_src, 32) || !aligned(v_src, 32) || (src_layer_stride * 2) % 32 ||
      g.plane_row_b % 32 || g.head_off_b % 32)
    return KVX_ERR_INVALID_ARG;
  SignalReq rq;
  rq.counters = static_cast<uint32_t*>(counters);
  rq.peer_flags = static_cast<uint32_t*>(peer_ready_flags);
  rq.ready_value = ready_value;
  rq.free_flag = static_cast<const uint32_t*>(free_flag);
  rq.free_value = free_value;
  rq.ctl = static_cast<kvx::Ctl*>(ctl);
  rq.layers_per_chunk = layers_per_chunk;
  rq.n_layers = n_layers;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (bits) {
    case 2: return dispatch_quant<2>(group, g, codes, scale, zero, s, rq);
    case 8: return dispatch_quant<8>(group, g, codes, scale, zero, s, rq);
    default: return dispatch_quant<4>(group, g, codes, scale, zero, s, rq);
  }
}

int kvx_dequant_scatter_paged(const void* codes, const void* scale, const void* zero,
                              int64_t payload_layer_stride, const int64_t* dst_slots,
                              int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim,
                              int group, int bits, void* k_cache, void* v_cache,
                              int64_t dst_layer_stride, int plane_heads, int head_offset,
                              void* stream) {
  int rc = valid_format(head_dim, group, bits);
  if (rc) return rc;
  kvx::Geo g;
  rc = make_geo(g, k_cache, v_cache, dst_layer_stride, dst_slots, n_layers, n_tokens, n_heads,
                head_dim, group, bits, payload_layer_stride, 2, 0, plane_heads, head_offset);
  if (rc) return rc;
  if (g.n_token_rows == 0) return KVX_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (bits == 16) {
    if (!codes || !aligned(codes, 16)) return KVX_ERR_INVALID_ARG;
    auto k = kvx::scatter16_kernel<kUnroll>;
    k<<<grid_for(k, g.n_token_rows), kThreads, 0, s>>>(g, static_cast<const uint8_t*>(codes));
    return cudaGetLastError();
  }
  if (!codes || !scale || !zero || !aligned(codes, 8 * bits) || !aligned(scale, 2) ||
      !aligned(zero, 2))
    return KVX_ERR_INVALID_ARG;
  if (k_cache && (!aligned(k_cache, 32) || !aligned(v_cache, 32) || (dst_layer_stride * 2) % 32 ||
                  g.plane_row_b % 32 || g.head_off_b % 32))
    return KVX_ERR_INVALID_ARG;  // 256-bit stores
  switch (bits) {
    case 2: return dispatch_dequant<2>(group, g, codes, scale, zero, s);
    case 8: return dispatch_dequant<8>(group, g, codes, scale, zero, s);
    default: return dispatch_dequant<4>(group, g, codes, scale, zero, s);
  }
}

int kvx_pull_dequant_scatter_paged(const void* codes, const void* scale, const void* zero,
                                   int64_t payload_layer_stride, const int64_t* dst_slots,
                                   int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim,
                                   int group, int bits, void* k_cache, void* v_cache,
                                   int64_t dst_layer_stride, int plane_heads, int head_offset,
                                   const void* ready_flags, uint32_t ready_value,
                                   int layers_per_chunk, void* done_counter, void* peer_free_flag,
                                   void* ctl, int flags, void* stream) {
  int rc = valid_format(head_dim, group, bits);
  if (rc) return rc;
  kvx::Geo g;
  rc = make_geo(g, k_cache, v_cache, dst_layer_stride, dst_slots, n_layers, n_tokens, n_heads,
                head_dim, group, bits, payload_layer_stride, 2, 0, plane_heads, head_offset);
  if (rc) return rc;
  if (g.n_token_rows == 0) return KVX_OK;
  if ((ready_flags && (!aligned(ready_flags, 4) || layers_per_chunk < 1)) || !aligned(ctl, 8) ||
      (flags & ~(KVX_PULL_PDL | KVX_PULL_CHAINED)) ||
      ((flags & KVX_PULL_CHAINED) && !(flags & KVX_PULL_PDL)))
    return KVX_ERR_INVALID_ARG;
  if ((done_counter != nullptr) != (peer_free_flag != nullptr) ||
      (done_counter && (!ready_flags || !aligned(done_counter, 4) || !aligned(peer_free_flag, 4))))
    return KVX_ERR_INVALID_ARG;
  PullDone done;
  done.done_counter = static_cast<uint32_t*>(done_counter);
  done.peer_free = static_cast<uint32_t*>(peer_free_flag);
  if (bits != 16 && codes && scale && zero && k_cache && aligned(k_cache, 32) &&
      aligned(v_cache, 32) && (dst_layer_stride * 2) % 32 == 0 && g.plane_row_b % 32 == 0 &&
      g.head_off_b % 32 == 0 && aligned(codes, 8 * bits)) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t* rf = static_cast<const uint32_t*>(ready_flags);
    kvx::Ctl* c = static_cast<kvx::Ctl*>(ctl);
    const bool pdl = flags & KVX_PULL_PDL;
    done.chained = (flags & KVX_PULL_CHAINED) != 0;
    const int lpc = layers_per_chunk;
    bool ok = false;
    cudaError_t e;
    switch (bits) {
      case 2: e = dispatch_pull<2>(group, g, codes, scale, zero, s, &ok, rf, ready_value, lpc, done, c, pdl); break;
      case 8: e = dispatch_pull<8>(group, g, codes, scale, zero, s, &ok, rf, ready_value, lpc, done, c, pdl); break;
      default: e = dispatch_pull<4>(group, g, codes, scale, zero, s, &ok, rf, ready_value, lpc, done, c, pdl); break;
    }
    if (e != cudaSuccess) return e;
    if (ok) return KVX_OK;
  }
  // shapes the bulk path cannot stage (16-bit, unaligned rows): per-lane loads,
  // which cannot wait in-kernel -- callers pass ready_flags only for bulk shapes
  if (ready_flags || done_counter) return KVX_ERR_UNSUPPORTED;
  return kvx_dequant_scatter_paged(codes, scale, zero, payload_layer_stride, dst_slots, n_layers,
                                   n_tokens, n_heads, head_dim, group, bits, k_cache, v_cache,
                                   dst_layer_stride, plane_heads, head_offset, stream);
}

int kvx_pull_supported(int64_t n_tokens, int n_heads, int head_dim, int group, int bits) {
  if (valid_format(head_dim, group, bits) || bits == 16 || n_tokens < 1) return 0;
  const int64_t row = int64_t(n_heads) * head_dim;
  return (2 * n_tokens * row * bits / 8) % 16 == 0 && (2 * n_tokens * (row / group) * 2) % 16 == 0;
}

// ---- "kivi" format: per-channel K groups + fp16 residual window, V per token --

struct KiviSignal {  // fused kivi prefill: device doorbells per layer chunk
  uint32_t* counters = nullptr;    // [2][kMaxSignalChunks] (K, V)
  uint32_t* peer_flags = nullptr;  // ready row: K chunks at [c], V chunks at [KVX_KIVI_V_FLAGS + c]
  int layers_per_chunk = 1;
  uint32_t ready_value = 0;
  kvx::Ctl* ctl = nullptr;
};

static int kivi_quant(const void* k_src, const void* v_src, int64_t src_layer_stride,
                      int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim, int group,
                      int bits, const int64_t* group_starts, int64_t n_groups,
                      const int64_t* residual_tokens, int64_t n_residual, void* payload,
                      int64_t payload_layer_stride, const int64_t* seg_offsets, void* stream,
                      const KiviSignal& ks = KiviSignal()) {
  int rc = kivi_check(head_dim, group, bits);
  if (rc) return rc;
  if (n_layers < 0 || n_tokens < 0 || n_heads <= 0 || n_groups < 0 || n_residual < 0 ||
      n_groups * group + n_residual != n_tokens || !seg_offsets || payload_layer_stride % 16)
    return KVX_ERR_INVALID_ARG;
  if (n_layers == 0 || n_tokens == 0) return KVX_OK;
  if (!k_src || !v_src || !payload || (n_groups && !group_starts) || (n_residual && !residual_tokens))
    return KVX_ERR_INVALID_ARG;
  if (kivi_offsets_bad(seg_offsets, payload_layer_stride, bits)) return KVX_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(payload);
  const int row_elems = n_heads * head_dim;
  cudaError_t e = cudaSuccess;
  if (n_groups) {  // K per channel first: the decode side starts pulling it first
    kvx::KchanGeo kg;
    kg.k_plane = static_cast<const char*>(k_src);
    kg.layer_stride_b = src_layer_stride * 2;
    kg.group_starts = group_starts;
    kg.n_groups = n_groups;
    kg.row_elems = row_elems;
    kg.n_layers = n_layers;
    kg.codes = base + seg_offsets[0];
    kg.scale = base + seg_offsets[1];
    kg.zero = base + seg_offsets[2];
    kg.payload_ls = payload_layer_stride;
    uint32_t* cnt = ks.counters;
    uint32_t* fl = ks.peer_flags;
    const int lpc = ks.layers_per_chunk;
    const uint32_t rv = ks.ready_value;
    if (bits == 4)
      e = group == 32 ? launch_kchan_quant<4, 32>(kg, s, cnt, fl, lpc, rv)
                      : launch_kchan_quant<4, 64>(kg, s, cnt, fl, lpc, rv);
    else
      e = group == 32 ? launch_kchan_quant<8, 32>(kg, s, cnt, fl, lpc, rv)
                      : launch_kchan_quant<8, 64>(kg, s, cnt, fl, lpc, rv);
    if (e != cudaSuccess) return e;
  } else if (ks.peer_flags) {
    // no per-channel groups (every request shorter than a group): the K
    // doorbells carry nothing, ring them in stream order
    const int nc = int((n_layers + ks.layers_per_chunk - 1) / ks.layers_per_chunk);
    for (int c = 0; c < nc; ++c) {
      rc = kvx_stream_signal(ks.peer_flags + c, ks.ready_value, stream);
      if (rc) return rc;
    }
  }
  if (n_residual) {  // residual window: fp16 rows gathered into the payload
    kvx::Geo g;
    rc = make_geo(g, k_src, k_src, src_layer_stride, residual_tokens, n_layers, n_residual, n_heads,
                  head_dim, group, 16, payload_layer_stride, 1, 0);
    if (rc) return rc;
    auto k = kvx::pack16_kernel<kUnroll>;
    k<<<grid_for(k, g.n_token_rows), kThreads, 0, s>>>(g, reinterpret_cast<uint8_t*>(base + seg_offsets[3]));
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  {  // V per token (its doorbells, rung after the K and residual kernels in
     // stream order, publish the whole chunk)
    kvx::Geo g;
    rc = make_geo(g, v_src, v_src, src_layer_stride, nullptr, n_layers, n_tokens, n_heads, head_dim,
                  group, bits, payload_layer_stride, 1, 1);
    if (rc) return rc;
    SignalReq rq;
    if (ks.peer_flags) {
      rq.counters = ks.counters + kvx::kMaxSignalChunks;
      rq.peer_flags = ks.peer_flags + KVX_KIVI_V_FLAGS;
      rq.ready_value = ks.ready_value;
      rq.ctl = ks.ctl;
      rq.layers_per_chunk = ks.layers_per_chunk;
      rq.n_layers = n_layers;
    }
    e = bits == 4 ? dispatch_quant<4>(group, g, base + seg_offsets[4], base + seg_offsets[5],
                                      base + seg_offsets[6], s, rq)
                  : dispatch_quant<8>(group, g, base + seg_offsets[4], base + seg_offsets[5],
                                      base + seg_offsets[6], s, rq);
  }
  return e;
}

int kvx_quant_pack_kivi(const void* k_src, const void* v_src, int64_t src_layer_stride,
                        int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim, int group,
                        int bits, const int64_t* group_starts, int64_t n_groups,
                        const int64_t* residual_tokens, int64_t n_residual, void* payload,
                        int64_t payload_layer_stride, const int64_t* seg_offsets, void* stream) {
  return kivi_quant(k_src, v_src, src_layer_stride, n_layers, n_tokens, n_heads, head_dim, group,
                    bits, group_starts, n_groups, residual_tokens, n_residual, payload,
                    payload_layer_stride, seg_offsets, stream);
}

int kvx_quant_pack_kivi_signal(const void* k_src, const void* v_src, int64_t src_layer_stride,
                               int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim,
                               int group, int bits, const int64_t* group_starts, int64_t n_groups,
                               const int64_t* residual_tokens, int64_t n_residual, void* payload,
                               int64_t payload_layer_stride, const int64_t* seg_offsets,
                               void* counters, void* peer_ready_flags, int layers_per_chunk,
                               uint32_t ready_value, const void* free_flag, uint32_t free_value,
                               void* ctl, void* stream) {
  if (!counters || !peer_ready_flags || layers_per_chunk < 1 || !aligned(counters, 4) ||
      !aligned(peer_ready_flags, 4) || !aligned(free_flag, 4) || !aligned(ctl, 8))
    return KVX_ERR_INVALID_ARG;
  if (n_layers > 0 && (n_layers + layers_per_chunk - 1) / layers_per_chunk > KVX_KIVI_V_FLAGS)
    return KVX_ERR_INVALID_ARG;
  if (free_flag) {  // hold the launch in the GPU front-end until the queue slot is free
    int rc = kvx_stream_wait(free_flag, free_value, stream);
    if (rc) return rc;
  }
  KiviSignal ks;
  ks.counters = static_cast<uint32_t*>(counters);
  ks.peer_flags = static_cast<uint32_t*>(peer_ready_flags);
  ks.layers_per_chunk = layers_per_chunk;
  ks.ready_value = ready_value;
  ks.ctl = static_cast<kvx::Ctl*>(ctl);
  return kivi_quant(k_src, v_src, src_layer_stride, n_layers, n_tokens, n_heads, head_dim, group,
                    bits, group_starts, n_groups, residual_tokens, n_residual, payload,
                    payload_layer_stride, seg_offsets, stream, ks);
}

static int kivi_dequant(const void* payload, int64_t payload_layer_stride,
                        const int64_t* seg_offsets, const int64_t* dst_slots,
                        const int64_t* group_starts, int64_t n_groups,
                        const int64_t* residual_dst_slots, int64_t n_residual, int64_t n_layers,
                        int64_t n_tokens, int n_heads, int head_dim, int group, int bits,
                        void* k_cache, void* v_cache, int64_t dst_layer_stride, void* stream,
                        bool bulk, const uint32_t* ready = nullptr, uint32_t ready_value = 0,
                        int layers_per_chunk = 1, kvx::Ctl* ctl = nullptr,
                        const PullDone& done = PullDone(), bool pdl = false) {
  int rc = kivi_check(head_dim, group, bits);
  if (rc) return rc;
  if (n_layers < 0 || n_tokens < 0 || n_heads <= 0 || n_groups < 0 || n_residual < 0 ||
      n_groups * group + n_residual != n_tokens || !seg_offsets || payload_layer_stride % 16)
    return KVX_ERR_INVALID_ARG;
  if (n_layers == 0 || n_tokens == 0) return KVX_OK;
  if (!payload || !dst_slots || !k_cache || !v_cache || !aligned(k_cache, 32) ||
      !aligned(v_cache, 32) || (dst_layer_stride * 2) % 32 || (n_groups && !group_starts) ||
      (n_residual && !residual_dst_slots))
    return KVX_ERR_INVALID_ARG;
  if (kivi_offsets_bad(seg_offsets, payload_layer_stride, bits)) return KVX_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const char* base = static_cast<const char*>(payload);
  cudaError_t e = cudaSuccess;
  bool fused = false;  // K groups and V rows in ONE pull kernel (pull_kivi_kernel)
  static const bool fuse_ok = std::getenv("KVX_KIVI_TWO_KERNELS") == nullptr;
  if (bulk && n_groups && fuse_ok) {
    kvx::KchanGeo kg;
    kg.k_plane = nullptr;
    kg.layer_stride_b = 0;
    kg.group_starts = group_starts;
    kg.n_groups = n_groups;
    kg.row_elems = n_heads * head_dim;
    kg.n_layers = n_layers;
    kg.codes = const_cast<char*>(base + seg_offsets[0]);
    kg.scale = const_cast<char*>(base + seg_offsets[1]);
    kg.zero = const_cast<char*>(base + seg_offsets[2]);
    kg.payload_ls = payload_layer_stride;
    kvx::Geo gv;
    rc = make_geo(gv, v_cache, v_cache, dst_layer_stride, dst_slots, n_layers, n_tokens, n_heads,
                  head_dim, group, bits, payload_layer_stride, 1, 1);
    if (rc) return rc;
    if (gv.plane_row_b % 32 == 0) {
      const char *vc = base + seg_offsets[4], *vs = base + seg_offsets[5], *vz = base + seg_offsets[6];
      // the residual fp16 K rows ride in the same kernel: the slot can be
      // freed by its last CTA in every case
      kvx::KiviResidual kr = {};
      kr.rows = base + seg_offsets[3];
      kr.payload_ls = payload_layer_stride;
      kr.dst_slots = residual_dst_slots;
      kr.n_rows = n_residual;
      kr.row_bytes = n_heads * head_dim * 2;
      const int64_t dls = dst_layer_stride * 2;
      const int lpc = layers_per_chunk;
      if (bits == 4)
        e = group == 32 ? launch_kivi_pull<4, 32>(kg, gv, vc, vs, vz, dst_slots, k_cache, dls, s, &fused, ready, ready_value, lpc, ctl, done, kr)
                        : launch_kivi_pull<4, 64>(kg, gv, vc, vs, vz, dst_slots, k_cache, dls, s, &fused, ready, ready_value, lpc, ctl, done, kr);
      else
        e = group == 32 ? launch_kivi_pull<8, 32>(kg, gv, vc, vs, vz, dst_slots, k_cache, dls, s, &fused, ready, ready_value, lpc, ctl, done, kr)
                        : launch_kivi_pull<8, 64>(kg, gv, vc, vs, vz, dst_slots, k_cache, dls, s, &fused, ready, ready_value, lpc, ctl, done, kr);
      if (e != cudaSuccess) return e;
    }
  }
  if (n_groups && !fused) {
    kvx::KchanGeo kg;
    kg.k_plane = nullptr;
    kg.layer_stride_b = 0;
    kg.group_starts = group_starts;
    kg.n_groups = n_groups;
    kg.row_elems = n_heads * head_dim;
    kg.n_layers = n_layers;
    kg.codes = const_cast<char*>(base + seg_offsets[0]);
    kg.scale = const_cast<char*>(base + seg_offsets[1]);
    kg.zero = const_cast<char*>(base + seg_offsets[2]);
    kg.payload_ls = payload_layer_stride;
    const int64_t dls = dst_layer_stride * 2;
    bool ok = false;
    if (bulk) {
      const int lpc = layers_per_chunk;
      if (bits == 4)
        e = group == 32
                ? launch_kchan_pull<4, 32>(kg, dst_slots, k_cache, dls, s, &ok, ready, ready_value, lpc, ctl, pdl)
                : launch_kchan_pull<4, 64>(kg, dst_slots, k_cache, dls, s, &ok, ready, ready_value, lpc, ctl, pdl);
      else
        e = group == 32
                ? launch_kchan_pull<8, 32>(kg, dst_slots, k_cache, dls, s, &ok, ready, ready_value, lpc, ctl, pdl)
                : launch_kchan_pull<8, 64>(kg, dst_slots, k_cache, dls, s, &ok, ready, ready_value, lpc, ctl, pdl);
      if (e != cudaSuccess) return e;
      if (!ok && ready) return KVX_ERR_UNSUPPORTED;  // per-lane kernels cannot wait in-kernel
    }
    if (!ok) {
      if (bits == 4)
        e = group == 32 ? launch_kchan_dequant<4, 32>(kg, dst_slots, k_cache, dls, s)
                        : launch_kchan_dequant<4, 64>(kg, dst_slots, k_cache, dls, s);
      else
        e = group == 32 ? launch_kchan_dequant<8, 32>(kg, dst_slots, k_cache, dls, s)
                        : launch_kchan_dequant<8, 64>(kg, dst_slots, k_cache, dls, s);
      if (e != cudaSuccess) return e;
    }
  }
  if (!fused) {
    kvx::Geo g;
    rc = make_geo(g, v_cache, v_cache, dst_layer_stride, dst_slots, n_layers, n_tokens, n_heads,
                  head_dim, group, bits, payload_layer_stride, 1, 1);
    if (rc) return rc;
    const char *vc = base + seg_offsets[4], *vs = base + seg_offsets[5], *vz = base + seg_offsets[6];
    bool ok = false;
    if (bulk && aligned(v_cache, 32) && g.plane_row_b % 32 == 0) {
      // in-kernel slot release only without residual rows (they are read
      // after this kernel); otherwise the caller releases the slot after the call
      PullDone pd = n_residual ? PullDone() : done;
      const uint32_t* vready = ready ? ready + KVX_KIVI_V_FLAGS : nullptr;
      e = bits == 4 ? dispatch_pull<4>(group, g, vc, vs, vz, s, &ok, vready, ready_value,
                                       layers_per_chunk, pd, ctl, pdl)
                    : dispatch_pull<8>(group, g, vc, vs, vz, s, &ok, vready, ready_value,
                                       layers_per_chunk, pd, ctl, pdl);
      if (e != cudaSuccess) return e;
    }
    if (!ok && ready) return KVX_ERR_UNSUPPORTED;  // per-lane kernels cannot wait in-kernel
    if (!ok)
      e = bits == 4 ? dispatch_dequant<4>(group, g, vc, vs, vz, s)
                    : dispatch_dequant<8>(group, g, vc, vs, vz, s);
  }
  if (e != cudaSuccess) return e;
  // residual fp16 rows last: once the V kernel has seen every chunk's
  // doorbell, the whole payload is published, so these per-lane reads need
  // no wait of their own
  if (n_residual && !fused) {
    kvx::Geo g;
    rc = make_geo(g, k_cache, k_cache, dst_layer_stride, residual_dst_slots, n_layers, n_residual,
                  n_heads, head_dim, group, 16, payload_layer_stride, 1, 0);
    if (rc) return rc;
    auto k = kvx::scatter16_kernel<kUnroll>;
    k<<<grid_for(k, g.n_token_rows), kThreads, 0, s>>>(
        g, reinterpret_cast<const uint8_t*>(base + seg_offsets[3]));
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // the two-kernel path could not free the slot in-kernel (the residual
    // rows are read after the V pull): release it in stream order
    if (done.peer_free) return kvx_stream_signal(done.peer_free, ready_value, stream);
  }
  return e;
}

int kvx_dequant_scatter_paged_kivi(const void* payload, int64_t payload_layer_stride,
                                   const int64_t* seg_offsets, const int64_t* dst_slots,
                                   const int64_t* group_starts, int64_t n_groups,
                                   const int64_t* residual_dst_slots, int64_t n_residual,
                                   int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim,
                                   int group, int bits, void* k_cache, void* v_cache,
                                   int64_t dst_layer_stride, void* stream) {
  return kivi_dequant(payload, payload_layer_stride, seg_offsets, dst_slots, group_starts,
                      n_groups, residual_dst_slots, n_residual, n_layers, n_tokens, n_heads,
                      head_dim, group, bits, k_cache, v_cache, dst_layer_stride, stream, false);
}

int kvx_pull_dequant_scatter_paged_kivi(const void* payload, int64_t payload_layer_stride,
                                        const int64_t* seg_offsets, const int64_t* dst_slots,
                                        const int64_t* group_starts, int64_t n_groups,
                                        const int64_t* residual_dst_slots, int64_t n_residual,
                                        int64_t n_layers, int64_t n_tokens, int n_heads,
                                        int head_dim, int group, int bits, void* k_cache,
                                        void* v_cache, int64_t dst_layer_stride,
                                        const void* ready_flags, uint32_t ready_value,
                                        int layers_per_chunk, void* done_counter,
                                        void* peer_free_flag, void* ctl, int flags,
                                        void* stream) {
  if ((ready_flags && (!aligned(ready_flags, 4) || layers_per_chunk < 1)) || !aligned(ctl, 8) ||
      (flags & ~KVX_PULL_PDL))  // the kivi pull has no chained variant
    return KVX_ERR_INVALID_ARG;
  if ((done_counter != nullptr) != (peer_free_flag != nullptr) ||
      (done_counter && (!ready_flags || !aligned(done_counter, 4) || !aligned(peer_free_flag, 4))))
    return KVX_ERR_INVALID_ARG;
  PullDone done;
  done.done_counter = static_cast<uint32_t*>(done_counter);
  done.peer_free = static_cast<uint32_t*>(peer_free_flag);
  return kivi_dequant(payload, payload_layer_stride, seg_offsets, dst_slots, group_starts,
                      n_groups, residual_dst_slots, n_residual, n_layers, n_tokens, n_heads,
                      head_dim, group, bits, k_cache, v_cache, dst_layer_stride, stream, true,
                      static_cast<const uint32_t*>(ready_flags), ready_value, layers_per_chunk,
                      static_cast<kvx::Ctl*>(ctl), done, (flags & KVX_PULL_PDL) != 0);
}

// ---- transport -------------------------------------------------------------

int kvx_enable_peer(int a, int b) {
  if (a == b) return KVX_OK;
  int ab = 0, ba = 0;
  cudaError_t e = cudaDeviceCanAccessPeer(&ab, a, b);
  if (e != cudaSuccess) return e;
  e = cudaDeviceCanAccessPeer(&ba, b, a);
  if (e != cudaSuccess) return e;
  if (!ab || !ba) return KVX_ERR_NO_PATH;
  int cur = 0;
  cudaGetDevice(&cur);
  int pairs[2][2] = {{a, b}, {b, a}};
  for (auto& p : pairs) {
    cudaSetDevice(p[0]);
    e = cudaDeviceEnablePeerAccess(p[1], 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
      cudaGetLastError();
      e = cudaSuccess;
    }
    if (e != cudaSuccess) break;
  }
  cudaSetDevice(cur);
  return e;
}

int kvx_copy_peer(void* dst, int dst_dev, const void* src, int src_dev, size_t n, void* stream) {
  if (n == 0) return KVX_OK;
  return cudaMemcpyPeerAsync(dst, dst_dev, src, src_dev, n, static_cast<cudaStream_t>(stream));
}

int kvx_memcpy_async(void* dst, const void* src, size_t n, void* stream) {
  if (n == 0) return KVX_OK;
  if (!dst || !src) return KVX_ERR_INVALID_ARG;
  return cudaMemcpyAsync(dst, src, n, cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
}

int kvx_malloc(void** ptr, size_t n) {
  if (!ptr) return KVX_ERR_INVALID_ARG;
  return cudaMalloc(ptr, n ? n : 256);
}

int kvx_free(void* ptr) { return ptr ? cudaFree(ptr) : KVX_OK; }

int kvx_memset_async(void* ptr, int value, size_t n, void* stream) {
  return cudaMemsetAsync(ptr, value, n, static_cast<cudaStream_t>(stream));
}

int kvx_ipc_handle_size(void) { return int(sizeof(cudaIpcMemHandle_t)); }

int kvx_ipc_get_handle(void* ptr, void* out) {
  if (!ptr || !out) return KVX_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e != cudaSuccess) return e;
  memcpy(out, &h, sizeof(h));
  return KVX_OK;
}

int kvx_ipc_open(const void* handle, void** ptr_out) {
  if (!handle || !ptr_out) return KVX_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e == cudaSuccess) return KVX_OK;
  cudaGetLastError();
  // a malformed handle is the caller's error; anything else means this GPU
  // cannot map the partner's memory: no path (costs.py:63-64's NoPath)
  if (e == cudaErrorInvalidValue || e == cudaErrorInvalidResourceHandle) return e;
  return KVX_ERR_NO_PATH;
}

int kvx_ipc_close(void* ptr) { return ptr ? cudaIpcCloseMemHandle(ptr) : KVX_OK; }

int kvx_stream_memops_supported(int* supported) {
  resolve_driver();
  if (supported) *supported = (g_drv_status == KVX_OK);
  return KVX_OK;
}

int kvx_stream_signal(void* flag, uint32_t value, void* stream) {
  resolve_driver();
  if (g_drv_status) return g_drv_status;
  if (!flag || !aligned(flag, 4)) return KVX_ERR_INVALID_ARG;
  CUresult r = g_write32(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                         CU_STREAM_WRITE_VALUE_DEFAULT);
  return r == CUDA_SUCCESS ? KVX_OK : KVX_ERR_UNSUPPORTED;
}

int kvx_stream_wait(const void* flag, uint32_t value, void* stream) {
  resolve_driver();
  if (g_drv_status) return g_drv_status;
  if (!flag || !aligned(flag, 4)) return KVX_ERR_INVALID_ARG;
  CUresult r = g_wait32(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                        CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? KVX_OK : KVX_ERR_UNSUPPORTED;
}

#ifdef KVX_TRACE
// A/B trace builds only (not part of include/kvx.h): copy the timeline ring
// of kernel kind 0 (K1-signal) or 1 (K3-bulk) to host memory.
int kvx_trace_read(int kind, void* host_out, unsigned int* n_out) {
  if (kind < 0 || kind > 1 || !host_out || !n_out) return KVX_ERR_INVALID_ARG;
  unsigned int n[2];
  cudaError_t e = cudaMemcpyFromSymbol(n, kvx::g_trace_n, sizeof(n));
  if (e != cudaSuccess) return e;
  *n_out = n[kind];
  return cudaMemcpyFromSymbol(host_out, kvx::g_trace, sizeof(kvx::g_trace[0]),
                              kind * sizeof(kvx::g_trace[0]));
}
#endif

int kvx_stream_wait_eq(const void* flag, uint32_t value, void* stream) {
  resolve_driver();
  if (g_drv_status) return g_drv_status;
  if (!flag || !aligned(flag, 4)) return KVX_ERR_INVALID_ARG;
  CUresult r = g_wait32(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                        CU_STREAM_WAIT_VALUE_EQ);
  return r == CUDA_SUCCESS ? KVX_OK : KVX_ERR_UNSUPPORTED;
}


// ---- host-mapped control block ---------------------------------------------

int kvx_ctl_alloc(void** ctl_out) {
  if (!ctl_out) return KVX_ERR_INVALID_ARG;
  void* p = nullptr;
  cudaError_t e = cudaHostAlloc(&p, sizeof(kvx::Ctl), cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess) return e;
  memset(p, 0, sizeof(kvx::Ctl));
  void* d = nullptr;
  e = cudaHostGetDevicePointer(&d, p, 0);
  if (e != cudaSuccess || d != p) {  // UVA: the kernels use the host address
    cudaFreeHost(p);
    return e != cudaSuccess ? int(e) : KVX_ERR_UNSUPPORTED;
  }
  *ctl_out = p;
  return KVX_OK;
}

int kvx_ctl_free(void* ctl) { return ctl ? cudaFreeHost(ctl) : KVX_OK; }

// ---- chunk plan and the native pair channel --------------------------------

int kvx_handoff_chunk_plan(int64_t n_layers, int64_t n_tokens, int n_heads, int head_dim,
                           int layerwise, int* layers_per_chunk, int* n_chunks) {
  if (n_layers < 1 || n_tokens < 0 || n_heads < 1 || head_dim < 32 || !layers_per_chunk ||
      !n_chunks)
    return KVX_ERR_INVALID_ARG;
  int64_t n;
  if (layerwise) {
    n = n_layers < kvx::kMaxSignalChunks ? n_layers : kvx::kMaxSignalChunks;
  } else {
    // layer-granular doorbells, but every K1 warp should own several items
    // per chunk (one fence + atomic per warp per chunk): >= 4 items per
    // resident K1 warp (148 SMs x 2 CTAs x 8 warps) in every chunk
    const int64_t cpr = int64_t(n_heads) * head_dim / 32;
    const int64_t items = n_layers * 2 * n_tokens * ((cpr + 31) / 32);
    n = items / (4 * 148 * 2 * 8);
    if (n > n_layers) n = n_layers;
    if (n > kvx::kMaxSignalChunks) n = kvx::kMaxSignalChunks;
    if (n < 1) n = 1;
  }
  const int64_t lpc = (n_layers + n - 1) / n;
  *layers_per_chunk = int(lpc);
  *n_chunks = int((n_layers + lpc - 1) / lpc);
  return KVX_OK;
}

}  // extern "C"

namespace {
constexpr int kFlagReadyBase = 0;                            // ready[h][c]: h * 64 + c
constexpr int kFlagFreeBase = kvx::kMaxSignalChunks * 8;     // free[h]: 512 + h
constexpr int kPairScratch = kvx::kMaxSignalChunks + 1;      // u32 per queue slot

int64_t round256(int64_t x) { return (x + 255) / 256 * 256; }
}  // namespace

struct kvx_pair {
  int role = 0;  // KVX_ROLE_PREFILL / KVX_ROLE_DECODE
  int dev = 0;
  int64_t n_layers = 0, max_tokens = 0;
  int n_heads = 0, head_dim = 0, bits = 4, group = 128, queue_depth = 1, layerwise = 0;
  uint32_t* local_flags = nullptr;  // this GPU's doorbell page
  uint32_t* peer_flags = nullptr;   // the partner's page (IPC / peer mapped)
  char* payload = nullptr;          // the prefill GPU's queue (local on P, mapped on D)
  int64_t slot_bytes = 0;
  kvx::Ctl* ctl = nullptr;
  uint32_t* scratch = nullptr;      // [queue_depth][65] (device, zero between launches)
};

namespace {
// Sequence protocol: hand-off e (1, 2, ...) uses queue slot h = e % Q for the
// v-th time, v = (e - 1) / Q + 1.  P waits free[h] >= v - 1, rings
// ready[h][c] = v; D waits ready[h][c] >= v and sets free[h] = v.
void seq_of(const kvx_pair* p, uint64_t e, int* h, uint32_t* v) {
  *h = int(e % uint64_t(p->queue_depth));
  *v = uint32_t((e - 1) / uint64_t(p->queue_depth) + 1);
}

// Per-layer segment stride of a queue slot's payload (= datapath.PackedLayout).
int64_t pair_layer_stride(const kvx_pair* p, int64_t n_tokens, int64_t* scale_off,
                          int64_t* zero_off) {
  const int64_t rows = 2 * n_tokens * p->n_heads;
  const int64_t codes = rows * p->head_dim * p->bits / 8;
  const int64_t meta = rows * (p->head_dim / p->group) * 2;
  *scale_off = round256(codes);
  *zero_off = *scale_off + round256(meta);
  return *zero_off + round256(meta);
}

int pair_check(const kvx_pair* p, uint64_t e, int64_t n_tokens, int plane_heads, int head_offset) {
  if (!p || e < 1) return KVX_ERR_INVALID_ARG;
  if (n_tokens < 0 || n_tokens > p->max_tokens) return KVX_ERR_INVALID_ARG;
  const int ph = plane_heads ? plane_heads : p->n_heads;
  if (head_offset < 0 || head_offset + p->n_heads > ph) return KVX_ERR_INVALID_ARG;
  if (current_device() != p->dev) return KVX_ERR_INVALID_ARG;
  return KVX_OK;
}
}  // namespace

extern "C" {

int kvx_pair_create(int role, int64_t n_layers, int64_t max_tokens, int n_heads, int head_dim,
                    int bits, int group, int queue_depth, int layerwise, void* local_flags,
                    void* peer_flags, void* payload, int64_t slot_bytes, void* ctl,
                    void** pair_out) {
  if (!pair_out || (role != KVX_ROLE_PREFILL && role != KVX_ROLE_DECODE)) return KVX_ERR_INVALID_ARG;
  int rc = valid_format(head_dim, group, bits);
  if (rc || bits == 16) return KVX_ERR_INVALID_ARG;
  if (n_layers < 1 || max_tokens < 1 || n_heads < 1 || queue_depth < 1 || queue_depth > 8 ||
      !local_flags || !peer_flags || !payload || !aligned(local_flags, 4) ||
      !aligned(peer_flags, 4) || !aligned(payload, 256) || slot_bytes % 256 || !aligned(ctl, 8))
    return KVX_ERR_INVALID_ARG;
  auto* p = new (std::nothrow) kvx_pair();
  if (!p) return cudaErrorMemoryAllocation;
  p->role = role;
  p->dev = current_device();
  p->n_layers = n_layers;
  p->max_tokens = max_tokens;
  p->n_heads = n_heads;
  p->head_dim = head_dim;
  p->bits = bits;
  p->group = group;
  p->queue_depth = queue_depth;
  p->layerwise = layerwise ? 1 : 0;
  p->local_flags = static_cast<uint32_t*>(local_flags);
  p->peer_flags = static_cast<uint32_t*>(peer_flags);
  p->payload = static_cast<char*>(payload);
  p->slot_bytes = slot_bytes;
  p->ctl = static_cast<kvx::Ctl*>(ctl);
  int64_t so, zo;
  if (pair_layer_stride(p, max_tokens, &so, &zo) * n_layers > slot_bytes) {
    delete p;
    return KVX_ERR_INVALID_ARG;
  }
  const size_t sb = size_t(queue_depth) * kPairScratch * 4;
  cudaError_t e = cudaMalloc(&p->scratch, sb);
  if (e == cudaSuccess) e = cudaMemset(p->scratch, 0, sb);
  if (e != cudaSuccess) {
    cudaFree(p->scratch);
    delete p;
    return e;
  }
  *pair_out = p;
  return KVX_OK;
}

int kvx_pair_destroy(void* pair) {
  auto* p = static_cast<kvx_pair*>(pair);
  if (!p) return KVX_OK;
  cudaError_t e = cudaFree(p->scratch);
  delete p;
  return e;
}

int kvx_pair_send(void* pair, uint64_t epoch, const void* k_src, const void* v_src,
                  int64_t src_layer_stride, const int64_t* src_slots, int64_t n_tokens,
                  int plane_heads, int head_offset, int flags, void* stream) {
  auto* p = static_cast<kvx_pair*>(pair);
  int rc = pair_check(p, epoch, n_tokens, plane_heads, head_offset);
  if (rc) return rc;
  if (p->role != KVX_ROLE_PREFILL || (flags & ~(KVX_PAIR_GATE | KVX_PAIR_PDL)))
    return KVX_ERR_INVALID_ARG;
  if (n_tokens == 0) return KVX_OK;
  int h;
  uint32_t v;
  seq_of(p, epoch, &h, &v);
  int lpc, nc;
  rc = kvx_handoff_chunk_plan(p->n_layers, n_tokens, p->n_heads, p->head_dim, p->layerwise, &lpc,
                              &nc);
  if (rc) return rc;
  int64_t so, zo;
  const int64_t ls = pair_layer_stride(p, n_tokens, &so, &zo);
  char* base = p->payload + int64_t(h) * p->slot_bytes;
  uint32_t* free_flag = p->local_flags + kFlagFreeBase + h;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
#ifdef KVX_TRACE
  g_trace_epoch = uint32_t(epoch);
#endif
  if ((flags & KVX_PAIR_GATE) && v > 1) {
    // hold the prefill side in the GPU front-end (no SMs held) until the
    // decode side has consumed the slot's previous use; K1 re-checks in-kernel
    rc = kvx_stream_wait(free_flag, v - 1, stream);
    if (rc) return rc;
  }
  if (!(flags & KVX_PAIR_PDL))
    return kvx_quant_pack_signal(k_src, v_src, src_layer_stride, src_slots, p->n_layers, n_tokens,
                                 p->n_heads, p->head_dim, p->group, p->bits, base, base + so,
                                 base + zo, ls, plane_heads, head_offset,
                                 p->scratch + h * kPairScratch,
                                 p->peer_flags + kFlagReadyBase + h * 64, lpc, v, free_flag, v - 1,
                                 p->ctl, s);
  // PDL: K1 launched behind the stream's previous kernel (typically the
  // previous hand-off's K1, which signals once its items are done); its CTAs
  // wait (griddepcontrol.wait) for that grid before reading anything
  kvx::Geo g;
  rc = make_geo(g, k_src, v_src, src_layer_stride, src_slots, p->n_layers, n_tokens, p->n_heads,
                p->head_dim, p->group, p->bits, ls, 2, 0, plane_heads, head_offset);
  if (rc) return rc;
  if (!aligned(k_src, 32) || !aligned(v_src, 32) || (src_layer_stride * 2) % 32 ||
      g.plane_row_b % 32 || g.head_off_b % 32)
    return KVX_ERR_INVALID_ARG;
  SignalReq rq;
  rq.counters = p->scratch + h * kPairScratch;
  rq.peer_flags = p->peer_flags + kFlagReadyBase + h * 64;
  rq.ready_value = v;
  rq.free_flag = free_flag;
  rq.free_value = v - 1;
  rq.ctl = p->ctl;
  rq.layers_per_chunk = lpc;
  rq.n_layers = p->n_layers;
  rq.pdl = true;
  char* codes = base;
  switch (p->bits) {
    case 2: return dispatch_quant<2>(p->group, g, codes, base + so, base + zo, s, rq);
    case 8: return dispatch_quant<8>(p->group, g, codes, base + so, base + zo, s, rq);
    default: return dispatch_quant<4>(p->group, g, codes, base + so, base + zo, s, rq);
  }
}

int kvx_pair_recv(void* pair, uint64_t epoch, void* k_cache, void* v_cache,
                  int64_t dst_layer_stride, const int64_t* dst_slots, int64_t n_tokens,
                  int plane_heads, int head_offset, int flags, void* stream) {
  auto* p = static_cast<kvx_pair*>(pair);
  int rc = pair_check(p, epoch, n_tokens, plane_heads, head_offset);
  if (rc) return rc;
  if (p->role != KVX_ROLE_DECODE || (flags & ~(KVX_PAIR_GATE | KVX_PAIR_PDL | KVX_PAIR_CHAINED)) ||
      ((flags & KVX_PAIR_CHAINED) && !(flags & KVX_PAIR_PDL)) || !dst_slots)
    return KVX_ERR_INVALID_ARG;
  if (n_tokens == 0) return KVX_OK;
  if (!kvx_pull_supported(n_tokens, p->n_heads, p->head_dim, p->group, p->bits))
    return KVX_ERR_UNSUPPORTED;
  int h;
  uint32_t v;
  seq_of(p, epoch, &h, &v);
  int lpc, nc;
  rc = kvx_handoff_chunk_plan(p->n_layers, n_tokens, p->n_heads, p->head_dim, p->layerwise, &lpc,
                              &nc);
  if (rc) return rc;
  int64_t so, zo;
  const int64_t ls = pair_layer_stride(p, n_tokens, &so, &zo);
  const char* base = p->payload + int64_t(h) * p->slot_bytes;
  uint32_t* ready = p->local_flags + kFlagReadyBase + h * 64;
#ifdef KVX_TRACE
  g_trace_epoch = uint32_t(epoch);
#endif
  if (flags & KVX_PAIR_GATE) {
    // launch only once the first chunk is published: a pull never sits on
    // the SMs waiting for an idle prefill side
    rc = kvx_stream_wait(ready, v, stream);
    if (rc) return rc;
  }
  return kvx_pull_dequant_scatter_paged(base, base + so, base + zo, ls, dst_slots, p->n_layers,
                                        n_tokens, p->n_heads, p->head_dim, p->group, p->bits,
                                        k_cache, v_cache, dst_layer_stride, plane_heads,
                                        head_offset, ready, v, lpc, p->scratch + h * kPairScratch,
                                        p->peer_flags + kFlagFreeBase + h, p->ctl,
                                        ((flags & KVX_PAIR_PDL) ? KVX_PULL_PDL : 0) |
                                            ((flags & KVX_PAIR_CHAINED) ? KVX_PULL_CHAINED : 0),
                                        stream);
}

int kvx_pair_recv_many(void* pair, uint64_t first_epoch, int count, void* k_cache, void* v_cache,
                       int64_t dst_layer_stride, const int64_t* const* dst_slots,
                       const int64_t* n_tokens, int plane_heads, int head_offset, int flags,
                       void* stream) {
  auto* p = static_cast<kvx_pair*>(pair);
  if (!p || p->role != KVX_ROLE_DECODE || count < 1 || !dst_slots || !n_tokens ||
      (flags & ~KVX_PAIR_PDL))
    return KVX_ERR_INVALID_ARG;
  if (count > p->queue_depth || count > kvx::kMaxPullMany) return KVX_ERR_INVALID_ARG;
  for (int i = 0; i < count; ++i) {
    int rc = pair_check(p, first_epoch + uint64_t(i), n_tokens[i], plane_heads, head_offset);
    if (rc) return rc;
    if (n_tokens[i] < 1 || !dst_slots[i]) return KVX_ERR_INVALID_ARG;
    if (!kvx_pull_supported(n_tokens[i], p->n_heads, p->head_dim, p->group, p->bits))
      return KVX_ERR_UNSUPPORTED;
  }
  kvx::Geo g;
  int rc = make_geo(g, k_cache, v_cache, dst_layer_stride, nullptr, p->n_layers, 1, p->n_heads,
                    p->head_dim, p->group, p->bits, 256, 2, 0, plane_heads, head_offset);
  if (rc) return rc;
  if (!aligned(k_cache, 32) || !aligned(v_cache, 32) || (dst_layer_stride * 2) % 32 ||
      g.plane_row_b % 32 || g.head_off_b % 32)
    return KVX_ERR_INVALID_ARG;
  kvx::PullMany pm;
  std::memset(&pm, 0, sizeof(pm));
  pm.count = count;
  pm.ctl = p->ctl;
  int h0 = 0;
  for (int i = 0; i < count; ++i) {
    int h;
    uint32_t v;
    seq_of(p, first_epoch + uint64_t(i), &h, &v);
    if (i == 0) h0 = h;
    int lpc, nc;
    rc = kvx_handoff_chunk_plan(p->n_layers, n_tokens[i], p->n_heads, p->head_dim, p->layerwise,
                                &lpc, &nc);
    if (rc) return rc;
    int64_t so, zo;
    const int64_t ls = pair_layer_stride(p, n_tokens[i], &so, &zo);
    const char* base = p->payload + int64_t(h) * p->slot_bytes;
    kvx::PullPart& P = pm.part[i];
    P.codes = reinterpret_cast<const uint8_t*>(base);
    P.scale = reinterpret_cast<const __half*>(base + so);
    P.zero = reinterpret_cast<const __half*>(base + zo);
    P.payload_ls = ls;
    P.slots = dst_slots[i];
    P.n_tokens = n_tokens[i];
    P.ready = p->local_flags + kFlagReadyBase + h * 64;
    P.ready_value = v;
    P.layers_per_chunk = lpc;
    P.peer_free = p->peer_flags + kFlagFreeBase + h;
  }
  pm.done_counter = p->scratch + h0 * kPairScratch;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool pdl = flags & KVX_PAIR_PDL;
  bool ok = false;
  cudaError_t e;
  switch (p->bits) {
    case 2: e = p->group == 32 ? launch_pull_many<2, 32>(g, p->n_layers, pm, s, &ok, pdl)
              : p->group == 64 ? launch_pull_many<2, 64>(g, p->n_layers, pm, s, &ok, pdl)
                               : launch_pull_many<2, 128>(g, p->n_layers, pm, s, &ok, pdl); break;
    case 8: e = p->group == 32 ? launch_pull_many<8, 32>(g, p->n_layers, pm, s, &ok, pdl)
              : p->group == 64 ? launch_pull_many<8, 64>(g, p->n_layers, pm, s, &ok, pdl)
                               : launch_pull_many<8, 128>(g, p->n_layers, pm, s, &ok, pdl); break;
    default: e = p->group == 32 ? launch_pull_many<4, 32>(g, p->n_layers, pm, s, &ok, pdl)
               : p->group == 64 ? launch_pull_many<4, 64>(g, p->n_layers, pm, s, &ok, pdl)
                                : launch_pull_many<4, 128>(g, p->n_layers, pm, s, &ok, pdl); break;
  }
  if (e != cudaSuccess) return e;
  return ok ? KVX_OK : KVX_ERR_UNSUPPORTED;
}

}  // extern "C"

// ---- NCCL pair pool ------------------------------------------
// The paper pre-builds NCCL groups for its async SendRecv hand-offs.  These
// entry points give a serving engine the same thing through the C-ABI.  NCCL
// is resolved at run time (dlopen of the libnccl.so.2 already loaded by the
// process -- torch's -- else the system one), so the library has no link-time
// NCCL dependency and never mixes two NCCL builds in one process.
namespace {
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  bool ok = false;
};

const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.send && api.recv &&
             api.group_start && api.group_end;
  });
  return api;
}

int nccl_rc(ncclResult_t r) { return r == ncclSuccess ? KVX_OK : KVX_ERR_NCCL; }
}  // namespace

extern "C" {

int kvx_nccl_unique_id_size(void) { return int(sizeof(ncclUniqueId)); }

int kvx_nccl_get_unique_id(void* id_out) {
  if (!id_out) return KVX_ERR_INVALID_ARG;
  const NcclApi& a = nccl_api();
  if (!a.ok) return KVX_ERR_UNSUPPORTED;
  ncclUniqueId id;
  int rc = nccl_rc(a.get_unique_id(&id));
  if (rc == KVX_OK) std::memcpy(id_out, &id, sizeof(id));
  return rc;
}

int kvx_nccl_pair_init(const void* unique_id, int n_ranks, int rank, void** comm_out) {
  if (!unique_id || !comm_out || n_ranks < 1 || rank < 0 || rank >= n_ranks)
    return KVX_ERR_INVALID_ARG;
  const NcclApi& a = nccl_api();
  if (!a.ok) return KVX_ERR_UNSUPPORTED;
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  int rc = nccl_rc(a.comm_init_rank(&comm, n_ranks, id, rank));
  if (rc == KVX_OK) *comm_out = comm;
  return rc;
}

int kvx_nccl_sendrecv(void* comm, const void* send_buf, size_t send_bytes, int send_peer,
                      void* recv_buf, size_t recv_bytes, int recv_peer, void* stream) {
  if (!comm || (send_peer >= 0 && send_bytes && !send_buf) ||
      (recv_peer >= 0 && recv_bytes && !recv_buf))
    return KVX_ERR_INVALID_ARG;
  const NcclApi& a = nccl_api();
  if (!a.ok) return KVX_ERR_UNSUPPORTED;
  auto c = static_cast<ncclComm_t>(comm);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc = nccl_rc(a.group_start());
  if (rc) return rc;
  if (send_peer >= 0 && send_bytes)
    rc = nccl_rc(a.send(send_buf, send_bytes, ncclUint8, send_peer, c, s));
  if (rc == KVX_OK && recv_peer >= 0 && recv_bytes)
    rc = nccl_rc(a.recv(recv_buf, recv_bytes, ncclUint8, recv_peer, c, s));
  const int rc2 = nccl_rc(a.group_end());
  return rc ? rc : rc2;
}

int kvx_nccl_pair_destroy(void* comm) {
  if (!comm) return KVX_OK;
  const NcclApi& a = nccl_api();
  if (!a.ok) return KVX_ERR_UNSUPPORTED;
  return nccl_rc(a.comm_destroy(static_cast<ncclComm_t>(comm)));
}

}  // extern "C"
