// "kivi" format kernels (PAPER.md:490-492 borrows KIVI):
// keys quantised PER CHANNEL over groups of G consecutive tokens of one
// request (the request's last n % G tokens travel as fp16, the residual
// window), values per token as in the default format.  Same scalar
// arithmetic as K1/K3 (bit-exact with oracle/kvq_oracle.py quant_pack_kivi).
#pragma once

#include "kvx_kernels.cuh"

namespace kvx {

struct KchanGeo {
  const char* k_plane;      // K plane of layer 0 (dense source [T, H*D] per layer)
  int64_t layer_stride_b;   // bytes between source layers
  const int64_t* group_starts;  // [n_groups] first token of each group (batch order)
  int64_t n_groups;
  int row_elems;            // H*D
  int64_t n_layers;
  char* codes;              // payload: Kc of layer 0
  char* scale;              // Ks of layer 0
  char* zero;               // Kz of layer 0
  int64_t payload_ls;       // bytes between payload layers
};

// Per-chunk doorbells of the kchan quantiser (the fused kivi prefill side):
// items are CTA-strided (item i -> CTA i % gridDim.x) in layer-major order, so
// the CTAs owning items of chunk c = [a, b) number min(b - a, gridDim.x); the
// last of them to finish its share rings peer_flags[c] = ready_value.
struct KchanSignal {
  uint32_t* counters;       // [kMaxSignalChunks] zero between launches (reset in-kernel)
  uint32_t* peer_flags;     // decode-side K doorbells (IPC/peer mapped), null = none
  int64_t items_per_chunk;  // n_groups * cblocks * layers_per_chunk
  uint32_t ready_value;
};

// One lane's share of a per-channel K group: TH of the group's G tokens x 8
// adjacent channels (w[j] = token j's 8 fp16), the G / TH lanes of a group
// adjacent in the warp.  min/max over the lane's tokens, then across the
// group's lanes with log2(G / TH) shuffles; the group's lanes split the 8
// channels' IEEE division and reciprocal between them and share the results
// (K1-kivi 1.99 -> 1.78 ms at N=1 config 2, profiles/r02_bench/kchan_ab_n1.log);
// the lane with half == 0 stores the 8 scales and zeros (16 B each), every
// lane quantises its own tokens
// (8 nibbles = one 32-bit store per token at 4-bit).  Warp-uniform call:
// inactive lanes (channels past the row) take part in the shuffles.
template <int BITS, int G, int TH>
__device__ __forceinline__ void kchan_quant_lanes(const KchanGeo& g, const uint4 (&w)[TH],
                                                  bool active, int half, int64_t layer, int64_t k,
                                                  int ch) {
  constexpr uint32_t QMAX = (1u << BITS) - 1u;
  constexpr float QMAXF = float(QMAX);
  constexpr int LPC = G / TH;
  __half2 mn[4], mx[4];
  mn[0] = mx[0] = u32_as_h2(w[0].x);
  mn[1] = mx[1] = u32_as_h2(w[0].y);
  mn[2] = mx[2] = u32_as_h2(w[0].z);
  mn[3] = mx[3] = u32_as_h2(w[0].w);
#pragma unroll
  for (int j = 1; j < TH; ++j) {
    const uint32_t v[4] = {w[j].x, w[j].y, w[j].z, w[j].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      mn[i] = __hmin2(mn[i], u32_as_h2(v[i]));
      mx[i] = __hmax2(mx[i], u32_as_h2(v[i]));
    }
  }
#pragma unroll
  for (int off = 1; off < LPC; off <<= 1)  // combine the lanes' token slices
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      mn[i] = __hmin2(mn[i], u32_as_h2(__shfl_xor_sync(0xffffffffu, h2_as_u32(mn[i]), off)));
      mx[i] = __hmax2(mx[i], u32_as_h2(__shfl_xor_sync(0xffffffffu, h2_as_u32(mx[i]), off)));
    }
  // scale / zero / reciprocal of the 8 channels: the group's LPC lanes hold
  // the same min/max, so each computes 8 / LPC of the channels (IEEE
  // division and reciprocal are the costly part) and the results are shared
  // with one shuffle per channel and value
  constexpr int PER = 8 / LPC > 0 ? 8 / LPC : 1;
  float lzf[PER], linv[PER];
  uint32_t lsz[PER];  // (scale16, zero16) of the lane's channels
  bool sub = false;
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    const int c = LPC >= 8 ? half : m * LPC + half;  // this lane's m-th channel
    const __half2 mnp = mn[0], mxp = mx[0];
    float fmn = __low2float(mnp), fmx = __low2float(mxp);
#pragma unroll
    for (int cc = 1; cc < 8; ++cc)  // select channel c without dynamic register indexing
      if (cc == c) {
        fmn = (cc & 1) ? __high2float(mn[cc >> 1]) : __low2float(mn[cc >> 1]);
        fmx = (cc & 1) ? __high2float(mx[cc >> 1]) : __low2float(mx[cc >> 1]);
      }
    const __half z16 = __float2half_rn(__fadd_rn(fmn, 0.0f));
    const __half s16 = __float2half_rn(__fadd_rn(__fdiv_rn(__fsub_rn(fmx, fmn), QMAXF), 0.0f));
    const float sv = __half2float(s16);
    linv[m] = (sv != 0.0f) ? __frcp_rn(sv) : 0.0f;
    lzf[m] = __half2float(z16);
    lsz[m] = h2_as_u32(__halves2half2(s16, z16));
    sub |= sv != 0.0f && sv < 6.103515625e-05f;
  }
  float zf[8], inv[8];
  uint32_t sz[8];
  const int base = (threadIdx.x & 31) & ~(LPC - 1);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int m = LPC >= 8 ? 0 : c / LPC;
    const int src = base + (LPC >= 8 ? c : c % LPC);
    zf[c] = __shfl_sync(0xffffffffu, lzf[m], src);
    inv[c] = __shfl_sync(0xffffffffu, linv[m], src);
    sz[c] = __shfl_sync(0xffffffffu, lsz[m], src);
  }
  const bool clamp = __any_sync(0xffffffffu, active && sub);
  if (!active) return;
  char* lc = g.codes + layer * g.payload_ls;
  if (half == 0) {  // one lane of the group writes the 8 scales / zeros (16 B each)
    const int64_t meta = (k * g.row_elems + ch) * 2;
    uint4 sv, zv;  // sz[c] = (scale16, zero16): low halves -> scales, high -> zeros
    sv.x = prmt(sz[0], sz[1], 0x5410); sv.y = prmt(sz[2], sz[3], 0x5410);
    sv.z = prmt(sz[4], sz[5], 0x5410); sv.w = prmt(sz[6], sz[7], 0x5410);
    zv.x = prmt(sz[0], sz[1], 0x7632); zv.y = prmt(sz[2], sz[3], 0x7632);
    zv.z = prmt(sz[4], sz[5], 0x7632); zv.w = prmt(sz[6], sz[7], 0x7632);
    *reinterpret_cast<uint4*>(g.scale + layer * g.payload_ls + meta) = sv;
    *reinterpret_cast<uint4*>(g.zero + layer * g.payload_ls + meta) = zv;
  }
  unsigned long long invv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    asm("mov.b64 %0, {%1, %2};" : "=l"(invv[i]) : "f"(inv[2 * i]), "f"(inv[2 * i + 1]));
#pragma unroll
  for (int j = 0; j < TH; ++j) {
    const uint32_t v[4] = {w[j].x, w[j].y, w[j].z, w[j].w};
    uint32_t b[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      unsigned long long x, r;
      asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(sub_lo(v[i], zf[2 * i])), "f"(sub_hi(v[i], zf[2 * i + 1])));
      asm("{.reg .b64 mg; mov.b64 mg, {%3, %3}; fma.rn.f32x2 %0, %1, %2, mg;}"
          : "=l"(r) : "l"(x), "l"(invv[i]), "f"(8388608.0f));
      b[2 * i] = uint32_t(r);
      b[2 * i + 1] = uint32_t(r >> 32);
    }
    if (clamp) {
#pragma unroll
      for (int i = 0; i < 8; ++i) b[i] = min(b[i] - 0x4B000000u, QMAX);
    }
    const int64_t row = k * G + half * TH + j;  // group-major payload row
    char* dst = lc + (row * g.row_elems + ch) * BITS / 8;
    if constexpr (BITS == 4) {
      *reinterpret_cast<uint32_t*>(dst) =
          bytes4(lea4(b[1], b[0]), lea4(b[3], b[2]), lea4(b[5], b[4]), lea4(b[7], b[6]));
    } else {
      *reinterpret_cast<uint2*>(dst) =
          make_uint2(bytes4(b[0], b[1], b[2], b[3]), bytes4(b[4], b[5], b[6], b[7]));
    }
  }
}

// G/16 lanes own 8 adjacent channels x G tokens, each lane loading 16 of the
// group's tokens with 16-byte loads (a warp reads 256-byte row segments).
// (A TMA-staged variant -- G row copies per (group, channel block) span into
// a shared-memory ring -- measured 1-21 % slower: the K1 step is bound by
// issue slots, not by loads in flight; profiles/r02_bench/kchan_ab_n1.log.)
template <int BITS, int G>
__global__ void __launch_bounds__(128) quant_pack_kchan_kernel(KchanGeo g, KchanSignal sig) {
  constexpr int TH = 16;      // tokens per lane (16 x 16 B = 64 registers of data)
  constexpr int LPC = G / TH;  // lanes sharing one 8-channel block (2 at G=32, 4 at G=64)
  constexpr int CTA_CH = 4 * (32 / LPC) * 8;  // channels per 128-thread CTA
  const int lane = threadIdx.x & 31;
  const int half = lane % LPC;  // which TH-token slice of the group
  const int cbw = (threadIdx.x >> 5) * (32 / LPC) + lane / LPC;  // 8-channel block in the CTA
  const int cblocks = (g.row_elems + CTA_CH - 1) / CTA_CH;
  const int64_t n_items = g.n_layers * g.n_groups * cblocks;
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int64_t lg = item / cblocks;
    const int cb = int(item - lg * cblocks);
    const int64_t layer = lg / g.n_groups;
    const int64_t k = lg - layer * g.n_groups;
    const int ch = cb * CTA_CH + cbw * 8;
    const bool active = ch < g.row_elems;
    const int64_t t0 = __ldg(g.group_starts + k) + half * TH;
    const char* src = g.k_plane + layer * g.layer_stride_b + (t0 * g.row_elems + ch) * 2;
    uint4 w[TH];
#pragma unroll
    for (int j = 0; j < TH; ++j) {
      if (active) {
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(w[j].x), "=r"(w[j].y), "=r"(w[j].z), "=r"(w[j].w)
                     : "l"(src + int64_t(j) * g.row_elems * 2));
      } else {
        w[j] = make_uint4(0, 0, 0, 0);
      }
    }
    kchan_quant_lanes<BITS, G, TH>(g, w, active, half, layer, k, ch);
    if (sig.peer_flags) {  // fused kivi prefill: this CTA's share of a chunk is done
      const int64_t c = item / sig.items_per_chunk;
      const int64_t nxt = item + gridDim.x;
      if (nxt >= n_items || nxt / sig.items_per_chunk != c) {
        __threadfence();  // this thread's payload stores, device-wide
        __syncthreads();
        if (threadIdx.x == 0) {
          const int64_t a = c * sig.items_per_chunk;
          const int64_t b = min(n_items, a + sig.items_per_chunk);
          const uint32_t owners = uint32_t(min(b - a, int64_t(gridDim.x)));
          __threadfence();
          if (atomicAdd(sig.counters + c, 1u) + 1 == owners) {
            sig.counters[c] = 0u;  // zero again for the next launch
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(sig.peer_flags + c),
                         "r"(sig.ready_value)
                         : "memory");
          }
        }
      }
    }
  }
}

// Dequantise per-channel-grouped K rows into the paged cache.  Warp per
// (layer, group k, block of 32 chunks): each lane loads the 32 scales and 32
// zeros of its channels ONCE (they are shared by the group's G rows -- over
// NVLink re-reading them per row would cost 8x the code bytes) and then walks
// the G rows: 16 B of codes in, 64 B of fp16 out per row.
template <int BITS>
__device__ __forceinline__ void kchan_dequant_store(const uint32_t (&cw)[BITS], const uint32_t (&sw)[16],
                                                    const uint32_t (&zw)[16], char* dst) {
  const __half2 k1024 = u32_as_h2(0x64006400u), kmax = u32_as_h2(0x7BFF7BFFu);
  U4 o[4];
#pragma unroll
  for (int v = 0; v < 4; ++v) {  // 8 elements per output vector
    uint32_t p[4];
    if constexpr (BITS == 4) {
      const uint32_t cc = cw[v];
      const uint32_t a0 = lop3_and_or(cc, 0x000F000Fu, 0x64006400u);
      const uint32_t a1 = lop3_and_or(cc >> 4, 0x000F000Fu, 0x64006400u);
      const uint32_t a2 = lop3_and_or(cc >> 8, 0x000F000Fu, 0x64006400u);
      const uint32_t a3 = lop3_and_or(cc >> 12, 0x000F000Fu, 0x64006400u);
      p[0] = prmt(a0, a1, 0x5410);
      p[1] = prmt(a2, a3, 0x5410);
      p[2] = prmt(a0, a1, 0x7632);
      p[3] = prmt(a2, a3, 0x7632);
    } else {
      p[0] = prmt(cw[2 * v], 0x64646464u, 0x4140);
      p[1] = prmt(cw[2 * v], 0x64646464u, 0x4342);
      p[2] = prmt(cw[2 * v + 1], 0x64646464u, 0x4140);
      p[3] = prmt(cw[2 * v + 1], 0x64646464u, 0x4342);
    }
    uint32_t* ov = &o[v].x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __half2 qh = __hsub2(u32_as_h2(p[i]), k1024);
      const __half2 y = __hfma2(qh, u32_as_h2(sw[4 * v + i]), u32_as_h2(zw[4 * v + i]));
      ov[i] = h2_as_u32(__hmin2(y, kmax));
    }
  }
  st256(dst, o[0], o[1]);
  st256(dst + 32, o[2], o[3]);
}

template <int BITS>
__device__ __forceinline__ void kchan_load_codes(const char* p, uint32_t (&cw)[BITS]) {
  if constexpr (BITS == 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    cw[0] = v.x; cw[1] = v.y; cw[2] = v.z; cw[3] = v.w;
  } else {
    const uint4 v0 = reinterpret_cast<const uint4*>(p)[0];
    const uint4 v1 = reinterpret_cast<const uint4*>(p)[1];
    cw[0] = v0.x; cw[1] = v0.y; cw[2] = v0.z; cw[3] = v0.w;
    cw[4] = v1.x; cw[5] = v1.y; cw[6] = v1.z; cw[7] = v1.w;
  }
}

template <int BITS, int G>
__global__ void __launch_bounds__(256) dequant_kchan_kernel(KchanGeo g, const int64_t* dst_slots,
                                                           char* k_cache, int64_t dst_layer_stride_b) {
  constexpr int CB = 32 * BITS / 8;  // code bytes per 32-channel chunk
  constexpr int U = 4;               // rows in flight per lane
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int cpr = g.row_elems / 32;
  const int cblk = (cpr + 31) / 32;
  const int64_t items = g.n_layers * g.n_groups * cblk;
  for (int64_t it = warp; it < items; it += n_warps) {
    const int64_t lg = it / cblk;
    const int c = int(it - lg * cblk) * 32 + lane;
    const int64_t layer = lg / g.n_groups;
    const int64_t k = lg - layer * g.n_groups;
    if (c >= cpr) continue;
    const char* lc = g.codes + layer * g.payload_ls;
    const char* ls = g.scale + layer * g.payload_ls + (k * g.row_elems + c * 32) * 2;
    const char* lz = g.zero + layer * g.payload_ls + (k * g.row_elems + c * 32) * 2;
    uint32_t sw[16], zw[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 a = reinterpret_cast<const uint4*>(ls)[i];
      const uint4 b = reinterpret_cast<const uint4*>(lz)[i];
      sw[4 * i] = a.x; sw[4 * i + 1] = a.y; sw[4 * i + 2] = a.z; sw[4 * i + 3] = a.w;
      zw[4 * i] = b.x; zw[4 * i + 1] = b.y; zw[4 * i + 2] = b.z; zw[4 * i + 3] = b.w;
    }
    const int64_t t0 = __ldg(g.group_starts + k);
    char* kplane = k_cache + layer * dst_layer_stride_b;
    for (int j0 = 0; j0 < G; j0 += U) {
      uint32_t cw[U][BITS];
      int64_t pos[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t row = k * G + j0 + u;
        pos[u] = __ldg(dst_slots + t0 + j0 + u);
        kchan_load_codes<BITS>(lc + (row * g.row_elems) * BITS / 8 + int64_t(c) * CB, cw[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (pos[u] >= 0)
          kchan_dequant_store<BITS>(cw[u], sw, zw, kplane + pos[u] * g.row_elems * 2 + int64_t(c) * 64);
    }
  }
}

// Bulk-staged variant of dequant_kchan_kernel for a payload read over NVLink
// (the kivi format's pull transport).  Span = (layer, group k, slab of S
// channels): one producer thread stages the group's G code-row slices
// (S*BITS/8 bytes each) plus the slab's S scales and S zeros with
// cp.async.bulk into a STAGES-deep shared-memory ring; 8 consumer warps
// dequantise from shared memory (each thread keeps one 32-channel chunk's
// scales/zeros in registers across the rows it walks) into the paged cache.
struct KchanBulk {
  int slab;          // S channels per span: 32 * 2^n, S/32 divides 256
  int slabs;         // ceil(row_elems / S)
  int64_t n_spans;   // n_layers * n_groups * slabs
  int stage_bytes;   // G * S * BITS/8 + 4 * S
  // per-chunk doorbells (nullable): wait ready[layer / layers_per_chunk] >=
  // ready_value (the hand-off's sequence number) before a span's bulk reads
  // -- one launch consumes a whole hand-off while the prefill side is still
  // producing it
  const uint32_t* ready;
  uint32_t ready_value;
  Ctl* ctl;  // nullable
  int layers_per_chunk;
};

// One K span of the kivi pull: (layer, group k, slab of S channels) -- the
// group's G code-row slices, then its S scales and S zeros, into a stage.
template <int BITS, int G>
__device__ __forceinline__ void kchan_issue_span(const KchanGeo& g, const KchanBulk& kb,
                                                 int64_t sp, uint8_t* buf, uint64_t* bar) {
  const int S = kb.slab;
  const int code_slice = S * BITS / 8;
  const int64_t lg = sp / kb.slabs;
  const int c0 = int(sp - lg * kb.slabs) * S;
  const int64_t layer = lg / g.n_groups, grp = lg - layer * g.n_groups;
  const int ns = min(S, g.row_elems - c0);
  const uint32_t rb = uint32_t(ns) * BITS / 8, mb = uint32_t(ns) * 2;
  mbar_expect_tx(bar, G * rb + 2 * mb);
  const char* lc = g.codes + layer * g.payload_ls + int64_t(c0) * BITS / 8;
  if (ns == g.row_elems && code_slice == int(rb)) {
    // the slab is whole rows: the group's G code rows are one range
    bulk_g2s(buf, lc + grp * G * int64_t(g.row_elems) * BITS / 8, G * rb, bar);
  } else {
    for (int j = 0; j < G; ++j)
      bulk_g2s(buf + j * code_slice, lc + (grp * G + j) * int64_t(g.row_elems) * BITS / 8, rb,
               bar);
  }
  const int64_t meta = (grp * g.row_elems + c0) * 2;
  bulk_g2s(buf + G * code_slice, g.scale + layer * g.payload_ls + meta, mb, bar);
  bulk_g2s(buf + G * code_slice + 2 * S, g.zero + layer * g.payload_ls + meta, mb, bar);
}

// Consumers of one staged K span: each thread keeps one 32-channel chunk's
// scales and zeros in registers and walks the group's rows.
template <int BITS, int G, int CONSUMERS>
__device__ __forceinline__ void kchan_consume_span(const KchanGeo& g, const KchanBulk& kb,
                                                   int64_t sp, const uint8_t* buf,
                                                   const int64_t* __restrict__ dst_slots,
                                                   char* k_cache, int64_t dst_ls_b) {
  constexpr int CB = 32 * BITS / 8;
  const int S = kb.slab;
  const int code_slice = S * BITS / 8;
  const int nck = S / 32;           // 32-channel chunks per full slab
  const int c = threadIdx.x % nck;  // this thread's chunk (fixed across spans)
  const int jstep = (CONSUMERS * 32) / nck;
  const int64_t lg = sp / kb.slabs;
  const int c0 = int(sp - lg * kb.slabs) * S;
  const int64_t layer = lg / g.n_groups, grp = lg - layer * g.n_groups;
  const int ns = min(S, g.row_elems - c0);
  if (c * 32 >= ns) return;
  const uint4* sv = reinterpret_cast<const uint4*>(buf + G * code_slice + c * 64);
  const uint4* zv = reinterpret_cast<const uint4*>(buf + G * code_slice + 2 * S + c * 64);
  uint32_t sw[16], zw[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 a = sv[i], b = zv[i];
    sw[4 * i] = a.x; sw[4 * i + 1] = a.y; sw[4 * i + 2] = a.z; sw[4 * i + 3] = a.w;
    zw[4 * i] = b.x; zw[4 * i + 1] = b.y; zw[4 * i + 2] = b.z; zw[4 * i + 3] = b.w;
  }
  const int64_t t0 = __ldg(g.group_starts + grp);
  char* kplane = k_cache + layer * dst_ls_b + int64_t(c0 + c * 32) * 2;
  for (int j = threadIdx.x / nck; j < G; j += jstep) {
    const int64_t pos = __ldg(dst_slots + t0 + j);
    if (pos < 0) continue;
    uint32_t cw[BITS];
    kchan_load_codes<BITS>(reinterpret_cast<const char*>(buf + j * code_slice + c * CB), cw);
    kchan_dequant_store<BITS>(cw, sw, zw, kplane + pos * int64_t(g.row_elems) * 2);
  }
}

template <int BITS, int G, int STAGES>
__global__ void __launch_bounds__(288, 1) pull_kchan_kernel(KchanGeo g, KchanBulk kb,
                                                            const int64_t* __restrict__ dst_slots,
                                                            char* k_cache, int64_t dst_ls_b) {
  constexpr int CONSUMERS = 8;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  __shared__ uint32_t s_abort;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CONSUMERS);
    }
    s_abort = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == CONSUMERS) {  // ---- producer: one elected thread
    if (lane == 0) {
      int64_t ready_chunk = -1;
      uint32_t k = 0;
      bool ok = true;
      for (int64_t sp = blockIdx.x; sp < kb.n_spans; sp += gridDim.x, ++k) {
        const int st = k % STAGES;
        if (k >= STAGES) mbar_wait(&empty[st], ((k / STAGES) & 1) ^ 1);
        const int64_t layer = (sp / kb.slabs) / g.n_groups;
        if (kb.ready && ok) {
          const int64_t c = layer / kb.layers_per_chunk;
          if (c > ready_chunk) {
            ok = wait_ready(kb.ready + c, kb.ready_value, kb.ctl);
            if (!ok) *reinterpret_cast<volatile uint32_t*>(&s_abort) = 1u;
            ready_chunk = c;
          }
        }
        if (!ok) {  // aborted: release the consumers span by span, no data
          mbar_arrive_empty_phase(&full[st]);
          continue;
        }
        kchan_issue_span<BITS, G>(g, kb, sp, smem + st * kb.stage_bytes, &full[st]);
      }
      // PDL (launched behind the previous hand-off's pull): every span of this
      // CTA is requested, the stream's next kernel may be scheduled
      pdl_launch_dependents();
    }
  } else {  // ---- consumers
    pdl_wait();  // the slot mapping, group starts and the cache are stream-ordered
    uint32_t k = 0;
    for (int64_t sp = blockIdx.x; sp < kb.n_spans; sp += gridDim.x, ++k) {
      const int st = k % STAGES;
      mbar_wait(&full[st], (k / STAGES) & 1);
      if (!*reinterpret_cast<volatile uint32_t*>(&s_abort))
        kchan_consume_span<BITS, G, CONSUMERS>(g, kb, sp, smem + st * kb.stage_bytes, dst_slots,
                                               k_cache, dst_ls_b);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
}

// The residual window of a kivi payload (each request's last n mod G tokens,
// K rows as fp16): rows_per_span rows of one layer per span.
struct KiviResidual {
  const char* rows;           // Kr of layer 0 (payload segment)
  int64_t payload_ls;
  const int64_t* dst_slots;   // [n_rows] paged positions of the residual tokens
  int64_t n_rows;             // residual tokens per layer (0 = none)
  int row_bytes;              // H * D * 2
  int rows_per_span;
  int spans_per_layer;
  int64_t n_spans;            // n_layers * spans_per_layer
};

// The kivi pull as ONE kernel: the per-channel K spans (kchan_*_span) and the
// per-token V spans (bulk_consume_span) share one span space -- K first, then
// V -- and one stage ring sized for the larger kind, so the V rows stream in
// right behind the K groups with no kernel boundary between them.  K spans
// wait on ready[c], V spans on ready[KVX_KIVI_V_FLAGS + c] (c = layer chunk).
// In-kernel completion as in pull_dequant_scatter_kernel (bg.done_counter /
// peer_free, only without residual rows).
template <int BITS, int G, int STAGES>
__global__ void __launch_bounds__(288, 1) pull_kivi_kernel(KchanGeo kg, KchanBulk kb, Geo g,
                                                           BulkGeo bg,
                                                           const uint8_t* __restrict__ vcodes,
                                                           const __half* __restrict__ vscale,
                                                           const __half* __restrict__ vzero,
                                                           const int64_t* __restrict__ dst_slots,
                                                           char* k_cache, int64_t dst_ls_b,
                                                           int stage_bytes, KiviResidual kr) {
  constexpr int CONSUMERS = 8;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  __shared__ uint32_t s_abort;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CONSUMERS);
    }
    s_abort = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nk = kb.n_spans;
  const int64_t nkv = nk + int64_t(bg.n_spans);  // then the residual spans
  const int64_t n_all = nkv + kr.n_spans;
  const int64_t two_t = g.n_tokens;  // V only: one plane
  if (warp == CONSUMERS) {  // ---- producer
    if (lane == 0) {
      int64_t ready_k = -1, ready_v = -1;
      uint32_t k = 0;
      bool ok = true;
      for (int64_t sp = blockIdx.x; sp < n_all; sp += gridDim.x, ++k) {
        const int st = k % STAGES;
        if (k >= STAGES) mbar_wait(&empty[st], ((k / STAGES) & 1) ^ 1);
        uint8_t* buf = smem + st * stage_bytes;
        if (sp < nk) {
          const int64_t c = ((sp / kb.slabs) / kg.n_groups) / kb.layers_per_chunk;
          if (kb.ready && ok && c > ready_k) {
            ok = wait_ready(kb.ready + c, kb.ready_value, kb.ctl);
            ready_k = c;
          }
          if (!ok) {
            *reinterpret_cast<volatile uint32_t*>(&s_abort) = 1u;
            mbar_arrive_empty_phase(&full[st]);
            continue;
          }
          kchan_issue_span<BITS, G>(kg, kb, sp, buf, &full[st]);
        } else if (sp >= nkv) {  // residual fp16 K rows: published with V's chunk
          const int64_t rsp = sp - nkv;
          const int64_t layer = rsp / kr.spans_per_layer;
          const int64_t c = layer / bg.layers_per_chunk;
          if (bg.ready && ok && c > ready_v) {
            ok = wait_ready(bg.ready + c, bg.ready_value, bg.ctl);
            ready_v = c;
          }
          if (!ok) {
            *reinterpret_cast<volatile uint32_t*>(&s_abort) = 1u;
            mbar_arrive_empty_phase(&full[st]);
            continue;
          }
          const int64_t r0 = (rsp - layer * kr.spans_per_layer) * kr.rows_per_span;
          const int rows = int(min(int64_t(kr.rows_per_span), kr.n_rows - r0));
          const uint32_t nb = uint32_t(rows) * kr.row_bytes;
          mbar_expect_tx(&full[st], nb);
          bulk_g2s(buf, kr.rows + layer * kr.payload_ls + r0 * kr.row_bytes, nb, &full[st]);
        } else {
          const uint32_t vsp = uint32_t(sp - nk);
          const uint32_t layer = vsp / bg.spans_per_layer;
          const int64_t c = int64_t(layer) / bg.layers_per_chunk;
          if (bg.ready && ok && c > ready_v) {
            ok = wait_ready(bg.ready + c, bg.ready_value, bg.ctl);
            ready_v = c;
          }
          if (!ok) {
            *reinterpret_cast<volatile uint32_t*>(&s_abort) = 1u;
            mbar_arrive_empty_phase(&full[st]);
            continue;
          }
          const int64_t r0 = int64_t(vsp - layer * bg.spans_per_layer) * bg.rows_per_span;
          const int rows = int(min(int64_t(bg.rows_per_span), two_t - r0));
          const uint32_t cb = rows * bg.code_row_bytes, mb = rows * bg.meta_row_bytes;
          mbar_expect_tx(&full[st], cb + 2 * mb);
          bulk_g2s(buf, vcodes + layer * g.codes_ls + r0 * bg.code_row_bytes, cb, &full[st]);
          const char* sb = reinterpret_cast<const char*>(vscale) + layer * g.meta_ls;
          const char* zb = reinterpret_cast<const char*>(vzero) + layer * g.meta_ls;
          uint8_t* mbuf = buf + bg.rows_per_span * bg.code_row_bytes;
          bulk_g2s(mbuf, sb + r0 * bg.meta_row_bytes, mb, &full[st]);
          bulk_g2s(mbuf + bg.rows_per_span * bg.meta_row_bytes, zb + r0 * bg.meta_row_bytes, mb,
                   &full[st]);
        }
      }
    }
  } else {  // ---- consumers
    pdl_wait();
    uint32_t k = 0;
    for (int64_t sp = blockIdx.x; sp < n_all; sp += gridDim.x, ++k) {
      const int st = k % STAGES;
      const uint8_t* buf = smem + st * stage_bytes;
      mbar_wait(&full[st], (k / STAGES) & 1);
      if (!*reinterpret_cast<volatile uint32_t*>(&s_abort)) {
        if (sp < nk) {
          kchan_consume_span<BITS, G, CONSUMERS>(kg, kb, sp, buf, dst_slots, k_cache, dst_ls_b);
        } else if (sp >= nkv) {  // residual rows: 16-byte copies into the K cache
          const int64_t rsp = sp - nkv;
          const int64_t layer = rsp / kr.spans_per_layer;
          const int64_t r0 = (rsp - layer * kr.spans_per_layer) * kr.rows_per_span;
          const int rows = int(min(int64_t(kr.rows_per_span), kr.n_rows - r0));
          const int vpr = kr.row_bytes / 16;
          for (int i = threadIdx.x; i < rows * vpr; i += CONSUMERS * 32) {
            const int r = i / vpr, v = i - r * vpr;
            const int64_t pos = __ldg(kr.dst_slots + r0 + r);
            if (pos < 0) continue;
            const uint4 x = reinterpret_cast<const uint4*>(buf + int64_t(r) * kr.row_bytes)[v];
            reinterpret_cast<uint4*>(k_cache + layer * dst_ls_b + pos * int64_t(kr.row_bytes))[v] = x;
          }
        } else {
          const uint32_t vsp = uint32_t(sp - nk);
          const uint32_t layer = vsp / bg.spans_per_layer;
          const int64_t r0 = int64_t(vsp - layer * bg.spans_per_layer) * bg.rows_per_span;
          const int rows = int(min(int64_t(bg.rows_per_span), two_t - r0));
          bulk_consume_span<BITS, G, CONSUMERS>(g, bg.code_row_bytes, bg.meta_row_bytes,
                                                bg.rows_per_span, bg.cpr, buf, rows, r0, layer,
                                                warp, lane);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
  if (bg.done_counter) {  // in-kernel slot release (no residual rows)
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t inc = s_abort ? 0x10001u : 1u;
      const uint32_t total = atomicAdd(bg.done_counter, inc) + inc;
      if ((total & 0xFFFFu) == gridDim.x) {
        bg.done_counter[0] = 0u;
        if ((total >> 16) == 0u)
          asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(bg.peer_free),
                       "r"(bg.ready_value)
                       : "memory");
      }
    }
  }
}

}  // namespace kvx
