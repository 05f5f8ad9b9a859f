// Device code of the KV hand-off: K1 quantise+pack, K3 dequantise+paged scatter.
//
// Both kernels are HBM/NVLink-bandwidth kernels (no tensor cores: ~8 flops per
// 2.53 B moved).  Work unit = one "token row": the n_heads*head_dim fp16
// elements of one (layer, K|V, token) -- contiguous on the paged side (vLLM
// flash layout) and contiguous in the dense packed payload.  One warp owns a
// token row at a time (grid-stride over token rows), so slot lookups and
// index math are paid once per 2-8 KB instead of once per element.
//
// Thread -> data: lane handles 16-byte vectors (8 fp16) at vector index
// v = lane + 32*k (k < UNROLL) + 32*UNROLL*iter within the token row.  A
// quantisation group of G elements is G/8 consecutive lanes, so group
// min/max is a half2 hmin2 tree inside the lane plus log2(G/8) xor-shuffles.
//
// Format (bit-exact with oracle/, see include/kvx.h):
//   z = f16(min + 0); s = f16((max - min)/(2^b - 1) + 0)   [IEEE fp32]
//   q = s == 0 ? 0 : min(rint_even(RN32(x - z) * rcp_rn(s)), 2^b - 1)  [product exact]
//   x_hat = f16_rn(min(q*s + z, 65504))     [single-rounding fp16 FMA]
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

namespace kvx {

struct __align__(16) U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 ld_stream(const void* p) {
  // Read-once data: do not allocate in L1.
  U4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(void* p, const U4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint32_t h2_as_u32(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u32_as_h2(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t mask, uint32_t orv) {
  // (a & mask) | orv  in one LOP3
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(mask), "r"(orv));
  return r;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// ---------------------------------------------------------------------------
// Codes <-> 8 elements per lane
// ---------------------------------------------------------------------------
template <int BITS>
struct CodeVec;  // storage for the 8 codes of one 16-byte vector

template <>
struct CodeVec<4> {
  using T = uint32_t;
};
template <>
struct CodeVec<8> {
  using T = uint2;
};
template <>
struct CodeVec<2> {
  using T = uint16_t;
};

// Dequantise 8 codes to 8 fp16 with a single-rounding fp16 FMA.
template <int BITS>
__device__ __forceinline__ U4 dequant8(typename CodeVec<BITS>::T c, __half2 s2, __half2 z2) {
  const __half2 k1024 = u32_as_h2(0x64006400u);   // (1024, 1024)
  const __half2 kmax = u32_as_h2(0x7BFF7BFFu);    // (65504, 65504)
  uint32_t p[4];  // half2 pairs, each holding (1024 + q_a, 1024 + q_b)
  if constexpr (BITS == 4) {
    // pairs (n_j, n_{j+4}) by shift+LOP3, then PRMT back to element order.
    uint32_t a0 = lop3_and_or(c, 0x000F000Fu, 0x64006400u);        // (n0, n4)
    uint32_t a1 = lop3_and_or(c >> 4, 0x000F000Fu, 0x64006400u);   // (n1, n5)
    uint32_t a2 = lop3_and_or(c >> 8, 0x000F000Fu, 0x64006400u);   // (n2, n6)
    uint32_t a3 = lop3_and_or(c >> 12, 0x000F000Fu, 0x64006400u);  // (n3, n7)
    p[0] = prmt(a0, a1, 0x5410);  // (n0, n1)
    p[1] = prmt(a2, a3, 0x5410);  // (n2, n3)
    p[2] = prmt(a0, a1, 0x7632);  // (n4, n5)
    p[3] = prmt(a2, a3, 0x7632);  // (n6, n7)
  } else if constexpr (BITS == 8) {
    p[0] = prmt(c.x, 0x64646464u, 0x4140);
    p[1] = prmt(c.x, 0x64646464u, 0x4342);
    p[2] = prmt(c.y, 0x64646464u, 0x4140);
    p[3] = prmt(c.y, 0x64646464u, 0x4342);
  } else {
    uint32_t w = c;
    w = w | (w << 14);  // element 2i at bits [2i,2i+2), element 2i+1 moved to bit 16+2i
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = lop3_and_or(w >> (4 * i), 0x00030003u, 0x64006400u);
  }
  U4 out;
  uint32_t* o = &out.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __half2 qh = __hsub2(u32_as_h2(p[i]), k1024);  // exact
    __half2 y = __hfma2(qh, s2, z2);               // RN16(q*s + z), one rounding
    o[i] = h2_as_u32(__hmin2(y, kmax));            // saturate (+inf -> 65504)
  }
  return out;
}

// Token-row geometry shared by both kernels.
struct Geo {
  const char* k_plane;     // K plane of layer 0 (paged/dense side)
  const char* v_plane;     // V plane of layer 0
  int64_t layer_stride_b;  // bytes between layers on the paged/dense side
  const int64_t* slots;    // token -> position on the paged side (nullable)
  int64_t n_tokens;
  int64_t n_token_rows;    // n_layers * 2 * n_tokens
  int64_t codes_ls;        // payload: bytes between layers of the codes array
  int64_t meta_ls;         // payload: bytes between layers of scale / zero
  int row_elems;           // n_heads * head_dim
  int vecs;                // row_elems / 8
  int planes;              // planes per layer in this launch: 2 (K and V) or 1
  int plane0;              // first plane: 0 = K, 1 = V (planes == 1: which one)
  int64_t plane_row_b;     // bytes per token row on the paged side (all its heads)
  int64_t head_off_b;      // byte offset of this launch's head window in that row
#ifdef KVX_DEBUG
  int64_t dbg_rows;        // debug builds: token positions one layer plane holds (0 = unknown)
#endif
};

// Token row `pos` of a plane, at this launch's head window (TP head shards:
// a prefill rank packs, or a decode rank scatters, a sub-range of heads).
__device__ __forceinline__ const char* row_ptr(const Geo& g, const char* plane, int64_t pos) {
  return plane + pos * g.plane_row_b + g.head_off_b;
}

__device__ __forceinline__ const char* plane_ptr(const Geo& g, int kv, int64_t layer) {
  return (kv ? g.v_plane : g.k_plane) + layer * g.layer_stride_b;
}

__device__ __forceinline__ int64_t pos_of(const Geo& g, int64_t t) {
  const int64_t p = g.slots ? __ldg(g.slots + t) : t;
#ifdef KVX_DEBUG
  // debug builds (-DKVX_DEBUG, the sanitizer stand-in): a position past the
  // plane the caller's layer stride describes is an out-of-bounds access
  if (g.dbg_rows > 0 && p >= g.dbg_rows) {
    printf("kvx debug: token %lld -> position %lld outside the plane (%lld rows)\n",
           (long long)t, (long long)p, (long long)g.dbg_rows);
    __trap();
  }
#endif
  return p;
}

// Token row tr = (l*planes + p)*T + t -> (plane kv, layer, row inside the
// layer's payload).
__device__ __forceinline__ void split_tr(const Geo& g, int64_t tr, int& kv, int64_t& t,
                                         int64_t& layer, int64_t& lrow) {
  const int64_t lk = tr / g.n_tokens;
  t = tr - lk * g.n_tokens;
  layer = lk >> (g.planes - 1);
  kv = g.plane0 + int(lk - (layer << (g.planes - 1)));
  lrow = tr - layer * g.planes * g.n_tokens;
}

// ---------------------------------------------------------------------------
// K1: quantise + pack.  codes/scale/zero may be peer (NVLink push) pointers.
//
// Lane owns a 32-element chunk (64 B = two 256-bit LDG.E.256 loads); a group
// of G elements is G/32 consecutive lanes (4 at G=128), so per-group scalar
// work (one IEEE divide, one IEEE reciprocal) is amortised over 32 elements
// and the min/max reduction needs at most two shuffles.  Per element the
// fast path is FHADD (f16 - f32 -> f32, the exact-input subtraction), half an
// FFMA2 (t*inv + 2^23: fused multiply + round-half-even), and ~0.9 integer
// ops of nibble packing (LEA/PRMT on the raw float bits).  Work items are
// (token row, 32-chunk block); each warp software-pipelines its items
// (loads of item i+1 in flight while item i is computed).
// ---------------------------------------------------------------------------
struct FastDiv {  // n / d for n < 2^31 via mul-hi (host-precomputed magic)
  uint32_t d, m, s;
};

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return (__umulhi(n, f.m) + n) >> f.s;
}

struct ItemGeo {
  FastDiv ipr;      // items (32-chunk blocks) per token row
  FastDiv tokens;   // n_tokens
  int cpr;          // 32-element chunks per token row
  uint32_t n_items;
  // short rows (cpr < 32, a power of two -- e.g. a TP shard's few KV heads):
  // one item packs 2^rpi_shift consecutive rows of one layer so every lane
  // has a chunk; rpi_shift == 0 is the one-row-per-item geometry
  int rpi_shift;
  int cpr_shift;    // log2(cpr) when rows are packed
  FastDiv ipl;      // items per layer when rows are packed
  uint32_t pt;      // token rows per layer (planes * n_tokens)
};

// (token row, chunk) of this lane's share of ``item``; false = no work
// (beyond the row's chunks or the layer's rows; tr stays a valid row).
template <bool PACKED = true>
__device__ __forceinline__ bool item_row_chunk(const ItemGeo& ig, uint32_t item, int lane,
                                               uint32_t& tr, int& c) {
  if (!PACKED || ig.rpi_shift == 0) {
    tr = fdiv(item, ig.ipr);
    c = int(item - tr * ig.ipr.d) * 32 + lane;
    return c < ig.cpr;
  }
  const uint32_t layer = fdiv(item, ig.ipl);
  const uint32_t r = ((item - layer * ig.ipl.d) << ig.rpi_shift) + (uint32_t(lane) >> ig.cpr_shift);
  c = lane & (ig.cpr - 1);
  const bool ok = r < ig.pt;
  tr = layer * ig.pt + (ok ? r : 0u);
  return ok;
}

__device__ __forceinline__ void ld256(const void* p, uint32_t (&r)[8]) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "l"(p));
}

// x(f16, low or high half of h2) - z(f32) -> f32, one FHADD, exact inputs, RN.
__device__ __forceinline__ float sub_lo(uint32_t h2, float z) {
  float r;
  asm("{.reg .f16 l, h; mov.b32 {l, h}, %1; sub.rn.f32.f16 %0, l, %2;}" : "=f"(r) : "r"(h2), "f"(z));
  return r;
}
__device__ __forceinline__ float sub_hi(uint32_t h2, float z) {
  float r;
  asm("{.reg .f16 l, h; mov.b32 {l, h}, %1; sub.rn.f32.f16 %0, h, %2;}" : "=f"(r) : "r"(h2), "f"(z));
  return r;
}

// (a, b) * inv + 2^23 in one FFMA2; returns the raw bits of both results.
__device__ __forceinline__ void fma_magic2(float a, float b, float inv, uint32_t& ra,
                                           uint32_t& rb) {
  unsigned long long x, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a), "f"(b));
  asm("{.reg .b64 iv, mg; mov.b64 iv, {%2, %2}; mov.b64 mg, {%3, %3};"
      " fma.rn.f32x2 %0, %1, iv, mg;}"
      : "=l"(r) : "l"(x), "f"(inv), "f"(8388608.0f));
  ra = uint32_t(r);
  rb = uint32_t(r >> 32);
}

__device__ __forceinline__ uint32_t lea4(uint32_t hi, uint32_t lo) { return (hi << 4) + lo; }
__device__ __forceinline__ uint32_t lea2(uint32_t hi, uint32_t lo) { return (hi << 2) + lo; }

// Gather the low bytes of 4 words into one word: [a0, b0, c0, d0].
__device__ __forceinline__ uint32_t bytes4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return prmt(prmt(a, b, 0x0040u), prmt(c, d, 0x0040u), 0x5410u);
}

template <int BITS>
struct Chunk32 {  // packed codes of 32 elements
  static constexpr int WORDS = BITS;  // 32*BITS/32
  uint32_t w[WORDS];
};

// q bits (raw float bits with q in the low byte) of 32 elements -> packed codes.
template <int BITS>
__device__ __forceinline__ Chunk32<BITS> pack32(const uint32_t (&b)[32]) {
  Chunk32<BITS> out;
  if constexpr (BITS == 4) {
    uint32_t p[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) p[i] = lea4(b[2 * i + 1], b[2 * i]);
#pragma unroll
    for (int k = 0; k < 4; ++k) out.w[k] = bytes4(p[4 * k], p[4 * k + 1], p[4 * k + 2], p[4 * k + 3]);
  } else if constexpr (BITS == 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) out.w[k] = bytes4(b[4 * k], b[4 * k + 1], b[4 * k + 2], b[4 * k + 3]);
  } else {
    uint32_t p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      p[i] = lea4(lea2(b[4 * i + 3], b[4 * i + 2]), lea2(b[4 * i + 1], b[4 * i]));
#pragma unroll
    for (int k = 0; k < 2; ++k) out.w[k] = bytes4(p[4 * k], p[4 * k + 1], p[4 * k + 2], p[4 * k + 3]);
  }
  return out;
}

template <int BITS>
__device__ __forceinline__ void store_chunk(void* dst, const Chunk32<BITS>& c) {
  if constexpr (BITS == 4) {
    asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "r"(c.w[0]), "r"(c.w[1]),
                 "r"(c.w[2]), "r"(c.w[3]) : "memory");
  } else if constexpr (BITS == 8) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(c.w[0]),
                 "r"(c.w[1]), "r"(c.w[2]), "r"(c.w[3]), "r"(c.w[4]), "r"(c.w[5]), "r"(c.w[6]),
                 "r"(c.w[7]) : "memory");
  } else {
    asm volatile("st.global.v2.b32 [%0], {%1,%2};" ::"l"(dst), "r"(c.w[0]), "r"(c.w[1]) : "memory");
  }
}

struct K1Item {
  const char* src;   // this lane's 64 source bytes (valid iff active)
  char* codes;       // this lane's code bytes
  __half* scale;     // group scale slot (this lane's group)
  __half* zero;
  bool active;
};

template <int BITS, int G>
__device__ __forceinline__ K1Item k1_item(const Geo& g, const ItemGeo& ig, uint32_t item, int lane,
                                          uint8_t* codes, __half* scale, __half* zero) {
  constexpr int CB = 32 * BITS / 8;  // code bytes per chunk
  K1Item it;
  uint32_t tr;
  int c;  // chunk inside the token row
  const bool ok = item_row_chunk(ig, item, lane, tr, c);
  const uint32_t lk = fdiv(tr, ig.tokens);
  const uint32_t t = tr - lk * ig.tokens.d;
  const uint32_t layer = lk >> (g.planes - 1);
  const int kv = g.plane0 + int(lk - (layer << (g.planes - 1)));
  const uint32_t lrow = tr - layer * g.planes * ig.tokens.d;
  const int64_t pos = pos_of(g, t);
  const char* plane = plane_ptr(g, kv, layer);
  it.active = ok;
  it.src = row_ptr(g, plane, pos) + int64_t(c) * 64;
  it.codes = reinterpret_cast<char*>(codes) + int64_t(layer) * g.codes_ls +
             (int64_t(lrow) * ig.cpr + c) * CB;
  const int64_t gi = (int64_t(lrow) * ig.cpr + c) * 32 / G;
  it.scale = reinterpret_cast<__half*>(reinterpret_cast<char*>(scale) + int64_t(layer) * g.meta_ls) + gi;
  it.zero = reinterpret_cast<__half*>(reinterpret_cast<char*>(zero) + int64_t(layer) * g.meta_ls) + gi;
  return it;
}

// Packed codes of a lane whose four 16-byte source pieces were loaded in the
// rotated order j -> (j + rot) & 3 (K1-bulk's conflict-free shared-memory
// reads): min/max and the per-element rounding are order-free, only the code
// positions are not -- move code piece (m - rot) & 3 to piece m.
template <int BITS>
__device__ __forceinline__ void unrotate_codes(Chunk32<BITS>& c, int rot) {
  if constexpr (BITS == 2) {  // 16 bits of codes per piece, two pieces per word
    uint64_t v = (uint64_t(c.w[1]) << 32) | c.w[0];
    const int sh = 16 * rot;
    v = sh ? (v << sh) | (v >> (64 - sh)) : v;
    c.w[0] = uint32_t(v);
    c.w[1] = uint32_t(v >> 32);
  } else {
    constexpr int WP = BITS / 4 * 1;  // words per piece: 1 at 4-bit, 2 at 8-bit
    uint32_t t[4 * WP];
#pragma unroll
    for (int i = 0; i < 4 * WP; ++i) t[i] = c.w[i];
    if (rot & 2) {
#pragma unroll
      for (int i = 0; i < 2 * WP; ++i) {
        const uint32_t a = t[i];
        t[i] = t[i + 2 * WP];
        t[i + 2 * WP] = a;
      }
    }
    if (rot & 1) {  // (p0, p1, p2, p3) -> (p3, p0, p1, p2)
      uint32_t last[WP];
#pragma unroll
      for (int i = 0; i < WP; ++i) last[i] = t[3 * WP + i];
#pragma unroll
      for (int i = 4 * WP - 1; i >= WP; --i) t[i] = t[i - WP];
#pragma unroll
      for (int i = 0; i < WP; ++i) t[i] = last[i];
    }
#pragma unroll
    for (int i = 0; i < 4 * WP; ++i) c.w[i] = t[i];
  }
}

template <int BITS, int G, bool ROT = false>
__device__ __forceinline__ void k1_process(const K1Item& it, const uint32_t (&w)[16], int lane,
                                           int rot = 0) {
  constexpr int LPG = G / 32;
  constexpr float QMAXF = float((1 << BITS) - 1);
  constexpr uint32_t QMAX = (1u << BITS) - 1u;
  // group min and -max as one half2 (tree for ILP)
  __half2 mn[8], mx[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    mn[i] = __hmin2(u32_as_h2(w[2 * i]), u32_as_h2(w[2 * i + 1]));
    mx[i] = __hmax2(u32_as_h2(w[2 * i]), u32_as_h2(w[2 * i + 1]));
  }
#pragma unroll
  for (int st = 4; st > 0; st >>= 1)
#pragma unroll
    for (int i = 0; i < st; ++i) {
      mn[i] = __hmin2(mn[i], mn[i + st]);
      mx[i] = __hmax2(mx[i], mx[i + st]);
    }
  __half2 r = __halves2half2(__hmin(__low2half(mn[0]), __high2half(mn[0])),
                             __hneg(__hmax(__low2half(mx[0]), __high2half(mx[0]))));
#pragma unroll
  for (int off = LPG / 2; off > 0; off >>= 1)
    r = __hmin2(r, u32_as_h2(__shfl_xor_sync(0xffffffffu, h2_as_u32(r), off)));
  const float fmn = __low2float(r);
  const float fmx = -__high2float(r);
  const __half z16 = __float2half_rn(__fadd_rn(fmn, 0.0f));
  const float sq = __fdiv_rn(__fsub_rn(fmx, fmn), QMAXF);
  const __half s16 = __float2half_rn(__fadd_rn(sq, 0.0f));
  const float s = __half2float(s16);
  const float inv = (s != 0.0f) ? __frcp_rn(s) : 0.0f;
  const float z = __half2float(z16);
  // Only a subnormal scale can push rint(t*inv) past 2^bits-1.
  const bool clamp = __any_sync(0xffffffffu, it.active && s != 0.0f && s < 6.103515625e-05f);
  uint32_t b[32];
#pragma unroll
  for (int i = 0; i < 16; ++i) fma_magic2(sub_lo(w[i], z), sub_hi(w[i], z), inv, b[2 * i], b[2 * i + 1]);
  if (clamp) {
#pragma unroll
    for (int i = 0; i < 32; ++i) b[i] = min(b[i] - 0x4B000000u, QMAX);
  }
  Chunk32<BITS> out = pack32<BITS>(b);
  if constexpr (ROT) unrotate_codes<BITS>(out, rot);
  if (it.active) {
    store_chunk<BITS>(it.codes, out);
    if ((lane & (LPG - 1)) == 0) {
      *it.scale = s16;
      *it.zero = z16;
    }
  }
}

#ifndef KVX_K1_MIN_BLOCKS
#define KVX_K1_MIN_BLOCKS 2  // keep 2 CTAs (16 warps) per SM: <= 128 registers
#endif
#ifndef KVX_K1_PF
#define KVX_K1_PF 2  // items prefetched ahead per warp (A/B: profiles/r01_summary.md)
#endif
// Device-side doorbells for the fused quantise -> NVLink-pull pipeline: with
// `sig.peer_flags` set, every warp arrives once per layer chunk it touched,
// right after its last item of that chunk; the last arriving warp publishes
// the chunk to the decode GPU (fence.sys + st.release.sys into the peer's
// ready flag).  Warps walk items in global order, so chunks complete
// progressively while the kernel is still running: ONE launch feeds the
// decode side layer by layer, no per-chunk launches or host round trips.
constexpr int kMaxSignalChunks = 64;  // = transport.PULL_MAX_CHUNKS

// Hand-off timeline tracing (A/B builds only: -DKVX_TRACE, see
// tools/handoff_trace.py).  Per launch of K1-signal (kind 0) and K3-bulk with
// completion (kind 1): %globaltimer stamps of the key protocol events.
#ifdef KVX_TRACE
constexpr int kTraceLaunches = 4096;
__device__ unsigned long long g_trace[2][kTraceLaunches][4];
__device__ unsigned int g_trace_n[2];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define KVX_TRACE_STAMP(kind, launch, slot) \
  (g_trace[kind][(launch) % kTraceLaunches][slot] = gtimer())
#else
#define KVX_TRACE_STAMP(kind, launch, slot) ((void)0)
#endif

// Host-mapped control block of one channel (include/kvx.h, kvx_ctl): the
// host writes `abort`, the kernels report through `status`; `timeout_ns`
// bounds every in-kernel wait (0 = the 60 s default).  Nullable: without one
// a wait that times out traps (there is nowhere to report it).
struct Ctl {
  uint32_t abort;
  uint32_t status;
  unsigned long long timeout_ns;
};
constexpr uint32_t kStatusAborted = 1u;
constexpr uint32_t kStatusTimeout = 2u;
constexpr unsigned long long kDefaultTimeoutNs = 60ull * 1000000000ull;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Bounded, abortable spin until a doorbell reaches `value`.  Doorbells carry
// per-slot sequence numbers that only grow, so the test is the wrap-safe
// (int32)(*flag - value) >= 0, and a flag left over from an earlier use of
// the slot (always < value) can never satisfy it.  System-scope acquire: the
// flag is written by the partner GPU over NVLink.  Returns false -- after
// recording why in ctl->status -- when the host aborted the channel or the
// wait outlived ctl->timeout_ns; the kernel then winds down instead of
// trapping, so the CUDA context (and the decode GPU's KV cache) survive a
// lost partner.
__device__ __noinline__ bool spin_until_geq(const uint32_t* flag, uint32_t value, Ctl* ctl) {
  unsigned long long t0 = 0, limit = kDefaultTimeoutNs;
  for (uint32_t spin = 0;; ++spin) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    const int32_t d = int32_t(v - value);
#ifdef KVX_DEBUG
    // the sequence protocol: a doorbell is never ahead of the value awaited
    // (the partner cannot reuse a slot this side has not released)
    if (d > 0 && d < (1 << 29)) {
      printf("kvx debug: doorbell %u ahead of the awaited %u\n", v, value);
      __trap();
    }
#endif
    if (d >= 0) {
      // A live doorbell is at most the awaited value (the partner cannot run
      // a slot's use ahead of this side); a jump of >= 2^29 is the host's
      // abort poison (PairChannel.abort releasing the GPU front-end waits).
      if (d < (1 << 29)) return true;
      if (!ctl) __trap();
      asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(&ctl->status), "r"(kStatusAborted)
                   : "memory");
      return false;
    }
    if ((spin & 255u) == 255u) {  // every 256 polls: the abort word and the clock
      const unsigned long long now = globaltimer_ns();
      if (spin == 255u) {
        t0 = now;
        if (ctl) {
          unsigned long long tl;
          asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(tl) : "l"(&ctl->timeout_ns));
          if (tl) limit = tl;
        }
      }
      uint32_t ab = 0;
      if (ctl) asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(ab) : "l"(&ctl->abort));
      if (ab || now - t0 > limit) {
        if (!ctl) __trap();
        asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(&ctl->status),
                     "r"(ab ? kStatusAborted : kStatusTimeout)
                     : "memory");
        return false;
      }
    }
    __nanosleep(spin < 64 ? 32 : 256);
  }
}

// Programmatic dependent launch (kernels launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): let the next kernel of
// the stream be scheduled now / wait until every earlier grid of the stream
// has completed and its memory is visible.  Both are no-ops without PDL.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

struct SignalGeo {
  // [kMaxSignalChunks] chunk arrivals: zero at launch, and reset in-kernel by
  // each chunk's last arrival, so zero again after every launch
  uint32_t* counters;
  uint32_t* peer_flags;  // [n_chunks] decode-side ready flags (IPC/peer mapped), or null
  uint32_t items_per_chunk;
  FastDiv ipc;           // items_per_chunk as a multiply-shift (per-item chunk test)
  uint32_t ready_value;  // this hand-off's sequence number v: doorbells are set to v
  // queue slot free (nullable, this GPU's memory, written by the decode side
  // over NVLink): every CTA waits *free_flag >= free_value (v - 1: the
  // slot's previous use consumed) before it stores into the slot
  const uint32_t* free_flag;
  uint32_t free_value;
  Ctl* ctl;  // nullable
#ifdef KVX_TRACE
  uint32_t trace_id;  // trace builds: the hand-off's epoch (row of the timeline ring)
#endif
};

// Warps w in [lo, hi) that own at least one item i in [a, b) (item i -> warp i % W).
__device__ __forceinline__ uint32_t warps_owning(uint32_t a, uint32_t b, uint32_t W, uint32_t lo,
                                                 uint32_t hi) {
  auto ov = [](uint32_t x0, uint32_t x1, uint32_t y0, uint32_t y1) -> uint32_t {
    const uint32_t l = max(x0, y0), h = min(x1, y1);
    return h > l ? h - l : 0u;
  };
  if (b - a >= W) return hi - lo;
  const uint32_t w0 = a % W, w1 = (b - 1) % W;
  if (w0 <= w1) return ov(w0, w1 + 1, lo, hi);
  return ov(w0, W, lo, hi) + ov(0, w1 + 1, lo, hi);
}

// CTAs (8 warps each) owning at least one item of [a, b).
__device__ __forceinline__ uint32_t ctas_owning(uint32_t a, uint32_t b, uint32_t W) {
  if (b - a >= W) return W / 8;
  const uint32_t w0 = a % W, w1 = (b - 1) % W;
  if (w0 <= w1) return (w1 >> 3) - (w0 >> 3) + 1;
  const uint32_t c0 = ((W - 1) >> 3) - (w0 >> 3) + 1, c1 = (w1 >> 3) + 1;
  const uint32_t dup = (w1 >> 3) >= (w0 >> 3) ? (w1 >> 3) - (w0 >> 3) + 1 : 0u;
  return c0 + c1 - dup;
}

// Two-level arrival: warps count in shared memory, the CTA's last warp adds
// one to the global chunk counter, the last CTA rings the peer's doorbell
// (a same-address global atomic per warp would serialise for small hand-offs).
__device__ __forceinline__ void chunk_arrive(const SignalGeo& sig, uint32_t* cta_cnt, uint32_t c,
                                             uint32_t n_items, uint32_t n_warps, int lane,
                                             uint32_t ready_value) {
  __threadfence();  // this lane's payload stores, device-wide
  __syncwarp();
  if (lane == 0) {
    const uint32_t a = c * sig.items_per_chunk;
    const uint32_t b = min(n_items, a + sig.items_per_chunk);
    const uint32_t lo = blockIdx.x * (blockDim.x >> 5);
    const uint32_t mine = warps_owning(a, b, n_warps, lo, lo + (blockDim.x >> 5));
    if (atomicAdd_block(cta_cnt + c, 1u) + 1 == mine) {
      __threadfence();
      if (atomicAdd(sig.counters + c, 1u) + 1 == ctas_owning(a, b, n_warps)) {
        sig.counters[c] = 0u;  // every owner has arrived: ready for the next launch
        // st.release.sys is cumulative over the payload stores this thread has
        // observed through the arrival atomics (it carries its own MEMBAR.SYS)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(sig.peer_flags + c),
                     "r"(ready_value)
                     : "memory");
#ifdef KVX_TRACE
        if ((c + 1) * sig.items_per_chunk >= n_items) KVX_TRACE_STAMP(0, sig.trace_id, 2);
#endif
      }
    }
  }
}

template <int BITS, int G>
__global__ void __launch_bounds__(256, KVX_K1_MIN_BLOCKS) quant_pack_kernel(Geo g, ItemGeo ig,
                                                         uint8_t* __restrict__ codes,
                                                         __half* __restrict__ scale,
                                                         __half* __restrict__ zero,
                                                         SignalGeo sig) {
  // Ring of PF+1 register buffers: the loads of the next PF items are in
  // flight while the current one is quantised (all indices compile-time).
  constexpr int NB = KVX_K1_PF + 1;
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t n_warps = (gridDim.x * blockDim.x) >> 5;
  __shared__ uint32_t cta_cnt[kMaxSignalChunks];
  __shared__ uint32_t s_go;
#ifdef KVX_TRACE
  const uint32_t trace_id = sig.trace_id;
  if (sig.peer_flags && blockIdx.x == 0 && threadIdx.x == 0) KVX_TRACE_STAMP(0, trace_id, 0);
#endif
  // PDL launches (kvx_pair_send with KVX_PAIR_PDL): wait for the stream's
  // previous grid and its memory before reading anything (a no-op otherwise)
  pdl_wait();
  if (sig.peer_flags) {
    for (int i = threadIdx.x; i < kMaxSignalChunks; i += blockDim.x) cta_cnt[i] = 0u;
    if (threadIdx.x == 0) {
      // the decode side is done with this queue slot's previous use
      s_go = sig.free_flag ? spin_until_geq(sig.free_flag, sig.free_value, sig.ctl) : 1u;
      if (blockIdx.x == 0) KVX_TRACE_STAMP(0, trace_id, 1);
    }
    __syncthreads();
    if (!s_go) return;  // aborted / timed out (ctl->status says which)
  }
  const uint32_t ready_value = sig.ready_value;
  uint32_t w[NB][16];
  K1Item it[NB];
#pragma unroll
  for (int i = 0; i < NB - 1; ++i) {
    const uint32_t itm = warp + i * n_warps;
    if (itm < ig.n_items) {
      it[i] = k1_item<BITS, G>(g, ig, itm, lane, codes, scale, zero);
      if (it[i].active) {
        ld256(it[i].src, *reinterpret_cast<uint32_t(*)[8]>(&w[i][0]));
        ld256(it[i].src + 32, *reinterpret_cast<uint32_t(*)[8]>(&w[i][8]));
      }
    }
  }
  for (uint32_t base = warp; base < ig.n_items; base += NB * n_warps) {
#pragma unroll
    for (int st = 0; st < NB; ++st) {
      const uint32_t cur = base + st * n_warps;
      if (cur >= ig.n_items) goto k1_done;  // warp-uniform
      const uint32_t pre = cur + (NB - 1) * n_warps;
      const int pb = (st + NB - 1) % NB;
      if (pre < ig.n_items) {
        it[pb] = k1_item<BITS, G>(g, ig, pre, lane, codes, scale, zero);
        if (it[pb].active) {
          ld256(it[pb].src, *reinterpret_cast<uint32_t(*)[8]>(&w[pb][0]));
          ld256(it[pb].src + 32, *reinterpret_cast<uint32_t(*)[8]>(&w[pb][8]));
        }
      }
      k1_process<BITS, G>(it[st], w[st], lane);
      if (sig.peer_flags) {
        const uint32_t c = fdiv(cur, sig.ipc);
        const uint32_t nxt = cur + n_warps;
        if (nxt >= ig.n_items || fdiv(nxt, sig.ipc) != c)
          chunk_arrive(sig, cta_cnt, c, ig.n_items, n_warps, lane, ready_value);
      }
    }
  }
k1_done:
  // this warp's items are done: the stream's next kernel may be scheduled
  // (it waits for this grid's completion before it reads anything)
  pdl_launch_dependents();
#ifdef KVX_TRACE
  if (sig.peer_flags) {  // trace builds: stamp the last CTA's exit
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(sig.counters + kMaxSignalChunks, 1u) == gridDim.x - 1) {
      sig.counters[kMaxSignalChunks] = 0u;
      KVX_TRACE_STAMP(0, trace_id, 3);
      atomicMax(&g_trace_n[0], trace_id + 1);
    }
  }
#endif
  return;
}

// 16-bit passthrough on the prefill side: copy rows into the dense payload.
template <int UNROLL>
__global__ void __launch_bounds__(256) pack16_kernel(Geo g, uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t tr = warp; tr < g.n_token_rows; tr += n_warps) {
    int kv;
    int64_t t, layer, lrow;
    split_tr(g, tr, kv, t, layer, lrow);
    const int64_t pos = pos_of(g, t);
    const char* plane = plane_ptr(g, kv, layer);
    const U4* src = reinterpret_cast<const U4*>(row_ptr(g, plane, pos));
    U4* dst = reinterpret_cast<U4*>(out + layer * g.codes_ls) + lrow * g.vecs;
    for (int base = 0; base < g.vecs; base += 32 * UNROLL) {
      U4 v[UNROLL];
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) {
        const int vi = base + k * 32 + lane;
        if (vi < g.vecs) v[k] = ld_stream(src + vi);
      }
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) {
        const int vi = base + k * 32 + lane;
        if (vi < g.vecs) st_stream(dst + vi, v[k]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K3: unpack + dequantise + scatter into the paged cache.  codes/scale/zero
// may be peer (NVLink pull) pointers.  Token rows with slot < 0 are skipped.
// ---------------------------------------------------------------------------
// Lane owns a 32-element chunk: one 16-byte code load (4-bit; 32 B at 8-bit,
// 8 B at 2-bit) -- wide requests matter when the payload is read over NVLink
// -- and two 256-bit stores into the paged cache.  Items and software
// pipelining as in K1.
struct K3Item {
  const char* codes;
  const __half* scale;
  const __half* zero;
  char* dst;
  bool active;
};

template <int BITS, int G, bool PACKED>
__device__ __forceinline__ K3Item k3_item(const Geo& g, const ItemGeo& ig, uint32_t item, int lane,
                                          const uint8_t* codes, const __half* scale,
                                          const __half* zero) {
  constexpr int CB = 32 * BITS / 8;
  K3Item it;
  uint32_t tr;
  int c;
  const bool ok = item_row_chunk<PACKED>(ig, item, lane, tr, c);
  const uint32_t lk = fdiv(tr, ig.tokens);
  const uint32_t t = tr - lk * ig.tokens.d;
  const uint32_t layer = lk >> (g.planes - 1);
  const int kv = g.plane0 + int(lk - (layer << (g.planes - 1)));
  const uint32_t lrow = tr - layer * g.planes * ig.tokens.d;
  const int64_t pos = pos_of(g, t);
  char* plane = const_cast<char*>(plane_ptr(g, kv, layer));
  it.active = ok && (pos >= 0);  // pos < 0: padding token, skipped
  it.dst = const_cast<char*>(row_ptr(g, plane, pos)) + int64_t(c) * 64;
  it.codes = reinterpret_cast<const char*>(codes) + int64_t(layer) * g.codes_ls +
             (int64_t(lrow) * ig.cpr + c) * CB;
  const int64_t gi = (int64_t(lrow) * ig.cpr + c) * 32 / G;
  it.scale = reinterpret_cast<const __half*>(reinterpret_cast<const char*>(scale) +
                                             int64_t(layer) * g.meta_ls) + gi;
  it.zero = reinterpret_cast<const __half*>(reinterpret_cast<const char*>(zero) +
                                            int64_t(layer) * g.meta_ls) + gi;
  return it;
}

template <int BITS>
struct K3Data {
  Chunk32<BITS> c;
  __half s, z;
};

template <int BITS>
__device__ __forceinline__ void k3_load(const K3Item& it, K3Data<BITS>& d) {
  if (!it.active) return;
  if constexpr (BITS == 4) {
#ifndef KVX_K3_PLAIN_HINTS  // L2 fetches 256 B around each code load (A/B: ~0.5 %)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(d.c.w[0]), "=r"(d.c.w[1]), "=r"(d.c.w[2]), "=r"(d.c.w[3])
                 : "l"(it.codes));
#else
    asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(d.c.w[0]), "=r"(d.c.w[1]), "=r"(d.c.w[2]), "=r"(d.c.w[3])
                 : "l"(it.codes));
#endif
  } else if constexpr (BITS == 8) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(d.c.w[0]), "=r"(d.c.w[1]), "=r"(d.c.w[2]), "=r"(d.c.w[3]),
                   "=r"(d.c.w[4]), "=r"(d.c.w[5]), "=r"(d.c.w[6]), "=r"(d.c.w[7])
                 : "l"(it.codes));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.v2.b32 {%0,%1}, [%2];"
                 : "=r"(d.c.w[0]), "=r"(d.c.w[1])
                 : "l"(it.codes));
  }
  d.s = __ldg(it.scale);
  d.z = __ldg(it.zero);
}

__device__ __forceinline__ void st256(void* p, const U4& a, const U4& b) {
#ifndef KVX_K3_PLAIN_HINTS  // streaming (evict-first) stores of the fp16 cache rows
  // (A/B, profiles/r02_bench/k3_hints_n1.log: config 2 K3 1.750 -> 1.743 ms,
  // config-4 pair shape 0.580 -> 0.570 ms; -DKVX_K3_PLAIN_HINTS restores the plain form)
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
               "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
#else
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
               "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
#endif
}

template <int BITS>
__device__ __forceinline__ void k3_process(const K3Item& it, const K3Data<BITS>& d) {
  if (!it.active) return;
  const __half2 s2 = __half2half2(d.s), z2 = __half2half2(d.z);
  U4 o[4];
  if constexpr (BITS == 4) {
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = dequant8<4>(d.c.w[i], s2, z2);
  } else if constexpr (BITS == 8) {
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = dequant8<8>(make_uint2(d.c.w[2 * i], d.c.w[2 * i + 1]), s2, z2);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      o[i] = dequant8<2>(uint16_t(d.c.w[i >> 1] >> (16 * (i & 1))), s2, z2);
  }
  st256(it.dst, o[0], o[1]);
  st256(it.dst + 32, o[2], o[3]);
}

#ifndef KVX_K3_PF
#define KVX_K3_PF 2  // items prefetched ahead per warp (A/B: profiles/r01_summary.md)
#endif
// PACKED: the short-row item geometry (ItemGeo::rpi_shift > 0), a separate
// instantiation so the common one keeps its register budget (48 vs 58).
template <int BITS, int G, bool PACKED = false>
#ifndef KVX_K3_MIN_BLOCKS
#define KVX_K3_MIN_BLOCKS 1
#endif
__global__ void __launch_bounds__(256, KVX_K3_MIN_BLOCKS) dequant_scatter_kernel(Geo g, ItemGeo ig,
                                                              const uint8_t* __restrict__ codes,
                                                              const __half* __restrict__ scale,
                                                              const __half* __restrict__ zero) {
  constexpr int NB = KVX_K3_PF + 1;
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t n_warps = (gridDim.x * blockDim.x) >> 5;
  K3Item it[NB];
  K3Data<BITS> d[NB];
#pragma unroll
  for (int i = 0; i < NB - 1; ++i) {
    const uint32_t itm = warp + i * n_warps;
    if (itm < ig.n_items) {
      it[i] = k3_item<BITS, G, PACKED>(g, ig, itm, lane, codes, scale, zero);
      k3_load<BITS>(it[i], d[i]);
    }
  }
  for (uint32_t base = warp; base < ig.n_items; base += NB * n_warps) {
#pragma unroll
    for (int st = 0; st < NB; ++st) {
      const uint32_t cur = base + st * n_warps;
      if (cur >= ig.n_items) return;  // warp-uniform
      const uint32_t pre = cur + (NB - 1) * n_warps;
      const int pb = (st + NB - 1) % NB;
      if (pre < ig.n_items) {
        it[pb] = k3_item<BITS, G, PACKED>(g, ig, pre, lane, codes, scale, zero);
        k3_load<BITS>(it[pb], d[pb]);
      }
      k3_process<BITS>(it[st], d[st]);
    }
  }
}

// 16-bit passthrough on the decode side: scatter the raw fp16 rows.
template <int UNROLL>
__global__ void __launch_bounds__(256) scatter16_kernel(Geo g, const uint8_t* __restrict__ in) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t tr = warp; tr < g.n_token_rows; tr += n_warps) {
    int kv;
    int64_t t, layer, lrow;
    split_tr(g, tr, kv, t, layer, lrow);
    const int64_t pos = pos_of(g, t);
    if (pos < 0) continue;
    char* plane = const_cast<char*>(plane_ptr(g, kv, layer));
    U4* dst = reinterpret_cast<U4*>(const_cast<char*>(row_ptr(g, plane, pos)));
    const U4* src = reinterpret_cast<const U4*>(in + layer * g.codes_ls) + lrow * g.vecs;
    for (int base = 0; base < g.vecs; base += 32 * UNROLL) {
      U4 v[UNROLL];
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) {
        const int vi = base + k * 32 + lane;
        if (vi < g.vecs) v[k] = ld_stream(src + vi);
      }
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) {
        const int vi = base + k * 32 + lane;
        if (vi < g.vecs) st_stream(dst + vi, v[k]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K3-bulk: TMA-staged pull + dequantise + paged scatter.
//
// For a payload that sits in another GPU's HBM (fused NVLink pull) the load
// side is what limits: per-lane LDGs become many small NVLink reads.  Here one
// producer thread per CTA streams "spans" (R consecutive token rows of one
// layer: codes, scales and zeros are each ONE contiguous range) into a
// STAGES-deep shared-memory ring with cp.async.bulk (the bulk-copy/TMA
// engine; large requests over NVLink), completion tracked by mbarrier
// transaction counts.  Eight consumer warps dequantise out of shared memory
// (16-byte conflict-free LDS per lane) and write 64 B per lane into the paged
// cache; each warp releases the stage through an "empty" mbarrier.
// ---------------------------------------------------------------------------
struct BulkGeo {
  // per-chunk doorbells (nullable): the producer waits ready[c] >= ready_value
  // (this hand-off's sequence number) before the chunk's bulk reads
  const uint32_t* ready;
  uint32_t ready_value;
  // in-kernel completion (nullable): a u32 counting CTA exits (low 16 bits)
  // and aborted CTAs (high bits), zero between launches.  The last CTA out
  // sets *peer_free = ready_value on the prefill GPU (queue slot consumed) --
  // no stream-memop node after the kernel -- unless a CTA aborted
  uint32_t* done_counter;
  uint32_t* peer_free;
  Ctl* ctl;              // nullable
#ifdef KVX_TRACE
  uint32_t trace_id;     // trace builds: the hand-off's epoch
#endif
  int layers_per_chunk;
  int chained;           // KVX_PULL_CHAINED: only the completion waits for the previous grid
  int rows_per_span;     // R
  int spans_per_layer;   // ceil(2T / R)
  uint32_t n_spans;      // n_layers * spans_per_layer
  int code_row_bytes;    // row_elems * bits / 8  (multiple of 16)
  int meta_row_bytes;    // row_elems / G * 2     (multiple of 16)
  int stage_bytes;       // R * (code_row_bytes + 2 * meta_row_bytes)
  int cpr;               // 32-element chunks per token row
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Block (producer thread only) until the prefill side has published chunk c
// (doorbell >= this hand-off's sequence number).  The doorbell lives in this
// GPU's memory and is written over NVLink by the prefill GPU (K1's last
// arriving warp, or a stream memop); the acquire + proxy fence order the
// following bulk reads of the peer payload.  False = aborted / timed out.
__device__ __forceinline__ bool wait_ready(const uint32_t* flag, uint32_t value, Ctl* ctl) {
  if (!spin_until_geq(flag, value, ctl)) return false;
  // the bulk copies that follow read through the async proxy
  asm volatile("fence.proxy.async.global;" ::: "memory");
  return true;
}

// Producer side of a span whose chunk was never published (abort): complete
// the stage's phase without data so the consumers move on.
__device__ __forceinline__ void mbar_arrive_empty_phase(uint64_t* bar) { mbar_arrive(bar); }

__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Consumer side of one staged span (R token rows of one layer: codes, then
// the scales, then the zeros, each a contiguous block of the stage buffer):
// dequantise and scatter the rows into the paged cache.  Short rows (fewer
// than 32 chunks, e.g. a TP shard's few KV heads): a warp covers 32 / cpr
// rows per pass so every lane has a chunk.
template <int BITS, int G, int CONSUMERS>
__device__ __forceinline__ void bulk_consume_span(const Geo& g, int code_row_bytes,
                                                  int meta_row_bytes, int rows_per_span, int cpr,
                                                  const uint8_t* buf, int rows, int64_t r0,
                                                  uint32_t layer, int warp, int lane) {
  constexpr int CB = 32 * BITS / 8;
  constexpr int LPG = G / 32;
  const __half* sbuf = reinterpret_cast<const __half*>(buf + rows_per_span * code_row_bytes);
  const __half* zbuf = sbuf + rows_per_span * meta_row_bytes / 2;
  const int rpw = (cpr < 32 && (32 % cpr) == 0) ? 32 / cpr : 1;
  const int sub = rpw > 1 ? lane / cpr : 0;
  const int cl = rpw > 1 ? lane % cpr : lane;
  const int gpr = meta_row_bytes / 2;
  for (int rb = warp * rpw; rb < rows; rb += CONSUMERS * rpw) {
    const int r = rb + sub;
    if (r >= rows) continue;
    const int64_t lrow = r0 + r;
    const int p = lrow >= g.n_tokens;
    const int kv = g.plane0 + p;
    const int64_t t = lrow - p * g.n_tokens;
    const int64_t pos = pos_of(g, t);
    if (pos < 0) continue;  // padding token
    char* dst = const_cast<char*>(row_ptr(g, plane_ptr(g, kv, layer), pos));
    const uint8_t* crow = buf + r * code_row_bytes;
    for (int c = cl; c < cpr; c += 32) {
      K3Data<BITS> d;
      if constexpr (BITS == 2) {
        const uint2 v = *reinterpret_cast<const uint2*>(crow + c * CB);
        d.c.w[0] = v.x;
        d.c.w[1] = v.y;
      } else {
#pragma unroll
        for (int i = 0; i < Chunk32<BITS>::WORDS / 4; ++i) {
          const uint4 v = reinterpret_cast<const uint4*>(crow + c * CB)[i];
          d.c.w[4 * i] = v.x;
          d.c.w[4 * i + 1] = v.y;
          d.c.w[4 * i + 2] = v.z;
          d.c.w[4 * i + 3] = v.w;
        }
      }
      d.s = sbuf[r * gpr + c / LPG];
      d.z = zbuf[r * gpr + c / LPG];
      K3Item it;
      it.active = true;
      it.dst = dst + int64_t(c) * 64;
      k3_process<BITS>(it, d);
    }
  }
}

template <int BITS, int G, int STAGES>
__global__ void __launch_bounds__(288, 1) pull_dequant_scatter_kernel(
    Geo g, BulkGeo bg, const uint8_t* __restrict__ codes, const __half* __restrict__ scale,
    const __half* __restrict__ zero) {
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
  const int64_t two_t = int64_t(g.planes) * g.n_tokens;  // payload rows per layer
#ifdef KVX_TRACE
  const uint32_t trace_id = bg.trace_id;
  if (bg.done_counter && blockIdx.x == 0 && threadIdx.x == 0) KVX_TRACE_STAMP(1, trace_id, 0);
#endif
  if (warp == CONSUMERS) {  // ---- producer: one elected thread
    // The producer touches only this hand-off's queue slot (peer payload) and
    // its doorbells -- nothing an earlier kernel of this stream writes -- so
    // it runs ahead of pdl_wait: the first STAGES spans are in flight before
    // the previous hand-off's pull has finished.
    if (lane == 0) {
      uint32_t k = 0;
      int ready_chunk = -1;  // highest chunk known to be published
      bool ok = true;
      for (uint32_t sp = blockIdx.x; sp < bg.n_spans; sp += gridDim.x, ++k) {
        const int st = k % STAGES;
        if (k >= STAGES) mbar_wait(&empty[st], ((k / STAGES) & 1) ^ 1);
        const uint32_t layer = sp / bg.spans_per_layer;
        if (bg.ready && ok) {
          const int c = int(layer) / bg.layers_per_chunk;
          if (c > ready_chunk) {
            ok = wait_ready(bg.ready + c, bg.ready_value, bg.ctl);
            if (!ok) *reinterpret_cast<volatile uint32_t*>(&s_abort) = 1u;
            ready_chunk = c;
#ifdef KVX_TRACE
            if (bg.done_counter && blockIdx.x == 0 && c == 0) KVX_TRACE_STAMP(1, trace_id, 1);
#endif
          }
        }
        if (!ok) {  // aborted: release the consumers span by span, no data
          mbar_arrive_empty_phase(&full[st]);
          continue;
        }
        const int64_t r0 = int64_t(sp - layer * bg.spans_per_layer) * bg.rows_per_span;
        const int rows = int(min(int64_t(bg.rows_per_span), two_t - r0));
        uint8_t* buf = smem + st * bg.stage_bytes;
        const uint32_t cb = rows * bg.code_row_bytes, mb = rows * bg.meta_row_bytes;
        mbar_expect_tx(&full[st], cb + 2 * mb);
        bulk_g2s(buf, codes + layer * g.codes_ls + r0 * bg.code_row_bytes, cb, &full[st]);
        const char* sbase = reinterpret_cast<const char*>(scale) + layer * g.meta_ls;
        const char* zbase = reinterpret_cast<const char*>(zero) + layer * g.meta_ls;
        uint8_t* mbuf = buf + bg.rows_per_span * bg.code_row_bytes;
        bulk_g2s(mbuf, sbase + r0 * bg.meta_row_bytes, mb, &full[st]);
        bulk_g2s(mbuf + bg.rows_per_span * bg.meta_row_bytes, zbase + r0 * bg.meta_row_bytes, mb,
                 &full[st]);
      }
      // PDL: every span of this CTA is requested -- the stream's next kernel
      // (the next hand-off's pull) may be scheduled now; its producer starts
      // streaming its own queue slot while this grid's last spans drain, and
      // its consumers wait (pdl_wait) until this grid has completed.  (At the
      // top of the kernel instead, every queued pull became resident at once
      // and hand-offs of 512+ tokens ran 4x slower: 270 vs 68 us at 512
      // tokens, cfg4 pair 2,637 vs 2,852 GB/s; profiles/r02_pdl_ab.md.)
      pdl_launch_dependents();
    }
  } else {
  // ---- consumers: the slot mapping and the cache are stream-ordered inputs
#ifndef KVX_K3_NO_PDL_WAIT  // A/B only: measures what the stream-order wait costs
  // chained pulls (the caller's promise, kvx.h KVX_PULL_CHAINED): this
  // hand-off's blocks and slot mapping do not depend on the previous pull, so
  // the cache writes overlap its drain; the completion below still waits
  if (!bg.chained) pdl_wait();
#endif
  uint32_t k = 0;
  for (uint32_t sp = blockIdx.x; sp < bg.n_spans; sp += gridDim.x, ++k) {
    const int st = k % STAGES;
    const uint32_t layer = sp / bg.spans_per_layer;
    const int64_t r0 = int64_t(sp - layer * bg.spans_per_layer) * bg.rows_per_span;
    const int rows = int(min(int64_t(bg.rows_per_span), two_t - r0));
    const uint8_t* buf = smem + st * bg.stage_bytes;
    mbar_wait(&full[st], (k / STAGES) & 1);
    if (*reinterpret_cast<volatile uint32_t*>(&s_abort)) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      continue;
    }
    bulk_consume_span<BITS, G, CONSUMERS>(g, bg.code_row_bytes, bg.meta_row_bytes,
                                          bg.rows_per_span, bg.cpr, buf, rows, r0, layer, warp,
                                          lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  }  // consumers

  if (bg.done_counter) {
    // The free flag only has to say "every read of the peer slot is
    // complete": each bulk read completed (its mbarrier phase) before the
    // consumers used the bytes, and every CTA counts itself done after that.
    // The cache stores need no ordering against the flag (the prefill side
    // never reads them), so neither a per-CTA fence nor a system-scope release
    // is needed -- they cost ~1 us and ~3.5 us on the critical path of every
    // hand-off (tools/handoff_trace.py).  Thread 0 is a consumer: it has
    // passed pdl_wait, so the previous use of these counters has completed.
    __syncthreads();  // this CTA has consumed every span it owned
    if (threadIdx.x == 0) {
      // chained: the previous pull (same counters' previous user Q hand-offs
      // back, and the previous slot's free flag) completes before this CTA
      // counts itself -- completions stay in hand-off order
      if (bg.chained) pdl_wait();
      // one atomic per CTA: low 16 bits count exits, high bits aborted CTAs
      const uint32_t inc = s_abort ? 0x10001u : 1u;
      const uint32_t total = atomicAdd(bg.done_counter, inc) + inc;
      if ((total & 0xFFFFu) == gridDim.x) {  // last CTA of the launch
        bg.done_counter[0] = 0u;
        KVX_TRACE_STAMP(1, trace_id, 2);
        if ((total >> 16) == 0u)
          asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(bg.peer_free), "r"(bg.ready_value)
                       : "memory");
#ifdef KVX_TRACE
        KVX_TRACE_STAMP(1, trace_id, 3);
        atomicMax(&g_trace_n[1], trace_id + 1);
#endif
      }
    }
  } else if (bg.chained && threadIdx.x == 0) {
    pdl_wait();  // chained: never complete before the previous grid
  }
}

// ---------------------------------------------------------------------------
// K3-bulk over several queued hand-offs in ONE launch (the decode side's pull
// of everything queued after a decode round).  The parts are
// consecutive queue slots of one pair landing in one paged cache; their spans
// are concatenated (part by part, layer-major within a part) and CTA-strided
// exactly like the single pull, each part waiting on its own chunk doorbells.
// The last CTA out frees every part's slot.  Amortises the per-launch ramp,
// tail and host cost that dominate short hand-offs.
// ---------------------------------------------------------------------------
constexpr int kMaxPullMany = 8;  // = the queue depth bound

struct PullPart {
  const uint8_t* codes;   // the slot's payload: codes / scales / zeros of layer 0
  const __half* scale;
  const __half* zero;
  int64_t payload_ls;     // bytes between payload layers (per-layer segments)
  const int64_t* slots;   // token -> paged position
  int64_t n_tokens;
  const uint32_t* ready;  // this part's chunk doorbells (this GPU), ready[c] >= ready_value
  uint32_t ready_value;
  int layers_per_chunk;
  uint32_t* peer_free;    // the slot's free flag on the prefill GPU
  uint32_t span0;         // first span of the part in the launch's span space
  int spans_per_layer;
  int rows_per_span;      // <= PullMany::stage_rows
};

struct PullMany {
  PullPart part[kMaxPullMany];
  int count;
  uint32_t n_spans;
  uint32_t* done_counter;  // as BulkGeo::done_counter
  Ctl* ctl;
  int code_row_bytes, meta_row_bytes, stage_bytes, cpr;
  int stage_rows;          // rows a stage holds (scales start at stage_rows * code_row_bytes)
};

template <int BITS, int G, int STAGES>
__global__ void __launch_bounds__(288, 1) pull_many_kernel(Geo g, const __grid_constant__ PullMany pm) {
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
      uint32_t k = 0;
      int i = 0, ready_chunk = -1;
      bool ok = true;
      for (uint32_t sp = blockIdx.x; sp < pm.n_spans; sp += gridDim.x, ++k) {
        const int st = k % STAGES;
        if (k >= STAGES) mbar_wait(&empty[st], ((k / STAGES) & 1) ^ 1);
        while (i + 1 < pm.count && sp >= pm.part[i + 1].span0) {
          ++i;
          ready_chunk = -1;
        }
        const PullPart& P = pm.part[i];
        const uint32_t local = sp - P.span0;
        const uint32_t layer = local / P.spans_per_layer;
        if (ok) {
          const int c = int(layer) / P.layers_per_chunk;
          if (c > ready_chunk) {
            ok = wait_ready(P.ready + c, P.ready_value, pm.ctl);
            if (!ok) *reinterpret_cast<volatile uint32_t*>(&s_abort) = 1u;
            ready_chunk = c;
          }
        }
        if (!ok) {
          mbar_arrive_empty_phase(&full[st]);
          continue;
        }
        const int64_t two_t = 2 * P.n_tokens;
        const int64_t r0 = int64_t(local - layer * P.spans_per_layer) * P.rows_per_span;
        const int rows = int(min(int64_t(P.rows_per_span), two_t - r0));
        uint8_t* buf = smem + st * pm.stage_bytes;
        const uint32_t cb = rows * pm.code_row_bytes, mb = rows * pm.meta_row_bytes;
        mbar_expect_tx(&full[st], cb + 2 * mb);
        const char* seg = reinterpret_cast<const char*>(P.codes) + int64_t(layer) * P.payload_ls;
        bulk_g2s(buf, seg + r0 * pm.code_row_bytes, cb, &full[st]);
        const char* sbase = reinterpret_cast<const char*>(P.scale) + int64_t(layer) * P.payload_ls;
        const char* zbase = reinterpret_cast<const char*>(P.zero) + int64_t(layer) * P.payload_ls;
        uint8_t* mbuf = buf + pm.stage_rows * pm.code_row_bytes;
        bulk_g2s(mbuf, sbase + r0 * pm.meta_row_bytes, mb, &full[st]);
        bulk_g2s(mbuf + pm.stage_rows * pm.meta_row_bytes, zbase + r0 * pm.meta_row_bytes, mb,
                 &full[st]);
      }
      pdl_launch_dependents();  // as in pull_dequant_scatter_kernel
    }
  } else {
    pdl_wait();  // the slot mappings and the cache are stream-ordered inputs
    uint32_t k = 0;
    int i = 0;
    Geo gp = g;
    gp.slots = pm.part[0].slots;
    gp.n_tokens = pm.part[0].n_tokens;
    for (uint32_t sp = blockIdx.x; sp < pm.n_spans; sp += gridDim.x, ++k) {
      const int st = k % STAGES;
      while (i + 1 < pm.count && sp >= pm.part[i + 1].span0) {
        ++i;
        gp.slots = pm.part[i].slots;
        gp.n_tokens = pm.part[i].n_tokens;
      }
      const PullPart& P = pm.part[i];
      const uint32_t local = sp - P.span0;
      const uint32_t layer = local / P.spans_per_layer;
      const int64_t r0 = int64_t(local - layer * P.spans_per_layer) * P.rows_per_span;
      const int rows = int(min(int64_t(P.rows_per_span), 2 * P.n_tokens - r0));
      const uint8_t* buf = smem + st * pm.stage_bytes;
      mbar_wait(&full[st], (k / STAGES) & 1);
      if (*reinterpret_cast<volatile uint32_t*>(&s_abort)) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        continue;
      }
      bulk_consume_span<BITS, G, CONSUMERS>(gp, pm.code_row_bytes, pm.meta_row_bytes,
                                            pm.stage_rows, pm.cpr, buf, rows, r0, layer, warp,
                                            lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
  // completion: every part's slot is freed by the last CTA out (see the
  // single pull for why no fence is needed)
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t inc = s_abort ? 0x10001u : 1u;
    const uint32_t total = atomicAdd(pm.done_counter, inc) + inc;
    if ((total & 0xFFFFu) == gridDim.x) {
      pm.done_counter[0] = 0u;
      if ((total >> 16) == 0u)
        for (int j = 0; j < pm.count; ++j)
          asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(pm.part[j].peer_free),
                       "r"(pm.part[j].ready_value)
                       : "memory");
    }
  }
}

// ---------------------------------------------------------------------------
// K1-bulk: quantise + pack with the source rows staged by TMA.  One producer
// thread per CTA streams spans (R consecutive token rows of one (layer,
// K|V) plane; one cp.async.bulk per row, or one for the span when the rows
// are contiguous) into a STAGES-deep shared-memory ring; eight consumer
// warps quantise out of shared memory (each lane's 64-byte chunk read as
// four 16-byte loads in a bank-conflict-free rotated order) with the same
// arithmetic as K1 (k1_process).  The bytes in flight per SM are bounded by
// the ring, not by registers: K1's register prefetch holds ~64 KB per SM at
// 122 registers; the ring holds 2 CTAs x STAGES x ~16 KB.  Same doorbell
// contract as K1 (SignalGeo): per-chunk arrivals per CTA (spans are
// CTA-strided: owners of chunk c's spans = min(#spans, gridDim.x)).
// ---------------------------------------------------------------------------
struct K1BulkGeo {
  int rows_per_span;     // R
  int spans_per_plane;   // ceil(T / R)
  uint32_t n_spans;      // n_layers * planes * spans_per_plane
  int row_bytes;         // source bytes of one token row (n_heads * head_dim * 2)
  int stage_bytes;       // R * row_bytes
  int cpr;               // 32-element chunks per row
  int contiguous;        // 1: a span's rows are one contiguous source range
  uint32_t spans_per_chunk;  // spans of one doorbell chunk (signal path)
};

template <int BITS, int G, int STAGES>
__global__ void __launch_bounds__(288, 2) quant_pack_bulk_kernel(Geo g, K1BulkGeo kb,
                                                                 uint8_t* __restrict__ codes,
                                                                 __half* __restrict__ scale,
                                                                 __half* __restrict__ zero,
                                                                 SignalGeo sig) {
  constexpr int CONSUMERS = 8;
  constexpr int CB = 32 * BITS / 8;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  __shared__ uint32_t s_go;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_go = 1u;
  }
  pdl_wait();  // PDL launches: the stream's previous grid and its memory first
#ifdef KVX_TRACE
  if (sig.peer_flags && blockIdx.x == 0 && threadIdx.x == 0) KVX_TRACE_STAMP(0, sig.trace_id, 0);
#endif
  if (sig.peer_flags && threadIdx.x == 0 && sig.free_flag)
    s_go = spin_until_geq(sig.free_flag, sig.free_value, sig.ctl) ? 1u : 0u;
#ifdef KVX_TRACE
  if (sig.peer_flags && blockIdx.x == 0 && threadIdx.x == 0) KVX_TRACE_STAMP(0, sig.trace_id, 1);
#endif
  __syncthreads();
  if (!s_go) return;  // aborted / timed out before anything was stored
  const int64_t T = g.n_tokens;
  if (warp == CONSUMERS) {  // ---- producer
    if (lane == 0) {
      uint32_t k = 0;
      for (uint32_t sp = blockIdx.x; sp < kb.n_spans; sp += gridDim.x, ++k) {
        const int st = k % STAGES;
        if (k >= STAGES) mbar_wait(&empty[st], ((k / STAGES) & 1) ^ 1);
        const uint32_t lp = sp / kb.spans_per_plane;  // layer * planes + plane
        const uint32_t layer = lp / g.planes;
        const int kv = g.plane0 + int(lp - layer * g.planes);
        const int64_t t0 = int64_t(sp - lp * kb.spans_per_plane) * kb.rows_per_span;
        const int rows = int(min(int64_t(kb.rows_per_span), T - t0));
        uint8_t* buf = smem + st * kb.stage_bytes;
        mbar_expect_tx(&full[st], uint32_t(rows) * kb.row_bytes);
        const char* plane = plane_ptr(g, kv, layer);
        if (kb.contiguous) {
          bulk_g2s(buf, row_ptr(g, plane, t0), uint32_t(rows) * kb.row_bytes, &full[st]);
        } else {
          for (int r = 0; r < rows; ++r)
            bulk_g2s(buf + r * kb.row_bytes, row_ptr(g, plane, pos_of(g, t0 + r)), kb.row_bytes,
                     &full[st]);
        }
      }
    }
  } else {  // ---- consumers
    const int cpr = kb.cpr;
    const int rpw = (cpr < 32 && 32 % cpr == 0) ? 32 / cpr : 1;  // rows per warp pass
    const int sub = rpw > 1 ? lane / cpr : 0;
    const int cl = rpw > 1 ? lane % cpr : lane;
    const int blocks = rpw > 1 ? 1 : (cpr + 31) / 32;
    const int rot = (lane >> 1) & 3;  // rotated 16-byte order: conflict-free LDS.128
    // this warp's first (row group, 32-chunk block) inside a span, and the
    // per-step advance of CONSUMERS items, precomputed once
    const int rb0 = warp / blocks, blk0 = warp - rb0 * blocks;
    const int drb = CONSUMERS / blocks, dblk = CONSUMERS - drb * blocks;
    const uint32_t code_row = uint32_t(cpr) * CB;      // code bytes per payload row
    const uint32_t meta_row = uint32_t(cpr) * 32 / G;  // groups per payload row
    uint32_t k = 0;
    for (uint32_t sp = blockIdx.x; sp < kb.n_spans; sp += gridDim.x, ++k) {
      const int st = k % STAGES;
      const uint32_t lp = sp / kb.spans_per_plane;
      const uint32_t layer = lp / g.planes;
      const int p = int(lp - layer * g.planes);
      const int64_t t0 = int64_t(sp - lp * kb.spans_per_plane) * kb.rows_per_span;
      const int rows = int(min(int64_t(kb.rows_per_span), T - t0));
      const uint8_t* buf = smem + st * kb.stage_bytes;
      // payload row of the span's first token row
      const int64_t lrow0 = int64_t(p) * T + t0;
      char* ccodes = reinterpret_cast<char*>(codes) + int64_t(layer) * g.codes_ls +
                     lrow0 * code_row;
      __half* cscale = reinterpret_cast<__half*>(reinterpret_cast<char*>(scale) +
                                                 int64_t(layer) * g.meta_ls) + lrow0 * meta_row;
      __half* czero = reinterpret_cast<__half*>(reinterpret_cast<char*>(zero) +
                                                int64_t(layer) * g.meta_ls) + lrow0 * meta_row;
      mbar_wait(&full[st], (k / STAGES) & 1);
      for (int rb = rb0, blk = blk0; rb * rpw < rows;) {
        const int r = rb * rpw + sub;
        const int c = blk * 32 + cl;
        K1Item it;
        it.active = r < rows && c < cpr;
        const int rr = it.active ? r : 0, cc = it.active ? c : 0;
        const uint8_t* src = buf + rr * kb.row_bytes + cc * 64;
        uint32_t w[16];  // piece j holds source piece (j + rot) & 3
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 v = *reinterpret_cast<const uint4*>(src + ((j + rot) & 3) * 16);
          w[4 * j] = v.x;
          w[4 * j + 1] = v.y;
          w[4 * j + 2] = v.z;
          w[4 * j + 3] = v.w;
        }
        it.src = nullptr;
        it.codes = ccodes + uint32_t(rr) * code_row + uint32_t(cc) * CB;
        const uint32_t gi = uint32_t(rr) * meta_row + uint32_t(cc) * 32 / G;
        it.scale = cscale + gi;
        it.zero = czero + gi;
        k1_process<BITS, G, true>(it, w, lane, rot);
        rb += drb;
        blk += dblk;
        if (blk >= blocks) {
          blk -= blocks;
          ++rb;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (sig.peer_flags) {  // this CTA's share of a doorbell chunk is done
        const uint32_t c = sp / kb.spans_per_chunk;
        const uint32_t nxt = sp + gridDim.x;
        if (nxt >= kb.n_spans || nxt / kb.spans_per_chunk != c) {
          __threadfence();  // this thread's payload stores, device-wide
          asm volatile("bar.sync 1, %0;" ::"r"(CONSUMERS * 32) : "memory");
          if (threadIdx.x == 0) {
            const uint32_t a = c * kb.spans_per_chunk;
            const uint32_t b = min(kb.n_spans, a + kb.spans_per_chunk);
            const uint32_t owners = min(b - a, gridDim.x);
            __threadfence();
            if (atomicAdd(sig.counters + c, 1u) + 1 == owners) {
              sig.counters[c] = 0u;
              asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(sig.peer_flags + c),
                           "r"(sig.ready_value)
                           : "memory");
#ifdef KVX_TRACE
              if (nxt >= kb.n_spans || b >= kb.n_spans) KVX_TRACE_STAMP(0, sig.trace_id, 2);
#endif
            }
          }
        }
      }
    }
    // every consumer of this CTA is done with its spans: the stream's next
    // kernel may be scheduled (PDL; it waits for this grid before reading)
    pdl_launch_dependents();
#ifdef KVX_TRACE
    if (sig.peer_flags) {  // trace builds: stamp the last CTA's exit
      asm volatile("bar.sync 1, %0;" ::"r"(CONSUMERS * 32) : "memory");
      if (threadIdx.x == 0 && atomicAdd(sig.counters + kMaxSignalChunks, 1u) == gridDim.x - 1) {
        sig.counters[kMaxSignalChunks] = 0u;
        KVX_TRACE_STAMP(0, sig.trace_id, 3);
        atomicMax(&g_trace_n[0], sig.trace_id + 1);
      }
    }
#endif
  }
}

}  // namespace kvx
