/*
 * C restatement of the KV hand-off oracle (TEST INFRASTRUCTURE ONLY).
 *
 * Same bit-exact format as oracle/kvq_oracle.py; used by the
 * tests as a second, independent restatement and by bench.py as the CPU
 * baseline / `--impl reference` arm ("port": the reference ships no CPU
 * quantiser).  Never linked into the product.
 *
 *   group  = G contiguous elements of one (layer, K|V, token, head) row
 *   zero16 = f16(mn + 0.0f); scale16 = f16((mx - mn) / (2^bits-1) + 0.0f)
 *   q      = s == 0 ? 0 : min(rint_even(RN32(x - z) * RN32(1/s)), 2^bits-1)
 *            (product exact, one rounding: fmaf(t, inv, 1.5*2^23) - 1.5*2^23,
 *            the same fused step the GPU issues as FFMA)
 *   x_hat  = f16_rn(min(q * s + z, 65504))  (one rounding of the exact sum)
 *
 * Two builds of the same arithmetic:
 *  - the scalar statement (always compiled; used when the CPU lacks AVX2/F16C),
 *  - an AVX2 + F16C + FMA path (oracle/Makefile builds with -mavx2 -mf16c
 *    -mfma), so that the CPU baseline is an optimised port rather than a
 *    soft-float one.  F16C's vcvtps2ph/vcvtph2ps round to nearest even, the
 *    quantiser's rounding is one FMA against the 1.5*2^23 shifter, and the
 *    dequantiser's single rounding of q*s + z to fp16 is done as an exact
 *    TwoSum in fp32 -> round-to-odd fp32 -> RN fp16 (round-to-odd onto 24
 *    bits followed by RN onto 11 bits equals one RN of the exact value).
 *  tests/test_oracle.py checks this file against the numpy oracle bit for bit.
 *
 * Build (oracle/Makefile): gcc -O3 -mavx2 -mf16c -mfma -fopenmp
 *                          -ffp-contract=off -fno-fast-math
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#if defined(__AVX2__) && defined(__F16C__) && defined(__FMA__)
#include <immintrin.h>
#define KVQ_SIMD 1
#else
#define KVQ_SIMD 0
#endif

typedef _Float16 f16;

static inline float h2f(uint16_t h) {
  f16 v;
  memcpy(&v, &h, 2);
  return (float)v;
}
static inline uint16_t f2h(float f) {
  f16 v = (f16)f; /* IEEE round-to-nearest-even */
  uint16_t h;
  memcpy(&h, &v, 2);
  return h;
}

static int check(int head_dim, int group, int bits) {
  if (bits != 2 && bits != 4 && bits != 8) return 1;
  if (group != 32 && group != 64 && group != 128) return 2;
  if (head_dim <= 0 || head_dim % group) return 3;
  return 0;
}

void kvq_set_threads(int n) {
#ifdef _OPENMP
  extern void omp_set_num_threads(int);
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int kvq_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

int kvq_simd(void) { return KVQ_SIMD; }

/* scale16 / zero16 of one group from its fp32 min and max */
static inline void group_params(float mn, float mx, int qmax, uint16_t* s16, uint16_t* z16) {
  *z16 = f2h(mn + 0.0f);
  float d = mx - mn;
  *s16 = f2h(d / (float)qmax + 0.0f);
}

/* q of one element: one rounding of the exact product t*inv to an integer */
static inline int quant_one(float x, float z, float inv, int qmax) {
  const float shifter = 12582912.0f; /* 1.5 * 2^23 */
  float t = x - z;
  float r = fmaf(t, inv, shifter) - shifter;
  r = r < 0.0f ? 0.0f : (r > (float)qmax ? (float)qmax : r);
  return (int)r;
}

/* RN16(min(q*s + z, 65504)) with one rounding: TwoSum, round-to-odd, RN. */
static inline float sum_round_odd(float p, float z) {
  float r = p + z;
  float bp = r - z;
  float e = (p - bp) + (z - (r - bp));
  if (e != 0.0f) {
    uint32_t u;
    memcpy(&u, &r, 4);
    if (!(u & 1u)) {
      uint32_t ue;
      memcpy(&ue, &e, 4);
      uint32_t same = ((u ^ ue) >> 31) == 0;
      u = same ? u + 1 : u - 1;
      memcpy(&r, &u, 4);
    }
  }
  return r < 65504.0f ? r : 65504.0f;
}

static void quant_row_scalar(const uint16_t* x, int head_dim, int group, int bits, uint8_t* out,
                             uint16_t* scale, uint16_t* zero) {
  const int ng = head_dim / group, qmax = (1 << bits) - 1, per = 8 / bits;
  memset(out, 0, (size_t)head_dim * bits / 8);
  for (int g = 0; g < ng; ++g) {
    float mn = INFINITY, mx = -INFINITY;
    for (int i = 0; i < group; ++i) {
      float v = h2f(x[g * group + i]);
      mn = v < mn ? v : mn;
      mx = v > mx ? v : mx;
    }
    uint16_t s16, z16;
    group_params(mn, mx, qmax, &s16, &z16);
    float s = h2f(s16), z = h2f(z16);
    scale[g] = s16;
    zero[g] = z16;
    float inv = s != 0.0f ? 1.0f / s : 0.0f;
    for (int i = 0; i < group; ++i) {
      int e = g * group + i;
      int q = s != 0.0f ? quant_one(h2f(x[e]), z, inv, qmax) : 0;
      out[e / per] |= (uint8_t)(q << ((e % per) * bits));
    }
  }
}

static void dequant_row_scalar(const uint8_t* c, const uint16_t* scale, const uint16_t* zero,
                               int head_dim, int group, int bits, uint16_t* out) {
  const int per = 8 / bits, mask = (1 << bits) - 1;
  for (int e = 0; e < head_dim; ++e) {
    int g = e / group;
    float s = h2f(scale[g]), z = h2f(zero[g]);
    int q = (c[e / per] >> ((e % per) * bits)) & mask;
    out[e] = f2h(sum_round_odd((float)q * s, z)); /* q*s exact in fp32 */
  }
}

#if KVQ_SIMD
static inline __m256 load8h(const uint16_t* p) {
  return _mm256_cvtph_ps(_mm_loadu_si128((const __m128i*)p));
}

static void quant_row_simd(const uint16_t* x, int head_dim, int group, int bits, uint8_t* out,
                           uint16_t* scale, uint16_t* zero) {
  const int ng = head_dim / group, qmax = (1 << bits) - 1, nv = group / 8;
  const __m256 shifter = _mm256_set1_ps(12582912.0f), vq = _mm256_set1_ps((float)qmax);
  const __m256 zf = _mm256_setzero_ps();
  for (int g = 0; g < ng; ++g) {
    const uint16_t* xg = x + g * group;
    __m256 vmn = load8h(xg), vmx = vmn;
    for (int v = 1; v < nv; ++v) {
      __m256 a = load8h(xg + 8 * v);
      vmn = _mm256_min_ps(a, vmn);
      vmx = _mm256_max_ps(a, vmx);
    }
    float lo[8], hi[8];
    _mm256_storeu_ps(lo, vmn);
    _mm256_storeu_ps(hi, vmx);
    float mn = lo[0], mx = hi[0];
    for (int i = 1; i < 8; ++i) {
      mn = lo[i] < mn ? lo[i] : mn;
      mx = hi[i] > mx ? hi[i] : mx;
    }
    uint16_t s16, z16;
    group_params(mn, mx, qmax, &s16, &z16);
    scale[g] = s16;
    zero[g] = z16;
    float s = h2f(s16);
    const __m256 vz = _mm256_set1_ps(h2f(z16));
    const __m256 vinv = _mm256_set1_ps(s != 0.0f ? 1.0f / s : 0.0f);
    uint8_t* og = out + (size_t)g * group * bits / 8;
    for (int v = 0; v < nv; ++v) {
      __m256 r = _mm256_sub_ps(_mm256_fmadd_ps(_mm256_sub_ps(load8h(xg + 8 * v), vz), vinv, shifter),
                               shifter);
      r = _mm256_min_ps(_mm256_max_ps(r, zf), vq); /* s == 0: inv == 0 -> r == 0 */
      __m128i q32lo, q32hi;
      __m256i qi = _mm256_cvttps_epi32(r);
      q32lo = _mm256_castsi256_si128(qi);
      q32hi = _mm256_extracti128_si256(qi, 1);
      __m128i q16 = _mm_packus_epi32(q32lo, q32hi);  /* 8 x u16 */
      __m128i q8 = _mm_packus_epi16(q16, q16);       /* 8 x u8 in the low 64 bits */
      uint64_t b;
      _mm_storel_epi64((__m128i*)&b, q8);
      if (bits == 8) {
        memcpy(og + 8 * v, &b, 8);
      } else if (bits == 4) {
        /* byte j = q[2j] | q[2j+1] << 4 */
        uint64_t even = b & 0x00FF00FF00FF00FFull, odd = (b >> 8) & 0x00FF00FF00FF00FFull;
        uint64_t pr = even | (odd << 4); /* 16-bit lanes hold one byte each */
        uint32_t w = (uint32_t)(pr & 0xFF) | (uint32_t)((pr >> 16) & 0xFF) << 8 |
                     (uint32_t)((pr >> 32) & 0xFF) << 16 | (uint32_t)((pr >> 48) & 0xFF) << 24;
        memcpy(og + 4 * v, &w, 4);
      } else {
        uint16_t w = 0;
        for (int i = 0; i < 8; ++i) w |= (uint16_t)(((b >> (8 * i)) & 3u) << (2 * i));
        memcpy(og + 2 * v, &w, 2);
      }
    }
  }
}

/* 8 codes starting at element 8*v of a row, as int32 lanes */
static inline __m256i codes8(const uint8_t* c, int v, int bits) {
  if (bits == 8) return _mm256_cvtepu8_epi32(_mm_loadl_epi64((const __m128i*)(c + 8 * v)));
  if (bits == 4) {
    uint32_t w;
    memcpy(&w, c + 4 * v, 4);
    return _mm256_and_si256(_mm256_srlv_epi32(_mm256_set1_epi32((int)w),
                                              _mm256_setr_epi32(0, 4, 8, 12, 16, 20, 24, 28)),
                            _mm256_set1_epi32(15));
  }
  uint16_t w;
  memcpy(&w, c + 2 * v, 2);
  return _mm256_and_si256(_mm256_srlv_epi32(_mm256_set1_epi32(w),
                                            _mm256_setr_epi32(0, 2, 4, 6, 8, 10, 12, 14)),
                          _mm256_set1_epi32(3));
}

static void dequant_row_simd(const uint8_t* c, const uint16_t* scale, const uint16_t* zero,
                             int head_dim, int group, int bits, uint16_t* out) {
  const int nvg = group / 8;
  const __m256i one = _mm256_set1_epi32(1), signm = _mm256_set1_epi32((int)0x80000000u);
  const __m256 kmax = _mm256_set1_ps(65504.0f), fz = _mm256_setzero_ps();
  for (int v = 0; v < head_dim / 8; ++v) {
    int g = v / nvg;
    const __m256 s = _mm256_set1_ps(h2f(scale[g])), z = _mm256_set1_ps(h2f(zero[g]));
    __m256 p = _mm256_mul_ps(_mm256_cvtepi32_ps(codes8(c, v, bits)), s); /* exact */
    __m256 r = _mm256_add_ps(p, z);
    __m256 bp = _mm256_sub_ps(r, z);
    __m256 e = _mm256_add_ps(_mm256_sub_ps(p, bp), _mm256_sub_ps(z, _mm256_sub_ps(r, bp)));
    /* round to odd: an inexact r with an even last bit steps one ulp toward e */
    __m256i ri = _mm256_castps_si256(r);
    __m256i inexact = _mm256_castps_si256(_mm256_cmp_ps(e, fz, _CMP_NEQ_OQ));
    __m256i even = _mm256_cmpeq_epi32(_mm256_and_si256(ri, one), _mm256_setzero_si256());
    __m256i same = _mm256_cmpeq_epi32(
        _mm256_and_si256(_mm256_xor_si256(ri, _mm256_castps_si256(e)), signm),
        _mm256_setzero_si256());
    __m256i step = _mm256_or_si256(_mm256_and_si256(same, one),
                                   _mm256_andnot_si256(same, _mm256_set1_epi32(-1)));
    ri = _mm256_add_epi32(ri, _mm256_and_si256(_mm256_and_si256(inexact, even), step));
    r = _mm256_min_ps(_mm256_castsi256_ps(ri), kmax);
    _mm_storeu_si128((__m128i*)(out + 8 * v), _mm256_cvtps_ph(r, _MM_FROUND_TO_NEAREST_INT));
  }
}
#define quant_row quant_row_simd
#define dequant_row dequant_row_simd
#else
#define quant_row quant_row_scalar
#define dequant_row dequant_row_scalar
#endif

/* src: fp16 bits [rows, head_dim] (row stride = head_dim). */
int kvq_quant_pack(const uint16_t* src, int64_t rows, int head_dim, int group, int bits,
                   uint8_t* codes, uint16_t* scale, uint16_t* zero) {
  int rc = check(head_dim, group, bits);
  if (rc) return rc;
  const int ng = head_dim / group;
  const int64_t cbytes = (int64_t)head_dim * bits / 8;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r)
    quant_row(src + r * head_dim, head_dim, group, bits, codes + r * cbytes, scale + r * ng,
              zero + r * ng);
  return 0;
}

int kvq_dequant(const uint8_t* codes, const uint16_t* scale, const uint16_t* zero, int64_t rows,
                int head_dim, int group, int bits, uint16_t* out) {
  int rc = check(head_dim, group, bits);
  if (rc) return rc;
  const int ng = head_dim / group;
  const int64_t cbytes = (int64_t)head_dim * bits / 8;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r)
    dequant_row(codes + r * cbytes, scale + r * ng, zero + r * ng, head_dim, group, bits,
                out + r * head_dim);
  return 0;
}

/* The scalar statement, callable on its own (tests pin SIMD == scalar). */
int kvq_quant_pack_scalar(const uint16_t* src, int64_t rows, int head_dim, int group, int bits,
                          uint8_t* codes, uint16_t* scale, uint16_t* zero) {
  int rc = check(head_dim, group, bits);
  if (rc) return rc;
  const int ng = head_dim / group;
  const int64_t cbytes = (int64_t)head_dim * bits / 8;
  for (int64_t r = 0; r < rows; ++r)
    quant_row_scalar(src + r * head_dim, head_dim, group, bits, codes + r * cbytes,
                     scale + r * ng, zero + r * ng);
  return 0;
}

int kvq_dequant_scalar(const uint8_t* codes, const uint16_t* scale, const uint16_t* zero,
                       int64_t rows, int head_dim, int group, int bits, uint16_t* out) {
  int rc = check(head_dim, group, bits);
  if (rc) return rc;
  const int ng = head_dim / group;
  const int64_t cbytes = (int64_t)head_dim * bits / 8;
  for (int64_t r = 0; r < rows; ++r)
    dequant_row_scalar(codes + r * cbytes, scale + r * ng, zero + r * ng, head_dim, group, bits,
                       out + r * head_dim);
  return 0;
}

/* Dequantise rows [n_lk = L*2][T][H] and scatter into paged caches laid out
 * [L][num_blocks*block_size][H][D] (k and v planes, layer_stride elements
 * apart); slot < 0 is skipped.  bits == 16 is a passthrough copy. */
int kvq_dequant_scatter_paged(const uint8_t* codes, const uint16_t* scale, const uint16_t* zero,
                              const int64_t* slots, int64_t n_layers, int64_t tokens, int heads,
                              int head_dim, int group, int bits, uint16_t* k_cache,
                              uint16_t* v_cache, int64_t layer_stride) {
  if (bits != 16) {
    int rc = check(head_dim, group, bits);
    if (rc) return rc;
  }
  const int ng = bits == 16 ? 0 : head_dim / group;
  const int64_t cbytes = (int64_t)head_dim * bits / 8;
  const int64_t n_lk = n_layers * 2;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t lk = 0; lk < n_lk; ++lk) {
    for (int64_t t = 0; t < tokens; ++t) {
      int64_t slot = slots[t];
      if (slot < 0) continue;
      uint16_t* plane = ((lk & 1) ? v_cache : k_cache) + (lk >> 1) * layer_stride;
      for (int h = 0; h < heads; ++h) {
        int64_t row = (lk * tokens + t) * heads + h;
        uint16_t* dst = plane + (slot * heads + h) * head_dim;
        if (bits == 16) {
          memcpy(dst, codes + row * cbytes, (size_t)head_dim * 2);
        } else {
          dequant_row(codes + row * cbytes, scale + row * ng, zero + row * ng, head_dim, group,
                      bits, dst);
        }
      }
    }
  }
  return 0;
}
