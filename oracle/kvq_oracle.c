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
 *            (product exact, one rounding: the GPU's fused FFMA(t, inv, 2^23))
 *   x_hat  = f16_rn(min(q * s + z, 65504))  (exact in double, one rounding)
 *
 * Build (oracle/Makefile): gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

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

/* src: fp16 bits [rows, head_dim] (row stride = head_dim). */
int kvq_quant_pack(const uint16_t* src, int64_t rows, int head_dim, int group, int bits,
                   uint8_t* codes, uint16_t* scale, uint16_t* zero) {
  int rc = check(head_dim, group, bits);
  if (rc) return rc;
  const int ng = head_dim / group;
  const int qmax = (1 << bits) - 1;
  const int per = 8 / bits;
  const int64_t cbytes = (int64_t)head_dim * bits / 8;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    const uint16_t* x = src + r * head_dim;
    uint8_t* out = codes + r * cbytes;
    memset(out, 0, (size_t)cbytes);
    for (int g = 0; g < ng; ++g) {
      float mn = INFINITY, mx = -INFINITY;
      for (int i = 0; i < group; ++i) {
        float v = h2f(x[g * group + i]);
        mn = v < mn ? v : mn;
        mx = v > mx ? v : mx;
      }
      uint16_t z16 = f2h(mn + 0.0f);
      volatile float d = mx - mn; /* keep IEEE ops discrete */
      float sq = d / (float)qmax;
      uint16_t s16 = f2h(sq + 0.0f);
      float s = h2f(s16), z = h2f(z16);
      scale[r * ng + g] = s16;
      zero[r * ng + g] = z16;
      float inv = s != 0.0f ? 1.0f / s : 0.0f;
      for (int i = 0; i < group; ++i) {
        int e = g * group + i;
        int q = 0;
        if (s != 0.0f) {
          volatile float t = h2f(x[e]) - z;          /* RN32(x - z) */
          double u = (double)t * (double)inv;         /* exact product */
          double rq = nearbyint(u);                   /* one rounding, half-to-even */
          rq = rq < 0.0 ? 0.0 : (rq > (double)qmax ? (double)qmax : rq);
          q = (int)rq;
        }
        out[e / per] |= (uint8_t)(q << ((e % per) * bits));
      }
    }
  }
  return 0;
}

static inline void dequant_row(const uint8_t* c, const uint16_t* scale, const uint16_t* zero,
                               int head_dim, int group, int bits, uint16_t* out) {
  const int per = 8 / bits;
  const int mask = (1 << bits) - 1;
  for (int e = 0; e < head_dim; ++e) {
    int g = e / group;
    float s = h2f(scale[g]), z = h2f(zero[g]);
    int q = (c[e / per] >> ((e % per) * bits)) & mask;
    double y = (double)q * (double)s + (double)z; /* exact: multiples of 2^-24 < 2^25 */
    y = y < 65504.0 ? y : 65504.0;
    f16 hv = (f16)y; /* single correct rounding double -> half */
    memcpy(&out[e], &hv, 2);
  }
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
