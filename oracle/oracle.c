/* CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h). */
#include "oracle.h"

#include <omp.h>
#include <string.h>

static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static float value_k(uint64_t key, uint64_t i) {
  const uint64_t z = splitmix64(key ^ i);
  return (float)(int32_t)(z >> 40) * (1.0f / 8388608.0f) - 1.0f;
}

float oracle_value(uint64_t seed, uint64_t i) { return value_k(splitmix64(seed), i); }

int oracle_threads(void) { return omp_get_max_threads(); }

void oracle_fill_input(const oc_desc* d, uint64_t seed, int64_t c_logical, float* in,
                       int64_t img_begin, int64_t img_count) {
  const int64_t Cb = d->nIfm / 16, H = d->ifh, W = d->ifw;
  const uint64_t key = splitmix64(seed);
  if (c_logical <= 0 || c_logical > d->nIfm) c_logical = d->nIfm;
#pragma omp parallel for schedule(static)
  for (int64_t n = img_begin; n < img_begin + img_count; ++n)
    for (int64_t cb = 0; cb < Cb; ++cb)
      for (int64_t h = 0; h < H; ++h)
        for (int64_t w = 0; w < W; ++w)
          for (int64_t c16 = 0; c16 < 16; ++c16) {
            const int64_t c = cb * 16 + c16;
            float v = 0.f;
            if (c < c_logical) v = value_k(key, (uint64_t)(((n * c_logical + c) * H + h) * W + w));
            in[((((n * Cb + cb) * H + h) * W + w) * 16) + c16] = v;
          }
}

void oracle_fill_filter(const oc_desc* d, uint64_t seed, int64_t c_logical, float* flt) {
  const int64_t Cb = d->nIfm / 16, Kb = d->nOfm / 16, R = d->kh, S = d->kw;
  const uint64_t key = splitmix64(seed);
  if (c_logical <= 0 || c_logical > d->nIfm) c_logical = d->nIfm;
#pragma omp parallel for schedule(static)
  for (int64_t kb = 0; kb < Kb; ++kb)
    for (int64_t cb = 0; cb < Cb; ++cb)
      for (int64_t r = 0; r < R; ++r)
        for (int64_t s = 0; s < S; ++s)
          for (int64_t c16 = 0; c16 < 16; ++c16)
            for (int64_t k16 = 0; k16 < 16; ++k16) {
              const int64_t c = cb * 16 + c16, k = kb * 16 + k16;
              float v = 0.f;
              if (c < c_logical) v = value_k(key, (uint64_t)(((k * c_logical + c) * R + r) * S + s));
              flt[(((((kb * Cb + cb) * R + r) * S + s) * 16 + c16) * 16) + k16] = v;
            }
}

void oracle_pad_input(const oc_desc* d, const float* in, float* inp, int64_t img_count) {
  const int64_t Cb = d->nIfm / 16, H = d->ifh, W = d->ifw;
  const int64_t Hp = (d->ofh - 1) * d->stride_h + d->kh, Wp = (d->ofw - 1) * d->stride_w + d->kw;
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < img_count; ++n)
    for (int64_t cb = 0; cb < Cb; ++cb)
      for (int64_t hp = 0; hp < Hp; ++hp)
        for (int64_t wp = 0; wp < Wp; ++wp) {
          const int64_t h = hp - d->pad_h, w = wp - d->pad_w;
          float* dst = inp + (((n * Cb + cb) * Hp + hp) * Wp + wp) * 16;
          if (h >= 0 && h < H && w >= 0 && w < W)
            memcpy(dst, in + (((n * Cb + cb) * H + h) * W + w) * 16, 64);
          else
            memset(dst, 0, 64);
        }
}

/* One band call (presets.hpp:82-84,112-118). The (ofm, ifm) loops are
 * interchanged for vectorisation; per output element the accumulation still
 * runs over ifm = 0..15 in order, so results are those of the band order. */
static inline void band(float* restrict o, const float* restrict f, const float* restrict x,
                        int64_t ofw, int64_t sw) {
  /* Register-blocked over 4 output pixels (independent elements) for ILP;
   * each element's accumulation order over ifm is unchanged. */
  int64_t oi = 0;
  for (; oi + 4 <= ofw; oi += 4) {
    float acc[4][16];
    for (int j = 0; j < 4; ++j)
      for (int k = 0; k < 16; ++k) acc[j][k] = o[(oi + j) * 16 + k];
    for (int ifm = 0; ifm < 16; ++ifm) {
      const float* fr = f + ifm * 16;
      for (int j = 0; j < 4; ++j) {
        const float xv = x[(oi + j) * sw * 16 + ifm];
        for (int k = 0; k < 16; ++k) acc[j][k] = acc[j][k] + fr[k] * xv;
      }
    }
    for (int j = 0; j < 4; ++j)
      for (int k = 0; k < 16; ++k) o[(oi + j) * 16 + k] = acc[j][k];
  }
  for (; oi < ofw; ++oi) {
    float acc[16];
    for (int k = 0; k < 16; ++k) acc[k] = o[oi * 16 + k];
    for (int ifm = 0; ifm < 16; ++ifm) {
      const float xv = x[oi * sw * 16 + ifm];
      for (int k = 0; k < 16; ++k) acc[k] = acc[k] + f[ifm * 16 + k] * xv;
    }
    for (int k = 0; k < 16; ++k) o[oi * 16 + k] = acc[k];
  }
}

void oracle_gemm_microkernel(const oc_desc* d, float* out, const float* flt, const float* in) {
  band(out, flt, in, d->ofw, d->stride_w);
}

void oracle_conv_fig5(const oc_desc* d, const float* inp, const float* flt, float* out,
                      int64_t img_begin, int64_t img_count) {
  const int64_t Kb = d->nOfm / 16, Cb = d->nIfm / 16, P = d->ofh, Q = d->ofw, R = d->kh,
                S = d->kw, sh = d->stride_h, sw = d->stride_w;
  const int64_t Hp = (P - 1) * sh + R, Wp = (Q - 1) * sw + S;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t img = img_begin; img < img_begin + img_count; ++img)
    for (int64_t ofm_tile = 0; ofm_tile < Kb; ++ofm_tile)
      for (int64_t ifm_tile = 0; ifm_tile < Cb; ++ifm_tile)
        for (int64_t oj = 0; oj < P; ++oj)
          for (int64_t kj = 0; kj < R; ++kj)
            for (int64_t ki = 0; ki < S; ++ki)
              band(out + (((img * Kb + ofm_tile) * P + oj) * Q) * 16,                       /* &output[img][ofm_tile][oj][0][0] */
                   flt + ((((ofm_tile * Cb + ifm_tile) * R + kj) * S + ki) * 16) * 16,     /* &filter[ofm_tile][ifm_tile][kj][ki][0][0] */
                   inp + ((((img * Cb + ifm_tile) * Hp + (oj * sh + kj)) * Wp) + ki) * 16, /* &input[img][ifm_tile][oj*sh+kj][ki][0] */
                   Q, sw);
}

void oracle_conv_f64(const oc_desc* d, const float* in, const float* flt, double* out,
                     int64_t img_begin, int64_t img_count) {
  const int64_t Kb = d->nOfm / 16, Cb = d->nIfm / 16, P = d->ofh, Q = d->ofw, R = d->kh,
                S = d->kw, H = d->ifh, W = d->ifw;
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int64_t n = img_begin; n < img_begin + img_count; ++n)
    for (int64_t kb = 0; kb < Kb; ++kb)
      for (int64_t p = 0; p < P; ++p)
        for (int64_t q = 0; q < Q; ++q) {
          double acc[16] = {0};
          for (int64_t cb = 0; cb < Cb; ++cb)
            for (int64_t r = 0; r < R; ++r) {
              const int64_t h = p * d->stride_h + r - d->pad_h;
              if (h < 0 || h >= H) continue;
              for (int64_t s = 0; s < S; ++s) {
                const int64_t w = q * d->stride_w + s - d->pad_w;
                if (w < 0 || w >= W) continue;
                const float* x = in + (((n * Cb + cb) * H + h) * W + w) * 16;
                const float* f = flt + ((((kb * Cb + cb) * R + r) * S + s) * 16) * 16;
                for (int c = 0; c < 16; ++c)
                  for (int k = 0; k < 16; ++k) acc[k] += (double)x[c] * (double)f[c * 16 + k];
              }
            }
          double* o = out + (((n * Kb + kb) * P + p) * Q + q) * 16;
          for (int k = 0; k < 16; ++k) o[k] = acc[k];
        }
}
