/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the timed CPU baseline — never as part of the product path.
 *
 * A plain-C restatement of the reference's conv nest (ConvPreset::build,
 * /root/reference/proj/include/nestrank/presets.hpp:60-127; paper Fig. 5,
 * PAPER.md:504-536), executed in the reference's program order
 * (for_each_iteration, include/nestrank/oracle.hpp:22-43).
 *
 * Pinning: the reference computes nothing numerically (the microkernel is
 * external LIBXSMM). The restatement is pinned
 * bit-exactly against an interpreter built from the reference's OWN headers
 * (oracle/ref_interp.cpp -> oracle/_ref/libref_interp.so): ConvPreset::build()
 * walked by oracle_detail::for_each_iteration with the ArrayRef subscripts
 * evaluated per iteration. Golden outputs of that interpreter are committed
 * under tests/golden/ (generator: tests/golden/make_golden.py).
 */
#ifndef PSCONV_ORACLE_H
#define PSCONV_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same field order as conv_desc in include/psconv.h; ifh/ifw resolved. */
typedef struct oc_desc {
  int64_t nImg, nOfm, nIfm, ofh, ofw, kh, kw, stride_h, stride_w, gemm_block;
  int64_t pad_h, pad_w, ifh, ifw;
} oc_desc;

/* Seeded generator (same function as the device generator, psconv.h). */
float oracle_value(uint64_t seed, uint64_t logical_index);
void oracle_fill_input(const oc_desc* d, uint64_t seed, int64_t c_logical, float* in_nchw16c,
                       int64_t img_begin, int64_t img_count);
void oracle_fill_filter(const oc_desc* d, uint64_t seed, int64_t c_logical, float* flt);

/* Copies NCHW16c input into the reference-implied pre-padded extent
 * Hp = (ofh-1)*stride_h + kh, Wp = (ofw-1)*stride_w + kw (presets.hpp:88-91),
 * zero border of pad_h/pad_w. Images [0, img_count). */
void oracle_pad_input(const oc_desc* d, const float* in, float* in_padded, int64_t img_count);

/* Fig. 5 in the identity order img, ofm_tile, ifm_tile, oj, kj, ki with the
 * band (oi, ofm, ifm) innermost: output += conv over images
 * [img_begin, img_begin+img_count) of the pre-padded input (arrays indexed
 * from image 0). fp32, no FMA contraction: per output element the sum runs
 * over (ifm_tile, kj, ki, ifm) in program order, exactly as the reference IR
 * executes. OpenMP over img (presets.hpp:125 annotation). */
void oracle_conv_fig5(const oc_desc* d, const float* in_padded, const float* flt, float* out,
                      int64_t img_begin, int64_t img_count);

/* The band as a 3-pointer microkernel (presets.hpp:116-123). */
void oracle_gemm_microkernel(const oc_desc* d, float* out, const float* flt, const float* in);

/* float64 direct convolution of the unpadded input (error attribution). */
void oracle_conv_f64(const oc_desc* d, const float* in, const float* flt, double* out,
                     int64_t img_begin, int64_t img_count);

int oracle_threads(void);

#ifdef __cplusplus
}
#endif
#endif
