/*
 * psconv.h — C ABI of the B200-native blocked direct-convolution forward path
 * (the computation PolyScientist, arXiv 2002.02145, tunes: Fig. 5 of the paper).
 *
 * This is the drop-in boundary. Every entry point is plain C: integers, plain
 * pointers and sizes, no C++ or torch types. Each one states the reference
 * interface (under /root/reference/proj) it replaces.
 *
 * Tensor layouts are the reference's ArrayRef subscripts
 * (include/nestrank/presets.hpp:93-97):
 *   input  NCHW16c    [nImg][nIfm/16][ifh][ifw][16]          (c innermost)
 *   filter KCRS16c16k [nOfm/16][nIfm/16][kh][kw][16c][16k]   (k innermost)
 *   output NKPQ16k    [nImg][nOfm/16][ofh][ofw][16]          (k innermost)
 * all fp32, dense, 16-byte aligned.
 *
 * Status codes follow the reference CLI's exit-code classes
 * (include/nestrank/cli.hpp:290-321, README.md:86-87): 0 ok, 2 input/config
 * error (ConfigRejectedError & co.), 1 runtime/analysis error. Nothing throws
 * across this boundary; conv_last_error() returns the thread's last message.
 */
#ifndef PSCONV_H
#define PSCONV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSCONV_OK 0
#define PSCONV_ERR_RUNTIME 1 /* reference exit status 1 (analysis / runtime) */
#define PSCONV_ERR_CONFIG 2  /* reference exit status 2 (input / config)     */

/* Arithmetic modes of the GPU path (BASELINE.json north_star). */
#define PSCONV_MODE_3XTF32 0 /* fp32-faithful: D += Alo*Bhi + Ahi*Blo + Ahi*Bhi */
#define PSCONV_MODE_TF32 1   /* fast mode: one TF32 product per MAC            */
#define PSCONV_MODE_F16X2 2  /* fp32-faithful: power-of-two scaled fp16 hi/lo split,
                                D += Alo*Bhi + Ahi*Blo + Ahi*Bhi as K=16 f16 MMAs */

/* conv_fwd flags */
#define PSCONV_FLAG_ACCUMULATE 1u /* out += conv (the reference body is `+=`,
                                     presets.hpp:112); default overwrites   */
#define PSCONV_FLAG_PREPACKED 2u  /* use the filter already prepacked into the
                                     plan by conv_plan_prepack (flt ignored) */
#define PSCONV_FLAG_RELU 4u       /* fused epilogue: out = max(conv (+ bias), 0);
                                     not with PSCONV_FLAG_ACCUMULATE            */

/*
 * Conv-layer descriptor. Replaces nestrank::ConvPreset (presets.hpp:13-23):
 * the first ten fields are the reference's, in the `conv:` CSV order
 * nImg,nOfm,nIfm,ofh,ofw,kh,kw,stride_h,stride_w,gemm_block (presets.hpp:25).
 * Extension fields (the reference has no padding, presets.hpp:88-91):
 *   pad_h, pad_w  zero padding; 0 reproduces the reference exactly.
 *   ifh, ifw      input extent; 0 means the reference-implied extent
 *                 (ofh-1)*stride_h + kh - 2*pad_h (and likewise for w).
 */
typedef struct conv_desc {
  int64_t nImg, nOfm, nIfm, ofh, ofw, kh, kw, stride_h, stride_w, gemm_block;
  int64_t pad_h, pad_w, ifh, ifw;
} conv_desc;

/* Parses "conv:<10 ints>" (reference form, presets.hpp:26-50; the "conv:"
 * prefix is optional, as in cli.hpp:54-66) or the extended forms with 12
 * (+pad_h,pad_w) or 14 (+ifh,ifw) integers. Validates. Returns 0 or 2. */
int conv_desc_parse(const char* text, conv_desc* out);

/* Same rules as ConvPreset::validate (presets.hpp:52-58) plus the extension
 * fields. Fills ifh/ifw when 0. Returns 0 or 2. gemm_block must be 16 for
 * the GPU path (checked by conv_plan_create, not here). */
int conv_desc_validate(conv_desc* d);

/* Formats the descriptor back to its `conv:` string (10 ints when the
 * extension fields are at their defaults, else 14). Returns 0, or 2 when
 * the buffer is too small. */
int conv_desc_format(const conv_desc* d, char* buf, size_t len);

/* ---------------------------------------------------------------------------
 * Nest-document front end. Reads the reference's textual
 * loop-nest format (parse_nest, loopnest.hpp:340-523; samples/conv2d.nest,
 * samples/matmul.nest) and recognises the computation:
 *   NEST_KIND_CONV  the blocked direct convolution of presets.hpp:60-127 with
 *                   any variable names and outer-loop order -> desc + recipe
 *                   ("perm=..." over the reference loop names, variants.hpp);
 *   NEST_KIND_GEMM  C[i][j] += A[i][k] * B[k][j] -> M, N, K, and desc = the
 *                   same product as a 1x1 convolution over M "images": row-major
 *                   A[M][K] IS NCHW16c and C[M][N] IS NKPQ16k at H = W = 1;
 *                   B[K][N] is blocked by gemm_pack_b (desc is validated and
 *                   runnable only when N, K % 16 == 0).
 * Returns 0, or 2 (parse error / unsupported computation; conv_last_error). */
#define NEST_KIND_CONV 1
#define NEST_KIND_GEMM 2
typedef struct nest_info {
  int32_t kind, reserved;
  conv_desc desc;
  int64_t M, N, K;
  char recipe[256];
} nest_info;
int nest_parse(const char* text, nest_info* out);

/* Row-major B[K][N] (device) -> the KCRS16c16k filter of the 1x1 convolution
 * that computes C = A * B (K input channels, N output channels). */
int gemm_pack_b(const float* b_rowmajor, float* b_blocked, int64_t K, int64_t N, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * CPU microkernel with the reference's call convention. Replaces the external
 * `gemm_microkernel(out, flt, in)` named by ConvPreset::build
 * (presets.hpp:116-123; MicrokernelSpec loopnest.hpp:139-148): a small GEMM
 * over the band (oi, ofm, ifm):
 *   out[oi*16+ofm] += flt[ifm*16+ofm] * in[oi*stride_w*16+ifm]
 * for oi < ofw. Like LIBXSMM, the shape (ofw, stride_w, block) is bound at
 * dispatch time; the returned function takes only the three pointers.
 */
typedef void (*gemm_microkernel_fn)(float* out, const float* flt, const float* in);

/* Returns 2 if the descriptor is invalid or gemm_block != 16, or
 * ofw*stride_w > 4096 (no specialisation). */
int gemm_microkernel_dispatch(const conv_desc* d, gemm_microkernel_fn* fn);

/* Batch-reduce form (north_star BRGEMM): folds `count` (ifm_tile,kj,ki)
 * blocks into one call on one output row:
 *   for i < count: gemm_microkernel(out, flt_blocks[i], in_rows[i]). */
int brgemm_f32(const conv_desc* d, float* out, const float* const* flt_blocks,
               const float* const* in_rows, int64_t count);

/* ---------------------------------------------------------------------------
 * GPU layer entry (sm_100a). A plan binds a descriptor, a mode and a schedule.
 * The schedule is chosen by the selector from the reference's recipe space
 * (variants.hpp:16-65: "perm=...;tile=oj:T") extended with an optional GPU
 * clause ";gpu=bn:B,box:QxPxN,cl:1|2,kg:K,ks:S,eg:1|2,os:4|8|12|16,..." (the full key list and
 * meanings: INTEGRATION.md "Recipe grammar"). recipe == NULL lets the selector choose.
 */
typedef struct conv_plan conv_plan;

int conv_plan_create(const conv_desc* d, int mode, int device, const char* recipe_or_null,
                     conv_plan** out);

/* Backward-data plan (neighbouring ops): for the FORWARD
 * descriptor d, a plan whose conv_fwd / conv_fwd_host computes dX = dL/dInput
 * from dY = dL/dOutput and the forward filter:
 *   in  = dY  [N][nOfm/16][ofh][ofw][16]   (NKPQ16k of the forward output)
 *   flt = W   KCRS16c16k of the forward layer (transposed and flipped inside)
 *   out = dX  [N][nIfm/16][ifh][ifw][16]   (NCHW16c of the forward input)
 * Stride 1: the transposed convolution conv(dY, W^T flipped, pad = k - 1 - pad) on
 * the same kernel. Stride s > 1: dX splits into stride_h x stride_w output phases
 * (h mod stride_h, w mod stride_w); each is a stride-1 transposed conv over dY with
 * the phase's forward taps (r = stride_h*u + rho) and asymmetric implied padding,
 * stored through a strided view of dX (phases without taps, e.g. 3 of 4 for a 1x1
 * stride-2 layer, are zero-filled). conv_plan_recipe lists the phases' schedules.
 * Returns 0 / 2 (a phase would need negative padding, e.g. 2x2 / stride 2 / pad 1) / 1. */
int conv_plan_create_bwd_data(const conv_desc* d, int mode, int device, const char* recipe_or_null,
                              conv_plan** out);
/* Backward-weight plan: for the FORWARD descriptor d (any
 * stride / padding), dW = dL/dFilter from the forward input X and dY:
 *   dW[k][c][r][s] = sum_{n,p,q} X[n][c][p*sh+r-pad_h][q*sw+s-pad_w] * dY[n][k][p][q]
 * computed by a pixel-major implicit GEMM (per tap, the reduction runs over the
 * pixels; both operands are read by TMA straight from NCHW16c / NKPQ16k as MN-major
 * tf32 tiles), split over pixel ranges with the partials added in split order
 * (bitwise reproducible). tf32 / 3xtf32 modes. recipe_or_null: NULL, or
 * "gpu=sw:S,kn:K,cn:C,nt:T,box:QxP,sp:SPLITS,st:STAGES,ch:K8" overriding the tile
 * roles (sw), channels / taps per tile, pixel box, splits, ring depth, 3xTF32
 * accumulation chunk. Returns 0 / 2 / 1. */
int conv_plan_create_bwd_weight(const conv_desc* d, int mode, int device, const char* recipe_or_null,
                                conv_plan** out);
/* The backward-weight geometry conv_plan_create_bwd_weight would choose on a GPU with
 * num_sms SMs (host only, no device): its recipe plus tiles / units / stage bytes. 0 / 2. */
int conv_wgrad_describe(const conv_desc* d, int mode, int num_sms, const char* recipe_or_null, char* buf,
                        size_t len);
/* Runs a backward-weight plan: x = X (NCHW16c), dy = dY (NKPQ16k), dw = dW
 * (KCRS16c16k, overwritten), all device arrays of the forward layer's sizes.
 * Stream-ordered, no allocation (the split workspace is the plan's). */
int conv_bwd_weight(const conv_plan* p, const float* x, const float* dy, float* dw, void* cuda_stream);
void conv_plan_destroy(conv_plan* p);

/* The plan's recipe id in the reference's grammar plus the gpu clause. */
const char* conv_plan_recipe(const conv_plan* p);

/* Runs the forward conv on images [img_begin, img_begin+img_count) of the
 * caller's device arrays (full-size, pointer to image 0), stream-ordered on
 * `cuda_stream` (a cudaStream_t; NULL = legacy default). Does not allocate
 * and does not synchronise. Each call first repacks `flt` into the plan's
 * K-major operand buffer (the tcgen05 tf32 B-operand layout; plus the
 * hi/lo split in 3xTF32 mode), so calls on ONE plan must be stream-ordered;
 * use one plan per concurrent stream. */
int conv_fwd(const conv_plan* p, const float* in, const float* flt, float* out, int64_t img_begin,
             int64_t img_count, void* cuda_stream, unsigned flags);

/* conv_fwd with a fused epilogue (the reference body is a
 * bare `+=`, presets.hpp:112): out = conv(in, flt) + bias[k] (bias: nOfm fp32
 * device values, or NULL), then ReLU when PSCONV_FLAG_RELU. With
 * PSCONV_FLAG_ACCUMULATE the bias is added into out as well (no ReLU).
 * conv_fwd(...) == conv_fwd_ex(..., bias = NULL, ...). */
int conv_fwd_ex(const conv_plan* p, const float* in, const float* flt, float* out, const float* bias,
                int64_t img_begin, int64_t img_count, void* cuda_stream, unsigned flags);

/* conv_fwd on HOST buffers (the reference's emitted driver computes on host
 * arrays, emit.hpp:60-134 / tests/golden/conv_identity.c): h_in / h_flt /
 * h_out are host pointers in the same layouts as conv_fwd (pinned memory gives
 * full copy/compute overlap). The image range is streamed through the device
 * in ~32 MB chunks, double buffered: the copy-in of chunk i+1, the kernel of
 * chunk i and the copy-out of chunk i-1 overlap on two plan-owned copy streams
 * and `cuda_stream`. Stream-ordered like conv_fwd: starts after prior work on
 * cuda_stream; h_out is complete when cuda_stream reaches this point. The plan
 * allocates its staging buffers on first use (released by conv_plan_destroy).
 * Returns 0 / 1 / 2. */
int conv_fwd_host(const conv_plan* p, const float* h_in, const float* h_flt, float* h_out,
                  int64_t img_begin, int64_t img_count, void* cuda_stream, unsigned flags);

/* Repacks a filter into the plan once (weights held constant, e.g. inference);
 * later conv_fwd calls with PSCONV_FLAG_PREPACKED skip the repack launch. */
int conv_plan_prepack(conv_plan* p, const float* flt, void* cuda_stream);

/* Number of kernel launches conv_fwd issues per call (for launch accounting). */
int conv_plan_launches(const conv_plan* p);

/* Emits the plan's driver loop nest as C text in the reference emitter's
 * format (emit.hpp:60-134; golden tests/golden/conv_identity.c). Returns the
 * number of bytes needed (excluding NUL); writes at most len-1 bytes. */
int64_t conv_plan_emit(const conv_plan* p, char* buf, size_t len);

/* Same emission without a plan or a GPU: any reference-legal recipe
 * (recipe NULL or "" = identity order). Returns bytes needed, or -2/-1. */
int64_t conv_emit_driver(const conv_desc* d, const char* recipe, char* buf, size_t len);

/* ---------------------------------------------------------------------------
 * Schedule selector (the paper's reuse-model ranking, re-expressed for B200).
 * Ranks candidate recipes for a descriptor by a closed-form SMEM/L2/HBM
 * traffic + tensor-pipe model. Writes up to k recipe ids separated by '\n'
 * into buf (best first) with their modelled microseconds into us_out (may be
 * NULL). Returns the number written, or -2 / -1 on config / runtime error.
 */
int conv_select_topk(const conv_desc* d, int mode, int k, char* buf, size_t len, double* us_out);
/* The same with the caller's assertion that only the first c_logical of the nIfm input channels
 * are non-zero (0 = all; the descriptor cannot carry it): with c_logical <= 4 and nIfm = 16 the
 * few-channel kernel's recipes (gpu=...,pp:C -- the ResNet stem) join the ranking. */
int conv_select_topk_ex(const conv_desc* d, int mode, int c_logical, int k, char* buf, size_t len,
                        double* us_out);

/* ---------------------------------------------------------------------------
 * Pairwise DNN ranker (PolyScientist-DNN; reference
 * dnnrank.hpp:87-438 PairwiseRanker, pipeline.hpp:98-173). Same net (8-64-32-
 * 16-8-2, relu/relu/softsign/relu/softmax, theta 0.6), joint pair
 * normalisation, seeded mini-batch training, "pairnet 1" weights text and
 * round-robin tournament ranking; the per-variant statistics are the B200
 * model's resource times (conv_model_stats: MMA, shared memory, operand-row
 * delivery, HBM; us) instead of cache working sets.
 */
/* stats[4] of one recipe. Returns 0 / 2. */
int conv_model_stats(const conv_desc* d, int mode, const char* recipe, double* stats);
/* Trains on dataset rows "a0 a1 a2 a3 b0 b1 b2 b3 A|B" (the reference pairs
 * format with real-valued statistics); holds out floor((1-split)*n) seeded-
 * shuffled rows; writes the weights text; acc[0] = train, acc[1] = holdout
 * accuracy (-1 if none). Returns 0 / 2. */
int ranker_train(const char* dataset, int epochs, double learning_rate, uint64_t seed, double split,
                 char* weights, size_t len, double* acc);
/* 0 = A faster, 1 = B faster, 2 = draw (neither softmax output > theta); prob
 * (may be NULL) receives both outputs. Negative status on error. */
int ranker_compare(const char* weights, const double* a, const double* b, double* prob);
/* conv_select_topk with the tournament instead of the cost model (ties by
 * modelled cost, then id); *symmetry = fraction of order-consistent games. */
int conv_select_topk_dnn(const conv_desc* d, int mode, int k, const char* weights, char* buf, size_t len,
                         double* symmetry);

/* Modelled time (microseconds) of one recipe, -1 on error. */
double conv_model_us(const conv_desc* d, int mode, const char* recipe);

/* Machine constants of the selector's model (the reference's machine file,
 * cachefit.hpp:43-106, re-expressed for B200): "<key> <value>" lines with keys
 * hbm_gbs, tf32_tflops, clock_ghz, sms, l2_bytes ('#' comments). The Python
 * layer feeds this pod's MEASURED_PEAKS.json at import. Not thread-safe with a
 * concurrent ranking. Returns 0 / 2. */
int conv_select_set_machine(const char* text);

/* ---------------------------------------------------------------------------
 * Device-side helpers (same stream semantics as conv_fwd).
 * Seeded generator: value(seed, i) = (int)(splitmix64(splitmix64(seed) ^ i) >> 40) * 2^-23 - 1,
 * i = logical NCHW (activations) or KCRS (weights) index; exactly
 * representable in fp32 and independent of layout and sharding.
 * c_logical < nIfm zero-fills the padded channels (ResNet-50 stem 3 -> 16). */
int conv_fill_input(const conv_desc* d, uint64_t seed, int64_t c_logical, float* in,
                    int64_t img_begin, int64_t img_count, void* cuda_stream);
int conv_fill_filter(const conv_desc* d, uint64_t seed, int64_t c_logical, float* flt,
                     void* cuda_stream);
/* Layout packing (a9): NCHW -> NCHW16c, KCRS -> KCRS16c16k, NKPQ16k -> NKPQ. */
int conv_pack_input(const conv_desc* d, const float* nchw, int64_t c_logical, float* nchw16c,
                    void* cuda_stream);
int conv_pack_filter(const conv_desc* d, const float* kcrs, int64_t c_logical, float* kcrs16c16k,
                     void* cuda_stream);
int conv_unpack_output(const conv_desc* d, const float* nkpq16k, float* nkpq, void* cuda_stream);

/* Thread-local message of the last failing call ("" if none). */
const char* conv_last_error(void);

/* Library / device introspection. */
const char* psconv_version(void);
int psconv_device_sm_count(int device);

#ifdef __cplusplus
}
#endif

#endif /* PSCONV_H */
