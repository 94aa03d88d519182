// Probe: does TMA multicast of a tile shared by the CTAs of a cluster raise the per-SM operand
// delivery of an L2-bound loop (B200, sm_100a)?  Every CTA streams, per iteration, a 32 KB "A"
// box of its own (64-B rows, like NCHW16c pixels) and a 16 KB "B" box that all CTAs of the
// cluster need (the filter block of their common N tile), through a ring of 4 stages with no
// consumer work (a stage is released as soon as it lands), all 148 SMs running:
//   unicast : every CTA loads the whole B box itself            (what conv_fwd_sm100 does)
//   mcast   : CTA r loads rows [r*R/CS, (r+1)*R/CS) of B and multicasts them to the cluster
// Reports bytes landed per cycle per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_02145_b200/csrc \
//        tools/probe_mcast.cu -o tools/probe_mcast -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100_ptx.cuh"
using namespace psconv;

constexpr int kStages = 4, kIters = 1024, kABytes = 32768, kBBytes = 16384, kStageBytes = kABytes + kBBytes;

template <int CS, bool MC, bool SAMEB = false>
__global__ void k_probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                        long long* out, int scatter) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kStages], empty[kStages];
  uint32_t rank = 0;
  if (CS > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], MC ? CS : 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (CS > 1) ptx::cluster_sync_all();
  if (threadIdx.x == 0) {
    const int cta = blockIdx.x;
    const int cl = SAMEB ? 0 : cta / CS;  // SAMEB: every cluster reads the same B box at the same time
    constexpr int kBRows = 256 / (MC ? CS : 1);  // B rows this CTA loads
    long long t0 = clock64();
    for (int it = 0; it < kIters + kStages - 1; ++it) {
      if (it < kIters) {
        const int s = it % kStages;
        if (it >= kStages) ptx::mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
        ptx::mbar_expect_tx(&full[s], kStageBytes);
        // A: 128 rows of 64 B, a different box per CTA and iteration (L2-resident 32 MB window)
        // scatter: 4 x 128 rows 100,352 B apart (box 1x1x128 of a 7x7 layer: one pixel of 128 images)
        if (scatter) ptx::tma_load_3d(sm + s * kStageBytes, &ma, &full[s], 0, (cta & 1) * 128, ((it * 37 + cta * 4) % 392) * 4);
        else ptx::tma_load_3d(sm + s * kStageBytes, &ma, &full[s], 0, (it & 7) * 256, (cta % 80) * 2);
        // B: 128 rows of 64 B shared by the cluster (and re-read from L2 by everyone)
        uint8_t* db = sm + s * kStageBytes + kABytes;
        if (!MC)
          ptx::tma_load_3d(db, &mb, &full[s], 0, 0, (it + cl) & 31);
        else
          ptx::tma_load_3d_mc(db + rank * kBRows * 64, &mb, &full[s], 0, rank * kBRows, (it + cl) & 31,
                              static_cast<uint16_t>((1u << CS) - 1));
      }
      const int c = it - (kStages - 1);
      if (c >= 0) {
        const int s = c % kStages;
        ptx::mbar_wait(&full[s], (c / kStages) & 1);
        if (!MC) {
          ptx::mbar_arrive(&empty[s]);
        } else {
          for (uint32_t r = 0; r < CS; ++r) ptx::mbar_arrive_remote(ptx::mapa(&empty[s], r));
        }
      }
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  __syncthreads();
  if (CS > 1) ptx::cluster_sync_all();
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int CS, bool MC, bool SAMEB = false>
void run(const CUtensorMap& ma, const CUtensorMap& mb, long long* out, int grid, const char* tag, int scatter = 0) {
  cudaFuncSetAttribute(k_probe<CS, MC, SAMEB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (CS > 4) cudaFuncSetAttribute(k_probe<CS, MC, SAMEB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid / CS * CS);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = CS > 1 ? 1 : 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_probe<CS, MC, SAMEB>, ma, mb, out, scatter);
    if (e != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess) {
      printf("%s: %s\n", tag, cudaGetErrorString(e));
      return;
    }
  }
  long long h = 0;
  cudaMemcpy(&h, out, sizeof(h), cudaMemcpyDeviceToHost);
  const double per_iter = double(h) / kIters;
  printf("grid %3d cluster %d %-8s: %7.1f cycles per 48 KB stage -> %5.1f B/cycle/SM landed (L2 reads %5.1f B/cycle/SM)\n",
         int(cfg.gridDim.x), CS, tag, per_iter, kStageBytes / per_iter,
         (double(kABytes) + double(kBBytes) / (MC ? CS : 1)) / per_iter);
}

int main() {
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fnp);
  float* buf;
  const size_t bytes = size_t(160) * 4096 * 64;  // A: [cta 160][rows 4096][16 fp32] = 40 MB
  cudaMalloc(&buf, bytes + (32 << 14));
  cudaMemset(buf, 0, bytes + (32 << 14));
  long long* out;
  cudaMalloc(&out, 64);
  CUtensorMap ma, mb;
  {
    cuuint64_t dims[3] = {16, 4096, 160};
    cuuint64_t str[2] = {64, 4096 * 64};
    cuuint32_t box[3] = {16, 256, 2};
    cuuint32_t es[3] = {1, 1, 1};
    enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  CUtensorMap ms;  // scattered A rows: [16][n 256 @ 100352 B][cb*px 1568 @ 64 B], box 16 x 128 x 4
  {
    cuuint64_t dims[3] = {16, 256, 1568};
    cuuint64_t str[2] = {100352, 64};
    cuuint32_t box[3] = {16, 128, 4};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&ms, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode ms failed %d\n", r);
  }
  auto encode_b = [&](int rows) {
    cuuint64_t dims[3] = {16, 256, 32};
    cuuint64_t str[2] = {64, 256 * 64};
    cuuint32_t box[3] = {16, cuuint32_t(rows), 1};
    cuuint32_t es[3] = {1, 1, 1};
    enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, reinterpret_cast<uint8_t*>(buf) + bytes, dims, str, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  for (int grid : {8, 148}) {
    encode_b(256);
    run<1, false>(ma, mb, out, grid, "unicast");
    run<1, false, true>(ma, mb, out, grid, "uni-sameB");
    run<1, false>(ms, mb, out, grid, "scatterA", 1);
    run<2, false>(ms, mb, out, grid, "scatterA", 1);
    run<2, false, true>(ma, mb, out, grid, "uni-sameB");
    run<2, false>(ma, mb, out, grid, "unicast");
    run<4, false>(ma, mb, out, grid, "unicast");
    encode_b(128);
    run<2, true>(ma, mb, out, grid, "mcast");
    encode_b(64);
    run<4, true>(ma, mb, out, grid, "mcast");
    encode_b(32);
    run<8, true>(ma, mb, out, grid, "mcast");
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
