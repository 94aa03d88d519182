// The reference-side binding in use (tests/test_adapter.py builds this against the reference
// headers + include/): a reference-EMITTED driver (emit_source text for PRESET_CSV, included
// as EMITTED_DRIVER) runs with the psconv CPU microkernel bound through
// nestrank::b200::microkernel; with -DWITH_GPU the same arrays also go through
// nestrank::b200::Layer (conv_fwd_host, 3xTF32) and both outputs are written.
//   adapter_demo <in_padded.bin> <flt.bin> <out_cpu.bin> [<out_gpu.bin>]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "nestrank_b200/psconv_binding.hpp"
#ifdef WITH_GPU
#include <cuda_runtime.h>
#endif

static gemm_microkernel_fn gemm_microkernel_ptr;
#define gemm_microkernel(o, f, i) gemm_microkernel_ptr((o), (f), (i))

static std::vector<float> load(const char* path, size_t n) {
  std::vector<float> v(n);
  FILE* f = std::fopen(path, "rb");
  if (!f || std::fread(v.data(), sizeof(float), n, f) != n) {
    std::fprintf(stderr, "cannot read %s\n", path);
    std::exit(3);
  }
  std::fclose(f);
  return v;
}

static void save(const char* path, const std::vector<float>& v) {
  FILE* f = std::fopen(path, "wb");
  std::fwrite(v.data(), sizeof(float), v.size(), f);
  std::fclose(f);
}

int main(int argc, char** argv) {
  if (argc < 4) return 2;
  const nestrank::ConvPreset p = nestrank::ConvPreset::parse(PRESET_CSV);
  const long hp = (p.ofh - 1) * p.stride_h + p.kh, wp = (p.ofw - 1) * p.stride_w + p.kw;
  const long kb = p.nOfm / p.gemm_block, cb = p.nIfm / p.gemm_block;
  std::vector<float> in = load(argv[1], size_t(p.nImg) * p.nIfm * hp * wp);
  std::vector<float> flt = load(argv[2], size_t(p.nOfm) * p.nIfm * p.kh * p.kw);
  std::vector<float> out(size_t(p.nImg) * p.nOfm * p.ofh * p.ofw, 0.f);
  gemm_microkernel_ptr = nestrank::b200::microkernel(p);
  {
    // array views with the ArrayRef subscripts of presets.hpp:93-97
    auto output = reinterpret_cast<float (*)[KB][OFH][OFW][16]>(out.data());
    auto filter = reinterpret_cast<const float (*)[CB][KH][KW][16][16]>(flt.data());
    auto input = reinterpret_cast<const float (*)[CB][HP][WP][16]>(in.data());
    (void)kb;
    (void)cb;
    int ofm_tile, ifm_tile, oj, kj, ki;  // the emitted pragma names them private
    (void)ofm_tile, (void)ifm_tile, (void)oj, (void)kj, (void)ki;
#include EMITTED_DRIVER
  }
  save(argv[3], out);
#ifdef WITH_GPU
  if (argc > 4) {
    nestrank::b200::Layer layer(p, "", 0, PSCONV_MODE_3XTF32);
    std::vector<float> gout(out.size(), -1.f);
    layer.forward_host(in.data(), flt.data(), gout.data(), 0, p.nImg);
    if (cudaDeviceSynchronize() != cudaSuccess) return 4;
    save(argv[4], gout);
    std::printf("gpu recipe %s\n", layer.recipe().c_str());
  }
#endif
  return 0;
}
