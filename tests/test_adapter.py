"""The reference-side binding of INTEGRATION.md, compiled and run.

include/nestrank_b200/psconv_binding.hpp is built against the reference headers where they lie
(/root/reference/proj/include) around a driver printed by the reference emitter itself
(emit_source, emit.hpp:60-134), with the psconv CPU microkernel bound through
nestrank::b200::microkernel (gemm_microkernel_dispatch): the C++ program's output must equal
the oracle. The GPU variant (prebuilt here by oracle/build_adapter.py --gpu, it travels in
oracle/_ref/) also runs nestrank::b200::Layer (conv_fwd_host) on the same arrays.
"""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


class P:
    def __init__(self, csv):
        (self.nImg, self.nOfm, self.nIfm, self.ofh, self.ofw, self.kh, self.kw, self.stride_h,
         self.stride_w, self.gemm_block) = [int(x) for x in csv.split(",")]
        self.pad_h = self.pad_w = 0
        self.ifh = (self.ofh - 1) * self.stride_h + self.kh
        self.ifw = (self.ofw - 1) * self.stride_w + self.kw


def _run(exe, csv, tmp_path, gpu):
    p = P(csv)
    x = oracle.fill_input(p, 77)
    w = oracle.fill_filter(p, 88)
    (tmp_path / "in.bin").write_bytes(np.ascontiguousarray(x).tobytes())
    (tmp_path / "flt.bin").write_bytes(np.ascontiguousarray(w).tobytes())
    args = [exe, str(tmp_path / "in.bin"), str(tmp_path / "flt.bin"), str(tmp_path / "cpu.bin")]
    if gpu:
        args.append(str(tmp_path / "gpu.bin"))
    subprocess.run(args, check=True, timeout=300)
    ref = oracle.conv(p, x, w).ravel()
    cpu = np.fromfile(tmp_path / "cpu.bin", np.float32)
    gpu_out = np.fromfile(tmp_path / "gpu.bin", np.float32) if gpu else None
    return ref, cpu, gpu_out


@pytest.mark.skipif(not (os.path.isdir(REF_INC) and oracle.ref_available()),
                    reason="reference headers / emitter not present (build container only)")
@pytest.mark.parametrize("csv", ["2,32,48,7,5,3,3,2,2,16", "3,16,32,6,6,1,1,1,1,16"])
def test_adapter_emitted_driver_with_psconv_microkernel(tmp_path, csv):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from build_adapter import build
    exe = build(csv, gpu=False, out_dir=str(tmp_path))
    ref, cpu, _ = _run(exe, csv, tmp_path, gpu=False)
    # the emitted driver calls the microkernel in the reference's program order: the same
    # fp32 accumulation order as the oracle
    assert oracle.rel_l2(cpu, ref) < 1e-6


@pytest.mark.gpu
def test_adapter_gpu_layer():
    exe = os.path.join(ROOT, "oracle", "_ref", "b200_adapter_demo_gpu")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/b200_adapter_demo_gpu not built (needs the reference headers)")
    import tempfile
    import pathlib
    csv = json.load(open(exe + ".json"))["csv"]
    with tempfile.TemporaryDirectory() as d:
        ref, cpu, gpu = _run(exe, csv, pathlib.Path(d), gpu=True)
    assert oracle.rel_l2(cpu, ref) < 1e-6
    assert oracle.rel_l2(gpu, ref) <= 1e-5, "nestrank::b200::Layer (3xTF32) vs the oracle"


def test_plain_c_program_links_the_abi(tmp_path):
    """include/psconv.h is plain C: a C11 program parses a `conv:` descriptor, formats it
    back, dispatches the 3-pointer microkernel and runs one call (no GPU needed)."""
    src = tmp_path / "abi.c"
    src.write_text(r'''
#include <stdio.h>
#include <string.h>
#include "psconv.h"
int main(void) {
  conv_desc d;
  if (conv_desc_parse("conv:2,32,32,4,4,3,3,1,1,16", &d) != PSCONV_OK) return 1;
  char buf[128];
  if (conv_desc_format(&d, buf, sizeof buf) != PSCONV_OK || strcmp(buf, "conv:2,32,32,4,4,3,3,1,1,16")) return 2;
  if (conv_desc_parse("conv:2,30,32,4,4,3,3,1,1,16", &d) != PSCONV_ERR_CONFIG) return 3;
  conv_desc_parse("conv:1,16,16,1,2,1,1,1,1,16", &d);
  gemm_microkernel_fn mk = 0;
  if (gemm_microkernel_dispatch(&d, &mk) != PSCONV_OK || !mk) return 4;
  float out[32] = {0}, flt[256], in[32];
  for (int i = 0; i < 256; ++i) flt[i] = (float)(i % 7) - 3.f;
  for (int i = 0; i < 32; ++i) in[i] = (float)(i % 5) - 2.f;
  mk(out, flt, in);
  for (int oi = 0; oi < 2; ++oi)
    for (int k = 0; k < 16; ++k) {
      float s = 0.f;
      for (int c = 0; c < 16; ++c) s += flt[c * 16 + k] * in[oi * 16 + c];
      if (s != out[oi * 16 + k]) return 5;
    }
  printf("ok %s\n", psconv_version());
  return 0;
}
''')
    lib_dir = os.path.join(ROOT, "paper_2002_02145_b200")
    exe = tmp_path / "abi"
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Werror", f"-I{os.path.join(ROOT, 'include')}", str(src),
                           "-o", str(exe), f"-L{lib_dir}", "-lpsconv", f"-Wl,-rpath,{lib_dir}"])
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0 and out.stdout.startswith("ok"), (out.returncode, out.stdout, out.stderr)
