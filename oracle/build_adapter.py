"""Builds oracle/_ref/b200_adapter_demo*: the reference-side binding
(include/nestrank_b200/psconv_binding.hpp) compiled against the reference headers WHERE THEY
LIE (/root/reference/proj/include) around a driver the REFERENCE EMITTER printed
(emit_source, emit.hpp:60-134, via oracle/_ref/libref_interp.so) -- test infrastructure for
tests/test_adapter.py (INTEGRATION.md's adapter, proven at the C++ level).

  python oracle/build_adapter.py [--gpu] [--csv 2,32,48,7,5,3,3,2,2,16] [--out DIR]
Outputs only into oracle/_ref/ (or --out); links paper_2002_02145_b200/libpsconv.so.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_INC = os.environ.get("REF_INCLUDE", "/root/reference/proj/include")
DEFAULT_CSV = "2,32,48,7,5,3,3,2,2,16"


def build(csv: str, gpu: bool, out_dir: str) -> str:
    sys.path.insert(0, ROOT)
    import oracle
    v = [int(x) for x in csv.split(",")]
    n, K, C, P, Q, R, S, sh, sw, blk = v
    text = oracle.ref_emit(csv, None)  # the reference emitter's identity driver
    os.makedirs(out_dir, exist_ok=True)
    tag = "gpu" if gpu else "cpu"
    inc = os.path.join(out_dir, f"adapter_emitted_{tag}.inc")
    with open(inc, "w") as fh:
        fh.write(text)
    exe = os.path.join(out_dir, f"b200_adapter_demo_{tag}")
    defs = {"PRESET_CSV": f'"{csv}"', "KB": K // blk, "CB": C // blk, "OFH": P, "OFW": Q, "KH": R,
            "KW": S, "HP": (P - 1) * sh + R, "WP": (Q - 1) * sw + S, "EMITTED_DRIVER": f'"{inc}"'}
    lib_dir = os.path.join(ROOT, "paper_2002_02145_b200")
    cmd = ["g++", "-std=c++20", "-O2", "-fopenmp", f"-I{REF_INC}", f"-I{os.path.join(ROOT, 'include')}"]
    cmd += [f"-D{k}={val}" for k, val in defs.items()]
    if gpu:
        cmd += ["-DWITH_GPU", "-I/usr/local/cuda/include"]
    cmd += [os.path.join(ROOT, "tests", "adapter", "adapter_demo.cpp"), "-o", exe, f"-L{lib_dir}", "-lpsconv",
            f"-Wl,-rpath,{lib_dir}", "-Wl,-rpath,$ORIGIN/../../paper_2002_02145_b200"]
    if gpu:
        cmd += ["-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.check_call(cmd)
    with open(exe + ".json", "w") as fh:
        json.dump({"csv": csv, "gpu": gpu}, fh)
    return exe


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpu", action="store_true")
    ap.add_argument("--csv", default=DEFAULT_CSV)
    ap.add_argument("--out", default=os.path.join(HERE, "_ref"))
    a = ap.parse_args()
    if not os.path.isdir(os.path.join(REF_INC, "nestrank")):
        print("build_adapter: reference headers not found; skipping", file=sys.stderr)
        return 0
    print(build(a.csv, a.gpu, a.out))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
