"""Pins the oracle to the REFERENCE ITSELF at BASELINE sizes (VERDICT r1 item 1 / SURVEY §8c
step 2): one-image slices of cfg1/2/3/5 and of the ResNet-50 stem (its first 16-channel
output block), each executed by the reference's own IR -- ConvPreset::build +
oracle_detail::for_each_iteration with the ArrayRef subscripts evaluated per point
(oracle/ref_interp.cpp over /root/reference/proj/include, presets.hpp:60-127,
oracle.hpp:22-43) -- on the seeded inputs of the named workload (the slice's global image
index keys the generator, so it is the same image the GPU computes at full N).

Writes tests/golden/slices.json: per slice the reference output's sha256 (fp32 bytes), its
iteration count and its relative L2 vs the float64 direct conv. The CPU tests recompute the
oracle on the same slice and require the identical sha256 (bit-exact), without needing
/root/reference; where the reference interpreter is built they also re-run it live.

Run here (needs /root/reference + oracle/build_ref.sh):  python tests/golden/make_slices.py
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

# (name, workload conv string (14 fields), logical C, seed id, image, output-channel blocks)
SLICES = [
    ("cfg1", "conv:28,64,64,56,56,3,3,1,1,16,1,1,56,56", 64, 1, 27, None),
    ("cfg2", "conv:28,64,256,56,56,1,1,1,1,16,0,0,56,56", 256, 2, 27, None),
    ("cfg3", "conv:56,128,128,28,28,3,3,2,2,16,1,1,56,56", 128, 3, 55, None),
    ("cfg5", "conv:2048,256,256,14,14,3,3,1,1,16,1,1,14,14", 256, 5, 2047, None),
    ("r50_stem", "conv:256,64,16,112,112,7,7,2,2,16,3,3,224,224", 3, 100, 255, 1),
]


class P:
    """ConvPreset-like record (no dependency on the product package)."""

    def __init__(self, conv):
        v = [int(x) for x in conv.split(":", 1)[1].split(",")]
        (self.nImg, self.nOfm, self.nIfm, self.ofh, self.ofw, self.kh, self.kw, self.stride_h,
         self.stride_w, self.gemm_block, self.pad_h, self.pad_w, self.ifh, self.ifw) = v

    def csv10(self):
        return ",".join(str(getattr(self, k)) for k in (
            "nImg", "nOfm", "nIfm", "ofh", "ofw", "kh", "kw", "stride_h", "stride_w", "gemm_block"))


def slice_inputs(conv, c_log, cfg_id, img, kblocks):
    """(one-image sliced descriptor, its input, its filter) with the workload's seeds."""
    full = P(conv)
    sx, sw = 1000 + cfg_id, 2000 + cfg_id
    x = oracle.fill_input(full, sx, c_log, img_begin=img, img_count=1)
    w = oracle.fill_filter(full, sw, c_log)
    s = P(conv)
    s.nImg = 1
    if kblocks is not None:
        s.nOfm = 16 * kblocks
        w = np.ascontiguousarray(w[:kblocks])
    return s, x, w


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.float32).tobytes()).hexdigest()


def main():
    assert oracle.ref_available(), "build oracle/_ref first (oracle/build_ref.sh)"
    out = []
    for name, conv, c_log, cfg_id, img, kb in SLICES:
        s, x, w = slice_inputs(conv, c_log, cfg_id, img, kb)
        t = time.time()
        ref, n = oracle.ref_interp(s.csv10(), oracle.pad_input(s, x), w, (1, s.nOfm // 16, s.ofh, s.ofw, 16))
        dt = time.time() - t
        f64 = oracle.conv_f64(s, x, w)
        out.append({"name": name, "conv": conv, "c_logical": c_log, "cfg_id": cfg_id, "image": img,
                    "ofm_blocks": kb, "ref_csv10": s.csv10(), "iterations": n, "sha256": sha(ref),
                    "rel_l2_vs_f64": oracle.rel_l2(ref, f64), "ref_seconds": round(dt, 2)})
        print(out[-1], flush=True)
    with open(os.path.join(HERE, "slices.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
