"""Generates tests/golden/* from the REFERENCE ITSELF, run in the build container.

The reference (arXiv 2002.02145 artefact "nestrank", /root/reference/proj) has no numeric
golden vectors for the conv path -- its arithmetic is the external LIBXSMM microkernel
 -- so these fixtures are produced by executing the reference's own code:

* numeric goldens: oracle/_ref/libref_interp.so = ConvPreset::parse(...).build()
  [+ apply_recipe] walked by oracle_detail::for_each_iteration with the ArrayRef subscripts
  evaluated per point (oracle/ref_interp.cpp), in fp32, on seeded inputs pre-padded to the
  reference-implied extent (presets.hpp:88-91);
* emission goldens: the reference emitter emit_source (emit.hpp:60-134) for several recipes
  (the identity one equals the reference's own tests/golden/conv_identity.c).

Run here (needs /root/reference + `oracle/build_ref.sh`):  python tests/golden/make_golden.py
The outputs are small and committed; tests never need /root/reference at run time.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

# (name, reference conv CSV (10 ints, no padding: input is pre-padded), seeds, recipes)
CASES = [
    ("default", "2,32,32,4,4,3,3,1,1,16", (11, 22),
     [None, "perm=oj,ofm_tile,ifm_tile,kj,ki;tile=oj:3", "perm=kj,ki,oj,ofm_tile,ifm_tile"]),
    ("stride2", "1,16,32,5,7,3,3,2,2,16", (33, 44), [None, "perm=ifm_tile,ofm_tile,oj,kj,ki"]),
    ("pointwise", "2,32,16,6,6,1,1,1,1,16", (55, 66), [None]),
    ("rect", "1,16,16,3,4,2,3,1,2,16", (77, 88), [None, "tile=oj:2"]),
    ("c48k32", "1,32,48,5,5,3,3,1,1,16", (99, 111), [None]),
]

EMIT = [
    ("default", "2,32,32,4,4,3,3,1,1,16", None),
    ("default", "2,32,32,4,4,3,3,1,1,16", "perm=ofm_tile,ifm_tile,oj,kj,ki"),
    ("default", "2,32,32,4,4,3,3,1,1,16", "perm=oj,ofm_tile,ifm_tile,kj,ki;tile=oj:3"),
    ("default", "2,32,32,4,4,3,3,1,1,16", "perm=kj,ki,oj,ofm_tile,ifm_tile;tile=oj:2,ifm_tile:2"),
    ("default", "2,32,32,4,4,3,3,1,1,16", "perm=img,ki"),
    ("cfg1", "28,64,64,56,56,3,3,1,1,16", None),
    ("cfg3", "56,128,128,28,28,3,3,2,2,16", "perm=oj,ofm_tile,ifm_tile,kj,ki;tile=oj:4"),
]


class P:  # minimal ConvPreset-like record for the oracle binding
    def __init__(self, csv):
        v = [int(x) for x in csv.split(",")]
        (self.nImg, self.nOfm, self.nIfm, self.ofh, self.ofw, self.kh, self.kw, self.stride_h,
         self.stride_w, self.gemm_block) = v
        self.pad_h = self.pad_w = 0
        self.ifh = (self.ofh - 1) * self.stride_h + self.kh
        self.ifw = (self.ofw - 1) * self.stride_w + self.kw


def main():
    assert oracle.ref_available(), "build oracle/_ref first (oracle/build_ref.sh)"
    index = {"numeric": [], "emit": []}
    for name, csv, (sx, sw), recipes in CASES:
        p = P(csv)
        x = oracle.fill_input(p, sx)
        w = oracle.fill_filter(p, sw)
        xp = oracle.pad_input(p, x)  # pad 0: identical to x
        arrays = {"input": x, "filter": w}
        for i, rec in enumerate(recipes):
            out, n = oracle.ref_interp(csv, xp, w, (p.nImg, p.nOfm // 16, p.ofh, p.ofw, 16), rec)
            arrays[f"output_{i}"] = out
            index["numeric"].append({"case": name, "conv": "conv:" + csv, "seeds": [sx, sw],
                                     "recipe": rec, "array": f"{name}.npz:output_{i}",
                                     "iterations": n})
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    for i, (name, csv, rec) in enumerate(EMIT):
        fn = f"emit_{i}_{name}.c"
        with open(os.path.join(HERE, fn), "w") as fh:
            fh.write(oracle.ref_emit(csv, rec))
        index["emit"].append({"conv": "conv:" + csv, "recipe": rec, "file": fn})
    with open(os.path.join(HERE, "index.json"), "w") as fh:
        json.dump(index, fh, indent=1)
    print("wrote", len(index["numeric"]), "numeric and", len(index["emit"]), "emission goldens")


if __name__ == "__main__":
    main()
