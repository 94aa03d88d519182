"""ctypes binding of the C ABI in include/psconv.h (libpsconv.so, built in-tree).

The library is the product: sm_100a kernels + the host runtime (descriptor,
recipe/selector, plans). There is no fallback: if the shared object is missing
this module raises at import time.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("PSCONV_LIB_NAME", "libpsconv.so"))  # A/B builds (tools)

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build()); "
        "there is no CPU fallback for the GPU path")

lib = ctypes.CDLL(LIB_PATH)

c_i64 = ctypes.c_int64
c_vp = ctypes.c_void_p


class conv_desc(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in (
        "nImg", "nOfm", "nIfm", "ofh", "ofw", "kh", "kw", "stride_h", "stride_w", "gemm_block",
        "pad_h", "pad_w", "ifh", "ifw")]


class nest_info(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("reserved", ctypes.c_int32), ("desc", conv_desc),
                ("M", c_i64), ("N", c_i64), ("K", c_i64), ("recipe", ctypes.c_char * 256)]


gemm_microkernel_fn = ctypes.CFUNCTYPE(None, ctypes.POINTER(ctypes.c_float),
                                       ctypes.POINTER(ctypes.c_float),
                                       ctypes.POINTER(ctypes.c_float))

_P = ctypes.POINTER
_sigs = {
    "conv_desc_parse": (ctypes.c_int, [ctypes.c_char_p, _P(conv_desc)]),
    "conv_desc_validate": (ctypes.c_int, [_P(conv_desc)]),
    "conv_desc_format": (ctypes.c_int, [_P(conv_desc), ctypes.c_char_p, ctypes.c_size_t]),
    "gemm_microkernel_dispatch": (ctypes.c_int, [_P(conv_desc), _P(gemm_microkernel_fn)]),
    "brgemm_f32": (ctypes.c_int, [_P(conv_desc), c_vp, c_vp, c_vp, c_i64]),
    "conv_plan_create": (ctypes.c_int, [_P(conv_desc), ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                        _P(c_vp)]),
    "conv_plan_destroy": (None, [c_vp]),
    "conv_plan_recipe": (ctypes.c_char_p, [c_vp]),
    "conv_plan_create_bwd_data": (ctypes.c_int, [_P(conv_desc), ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                                  ctypes.POINTER(c_vp)]),
    "conv_fwd": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, ctypes.c_uint]),
    "conv_plan_create_bwd_weight": (ctypes.c_int, [_P(conv_desc), ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                                    ctypes.POINTER(c_vp)]),
    "conv_bwd_weight": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "conv_wgrad_describe": (ctypes.c_int, [_P(conv_desc), ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                           ctypes.c_char_p, ctypes.c_size_t]),
    "conv_model_stats": (ctypes.c_int, [_P(conv_desc), ctypes.c_int, ctypes.c_char_p,
                                         ctypes.POINTER(ctypes.c_double)]),
    "ranker_train": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.c_double, ctypes.c_uint64,
                                     ctypes.c_double, ctypes.c_char_p, ctypes.c_size_t,
                                     ctypes.POINTER(ctypes.c_double)]),
    "ranker_compare": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "conv_select_topk_dnn": (ctypes.c_int, [_P(conv_desc), ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                             ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_double)]),
    "nest_parse": (ctypes.c_int, [ctypes.c_char_p, _P(nest_info)]),
    "gemm_pack_b": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i64, c_vp]),
    "conv_fwd_ex": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, ctypes.c_uint]),
    "conv_fwd_host": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, ctypes.c_uint]),
    "conv_plan_launches": (ctypes.c_int, [c_vp]),
    "conv_plan_prepack": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "conv_plan_emit": (c_i64, [c_vp, ctypes.c_char_p, ctypes.c_size_t]),
    "conv_emit_driver": (c_i64, [_P(conv_desc), ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t]),
    "conv_select_topk": (ctypes.c_int, [_P(conv_desc), ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                        ctypes.c_size_t, _P(ctypes.c_double)]),
    "conv_model_us": (ctypes.c_double, [_P(conv_desc), ctypes.c_int, ctypes.c_char_p]),
    "conv_select_topk_ex": (ctypes.c_int, [_P(conv_desc), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_char_p, ctypes.c_size_t, _P(ctypes.c_double)]),
    "conv_select_set_machine": (ctypes.c_int, [ctypes.c_char_p]),
    "conv_fill_input": (ctypes.c_int, [_P(conv_desc), ctypes.c_uint64, c_i64, c_vp, c_i64, c_i64,
                                       c_vp]),
    "conv_fill_filter": (ctypes.c_int, [_P(conv_desc), ctypes.c_uint64, c_i64, c_vp, c_vp]),
    "conv_pack_input": (ctypes.c_int, [_P(conv_desc), c_vp, c_i64, c_vp, c_vp]),
    "conv_pack_filter": (ctypes.c_int, [_P(conv_desc), c_vp, c_i64, c_vp, c_vp]),
    "conv_unpack_output": (ctypes.c_int, [_P(conv_desc), c_vp, c_vp, c_vp]),
    "conv_last_error": (ctypes.c_char_p, []),
    "psconv_version": (ctypes.c_char_p, []),
    "psconv_device_sm_count": (ctypes.c_int, [ctypes.c_int]),
}
for _name, (_res, _args) in _sigs.items():
    if "PSCONV_LIB_NAME" in os.environ and not hasattr(lib, _name):
        continue  # older A/B build (tools only)
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sigs)
