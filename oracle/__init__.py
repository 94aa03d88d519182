"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Python binding of oracle/liboracle.so (plain-C restatement of the reference
conv nest, see oracle.h) and, where it was built, oracle/_ref/libref_interp.so
(the reference's own IR executed numerically, see ref_interp.cpp).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this package.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_REF = os.path.join(_HERE, "_ref", "libref_interp.so")

c_i64 = ctypes.c_int64
c_vp = ctypes.c_void_p


class oc_desc(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in (
        "nImg", "nOfm", "nIfm", "ofh", "ofw", "kh", "kw", "stride_h", "stride_w", "gemm_block",
        "pad_h", "pad_w", "ifh", "ifw")]


def _load():
    if not os.path.exists(_LIB):
        raise ImportError(f"{_LIB} missing: run `make oracle`")
    lib = ctypes.CDLL(_LIB)
    P = ctypes.POINTER(oc_desc)
    sig = {
        "oracle_value": (ctypes.c_float, [ctypes.c_uint64, ctypes.c_uint64]),
        "oracle_fill_input": (None, [P, ctypes.c_uint64, c_i64, c_vp, c_i64, c_i64]),
        "oracle_fill_filter": (None, [P, ctypes.c_uint64, c_i64, c_vp]),
        "oracle_pad_input": (None, [P, c_vp, c_vp, c_i64]),
        "oracle_conv_fig5": (None, [P, c_vp, c_vp, c_vp, c_i64, c_i64]),
        "oracle_gemm_microkernel": (None, [P, c_vp, c_vp, c_vp]),
        "oracle_conv_f64": (None, [P, c_vp, c_vp, c_vp, c_i64, c_i64]),
        "oracle_threads": (ctypes.c_int, []),
    }
    for k, (r, a) in sig.items():
        f = getattr(lib, k)
        f.restype, f.argtypes = r, a
    return lib


lib = _load()


def desc(p) -> oc_desc:
    """oc_desc from a ConvPreset-like object (ifh/ifw resolved by the caller or here)."""
    ifh = p.ifh or (p.ofh - 1) * p.stride_h + p.kh - 2 * p.pad_h
    ifw = p.ifw or (p.ofw - 1) * p.stride_w + p.kw - 2 * p.pad_w
    return oc_desc(p.nImg, p.nOfm, p.nIfm, p.ofh, p.ofw, p.kh, p.kw, p.stride_h, p.stride_w,
                   p.gemm_block, p.pad_h, p.pad_w, ifh, ifw)


def _p(a: np.ndarray) -> int:
    assert a.flags.c_contiguous
    return a.ctypes.data


def threads() -> int:
    return lib.oracle_threads()


def value(seed: int, idx: int) -> float:
    return lib.oracle_value(seed, idx)


def fill_input(p, seed: int, c_logical: int = 0, img_begin: int = 0, img_count=None) -> np.ndarray:
    d = desc(p)
    n = p.nImg - img_begin if img_count is None else img_count
    # the C routine indexes arrays from image 0: hand it a base shifted back by
    # img_begin images (only images [img_begin, img_begin+n) are written)
    out = np.zeros((n, p.nIfm // 16, d.ifh, d.ifw, 16), np.float32)
    img_bytes = 4 * (p.nIfm // 16) * d.ifh * d.ifw * 16
    lib.oracle_fill_input(ctypes.byref(d), seed, c_logical, _p(out) - img_begin * img_bytes,
                          img_begin, n)
    return out


def fill_filter(p, seed: int, c_logical: int = 0) -> np.ndarray:
    d = desc(p)
    out = np.zeros((p.nOfm // 16, p.nIfm // 16, p.kh, p.kw, 16, 16), np.float32)
    lib.oracle_fill_filter(ctypes.byref(d), seed, c_logical, _p(out))
    return out


def pad_input(p, inp: np.ndarray) -> np.ndarray:
    d = desc(p)
    n = inp.shape[0]
    hp = (p.ofh - 1) * p.stride_h + p.kh
    wp = (p.ofw - 1) * p.stride_w + p.kw
    out = np.empty((n, p.nIfm // 16, hp, wp, 16), np.float32)
    lib.oracle_pad_input(ctypes.byref(d), _p(np.ascontiguousarray(inp)), _p(out), n)
    return out


def conv_fig5(p, in_padded: np.ndarray, flt: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    """Fig. 5 identity-order fp32 conv over all images of ``in_padded`` (out += conv)."""
    d = desc(p)
    n = in_padded.shape[0]
    if out is None:
        out = np.zeros((n, p.nOfm // 16, p.ofh, p.ofw, 16), np.float32)
    lib.oracle_conv_fig5(ctypes.byref(d), _p(np.ascontiguousarray(in_padded)),
                         _p(np.ascontiguousarray(flt)), _p(out), 0, n)
    return out


def conv(p, inp: np.ndarray, flt: np.ndarray) -> np.ndarray:
    """Convenience: pad + Fig. 5 (fresh zero output)."""
    return conv_fig5(p, pad_input(p, inp), flt)


def conv_f64(p, inp: np.ndarray, flt: np.ndarray) -> np.ndarray:
    d = desc(p)
    n = inp.shape[0]
    out = np.zeros((n, p.nOfm // 16, p.ofh, p.ofw, 16), np.float64)
    lib.oracle_conv_f64(ctypes.byref(d), _p(np.ascontiguousarray(inp)),
                        _p(np.ascontiguousarray(flt)), _p(out), 0, n)
    return out


def rel_l2(got, ref) -> float:
    got = np.asarray(got, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    den = np.linalg.norm(ref.ravel())
    return float(np.linalg.norm((got - ref).ravel()) / (den if den else 1.0))


def max_abs(got, ref) -> float:
    return float(np.max(np.abs(np.asarray(got, np.float64).ravel() - np.asarray(ref, np.float64).ravel())))


# ----------------------------------------------------------------- reference IR
def ref_available() -> bool:
    return os.path.exists(_REF)


def _ref():
    lib_r = ctypes.CDLL(_REF)
    lib_r.ref_interp_conv.restype = c_i64
    lib_r.ref_interp_conv.argtypes = [ctypes.c_char_p, ctypes.c_char_p, c_vp, c_vp, c_vp]
    lib_r.ref_emit.restype = c_i64
    lib_r.ref_emit.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t]
    lib_r.ref_interp_error.restype = ctypes.c_char_p
    return lib_r


def ref_interp(csv10: str, in_padded: np.ndarray, flt: np.ndarray, out_shape, recipe: str | None = None):
    """Runs the reference IR (ConvPreset::build + for_each_iteration) numerically."""
    r = _ref()
    out = np.zeros(out_shape, np.float32)
    n = r.ref_interp_conv(csv10.encode(), recipe.encode() if recipe else None,
                          _p(np.ascontiguousarray(in_padded)), _p(np.ascontiguousarray(flt)), _p(out))
    if n < 0:
        raise RuntimeError(r.ref_interp_error().decode())
    return out, int(n)


def ref_emit(csv10: str, recipe: str | None = None) -> str:
    r = _ref()
    n = r.ref_emit(csv10.encode(), recipe.encode() if recipe else None, None, 0)
    if n < 0:
        raise RuntimeError(r.ref_interp_error().decode())
    buf = ctypes.create_string_buffer(int(n) + 1)
    r.ref_emit(csv10.encode(), recipe.encode() if recipe else None, buf, len(buf))
    return buf.value.decode()
