"""B200-native blocked direct-convolution forward (the PolyScientist hot path).

Python mirror of the reference's operator interface for this path, over the C
ABI in include/psconv.h:

* :class:`ConvPreset` — the conv-layer descriptor (reference
  ``nestrank::ConvPreset``, include/nestrank/presets.hpp:13-58): same fields,
  same ``conv:`` CSV, same validation and error class (``ConfigRejectedError``,
  common.hpp:26 — CLI exit status 2), plus the padding / input-extent extension.
* :class:`ConvPlan` — one layer on one GPU: a descriptor, an arithmetic mode
  (3xTF32 fp32-faithful, or TF32) and a schedule in the reference's recipe
  grammar (variants.hpp:16-65).
* :func:`gemm_microkernel` — the 3-pointer CPU microkernel contract
  (presets.hpp:116-123).

The GPU path has no fallback: this package fails at import when libpsconv.so
is missing, and ConvPlan creation fails on anything but an sm_100 device.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, fields

from . import _lib
from ._lib import conv_desc, lib

__all__ = [
    "Error", "ConfigRejectedError", "AnalysisError", "ConvPreset", "ConvPlan", "MODE_3XTF32",
    "MODE_TF32", "MODE_F16X2", "WgradPlan", "FLAG_ACCUMULATE", "emit_driver", "select_topk", "model_us", "gemm_microkernel",
    "brgemm", "fill_input", "fill_filter", "version", "parse_nest", "NestInfo", "GemmPlan",
    "model_stats", "ranker_train", "ranker_compare", "default_ranker_weights", "pack_input",
    "pack_filter", "unpack_output", "set_machine", "load_measured_peaks",
]

MODE_3XTF32 = 0
MODE_TF32 = 1
MODE_F16X2 = 2  # fp32-faithful: power-of-two scaled fp16 hi/lo split (three K=16 f16 MMAs)
FLAG_ACCUMULATE = 1
FLAG_PREPACKED = 2
FLAG_RELU = 4
_MODES = {"3xtf32": MODE_3XTF32, "tf32": MODE_TF32, "f16x2": MODE_F16X2}


class Error(RuntimeError):
    """Base error (reference nestrank::Error, common.hpp:11-13)."""


class ConfigRejectedError(Error):
    """Input / config error: status 2 (reference ConfigRejectedError & co.)."""


class AnalysisError(Error):
    """Runtime / analysis error: status 1."""


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = (lib.conv_last_error() or b"").decode()
    if rc == 2:
        raise ConfigRejectedError(msg)
    raise AnalysisError(msg or f"psconv error {rc}")


def version() -> str:
    return lib.psconv_version().decode()


@dataclass
class ConvPreset:
    """Conv-layer descriptor; field order = the reference ``conv:`` CSV order."""
    nImg: int = 2
    nOfm: int = 32
    nIfm: int = 32
    ofh: int = 4
    ofw: int = 4
    kh: int = 3
    kw: int = 3
    stride_h: int = 1
    stride_w: int = 1
    gemm_block: int = 16
    pad_h: int = 0
    pad_w: int = 0
    ifh: int = 0
    ifw: int = 0

    # -- reference interface -------------------------------------------------
    @classmethod
    def parse(cls, csv: str) -> "ConvPreset":
        """``conv:nImg,...,gemm_block[,pad_h,pad_w[,ifh,ifw]]`` (presets.hpp:26-50)."""
        d = conv_desc()
        _check(lib.conv_desc_parse(csv.encode(), ctypes.byref(d)))
        return cls._from_c(d)

    def validate(self) -> "ConvPreset":
        d = self.to_c()
        _check(lib.conv_desc_validate(ctypes.byref(d)))
        self.ifh, self.ifw = d.ifh, d.ifw
        return self

    # -- helpers ---------------------------------------------------------------
    @classmethod
    def _from_c(cls, d: conv_desc) -> "ConvPreset":
        return cls(**{f.name: int(getattr(d, f.name)) for f in fields(cls)})

    def to_c(self) -> conv_desc:
        return conv_desc(**{f.name: int(getattr(self, f.name)) for f in fields(self)})

    def __str__(self) -> str:
        d = self.to_c()
        buf = ctypes.create_string_buffer(512)
        _check(lib.conv_desc_format(ctypes.byref(d), buf, len(buf)))
        return buf.value.decode()

    @property
    def csv10(self) -> str:
        return ",".join(str(getattr(self, n)) for n in (
            "nImg", "nOfm", "nIfm", "ofh", "ofw", "kh", "kw", "stride_h", "stride_w", "gemm_block"))

    def flops(self, c_logical: int | None = None, n_img: int | None = None) -> int:
        """Algorithmic FLOPs 2*N*K*C*P*Q*R*S (logical C)."""
        c = c_logical or self.nIfm
        n = self.nImg if n_img is None else n_img
        return 2 * n * self.nOfm * c * self.ofh * self.ofw * self.kh * self.kw

    def input_elems(self, n_img: int | None = None) -> int:
        v = self.validate()
        return (self.nImg if n_img is None else n_img) * v.nIfm * v.ifh * v.ifw

    def filter_elems(self) -> int:
        return self.nOfm * self.nIfm * self.kh * self.kw

    def output_elems(self, n_img: int | None = None) -> int:
        return (self.nImg if n_img is None else n_img) * self.nOfm * self.ofh * self.ofw


def _stream_ptr(stream) -> int:
    if stream is None:
        try:
            import torch
            return torch.cuda.current_stream().cuda_stream
        except Exception:  # noqa: BLE001
            return 0
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


def _ptr(t) -> int:
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    if hasattr(t, "ctypes"):  # numpy array (host buffers for forward_host)
        return t.ctypes.data
    return int(t)


class WgradPlan:
    """Backward-weight plan of a forward layer (C ABI conv_plan_create_bwd_weight):
    forward(x, dy, dw) computes dW (KCRS16c16k) from X (NCHW16c) and dY (NKPQ16k) with the
    pixel-major wgrad kernel (MN-major tf32 operands straight from the activation layouts,
    split over pixel ranges, partials added in split order)."""

    def __init__(self, preset: "ConvPreset", mode="3xtf32", device: int = 0, recipe: str | None = None,
                 c_logical: int = 0):
        """c_logical < 16 on a one-block (nIfm = 16) layer whose padded input channels are zero
        (the ResNet stem): the tap-folded path (recipe pp:C)."""
        if isinstance(mode, str):
            mode = _MODES[mode.lower()]
        if c_logical and c_logical < 16 and preset.nIfm == 16 and not (recipe and "pp:" in recipe):
            recipe = f"{recipe},pp:{c_logical}" if recipe and "gpu=" in recipe else f"gpu=pp:{c_logical}"
        self.preset = ConvPreset(**{f.name: getattr(preset, f.name) for f in fields(preset)}).validate()
        self.mode = mode
        self.device = device
        self._d = self.preset.to_c()
        h = ctypes.c_void_p()
        _check(lib.conv_plan_create_bwd_weight(ctypes.byref(self._d), mode, device,
                                               recipe.encode() if recipe else None, ctypes.byref(h)))
        self._h = h

    @property
    def recipe(self) -> str:
        """The wgrad kernel's geometry (gpu=sw:,kn:,cn:,nt:,box:,sp:,st:,ch:)."""
        return lib.conv_plan_recipe(self._h).decode()

    @staticmethod
    def describe(preset: "ConvPreset", mode="3xtf32", num_sms: int = 148, recipe: str | None = None) -> str:
        """The geometry a plan would choose on a GPU with num_sms SMs (host only)."""
        if isinstance(mode, str):
            mode = _MODES[mode.lower()]
        d = preset.to_c()
        buf = ctypes.create_string_buffer(512)
        _check(lib.conv_wgrad_describe(ctypes.byref(d), mode, num_sms, recipe.encode() if recipe else None,
                                       buf, len(buf)))
        return buf.value.decode()

    def forward(self, x, dy, dw, stream=None) -> None:
        _check(lib.conv_bwd_weight(self._h, _ptr(x), _ptr(dy), _ptr(dw), _stream_ptr(stream)))

    __call__ = forward

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.conv_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass


def _cached_bwd_data_recipe(preset: "ConvPreset", mode: int) -> str | None:
    """Backward data of a stride-1 layer is the forward conv of its transposed descriptor
    (channels swapped, padding k - 1 - pad), which is often another layer's forward shape (the
    ResNet 3x3s, the 1x1 pairs 64->256 / 256->64 ...): reuse that shape's measured recipe from
    the committed plan cache. Strided layers run per-phase child plans (selector choice)."""
    if preset.stride_h != 1 or preset.stride_w != 1:
        return None
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "plans_b200.json")
    try:
        with open(path) as fh:
            cache = json.load(fh)
    except (OSError, ValueError):
        return None
    p = preset
    t = ConvPreset(nImg=p.nImg, nOfm=p.nIfm, nIfm=p.nOfm, ofh=p.ifh, ofw=p.ifw, kh=p.kh, kw=p.kw, stride_h=1,
                   stride_w=1, gemm_block=p.gemm_block, pad_h=p.kh - 1 - p.pad_h, pad_w=p.kw - 1 - p.pad_w,
                   ifh=p.ofh, ifw=p.ofw)
    try:
        t.validate()
    except Error:
        return None
    name = {v: k for k, v in _MODES.items()}.get(mode, mode)
    e = cache.get(f"{t}|{name}")
    if not e or "pp:" in e["recipe"] or "fold:" in e["recipe"]:
        return None
    return e["recipe"]


class ConvPlan:
    """One conv layer bound to a device, a mode and a schedule (recipe)."""

    def __init__(self, preset: ConvPreset, mode="3xtf32", device: int = 0,
                 recipe: str | None = None, bwd_data: bool = False):
        """bwd_data=True: the backward-data plan of the forward layer `preset`; forward(dy, w,
        dx) then computes dX from dY (NKPQ16k) and the forward filter (strided layers: one
        stride-1 transposed conv per output phase, C ABI conv_plan_create_bwd_data)."""
        if isinstance(mode, str):
            mode = _MODES[mode.lower()]
        self.preset = ConvPreset(**{f.name: getattr(preset, f.name) for f in fields(preset)}).validate()
        self.mode = mode
        self.device = device
        self.bwd_data = bwd_data
        if bwd_data and recipe is None:
            recipe = _cached_bwd_data_recipe(self.preset, mode)
        self._d = self.preset.to_c()
        h = ctypes.c_void_p()
        create = lib.conv_plan_create_bwd_data if bwd_data else lib.conv_plan_create
        _check(create(ctypes.byref(self._d), mode, device, recipe.encode() if recipe else None,
                      ctypes.byref(h)))
        self._h = h

    @property
    def recipe(self) -> str:
        return lib.conv_plan_recipe(self._h).decode()

    @property
    def launches(self) -> int:
        return lib.conv_plan_launches(self._h)

    def emit(self) -> str:
        n = lib.conv_plan_emit(self._h, None, 0)
        if n < 0:
            _check(int(-n))
        buf = ctypes.create_string_buffer(int(n) + 1)
        lib.conv_plan_emit(self._h, buf, len(buf))
        return buf.value.decode()

    def prepack(self, flt, stream=None) -> None:
        """Repack a constant filter once; then forward(..., prepacked=True) skips that launch."""
        _check(lib.conv_plan_prepack(self._h, _ptr(flt), _stream_ptr(stream)))

    def forward(self, inp, flt, out, img_begin: int = 0, img_count: int | None = None,
                stream=None, accumulate: bool = False, prepacked: bool = False,
                bias=None, relu: bool = False) -> None:
        """Device pointers or CUDA tensors in NCHW16c / KCRS16c16k / NKPQ16k. Optional fused
        epilogue: + bias[nOfm] (device), ReLU (C ABI conv_fwd_ex)."""
        if img_count is None:
            img_count = self.preset.nImg - img_begin
        flags = ((FLAG_ACCUMULATE if accumulate else 0) | (FLAG_PREPACKED if prepacked else 0)
                 | (FLAG_RELU if relu else 0))
        if bias is None and not relu:
            _check(lib.conv_fwd(self._h, _ptr(inp), 0 if flt is None else _ptr(flt), _ptr(out),
                                img_begin, img_count, _stream_ptr(stream), flags))
        else:
            _check(lib.conv_fwd_ex(self._h, _ptr(inp), 0 if flt is None else _ptr(flt), _ptr(out),
                                   0 if bias is None else _ptr(bias), img_begin, img_count,
                                   _stream_ptr(stream), flags))

    __call__ = forward

    def graph(self, inp, flt, out, img_begin: int = 0, img_count: int | None = None,
              accumulate: bool = False, prepacked: bool = True):
        """Capture this call (fixed pointers) into a CUDA graph: returns a torch.cuda.CUDAGraph
        whose replay() re-runs the conv (launch + PDL edges, plus a split-K flag reset when the
        schedule splits tail tiles) with less host and launch overhead than forward() --
        serving loops over the same buffers. One warm-up call runs first (lazy allocations)."""
        import torch
        dev = torch.device("cuda", self.device)
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            self.forward(inp, flt, out, img_begin, img_count, stream=side, accumulate=accumulate,
                         prepacked=prepacked)
        torch.cuda.current_stream(dev).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            self.forward(inp, flt, out, img_begin, img_count, stream=side, accumulate=accumulate,
                         prepacked=prepacked)
        return g

    def forward_host(self, inp, flt, out, img_begin: int = 0, img_count: int | None = None,
                     stream=None, accumulate: bool = False, prepacked: bool = False) -> None:
        """conv on HOST buffers (CPU tensors / numpy arrays; pinned for full overlap): the
        image range is streamed through the device in double-buffered chunks (C ABI
        conv_fwd_host). Stream-ordered: `out` is complete once `stream` reaches this call."""
        if img_count is None:
            img_count = self.preset.nImg - img_begin
        flags = (FLAG_ACCUMULATE if accumulate else 0) | (FLAG_PREPACKED if prepacked else 0)
        _check(lib.conv_fwd_host(self._h, _ptr(inp), 0 if flt is None else _ptr(flt), _ptr(out),
                                 img_begin, img_count, _stream_ptr(stream), flags))

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.conv_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


@dataclass
class NestInfo:
    """What a reference nest document computes (C ABI nest_parse)."""
    kind: str                    # "conv" or "gemm"
    preset: ConvPreset           # the conv descriptor (gemm: the equivalent 1x1 conv)
    recipe: str                  # conv: outer-loop order as a reference recipe id
    M: int = 0
    N: int = 0
    K: int = 0


def parse_nest(text: str) -> NestInfo:
    """Reads a reference nest document (loopnest.hpp:340-523 grammar; e.g. samples/conv2d.nest,
    samples/matmul.nest) and recognises the computation."""
    info = _lib.nest_info()
    _check(lib.nest_parse(text.encode(), ctypes.byref(info)))
    kind = {1: "conv", 2: "gemm"}[info.kind]
    return NestInfo(kind, ConvPreset._from_c(info.desc), info.recipe.decode(), info.M, info.N, info.K)


class GemmPlan:
    """C[M][N] = A[M][K] @ B[K][N] (row-major fp32, device) on the conv kernel: row-major A
    is NCHW16c and C is NKPQ16k at H = W = 1, so the product is a 1x1 convolution over M
    "images"; B is blocked once per call by gemm_pack_b (N, K multiples of 16)."""

    def __init__(self, M: int, N: int, K: int, mode="3xtf32", device: int = 0,
                 recipe: str | None = None):
        self.M, self.N, self.K = M, N, K
        self.conv = ConvPlan(ConvPreset.parse(f"conv:{M},{N},{K},1,1,1,1,1,1,16"), mode=mode,
                             device=device, recipe=recipe)
        self._bblk = None

    @property
    def recipe(self) -> str:
        return self.conv.recipe

    def forward(self, a, b, c, stream=None) -> None:
        import torch
        if self._bblk is None:
            self._bblk = torch.empty(self.K * self.N, dtype=torch.float32,
                                     device=torch.device("cuda", self.conv.device))
        _check(lib.gemm_pack_b(_ptr(b), _ptr(self._bblk), self.K, self.N, _stream_ptr(stream)))
        self.conv.forward(a, self._bblk, c, stream=stream)

    __call__ = forward


def emit_driver(preset: ConvPreset, recipe: str | None = None) -> str:
    """Driver loop nest text in the reference emitter's format (emit.hpp:60-134)."""
    d = preset.to_c()
    rc = lib.conv_emit_driver(ctypes.byref(d), recipe.encode() if recipe else None, None, 0)
    if rc < 0:
        _check(int(-rc))
    buf = ctypes.create_string_buffer(int(rc) + 1)
    lib.conv_emit_driver(ctypes.byref(d), recipe.encode() if recipe else None, buf, len(buf))
    return buf.value.decode()


def select_topk(preset: ConvPreset, mode="3xtf32", k: int = 5, ranker: str = "cost",
                weights: str | None = None, c_logical: int = 0):
    """Ranked recipes, best first: [(recipe, modelled_us), ...]. ranker="cost" sorts by the
    closed-form model (costrank.hpp:31-40 analogue); ranker="dnn" runs the pairwise-net
    tournament with `weights` (pairnet text; default: the shipped B200 weights)."""
    if isinstance(mode, str):
        mode = _MODES[mode.lower()]
    d = preset.to_c()
    buf = ctypes.create_string_buffer(1 << 16)
    if ranker == "dnn":
        w = (weights if weights is not None else default_ranker_weights()).encode()
        sym = ctypes.c_double()
        n = lib.conv_select_topk_dnn(ctypes.byref(d), mode, k, w, buf, len(buf), ctypes.byref(sym))
        if n < 0:
            _check(-n)
        ids = buf.value.decode().split("\n") if n else []
        mname = {v: k for k, v in _MODES.items()}[mode]
        return [(r, model_us(preset, r, mname)) for r in ids]
    us = (ctypes.c_double * k)()
    # (c_logical: the caller's assertion that only that many input channels are non-zero --
    # lets the model rank the few-channel kernel, recipe pp:C)
    n = lib.conv_select_topk_ex(ctypes.byref(d), mode, int(c_logical), k, buf, len(buf), us)
    if n < 0:
        _check(-n)
    ids = buf.value.decode().split("\n") if n else []
    return list(zip(ids, [us[i] for i in range(n)]))


def model_stats(preset: ConvPreset, recipe: str, mode="3xtf32") -> list[float]:
    """The pairwise ranker's four statistics of one recipe (us: MMA, shared memory, operand
    rows, HBM) from the closed-form model."""
    if isinstance(mode, str):
        mode = _MODES[mode.lower()]
    d = preset.to_c()
    st = (ctypes.c_double * 4)()
    _check(lib.conv_model_stats(ctypes.byref(d), mode, recipe.encode(), st))
    return list(st)


def ranker_train(dataset: str, epochs: int = 300, learning_rate: float = 0.01, seed: int = 1,
                 split: float = 0.8) -> tuple[str, float, float]:
    """Trains the pairwise net on dataset rows "a0..a3 b0..b3 A|B"; returns (weights text,
    train accuracy, holdout accuracy or -1)."""
    buf = ctypes.create_string_buffer(1 << 20)
    acc = (ctypes.c_double * 2)()
    _check(lib.ranker_train(dataset.encode(), epochs, learning_rate, seed, split, buf, len(buf), acc))
    return buf.value.decode(), acc[0], acc[1]


def ranker_compare(weights: str, a, b) -> tuple[int, float, float]:
    """(0 A faster | 1 B faster | 2 draw, p_A, p_B)."""
    arr = ctypes.c_double * 4
    prob = (ctypes.c_double * 2)()
    r = lib.ranker_compare(weights.encode(), arr(*a), arr(*b), prob)
    if r < 0:
        _check(-r)
    return r, prob[0], prob[1]


def default_ranker_weights() -> str:
    """The shipped B200 weights (tools/train_ranker.py)."""
    import os
    path = os.path.join(os.path.dirname(__file__), "ranker_b200.pairnet")
    with open(path) as f:
        return f.read()


def model_us(preset: ConvPreset, recipe: str, mode="3xtf32") -> float:
    if isinstance(mode, str):
        mode = _MODES[mode.lower()]
    d = preset.to_c()
    v = lib.conv_model_us(ctypes.byref(d), mode, recipe.encode())
    if v < 0:
        _check(2)
    return v


def gemm_microkernel(preset: ConvPreset):
    """The dispatched 3-pointer CPU microkernel (a ctypes function)."""
    d = preset.to_c()
    fn = _lib.gemm_microkernel_fn()
    _check(lib.gemm_microkernel_dispatch(ctypes.byref(d), ctypes.byref(fn)))
    return fn


def brgemm(preset: ConvPreset, out_ptr: int, flt_ptrs, in_ptrs) -> None:
    d = preset.to_c()
    n = len(flt_ptrs)
    fa = (ctypes.c_void_p * n)(*flt_ptrs)
    ia = (ctypes.c_void_p * n)(*in_ptrs)
    _check(lib.brgemm_f32(ctypes.byref(d), out_ptr, fa, ia, n))


def pack_input(preset: ConvPreset, nchw, out, c_logical: int = 0, stream=None) -> None:
    """NCHW (c_logical channels) -> NCHW16c of `preset` (device buffers; channels >= c_logical
    zero-filled): the blocked layout of the reference's input ArrayRef (presets.hpp:93-97)."""
    d = preset.to_c()
    _check(lib.conv_pack_input(ctypes.byref(d), _ptr(nchw), c_logical, _ptr(out), _stream_ptr(stream)))


def pack_filter(preset: ConvPreset, kcrs, out, c_logical: int = 0, stream=None) -> None:
    """KCRS (c_logical input channels) -> KCRS16c16k (presets.hpp:93-97 filter subscripts)."""
    d = preset.to_c()
    _check(lib.conv_pack_filter(ctypes.byref(d), _ptr(kcrs), c_logical, _ptr(out), _stream_ptr(stream)))


def unpack_output(preset: ConvPreset, nkpq16k, out, stream=None) -> None:
    """NKPQ16k (the reference's output ArrayRef) -> plain NKPQ."""
    d = preset.to_c()
    _check(lib.conv_unpack_output(ctypes.byref(d), _ptr(nkpq16k), _ptr(out), _stream_ptr(stream)))


def set_machine(**consts: float) -> None:
    """Selector machine constants (C ABI conv_select_set_machine): hbm_gbs, tf32_tflops,
    clock_ghz, sms, l2_bytes."""
    text = "\n".join(f"{k} {float(v)!r}" for k, v in consts.items())
    _check(lib.conv_select_set_machine(text.encode()))


def load_measured_peaks(path: str | None = None) -> dict | None:
    """Feeds the pod's measured peaks (MEASURED_PEAKS.json: HBM copy GB/s, cuBLAS bf16
    TFLOP/s -> tf32 = bf16 / 2) to the selector's model; returns what was set, or None when
    the file is absent (the model keeps its built-in constants)."""
    import json
    import os
    path = path or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            j = json.load(fh)
        consts = {"hbm_gbs": float(j["hbm_gbs"]), "tf32_tflops": float(j["bf16_tflops"]) / 2.0}
    except (OSError, KeyError, ValueError, TypeError):
        return None
    set_machine(**consts)
    return consts


def fill_input(preset: ConvPreset, seed: int, inp, c_logical: int = 0, img_begin: int = 0,
               img_count: int | None = None, stream=None) -> None:
    """Seeded uniform[-1,1) activations on the device (NCHW16c, logical-index keyed)."""
    d = preset.to_c()
    if img_count is None:
        img_count = preset.nImg - img_begin
    _check(lib.conv_fill_input(ctypes.byref(d), seed, c_logical, _ptr(inp), img_begin, img_count,
                               _stream_ptr(stream)))


def fill_filter(preset: ConvPreset, seed: int, flt, c_logical: int = 0, stream=None) -> None:
    d = preset.to_c()
    _check(lib.conv_fill_filter(ctypes.byref(d), seed, c_logical, _ptr(flt), _stream_ptr(stream)))


MACHINE = load_measured_peaks()  # this pod's peaks into the selector (None: built-in constants)
