"""Measurement harness for the conv path (SURVEY.md §8 a9 "bench harness", §8 d).

Shared by bench.py: roofline arithmetic, clock sampling, and the two timing protocols of a
layer on one GPU.

* single launch: L2 flushed (256 MiB write + read-back) before every timed step, CUDA events
  on the launching stream around (filter repack +) conv -- the driver's step protocol. It
  includes the per-launch floor of an isolated launch (~5-6 us for an empty 148-CTA kernel
  after the flush, tools/probe_launch.cu), which dominates layers under ~20 us.
* steady state: back-to-back launches cycling through R input/output sets whose combined
  footprint exceeds 2x the 126 MB L2 (each launch reads inputs last touched R-1 launches
  earlier, evicted by the other sets), CUDA events around batches, for >= 0.3 s so the
  nvidia-smi clock record of the layer covers the timed region. This is how the layers run
  inside a network pass (PDL overlaps a launch's prologue with the previous kernel's tail);
  per-launch time = batch time / launches.

Roofline: the slower of FLOPs at the mode's tensor peak (tf32 = measured
cuBLAS bf16 / 2; 3xTF32 = tf32 / 3; f16x2 = bf16 / 3) and compulsory bytes at the measured
HBM copy bandwidth (MEASURED_PEAKS.json).
"""
from __future__ import annotations

import json
import math
import os
import statistics
import subprocess
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HBM_FALLBACK_GBS, BF16_FALLBACK_TFLOPS = 6650.0, 1590.0  # B200_PROFILING.md fallback
L2_BYTES = 126 * (1 << 20)


def peaks():
    """(hbm GB/s, bf16 TFLOP/s, source) -- this pod's MEASURED_PEAKS.json, else the fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            j = json.load(fh)
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), "MEASURED_PEAKS.json (measured)"
    except (OSError, KeyError, ValueError):
        return HBM_FALLBACK_GBS, BF16_FALLBACK_TFLOPS, "B200_PROFILING.md fallback"


def mode_peak_tflops(mode: str, bf16: float) -> float:
    return {"tf32": bf16 / 2.0, "3xtf32": bf16 / 6.0, "f16x2": bf16 / 3.0}[mode]


def compulsory_bytes(p, c_logical=None) -> int:
    """4*(distinct input elements touched + K*C_L*R*S + N*K*P*Q), C_L = the layout channel
    count (the stem's C = 3 padded to 16 is read as 16)."""
    rows = {oj * p.stride_h + kj - p.pad_h for oj in range(p.ofh) for kj in range(p.kh)}
    cols = {oi * p.stride_w + ki - p.pad_w for oi in range(p.ofw) for ki in range(p.kw)}
    ifh = p.ifh or (p.ofh - 1) * p.stride_h + p.kh - 2 * p.pad_h
    ifw = p.ifw or (p.ofw - 1) * p.stride_w + p.kw - 2 * p.pad_w
    nr = sum(1 for r in rows if 0 <= r < ifh)
    nc = sum(1 for c in cols if 0 <= c < ifw)
    touched_in = p.nImg * p.nIfm * nr * nc
    return 4 * (touched_in + p.nOfm * p.nIfm * p.kh * p.kw + p.nImg * p.nOfm * p.ofh * p.ofw)


def flops(p, c_logical=None, n_img=None) -> int:
    """2*N*K*C*P*Q*R*S with the logical C."""
    c = c_logical or p.nIfm
    n = p.nImg if n_img is None else n_img
    return 2 * n * p.nOfm * c * p.ofh * p.ofw * p.kh * p.kw


def roofline(p, c_logical, mode, hbm_gbs, bf16_tflops, n_img=None) -> dict:
    """Roofline time and bound of one launch over n_img images (default all)."""
    n = p.nImg if n_img is None else n_img
    f = flops(p, c_logical, n)
    b = compulsory_bytes(p, c_logical) * n / p.nImg
    pk = mode_peak_tflops(mode, bf16_tflops)
    t_tensor = f / (pk * 1e12)
    t_hbm = b / (hbm_gbs * 1e9)
    return {"flops": f, "bytes": b, "peak_tflops": pk, "t_tensor_s": t_tensor, "t_hbm_s": t_hbm,
            "bound": "tensor" if t_tensor >= t_hbm else "hbm", "t_roof_s": max(t_tensor, t_hbm)}


def roofline_entry(roof, kernel_ms, hbm_gbs) -> dict:
    """The bench line's roofline object for a kernel of average duration kernel_ms."""
    if roof["bound"] == "tensor":
        a = roof["flops"] / (kernel_ms * 1e-3) / 1e12
        return {"bound": "tensor", "achieved": round(a, 2), "peak": round(roof["peak_tflops"], 2),
                "unit": "TFLOP/s", "frac": round(a / roof["peak_tflops"], 4)}
    a = roof["bytes"] / (kernel_ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": round(a, 1), "peak": hbm_gbs, "unit": "GB/s",
            "frac": round(a / hbm_gbs, 4)}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during a measurement window (the
    recipe's clocks line, B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device, period_ms: int = 50):
        self.device = device
        self.period_ms = period_ms
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.device), "-lms", str(self.period_ms)], stdout=self.fh,
                stderr=subprocess.DEVNULL)
            time.sleep(0.15)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.06)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            self.fh.close()

    def summary(self) -> dict:
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        rows = []
        with open(self.path) as fh:
            for line in fh:
                f = [x.strip() for x in line.split(",")]
                if len(f) < 8:
                    continue
                try:
                    rows.append((float(f[0]), float(f[1]), float(f[2]), f[3], f[4], f[5], f[6], f[7]))
                except ValueError:
                    continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        mx = max(r[1] for r in rows)
        load = [r for r in rows if r[2] > 250.0] or rows  # under load: board power above idle
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in load:
            for n, v in zip(names, r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(rows), "samples_under_load": len(load),
                "power_w_max": max(r[2] for r in rows)}


def clocks_ok(c: dict) -> bool:
    """The recipe's rejection rule: no hw / thermal slowdown, SM clock not pinned low."""
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    if bad & set(c.get("reasons", [])):
        return False
    sm, mx = c.get("sm_mhz"), c.get("sm_max_mhz")
    if sm and mx and sm < 0.6 * mx and "sw_power_cap" not in c.get("reasons", []):
        return False
    return True


class LayerBench:
    """Device buffers of one layer (seeded inputs of the named workload) and the two timing
    protocols. `sets` extra input/output copies make the steady-state footprint > 2x L2."""

    def __init__(self, ps, preset, c_logical, seeds, device, img_begin=0, img_count=None):
        import torch
        self.torch = torch
        self.ps = ps
        self.p = preset
        self.c_logical = c_logical
        self.dev = torch.device("cuda", device)
        self.b0 = img_begin
        self.n = preset.nImg - img_begin if img_count is None else img_count
        self.in_img = preset.input_elems(n_img=1)
        self.out_img = preset.output_elems(n_img=1)
        self.x = torch.empty(preset.input_elems(), dtype=torch.float32, device=self.dev)
        self.w = torch.empty(preset.filter_elems(), dtype=torch.float32, device=self.dev)
        self.y = torch.zeros(preset.output_elems(), dtype=torch.float32, device=self.dev)
        ps.fill_input(preset, seeds[0], self.x, c_logical=c_logical, img_begin=self.b0, img_count=self.n)
        ps.fill_filter(preset, seeds[1], self.w, c_logical=c_logical)
        self.stream = torch.cuda.current_stream(self.dev)
        self._sets = None

    # -- single launch after an L2 flush -------------------------------------------------
    def single(self, plan, flush, steps, warmup, prepack_in_step=True):
        """Per-step (repack + conv) and conv-only event times in ms (lists); L2 flushed before
        every step. With prepack_in_step=False the step is the conv alone (prepacked filter).

        Two passes of `steps` L2-flushed launches each: the step pass records events only around
        the whole step (an event between the repack and the conv launch would serialise them:
        the conv's prologue overlaps the repack through PDL, so a middle event adds ~6 us to a
        step of a small layer, tools/step_overhead.py); after a short idle, the kernel pass
        times the conv alone on the prepacked filter."""
        torch, st = self.torch, self.stream

        def one():
            if prepack_in_step:
                plan.prepack(self.w, st)
            plan.forward(self.x, None, self.y, self.b0, self.n, st, prepacked=True)

        if not prepack_in_step:
            plan.prepack(self.w, st)
        for _ in range(warmup):
            one()
        torch.cuda.synchronize()
        # two passes, each started from the same idle power state (the sw power cap lowers the
        # clocks under sustained load: a pass run right after the other, or alternating with it,
        # measured up to 5% slower on cfg5)
        ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(2)) for _ in range(steps)]
        for e0, e1 in ev:
            flush()
            e0.record(st)
            one()
            e1.record(st)
        torch.cuda.synchronize()
        step = [a.elapsed_time(b) for a, b in ev]
        time.sleep(0.3)
        for e0, e1 in ev:
            flush()
            e0.record(st)
            plan.forward(self.x, None, self.y, self.b0, self.n, st, prepacked=True)
            e1.record(st)
        torch.cuda.synchronize()
        return step, [a.elapsed_time(b) for a, b in ev]

    # -- steady state: rotating sets, back-to-back launches -------------------------------
    def _rotating_sets(self):
        if self._sets is None:
            torch = self.torch
            per = 4 * self.n * (self.in_img + self.out_img)
            r = max(2, min(16, math.ceil(2 * L2_BYTES / max(per, 1))))
            free, _ = torch.cuda.mem_get_info(self.dev)
            r = max(2, min(r, int(0.5 * free // max(per, 1)) + 1))
            xs = [self.x[self.b0 * self.in_img:(self.b0 + self.n) * self.in_img]]
            ys = [self.y[self.b0 * self.out_img:(self.b0 + self.n) * self.out_img]]
            for _ in range(r - 1):
                xs.append(xs[0].clone())
                ys.append(torch.empty_like(ys[0]))
            self._sets = (xs, ys)
        return self._sets

    def steady(self, plan, min_seconds=0.3, batch_ms=4.0):
        """Per-launch ms of back-to-back conv launches (prepacked filter) over the rotating
        sets; median over batches of >= batch_ms, batches repeated for >= min_seconds.
        Returns (ms per launch, launches timed, sets)."""
        torch, st = self.torch, self.stream
        xs, ys = self._rotating_sets()
        r = len(xs)
        plan.prepack(self.w, st)

        def launch(i):
            plan.forward(xs[i % r], None, ys[i % r], 0, self.n, st, prepacked=True)

        for i in range(2 * r):
            launch(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for i in range(r):
            launch(i)
        e1.record(st)
        torch.cuda.synchronize()
        est = max(e0.elapsed_time(e1) / r, 1e-3)
        per_batch = max(r, int(math.ceil(batch_ms / est / r)) * r)
        times, total, t_start = [], 0, time.perf_counter()
        while True:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for i in range(per_batch):
                launch(i)
            e1.record(st)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / per_batch)
            total += per_batch
            if time.perf_counter() - t_start >= min_seconds and len(times) >= 3:
                break
        return statistics.median(times), total, r

    def output_images(self, images):
        """Host copies (numpy) of the given global image indices of the current output."""
        out = {}
        for i in images:
            out[i] = self.y[i * self.out_img:(i + 1) * self.out_img].cpu().numpy()
        return out

    def release(self):
        self._sets = None
        self.x = self.w = self.y = None


def tf32_gemm_tflops(device=0, n=8192, reps=10) -> float:
    """Live cuBLAS TF32 GEMM (fp32 in/out, tf32 tensor cores), best of reps (burst)."""
    import torch
    dev = torch.device("cuda", device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        a = torch.randn(n, n, device=dev)
        b = torch.randn(n, n, device=dev)
        c = torch.empty(n, n, device=dev)
        for _ in range(3):
            torch.matmul(a, b, out=c)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
