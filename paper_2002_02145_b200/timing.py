"""Timing helpers shared by bench.py, the tuner and the sweep tools."""
from __future__ import annotations


class L2Flush:
    """Evicts the 126 MB L2 between timed iterations: writes a 256 MiB buffer (larger than
    L2), then reads it back so the dirty lines of that write are written back to HBM before
    the timed region starts (otherwise ~126 MB of write-back lands inside the next timed
    kernel and inflates small kernels by up to ~40%, measured on cfg2)."""

    def __init__(self, device, mib: int = 256):
        import torch
        self.buf = torch.empty(mib * (1 << 20) // 4, dtype=torch.float32, device=device)
        self.acc = torch.empty((), dtype=torch.float32, device=device)

    def __call__(self):
        import torch
        self.buf.fill_(1.0)
        torch.sum(self.buf, dim=0, out=self.acc)
