"""Host<->device copy bandwidth on this box (the e2e leg's bound): pinned H2D alone,
D2H alone, and both at once on two streams. python tools/pcie_probe.py [MB]"""
import sys
import torch

mb = int(sys.argv[1]) if len(sys.argv) > 1 else 400
n = mb * 2**20 // 4
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, device="cuda")
d_out = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=5):
    best = 1e9
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_event(e0)
        s2.wait_event(e0)
        if h2d:
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for name, a, b in (("h2d", 1, 0), ("d2h", 0, 1), ("both", 1, 1)):
    ms = run(a, b)
    print(f"{name}: {mb} MB each way in {ms:.3f} ms -> {mb * 2**20 * (a + b) / ms / 1e6:.1f} GB/s total")


# chunked, duplex: H2D chunk i+1 overlaps D2H chunk i (the conv_fwd_host pattern
# without the kernel)
def chunked(chunk_mb, reps=5):
    cn = chunk_mb * 2**20 // 4
    k = n // cn
    best = 1e9
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_event(e0)
        s2.wait_event(e0)
        for i in range(k):
            with torch.cuda.stream(s1):
                d_in[i * cn:(i + 1) * cn].copy_(h_in[i * cn:(i + 1) * cn], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s1)
            s2.wait_event(ev)
            with torch.cuda.stream(s2):
                h_out[i * cn:(i + 1) * cn].copy_(d_in[i * cn:(i + 1) * cn], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, k


for cmb in (8, 32, 64):
    ms, k = chunked(cmb)
    print(f"chunked {cmb} MB x {k}: {ms:.3f} ms -> {2 * k * cmb * 2**20 / ms / 1e6:.1f} GB/s total")
