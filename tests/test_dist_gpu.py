"""The N>1 (minibatch-split) path on the real kernel, world size 2 on one GPU.

This environment exposes one B200, and NCCL refuses two ranks on one device, so the ranks
use gloo for their collectives while each runs the real conv_fwd on cuda:0 over its image
shard (independent launches in two processes: no kernel waits on another rank's kernel).
The shards are gathered (variable sizes, dist.gather_shards) and checked against the CPU
oracle; bench.py's own multi-rank path is run the same way under torchrun.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, conv, c_log, cfg_id, mode, result_path):
    import paper_2002_02145_b200 as ps
    from paper_2002_02145_b200 import tune
    from paper_2002_02145_b200.dist import gather_shards, image_range, max_over_ranks
    from paper_2002_02145_b200.workloads import seeds, with_images
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    p = ps.ConvPreset.parse(conv)
    b0, n = image_range(rank, world, p.nImg)
    sx, sw = seeds(cfg_id)
    x = torch.empty(p.input_elems(), device=dev)
    w = torch.empty(p.filter_elems(), device=dev)
    y = torch.full((p.output_elems(),), float("nan"), device=dev)
    ps.fill_input(p, sx, x, c_logical=c_log, img_begin=b0, img_count=n)  # this rank's images only
    ps.fill_filter(p, sw, w, c_logical=c_log)
    # the schedule of this rank's shard (as bench.py chooses it), rank 0's broadcast to all
    obj = [None]
    if rank == 0:
        local = ps.ConvPreset.parse(with_images(conv, n))
        obj[0] = tune.lookup(local, mode) or ps.select_topk(local, mode, 1)[0][0]
    dist.broadcast_object_list(obj, src=0)
    plan = ps.ConvPlan(p, mode=mode, device=0, recipe=obj[0])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.forward(x, w, y, img_begin=b0, img_count=n)
    e1.record()
    torch.cuda.synchronize()
    t = max_over_ranks(e0.elapsed_time(e1))
    per = p.output_elems(n_img=1)
    full = gather_shards(y[b0 * per:(b0 + n) * per].cpu(), p.nImg, per)
    if rank == 0:
        np.save(result_path, full.numpy())
        assert t > 0
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("conv,c_log,cfg_id,mode", [
    ("conv:28,64,64,56,56,3,3,1,1,16,1,1,56,56", 64, 1, "3xtf32"),   # cfg1: 14 + 14 images
    ("conv:5,256,256,14,14,3,3,1,1,16,1,1,14,14", 256, 5, "tf32"),    # uneven: 2 + 3 images
])
def test_two_ranks_real_kernel_gathered_vs_oracle(tmp_path, conv, c_log, cfg_id, mode):
    import oracle
    from paper_2002_02145_b200.workloads import seeds
    res = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(2, _free_port(), conv, c_log, cfg_id, mode, res), nprocs=2, join=True)
    p = __import__("paper_2002_02145_b200").ConvPreset.parse(conv)
    sx, sw = seeds(cfg_id)
    full = np.load(res)
    assert np.isfinite(full).all(), "a shard was not written"
    ref = oracle.conv(p, oracle.fill_input(p, sx, c_log), oracle.fill_filter(p, sw, c_log)).ravel()
    tol = {"3xtf32": 1e-5, "tf32": 5e-3}[mode]
    assert oracle.rel_l2(full, ref) <= tol


@pytest.mark.gpu
def test_bench_two_ranks_under_torchrun():
    """bench.py's N>1 path end to end (torchrun, 2 ranks on the one GPU, gloo collectives):
    per-shard schedule, max-over-ranks timing, variable-size all-gather, oracle verification."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--dist-backend", "gloo", "--workload", "cfg1", "--layers", "none", "--no-f16x2",
           "--steps", "3", "--warmup", "3"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    r = json.loads(lines[0])
    assert r["n_gpus"] == 2 and r["run"]["images_per_gpu"] == 14
    assert r["verified"]["pass"] and r["verified"]["gather"].startswith("gloo")
    assert r["cpu_baseline"]["kind"] in ("reference", "port")
