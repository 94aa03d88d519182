"""Multi-process sharding path on CPU (gloo, world_size 2): each rank computes its image shard
(the CPU oracle stands in for the per-GPU conv_fwd), shards are gathered, and the result must
equal the single-process conv bit-exactly (images are independent units)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2002_02145_b200.dist import image_range  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, conv, result_path):
    import oracle
    import paper_2002_02145_b200 as ps
    from paper_2002_02145_b200.dist import gather_shards, max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = ps.ConvPreset.parse(conv)
    b0, n = image_range(rank, world, p.nImg)
    x = oracle.fill_input(p, 1234, img_begin=b0, img_count=n)   # keyed by global image index
    w = oracle.fill_filter(p, 5678)
    out = oracle.conv(ps.ConvPreset.parse(conv.replace(f"conv:{p.nImg},", f"conv:{n},", 1)), x, w) \
        if n else np.zeros((0,), np.float32)
    per = p.output_elems(n_img=1)
    full = gather_shards(torch.from_numpy(out.ravel().copy()), p.nImg, per)
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        np.save(result_path, full.numpy())
        assert t == world
    dist.destroy_process_group()


@pytest.mark.parametrize("conv", ["conv:5,32,32,6,6,3,3,1,1,16,1,1,6,6",
                                  "conv:4,16,32,5,5,3,3,2,2,16,1,1,10,10"])
def test_two_rank_shards_equal_full(tmp_path, conv):
    import oracle
    import paper_2002_02145_b200 as ps
    world = 2
    res = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(world, _free_port(), conv, res), nprocs=world, join=True)
    p = ps.ConvPreset.parse(conv)
    ref = oracle.conv(p, oracle.fill_input(p, 1234), oracle.fill_filter(p, 5678)).ravel()
    assert np.array_equal(np.load(res), ref)


def test_image_ranges_cover_exactly():
    for n in (1, 5, 28, 2048):
        for world in (1, 2, 3, 4, 8):
            got = [image_range(r, world, n) for r in range(world)]
            assert sum(c for _, c in got) == n
            assert all(got[i][0] + got[i][1] == got[i + 1][0] for i in range(world - 1))
    assert image_range(0, 8, 2048) == (0, 256) and image_range(7, 8, 2048) == (1792, 256)
