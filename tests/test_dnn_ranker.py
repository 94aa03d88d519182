"""Pairwise DNN ranker (reference dnnrank.hpp PairwiseRanker,
pipeline.hpp:98-173): training determinism, weights round trip, dataset validation, and the
tournament ranking over the B200 candidate space. CPU only."""
import random

import pytest

ps = pytest.importorskip("paper_2002_02145_b200")


def _synthetic(n=400, seed=3):
    """Variant A wins iff its total modelled time is smaller (a learnable rule)."""
    rnd = random.Random(seed)
    rows = []
    for _ in range(n):
        a = [rnd.uniform(1, 100) for _ in range(4)]
        b = [rnd.uniform(1, 100) for _ in range(4)]
        rows.append(" ".join(f"{v:.4f}" for v in a + b) + (" A" if sum(a) < sum(b) else " B"))
    return "# a0 a1 a2 a3 b0 b1 b2 b3 winner\n" + "\n".join(rows) + "\n"


def test_train_learns_and_is_deterministic():
    data = _synthetic()
    w1, tr1, ho1 = ps.ranker_train(data, epochs=300, learning_rate=0.01, seed=7, split=0.8)
    w2, tr2, ho2 = ps.ranker_train(data, epochs=300, learning_rate=0.01, seed=7, split=0.8)
    assert w1 == w2 and tr1 == tr2 and ho1 == ho2  # deterministic under the seed
    assert tr1 > 0.9 and ho1 > 0.85
    assert w1.startswith("pairnet 1\ndims 8 64 32 16 8 2\nactivations relu relu softsign relu softmax\n")
    r, pa, pb = ps.ranker_compare(w1, [1, 1, 1, 1], [90, 90, 90, 90])
    assert r == 0 and pa > pb


def test_zero_epochs_and_bad_inputs():
    w, _, _ = ps.ranker_train(_synthetic(40), epochs=0, seed=1, split=1.0)
    assert "theta 0.59999999999999998" in w or "theta 0.6" in w
    for bad in ["", "1 2 3 A\n", "1 2 3 4 5 6 7 8 C\n", "1 2 3 4 5 6 7 8 A extra\n"]:
        with pytest.raises(ps.ConfigRejectedError):
            ps.ranker_train(bad)
    with pytest.raises(ps.ConfigRejectedError):
        ps.ranker_compare("pairnet 2\n", [1, 1, 1, 1], [1, 1, 1, 1])
    with pytest.raises(ps.ConfigRejectedError):
        ps.ranker_compare(w, [0, 0, 0, 0], [0, 0, 0, 0])


def test_tournament_over_candidates():
    p = ps.ConvPreset.parse("conv:2048,256,256,14,14,3,3,1,1,16,1,1,14,14")
    st = ps.model_stats(p, "perm=ofm_tile,ifm_tile,oj,kj,ki;gpu=bn:256,box:2x1x64,cl:1", "3xtf32")
    assert len(st) == 4 and all(v >= 0 for v in st) and st[0] > 0
    ranked = ps.select_topk(p, "3xtf32", k=5, ranker="dnn")
    assert len(ranked) == 5 and len({r for r, _ in ranked}) == 5
    for r, _ in ranked:
        ps.emit_driver(p, r.split(";gpu=")[0])  # every ranked id is a legal reference recipe
