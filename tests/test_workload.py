"""Pins of the shared input generator (workload/gen.py)."""
import numpy as np
import pytest
import torch

from workload import gen


def test_mix64_tensor_matches_integer_definition():
    xs = [0, 1, 2, 12345, (1 << 63) - 1, (1 << 63), (1 << 64) - 1, 0xDEADBEEFCAFEF00D]
    t = torch.tensor([gen._signed(x) for x in xs], dtype=torch.int64)
    got = [int(v) & gen.MASK64 for v in gen.mix64(t).tolist()]
    assert got == [gen.mix64_py(x) for x in xs]


def test_zipf_normalisation(golden):
    ex = golden["zipf"][0]            # alpha=1, m=3 -> P(1) = 6/11
    cdf = gen.zipf_cdf(ex["m"], ex["alpha"], "cpu")
    assert abs(float(cdf[0]) - ex["p_top_num"] / ex["p_top_den"]) < 1e-15
    # m = 1 -> always rank 0
    u = torch.rand(100, dtype=torch.float64)
    assert (gen.zipf_rank(u, 1, 1.0) == 0).all()


def test_zipf_empirical_frequencies():
    u = gen.uniform(gen.stream(gen.SEED, 0, 0, torch.arange(200000)))
    r = gen.zipf_rank(u, 5, 1.0)
    freq = torch.bincount(r, minlength=5).double() / r.numel()
    p = 1.0 / torch.arange(1, 6, dtype=torch.float64)
    p /= p.sum()
    assert (freq - p).abs().max() < 5e-3


@pytest.mark.parametrize("n", [1, 2, 3, 39, 1000, 4099])
def test_permutation_is_bijection(n):
    r = torch.arange(n, dtype=torch.int64)
    y = gen.permute(r, n, salt=5)
    assert sorted(y.tolist()) == list(range(n))


def test_skew_calibration(golden):
    """the top 10% of Criteo rows take ~90% of accesses at alpha=0.7."""
    ex = golden["skew"][0]
    cards = gen.cards_for("criteo")
    ps = []
    for c in cards:
        p = np.arange(1, c + 1, dtype=np.float64) ** -ex["alpha"]
        ps.append(p / p.sum() / len(cards))
    p = np.sort(np.concatenate(ps))[::-1]
    share = p[: len(p) // 10].sum()
    assert ex["top10_share_min"] <= share <= ex["top10_share_max"]


def test_criteo_keys_shape_range_determinism():
    cards = gen.cards_for("toy")
    k1 = gen.criteo_keys(0, 3, 2, 128, cards)
    k2 = gen.criteo_keys(0, 3, 2, 128, cards)
    assert k1.shape == (2, 128 * 26)
    assert torch.equal(k1, k2)
    assert int(k1.min()) >= 0 and int(k1.max()) < sum(cards)
    offs = np.cumsum([0] + cards)
    f = np.arange(128 * 26) % 26
    kk = k1[0].numpy()
    assert ((kk >= offs[f]) & (kk < offs[f + 1])).all()
    assert not torch.equal(k1[0], gen.criteo_keys(1, 3, 1, 128, cards)[0])


def test_reddit_keys_distinct():
    k = gen.reddit_keys(0, 0, 2000, R=5000)
    assert k.numel() == 2000 and torch.unique(k).numel() == 2000
    assert int(k.min()) >= 0 and int(k.max()) < 5000


def test_grads_exact_range():
    g = gen.grads(0, 0, 64, 8)
    assert g.dtype == torch.float32
    assert float(g.abs().max()) < 2.0 ** -5
    q = g.double() * 2 ** 28
    assert torch.equal(q, q.round())


def test_scaled_cards():
    c = gen.cards_for("scale")
    assert sum(c) == 24_000_000 and len(c) == 26 and min(c) >= 1
