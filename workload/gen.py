"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module is *input generation only*: it holds none of the HET method's
arithmetic (no dedup, no cache protocol, no SGD).  Both `oracle/` (through the
tests) and the CUDA path (through `bench.py` / the tests) draw their keys and
gradients from here, so the two sides see bit-identical inputs.

Recipe (restated in DESIGN.md "Input recipe"):

* RNG: counter-based ``mix64`` = the splitmix64 finalizer.  The stream for
  (worker i, iteration t, slot j) is ``h = mix64(mix64(mix64(seed ^ i) ^ t) ^ j)``
  and a uniform is ``u = (h >> 11) * 2**-53``.
* Criteo-shaped keys: per sample b and field f, a rank r ~ Zipf(alpha, n_f) by
  inverse CDF, then ``key = offset_f + pi_f(r)`` where ``pi_f`` is a seeded
  bijection of [0, n_f) (4-round Feistel network with cycle walking), so hot
  ids scatter across owners.  Keys are sample-major: ``keys[b*F + f]``.
  The paper's skew statistic (top 10% of Criteo embeddings take 90% of the
  updates, §2.3) calibrates alpha = 0.7.
* Reddit-shaped keys: K distinct node ids per worker-iteration, Zipf(1.0)
  draws over a permuted id space, duplicates rejected, draw order kept
  (GNN batches hold unique ids, §5.1).
* Gradients: ``G[pos][d] = (int32)((h >> 40) - 2**23) * 2**-28`` with h from
  the stream (seed + 1, i, t, pos*D + d): exact fp32 values in [-2^-5, 2^-5).

All tensor arithmetic is int64 torch ops (two's-complement wrap, logical
shifts emulated with masks), so the same function runs on CPU for the oracle
and on CUDA for the bench; ``mix64_py`` is the plain-integer definition the
tests pin it against.
"""
from __future__ import annotations

import math
from functools import lru_cache

import torch

SEED = 2112072210
MASK64 = (1 << 64) - 1
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB


def _signed(c: int) -> int:
    return c - (1 << 64) if c >= (1 << 63) else c


_C1S = _signed(_C1)
_C2S = _signed(_C2)

# Criteo-Kaggle per-field cardinalities (26 categorical fields); sum 33,762,577
# (BASELINE.json configs[1] "~33.8M-row table").
CRITEO_CARDS = [1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145,
                5683, 8351593, 3194, 27, 14992, 5461306, 10, 5652, 2173, 4,
                7046547, 18, 15, 286181, 105, 142572]
TOY_CARDS = [39] * 12 + [38] * 14          # 1,000 rows (BASELINE.json configs[0])
REDDIT_ROWS = 232965                       # BASELINE.json configs[2]


# ----------------------------------------------------------------------------
# mix64: plain-integer definition and the tensor version
# ----------------------------------------------------------------------------
def mix64_py(x: int) -> int:
    """splitmix64 finalizer on a Python int (mod 2^64)."""
    x &= MASK64
    x ^= x >> 30
    x = (x * _C1) & MASK64
    x ^= x >> 27
    x = (x * _C2) & MASK64
    x ^= x >> 31
    return x


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of an int64 tensor viewed as uint64."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def mix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finalizer on an int64 tensor viewed as uint64 (wrapping)."""
    x = x ^ _srl(x, 30)
    x = x * _C1S
    x = x ^ _srl(x, 27)
    x = x * _C2S
    x = x ^ _srl(x, 31)
    return x


def stream_base(seed: int, i: int, t: int) -> int:
    """mix64(mix64(seed ^ i) ^ t) as a Python int: the per-(worker, iteration) prefix."""
    return mix64_py(mix64_py((seed ^ i) & MASK64) ^ (t & MASK64))


def stream(seed: int, i: int, t: int, j: torch.Tensor) -> torch.Tensor:
    """h = mix64(mix64(mix64(seed ^ i) ^ t) ^ j) for a tensor of slots j."""
    return mix64(j ^ _signed(stream_base(seed, i, t)))


def uniform(h: torch.Tensor) -> torch.Tensor:
    return _srl(h, 11).to(torch.float64) * (2.0 ** -53)


# ----------------------------------------------------------------------------
# field layouts
# ----------------------------------------------------------------------------
def scaled_cards(total: int, base=CRITEO_CARDS) -> list[int]:
    """Criteo fields scaled proportionally to `total` rows (>= 1 each); the
    rounding remainder goes to the largest field (SURVEY.md §8(d) 'scale')."""
    s = sum(base)
    cards = [max(1, (c * total) // s) for c in base]
    big = max(range(len(base)), key=lambda f: base[f])
    cards[big] += total - sum(cards)
    assert sum(cards) == total and min(cards) >= 1
    return cards


def cards_for(name: str) -> list[int]:
    if name == "toy":
        return list(TOY_CARDS)
    if name in ("criteo", "wdl", "dcn"):
        return list(CRITEO_CARDS)
    if name == "scale":
        return scaled_cards(24_000_000)
    raise ValueError(name)


# ----------------------------------------------------------------------------
# Zipf inverse CDF and seeded permutations
# ----------------------------------------------------------------------------
@lru_cache(maxsize=64)
def _zipf_cdf_cpu(n: int, alpha: float) -> torch.Tensor:
    r = torch.arange(1, n + 1, dtype=torch.float64)
    p = r.pow(-alpha)
    cdf = torch.cumsum(p, 0)
    cdf /= cdf[-1].clone()
    cdf[-1] = 1.0
    return cdf


_cdf_dev_cache: dict = {}


def zipf_cdf(n: int, alpha: float, device) -> torch.Tensor:
    device = torch.device(device)
    if device.type == "cpu":
        return _zipf_cdf_cpu(n, alpha)
    k = (n, alpha, str(device))
    if k not in _cdf_dev_cache:
        _cdf_dev_cache[k] = _zipf_cdf_cpu(n, alpha).to(device)
    return _cdf_dev_cache[k]


def zipf_rank(u: torch.Tensor, n: int, alpha: float) -> torch.Tensor:
    """Smallest r in [0, n) with CDF[r] > u  (P(r) proportional to (r+1)^-alpha)."""
    cdf = zipf_cdf(n, alpha, u.device)
    r = torch.searchsorted(cdf, u.contiguous(), right=True)
    return r.clamp_(max=n - 1)


def _feistel_params(n: int, salt: int):
    b = max(2, (n - 1).bit_length())
    b += b & 1
    half = b // 2
    keys = [_signed(mix64_py((SEED ^ 0x5045524D00000000 ^ (salt * 0x9E3779B97F4A7C15) ^ r) & MASK64))
            for r in range(4)]
    return half, (1 << half) - 1, keys


def _feistel(x: torch.Tensor, half: int, mask: int, keys) -> torch.Tensor:
    L = x >> half
    R = x & mask
    for k in keys:
        L, R = R, L ^ (mix64(R ^ k) & mask)
    return (L << half) | R


def permute(r: torch.Tensor, n: int, salt: int) -> torch.Tensor:
    """Seeded bijection of [0, n) (Feistel on [0, 2^b) + cycle walking)."""
    if n == 1:
        return torch.zeros_like(r)
    half, mask, keys = _feistel_params(n, salt)
    y = _feistel(r, half, mask, keys)
    bad = y >= n
    while bool(bad.any()):
        y[bad] = _feistel(y[bad], half, mask, keys)
        bad = y >= n
    return y


# ----------------------------------------------------------------------------
# public generators
# ----------------------------------------------------------------------------
def criteo_keys(i: int, t0: int, T: int, B: int, cards: list[int], alpha: float = 0.7,
                seed: int = SEED, device="cpu") -> torch.Tensor:
    """Keys for worker i, iterations t0..t0+T-1: int64 [T, B*F], sample-major."""
    F = len(cards)
    offs = [0]
    for c in cards[:-1]:
        offs.append(offs[-1] + c)
    j = torch.arange(B * F, dtype=torch.int64, device=device)
    bases = torch.tensor([_signed(stream_base(seed, i, t)) for t in range(t0, t0 + T)],
                         dtype=torch.int64, device=device)
    h = mix64(bases[:, None] ^ j[None, :])                     # [T, B*F]
    u = uniform(h).view(T, B, F)
    out = torch.empty(T, B, F, dtype=torch.int64, device=device)
    for f in range(F):
        r = zipf_rank(u[:, :, f].reshape(-1), cards[f], alpha)
        out[:, :, f] = (offs[f] + permute(r, cards[f], f + 1)).view(T, B)
    return out.view(T, B * F)


def reddit_keys(i: int, t: int, K: int, R: int = REDDIT_ROWS, alpha: float = 1.0,
                seed: int = SEED, device="cpu", chunk: int = 16384) -> torch.Tensor:
    """K distinct node ids for worker i, iteration t (draw order kept)."""
    assert K <= R
    seen = torch.zeros(R, dtype=torch.bool, device=device)
    got = []
    have = 0
    j0 = 0
    while have < K:
        j = torch.arange(j0, j0 + chunk, dtype=torch.int64, device=device)
        j0 += chunk
        ids = permute(zipf_rank(uniform(stream(seed, i, t, j)), R, alpha), R, 0xEDD17)
        # first occurrence within the chunk, in draw order
        uniq, inv = torch.unique(ids, return_inverse=True)
        first = torch.full((uniq.numel(),), chunk, dtype=torch.int64, device=device)
        first.scatter_reduce_(0, inv, torch.arange(chunk, dtype=torch.int64, device=device), reduce="amin")
        order = torch.sort(first).values
        cand = ids[order]
        cand = cand[~seen[cand]]
        cand = cand[: K - have]
        seen[cand] = True
        got.append(cand)
        have += cand.numel()
    return torch.cat(got)


def grads(i: int, t: int, n: int, D: int, seed: int = SEED, device="cpu") -> torch.Tensor:
    """Synthetic exact-fp32 gradients [n, D] for worker i, iteration t."""
    j = torch.arange(n * D, dtype=torch.int64, device=device)
    h = stream(seed + 1, i, t, j)
    v = (_srl(h, 40) - (1 << 23)).to(torch.float32) * (2.0 ** -28)
    return v.view(n, D)


def dense_grads(i: int, t: int, P: int, seed: int = SEED, device="cpu") -> torch.Tensor:
    """Synthetic dense-model gradient buffer [P] (fp32) for worker i, iteration t."""
    j = torch.arange(P, dtype=torch.int64, device=device)
    h = stream(seed + 2, i, t, j)
    return (_srl(h, 40) - (1 << 23)).to(torch.float32) * (2.0 ** -28)
