"""placeholder; replaced below"""
from paper_2409_15097_b200.rng import MT19937_64, uniform_below


def alpaca_lengths(total: int, seed: int = 7, lo: int = 64, span: int = 449):
    """Config 2 segment lengths: L_i = 64 + uniform_below(gen, 449) from mt19937_64(seed), the last
    segment truncated so the lengths fill `total`."""
    gen = MT19937_64(seed)
    out, acc = [], 0
    while acc < total:
        length = lo + uniform_below(gen, span)
        length = min(length, total - acc)
        out.append(length)
        acc += length
    return out
