"""Pure-Python twin of the oracle's tau-nice sampler (SURVEY 8(c) "SAMPLE").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Written independently of
oracle/pcdm_oracle.c with Python big integers and a set, so that a slip in one
(a wrong shift, a swapped counter word, an off-by-one in the rejection bound)
shows up as a disagreement.  Small n / tau only: it is slow.

The law it implements is the tau-nice sampling of PAPER.md:436-438 (uniform
over all tau-subsets of [n]); the concrete counter layout and ownership rule
are the SURVEY 8(c) reading (the paper gives only the law).
"""
from __future__ import annotations

M32 = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """Philox4x32 with 10 rounds (Salmon et al., SC'11)."""
    x = [int(c) & M32 for c in ctr]
    k = [int(key[0]) & M32, int(key[1]) & M32]
    for rnd in range(10):
        if rnd:
            k = [(k[0] + 0x9E3779B9) & M32, (k[1] + 0xBB67AE85) & M32]
        a = 0xD2511F53 * x[0]
        c = 0xCD9E8D57 * x[2]
        x = [((c >> 32) ^ x[1] ^ k[0]) & M32, c & M32, ((a >> 32) ^ x[3] ^ k[1]) & M32, a & M32]
    return x


def draw(seed, k, rho, j, tag, n):
    out = philox4x32_10([j, k, rho, tag], [seed & M32, (seed >> 32) & M32])
    u = (out[1] << 32) | out[0]
    prod = u * n
    low = prod % (1 << 64)
    if low < ((1 << 64) - n) % n:
        return None
    return prod >> 64


def sample(seed, k, tau, n):
    assert 1 <= tau <= n
    comp = 2 * tau > n
    cnt = n - tau if comp else tau
    tag = 2 if comp else 1
    owner = {}          # value -> slot that owns it
    slot_val = [None] * cnt
    pending = list(range(cnt))
    rho = 0
    while pending:
        nxt = []
        for j in pending:
            v = draw(seed, k, rho, j, tag, n)
            if v is None or v in owner:
                nxt.append(j)
            else:
                owner[v] = j
                slot_val[j] = v
        pending = nxt
        rho += 1
    if comp:
        return [v for v in range(n) if v not in owner]
    return slot_val


# ---------------------------------------------------------------- other DU samplings (NEXT-1)
def word(seed, k, j, tag):
    out = philox4x32_10([j, k, 0, tag], [seed & M32, (seed >> 32) & M32])
    return (out[1] << 32) | out[0]


def threshold(p):
    """(always, floor(p * 2^64)) with exact rational arithmetic on the double p."""
    from fractions import Fraction
    if p >= 1.0:
        return True, 0
    if p <= 0.0:
        return False, 0
    return False, int(Fraction(p) * (1 << 64))


def sample_independent(seed, k, tau, n):
    picked = set()
    out = []
    for j in range(tau):
        rho = 0
        while True:
            v = draw(seed, k, rho, j, 3, n)
            if v is not None:
                break
            rho += 1
        out.append(-1 if v in picked else v)
        picked.add(v)
    return out


def sample_binomial(seed, k, tau, n, p_b):
    s = sample(seed, k, tau, n)
    always, T = threshold(p_b)
    return [v if always or word(seed, k, j, 4) < T else -1 for j, v in enumerate(s)]


def sample_du(seed, k, tau, n, q):
    assert 2 * tau <= n
    s = sample(seed, k, tau, n)
    u = word(seed, k, 0, 5)
    cum = 0.0
    K = tau
    for size in range(tau):
        cum += float(q[size])        # same left-to-right fp64 cumulative sums
        always, T = threshold(cum)
        if always or u < T:
            K = size
            break
    return [v if j < K else -1 for j, v in enumerate(s)]
