"""Oracle: splitmix64 and the SAMPLE-mode permutation pi_seed over [0, n).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

DESIGN.md reading R3 (a refinement of SURVEY Appendix A.1): a 4-round Feistel network on
b = max(2, ceil(log2 n)) bits, cycle-walked into [0, n) (so fewer than 2 walks are expected).
The halves are unbalanced when b is odd: x = (L, R) with |L| = ceil(b/2), |R| = floor(b/2); each
round maps (L, R) -> (R, L xor F_r(R)) so the half sizes alternate and return after 4 rounds.
F_r(x) = fmix32(x xor k_r) masked to the width of L, k_r = low 32 bits of
splitmix64(seed xor golden*(r+1)); fmix32 is MurmurHash3's 32-bit finaliser.  n < 2^32.
The CUDA library implements the same counter-based generator independently.
"""

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def splitmix64(z):
    z = (z + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


MASK32 = (1 << 32) - 1


def fmix32(h):
    h &= MASK32
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & MASK32
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & MASK32
    h ^= h >> 16
    return h


class Feistel:
    def __init__(self, n, seed):
        if n < 1:
            raise ValueError("empty domain")
        if n > (1 << 32):
            raise ValueError("domain larger than 2^32")
        self.n = n
        b = max(2, (n - 1).bit_length())          # ceil(log2 n) for n >= 2
        self.a = (b + 1) // 2                     # |L|
        self.c = b // 2                           # |R|
        self.keys = [splitmix64((seed ^ ((GOLDEN * (r + 1)) & MASK64)) & MASK64) & MASK32 for r in range(4)]

    def _E(self, x):
        a, c = self.a, self.c
        L, R = x >> c, x & ((1 << c) - 1)
        for k in self.keys:
            # (L: a bits, R: c bits) -> (R: c bits, L ^ F(R): a bits); sizes swap every round
            L, R = R, L ^ (fmix32(R ^ k) & ((1 << a) - 1))
            a, c = c, a
        return (L << c) | R

    def __call__(self, j):
        if not 0 <= j < self.n:
            raise IndexError(j)
        x = self._E(j)
        while x >= self.n:
            x = self._E(x)
        return x
