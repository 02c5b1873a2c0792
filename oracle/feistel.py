"""Oracle: splitmix64 and the SAMPLE-mode permutation pi_seed over [0, n).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SURVEY Appendix A.1 (reading R3 in DESIGN.md): a 4-round balanced Feistel network on
b = max(2, ceil(log2 n)) bits (rounded up to even), cycle-walked into [0, n).  The CUDA
library implements the same counter-based generator independently.
"""

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def splitmix64(z):
    z = (z + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


class Feistel:
    def __init__(self, n, seed):
        if n < 1:
            raise ValueError("empty domain")
        self.n = n
        b = max(2, (n - 1).bit_length())          # ceil(log2 n) for n >= 2
        if b % 2:
            b += 1
        self.h = b // 2
        self.mask = (1 << self.h) - 1
        self.keys = [splitmix64((seed ^ ((GOLDEN * (r + 1)) & MASK64)) & MASK64) for r in range(4)]

    def _E(self, x):
        L, R = x >> self.h, x & self.mask
        for k in self.keys:
            L, R = R, L ^ (splitmix64(R ^ k) & self.mask)
        return (L << self.h) | R

    def __call__(self, j):
        if not 0 <= j < self.n:
            raise IndexError(j)
        x = self._E(j)
        while x >= self.n:
            x = self._E(x)
        return x
