"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA-side bench.

This module holds none of the method's arithmetic (no decoding, validity, simulator, GP or
acquisition).  It only draws seeded random numbers and composes callables that each side
passes in from its own implementation.

Recipe (DESIGN.md §4 "Input recipe", after SURVEY §8(d) "Observed set and value
distributions"; the noise model follows SPEC wrap_noisy, and the paper's
simulator-noise ablation P:437):
  * observed configurations: CVI positions p_t = splitmix64(seed ^ 0x0B5E ^ t) mod N_cvi,
    t = 0, 1, ...; keep the first M distinct positions whose configuration passes the
    resource check.  (Profiling is out of scope; these stand in for profiled points.)
  * observed cost = cost_sim(x) * exp(0.3 * sin(sum_j w_j * digit_j/(n_j-1) + w0)) * (1 + noise*u)
    with w_j = 3 u(seed ^ 0xA0 ^ j), w0 = 3 u(seed ^ 0xB0), u = u(seed ^ 0xC0 ^ raw) in [-1, 1):
    a smooth structured simulator bias the GP can learn plus i.i.d. profiling noise.
"""

from __future__ import annotations

import math

MASK64 = (1 << 64) - 1


def splitmix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def u_pm1(z: int) -> float:
    """Uniform in [-1, 1) from a 64-bit counter."""
    return 2.0 * ((splitmix64(z & MASK64) >> 11) * 2.0 ** -53) - 1.0


def observed_set(M, seed, n_cvi, domain_sizes, unrank, is_valid, cost_sim, noise=0.05, max_draws=None):
    """Return (raws, costs) of M synthetic profiled configurations.

    unrank(p) -> (raw, digits);  is_valid(raw) -> bool (resource check);  cost_sim(raw) -> float.
    Each callable comes from the side that consumes the inputs (oracle or CUDA library).
    """
    d = len(domain_sizes)
    w = [3.0 * u_pm1(seed ^ 0xA0 ^ j) for j in range(d)]
    w0 = 3.0 * u_pm1(seed ^ 0xB0)
    seen = set()
    raws, costs = [], []
    t = 0
    max_draws = max_draws if max_draws is not None else 200 * max(M, 1) + 1000
    while len(raws) < M and t < max_draws:
        p = splitmix64(seed ^ 0x0B5E ^ t) % n_cvi
        t += 1
        if p in seen:
            continue
        seen.add(p)
        raw, digits = unrank(p)
        if not is_valid(raw):
            continue
        s = sum(w[j] * (digits[j] / (domain_sizes[j] - 1) if domain_sizes[j] > 1 else 0.0) for j in range(d))
        c = cost_sim(raw) * math.exp(0.3 * math.sin(s + w0)) * (1.0 + noise * u_pm1(seed ^ 0xC0 ^ raw))
        raws.append(int(raw))
        costs.append(float(c))
    if len(raws) < M:
        raise RuntimeError(f"only {len(raws)} valid observed points found")
    return raws, costs
