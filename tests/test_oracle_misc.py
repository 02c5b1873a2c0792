"""Pins for oracle/feistel.py, oracle/run.py top-k and the synthgen inputs (not gpu).

  * splitmix64: published reference outputs of Vigna's SplitMix64 (seed 0, seed 1234567);
  * Feistel: exhaustive bijectivity of pi_seed on [0, n) (SURVEY §8(c) row 'Feistel');
  * top-k: SIM-mode top-1 = brute-force argmin of the simulated cost, ties -> first in
    enumeration order (S:503-506 brute_force_optimum); k >= #valid returns every valid
    configuration; order (score desc, raw asc).
"""

import numpy as np
import pytest

import synthgen
from oracle import feistel, run, sim


def test_splitmix64_reference_vectors():
    # Vigna's reference: state += golden; mix.  seed 0 -> 0xE220A8397B1DCDAF
    assert feistel.splitmix64(0) == 0xE220A8397B1DCDAF
    s = 1234567
    outs = []
    for _ in range(3):
        outs.append(feistel.splitmix64(s))
        s = (s + feistel.GOLDEN) & feistel.MASK64
    assert outs == [6457827717110365317, 3203168211198807973, 9817491932198370423]
    assert synthgen.splitmix64(0) == feistel.splitmix64(0)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 1000, (1 << 20) - 3])
@pytest.mark.parametrize("seed", [0, 0xDEADBEEF])
def test_feistel_bijective(n, seed):
    pi = feistel.Feistel(n, seed)
    img = np.array([pi(j) for j in range(n)])
    assert img.min() >= 0 and img.max() < n
    assert len(np.unique(img)) == n


def test_feistel_not_identity():
    pi = feistel.Feistel(1000, 1)
    assert sum(pi(j) == j for j in range(1000)) < 20


@pytest.mark.parametrize("name", ["P0", "C1", "C2"])
def test_sim_top1_is_bruteforce_argmin(oracle_spaces, name):
    sp = oracle_spaces[name]
    fit = run.observed_fit(sp, [], [])
    n = sp.n_cvi()
    rec = run.score_batch(sp, fit, "range", 0, n, acq="sim")
    top = run.topk(rec, 5)
    # brute force: argmin over enumerate(space) of cost, ties -> first in enumeration order
    cost = np.where(rec["valid"], rec["cost"], np.inf)
    i = int(np.argmin(cost))                  # argmin returns the first minimum
    assert top[0][0] == int(rec["raw"][i])
    assert top[0][1] == pytest.approx(-np.log(cost[i]), rel=1e-15)
    scores = [s for _, s in top]
    assert scores == sorted(scores, reverse=True)


def test_topk_all_valid_when_k_large(oracle_spaces):
    sp = oracle_spaces["C1"]
    fit = run.observed_fit(sp, [], [])
    rec = run.score_batch(sp, fit, "range", 0, sp.n_cvi(), acq="lcb")
    top = run.topk(rec, 10_000)
    assert len(top) == int(rec["valid"].sum()) == 176
    keys = [(-s, r) for r, s in top]
    assert keys == sorted(keys)


def test_observed_set_recipe_deterministic(oracle_spaces):
    sp = oracle_spaces["C2"]

    def unrank(p):
        dg = sp.cvi_unrank(p)
        return sp.encode_raw(dg), dg

    def valid(raw):
        return bool(sim.simulate(sp, [sp.decode_raw(raw)])[1][0])

    def cost(raw):
        return float(sim.simulate(sp, [sp.decode_raw(raw)])[0][0])

    sizes = [f.n for f in sp.features]
    a = synthgen.observed_set(16, 5, sp.n_cvi(), sizes, unrank, valid, cost)
    b = synthgen.observed_set(16, 5, sp.n_cvi(), sizes, unrank, valid, cost)
    assert a == b and len(set(a[0])) == 16
    fit = run.observed_fit(sp, *a)
    assert fit.M == 16 and np.isfinite(fit.alpha).all()
