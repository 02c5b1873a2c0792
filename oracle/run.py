"""Oracle: score a batch of candidates and keep the exact top-k.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Batch semantics (SURVEY §8(a) a0, §8(b) as_score_args; reading R3):
  RANGE : candidate j of the batch is CVI position  begin + j
  SAMPLE: candidate j is CVI position  pi_seed(begin + j)   (oracle/feistel.py)
Order (reading R11): score descending, raw index ascending ("lowest index wins";
S:506 "ties -> first in enumeration order").  Masked candidates score -inf and never enter
the top-k; k > #valid returns every valid candidate.
"""

from __future__ import annotations

import numpy as np

from . import acq as _acq
from . import ensemble as _ens
from . import gp as _gp
from . import sim as _sim
from .feistel import Feistel


def positions(space, mode, begin, count, seed=0, plist=None):
    n = space.n_cvi()
    if mode == "list":
        # LIST (NEXT-2 batches): candidate j is plist[begin + j]; entries outside [0, n) stay as
        # given and are scored as masked by score_batch
        return [int(x) for x in plist[begin:begin + count]]
    if begin < 0 or count < 0 or begin + count > n:
        raise IndexError("batch exceeds the CVI range")
    if mode == "range":
        return list(range(begin, begin + count))
    if mode == "sample":
        pi = Feistel(n, seed)
        return [pi(begin + j) for j in range(count)]
    raise ValueError(mode)


def observed_fit(space, raws, costs):
    """Fit the GP to observed (raw, cost) pairs; masked or non-canonical raws are rejected."""
    digits = [space.decode_raw(int(r)) for r in raws]
    for dg in digits:
        if not space.structurally_valid(dg):
            raise ValueError("observed configuration is not valid (G1-G3)")
    if len(digits):
        cs, ok, _ = _sim.simulate(space, digits)
        if not np.all(ok):
            raise ValueError("observed configuration violates the resource check (G4)")
    else:
        cs = np.zeros(0)
    ens = None
    if space.gp.get("prior", "sim") == "ensemble" and len(digits):
        # NEXT-1: the regression-simulator ensemble as the prior mean (R20);
        # Unavailable -> the analytical simulator stays the prior
        ens = _ens.Ensemble(space, digits, costs, int(space.gp.get("ensemble_seed", 0)))
        if not ens.available:
            ens = None
    if ens is not None:
        fit = _gp.fit_observed_prior(space, digits, costs, ens.predict(space, digits))
    else:
        fit = _gp.fit_observed(space, digits, costs, cs)
    fit.ens = ens
    return fit


def evaluate(space, digits_list, fit, acq="ei", kappa=2.0, xi=0.0):
    """Per-candidate records for structurally valid configurations."""
    B = len(digits_list)
    rec = {"raw": np.array([space.encode_raw(dg) for dg in digits_list], dtype=np.uint64)}
    if B == 0:
        for k in ("cost", "mem", "mu", "s2", "score", "m0"):
            rec[k] = np.zeros(0)
        rec["valid"] = np.zeros(0, dtype=bool)
        return rec
    cost, ok, mem = _sim.simulate(space, digits_list)
    ens = getattr(fit, "ens", None)
    m0 = ens.predict(space, digits_list) if ens is not None else np.log(cost)
    X = _gp.features(space, digits_list)
    mu, s2, _ = fit.posterior(X, m0)
    if acq == "ei":
        if fit.M == 0:
            raise ValueError("EI needs at least one observation")
        score = _acq.ei_score(mu, s2, fit.fstar, xi)
    elif acq == "lcb":
        score = _acq.lcb_score(mu, s2, kappa)
    elif acq == "sim":
        score = _acq.sim_score(m0)
    else:
        raise ValueError(acq)
    score = np.where(ok, score, -np.inf)
    rec.update(cost=cost, mem=mem, valid=ok, m0=m0, mu=mu, s2=s2, score=score, X=X)
    return rec


def score_batch(space, fit, mode, begin, count, seed=0, acq="ei", kappa=2.0, xi=0.0, plist=None):
    pos = positions(space, mode, begin, count, seed, plist)
    n = space.n_cvi()
    inside = [0 <= p < n for p in pos]
    digits = [space.cvi_unrank(p) if ok else space.cvi_unrank(0) for p, ok in zip(pos, inside)]
    rec = evaluate(space, digits, fit, acq, kappa, xi)
    if not all(inside):
        out = ~np.array(inside, dtype=bool)
        rec["valid"] = rec["valid"] & ~out
        rec["score"] = np.where(out, -np.inf, rec["score"])
        rec["raw"] = np.where(out, np.uint64(np.iinfo(np.uint64).max), rec["raw"]).astype(np.uint64)
    rec["cvi"] = np.array(pos, dtype=np.int64)
    rec["digits"] = digits
    return rec


def topk(rec, k):
    """Exact top-k of valid records: (score desc, raw asc) -> list[(raw, score)]."""
    idx = [i for i in range(len(rec["score"])) if rec["valid"][i] and np.isfinite(rec["score"][i])]
    idx.sort(key=lambda i: (-rec["score"][i], int(rec["raw"][i])))
    return [(int(rec["raw"][i]), float(rec["score"][i])) for i in idx[:k]]
