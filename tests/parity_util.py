"""Shared helpers of the GPU parity tests: the same seeded inputs for the oracle and the CUDA path,
and the SURVEY A.7 tolerances."""

import math

import numpy as np

import synthgen
from conftest import space_path
from oracle import acq as oacq, run, sim, space as S

_ORACLE = {}


def oracle_space(name):
    if name not in _ORACLE:
        _ORACLE[name] = S.load_space(space_path(name))
    return _ORACLE[name]


def observed(o, M, seed=0):
    """The seeded observed set, generated with the ORACLE's decode/validity/simulator."""
    if M == 0:
        return [], []

    def unrank(p):
        dg = o.cvi_unrank(p)
        return o.encode_raw(dg), dg

    def valid(raw):
        return bool(sim.simulate(o, [o.decode_raw(raw)])[1][0])

    def cost(raw):
        return float(sim.simulate(o, [o.decode_raw(raw)])[0][0])

    return synthgen.observed_set(M, seed, o.n_cvi(), [f.n for f in o.features], unrank, valid, cost)


def oracle_records(o, fit, mode, begin, count, seed=0):
    """Per-candidate oracle records (prior m0, mu, s2, validity, raw) for a batch."""
    return run.score_batch(o, fit, mode, begin, count, seed, acq="lcb", kappa=0.0)


def oracle_scores(o, fit, rec, acq, kappa=2.0, xi=0.0):
    if acq == "ei":
        s = oacq.ei_score(rec["mu"], rec["s2"], fit.fstar, xi)
    elif acq == "lcb":
        s = oacq.lcb_score(rec["mu"], rec["s2"], kappa)
    else:
        s = oacq.sim_score(rec["m0"])
    return np.where(rec["valid"], s, -np.inf)


def oracle_topk(rec, scores, k):
    r = dict(rec)
    r["score"] = scores
    return run.topk(r, k)


def ei_tolerance_ok(gpu, ref, mu, s2, fstar, sf2, xi=0.0):
    """A.7: |d log EI| <= 1e-5 where z >= -3 and s2 >= 1e-3 sf2; elsewhere |d EI| <= 1e-5 sigma_f."""
    sig = np.sqrt(s2)
    with np.errstate(divide="ignore", invalid="ignore"):
        z = np.where(sig > 0, (fstar - mu - xi) / np.where(sig > 0, sig, 1), -np.inf)
    strict = (z >= -3) & (s2 >= 1e-3 * sf2)
    d_log = np.abs(gpu - ref)
    d_ei = np.abs(np.exp(gpu.astype(np.float64)) - np.exp(ref))
    ok = np.where(strict, d_log <= 1e-5, d_ei <= 1e-5 * math.sqrt(sf2))
    both_inf = np.isneginf(gpu) & np.isneginf(ref)
    return ok | both_inf
