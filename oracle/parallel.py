"""Oracle over all host cores: a full-size batch cut into contiguous shares, each share evaluated
by oracle/batch.py in a spawned worker process, the per-share results merged.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Used by the full-size parity tests and by
bench.py's cpu_baseline / --impl reference legs.  Merging is exact: valid counts add, and the
top-k of a union is the top-k of the shares' top-k lists under the same total order (score
descending, raw index ascending; reading R11).

Nothing here changes the arithmetic of the oracle: every candidate is decoded, checked,
simulated and scored by the batch forms of the scalar definitions (pinned against them in
tests/test_oracle_batch.py), in FP64.
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

from . import acq as _acq
from . import batch as _batch

_CTX = {}      # per-process context (set by _init in every spawned worker)
CHUNK = 1 << 15


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:           # pragma: no cover
        return os.cpu_count() or 1


def _one_thread_blas():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:                # pragma: no cover
        pass


def _positions(space, mode, begin, count, seed):
    ordinals = np.arange(begin, begin + count, dtype=np.int64)
    if mode == "range":
        return ordinals
    if mode == "sample":
        return _batch.feistel_batch(space.n_cvi(), seed, ordinals)
    raise ValueError(mode)


def score_positions(space, unranker, fit, pos, acq="ei", kappa=2.0, xi=0.0):
    """Per-candidate FP64 records for CVI positions `pos` (oracle/run.py's score_batch, batch form)."""
    dg, act, raw = unranker.unrank(pos)
    cost, ok, mem = _batch.simulate(space, dg, act)
    if space.gp.get("prior", "sim") != "sim":
        raise NotImplementedError("the batch oracle covers the analytical-simulator prior")
    with np.errstate(divide="ignore"):
        m0 = np.log(cost)
    score = np.full(len(pos), -np.inf)
    mu = np.full(len(pos), np.nan)
    s2 = np.full(len(pos), np.nan)
    v = np.nonzero(ok)[0]
    if len(v):
        if acq == "sim":
            score[v] = _acq.sim_score(m0[v])
        else:
            X = _batch.features(space, dg[v], act[v])
            mu[v], s2[v] = _batch.posterior(fit, X, m0[v])
            if acq == "ei":
                score[v] = _acq.ei_score(mu[v], s2[v], fit.fstar, xi)
            elif acq == "lcb":
                score[v] = _acq.lcb_score(mu[v], s2[v], kappa)
            else:
                raise ValueError(acq)
    return dict(raw=raw, valid=ok, m0=m0, mu=mu, s2=s2, score=score, digits=dg, active=act, cost=cost, mem=mem)


def _topk_of(raw, score, k):
    fin = np.isfinite(score)
    r, s = raw[fin], score[fin]
    order = np.lexsort((r, -s))[:k]
    return [(int(r[i]), float(s[i])) for i in order]


def _merge(lists, k):
    allr = [x for l in lists for x in l]
    allr.sort(key=lambda t: (-t[1], t[0]))
    return allr[:k]


def _work_score(args):
    lo, hi = args
    c = _CTX
    sp, U = c["space"], c["unranker"]
    top, nval = [], 0
    for b in range(lo, hi, CHUNK):
        n = min(CHUNK, hi - b)
        pos = _positions(sp, c["mode"], c["begin"] + b, n, c["seed"])
        rec = score_positions(sp, U, c["fit"], pos, c["acq"], c["kappa"], c["xi"])
        nval += int(rec["valid"].sum())
        top = _merge([top, _topk_of(rec["raw"], rec["score"], c["k"])], c["k"])
        if c.get("probe") is not None:
            c["probe"](b, rec)
    return top, nval


def _work_valid(args):
    lo, hi = args
    sp, U = _CTX["space"], _CTX["unranker"]
    nval = 0
    for b in range(lo, hi, CHUNK * 4):
        pos = np.arange(b, min(hi, b + CHUNK * 4), dtype=np.int64)
        dg, act, _ = U.unrank(pos)
        nval += int(_batch.simulate(sp, dg, act)[1].sum())
    return nval


def _shares(count, parts):
    parts = max(1, min(parts, count // CHUNK + 1))
    edges = [count * i // parts for i in range(parts + 1)]
    return [(edges[i], edges[i + 1]) for i in range(parts) if edges[i + 1] > edges[i]]


def _init(ctx, worker=True):
    """Worker start-up (spawned, not forked: the caller may hold a CUDA context and a threaded
    BLAS, and a fork of such a process deadlocked the parent's next multithreaded LAPACK call)."""
    if worker:
        _one_thread_blas()
    _CTX.clear()
    _CTX.update(ctx)
    _CTX["unranker"] = _batch.Unranker(ctx["space"])


class Pool:
    """A persistent set of `procs` spawned oracle workers for one space and fit."""

    def __init__(self, space, fit=None, procs=None):
        self.procs = procs or cores()
        self.ctx = dict(space=space, fit=fit)
        self.pool = None
        if self.procs > 1:
            self.pool = mp.get_context("spawn").Pool(self.procs, initializer=_init, initargs=(self.ctx,))
        else:
            _init(self.ctx, worker=False)

    def _map(self, fn, shares, extra):
        if self.pool is None:
            _CTX.update(extra)
            return [fn(x) for x in shares]
        return self.pool.map(fn, [(extra, x) for x in shares], chunksize=1)

    def topk(self, mode, begin, count, k, seed=0, acq="ei", kappa=2.0, xi=0.0):
        extra = dict(mode=mode, begin=begin, seed=seed, acq=acq, kappa=kappa, xi=xi, k=k)
        fn = _work_score if self.pool is None else _work_score_x
        res = self._map(fn, _shares(count, self.procs * 4), extra)
        return _merge([r[0] for r in res], k), sum(r[1] for r in res)

    def count_valid(self, begin, end):
        fn = _work_valid if self.pool is None else _work_valid_x
        return sum(self._map(fn, [(begin + a, begin + b) for a, b in _shares(end - begin, self.procs * 4)], {}))

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()
            self.pool = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def _work_score_x(arg):
    extra, share = arg
    _CTX.update(extra)
    return _work_score(share)


def _work_valid_x(arg):
    _, share = arg
    return _work_valid(share)


def topk(space, fit, mode, begin, count, k, seed=0, acq="ei", kappa=2.0, xi=0.0, procs=None):
    """Exact top-k (raw, score) and the valid count of a batch, over `procs` host processes."""
    with Pool(space, fit, procs) as P:
        return P.topk(mode, begin, count, k, seed, acq, kappa, xi)


def count_valid(space, begin=0, end=None, procs=None):
    """Number of CVI positions in [begin, end) that pass the resource check (G4)."""
    end = space.n_cvi() if end is None else end
    with Pool(space, None, procs) as P:
        return P.count_valid(begin, end)
