"""C-ABI library on the CPU (not gpu): it loads, exports every symbol include/autoscout.h declares,
and its HOST paths (space compile, CVI decode, simulator + FP64 resource check, Feistel, GP
fit, pool merge) agree with the oracle.  No compute kernel is launched here.
"""

import json
import os
import random
import re

import numpy as np
import pytest

from conftest import ROOT, space_path, space_text
from oracle import feistel, run, sim, space as S
import synthgen

A = pytest.importorskip("paper_2603_11603_b200.autoscout")

PRESETS = ("P0", "C1", "C2", "C3", "C4", "C5")


def test_exports_every_declared_symbol():
    with open(os.path.join(ROOT, "include", "autoscout.h")) as fh:
        hdr = fh.read()
    declared = set(re.findall(r"\b(autoscout_[a-z_0-9]+)\s*\(", hdr))
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(A.lib(), name), name
    assert declared == set(A.EXPORTS)


@pytest.fixture(scope="module")
def host_spaces():
    return {n: A.Space(space_path(n), -1) for n in PRESETS}


@pytest.mark.parametrize("name", PRESETS)
def test_counts_match_oracle(host_spaces, oracle_spaces, name):
    inf = host_spaces[name].info
    o = oracle_spaces[name]
    assert inf["n_raw"] == o.n_raw and inf["n_cvi"] == o.n_cvi() and inf["n_features"] == len(o.features)


@pytest.mark.parametrize("name", ["C1", "C3"])
def test_cvi_full_small(host_spaces, oracle_spaces, name):
    sp, o = host_spaces[name], oracle_spaces[name]
    raws = [o.encode_raw(d) for d in o.enumerate_cvi()]
    assert [sp.cvi_to_raw(p) for p in range(o.n_cvi())] == raws


@pytest.mark.parametrize("name", PRESETS)
def test_decode_simulate_match_oracle(host_spaces, oracle_spaces, name):
    sp, o = host_spaces[name], oracle_spaces[name]
    rng = random.Random(5)
    n = o.n_cvi()
    ps = [rng.randrange(n) for _ in range(300)] + [0, n - 1]
    digs = [o.cvi_unrank(p) for p in ps]
    cost, ok, mem = sim.simulate(o, digs)
    for p, dg, c, k, m in zip(ps, digs, cost, ok, mem):
        raw = o.encode_raw(dg)
        assert sp.cvi_to_raw(p) == raw
        gd, gv = sp.decode(raw)
        assert gd == dg and gv == bool(k)
        gc, gm, gok = sp.simulate(raw)
        assert gok == bool(k)
        assert gm == m                                   # bit-exact FP64 resource quantity (R7)
        assert gc == pytest.approx(c, rel=1e-13)


@pytest.mark.parametrize("name", ["P0", "C2", "C4"])
def test_decode_random_raw_validity(host_spaces, oracle_spaces, name):
    """Random raw indices (mostly non-canonical / invalid): validity bit = oracle G1-G4."""
    sp, o = host_spaces[name], oracle_spaces[name]
    rng = random.Random(9)
    for _ in range(400):
        raw = rng.randrange(o.n_raw)
        dg = o.decode_raw(raw)
        valid = o.structurally_valid(dg) and bool(sim.simulate(o, [dg])[1][0])
        gd, gv = sp.decode(raw)
        assert gd == dg and gv == valid


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_sample_to_cvi_is_oracle_feistel(host_spaces, oracle_spaces, name):
    sp, o = host_spaces[name], oracle_spaces[name]
    pi = feistel.Feistel(o.n_cvi(), 1234)
    for j in list(range(50)) + [o.n_cvi() - 1]:
        assert sp.sample_to_cvi(1234, j) == pi(j)


@pytest.mark.parametrize("name,M", [("C1", 16), ("C2", 64), ("C4", 40)])
def test_host_gp_fit_matches_oracle(oracle_spaces, name, M):
    o = oracle_spaces[name]
    sp = A.Space(space_path(name), -1)
    raws, costs = observed(o, M)
    fit = run.observed_fit(o, raws, costs)
    sp.observe(raws, costs)
    m, b, fstar = sp.observe_info()
    assert m == M
    assert b == pytest.approx(fit.b, rel=1e-13, abs=1e-15)
    assert fstar == pytest.approx(fit.fstar, rel=1e-15)


def test_async_observe_flag_on_host_only_handle(oracle_spaces):
    """set_async_observe on a host-only handle: accepted, observe() stays synchronous (the
    asynchronous fit exists for the device path), and the fit equals the oracle's."""
    o = oracle_spaces["C2"]
    sp = A.Space(space_path("C2"), -1)
    sp.set_async_observe(True)
    raws, costs = observed(o, 130)
    fit = run.observed_fit(o, raws, costs)
    sp.observe(raws, costs)
    m, b, fstar = sp.observe_info()
    assert m == 130
    assert b == pytest.approx(fit.b, rel=1e-13, abs=1e-15)
    sp.set_async_observe(False)
    sp.observe_clear()
    assert sp.observe_info()[0] == 0


def observed(o, M, seed=0):
    def unrank(p):
        dg = o.cvi_unrank(p)
        return o.encode_raw(dg), dg

    def valid(raw):
        return bool(sim.simulate(o, [o.decode_raw(raw)])[1][0])

    def cost(raw):
        return float(sim.simulate(o, [o.decode_raw(raw)])[0][0])

    return synthgen.observed_set(M, seed, o.n_cvi(), [f.n for f in o.features], unrank, valid, cost)


def test_observe_rejects_invalid(host_spaces, oracle_spaces):
    sp = A.Space(space_path("P0"), -1)
    o = oracle_spaces["P0"]
    bad = o.encode_raw(o.decode_raw(1))   # tp=1 ... ddp_bucket=2 with dp=1 -> non-canonical
    assert not o.structurally_valid(o.decode_raw(1))
    with pytest.raises(A.AutoscoutError) as e:
        sp.observe([bad], [1.0])
    assert e.value.status == "AS_ERR_INVALID_CONFIG"
    with pytest.raises(A.AutoscoutError) as e:
        sp.observe([0], [-1.0])
    assert e.value.status == "AS_ERR_INVALID_ARG"
    with pytest.raises(A.AutoscoutError) as e:
        sp.observe([o.n_raw], [1.0])
    assert e.value.status == "AS_ERR_INDEX_RANGE"


@pytest.mark.parametrize("mutate,status", [
    (lambda d: d.update(features=[]), "AS_ERR_SPACE_SCHEMA"),
    (lambda d: d["features"][0].update(domain=[]), "AS_ERR_SPACE_EMPTY"),
    (lambda d: d["features"][0].update(default=3), "AS_ERR_SPACE_SCHEMA"),
    (lambda d: d["features"][5]["requires"][0].update(feature="nope"), "AS_ERR_SPACE_SCHEMA"),
    (lambda d: d["features"][1].update(requires=[{"feature": "sp", "op": "==", "value": True}]), "AS_ERR_SPACE_CYCLE"),
    (lambda d: d["constraints"].append({"type": "product_eq_devices", "features": ["pp"]}) or
     d["constraints"].append({"type": "divides_const", "features": ["pp"], "const": "F_work"}) or
     d["model"].update(F_work=3), "AS_ERR_SPACE_EMPTY"),
    (lambda d: d["gp"].update(onehot_max_width=-1), "AS_ERR_SPACE_SCHEMA"),
    (lambda d: d["gp"].update(onehot_max_width=2.5), "AS_ERR_SPACE_SCHEMA"),
    (lambda d: d["gp"].update(kernel="cubic"), "AS_ERR_SPACE_SCHEMA"),
])
def test_space_errors(mutate, status):
    doc = json.loads(space_text("P0"))
    mutate(doc)
    with pytest.raises(A.AutoscoutError) as e:
        A.Space(doc, -1)
    assert e.value.status == status


def test_host_only_cannot_score(host_spaces):
    with pytest.raises(A.AutoscoutError) as e:
        host_spaces["C1"].score_batch(acq="sim", k=4)
    assert e.value.status == "AS_ERR_STATE"


def test_topk_merge_host():
    rng = np.random.default_rng(0)
    pools = np.zeros((3, 8), dtype=A.ENTRY_DTYPE)
    for p in range(3):
        sc = np.sort(rng.normal(size=8))[::-1]
        pools[p]["score"] = sc
        pools[p]["raw"] = rng.choice(10_000, 8, replace=False) + 10_000 * p
    pools[1]["score"][2] = pools[0]["score"][1]          # a tie across pools -> raw breaks it
    for p in range(3):                                   # keep each pool ordered (score desc, raw asc)
        order = sorted(range(8), key=lambda i: (-pools[p]["score"][i], pools[p]["raw"][i]))
        pools[p] = pools[p][order]
    allv = [(int(r), float(s)) for r, s in zip(pools["raw"].ravel(), pools["score"].ravel())]
    ref = sorted(allv, key=lambda t: (-t[1], t[0]))[:5]
    nocut = np.concatenate([A.no_cut()] * 3)
    got, cert = A.topk_merge(pools, [8, 8, 8], nocut, 5)
    assert got == ref and cert
    # a cut entry ranking before the 5th -> not certified
    cuts = nocut.copy()
    cuts[1]["score"] = ref[4][1] + 1.0
    cuts[1]["raw"] = 5
    got, cert = A.topk_merge(pools, [8, 8, 8], cuts, 5)
    assert not cert
    # a cut tied with the 5th score but with a larger raw index ranks after it -> certified
    cuts[1]["score"] = ref[4][1]
    cuts[1]["raw"] = ref[4][0] + 1
    got, cert = A.topk_merge(pools, [8, 8, 8], cuts, 5)
    assert cert and got == ref
