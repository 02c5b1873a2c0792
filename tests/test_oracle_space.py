"""Pins for oracle/space.py: decode, activity, G1/G2/G3 validity, CVI order (not gpu).

Pinned against: SPEC examples, Table 1 gates
(P:507), the north_star invariants (TP*PP*DP*CP = GPU count, layer/head divisibility),
SURVEY Appendix C counts (independent enumerator) and an exhaustive brute-force enumeration
over the full raw range (tests/brute.py) for P0, C1, C2, C3.
"""

import json
import random

import numpy as np
import pytest

from conftest import cfg_digits, golden, space_path, space_text
from oracle import space as S
from brute import enumerate_valid_raw

PRESETS = ("P0", "C1", "C2", "C3", "C4", "C5")


def tiny(features, constraints=(), hardware=None):
    return {"hardware": hardware or {"devices": [{"class": "x", "count": 8, "mem_gb": 80, "rel_throughput": 1.0}]},
            "features": features, "constraints": list(constraints), "model": {}}


def test_enumerate_two_free_bools():
    # S:96 "two independent boolean sparse features, no dense -> 4 configurations"
    sp = S.load_space(tiny([{"name": "a", "kind": "sparse", "domain": [False, True], "default": False},
                            {"name": "b", "kind": "sparse", "domain": [False, True], "default": False}]))
    assert sp.n_cvi() == 4
    assert [sp.encode_raw(d) for d in sp.enumerate_cvi()] == [0, 1, 2, 3]


def test_enumerate_gated_sp():
    # S:97 "tp in {1,2} and sp gated on tp>1 -> 3 configurations (tp=1/sp=Inactive; tp=2/sp in {T,F})"
    sp = S.load_space(tiny([{"name": "tp", "kind": "sparse", "domain": [1, 2], "default": 1},
                            {"name": "sp", "kind": "sparse", "domain": [False, True], "default": False,
                             "requires": [{"feature": "tp", "op": ">", "value": 1}]}]))
    assert sp.n_cvi() == 3
    assert [sp.encode_raw(d) for d in sp.enumerate_cvi()] == [0, 2, 3]
    # raw 1 = (tp=1, sp=T): sp inactive but not at its default -> non-canonical duplicate
    assert not sp.structurally_valid(sp.decode_raw(1))
    assert sp.activity(sp.decode_raw(1)) == [True, False]


@pytest.mark.parametrize("cfg,inactive", [
    ({"dp": 1, "tp": 2}, {"ddp", "ddp_bucket"}),          # S:69 "dp=1 -> ddp and ddp_bucket inactive"
    ({"tp": 1, "dp": 2}, {"tp_comm", "sp"}),              # S:70 "tp=1 -> tp_comm inactive"; P:507 sp requires tp>1
    ({"tp": 2, "dp": 2}, set()),                          # S:71 "tp=2, dp=2 -> all three dense features active"
])
def test_mask_examples(oracle_spaces, cfg, inactive):
    sp = oracle_spaces["P0"]
    dg = cfg_digits(sp, cfg)
    act = sp.activity(dg)
    got = {f.name for f, a in zip(sp.features, act) if not a}
    assert got == inactive


def test_is_feasible_examples(oracle_spaces):
    sp = oracle_spaces["P0"]
    # S:87 sp=True with tp=1 -> false
    assert not sp.structurally_valid(cfg_digits(sp, {"sp": True, "tp": 1}))
    # S:88 minimal configuration -> true
    assert sp.structurally_valid(cfg_digits(sp, {}))
    # S:89 pp=8, tp=8, dp=8 on 12 devices -> false
    assert not sp.structurally_valid(cfg_digits(sp, {"pp": 8, "tp": 8, "dp": 8}))


@pytest.mark.parametrize("mutate,kind", [
    (lambda d: d.update(features=[]), "schema"),
    (lambda d: d["features"][0].update(domain=[]), "empty_domain"),
    (lambda d: d["features"][5]["requires"][0].update(feature="nope"), "unknown_ref"),
    (lambda d: d["features"][0].update(default=3), "schema"),                      # S:30 default in domain
])
def test_load_errors(mutate, kind):
    doc = json.loads(space_text("P0"))
    mutate(doc)
    with pytest.raises(S.SpaceError) as e:
        S.load_space(doc)
    assert e.value.kind == kind


def test_load_cycle():
    # S:62 "f1.activation references f2, f2.activation references f1 -> cyclic-dependency error"
    doc = tiny([{"name": "f1", "kind": "sparse", "domain": [0, 1], "requires": [{"feature": "f2", "op": ">", "value": 0}]},
                {"name": "f2", "kind": "sparse", "domain": [0, 1], "requires": [{"feature": "f1", "op": ">", "value": 0}]}])
    with pytest.raises(S.SpaceError) as e:
        S.load_space(doc)
    assert e.value.kind == "cycle"


@pytest.mark.parametrize("name", PRESETS)
def test_counts_vs_survey(oracle_spaces, name):
    g = golden("counts.json")[name]
    sp = oracle_spaces[name]
    assert sp.n_raw == g["n_raw"]
    assert sp.n_cvi() == g["n_cvi"]


def test_p0_s33_world_rule():
    # S:33 reading (world divides the 12 devices) -> survey count 12,144; "order of magnitude 10^4"
    doc = json.loads(space_text("P0"))
    doc["constraints"][0]["divides_devices"] = True
    sp = S.load_space(doc)
    assert sp.n_cvi() == golden("counts.json")["P0_S33"]["n_cvi"]
    assert 1e3 < sp.n_cvi() < 1e5


@pytest.mark.parametrize("name", ["P0", "C1", "C2", "C3"])
def test_cvi_equals_bruteforce(oracle_spaces, name):
    with open(space_path(name)) as fh:
        doc = json.load(fh)
    sp = oracle_spaces[name]
    ref = enumerate_valid_raw(doc, sp.G)
    got = np.array([sp.encode_raw(d) for d in sp.enumerate_cvi()], dtype=np.int64)
    assert len(got) == len(ref)
    assert np.array_equal(got, ref)                       # same set AND ascending raw order


@pytest.mark.parametrize("name", PRESETS)
def test_unrank_rank_roundtrip(oracle_spaces, name):
    sp = oracle_spaces[name]
    rng = random.Random(7)
    n = sp.n_cvi()
    ps = sorted({0, n - 1} | {rng.randrange(n) for _ in range(60)})
    raws = []
    for p in ps:
        dg = sp.cvi_unrank(p)
        assert sp.structurally_valid(dg)
        assert sp.cvi_rank(dg) == p
        raws.append(sp.encode_raw(dg))
    assert raws == sorted(raws) and len(set(raws)) == len(raws)     # CVI order = raw order


@pytest.mark.parametrize("name", ["C1", "C2", "C4", "C5"])
def test_north_star_invariants(oracle_spaces, name):
    """TP*PP*DP*CP = GPU count; layer/head divisibility; Table 1 gates."""
    sp = oracle_spaces[name]
    rng = random.Random(3)
    n = sp.n_cvi()
    ps = range(n) if n < 5000 else [rng.randrange(n) for _ in range(1500)]
    M = sp.model
    for p in ps:
        dg = sp.cvi_unrank(p)
        act = sp.activity(dg)
        v = lambda k: sp.effective_value(sp.index[k], dg, act) if k in sp.index else 1
        assert v("pp") * v("tp") * v("dp") * v("cp") == sp.G
        assert M["L"] % (v("pp") * v("vpp")) == 0
        assert M["a"] % v("tp") == 0 and M["kv"] % v("tp") == 0
        assert M["GBS"] % (v("dp") * v("mbs")) == 0
        if "sp" in sp.index and v("tp") == 1:
            assert not act[sp.index["sp"]] and v("sp") is False       # P:507 sp requires tp>1
        for k in ("ovg", "ddp_bucket", "ddp", "dopt"):
            if k in sp.index and v("dp") == 1:
                assert not act[sp.index[k]]                           # P:510 gated on dp>1
        if "ep" in sp.index:
            assert v("dp") % v("ep") == 0 and M["E"] % v("ep") == 0
