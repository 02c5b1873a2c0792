"""Pins for oracle/sim.py (not gpu).

Pinned against: hand-evaluated SPEC formula values and SURVEY Appendix C.2 transcription
values (tests/golden/sim_values.json); SPEC examples S:500-502 and properties S:541-542;
the brute-force G4 counts of SURVEY Appendix C (tests/golden/counts.json); monotonicity of the
serving KV capacity in gpu_memory_utilization.
"""

import json

import numpy as np
import pytest

from conftest import cfg_digits, golden, space_text
from oracle import sim, space as S


@pytest.mark.parametrize("case", golden("sim_values.json")["cases"], ids=lambda c: c["space"] + str(sorted(c["cfg"].items()))[:40])
def test_golden_values(oracle_spaces, case):
    sp = oracle_spaces[case["space"]]
    dg = cfg_digits(sp, case["cfg"])
    assert sp.structurally_valid(dg)
    cost, ok, mem, terms = sim.simulate(sp, [dg], terms=True)
    assert ok[0]
    rel = 1e-12 if case["space"] == "P0" else 5e-9          # survey values printed to 9-10 significant digits
    assert cost[0] == pytest.approx(case["cost"], rel=rel)
    if "mem_gb" in case:
        assert mem[0] / 1e9 == pytest.approx(case["mem_gb"], rel=6e-6)   # printed to 6 significant digits
    if "TPOT" in case:
        assert terms["TPOT"][0] == pytest.approx(case["TPOT"], rel=5e-8)   # printed to 8 significant digits
    if "b" in case:
        assert terms["b"][0] == case["b"]
    if "kv_tok" in case:
        assert terms["kv_tok"][0] == case["kv_tok"]
    if "thr" in case:
        assert terms["thr"][0] == pytest.approx(case["thr"], rel=5e-6)


def _all_valid(sp):
    return list(sp.enumerate_cvi())


@pytest.mark.parametrize("name", ["P0", "C1", "C2", "C3"])
def test_valid_counts(oracle_spaces, name):
    sp = oracle_spaces[name]
    _, ok, _ = sim.simulate(sp, _all_valid(sp))
    assert int(ok.sum()) == golden("counts.json")[name]["n_valid"]


def test_spec_doubling_dp_halves_tcomp(oracle_spaces):
    # S:500 "doubling dp with all else fixed halves the world-divided t_comp term"
    sp = oracle_spaces["P0"]
    a = cfg_digits(sp, {"dp": 2, "mbs": 2})
    b = cfg_digits(sp, {"dp": 4, "mbs": 2})
    ta = sim.simulate(sp, [a], terms=True)[3]["t_comp"][0]
    tb = sim.simulate(sp, [b], terms=True)[3]["t_comp"][0]
    assert tb == pytest.approx(ta / 2, rel=1e-15)


def test_spec_ar_factors(oracle_spaces):
    # S:501 "ar: True multiplies t_comp by r_ar=1.33 and multiplies activation memory by 0.3"
    sp = oracle_spaces["P0"]
    f = sim.simulate(sp, [cfg_digits(sp, {"tp": 2, "mbs": 4, "ar": False})], terms=True)[3]
    t = sim.simulate(sp, [cfg_digits(sp, {"tp": 2, "mbs": 4, "ar": True})], terms=True)[3]
    assert t["t_comp"][0] == pytest.approx(1.33 * f["t_comp"][0], rel=1e-15)
    assert t["act_mem"][0] == pytest.approx(0.3 * f["act_mem"][0], rel=1e-15)


def test_spec_unsharded_params_infeasible():
    # S:502 "pp=tp=1 with P_mem exceeding one device's memory -> Infeasible"
    doc = json.loads(space_text("P0"))
    doc["model"]["P_mem"] = 90e9
    sp = S.load_space(doc)
    digs = [d for d in sp.enumerate_cvi()
            if sp.features[0].values[d[0]] == 1 and sp.features[1].values[d[1]] == 1]
    _, ok, _ = sim.simulate(sp, digs)
    assert len(digs) > 0 and not ok.any()


def test_spec_monotone_properties(oracle_spaces):
    # increasing tp_comm never increases t_tp; bucket_pen minimal at 4; sp never increases cost (tp>1)
    sp = oracle_spaces["P0"]
    digs = _all_valid(sp)
    cost, _, _, T = sim.simulate(sp, digs, terms=True)
    key = {}
    for i, d in enumerate(digs):
        key[tuple(d)] = i
    jt, js, jb = sp.index["tp_comm"], sp.index["sp"], sp.index["ddp_bucket"]
    for i, d in enumerate(digs):
        if d[jt] + 1 < sp.features[jt].n and sp.activity(d)[jt]:
            e = list(d); e[jt] += 1
            assert T["t_tp"][key[tuple(e)]] <= T["t_tp"][i]
        if d[js] == 0 and sp.activity(d)[js]:
            e = list(d); e[js] = 1
            assert cost[key[tuple(e)]] <= cost[i]
        if sp.activity(d)[jb]:
            e = list(d); e[jb] = sp.features[jb].values.index(4)
            assert T["bucket_pen"][key[tuple(e)]] <= T["bucket_pen"][i]


def test_pure(oracle_spaces):
    # S:541 "synthetic_cost is pure: repeated evaluations of one configuration are bit-identical"
    sp = oracle_spaces["C4"]
    dg = sp.cvi_unrank(12345)
    c1 = sim.simulate(sp, [dg] * 50)
    assert len(set(c1[0].tolist())) == 1 and len(set(c1[2].tolist())) == 1


def test_serve_kv_capacity_monotone_in_u(oracle_spaces):
    sp = oracle_spaces["C3"]
    ju = sp.index["u"]
    digs = _all_valid(sp)
    _, _, usable = sim.simulate(sp, digs)
    idx = {tuple(d): i for i, d in enumerate(digs)}
    for i, d in enumerate(digs):
        if d[ju] + 1 < sp.features[ju].n:
            e = list(d); e[ju] += 1
            assert usable[idx[tuple(e)]] >= usable[i]
