"""NEXT-3: Algorithm 1 over the library, host side (not gpu).

Pinned by the worked examples SPEC.md derives from the paper's formulas (acceptance 2-5,
S:615-626) -- Eq. 1, the difference-of-differences estimator,
the tournament's zigzag halving, MAPE and the one-way fidelity switch with
weak priors -- plus end-to-end runs on host-only handles (decode, activity,
subtree ranges and the simulator through the C ABI) against a brute-force optimum of the
synthetic truth.
"""

import math

import numpy as np
import pytest

import synthgen
from conftest import space_path
from paper_2603_11603_b200 import search as SE
from paper_2603_11603_b200.autoscout import Space


def test_ucb1_eq1_worked_example():
    # Q_S=3, N_S=2, Q_D=1, N_D=2, N_total=4, C(t)=1: 1.5 + 0.8326 vs 0.5 + 0.8326 -> Sparse
    assert SE.select_arm([3.0, 1.0], [2, 2], t=0, C0=1.0, gamma=1.0) == SE.SPARSE
    assert math.sqrt(math.log(4) / 2) == pytest.approx(0.8326, abs=1e-4)
    assert SE.select_arm([1.0, 3.0], [2, 2], t=0, C0=1.0, gamma=1.0) == SE.DENSE
    # an unpulled arm first, Sparse before Dense
    assert SE.select_arm([0.0, 5.0], [0, 5], t=3) == SE.SPARSE
    assert SE.select_arm([9.0, 0.0], [3, 0], t=3) == SE.DENSE
    assert SE.select_arm([0.0, 0.0], [0, 0], t=0) == SE.SPARSE
    # C(t) = C0 gamma^t: C0 = 1, gamma = 0.9, t = 10 -> 0.3487
    assert SE.exploration(1.0, 0.9, 10) == pytest.approx(0.3487, abs=1e-4)


def test_ucb1_shifts_to_exploitation():
    # C(t) -> 0: the arm with the higher mean reward wins although it was pulled more
    Q, N = [2.0, 0.9], [10, 2]          # means 0.2 vs 0.45
    assert SE.select_arm(Q, N, t=0, C0=1.414, gamma=0.99) == SE.DENSE
    assert SE.select_arm([6.0, 0.9], [10, 2], t=2000, C0=1.414, gamma=0.99) == SE.SPARSE   # 0.6 vs 0.45


def test_difference_of_differences():
    # (c_bb, c_bc, c_cb, c_cc) = (10, 8, 9, 6) -> D_sparse = 1.5, D_dense = 2.5
    d_s, d_d, r_s, r_d = SE.attribute(10.0, 8.0, 9.0, 6.0)
    assert (d_s, d_d) == (1.5, 2.5)
    assert (r_s, r_d) == pytest.approx((0.15, 0.25))
    assert SE.attribute(7.0, 7.0, 7.0, 7.0)[:2] == (0.0, 0.0)
    assert SE.attribute(5.0, 6.0, 7.0, 8.0)[2:] == (0.0, 0.0)      # candidates worse: clipped
    assert SE.attribute(5.0, 6.0, math.inf, math.inf)[2] == 0.0     # infeasible sparse candidate


def test_tournament_zigzag_halving():
    t = SE.Tournament(8)
    rounds = []
    rng = np.random.default_rng(1)
    while not t.done:
        order = list(t.order())
        rounds.append(order)
        for k in order:
            t.record(k, float(rng.random()))
    assert [len(r) for r in rounds] == [8, 4, 2]                      # 8 -> 4 -> 2 -> 1
    assert rounds[0] == sorted(rounds[0]) and rounds[1] == sorted(rounds[1])[::-1]
    assert rounds[2] == sorted(rounds[2])
    # cumulative rewards {2.0, 1.0, 3.0, 0.5}, 4 survivors -> {T3, T1}
    t4 = SE.Tournament(4)
    for k, r in zip(t4.order(), (2.0, 1.0, 3.0, 0.5)):
        t4.record(k, r)
    assert t4.survivors == [0, 2]
    t2 = SE.Tournament(2)
    for k in t2.order():
        t2.record(k, 1.0)
    assert t2.winner() == 0                                            # tie -> lower index


def test_mape_and_weak_priors():
    # predictions (100, 200) vs real (110, 180) -> mean(10/110, 20/180) = 0.1010
    assert SE.mape([(100.0, 110.0), (200.0, 180.0)]) == pytest.approx(0.1010, abs=1e-4)
    # lambda = 0.25, Q_S = 8, N_S = 4 -> Q_S = 2, N_S = 1, mean kept
    Q, N = SE.weak_prior([8.0, 3.0], [4, 6], 0.25)
    assert (Q[0], N[0]) == (2.0, 1.0)
    assert Q[1] / N[1] == pytest.approx(3.0 / 6)


@pytest.fixture(scope="module")
def p0():
    return Space(space_path("P0"), -1)


def test_dense_coordinate_search(p0):
    sp = SE.SearchSpace(p0)
    # tp = 2, dp = 2: tp_comm, ddp, ddp_bucket active; tp_comm at 12 (digit 0)
    dg = [0] * sp.d
    dg[sp.names.index("tp")] = 1
    dg[sp.names.index("dp")] = 1
    raw = sp.raw_of(sp.project(dg))
    act = sp.active_dense(raw)
    assert [sp.names[f] for f in act] == ["ddp", "tp_comm", "ddp_bucket"]
    st = SE.DenseState(coord=1)                      # tp_comm
    r1 = st.propose(sp, raw)
    assert sp.digits(r1)[sp.names.index("tp_comm")] == 1          # 12 -> 13
    st.update(sp, raw, improved=True)
    assert st.step[sp.names.index("tp_comm")] == 2                # doubling on success
    st.update(sp, raw, improved=False)
    assert st.step[sp.names.index("tp_comm")] == 1 and st.flip_used
    st.update(sp, raw, improved=False)
    assert st.coord == 2 and not st.flip_used                     # flip used -> next coordinate
    # boundary: tp_comm at its maximum with direction +1 -> one step down
    dg2 = sp.digits(raw)
    dg2[sp.names.index("tp_comm")] = sp.nvals[sp.names.index("tp_comm")] - 1
    top = sp.raw_of(dg2)
    st2 = SE.DenseState(coord=1)
    assert sp.digits(st2.propose(sp, top))[sp.names.index("tp_comm")] == sp.nvals[sp.names.index("tp_comm")] - 2


def truth(sp):
    """Synthetic "profiling" (the recipe of synthgen without noise): cost_sim times a smooth bias."""
    d = sp.d
    sizes = [len(f["domain"]) for f in sp.doc["features"]]
    w = [3.0 * synthgen.u_pm1(0xA0 ^ j) for j in range(d)]
    w0 = 3.0 * synthgen.u_pm1(0xB0)

    def real(raw):
        dg, _ = sp.decode(raw)
        c, _, ok = sp.simulate(raw)
        if not ok:
            return math.inf
        s = sum(w[j] * (dg[j] / (sizes[j] - 1) if sizes[j] > 1 else 0.0) for j in range(d))
        return c * math.exp(0.3 * math.sin(s + w0))
    return real


def test_fidelity_switch_rules(p0):
    real = truth(p0)
    # a perfect simulator never switches (acceptance 5a)
    r = SE.run(p0, real, SE.RunConfig(T=60, tau=5, seed=1, gpu_topk=False), sim_cost=real)
    assert r["mode"] == "sim" and not any(e.get("event") == "switch" for e in r["trace"])
    # a simulator 3x off switches at the first checkpoint, MAPE = |3c - c| / c = 2 (acceptance 5b)
    r = SE.run(p0, real, SE.RunConfig(T=30, tau=5, seed=1, gpu_topk=False), sim_cost=lambda x: 3.0 * real(x))
    sw = [e for e in r["trace"] if e.get("event") == "switch"]
    assert len(sw) == 1 and sw[0]["t"] == 5 and sw[0]["mape"] == pytest.approx(2.0)
    assert sw[0]["tree_nodes_after"] == sw[0]["tree_nodes"]            # tree retained (5c)
    assert len(sw[0]["reval"]) == 5                                    # top-K re-evaluation
    assert r["mode"] == "real"


def test_determinism(p0):
    real = truth(p0)
    a = SE.run(p0, real, SE.RunConfig(T=25, seed=7, gpu_topk=False))
    b = SE.run(p0, real, SE.RunConfig(T=25, seed=7, gpu_topk=False))
    assert a["trace"] == b["trace"] and a["best_raw"] == b["best_raw"]


def test_search_quality_C3_and_C1():
    """Budget 20 % of |space| iterations: the loop's median best is within 1 % of the brute-force
    optimum on C3 and C1, and never worse than random search given as many evaluations."""
    for name in ("C3", "C1"):
        sp = Space(space_path(name), -1)
        real = truth(sp)
        allc = np.array([real(sp.cvi_to_raw(p)) for p in range(sp.n_cvi)])
        best = allc.min()
        ours, rnd = [], []
        for seed in range(12):
            r = SE.run(sp, real, SE.RunConfig(T=int(0.2 * sp.n_cvi), seed=seed, gpu_topk=False))
            ours.append(r["best_cost"] / best)
            pick = np.random.default_rng(1000 + seed).choice(len(allc), r["real_evals"] + r["sim_evals"],
                                                             replace=False)
            rnd.append(allc[pick].min() / best)
        assert np.median(ours) <= 1.01, (name, sorted(ours))
        assert np.median(ours) <= np.median(rnd), (name, np.median(ours), np.median(rnd))
