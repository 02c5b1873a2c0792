"""Oracle: analytical iteration-time / serving simulator and the FP64 resource mask (G4).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Sources.  The paper's simulators are R^2-weighted linear regressions (Table 2
P:518-543, ensemble eq. P:545-548); the only analytical time+memory formula in the
reference is SPEC's `synthetic_cost`.  BASELINE.json's north_star asks for "the
low-fidelity analytical iteration-time and memory simulator", so (reading R6):
  * sim_mode "spec"    -- SPEC synthetic_cost verbatim, constants S:547 + R8.
  * sim_mode "derived" -- SURVEY Appendix A.3: the same terms with coefficients derived from
                          model/hardware descriptors + terms for vpp, recompute granularity,
                          tp overlap, distributed optimizer, EP dispatcher, CP.
  * sim_mode "serve"   -- SURVEY Appendix A.4 (vLLM-style decode step + KV capacity).

Everything is evaluated in FP64.  The resource quantities (training memory, serving usable
bytes / KV tokens) use only + - * / in exactly the order written below, with numpy
element-wise ufuncs (no FMA contraction), so that the CUDA path can reproduce them
bit-for-bit (reading R7).  The times need not be bit-exact.
"""

from __future__ import annotations

import numpy as np

TRAIN_KNOBS = ("pp", "vpp", "tp", "dp", "cp", "ep", "mbs", "ar", "arl", "sp", "tpov", "tp_comm",
               "dopt", "ovg", "ovp", "ddp_bucket", "ddp", "disp")
SERVE_KNOBS = ("tp", "max_num_seqs", "cpf", "mbt", "u")

# Values of knobs that a preset does not declare (SURVEY A.3 "Knobs absent from a preset").
NEUTRAL = {"pp": 1, "vpp": 1, "tp": 1, "dp": 1, "cp": 1, "ep": 1, "mbs": 1, "ar": "none", "arl": 1,
           "sp": False, "tpov": False, "tp_comm": 0, "dopt": False, "ovg": False, "ovp": False,
           "ddp_bucket": 4, "ddp": 1, "disp": "alltoall",
           "max_num_seqs": 1, "cpf": False, "mbt": 1, "u": 0.9}


def _ar_code(v):
    """ar: bool {F,T} -> {none, full}; categorical as-is.  0 none, 1 sel, 2 full."""
    if isinstance(v, bool):
        return 2 if v else 0
    return {"none": 0, "sel": 1, "full": 2}[v]


def knob_arrays(space, digits_list):
    """Per-knob arrays of effective values and activity over a batch of configurations."""
    names = TRAIN_KNOBS if space.sim_mode in ("spec", "derived") else SERVE_KNOBS
    B = len(digits_list)
    vals = {k: np.empty(B, dtype=np.float64) for k in names}
    acts = {k: np.zeros(B, dtype=bool) for k in names}
    present = {k: (k in space.index) for k in names}
    for b, dg in enumerate(digits_list):
        act = space.activity(dg)
        for k in names:
            if present[k]:
                j = space.index[k]
                v = space.effective_value(j, dg, act)
                acts[k][b] = act[j]
            else:
                v = NEUTRAL[k]
            if k == "ar":
                v = _ar_code(v)
            elif k == "disp":
                v = 1 if v == "allgather" else 0
            elif isinstance(v, bool):
                v = 1 if v else 0
            vals[k][b] = float(v)
    return vals, acts, present


def device_assignment(space, world):
    """Fill the fastest device class first; eff = min rel. throughput, cap = min memory of the
    classes used (S:490 'fill fastest class first; eff = min relative throughput'; S:496
    'per-device memory'; SURVEY A.3 'per device class: min cap of the classes used')."""
    classes = sorted(space.hardware["devices"], key=lambda c: -float(c["rel_throughput"]))
    eff = np.empty(len(world))
    cap = np.empty(len(world))
    for i, w in enumerate(world):
        rem = w
        e, c = np.inf, np.inf
        for cl in classes:
            if rem <= 0:
                break
            e = min(e, float(cl["rel_throughput"]))
            c = min(c, float(cl["mem_gb"]) * 1e9)
            rem -= int(cl["count"])
        eff[i], cap[i] = e, c
    return eff, cap


def simulate(space, digits_list, terms=False):
    """-> (cost [B] FP64 objective units, resource_ok [B] bool, mem_or_usable [B] FP64)
    [, dict of the named cost terms when terms=True]."""
    vals, acts, present = knob_arrays(space, digits_list)
    return simulate_knobs(space, vals, acts, present, terms)


def simulate_knobs(space, vals, acts, present, terms=False):
    """simulate() on per-knob arrays of effective values / activity (knob_arrays' output, or
    oracle/batch.py's vectorised equivalent for large batches)."""
    if space.sim_mode == "spec":
        out = _spec(space, vals, acts)
    elif space.sim_mode == "derived":
        out = _derived(space, vals, acts, present)
    elif space.sim_mode == "serve":
        out = _serve(space, vals, acts)
    else:
        raise ValueError(space.sim_mode)
    return out if terms else out[:3]


def _spec(space, V, A):
    """SPEC synthetic_cost, verbatim."""
    M = space.model
    pp, tp, dp, ep, cp, mbs = V["pp"], V["tp"], V["dp"], V["ep"], V["cp"], V["mbs"]
    ar = V["ar"] == 2
    sp = V["sp"] == 1
    world = pp * tp * dp * cp
    eff, cap = device_assignment(space, world.astype(np.int64))
    micro_steps = M["B"] / (dp * mbs)
    r = np.where(ar, M["r_ar"], 1.0)
    mbs_scale = 1.0 + 0.1 * np.log2(mbs)
    t_comp = M["F_work"] * r / (world * eff * mbs_scale)
    t_bubble = t_comp * (pp - 1.0) / micro_steps
    overlap = np.where(tp > 1, np.clip((V["tp_comm"] - 12.0) / 16.0, 0.0, 0.5), 0.0)
    t_tp = M["alpha_tp"] * (tp - 1.0) / tp * (1.0 - overlap) * np.where(sp & (tp > 1), 0.8, 1.0)
    bucket_pen = np.where(dp > 1, 1.0 + 0.1 * (np.log2(V["ddp_bucket"]) - 2.0) ** 2, 0.0)
    t_dp = M["alpha_dp"] * (dp - 1.0) / dp * bucket_pen
    t_ep = M["alpha_tp"] * 0.5 * (ep - 1.0) / ep
    cost = t_comp + t_bubble + t_tp + t_dp + t_ep
    # S:496, normative FP64 order (R7): ((P_mem/(pp*tp)) + (((A_mem*mbs)*f)/cp))
    m1 = M["P_mem"] / (pp * tp)
    m2 = M["A_mem"] * mbs
    m3 = m2 * np.where(ar, 0.3, 1.0)
    m4 = m3 / cp
    mem = m1 + m4
    return cost, mem <= cap, mem, dict(t_comp=t_comp, t_bubble=t_bubble, t_tp=t_tp, t_dp=t_dp, t_ep=t_ep,
                                      bucket_pen=bucket_pen, act_mem=m4, param_mem=m1)


def _bw(space, span):
    hw = space.hardware
    return np.where(span <= hw["gpus_per_node"], hw["bw_intra"], hw["bw_inter"])


def _derived(space, V, A, present):
    """SURVEY Appendix A.3 'Derived mode', term by term."""
    M, hw = space.model, space.hardware
    L, h, S, GBS, P = M["L"], M["h"], M["S"], M["GBS"], M["P"]
    a, kv = M.get("a", 1), M.get("kv", 1)
    P_exp, E, topk = M.get("P_exp", 0.0), M.get("E", 1), M.get("topk", 1)
    pp, vpp, tp, dp, cp, ep, mbs = (V[k] for k in ("pp", "vpp", "tp", "dp", "cp", "ep", "mbs"))
    ar = V["ar"]
    sp = V["sp"] == 1
    full = ar == 2
    sel = ar == 1
    world = pp * tp * dp * cp
    m = GBS / (dp * mbs)
    L_st = L / (pp * vpp)
    arl_active = A["arl"] if present["arl"] else np.zeros(len(pp), dtype=bool)
    f_rc = np.where(full, np.where(arl_active, np.minimum(1.0, V["arl"] / L_st), 1.0), 0.0)
    r = 1.0 + 0.33 * f_rc + np.where(sel, 0.03, 0.0)
    P_act = P - P_exp + P_exp * topk / E
    T_work = GBS * S * (6.0 * P_act + 12.0 * L * h * S) / (hw["peak_flops"] * hw["mfu0"])
    tpc_active = (A["tp_comm"] if present["tp_comm"] else np.zeros(len(pp), dtype=bool))
    steal = np.where(tpc_active, 0.5 * V["tp_comm"] / hw["n_sm"], 0.0)
    s_mbs = 1.0 + 0.1 * np.log2(mbs)
    t_comp = T_work * r * (1.0 + steal) / (world * s_mbs)
    t_bubble = t_comp * (pp - 1.0) / (m * vpp)
    ov = np.where((tp > 1) & tpc_active, np.clip((V["tp_comm"] - 12.0) / 16.0, 0.0, 0.5), 0.0)
    t_tp = np.where(tp > 1,
                    16.0 * L * GBS * S * h / (pp * dp * cp * _bw(space, tp)) * (tp - 1.0) / tp
                    * (1.0 - ov) * np.where(sp, 0.8, 1.0), 0.0)
    # P_loc in normative order: ((P - P_exp) + (P_exp/ep)) / (pp*tp)
    P_loc = ((P - P_exp) + (P_exp / ep)) / (pp * tp)
    bucket = V["ddp_bucket"]
    ovg = V["ovg"] == 1
    ovp = V["ovp"] == 1
    t_dp = np.where(dp > 1,
                    4.0 * P_loc / _bw(space, tp * cp * dp) * (dp - 1.0) / dp
                    * (1.0 + 0.1 * (np.log2(bucket) - 2.0) ** 2)
                    * np.where(ovg, 0.5, 1.0) * np.where(ovp, 0.75, 1.0), 0.0)
    t_ep = np.where(ep > 1,
                    8.0 * topk * L * GBS * S * h / (pp * dp * cp * np.where(sp, tp, 1.0) * _bw(space, tp * cp * ep))
                    * (ep - 1.0) / ep * np.where(V["disp"] == 1, 1.5, 1.0), 0.0)
    t_cp = np.where(cp > 1,
                    0.5 * 12.0 * L * GBS * S * kv * (h / a) / (pp * dp * _bw(space, tp * cp)) * (cp - 1.0) / cp, 0.0)
    cost = t_comp + t_bubble + t_tp + t_dp + t_ep + t_cp
    # ---- memory, normative FP64 order (SURVEY A.3 memory block, R7) ----
    dopt = V["dopt"] == 1
    bpp = np.where(dopt, 6.0 + 12.0 / dp, 18.0)
    act = np.where(sp, 34.0 / tp, 10.0 + 24.0 / tp)
    af = (1.0 - 0.7 * f_rc) - np.where(sel, 0.2, 0.0)
    t1 = P_loc * bpp
    t2 = float(L) * (S / cp)
    t2 = t2 * h
    t2 = t2 * mbs
    t2 = t2 * act
    t2 = t2 * af
    mem = t1 + t2
    _, cap = device_assignment(space, world.astype(np.int64))
    return cost, mem <= cap, mem, dict(t_comp=t_comp, t_bubble=t_bubble, t_tp=t_tp, t_dp=t_dp, t_ep=t_ep,
                                      t_cp=t_cp, act_mem=t2, param_mem=t1)


def _serve(space, V, A):
    """SURVEY Appendix A.4 (serving; no counterpart in PAPER/SPEC -- reading R6)."""
    M, hw = space.model, space.hardware
    L, h, kv, dh, ffn, P = M["L"], M["h"], M["kv"], M["dh"], M["ffn"], M["P"]
    P_in, P_out, mml = M["P_in"], M["P_out"], M["max_model_len"]
    w = M.get("w_tpot", 0.5)
    tp, ns, u = V["tp"], V["max_num_seqs"], V["u"]
    cpf = V["cpf"] == 1
    mbt = V["mbt"]
    _, cap = device_assignment(space, tp.astype(np.int64))
    W = 2.0 * P
    kvb = 4.0 * L * kv * dh / tp
    mbt_eff = np.where(cpf, mbt, float(mml))
    # usable bytes, normative order: ((u*cap - W/tp) - (((mbt_eff*(4h+2ffn))*2)/tp)) - 1e9
    t1 = u * cap
    t2 = W / tp
    t3 = mbt_eff * float(4 * h + 2 * ffn)
    t4 = t3 * 2.0
    t5 = t4 / tp
    usable = ((t1 - t2) - t5) - 1e9
    kv_tok = np.floor(usable / kvb)
    ok = (usable > 0) & (kv_tok >= mml)
    b = np.minimum(ns, np.floor(kv_tok / float(P_in + P_out)))
    b = np.where(ok, b, 1.0)      # times are meaningless for masked configs; keep them finite
    bw_hbm, peak, bw_intra = hw["bw_hbm"], hw["peak_flops"], hw["bw_intra"]
    T_w = (W / tp) / bw_hbm
    T_kv = b * (P_in + P_out / 2.0) * kvb / bw_hbm
    T_fl = 2.0 * P * b / (tp * peak)
    T_ar = np.where(tp > 1, 2.0 * L * (2.0 * (tp - 1.0) / tp * b * h * 2.0 / bw_intra + 5e-6), 0.0)
    t_sched = 5e-4
    t_dec = np.maximum(T_w + T_kv, T_fl) + T_ar + t_sched
    p = b * P_in / P_out
    T_pf = 2.0 * P / (tp * peak * 0.6)
    t_pf = np.where(cpf,
                    p * T_pf + np.maximum(0.0, p - (mbt - b)) / mbt * (T_w + t_sched),
                    (b / P_out) * (T_w + t_sched) + p * T_pf)
    TPOT = t_dec + t_pf
    thr = (space.G / tp) * b / TPOT
    cost = TPOT ** w * thr ** (-(1.0 - w))
    return cost, ok, usable, dict(TPOT=TPOT, thr=thr, b=b, kv_tok=kv_tok, t_dec=t_dec, t_pf=t_pf)
