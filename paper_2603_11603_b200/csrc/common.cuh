// Shared host/device definitions of the scoring path: device data layout, candidate decode,
// analytical simulator + FP64 resource check, acquisition.  Compiled for the host (observe,
// introspection) and for sm_100a (score / refine / mask kernels) from the same source.
//
// Formulas: SURVEY.md Appendix A (A.1 index spaces, A.2 bit-exact resource check, A.3 training
// simulator, A.4 serving simulator, A.5 surrogate/acquisition); readings in DESIGN.md §3.
#pragma once
#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define AS_HD __host__ __device__ __forceinline__
#else
#define AS_HD inline
#endif

namespace as {

constexpr int DMAX = 24;        // max features (3 x 8 digit bytes)
constexpr int VMAX = 64;        // max domain size (predicates are 64-bit digit masks)
constexpr int TUPW = 8;         // max features in one tail gating group
constexpr int MMAX = 256;       // max observed configurations (round-1 SMEM budget)
constexpr int MAX_CLS = 4;      // device classes of the simulated cluster

// ---- digit vector: 24 digits x 8 bits in three 64-bit words (feature j -> word j>>3, byte j&7)
struct DV {
  uint64_t w[3];
};
AS_HD uint32_t dv_get(const DV& v, int j) {
  uint64_t x = (j < 8) ? v.w[0] : ((j < 16) ? v.w[1] : v.w[2]);
  return static_cast<uint32_t>((x >> ((j & 7) * 8)) & 0xFFu);
}
AS_HD void dv_set(DV& v, int j, uint32_t d) {
  uint64_t m = ~(0xFFull << ((j & 7) * 8));
  uint64_t b = static_cast<uint64_t>(d) << ((j & 7) * 8);
  if (j < 8) v.w[0] = (v.w[0] & m) | b;
  else if (j < 16) v.w[1] = (v.w[1] & m) | b;
  else v.w[2] = (v.w[2] & m) | b;
}

// One entry of a per-structure tail-component list: the component's digits pre-placed in the
// digit vector, its contribution to the raw index, and its activity bits.
struct Tuple {
  DV dv;
  uint64_t raw;
  uint32_t act;
  uint32_t pad;
};

enum Knob {
  K_PP, K_VPP, K_TP, K_DP, K_CP, K_EP, K_MBS, K_AR, K_ARL, K_SP, K_TPOV, K_TPCOMM, K_DOPT, K_OVG,
  K_OVP, K_BUCKET, K_DDP, K_DISP, K_NS, K_CPF, K_MBT, K_U, NKNOB
};

struct SimParams {
  int mode;                  // 0 spec, 1 derived (A.3), 2 serve (A.4)
  int kf[NKNOB];             // feature index bound to each knob, -1 if the preset lacks it
  // digit extraction of a bound knob without per-call index arithmetic: digit vector word kw,
  // bit shift ks, table offset ko = kf * VMAX, activity bit kbit = 1 << kf
  int kw[NKNOB], ks[NKNOB], ko[NKNOB];
  uint32_t kbit[NKNOB];
  double neutral[NKNOB];     // value of an absent knob (A.3 "Knobs absent from a preset")
  int n_cls;                 // device classes, sorted by relative throughput (fastest first)
  int cls_count[MAX_CLS];
  double cls_cap[MAX_CLS];   // bytes
  double cls_eff[MAX_CLS];
  // SPEC mode constants (S:547 + DESIGN.md R8)
  double F_work, alpha_tp, alpha_dp, r_ar, B, P_mem, A_mem;
  // derived / serving constants (model + hardware descriptor)
  double L, h, a, kv, S, GBS, P, P_exp, E, topk, peak, mfu0, bw_intra, bw_inter, gpn, n_sm;
  double dh, ffn, P_in, P_out, mml, w_tpot, bw_hbm, G;
  // derived per-space constants of the cost terms (set by build_space; the resource check does not
  // use them).  Cost terms multiply by per-digit reciprocals instead of dividing (R7:
  // only the resource check is bit-exact; the cost agrees with the oracle to rounding).
  double inv_B, inv_GBS, inv_bw_intra, inv_bw_inter, half_inv_nsm, T_work, C_tp, C_ep, C_cp;
  double neutral_inv[NKNOB], neutral_lg2[NKNOB];
};

// ---- exact FP64 arithmetic for the resource check (A.2): no FMA contraction, fixed order.
#ifdef __CUDA_ARCH__
AS_HD double xadd(double a, double b) { return __dadd_rn(a, b); }
AS_HD double xsub(double a, double b) { return __dsub_rn(a, b); }
AS_HD double xmul(double a, double b) { return __dmul_rn(a, b); }
AS_HD double xdiv(double a, double b) { return __ddiv_rn(a, b); }
#else
AS_HD double xadd(double a, double b) { return a + b; }   // host: compiled with -ffp-contract=off
AS_HD double xsub(double a, double b) { return a - b; }
AS_HD double xmul(double a, double b) { return a * b; }
AS_HD double xdiv(double a, double b) { return a / b; }
#endif

struct Knobs {
  double v[NKNOB];
  double vi[NKNOB];  // 1 / value        (knobs in knob_has_inv)
  double lg[NKNOB];  // log2(value)      (knobs in knob_has_lg2)
  uint32_t act;  // bit k: knob k bound to an active feature
};
AS_HD constexpr bool knob_has_inv(int i) {
  return i == K_PP || i == K_VPP || i == K_TP || i == K_DP || i == K_CP || i == K_EP || i == K_MBS;
}
AS_HD constexpr bool knob_has_lg2(int i) { return i == K_MBS || i == K_BUCKET; }

// Effective knob values of a decoded canonical configuration: inactive features carry their
// default digit (G1), so the digit's value is the effective value.
// Tables: val / inv / lg2 [feature][digit] (inv and lg2 only read for the knobs that need them).
AS_HD void load_knobs(const SimParams& P, const double* val, const double* inv, const double* lg2, const DV& dv,
                      uint32_t act_bits, Knobs& k) {
  k.act = 0;
#pragma unroll
  for (int i = 0; i < NKNOB; ++i) {
    if (P.kf[i] >= 0) {
      const int kw = P.kw[i];
      const uint64_t w = kw == 0 ? dv.w[0] : (kw == 1 ? dv.w[1] : dv.w[2]);
      const int o = P.ko[i] + static_cast<int>((w >> P.ks[i]) & 0xFFu);
      k.v[i] = val[o];
      if (knob_has_inv(i)) k.vi[i] = inv[o];
      if (knob_has_lg2(i)) k.lg[i] = lg2[o];
      if (act_bits & P.kbit[i]) k.act |= (1u << i);
    } else {
      k.v[i] = P.neutral[i];
      if (knob_has_inv(i)) k.vi[i] = P.neutral_inv[i];
      if (knob_has_lg2(i)) k.lg[i] = P.neutral_lg2[i];
    }
  }
}

AS_HD void device_assignment(const SimParams& P, double world, double& eff, double& cap) {
  double rem = world;
  eff = INFINITY;
  cap = INFINITY;
  for (int i = 0; i < P.n_cls; ++i) {
    if (rem <= 0.0) break;
    eff = fmin(eff, P.cls_eff[i]);
    cap = fmin(cap, P.cls_cap[i]);
    rem -= static_cast<double>(P.cls_count[i]);
  }
}

AS_HD double bw_of(const SimParams& P, double span) { return span <= P.gpn ? P.bw_intra : P.bw_inter; }
AS_HD double inv_bw_of(const SimParams& P, double span) { return span <= P.gpn ? P.inv_bw_intra : P.inv_bw_inter; }
AS_HD double clamp(double x, double lo, double hi) { return fmin(fmax(x, lo), hi); }

// Simulator: cost in objective units (s/iter, or the scalarized serving cost), resource check.
// mem_out = training memory (bytes) or serving usable bytes.
AS_HD void simulate(const SimParams& P, const Knobs& k, double& cost, bool& ok, double& mem_out) {
  const double pp = k.v[K_PP], tp = k.v[K_TP], dp = k.v[K_DP], cp = k.v[K_CP], ep = k.v[K_EP],
               mbs = k.v[K_MBS];
  if (P.mode == 0) {  // ---- SPEC synthetic_cost, S:489-497 verbatim
    const bool ar = k.v[K_AR] == 2.0, sp = k.v[K_SP] == 1.0;
    const double world = pp * tp * dp * cp;
    double eff, cap;
    device_assignment(P, world, eff, cap);
    const double r = ar ? P.r_ar : 1.0;
    const double t_comp = P.F_work * r / (world * eff * (1.0 + 0.1 * k.lg[K_MBS]));
    const double t_bubble = t_comp * (pp - 1.0) * (dp * mbs) * P.inv_B;   // / micro, micro = B/(dp mbs)
    const double ov = tp > 1.0 ? clamp((k.v[K_TPCOMM] - 12.0) * 0.0625, 0.0, 0.5) : 0.0;
    const double t_tp = P.alpha_tp * (1.0 - k.vi[K_TP]) * (1.0 - ov) * ((sp && tp > 1.0) ? 0.8 : 1.0);
    const double lb = k.lg[K_BUCKET] - 2.0;
    const double bp = dp > 1.0 ? 1.0 + 0.1 * lb * lb : 0.0;
    const double t_dp = P.alpha_dp * (1.0 - k.vi[K_DP]) * bp;
    const double t_ep = P.alpha_tp * 0.5 * (1.0 - k.vi[K_EP]);
    cost = t_comp + t_bubble + t_tp + t_dp + t_ep;
    // S:496 in the normative order (R7): (P_mem/(pp*tp)) + (((A_mem*mbs)*f)/cp)
    const double m1 = xdiv(P.P_mem, xmul(pp, tp));
    const double m2 = xmul(P.A_mem, mbs);
    const double m3 = xmul(m2, ar ? 0.3 : 1.0);
    const double m4 = xdiv(m3, cp);
    const double mem = xadd(m1, m4);
    mem_out = mem;
    ok = mem <= cap;
    return;
  }
  if (P.mode == 1) {  // ---- derived mode, SURVEY A.3
    const double vpp = k.v[K_VPP];
    const double arc = k.v[K_AR];
    const bool full = arc == 2.0, sel = arc == 1.0, sp = k.v[K_SP] == 1.0;
    const double world = pp * tp * dp * cp;
    const double L_st = xdiv(P.L, xmul(pp, vpp));
    const bool arl_active = (k.act >> K_ARL) & 1u;
    const double f_rc = full ? (arl_active ? fmin(1.0, xdiv(k.v[K_ARL], L_st)) : 1.0) : 0.0;
    const double r = 1.0 + 0.33 * f_rc + (sel ? 0.03 : 0.0);
    const bool tpc_active = (k.act >> K_TPCOMM) & 1u;
    const double steal = tpc_active ? k.v[K_TPCOMM] * P.half_inv_nsm : 0.0;
    const double ipdc = k.vi[K_PP] * k.vi[K_DP] * k.vi[K_CP];         // 1 / (pp dp cp)
    const double t_comp = P.T_work * r * (1.0 + steal) * (ipdc * k.vi[K_TP]) / (1.0 + 0.1 * k.lg[K_MBS]);
    const double t_bubble = t_comp * (pp - 1.0) * (dp * mbs * P.inv_GBS) * k.vi[K_VPP];   // / (m vpp)
    const double ov = (tp > 1.0 && tpc_active) ? clamp((k.v[K_TPCOMM] - 12.0) * 0.0625, 0.0, 0.5) : 0.0;
    const double t_tp = tp > 1.0 ? P.C_tp * ipdc * inv_bw_of(P, tp) * (1.0 - k.vi[K_TP]) * (1.0 - ov) * (sp ? 0.8 : 1.0)
                                 : 0.0;
    const double P_loc = xdiv(xadd(P.P - P.P_exp, xdiv(P.P_exp, ep)), xmul(pp, tp));
    const double lb = k.lg[K_BUCKET] - 2.0;
    const bool ovg = k.v[K_OVG] == 1.0, ovp = k.v[K_OVP] == 1.0;
    const double t_dp = dp > 1.0 ? 4.0 * P_loc * inv_bw_of(P, tp * cp * dp) * (1.0 - k.vi[K_DP]) *
                                       (1.0 + 0.1 * lb * lb) * (ovg ? 0.5 : 1.0) * (ovp ? 0.75 : 1.0)
                                 : 0.0;
    const double t_ep = ep > 1.0 ? P.C_ep * ipdc * (sp ? k.vi[K_TP] : 1.0) * inv_bw_of(P, tp * cp * ep) *
                                       (1.0 - k.vi[K_EP]) * (k.v[K_DISP] == 1.0 ? 1.5 : 1.0)
                                 : 0.0;
    const double t_cp = cp > 1.0 ? P.C_cp * k.vi[K_PP] * k.vi[K_DP] * inv_bw_of(P, tp * cp) * (1.0 - k.vi[K_CP])
                                 : 0.0;
    cost = t_comp + t_bubble + t_tp + t_dp + t_ep + t_cp;
    // memory, normative FP64 order (R7)
    const bool dopt = k.v[K_DOPT] == 1.0;
    const double bpp = dopt ? xadd(6.0, xdiv(12.0, dp)) : 18.0;
    const double act = sp ? xdiv(34.0, tp) : xadd(10.0, xdiv(24.0, tp));
    const double af = xsub(xsub(1.0, xmul(0.7, f_rc)), sel ? 0.2 : 0.0);
    const double t1 = xmul(P_loc, bpp);
    double t2 = xmul(P.L, xdiv(P.S, cp));
    t2 = xmul(t2, P.h);
    t2 = xmul(t2, mbs);
    t2 = xmul(t2, act);
    t2 = xmul(t2, af);
    const double mem = xadd(t1, t2);
    double eff, cap;
    device_assignment(P, world, eff, cap);
    mem_out = mem;
    ok = mem <= cap;
    return;
  }
  // ---- serving, SURVEY A.4
  const double ns = k.v[K_NS], u = k.v[K_U], mbt = k.v[K_MBT];
  const bool cpf = k.v[K_CPF] == 1.0;
  double eff, cap;
  device_assignment(P, tp, eff, cap);
  const double W = 2.0 * P.P;
  const double kvb = xdiv(xmul(xmul(xmul(4.0, P.L), P.kv), P.dh), tp);
  const double mbt_eff = cpf ? mbt : P.mml;
  const double t1 = xmul(u, cap);
  const double t2 = xdiv(W, tp);
  const double t3 = xmul(mbt_eff, 4.0 * P.h + 2.0 * P.ffn);
  const double t4 = xmul(t3, 2.0);
  const double t5 = xdiv(t4, tp);
  const double usable = xsub(xsub(xsub(t1, t2), t5), 1e9);
  const double kv_tok = floor(xdiv(usable, kvb));
  ok = (usable > 0.0) && (kv_tok >= P.mml);
  mem_out = usable;
  double b = fmin(ns, floor(kv_tok / (P.P_in + P.P_out)));
  if (!ok) b = 1.0;
  const double T_w = (W / tp) / P.bw_hbm;
  const double T_kv = b * (P.P_in + P.P_out / 2.0) * kvb / P.bw_hbm;
  const double T_fl = 2.0 * P.P * b / (tp * P.peak);
  const double T_ar = tp > 1.0 ? 2.0 * P.L * (2.0 * (tp - 1.0) / tp * b * P.h * 2.0 / P.bw_intra + 5e-6) : 0.0;
  const double t_sched = 5e-4;
  const double t_dec = fmax(T_w + T_kv, T_fl) + T_ar + t_sched;
  const double p = b * P.P_in / P.P_out;
  const double T_pf = 2.0 * P.P / (tp * P.peak * 0.6);
  const double t_pf = cpf ? p * T_pf + fmax(0.0, p - (mbt - b)) / mbt * (T_w + t_sched)
                          : (b / P.P_out) * (T_w + t_sched) + p * T_pf;
  const double TPOT = t_dec + t_pf;
  const double thr = (P.G / tp) * b / TPOT;
  cost = pow(TPOT, P.w_tpot) * pow(thr, -(1.0 - P.w_tpot));
}

// ---- derived mode, partial evaluation per structure (gen kernel fast path).
// Every derived-mode cost term is a product of factors that depend on the structural prefix only
// (pp, vpp, tp, dp, cp, ep, mbs, ar, arl when they are prefix features) and per-candidate tail
// factors (tp_comm steal / overlap, sp, bucket penalty, ovg, ovp, dispatcher).  The structural
// products are evaluated once per structure on the host; the resource check of every structure
// is tabulated over the tail features it reads (sp, dopt, ... and their tail gates), computed
// with the normative FP64 order by the same simulate() (R7: bit-identical).  Costs agree with
// simulate() to FP64 re-association (the refine kernel still evaluates simulate() itself).
struct SimRec {
  double comp;        // T_work r ipdc vi_tp / (1 + 0.1 lg mbs)      t_comp = comp (1 + steal)
  double bub;         // (pp - 1) (dp mbs / GBS) vi_vpp              t_bubble = t_comp bub
  double tp;          // tp > 1: C_tp ipdc inv_bw(tp) (1 - vi_tp)     x (1 - ov) (sp ? 0.8 : 1)
  double dp;          // dp > 1: 4 P_loc inv_bw(tp cp dp) (1 - vi_dp) x (1 + 0.1 lb^2) ovg ovp
  double ep;          // ep > 1: C_ep ipdc inv_bw(tp cp ep) (1 - vi_ep) x (sp ? vi_tp : 1) disp
  double cp;          // t_cp
  double vi_tp;       // 1 / tp (t_ep's sequence-parallel factor)
  uint32_t tpgt1;     // tp > 1
  uint32_t pad;
  uint64_t memok;     // bit c: resource check passes for tail combination c
  uint64_t pad2;      // 80 B: five 16-byte loads
};
constexpr int SR_MAXCF = 4;   // tail features in the resource-check combination
struct SimFast {
  int on;
  int n_cf;
  int cf_w[SR_MAXCF], cf_s[SR_MAXCF];   // digit word / bit shift of combination feature i
  uint32_t cf_mul[SR_MAXCF];            // combination index = sum digit_i * cf_mul[i]
};
AS_HD uint32_t knob_digit(const SimParams& P, int i, const DV& dv) {
  const int kw = P.kw[i];
  const uint64_t w = kw == 0 ? dv.w[0] : (kw == 1 ? dv.w[1] : dv.w[2]);
  return static_cast<uint32_t>((w >> P.ks[i]) & 0xFFu);
}
AS_HD double knob_val(const SimParams& P, const double* val, int i, const DV& dv) {
  return P.kf[i] >= 0 ? val[P.ko[i] + static_cast<int>(knob_digit(P, i, dv))] : P.neutral[i];
}
// per-structure products from the structural knobs k (tail knob values in k are ignored)
AS_HD void simrec_base(const SimParams& P, const Knobs& k, SimRec& r) {
  const double pp = k.v[K_PP], tp = k.v[K_TP], dp = k.v[K_DP], cp = k.v[K_CP], ep = k.v[K_EP], mbs = k.v[K_MBS];
  const double vpp = k.v[K_VPP], arc = k.v[K_AR];
  const bool full = arc == 2.0, sel = arc == 1.0;
  const double L_st = xdiv(P.L, xmul(pp, vpp));
  const bool arl_active = (k.act >> K_ARL) & 1u;
  const double f_rc = full ? (arl_active ? fmin(1.0, xdiv(k.v[K_ARL], L_st)) : 1.0) : 0.0;
  const double rr = 1.0 + 0.33 * f_rc + (sel ? 0.03 : 0.0);
  const double ipdc = k.vi[K_PP] * k.vi[K_DP] * k.vi[K_CP];
  r.comp = P.T_work * rr * (ipdc * k.vi[K_TP]) / (1.0 + 0.1 * k.lg[K_MBS]);
  r.bub = (pp - 1.0) * (dp * mbs * P.inv_GBS) * k.vi[K_VPP];
  r.tp = tp > 1.0 ? P.C_tp * ipdc * inv_bw_of(P, tp) * (1.0 - k.vi[K_TP]) : 0.0;
  const double P_loc = xdiv(xadd(P.P - P.P_exp, xdiv(P.P_exp, ep)), xmul(pp, tp));
  r.dp = dp > 1.0 ? 4.0 * P_loc * inv_bw_of(P, tp * cp * dp) * (1.0 - k.vi[K_DP]) : 0.0;
  r.ep = ep > 1.0 ? P.C_ep * ipdc * inv_bw_of(P, tp * cp * ep) * (1.0 - k.vi[K_EP]) : 0.0;
  r.cp = cp > 1.0 ? P.C_cp * k.vi[K_PP] * k.vi[K_DP] * inv_bw_of(P, tp * cp) * (1.0 - k.vi[K_CP]) : 0.0;
  r.vi_tp = k.vi[K_TP];
  r.tpgt1 = tp > 1.0 ? 1u : 0u;
  r.pad = 0;
}
// cost + resource check of a candidate of structure record r (digits dv, activity act)
AS_HD void sim_fast(const SimParams& P, const SimFast& F, const double* val, const double* lg2, const SimRec& r,
                    const DV& dv, uint32_t act, double& cost, bool& ok) {
  const bool tpc_on = P.kf[K_TPCOMM] >= 0 && ((act & P.kbit[K_TPCOMM]) != 0u);
  const double v_tpc = knob_val(P, val, K_TPCOMM, dv);
  const bool sp = knob_val(P, val, K_SP, dv) == 1.0;
  const double lgb = P.kf[K_BUCKET] >= 0 ? lg2[P.ko[K_BUCKET] + static_cast<int>(knob_digit(P, K_BUCKET, dv))]
                                         : P.neutral_lg2[K_BUCKET];
  const bool ovg = knob_val(P, val, K_OVG, dv) == 1.0, ovp = knob_val(P, val, K_OVP, dv) == 1.0;
  const bool disp = knob_val(P, val, K_DISP, dv) == 1.0;
  const double steal = tpc_on ? v_tpc * P.half_inv_nsm : 0.0;
  const double t_comp = r.comp * (1.0 + steal);
  const double ov = (r.tpgt1 && tpc_on) ? clamp((v_tpc - 12.0) * 0.0625, 0.0, 0.5) : 0.0;
  const double lb = lgb - 2.0;
  cost = t_comp + t_comp * r.bub + r.tp * (1.0 - ov) * (sp ? 0.8 : 1.0) +
         r.dp * (1.0 + 0.1 * lb * lb) * (ovg ? 0.5 : 1.0) * (ovp ? 0.75 : 1.0) +
         r.ep * (sp ? r.vi_tp : 1.0) * (disp ? 1.5 : 1.0) + r.cp;
  uint32_t c = 0;
  for (int i = 0; i < F.n_cf; ++i) {
    const uint64_t w = F.cf_w[i] == 0 ? dv.w[0] : (F.cf_w[i] == 1 ? dv.w[1] : dv.w[2]);
    c += static_cast<uint32_t>((w >> F.cf_s[i]) & 0xFFu) * F.cf_mul[i];
  }
  ok = (r.memok >> c) & 1ull;
}

// ---- acquisition in FP64 (R10)
constexpr double LN_2PI = 1.8378770664093454835606594728112;
constexpr double INV_SQRT_2PI = 0.39894228040143267793994605993438;
constexpr double INV_SQRT2 = 0.70710678118654752440084436210485;

AS_HD double lnh(double z) {
  if (z >= -10.0) {
    const double phi = exp(-0.5 * z * z) * INV_SQRT_2PI;
    const double Phi = 0.5 * erfc(-z * INV_SQRT2);
    return log(phi + z * Phi);
  }
  const double z2 = z * z;
  const double z4 = z2 * z2;
  return -0.5 * z2 - 0.5 * LN_2PI - 2.0 * log(-z) +
         log1p(-3.0 / z2 + 15.0 / z4 - 105.0 / (z4 * z2) + 945.0 / (z4 * z4));
}

// acq: 0 EI (log EI), 1 LCB, 2 SIM
AS_HD double acquisition(int acq, double mu, double s2, double m0, double fstar, double xi, double kappa) {
  if (acq == 2) return -m0;
  const double sigma = sqrt(fmax(s2, 0.0));
  if (acq == 1) return kappa * sigma - mu;
  const double u = fstar - mu - xi;
  if (sigma == 0.0) return u > 0.0 ? log(u) : -INFINITY;
  return log(sigma) + lnh(u / sigma);
}

// ---- Matern-5/2 / RBF (A.5)
constexpr double SQRT5 = 2.2360679774997896964091736687313;
AS_HD double kernel64(int kind, double sf2, double r2) {
  const double r = sqrt(r2);
  if (kind == 0) return sf2 * (1.0 + SQRT5 * r + (5.0 / 3.0) * r2) * exp(-SQRT5 * r);
  return sf2 * exp(-0.5 * r2);
}

// ---- splitmix64 + Feistel permutation of [0, n) for SAMPLE mode (R3)
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
AS_HD uint64_t splitmix64(uint64_t z) {
  z += GOLDEN;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// SAMPLE-mode permutation (R3): 4-round Feistel on b = max(2, ceil(log2 n)) bits with
// alternating unbalanced halves (|L| = ceil(b/2), |R| = floor(b/2)), round function
// fmix32(R ^ k_r) masked to |L|, cycle-walked into [0, n).  n < 2^32.
struct FeistelKey {
  uint32_t k[4];
  uint64_t n;
  uint32_t a, c;   // |L|, |R| of the input layout
};
inline FeistelKey feistel_make(uint64_t n, uint64_t seed) {
  FeistelKey f;
  f.n = n;
  uint32_t b = 0;
  while ((1ull << b) < n) ++b;  // ceil(log2 n)
  if (b < 2) b = 2;
  f.a = (b + 1) / 2;
  f.c = b / 2;
  for (int r = 0; r < 4; ++r) f.k[r] = static_cast<uint32_t>(splitmix64(seed ^ (GOLDEN * static_cast<uint64_t>(r + 1))));
  return f;
}
AS_HD uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}
AS_HD uint32_t feistel_E(const FeistelKey& f, uint32_t x) {
  uint32_t a = f.a, c = f.c;
  uint32_t L = x >> c, R = x & ((1u << c) - 1u);
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t nl = R;
    R = L ^ (fmix32(R ^ f.k[r]) & ((1u << a) - 1u));
    L = nl;
    const uint32_t t = a;
    a = c;
    c = t;
  }
  return (L << c) | R;
}
AS_HD uint64_t feistel_pi(const FeistelKey& f, uint64_t j) {
  uint32_t x = feistel_E(f, static_cast<uint32_t>(j));
  while (x >= f.n) x = feistel_E(f, x);
  return x;
}

}  // namespace as
