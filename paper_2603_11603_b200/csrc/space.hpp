// Host-side space model: parsing/validation of the space JSON, the structural-prefix /
// tail-component decomposition that defines the compact valid index (CVI), exact host decode,
// and the FP64 GP fit of the observed set.  See DESIGN.md §5.1 for the layout.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"

namespace as {

struct Status {
  int code = 0;  // as_status
  std::string msg;
  bool ok() const { return code == 0; }
};

struct Atom {
  int ref;           // referenced (earlier) feature
  uint64_t allowed;  // digit mask of the referenced feature for which the comparison holds
};

struct FeatureH {
  std::string name;
  int n = 0;
  int dflt = 0;
  int vkind = 0;              // 0 number, 1 bool, 2 string
  bool dense = false;         // kind "dense" (coordinate-search knob)
  std::vector<double> num;    // numeric value of each digit (bool 0/1, string: index)
  std::vector<std::string> str;
  std::vector<Atom> req;
};

enum CType {
  C_PROD_EQ_DEV, C_PROD_LE_DEV_POW2, C_DIVIDES, C_DIVIDES_CONST, C_GBS_DIV, C_SEQ_2CP, C_GE,
  C_LE_CONST_DIV, C_MB_DIV_PP, C_IMPLIES
};

struct ConstraintH {
  int type;
  std::vector<int> f;            // product features / div features
  int a = -1, b = -1;            // divides a|b, ge a>=b, le_const_div feature a, mb: vpp,pp,dp,mbs in f
  double cval = 0;               // constant
  bool divides_devices = false;
  std::vector<Atom> iff, then;   // implies
  int last = 0;                  // highest referenced feature
};

struct HostSpace {
  std::string name;
  int d = 0;
  std::vector<FeatureH> feat;
  std::vector<ConstraintH> cons;
  double G = 0;
  uint64_t stride[DMAX] = {};
  uint64_t n_raw = 0;
  // CVI decomposition
  int n_prefix = 0;
  std::vector<int> comp_first, comp_width;
  int n_struct = 0;
  std::vector<uint64_t> prefix;   // [n_struct+1]
  std::vector<uint64_t> s_raw;    // [n_struct] raw base (ascending)
  std::vector<uint32_t> s_act;    // [n_struct]
  std::vector<DV> s_dv;           // [n_struct]
  std::vector<uint32_t> s_off, s_cnt;  // [n_struct * n_comp]
  std::vector<Tuple> tuples;
  uint64_t n_cvi = 0;
  uint64_t tail_span = 1;         // stride of the last prefix feature (raw size of one structure's tail)
  // value tables (VMAX per feature)
  std::vector<double> val;        // simulator values
  std::vector<double> inv, lg2;   // 1/value, log2(value) (cost terms; 0 where value == 0)
  std::vector<double> xt64;       // GP features x~ = phi / l
  std::vector<float> xt32;
  SimParams sim{};
  // GP hyper-parameters
  int kernel = 0;                 // 0 matern52, 1 rbf
  double sf2 = 0.1, sn2 = 1e-3, xi = 0.0, kappa = 2.0;
  int prior = 0;                  // gp.prior: 0 "sim" (ln cost_sim, R9), 1 "ensemble" (NEXT-1, R20)
  uint64_t ens_seed = 0;          // gp.ensemble_seed: holdout split of the regression simulators
  int onehot_max = 64;            // gp.onehot_max_width: one-hot r^2 width target of the TC kernel (impl. knob)
  std::vector<double> ls;
};

Status build_space(const char* json, HostSpace& S);
void feature_tables(HostSpace& S);   // x~ = phi / l tables from S.ls (after a lengthscale change)

// Exact host introspection.
void activity(const HostSpace& S, const int* dig, bool* act);
bool cvi_decode(const HostSpace& S, uint64_t p, DV& dv, uint32_t& act, uint64_t& raw);  // p < n_cvi
// raw -> digits; *structural = G1 + constraints (membership in the CVI); returns false if raw >= n_raw
uint64_t cvi_rank(const HostSpace& S, uint64_t raw, bool* member);   // #members with raw index < raw
bool raw_decode(const HostSpace& S, uint64_t raw, int* dig, DV& dv, uint32_t& act, bool& structural);
void simulate_host(const HostSpace& S, const DV& dv, uint32_t act, double& cost, bool& ok, double& mem);

// FP64 GP fit of the observed set (R9).
struct GPFit {
  int M = 0;
  double b = 0.0, fstar = INFINITY;
  std::vector<double> X;        // [M][d] x~ of observed
  std::vector<double> alpha;    // [M] K^-1 r
  std::vector<double> r;        // [M] residual y - m0 - b (the GP's observations; ML-II evidence)
  std::vector<double> Wl;       // [M][M] L^-1 (lower triangular, row-major)
  double w_fro = 0.0;           // ||L^-1||_F  (error bound of the FP32 screen)
};
Status gp_fit(const HostSpace& S, const std::vector<DV>& obs_dv, const std::vector<uint32_t>& obs_act,
              const std::vector<double>& cost, const std::vector<double>& cost_sim, GPFit& fit,
              const std::vector<double>* m0_prior = nullptr);

// Regression-simulator ensemble (NEXT-1; reading R20): four ridge-stabilised
// linear fits of ln c on the Table 2 knob subsets, R^2 on a seeded 20 % holdout, weights
// max(0,R^2)/sum.  on = false when every R^2 <= 0 (Unavailable).  The weighted sum of linear
// models is one linear model: m0(x) = c0 + sum_f tab[f][digit_f].
struct EnsembleFit {
  bool on = false;
  double c0 = 0.0;
  double r2[4] = {0, 0, 0, 0};
  double w[4] = {0, 0, 0, 0};
  std::vector<double> tab;        // [d * VMAX]
};
void ensemble_fit(const HostSpace& S, const std::vector<DV>& dv, const std::vector<double>& cost, EnsembleFit& e);
double ensemble_m0(const HostSpace& S, const EnsembleFit& e, const DV& dv);

}  // namespace as
