// Host-side space compiler: JSON -> validated feature/constraint model -> CVI structure tables.
// Compiled with -ffp-contract=off so the host FP64 resource check is bit-identical to the
// oracle's numpy evaluation and to the device's __dmul_rn/__dadd_rn path (R7).
#include "space.hpp"
#include "host_pool.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <numeric>
#include <set>

#include "json.hpp"

namespace as {

namespace {

enum { E_ARG = 1, E_SCHEMA = 2, E_CYCLE = 3, E_ORDER = 4, E_EMPTY = 5, E_CAP = 10, E_NUM = 9 };

Status err(int code, const std::string& m) { return Status{code, m}; }

bool cmp_num(double a, const std::string& op, double b) {
  if (op == ">") return a > b;
  if (op == ">=") return a >= b;
  if (op == "==") return a == b;
  if (op == "!=") return a != b;
  if (op == "<") return a < b;
  if (op == "<=") return a <= b;
  return false;
}

bool valid_op(const std::string& op) {
  return op == ">" || op == ">=" || op == "==" || op == "!=" || op == "<" || op == "<=";
}

// Build the allowed-digit mask of an atomic comparison "ref <op> value".
Status make_atom(const HostSpace& S, int ref, const std::string& op, const asj::Value& v, Atom& out) {
  const FeatureH& r = S.feat[ref];
  if (!valid_op(op)) return err(E_SCHEMA, "bad comparison operator '" + op + "'");
  out.ref = ref;
  out.allowed = 0;
  for (int k = 0; k < r.n; ++k) {
    bool hold;
    if (r.vkind == 2 || v.kind == asj::Value::String) {
      if (r.vkind != 2 || v.kind != asj::Value::String || (op != "==" && op != "!="))
        return err(E_SCHEMA, "categorical comparison must be ==/!= between strings (" + r.name + ")");
      hold = (op == "==") == (r.str[k] == v.str);
    } else {
      double b;
      if (v.kind == asj::Value::Bool) b = v.b ? 1.0 : 0.0;
      else if (v.kind == asj::Value::Number) b = v.num;
      else return err(E_SCHEMA, "predicate value must be a number, bool or string");
      hold = cmp_num(r.num[k], op, b);
    }
    if (hold) out.allowed |= (1ull << k);
  }
  return Status{};
}

const asj::Value* need(const asj::Value& o, const char* k) { return o.get(k); }

int feature_index(const HostSpace& S, const std::string& n) {
  for (int i = 0; i < S.d; ++i)
    if (S.feat[i].name == n) return i;
  return -1;
}

double model_const(const asj::Value* model, const std::string& k, double dflt, bool* found = nullptr) {
  const asj::Value* v = model ? model->get(k) : nullptr;
  if (found) *found = (v && v->kind == asj::Value::Number);
  if (!v || v->kind != asj::Value::Number) return dflt;
  return v->num;
}

}  // namespace

void activity(const HostSpace& S, const int* dig, bool* act) {
  for (int j = 0; j < S.d; ++j) {
    bool a = true;
    for (const Atom& at : S.feat[j].req) {
      if (!act[at.ref] || !((at.allowed >> dig[at.ref]) & 1ull)) { a = false; break; }
    }
    act[j] = a;
  }
}

static double eff_value(const HostSpace& S, int f, const int* dig, const bool* act) {
  const FeatureH& F = S.feat[f];
  return F.num[act[f] ? dig[f] : F.dflt];
}

static bool atom_holds(const Atom& a, const int* dig, const bool* act) {
  return act[a.ref] && ((a.allowed >> dig[a.ref]) & 1ull);
}

// One structural constraint on effective values (R5; same semantics as the oracle).
static bool constraint_ok(const HostSpace& S, const ConstraintH& c, const int* dig, const bool* act) {
  auto ev = [&](int f) { return eff_value(S, f, dig, act); };
  auto prod = [&](const std::vector<int>& fs) {
    double p = 1.0;
    for (int f : fs) p *= ev(f);
    return p;
  };
  auto imod = [](double a, double b) { return std::fmod(a, b) == 0.0; };
  switch (c.type) {
    case C_PROD_EQ_DEV: return prod(c.f) == S.G;
    case C_PROD_LE_DEV_POW2: {
      double w = prod(c.f);
      uint64_t wi = static_cast<uint64_t>(w);
      bool ok = w <= S.G && (wi & (wi - 1)) == 0;
      if (c.divides_devices) ok = ok && imod(S.G, w);
      return ok;
    }
    case C_DIVIDES: return imod(ev(c.b), ev(c.a));
    case C_DIVIDES_CONST: return imod(c.cval, prod(c.f));
    case C_GBS_DIV: return imod(c.cval, prod(c.f));
    case C_SEQ_2CP: {
      double cp = ev(c.a);
      return cp == 1.0 || imod(c.cval, 2.0 * cp);
    }
    case C_GE:
      if (!(act[c.a] && act[c.b])) return true;
      return ev(c.a) >= ev(c.b);
    case C_LE_CONST_DIV:
      if (!act[c.a]) return true;
      return ev(c.a) * prod(c.f) <= c.cval;
    case C_MB_DIV_PP: {  // f = {vpp, pp, dp, mbs}; cval = GBS
      if (ev(c.f[0]) <= 1.0) return true;
      double m = std::floor(c.cval / (ev(c.f[2]) * ev(c.f[3])));
      return imod(m, ev(c.f[1]));
    }
    case C_IMPLIES: {
      bool cond = true;
      for (const Atom& a : c.iff) cond = cond && atom_holds(a, dig, act);
      if (!cond) return true;
      for (const Atom& a : c.then)
        if (!atom_holds(a, dig, act)) return false;
      return true;
    }
  }
  return false;
}

static void dv_from_digits(const HostSpace& S, const int* dig, DV& dv) {
  dv.w[0] = dv.w[1] = dv.w[2] = 0;
  for (int j = 0; j < S.d; ++j) dv_set(dv, j, static_cast<uint32_t>(dig[j]));
}

static uint32_t act_bits(const HostSpace& S, const bool* act) {
  uint32_t b = 0;
  for (int j = 0; j < S.d; ++j)
    if (act[j]) b |= (1u << j);
  return b;
}

Status build_space(const char* json, HostSpace& S) {
  asj::Value doc;
  try {
    doc = asj::parse(json);
  } catch (const std::exception& e) {
    return err(E_SCHEMA, std::string("JSON: ") + e.what());
  }
  if (doc.kind != asj::Value::Object) return err(E_SCHEMA, "space document must be a JSON object");
  if (const asj::Value* n = doc.get("name"); n && n->kind == asj::Value::String) S.name = n->str;

  // ---------------------------------------------------------------- features
  const asj::Value* fs = doc.get("features");
  if (!fs || fs->kind != asj::Value::Array || fs->arr.empty())
    return err(E_SCHEMA, "space must declare at least one feature (SPEC.md:61)");
  S.d = static_cast<int>(fs->arr.size());
  if (S.d > DMAX) return err(E_CAP, "more than 24 features");
  S.feat.resize(S.d);
  std::map<std::string, int> idx;
  for (int i = 0; i < S.d; ++i) {
    const asj::Value& f = fs->arr[i];
    const asj::Value* nm = f.get("name");
    if (f.kind != asj::Value::Object || !nm || nm->kind != asj::Value::String)
      return err(E_SCHEMA, "feature needs a string name");
    if (idx.count(nm->str)) return err(E_SCHEMA, "duplicate feature name " + nm->str);
    idx[nm->str] = i;
    S.feat[i].name = nm->str;
  }
  // cycle detection over activation references
  {
    std::vector<std::vector<int>> g(S.d);
    for (int i = 0; i < S.d; ++i) {
      const asj::Value* rq = fs->arr[i].get("requires");
      if (!rq) continue;
      if (rq->kind != asj::Value::Array) return err(E_SCHEMA, "requires must be an array");
      for (const asj::Value& a : rq->arr) {
        const asj::Value* rf = a.get("feature");
        if (!rf || rf->kind != asj::Value::String || !idx.count(rf->str))
          return err(E_SCHEMA, "feature " + S.feat[i].name + " requires an unknown feature");
        g[i].push_back(idx[rf->str]);
      }
    }
    std::vector<int> st(S.d, 0);
    std::function<bool(int)> dfs = [&](int u) {
      st[u] = 1;
      for (int v : g[u]) {
        if (st[v] == 1) return false;
        if (st[v] == 0 && !dfs(v)) return false;
      }
      st[u] = 2;
      return true;
    };
    for (int u = 0; u < S.d; ++u)
      if (st[u] == 0 && !dfs(u)) return err(E_CYCLE, "cyclic activation dependency (SPEC.md:62)");
  }
  for (int i = 0; i < S.d; ++i) {
    const asj::Value& f = fs->arr[i];
    FeatureH& F = S.feat[i];
    const asj::Value* kind = f.get("kind");
    if (!kind || kind->kind != asj::Value::String || (kind->str != "sparse" && kind->str != "dense"))
      return err(E_SCHEMA, "feature " + F.name + ": kind must be sparse|dense");
    F.dense = kind->str == "dense";
    const asj::Value* dom = f.get("domain");
    if (!dom || dom->kind != asj::Value::Array) return err(E_SCHEMA, "feature " + F.name + ": domain must be an array");
    if (dom->arr.empty()) return err(E_EMPTY, "feature " + F.name + " has an empty domain (SPEC.md:58)");
    F.n = static_cast<int>(dom->arr.size());
    if (F.n > VMAX) return err(E_CAP, "feature " + F.name + ": domain larger than 64");
    const asj::Value::Kind k0 = dom->arr[0].kind;
    F.vkind = k0 == asj::Value::Number ? 0 : (k0 == asj::Value::Bool ? 1 : 2);
    if (k0 != asj::Value::Number && k0 != asj::Value::Bool && k0 != asj::Value::String)
      return err(E_SCHEMA, "feature " + F.name + ": domain values must be numbers, bools or strings");
    for (int k = 0; k < F.n; ++k) {
      const asj::Value& v = dom->arr[k];
      if (v.kind != k0) return err(E_SCHEMA, "feature " + F.name + ": mixed domain types");
      F.num.push_back(v.kind == asj::Value::Number ? v.num : (v.kind == asj::Value::Bool ? (v.b ? 1.0 : 0.0) : double(k)));
      F.str.push_back(v.kind == asj::Value::String ? v.str : std::string());
    }
    F.dflt = 0;
    if (const asj::Value* dv = f.get("default")) {
      int found = -1;
      for (int k = 0; k < F.n && found < 0; ++k) {
        const asj::Value& v = dom->arr[k];
        if (v.kind != dv->kind) continue;
        if ((v.kind == asj::Value::Number && v.num == dv->num) || (v.kind == asj::Value::Bool && v.b == dv->b) ||
            (v.kind == asj::Value::String && v.str == dv->str))
          found = k;
      }
      if (found < 0) return err(E_SCHEMA, "feature " + F.name + ": default not in domain (SPEC.md:30)");
      F.dflt = found;
    }
    if (const asj::Value* rq = f.get("requires")) {
      for (const asj::Value& a : rq->arr) {
        int ref = idx[a.get("feature")->str];
        if (ref >= i) return err(E_ORDER, "feature " + F.name + " requires a later feature (SPEC.md:30)");
        const asj::Value* op = a.get("op");
        const asj::Value* val = a.get("value");
        if (!op || op->kind != asj::Value::String || !val) return err(E_SCHEMA, "requires atom needs op and value");
        Atom at;
        Status st = make_atom(S, ref, op->str, *val, at);
        if (!st.ok()) return st;
        F.req.push_back(at);
      }
    }
  }
  // raw mixed radix
  S.stride[S.d - 1] = 1;
  for (int j = S.d - 2; j >= 0; --j) {
    unsigned __int128 s = static_cast<unsigned __int128>(S.stride[j + 1]) * S.feat[j + 1].n;
    if (s > (static_cast<unsigned __int128>(1) << 63)) return err(E_SCHEMA, "raw index range exceeds 2^63");
    S.stride[j] = static_cast<uint64_t>(s);
  }
  {
    unsigned __int128 nr = static_cast<unsigned __int128>(S.stride[0]) * S.feat[0].n;
    if (nr > (static_cast<unsigned __int128>(1) << 63)) return err(E_SCHEMA, "raw index range exceeds 2^63");
    S.n_raw = static_cast<uint64_t>(nr);
  }

  // ---------------------------------------------------------------- hardware / model
  const asj::Value* hw = doc.get("hardware");
  const asj::Value* model = doc.get("model");
  if (!hw || hw->kind != asj::Value::Object) return err(E_SCHEMA, "missing hardware object");
  const asj::Value* devs = hw->get("devices");
  if (!devs || devs->kind != asj::Value::Array || devs->arr.empty()) return err(E_SCHEMA, "hardware.devices must be a non-empty array");
  struct Cls { int count; double cap, eff; };
  std::vector<Cls> cls;
  S.G = 0;
  for (const asj::Value& c : devs->arr) {
    const asj::Value *cnt = c.get("count"), *mem = c.get("mem_gb"), *rel = c.get("rel_throughput");
    if (!cnt || !mem || !rel) return err(E_SCHEMA, "device class needs count, mem_gb, rel_throughput");
    cls.push_back({static_cast<int>(cnt->num), mem->num * 1e9, rel->num});
    S.G += cnt->num;
  }
  if (cls.size() > static_cast<size_t>(MAX_CLS)) return err(E_CAP, "more than 4 device classes");
  std::stable_sort(cls.begin(), cls.end(), [](const Cls& a, const Cls& b) { return a.eff > b.eff; });

  // ---------------------------------------------------------------- constraints
  std::vector<int> cref;  // features referenced by constraints
  if (const asj::Value* cs = doc.get("constraints")) {
    for (const asj::Value& c : cs->arr) {
      const asj::Value* t = c.get("type");
      if (!t || t->kind != asj::Value::String) return err(E_SCHEMA, "constraint needs a type");
      ConstraintH C;
      auto fidx = [&](const asj::Value* v, int& out) -> Status {
        if (!v || v->kind != asj::Value::String || feature_index(S, v->str) < 0)
          return err(E_SCHEMA, "constraint references an unknown feature");
        out = feature_index(S, v->str);
        return Status{};
      };
      auto flist = [&](const asj::Value* v) -> Status {
        if (!v || v->kind != asj::Value::Array) return err(E_SCHEMA, "constraint features must be an array");
        for (const asj::Value& x : v->arr) {
          int i;
          Status st = fidx(&x, i);
          if (!st.ok()) return st;
          C.f.push_back(i);
        }
        return Status{};
      };
      auto cst = [&](const asj::Value* v, double& out) -> Status {
        if (!v || v->kind != asj::Value::String) return err(E_SCHEMA, "constraint const must be a name");
        if (v->str == "G") { out = S.G; return Status{}; }
        bool found;
        out = model_const(model, v->str, 0, &found);
        if (!found) return err(E_SCHEMA, "unknown model constant " + v->str);
        return Status{};
      };
      auto atoms = [&](const asj::Value* v, std::vector<Atom>& out) -> Status {
        if (!v || v->kind != asj::Value::Array) return err(E_SCHEMA, "implies needs atom arrays");
        for (const asj::Value& a : v->arr) {
          int r;
          Status st = fidx(a.get("feature"), r);
          if (!st.ok()) return st;
          const asj::Value* op = a.get("op");
          const asj::Value* val = a.get("value");
          if (!op || !val) return err(E_SCHEMA, "atom needs op and value");
          Atom at;
          st = make_atom(S, r, op->str, *val, at);
          if (!st.ok()) return st;
          out.push_back(at);
        }
        return Status{};
      };
      Status st;
      const std::string& ty = t->str;
      if (ty == "product_eq_devices") { C.type = C_PROD_EQ_DEV; st = flist(c.get("features")); }
      else if (ty == "product_le_devices_pow2") {
        C.type = C_PROD_LE_DEV_POW2; st = flist(c.get("features"));
        if (const asj::Value* dd = c.get("divides_devices")) C.divides_devices = dd->kind == asj::Value::Bool && dd->b;
      } else if (ty == "divides") {
        C.type = C_DIVIDES; st = fidx(c.get("a"), C.a);
        if (st.ok()) st = fidx(c.get("b"), C.b);
      } else if (ty == "divides_const") { C.type = C_DIVIDES_CONST; st = flist(c.get("features")); if (st.ok()) st = cst(c.get("const"), C.cval); }
      else if (ty == "gbs_divisible") {
        C.type = C_GBS_DIV; st = flist(c.get("features"));
        bool f; C.cval = model_const(model, "GBS", 0, &f);
        if (st.ok() && !f) st = err(E_SCHEMA, "gbs_divisible needs model.GBS");
      } else if (ty == "seq_divisible_2cp") {
        C.type = C_SEQ_2CP; st = fidx(c.get("feature"), C.a);
        bool f; C.cval = model_const(model, "S", 0, &f);
        if (st.ok() && !f) st = err(E_SCHEMA, "seq_divisible_2cp needs model.S");
      } else if (ty == "ge") {
        C.type = C_GE; st = fidx(c.get("a"), C.a);
        if (st.ok()) st = fidx(c.get("b"), C.b);
      } else if (ty == "le_const_div") {
        C.type = C_LE_CONST_DIV; st = fidx(c.get("feature"), C.a);
        if (st.ok()) st = flist(c.get("div"));
        if (st.ok()) st = cst(c.get("const"), C.cval);
      } else if (ty == "microbatch_divisible_pp") {
        C.type = C_MB_DIV_PP;
        for (const char* k : {"vpp", "pp", "dp", "mbs"}) {
          int i;
          if (st.ok()) st = fidx(c.get(k), i);
          if (st.ok()) C.f.push_back(i);
        }
        bool f; C.cval = model_const(model, "GBS", 0, &f);
        if (st.ok() && !f) st = err(E_SCHEMA, "microbatch_divisible_pp needs model.GBS");
      } else if (ty == "implies") {
        C.type = C_IMPLIES; st = atoms(c.get("if"), C.iff);
        if (st.ok()) st = atoms(c.get("then"), C.then);
      } else {
        return err(E_SCHEMA, "unknown constraint type " + ty);
      }
      if (!st.ok()) return st;
      std::vector<int> refs = C.f;
      if (C.a >= 0) refs.push_back(C.a);
      if (C.b >= 0) refs.push_back(C.b);
      for (const Atom& a : C.iff) refs.push_back(a.ref);
      for (const Atom& a : C.then) refs.push_back(a.ref);
      C.last = refs.empty() ? 0 : *std::max_element(refs.begin(), refs.end());
      cref.insert(cref.end(), refs.begin(), refs.end());
      S.cons.push_back(C);
    }
  }

  // ---------------------------------------------------------------- structural prefix (R4)
  // smallest declaration-order prefix holding every constraint-referenced feature and, transitively,
  // every feature its activation predicates reference.
  {
    std::vector<bool> need(S.d, false);
    std::vector<int> stack(cref.begin(), cref.end());
    while (!stack.empty()) {
      int f = stack.back();
      stack.pop_back();
      if (need[f]) continue;
      need[f] = true;
      for (const Atom& a : S.feat[f].req) stack.push_back(a.ref);
    }
    S.n_prefix = 0;
    for (int j = 0; j < S.d; ++j)
      if (need[j]) S.n_prefix = j + 1;
  }
  // tail gating groups: connected components of gate edges among tail features; each must be a
  // contiguous run of features so the CVI order stays the raw order.
  {
    std::vector<int> par(S.d);
    std::iota(par.begin(), par.end(), 0);
    std::function<int(int)> find = [&](int x) { return par[x] == x ? x : par[x] = find(par[x]); };
    for (int j = S.n_prefix; j < S.d; ++j)
      for (const Atom& a : S.feat[j].req)
        if (a.ref >= S.n_prefix) par[find(j)] = find(a.ref);
    int j = S.n_prefix;
    while (j < S.d) {
      int r = find(j), e = j;
      while (e + 1 < S.d && find(e + 1) == r) ++e;
      for (int q = e + 1; q < S.d; ++q)
        if (find(q) == r) return err(E_ORDER, "tail gating group of " + S.feat[j].name + " is not contiguous");
      if (e - j + 1 > TUPW) return err(E_CAP, "tail gating group wider than 8 features");
      S.comp_first.push_back(j);
      S.comp_width.push_back(e - j + 1);
      j = e + 1;
    }
  }
  const int n_comp = static_cast<int>(S.comp_first.size());
  S.tail_span = S.n_prefix > 0 ? S.stride[S.n_prefix - 1] : S.n_raw;

  // ---------------------------------------------------------------- enumerate structures
  {
    int dig[DMAX] = {0};
    bool act[DMAX] = {false};
    std::map<std::vector<uint64_t>, uint32_t> list_cache;
    uint64_t acc = 0;
    Status failure;
    std::function<void(int)> rec_prefix;
    std::function<void(int, int, int, std::vector<Tuple>&)> rec_comp;
    rec_comp = [&](int c, int j, int end, std::vector<Tuple>& out) {
      if (j == end) {
        Tuple t{};
        for (int q = S.comp_first[c]; q < end; ++q) {
          dv_set(t.dv, q, static_cast<uint32_t>(dig[q]));
          t.raw += static_cast<uint64_t>(dig[q]) * S.stride[q];
          if (act[q]) t.act |= (1u << q);
        }
        out.push_back(t);
        return;
      }
      const FeatureH& F = S.feat[j];
      for (int v = 0; v < F.n; ++v) {
        dig[j] = v;
        bool a = true;
        for (const Atom& at : F.req)
          if (!act[at.ref] || !((at.allowed >> dig[at.ref]) & 1ull)) { a = false; break; }
        act[j] = a;
        if (!a && v != F.dflt) continue;  // G1
        rec_comp(c, j + 1, end, out);
      }
      dig[j] = S.feat[j].dflt;
    };
    rec_prefix = [&](int j) {
      if (!failure.ok()) return;
      if (j == S.n_prefix) {
        DV dv{};
        uint64_t raw = 0;
        for (int q = 0; q < S.n_prefix; ++q) {
          dv_set(dv, q, static_cast<uint32_t>(dig[q]));
          raw += static_cast<uint64_t>(dig[q]) * S.stride[q];
        }
        uint32_t ab = 0;
        for (int q = 0; q < S.n_prefix; ++q)
          if (act[q]) ab |= (1u << q);
        uint64_t tail = 1;
        for (int c = 0; c < n_comp; ++c) {
          std::vector<Tuple> lst;
          rec_comp(c, S.comp_first[c], S.comp_first[c] + S.comp_width[c], lst);
          std::vector<uint64_t> key;
          for (const Tuple& t : lst) { key.push_back(t.raw); key.push_back(t.act); }
          auto it = list_cache.find(key);
          uint32_t off;
          if (it == list_cache.end()) {
            off = static_cast<uint32_t>(S.tuples.size());
            S.tuples.insert(S.tuples.end(), lst.begin(), lst.end());
            list_cache[key] = off;
          } else {
            off = it->second;
          }
          S.s_off.push_back(off);
          S.s_cnt.push_back(static_cast<uint32_t>(lst.size()));
          tail *= lst.size();
        }
        if (tail >= (1ull << 32)) { failure = err(E_CAP, "a structure has >= 2^32 valid tails"); return; }
        S.prefix.push_back(acc);
        S.s_raw.push_back(raw);
        S.s_act.push_back(ab);
        S.s_dv.push_back(dv);
        acc += tail;
        return;
      }
      const FeatureH& F = S.feat[j];
      for (int v = 0; v < F.n; ++v) {
        dig[j] = v;
        bool a = true;
        for (const Atom& at : F.req)
          if (!act[at.ref] || !((at.allowed >> dig[at.ref]) & 1ull)) { a = false; break; }
        act[j] = a;
        if (!a && v != F.dflt) continue;  // G1
        bool ok = true;
        for (const ConstraintH& c : S.cons)
          if (c.last == j && !constraint_ok(S, c, dig, act)) { ok = false; break; }
        if (!ok) continue;
        rec_prefix(j + 1);
      }
      dig[j] = 0;
    };
    rec_prefix(0);
    if (!failure.ok()) return failure;
    S.n_struct = static_cast<int>(S.s_raw.size());
    S.prefix.push_back(acc);
    S.n_cvi = acc;
    if (S.n_cvi == 0) return err(E_EMPTY, "no configuration satisfies the constraints (SPEC.md:34)");
    if (S.n_cvi >= (1ull << 32)) return err(E_CAP, "n_cvi >= 2^32");
  }

  // ---------------------------------------------------------------- simulator binding
  const asj::Value* sm = doc.get("sim_mode");
  std::string mode = (sm && sm->kind == asj::Value::String) ? sm->str : "spec";
  SimParams& P = S.sim;
  P.mode = mode == "spec" ? 0 : (mode == "derived" ? 1 : (mode == "serve" ? 2 : -1));
  if (P.mode < 0) return err(E_SCHEMA, "sim_mode must be spec|derived|serve");
  static const char* train_names[NKNOB] = {"pp", "vpp", "tp", "dp", "cp", "ep", "mbs", "ar", "arl", "sp", "tpov",
                                           "tp_comm", "dopt", "ovg", "ovp", "ddp_bucket", "ddp", "disp",
                                           nullptr, nullptr, nullptr, nullptr};
  static const double neutral[NKNOB] = {1, 1, 1, 1, 1, 1, 1, 0, 1, 0, 0, 0, 0, 0, 0, 4, 1, 0, 1, 0, 1, 0.9};
  for (int k = 0; k < NKNOB; ++k) {
    P.neutral[k] = neutral[k];
    P.kf[k] = -1;
    const char* nm = nullptr;
    if (P.mode != 2) nm = train_names[k];
    else if (k == K_TP) nm = "tp";
    else if (k == K_NS) nm = "max_num_seqs";
    else if (k == K_CPF) nm = "cpf";
    else if (k == K_MBT) nm = "mbt";
    else if (k == K_U) nm = "u";
    if (nm) P.kf[k] = feature_index(S, nm);
    const int f = P.kf[k] >= 0 ? P.kf[k] : 0;
    P.kw[k] = f >> 3;
    P.ks[k] = (f & 7) * 8;
    P.ko[k] = f * VMAX;
    P.kbit[k] = P.kf[k] >= 0 ? (1u << f) : 0u;
  }
  S.val.assign(static_cast<size_t>(S.d) * VMAX, 0.0);
  for (int j = 0; j < S.d; ++j) {
    const FeatureH& F = S.feat[j];
    for (int v = 0; v < F.n; ++v) {
      double x = F.num[v];
      if (j == P.kf[K_AR]) {
        if (F.vkind == 1) x = F.num[v] != 0.0 ? 2.0 : 0.0;
        else if (F.vkind == 2) {
          if (F.str[v] == "none") x = 0;
          else if (F.str[v] == "sel") x = 1;
          else if (F.str[v] == "full") x = 2;
          else return err(E_SCHEMA, "ar values must be bool or none|sel|full");
        }
      } else if (j == P.kf[K_DISP] && F.vkind == 2) {
        if (F.str[v] == "alltoall") x = 0;
        else if (F.str[v] == "allgather") x = 1;
        else return err(E_SCHEMA, "disp values must be alltoall|allgather");
      }
      S.val[j * VMAX + v] = x;
    }
  }
  S.inv.assign(S.val.size(), 0.0);
  S.lg2.assign(S.val.size(), 0.0);
  for (size_t i = 0; i < S.val.size(); ++i) {
    const double x = S.val[i];
    S.inv[i] = x != 0.0 ? 1.0 / x : 0.0;
    S.lg2[i] = x > 0.0 ? std::log2(x) : 0.0;
  }
  P.n_cls = static_cast<int>(cls.size());
  for (int i = 0; i < P.n_cls; ++i) {
    P.cls_count[i] = cls[i].count;
    P.cls_cap[i] = cls[i].cap;
    P.cls_eff[i] = cls[i].eff;
  }
  auto mc = [&](const char* k, double d) { return model_const(model, k, d); };
  auto hc = [&](const char* k, double d) { return model_const(hw, k, d); };
  P.F_work = mc("F_work", 100); P.alpha_tp = mc("alpha_tp", 2.0); P.alpha_dp = mc("alpha_dp", 1.5);
  P.r_ar = mc("r_ar", 1.33); P.B = mc("B", 64); P.P_mem = mc("P_mem", 0); P.A_mem = mc("A_mem", 0);
  P.L = mc("L", 1); P.h = mc("h", 1); P.a = mc("a", 1); P.kv = mc("kv", 1); P.S = mc("S", 1);
  P.GBS = mc("GBS", 1); P.P = mc("P", 0); P.P_exp = mc("P_exp", 0); P.E = mc("E", 1); P.topk = mc("topk", 1);
  P.dh = mc("dh", 128); P.ffn = mc("ffn", 0); P.P_in = mc("P_in", 1); P.P_out = mc("P_out", 1);
  P.mml = mc("max_model_len", 1); P.w_tpot = mc("w_tpot", 0.5);
  P.peak = hc("peak_flops", 312e12); P.mfu0 = hc("mfu0", 0.5); P.bw_intra = hc("bw_intra", 240e9);
  P.bw_inter = hc("bw_inter", 25e9); P.gpn = hc("gpus_per_node", 8); P.n_sm = hc("n_sm", 108);
  P.bw_hbm = hc("bw_hbm", 2.039e12);
  P.G = S.G;
  P.inv_B = 1.0 / P.B;
  P.inv_GBS = 1.0 / P.GBS;
  P.inv_bw_intra = 1.0 / P.bw_intra;
  P.inv_bw_inter = 1.0 / P.bw_inter;
  P.half_inv_nsm = 0.5 / P.n_sm;
  {
    const double P_act = P.P - P.P_exp + P.P_exp * P.topk / P.E;
    P.T_work = P.GBS * P.S * (6.0 * P_act + 12.0 * P.L * P.h * P.S) / (P.peak * P.mfu0);
  }
  P.C_tp = 16.0 * P.L * P.GBS * P.S * P.h;
  P.C_ep = 8.0 * P.topk * P.L * P.GBS * P.S * P.h;
  P.C_cp = 0.5 * 12.0 * P.L * P.GBS * P.S * P.kv * (P.h / P.a);
  for (int k = 0; k < NKNOB; ++k) {
    P.neutral_inv[k] = P.neutral[k] != 0.0 ? 1.0 / P.neutral[k] : 0.0;
    P.neutral_lg2[k] = P.neutral[k] > 0.0 ? std::log2(P.neutral[k]) : 0.0;
  }

  // ---------------------------------------------------------------- GP hyper-parameters + features
  const asj::Value* gp = doc.get("gp");
  S.ls.assign(S.d, 1.0);
  if (gp) {
    if (const asj::Value* k = gp->get("kernel")) {
      if (k->str == "matern52") S.kernel = 0;
      else if (k->str == "rbf") S.kernel = 1;
      else return err(E_SCHEMA, "gp.kernel must be matern52|rbf");
    }
    if (const asj::Value* l = gp->get("lengthscale")) {
      if (l->kind == asj::Value::Number) S.ls.assign(S.d, l->num);
      else if (l->kind == asj::Value::Array && static_cast<int>(l->arr.size()) == S.d)
        for (int j = 0; j < S.d; ++j) S.ls[j] = l->arr[j].num;
      else return err(E_SCHEMA, "gp.lengthscale must be a number or an array of d numbers");
    }
    S.sf2 = model_const(gp, "sf2", 0.1);
    S.sn2 = model_const(gp, "sn2", 1e-3);
    S.xi = model_const(gp, "xi", 0.0);
    S.kappa = model_const(gp, "kappa", 2.0);
    if (const asj::Value* w = gp->get("onehot_max_width")) {
      if (w->kind != asj::Value::Number || !(w->num >= 0) || w->num != static_cast<int>(w->num))
        return err(E_SCHEMA, "gp.onehot_max_width must be a non-negative integer");
      S.onehot_max = static_cast<int>(w->num);
    }
    if (const asj::Value* pr = gp->get("prior")) {
      if (pr->kind != asj::Value::String || (pr->str != "sim" && pr->str != "ensemble"))
        return err(E_SCHEMA, "gp.prior must be sim|ensemble");
      S.prior = pr->str == "ensemble" ? 1 : 0;
    }
    if (const asj::Value* es = gp->get("ensemble_seed")) {
      if (es->kind != asj::Value::Number || !(es->num >= 0) || es->num != std::floor(es->num))
        return err(E_SCHEMA, "gp.ensemble_seed must be a non-negative integer");
      S.ens_seed = static_cast<uint64_t>(es->num);
    }
  }
  for (double l : S.ls)
    if (!(l > 0)) return err(E_SCHEMA, "gp.lengthscale must be positive");
  if (!(S.sf2 > 0) || !(S.sn2 > 0)) return err(E_SCHEMA, "gp.sf2 and gp.sn2 must be positive");
  feature_tables(S);
  return Status{};
}

void feature_tables(HostSpace& S) {
  S.xt64.assign(static_cast<size_t>(S.d) * VMAX, 0.0);
  S.xt32.assign(static_cast<size_t>(S.d) * VMAX, 0.0f);
  for (int j = 0; j < S.d; ++j)
    for (int v = 0; v < S.feat[j].n; ++v) {
      const double phi = S.feat[j].n > 1 ? double(v) / double(S.feat[j].n - 1) : 0.0;
      S.xt64[j * VMAX + v] = phi / S.ls[j];
      S.xt32[j * VMAX + v] = static_cast<float>(phi / S.ls[j]);
    }
}

bool cvi_decode(const HostSpace& S, uint64_t p, DV& dv, uint32_t& act, uint64_t& raw) {
  if (p >= S.n_cvi) return false;
  int lo = 0, hi = S.n_struct;
  while (hi - lo > 1) {
    int mid = (lo + hi) / 2;
    if (S.prefix[mid] <= p) lo = mid; else hi = mid;
  }
  const int n_comp = static_cast<int>(S.comp_first.size());
  uint64_t t = p - S.prefix[lo];
  dv = S.s_dv[lo];
  act = S.s_act[lo];
  raw = S.s_raw[lo];
  for (int c = n_comp - 1; c >= 0; --c) {
    const uint32_t off = S.s_off[static_cast<size_t>(lo) * n_comp + c], cnt = S.s_cnt[static_cast<size_t>(lo) * n_comp + c];
    const Tuple& tu = S.tuples[off + t % cnt];
    t /= cnt;
    dv.w[0] |= tu.dv.w[0]; dv.w[1] |= tu.dv.w[1]; dv.w[2] |= tu.dv.w[2];
    act |= tu.act;
    raw += tu.raw;
  }
  return true;
}

// Number of CVI members with raw index < raw (raw <= n_raw), and whether raw itself is a member.
// The CVI is ascending raw order (R4); the structural prefix is the most significant digit block,
// so members below raw are: every member of a structure whose prefix raw part is smaller, plus,
// inside the structure with an equal prefix, the tail combinations that compare lower group by
// group (tail groups are contiguous digit blocks, the earlier group more significant).
uint64_t cvi_rank(const HostSpace& S, uint64_t raw, bool* member) {
  if (member) *member = false;
  if (raw >= S.n_raw) return S.n_cvi;
  const uint64_t raw_p = raw - raw % S.tail_span, raw_t = raw % S.tail_span;
  const size_t i = static_cast<size_t>(std::lower_bound(S.s_raw.begin(), S.s_raw.end(), raw_p) - S.s_raw.begin());
  uint64_t r = S.prefix[i];
  if (i == static_cast<size_t>(S.n_struct) || S.s_raw[i] != raw_p) return r;
  const int n_comp = static_cast<int>(S.comp_first.size());
  for (int c = 0; c < n_comp; ++c) {
    // raw contribution of group c's digits in raw_t
    uint64_t contrib = 0;
    for (int f = S.comp_first[c]; f < S.comp_first[c] + S.comp_width[c]; ++f)
      contrib += ((raw_t / S.stride[f]) % S.feat[f].n) * S.stride[f];
    const uint32_t off = S.s_off[i * n_comp + c], cnt = S.s_cnt[i * n_comp + c];
    const Tuple* b = S.tuples.data() + off;
    const Tuple* e = b + cnt;
    const Tuple* lb = std::lower_bound(b, e, contrib, [](const Tuple& t, uint64_t v) { return t.raw < v; });
    uint64_t mult = 1;
    for (int h = c + 1; h < n_comp; ++h) mult *= S.s_cnt[i * n_comp + h];
    r += static_cast<uint64_t>(lb - b) * mult;
    if (lb == e || lb->raw != contrib) return r;
  }
  if (member) *member = true;
  return r;
}

bool raw_decode(const HostSpace& S, uint64_t raw, int* dig, DV& dv, uint32_t& act, bool& structural) {
  if (raw >= S.n_raw) return false;
  for (int j = 0; j < S.d; ++j) dig[j] = static_cast<int>((raw / S.stride[j]) % S.feat[j].n);
  bool a[DMAX];
  activity(S, dig, a);
  structural = true;
  for (int j = 0; j < S.d; ++j)
    if (!a[j] && dig[j] != S.feat[j].dflt) structural = false;
  for (const ConstraintH& c : S.cons)
    if (!constraint_ok(S, c, dig, a)) structural = false;
  dv_from_digits(S, dig, dv);
  act = act_bits(S, a);
  return true;
}

void simulate_host(const HostSpace& S, const DV& dv, uint32_t act, double& cost, bool& ok, double& mem) {
  Knobs k;
  load_knobs(S.sim, S.val.data(), S.inv.data(), S.lg2.data(), dv, act, k);
  simulate(S.sim, k, cost, ok, mem);
}

// ---------------------------------------------------------------- regression-simulator ensemble
// NEXT-1; Appendix B Table 2 + weight equation, SPEC.md
// fit_simulator / ensemble_predict; readings R20.
namespace {
const char* const kTable2[4][9] = {
    {"a100", "a40", "mbs", "tp", "pp", "dp", nullptr},                       // 3D-Parallelism
    {"a100", "a40", "mbs", "tp", "pp", "dp", "ep", "cp", "sp"},              // 5D-Parallelism
    {"a100", "a40", "mbs", "tp", "pp", "dp", "ddp_optim", nullptr},          // DDP-Aware
    {"a100", "a40", "mbs", "tp", "pp", "dp", "ar", "tp_comm", nullptr},      // Communication-Aware
};

std::vector<int> table2_columns(const HostSpace& S, int m) {
  std::vector<int> cols;
  for (int k = 0; k < 9 && kTable2[m][k]; ++k) {
    const std::string knob = kTable2[m][k];
    int f = -1;
    if (knob == "ddp_optim") {
      f = feature_index(S, "dopt");
      if (f < 0) f = feature_index(S, "ddp");
    } else {
      f = feature_index(S, knob);
    }
    if (f >= 0 && std::find(cols.begin(), cols.end(), f) == cols.end()) cols.push_back(f);
  }
  std::sort(cols.begin(), cols.end());
  return cols;
}

// (Z^T Z + 1e-6 I) g = Z^T (y - ybar) on standardised, non-constant columns (Cholesky)
void ridge_fit(const std::vector<std::vector<double>>& X, const std::vector<double>& y, double& beta0,
               std::vector<double>& beta) {
  const size_t n = y.size(), p = X.empty() ? 0 : X[0].size();
  double ybar = 0.0;
  for (double v : y) ybar += v;
  ybar /= static_cast<double>(n);
  beta.assign(p, 0.0);
  std::vector<double> mu(p, 0.0), sd(p, 0.0);
  std::vector<int> keep;
  for (size_t j = 0; j < p; ++j) {
    for (size_t i = 0; i < n; ++i) mu[j] += X[i][j];
    mu[j] /= static_cast<double>(n);
    for (size_t i = 0; i < n; ++i) sd[j] += (X[i][j] - mu[j]) * (X[i][j] - mu[j]);
    sd[j] = std::sqrt(sd[j] / static_cast<double>(n));
    if (sd[j] > 1e-9 * std::fmax(1.0, std::fabs(mu[j]))) keep.push_back(static_cast<int>(j));
  }
  const size_t q = keep.size();
  if (q > 0) {
    std::vector<double> A(q * q, 0.0), r(q, 0.0);
    for (size_t a = 0; a < q; ++a) {
      for (size_t b = 0; b <= a; ++b) {
        double acc = 0.0;
        for (size_t i = 0; i < n; ++i)
          acc += (X[i][keep[a]] - mu[keep[a]]) / sd[keep[a]] * ((X[i][keep[b]] - mu[keep[b]]) / sd[keep[b]]);
        A[a * q + b] = A[b * q + a] = acc;
      }
      A[a * q + a] += 1e-6;
      for (size_t i = 0; i < n; ++i) r[a] += (X[i][keep[a]] - mu[keep[a]]) / sd[keep[a]] * (y[i] - ybar);
    }
    for (size_t a = 0; a < q; ++a) {          // Cholesky A = L L^T in place (lower)
      for (size_t b = 0; b <= a; ++b) {
        double acc = A[a * q + b];
        for (size_t c = 0; c < b; ++c) acc -= A[a * q + c] * A[b * q + c];
        A[a * q + b] = (a == b) ? std::sqrt(acc) : acc / A[b * q + b];
      }
    }
    std::vector<double> g(q);
    for (size_t a = 0; a < q; ++a) {          // L z = r
      double acc = r[a];
      for (size_t c = 0; c < a; ++c) acc -= A[a * q + c] * g[c];
      g[a] = acc / A[a * q + a];
    }
    for (size_t a = q; a-- > 0;) {            // L^T g = z
      double acc = g[a];
      for (size_t c = a + 1; c < q; ++c) acc -= A[c * q + a] * g[c];
      g[a] = acc / A[a * q + a];
    }
    for (size_t a = 0; a < q; ++a) beta[keep[a]] = g[a] / sd[keep[a]];
  }
  beta0 = ybar;
  for (size_t j = 0; j < p; ++j) beta0 -= beta[j] * mu[j];
}
}  // namespace

void ensemble_fit(const HostSpace& S, const std::vector<DV>& dv, const std::vector<double>& cost, EnsembleFit& e) {
  e = EnsembleFit{};
  const int n = static_cast<int>(dv.size());
  if (n == 0) return;
  std::vector<double> y(n);
  for (int i = 0; i < n; ++i) y[i] = std::log(cost[i]);
  // seeded 80/20 split: holdout = the floor(n/5) (>= 1) smallest splitmix64(seed ^ 0xE45E ^ i)
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    return splitmix64(S.ens_seed ^ 0xE45Eull ^ static_cast<uint64_t>(a)) <
           splitmix64(S.ens_seed ^ 0xE45Eull ^ static_cast<uint64_t>(b));
  });
  const int nh = std::max(1, n / 5);
  std::vector<int> hold(order.begin(), order.begin() + std::min(nh, n)), train(order.begin() + std::min(nh, n), order.end());
  std::sort(hold.begin(), hold.end());
  std::sort(train.begin(), train.end());
  auto x_of = [&](int i, int f) { return S.feat[f].num[dv_get(dv[i], f)]; };
  double w_tot = 0.0;
  std::vector<std::vector<double>> coef(4, std::vector<double>(S.d, 0.0));
  double b0s[4] = {0, 0, 0, 0};
  for (int m = 0; m < 4; ++m) {
    const std::vector<int> cols = table2_columns(S, m);
    e.r2[m] = -INFINITY;
    if (static_cast<int>(train.size()) < static_cast<int>(cols.size()) + 2 || hold.empty()) continue;
    std::vector<std::vector<double>> X(train.size(), std::vector<double>(cols.size()));
    std::vector<double> yt(train.size());
    for (size_t i = 0; i < train.size(); ++i) {
      for (size_t j = 0; j < cols.size(); ++j) X[i][j] = x_of(train[i], cols[j]);
      yt[i] = y[train[i]];
    }
    double b0;
    std::vector<double> b;
    ridge_fit(X, yt, b0, b);
    // R^2 on the holdout; zero variance -> 0
    double ym = 0.0, yy = 0.0;
    for (int i : hold) {
      ym += y[i];
      yy += y[i] * y[i];
    }
    ym /= static_cast<double>(hold.size());
    double sst = 0.0, ssr = 0.0;
    for (int i : hold) {
      double yh = b0;
      for (size_t j = 0; j < cols.size(); ++j) yh += b[j] * x_of(i, cols[j]);
      sst += (y[i] - ym) * (y[i] - ym);
      ssr += (y[i] - yh) * (y[i] - yh);
    }
    e.r2[m] = (sst <= 1e-24 * yy) ? 0.0 : 1.0 - ssr / sst;
    b0s[m] = b0;
    for (size_t j = 0; j < cols.size(); ++j) coef[m][cols[j]] = b[j];
    w_tot += std::fmax(0.0, e.r2[m]);
  }
  if (!(w_tot > 0.0)) return;   // Unavailable: the prior stays ln cost_sim
  e.on = true;
  e.c0 = 0.0;
  std::vector<double> cf(S.d, 0.0);
  for (int m = 0; m < 4; ++m) {
    e.w[m] = std::fmax(0.0, e.r2[m]) / w_tot;
    e.c0 += e.w[m] * b0s[m];
    for (int f = 0; f < S.d; ++f) cf[f] += e.w[m] * coef[m][f];
  }
  e.tab.assign(static_cast<size_t>(S.d) * VMAX, 0.0);
  for (int f = 0; f < S.d; ++f)
    for (int v = 0; v < S.feat[f].n; ++v) e.tab[static_cast<size_t>(f) * VMAX + v] = cf[f] * S.feat[f].num[v];
}

double ensemble_m0(const HostSpace& S, const EnsembleFit& e, const DV& dv) {
  double m = e.c0;
  for (int f = 0; f < S.d; ++f) m += e.tab[static_cast<size_t>(f) * VMAX + dv_get(dv, f)];
  return m;
}

Status gp_fit(const HostSpace& S, const std::vector<DV>& obs_dv, const std::vector<uint32_t>& obs_act,
              const std::vector<double>& cost, const std::vector<double>& cost_sim, GPFit& fit,
              const std::vector<double>* m0_prior) {
  (void)obs_act;
  const int M = static_cast<int>(obs_dv.size());
  const int d = S.d;
  fit = GPFit{};
  fit.M = M;
  if (M == 0) return Status{};
  fit.X.resize(static_cast<size_t>(M) * d);
  std::vector<double> y(M), m0(M), r(M);
  for (int i = 0; i < M; ++i) {
    for (int j = 0; j < d; ++j) fit.X[i * d + j] = S.xt64[j * VMAX + dv_get(obs_dv[i], j)];
    y[i] = std::log(cost[i]);
    m0[i] = m0_prior ? (*m0_prior)[i] : std::log(cost_sim[i]);
  }
  double sum = 0.0;
  for (int i = 0; i < M; ++i) sum += y[i] - m0[i];
  fit.b = sum / M;
  fit.fstar = INFINITY;
  for (int i = 0; i < M; ++i) {
    r[i] = (y[i] - m0[i]) - fit.b;
    fit.fstar = std::fmin(fit.fstar, y[i]);
  }
  fit.r = r;
  // K = k(o_i, o_j) + sn2 I ; Cholesky K = L L^T.  Host threads (host_pool.hpp): every element is
  // computed by one task with the operations and order of the sequential loops, so the fit does not
  // depend on the thread count.
  HostPool& pool = HostPool::get();
  const bool par = M >= 128;  // below, the whole fit takes tens of microseconds: no thread wake-ups
  std::vector<double> L(static_cast<size_t>(M) * M, 0.0);
  pool.run(M, [&](int i) {
    for (int j = 0; j <= i; ++j) {
      double r2 = 0.0;
      for (int q = 0; q < d; ++q) {
        const double df = fit.X[i * d + q] - fit.X[j * d + q];
        r2 += df * df;
      }
      L[i * M + j] = kernel64(S.kernel, S.sf2, r2) + (i == j ? S.sn2 : 0.0);
    }
  }, par);
  // Right-looking Cholesky in column blocks of CB: factor the diagonal block, then the panel below
  // it (rows in parallel), then the trailing update A[i][j] -= L[i][q] L[j][q] for the block's q
  // (rows in parallel).  Each element still receives its updates in ascending q (the textbook
  // left-looking order), so the factor is identical to the unblocked loop; rows run unit-stride over
  // j through Lt = L^T.
  std::vector<double> Lt(static_cast<size_t>(M) * M, 0.0);
  constexpr int CB = 32;
  bool pd = true;
  for (int k0 = 0; k0 < M && pd; k0 += CB) {
    const int k1 = std::min(M, k0 + CB);
    for (int q = k0; q < k1; ++q) {          // diagonal block, sequential
      const double sq = L[q * M + q];
      if (!(sq > 0.0)) {
        pd = false;
        break;
      }
      const double lqq = std::sqrt(sq);
      L[q * M + q] = lqq;
      Lt[static_cast<size_t>(q) * M + q] = lqq;
      for (int i = q + 1; i < k1; ++i) {
        L[i * M + q] /= lqq;
        Lt[static_cast<size_t>(q) * M + i] = L[i * M + q];
      }
      const double* lq = Lt.data() + static_cast<size_t>(q) * M;
      for (int i = q + 1; i < k1; ++i) {
        const double liq = L[i * M + q];
        double* ai = L.data() + static_cast<size_t>(i) * M;
        for (int j = q + 1; j <= i; ++j) ai[j] -= liq * lq[j];
      }
    }
    if (!pd || k1 == M) break;
    pool.run(M - k1, [&](int t) {           // panel rows i >= k1: columns [k0, k1)
      const int i = k1 + t;
      double* ai = L.data() + static_cast<size_t>(i) * M;
      for (int q = k0; q < k1; ++q) {
        ai[q] /= L[q * M + q];
        Lt[static_cast<size_t>(q) * M + i] = ai[q];
        const double liq = ai[q];
        const double* lq = Lt.data() + static_cast<size_t>(q) * M;
        for (int j = q + 1; j < k1; ++j) ai[j] -= liq * lq[j];
      }
    }, par);
    pool.run(M - k1, [&](int t) {           // trailing update of row i: columns [k1, i]
      const int i = M - 1 - t;                // longest rows first
      double* ai = L.data() + static_cast<size_t>(i) * M;
      for (int q = k0; q < k1; ++q) {
        const double liq = ai[q];
        const double* lq = Lt.data() + static_cast<size_t>(q) * M;
        for (int j = k1; j <= i; ++j) ai[j] -= liq * lq[j];
      }
    }, par);
  }
  if (!pd) return err(E_NUM, "Cholesky of the GP covariance failed (not positive definite)");
  // alpha = L^-T L^-1 r
  std::vector<double> z(M);
  for (int i = 0; i < M; ++i) {
    double t = r[i];
    for (int q = 0; q < i; ++q) t -= L[i * M + q] * z[q];
    z[i] = t / L[i * M + i];
  }
  fit.alpha.assign(M, 0.0);
  for (int i = M - 1; i >= 0; --i) {
    double t = z[i];
    for (int q = i + 1; q < M; ++q) t -= L[q * M + i] * fit.alpha[q];
    fit.alpha[i] = t / L[i * M + i];
  }
  // W = L^-1 (lower triangular), row by row: W[i][c] = (delta_ic - sum_{q=c}^{i-1} L[i][q] W[q][c]) / L[i][i].
  // The sum is accumulated for all c of the row at once (axpy over the contiguous row W[q][0..q],
  // q ascending): the same operations in the same order per element as the column-by-column
  // form, but unit-stride and vectorisable.
  // Column ranges [c0, c1) in parallel, cut so that each holds about the same work ((M - c)^2 / 2
  // multiply-adds per column); inside a range the row-by-row axpy form, unit-stride in c.
  fit.Wl.assign(static_cast<size_t>(M) * M, 0.0);
  const int nr = std::min(M, 4 * pool.threads());
  std::vector<int> cut(nr + 1, M);
  {
    const double tot = static_cast<double>(M) * M * M / 6.0;
    double acc = 0.0;
    int r = 0;
    cut[0] = 0;
    for (int c = 0; c < M && r + 1 < nr; ++c) {
      acc += 0.5 * static_cast<double>(M - c) * (M - c);
      if (acc >= tot * (r + 1) / nr) cut[++r] = c + 1;
    }
    for (int q = r + 1; q <= nr; ++q) cut[q] = M;
  }
  pool.run(nr, [&](int rg) {
    const int c0 = cut[rg], c1 = cut[rg + 1];
    if (c0 >= c1) return;
    std::vector<double> t(static_cast<size_t>(c1 - c0));
    for (int i = c0; i < M; ++i) {
      const int ce = std::min(c1, i + 1);
      for (int c = c0; c < ce; ++c) t[c - c0] = (c == i) ? 1.0 : 0.0;
      for (int q = c0; q < i; ++q) {
        const double liq = L[i * M + q];
        const double* wq = fit.Wl.data() + static_cast<size_t>(q) * M;
        const int cq = std::min(c1, q + 1);
        for (int c = c0; c < cq; ++c) t[c - c0] -= liq * wq[c];
      }
      const double lii = L[i * M + i];
      for (int c = c0; c < ce; ++c) fit.Wl[static_cast<size_t>(i) * M + c] = t[c - c0] / lii;
    }
  }, par);
  double fro = 0.0;
  for (double w : fit.Wl) fro += w * w;
  fit.w_fro = std::sqrt(fro);
  return Status{};
}

}  // namespace as
