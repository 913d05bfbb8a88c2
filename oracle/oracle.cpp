// oracle.cpp — TEST INFRASTRUCTURE ONLY: a CPU restatement of the reference's batched-execution
// hot path, used by tests/ (and bench.py's CPU legs) as the parity checker for the B200 path.
// It is never linked into or called by the product (paper_2305_10611_b200/).
//
// What is restated, each with the reference lines it follows:
//   * primitive ops, fp32, separate mul + add, fixed i-k-j dense order .. proj/src/backend.cpp:105-181
//   * elementwise chain semantics ............................ proj/src/exec_batched.cpp:10-19
//   * depth scheduler (bucket key, map order, sorted ids) ..... proj/src/schedule.cpp:13-62
//   * zoo parameter / input generators (mt19937 streams) ...... proj/src/zoo.cpp:293-401
//   * the seven zoo models + fig5 evaluated unbatched, in program order, op by op, as the
//     sequential interpreter does (proj/src/reference.cpp:161-334 over the sources at
//     proj/src/zoo.cpp:26-279).
// Pinned against the compiled reference (oracle/_ref/mbatch_ref) through the golden fixtures in
// tests/golden/ (digests of params, inputs and outputs must be bitwise equal).
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <random>
#include <string>
#include <vector>

namespace {

// ---------------------------------------------------------------------------
// Values

struct HV {
  enum Kind { kTensor = 0, kInt = 1, kList = 2, kTuple = 3, kAdt = 4 };
  int kind = kTensor;
  int rows = 0, cols = 0;
  std::vector<float> d;
  long ival = 0;
  int ctor = 0;  // 0 Leaf, 1 Node
  std::vector<HV> items;

  static HV tensor(int r, int c) { HV v; v.kind = kTensor; v.rows = r; v.cols = c; v.d.assign(size_t(r) * c, 0.0f); return v; }
  static HV scalar(long x) { HV v; v.kind = kInt; v.ival = x; return v; }
  static HV list(std::vector<HV> it) { HV v; v.kind = kList; v.items = std::move(it); return v; }
  static HV tuple(std::vector<HV> it) { HV v; v.kind = kTuple; v.items = std::move(it); return v; }
  static HV adt(int ctor, std::vector<HV> it) { HV v; v.kind = kAdt; v.ctor = ctor; v.items = std::move(it); return v; }
};

void encode(const HV& v, std::vector<int32_t>& t, std::vector<float>& d) {
  t.push_back(v.kind);
  switch (v.kind) {
    case HV::kTensor: t.push_back(v.rows); t.push_back(v.cols); d.insert(d.end(), v.d.begin(), v.d.end()); return;
    case HV::kInt: t.push_back(static_cast<int32_t>(v.ival)); return;
    case HV::kAdt: t.push_back(v.ctor); [[fallthrough]];
    default:
      t.push_back(static_cast<int32_t>(v.items.size()));
      for (auto& it : v.items) encode(it, t, d);
  }
}

bool decode(const int32_t* t, int64_t nt, int64_t& ti, const float* d, int64_t nd, int64_t& di, HV& out) {
  if (ti >= nt) return false;
  out = HV{};
  out.kind = t[ti++];
  switch (out.kind) {
    case HV::kTensor: {
      if (ti + 2 > nt) return false;
      out.rows = t[ti++]; out.cols = t[ti++];
      int64_t n = int64_t(out.rows) * out.cols;
      if (n < 0 || di + n > nd) return false;
      out.d.assign(d + di, d + di + n);
      di += n;
      return true;
    }
    case HV::kInt: if (ti >= nt) return false; out.ival = t[ti++]; return true;
    case HV::kList: case HV::kTuple: case HV::kAdt: {
      if (out.kind == HV::kAdt) { if (ti >= nt) return false; out.ctor = t[ti++]; }
      if (ti >= nt) return false;
      int n = t[ti++];
      out.items.resize(n);
      for (int i = 0; i < n; ++i) if (!decode(t, nt, ti, d, nd, di, out.items[i])) return false;
      return true;
    }
  }
  return false;
}

void digest(const HV& v, uint64_t& h) {
  auto mix = [&](uint64_t x) { h ^= x; h *= 1099511628211ull; };
  if (v.kind == HV::kTensor) for (float f : v.d) { uint32_t b; std::memcpy(&b, &f, 4); mix(b); }
  else if (v.kind == HV::kInt) mix(static_cast<uint64_t>(v.ival));
  for (auto& it : v.items) digest(it, h);
}

// ---------------------------------------------------------------------------
// Primitive ops (proj/src/backend.cpp:94-181).  Every product and sum is a separately rounded
// fp32 operation; the TU is compiled with -ffp-contract=off (oracle/Makefile).

inline float sigmoid_f(float x) { return 1.0f / (1.0f + std::exp(-x)); }   // backend.cpp:96
inline float tanh_f(float x) { return std::tanh(x); }                       // backend.cpp:97
inline float relu_f(float x) { return x > 0.0f ? x : 0.0f; }                // backend.cpp:98

long g_prim_ops = 0;

// dense: c = 0; for i, for p ascending, for j: c[i,j] += a[i,p] * b[p,j]   (backend.cpp:116-131)
HV dense(const HV& a, const HV& b) {
  ++g_prim_ops;
  HV c = HV::tensor(a.rows, b.cols);
  int m = a.rows, k = a.cols, n = b.cols;
  for (int i = 0; i < m; ++i)
    for (int p = 0; p < k; ++p) {
      float av = a.d[size_t(i) * k + p];
      const float* brow = b.d.data() + size_t(p) * n;
      float* crow = c.d.data() + size_t(i) * n;
      for (int j = 0; j < n; ++j) crow[j] += av * brow[j];
    }
  return c;
}
HV add(const HV& a, const HV& b) { ++g_prim_ops; HV c = a; for (size_t i = 0; i < c.d.size(); ++i) c.d[i] = a.d[i] + b.d[i]; return c; }
HV mul(const HV& a, const HV& b) { ++g_prim_ops; HV c = a; for (size_t i = 0; i < c.d.size(); ++i) c.d[i] = a.d[i] * b.d[i]; return c; }
HV unary(const HV& a, float (*f)(float)) { ++g_prim_ops; HV c = a; for (auto& x : c.d) x = f(x); return c; }
HV sigm(const HV& a) { return unary(a, sigmoid_f); }
HV tanh_(const HV& a) { return unary(a, tanh_f); }
HV relu(const HV& a) { return unary(a, relu_f); }
HV concat(const HV& a, const HV& b) {  // axis 1 (backend.cpp:153-163)
  ++g_prim_ops;
  HV c = HV::tensor(a.rows, a.cols + b.cols);
  for (int r = 0; r < a.rows; ++r) {
    for (int j = 0; j < a.cols; ++j) c.d[size_t(r) * c.cols + j] = a.d[size_t(r) * a.cols + j];
    for (int j = 0; j < b.cols; ++j) c.d[size_t(r) * c.cols + a.cols + j] = b.d[size_t(r) * b.cols + j];
  }
  return c;
}
// argmax (1,n) -> first index of the max, stored as float (backend.cpp:164-173); scalar() then
// truncates to long (reference.cpp:199-205).
long argmax_scalar(const HV& a) {
  ++g_prim_ops;
  int best = 0;
  for (int i = 1; i < a.cols; ++i) if (a.d[i] > a.d[best]) best = i;
  return static_cast<long>(static_cast<float>(best));
}

// ---------------------------------------------------------------------------
// Zoo (proj/src/zoo.cpp)

struct Decl { std::string name; int kind; int rows, cols; int leaf_fields; };  // kind: 0 tensor param, 1 list input, 2 tree input, 3 tensor input, 4 int input
enum { kParamT = 0, kListIn = 1, kTreeIn = 2, kTensorIn = 3, kIntIn = 4 };

struct Model {
  std::string name;
  int H = 32, C = 8;
  std::vector<Decl> decls;  // module param order (params and instance inputs interleaved as declared)
  std::map<std::string, HV> params;
  std::vector<std::map<std::string, HV>> inputs;
  std::vector<HV> outputs;
  long prim_ops = 0;
  const HV& P(const std::string& n) const { return params.at(n); }
};

std::vector<Decl> decls_for(const std::string& name, int H, int C) {
  int H2 = 2 * H;
  auto p = [](const char* n, int r, int c) { return Decl{n, kParamT, r, c, 0}; };
  if (name == "rnn")
    return {p("rnn_bias", 1, H), p("rnn_i_wt", H, H), p("rnn_h_wt", H, H), p("rnn_init", 1, H),
            p("c_wt", H, C), p("cbias", 1, C), Decl{"inps", kListIn, 1, H, 0}};
  if (name == "birnn")
    return {p("f_rnn_bias", 1, H), p("f_rnn_i_wt", H, H), p("f_rnn_h_wt", H, H), p("f_rnn_init", 1, H),
            p("b_rnn_bias", 1, H), p("b_rnn_i_wt", H, H), p("b_rnn_h_wt", H, H), p("b_rnn_init", 1, H),
            Decl{"inps_list", kListIn, 1, H, 0}};
  if (name == "treelstm")
    return {p("x_wt", H, H), p("x_bias", 1, H), p("xn", 1, H), p("i_wt", H2, H), p("fl_wt", H2, H),
            p("fr_wt", H2, H), p("u_wt", H2, H), p("hz", 1, H), p("cz", 1, H), p("c_wt", H, C),
            p("cbias", 1, C), Decl{"t", kTreeIn, 1, H, 1}};
  if (name == "mvrnn")
    return {p("v_wt", H2, H), p("vbias", 1, H), p("c_wt", H, C), p("cbias", 1, C), Decl{"t", kTreeIn, 1, H, 2}};
  if (name == "nestedrnn")
    return {p("zb", 1, H), p("z_wt", H2, H), p("hb", 1, H), p("h_wt", H2, H), p("rb", 1, H), p("r_wt", H2, H),
            p("n_wt", H, 11), p("ibias", 1, H), p("i_wt", H, H), p("outer_init", 1, H),
            Decl{"xs", kListIn, 1, H, 0}};
  if (name == "drnn")
    return {p("obias", 1, H), p("o_wt", H, H), p("d_wt", H, 2), p("lbias", 1, H), p("l_wt", H, H),
            p("rbias", 1, H), p("r_wt", H, H), p("root_bias", 1, H), p("root_wt", H, H),
            Decl{"x", kTensorIn, 1, H, 0}, Decl{"fuel", kIntIn, 0, 0, 0}};
  if (name == "stackrnn")
    return {p("hbias", 1, H), p("s_wt", H2, H), p("a_wt", H, 2), p("ebias", 1, H), p("e_wt", H, H),
            p("pbias", 1, H), p("p_wt", H, H), p("rbias", 1, H), p("r_wt", H, H), p("obias", 1, H),
            p("o_wt", H2, H), p("init", 1, H), p("c_wt", H, C), p("cbias", 1, C), Decl{"toks", kListIn, 1, H, 0}};
  if (name == "fig5")
    return {p("a_wt", H, H), p("abias", 1, H), p("b_wt", H, H), p("bbias", 1, H),
            Decl{"x", kTensorIn, 1, H, 0}, Decl{"sel", kIntIn, 0, 0, 0}};
  return {};
}

// zoo.cpp:281-286
HV random_tensor(std::mt19937& rng, int r, int c) {
  std::uniform_real_distribution<float> dist(-0.5f, 0.5f);
  HV v = HV::tensor(r, c);
  for (auto& x : v.d) x = dist(rng);
  return v;
}

// zoo.cpp:293-301: full binary tree with `leaves` leaves.
HV random_tree(std::mt19937& rng, int leaves, const std::function<HV(std::mt19937&)>& leaf_fn) {
  if (leaves == 1) return leaf_fn(rng);
  std::uniform_int_distribution<int> split(1, leaves - 1);
  int left = split(rng);
  HV l = random_tree(rng, left, leaf_fn);
  HV r = random_tree(rng, leaves - left, leaf_fn);
  return HV::adt(1, {std::move(l), std::move(r)});
}

void make_params(Model& m, unsigned seed) {  // zoo.cpp:332-341
  std::mt19937 rng(seed * 7919u + 17u);
  m.params.clear();
  for (auto& d : m.decls)
    if (d.kind == kParamT) m.params[d.name] = random_tensor(rng, d.rows, d.cols);
}

void make_inputs(Model& m, unsigned seed, int batch) {  // zoo.cpp:343-401
  m.inputs.clear();
  for (int i = 0; i < batch; ++i) {
    std::mt19937 rng(seed * 104729u + 31u * i + 7u);
    std::map<std::string, HV> inst;
    for (auto& d : m.decls) {
      switch (d.kind) {
        case kParamT: break;
        case kListIn: {
          std::uniform_int_distribution<int> len_dist(4, 12);
          int len = len_dist(rng);
          std::vector<HV> items;
          for (int k = 0; k < len; ++k) items.push_back(random_tensor(rng, d.rows, d.cols));
          inst[d.name] = HV::list(std::move(items));
          break;
        }
        case kTreeIn: {
          std::uniform_int_distribution<int> leaves_dist(4, 16);
          int leaves = leaves_dist(rng);
          int H = m.H;
          int nf = d.leaf_fields;
          auto leaf_fn = [H, nf](std::mt19937& r) {
            std::vector<HV> f;
            f.push_back(random_tensor(r, 1, H));
            if (nf == 2) f.push_back(random_tensor(r, H, H));
            return HV::adt(0, std::move(f));
          };
          inst[d.name] = random_tree(rng, leaves, leaf_fn);
          break;
        }
        case kTensorIn: inst[d.name] = random_tensor(rng, d.rows, d.cols); break;
        case kIntIn: {
          if (d.name == "fuel") { std::uniform_int_distribution<int> fd(3, 4); inst[d.name] = HV::scalar(fd(rng)); }
          else if (d.name == "sel") inst[d.name] = HV::scalar(i % 2);
          else { std::uniform_int_distribution<int> dd(0, 7); inst[d.name] = HV::scalar(dd(rng)); }
          break;
        }
      }
    }
    m.inputs.push_back(std::move(inst));
  }
}

// ---------------------------------------------------------------------------
// Unbatched model evaluation, op by op in program order (zoo.cpp sources).

// @rnn (zoo.cpp:27-37): inp_linear = bias + dense(inp, i_wt); new_state = sigmoid(inp_linear + dense(state, h_wt))
std::vector<HV> eval_rnn_chain(const std::vector<HV>& inps, HV state, const HV& bias, const HV& i_wt, const HV& h_wt) {
  std::vector<HV> out;
  for (auto& inp : inps) {
    HV inp_linear = add(bias, dense(inp, i_wt));
    HV ns = sigm(add(inp_linear, dense(state, h_wt)));
    out.push_back(ns);
    state = ns;
  }
  return out;
}

HV eval_rnn(const Model& m, const std::map<std::string, HV>& in) {  // zoo.cpp:26-45
  auto res = eval_rnn_chain(in.at("inps").items, m.P("rnn_init"), m.P("rnn_bias"), m.P("rnn_i_wt"), m.P("rnn_h_wt"));
  std::vector<HV> out;
  for (auto& p : res) out.push_back(relu(add(m.P("cbias"), dense(p, m.P("c_wt")))));
  return HV::list(std::move(out));
}

HV eval_birnn(const Model& m, const std::map<std::string, HV>& in) {  // zoo.cpp:47-76
  const auto& xs = in.at("inps_list").items;
  std::vector<HV> rxs(xs.rbegin(), xs.rend());
  auto fwd = eval_rnn_chain(xs, m.P("f_rnn_init"), m.P("f_rnn_bias"), m.P("f_rnn_i_wt"), m.P("f_rnn_h_wt"));
  auto bwd = eval_rnn_chain(rxs, m.P("b_rnn_init"), m.P("b_rnn_bias"), m.P("b_rnn_i_wt"), m.P("b_rnn_h_wt"));
  std::reverse(bwd.begin(), bwd.end());
  std::vector<HV> out;
  for (size_t i = 0; i < fwd.size(); ++i) out.push_back(concat(fwd[i], bwd[i]));
  return HV::list(std::move(out));
}

// @tcell (zoo.cpp:84-92) -> (tanh(c), c)
std::pair<HV, HV> tcell(const Model& m, const HV& xt, const HV& lh, const HV& lc, const HV& rh, const HV& rc) {
  HV hcat = concat(lh, rh);
  HV i = sigm(add(dense(hcat, m.P("i_wt")), xt));
  HV fl = sigm(add(dense(hcat, m.P("fl_wt")), xt));
  HV fr = sigm(add(dense(hcat, m.P("fr_wt")), xt));
  HV u = tanh_(add(dense(hcat, m.P("u_wt")), xt));
  HV c = add(mul(i, u), add(mul(fl, lc), mul(fr, rc)));
  return {tanh_(c), c};
}

std::pair<HV, HV> tlstm(const Model& m, const HV& t) {  // zoo.cpp:94-107
  if (t.ctor == 0) {
    HV xt = add(m.P("x_bias"), dense(t.items[0], m.P("x_wt")));
    return tcell(m, xt, m.P("hz"), m.P("cz"), m.P("hz"), m.P("cz"));
  }
  auto l = tlstm(m, t.items[0]);
  auto r = tlstm(m, t.items[1]);
  return tcell(m, m.P("xn"), l.first, l.second, r.first, r.second);
}

HV eval_treelstm(const Model& m, const std::map<std::string, HV>& in) {  // zoo.cpp:109-116
  auto res = tlstm(m, in.at("t"));
  return relu(add(m.P("cbias"), dense(res.first, m.P("c_wt"))));
}

std::pair<HV, HV> mv(const Model& m, const HV& t) {  // zoo.cpp:124-136
  if (t.ctor == 0) return {t.items[0], t.items[1]};
  auto l = mv(m, t.items[0]);
  auto r = mv(m, t.items[1]);
  HV lv_rm = dense(l.first, r.second);
  HV rv_lm = dense(r.first, l.second);
  HV v = tanh_(add(m.P("vbias"), dense(concat(lv_rm, rv_lm), m.P("v_wt"))));
  return {v, add(l.second, r.second)};
}

HV eval_mvrnn(const Model& m, const std::map<std::string, HV>& in) {  // zoo.cpp:138-143
  auto res = mv(m, in.at("t"));
  return relu(add(m.P("cbias"), dense(res.first, m.P("c_wt"))));
}

HV eval_nestedrnn(const Model& m, const std::map<std::string, HV>& in) {  // zoo.cpp:145-174
  HV h = m.P("outer_init");
  for (auto& x : in.at("xs").items) {
    HV cat = concat(x, h);
    HV z = sigm(add(m.P("zb"), dense(cat, m.P("z_wt"))));
    HV hc = tanh_(add(m.P("hb"), dense(cat, m.P("h_wt"))));
    HV zr = sigm(add(m.P("rb"), dense(cat, m.P("r_wt"))));
    HV hmix = add(mul(z, hc), mul(zr, h));
    long n = argmax_scalar(dense(hmix, m.P("n_wt")));
    HV s = hmix;
    for (long k = n + 25; k > 0; --k) s = sigm(add(m.P("ibias"), dense(s, m.P("i_wt"))));  // @inner
    h = s;
  }
  return h;
}

void drnn_gen(const Model& m, const HV& h, long fuel, std::vector<HV>& out) {  // zoo.cpp:184-199
  HV o = tanh_(add(m.P("obias"), dense(h, m.P("o_wt"))));
  if (fuel <= 0) { out.push_back(o); return; }
  long d = argmax_scalar(dense(o, m.P("d_wt")));
  if (d == 0) { out.push_back(o); return; }
  HV lh = tanh_(add(m.P("lbias"), dense(o, m.P("l_wt"))));
  HV rh = tanh_(add(m.P("rbias"), dense(o, m.P("r_wt"))));
  std::vector<HV> lt, rt;
  drnn_gen(m, lh, fuel - 1, lt);
  drnn_gen(m, rh, fuel - 1, rt);
  out.push_back(o);
  for (auto& v : lt) out.push_back(std::move(v));
  for (auto& v : rt) out.push_back(std::move(v));
}

HV eval_drnn(const Model& m, const std::map<std::string, HV>& in) {  // zoo.cpp:201-208
  HV h0 = tanh_(add(m.P("root_bias"), dense(in.at("x"), m.P("root_wt"))));
  std::vector<HV> out;
  drnn_gen(m, h0, in.at("fuel").ival, out);
  return HV::list(std::move(out));
}

HV eval_stackrnn(const Model& m, const std::map<std::string, HV>& in) {  // zoo.cpp:211-240
  HV h = m.P("init");
  for (auto& x : in.at("toks").items) {
    HV h2 = sigm(add(m.P("hbias"), dense(concat(x, h), m.P("s_wt"))));
    long a = argmax_scalar(dense(h2, m.P("a_wt")));
    HV h0, h1;
    if (a == 0) {
      h0 = tanh_(add(m.P("ebias"), dense(h2, m.P("e_wt"))));
      h1 = relu(add(m.P("pbias"), dense(h2, m.P("p_wt"))));
    } else {
      h0 = tanh_(add(m.P("rbias"), dense(h2, m.P("r_wt"))));
      h1 = h0;
    }
    h = sigm(add(m.P("obias"), dense(concat(h0, h1), m.P("o_wt"))));
  }
  return relu(add(m.P("cbias"), dense(h, m.P("c_wt"))));
}

HV eval_fig5(const Model& m, const std::map<std::string, HV>& in) {  // zoo.cpp:243-259
  auto common = [&](const HV& v) { return sigm(add(m.P("bbias"), dense(v, m.P("b_wt")))); };
  auto extra = [&](const HV& v) { return relu(add(m.P("abias"), dense(v, m.P("a_wt")))); };
  HV r = in.at("sel").ival == 0 ? common(in.at("x")) : common(extra(in.at("x")));
  return common(r);
}

HV eval_instance(const Model& m, const std::map<std::string, HV>& in) {
  if (m.name == "rnn") return eval_rnn(m, in);
  if (m.name == "birnn") return eval_birnn(m, in);
  if (m.name == "treelstm") return eval_treelstm(m, in);
  if (m.name == "mvrnn") return eval_mvrnn(m, in);
  if (m.name == "nestedrnn") return eval_nestedrnn(m, in);
  if (m.name == "drnn") return eval_drnn(m, in);
  if (m.name == "stackrnn") return eval_stackrnn(m, in);
  if (m.name == "fig5") return eval_fig5(m, in);
  return HV{};
}

void encode_inputs(const Model& m, std::vector<int32_t>& t, std::vector<float>& d) {
  for (auto& inst : m.inputs)
    for (auto& dc : m.decls)
      if (dc.kind != kParamT) encode(inst.at(dc.name), t, d);
}

}  // namespace

struct orc_model : Model {
  std::vector<std::string> param_names;
};

extern "C" {

orc_model* orc_model_create(const char* name, int hidden, unsigned seed) {
  auto decls = decls_for(name, hidden, 8);
  if (decls.empty()) return nullptr;
  auto* m = new orc_model;
  m->name = name;
  m->H = hidden;
  m->decls = decls;
  for (auto& d : decls) if (d.kind == kParamT) m->param_names.push_back(d.name);
  make_params(*m, seed);
  return m;
}

void orc_model_destroy(orc_model* m) { delete m; }

int orc_make_inputs(orc_model* m, unsigned seed, int batch) {
  if (!m || batch < 1) return -1;
  make_inputs(*m, seed, batch);
  return 0;
}

int orc_set_inputs(orc_model* m, int batch, const int32_t* toks, int64_t ntok, const float* data, int64_t ndata) {
  int64_t ti = 0, di = 0;
  m->inputs.clear();
  for (int i = 0; i < batch; ++i) {
    std::map<std::string, HV> inst;
    for (auto& dc : m->decls) {
      if (dc.kind == kParamT) continue;
      HV v;
      if (!decode(toks, ntok, ti, data, ndata, di, v)) return -1;
      inst[dc.name] = std::move(v);
    }
    m->inputs.push_back(std::move(inst));
  }
  return (ti == ntok && di == ndata) ? 0 : -1;
}

int64_t orc_inputs_ntok(const orc_model* m) { std::vector<int32_t> t; std::vector<float> d; encode_inputs(*m, t, d); return int64_t(t.size()); }
int64_t orc_inputs_ndata(const orc_model* m) { std::vector<int32_t> t; std::vector<float> d; encode_inputs(*m, t, d); return int64_t(d.size()); }
int orc_get_inputs(const orc_model* m, int32_t* toks, float* data) {
  std::vector<int32_t> t; std::vector<float> d;
  encode_inputs(*m, t, d);
  std::memcpy(toks, t.data(), t.size() * 4);
  std::memcpy(data, d.data(), d.size() * 4);
  return 0;
}

uint64_t orc_params_digest(const orc_model* m) {
  uint64_t h = 1469598103934665603ull;
  for (auto& d : m->decls) if (d.kind == kParamT) digest(m->params.at(d.name), h);
  return h;
}
uint64_t orc_inputs_digest(const orc_model* m) {
  uint64_t h = 1469598103934665603ull;
  for (auto& inst : m->inputs)
    for (auto& d : m->decls) if (d.kind != kParamT) digest(inst.at(d.name), h);
  return h;
}

int orc_evaluate(orc_model* m) {
  g_prim_ops = 0;
  m->outputs.clear();
  for (auto& inst : m->inputs) m->outputs.push_back(eval_instance(*m, inst));
  m->prim_ops = g_prim_ops;
  return 0;
}

int64_t orc_last_prim_ops(const orc_model* m) { return m->prim_ops; }

int64_t orc_outputs_ntok(const orc_model* m) { std::vector<int32_t> t; std::vector<float> d; for (auto& o : m->outputs) encode(o, t, d); return int64_t(t.size()); }
int64_t orc_outputs_ndata(const orc_model* m) { std::vector<int32_t> t; std::vector<float> d; for (auto& o : m->outputs) encode(o, t, d); return int64_t(d.size()); }
int orc_get_outputs(const orc_model* m, int32_t* toks, float* data) {
  std::vector<int32_t> t; std::vector<float> d;
  for (auto& o : m->outputs) encode(o, t, d);
  std::memcpy(toks, t.data(), t.size() * 4);
  std::memcpy(data, d.data(), d.size() * 4);
  return 0;
}
uint64_t orc_outputs_digest(const orc_model* m) {
  uint64_t h = 1469598103934665603ull;
  for (auto& o : m->outputs) digest(o, h);
  return h;
}

int orc_num_params(const orc_model* m) { return int(m->param_names.size()); }
const char* orc_param_name(const orc_model* m, int i) { return m->param_names.at(i).c_str(); }
int orc_param_shape(const orc_model* m, int i, int* rows, int* cols) {
  const HV& v = m->params.at(m->param_names.at(i));
  *rows = v.rows; *cols = v.cols;
  return 0;
}
const float* orc_param_data(const orc_model* m, int i) { return m->params.at(m->param_names.at(i)).d.data(); }

int orc_exec_primop(int op, int nin, const float* const* ins, const int* rows, const int* cols,
                    float* out, int out_rows, int out_cols, float fill) {
  int n = out_rows * out_cols;
  switch (op) {
    case 0: {  // dense (backend.cpp:116-131)
      if (nin != 2 || cols[0] != rows[1]) return -1;
      int m = rows[0], k = cols[0], nn = cols[1];
      for (int i = 0; i < m * nn; ++i) out[i] = 0.0f;
      for (int i = 0; i < m; ++i)
        for (int p = 0; p < k; ++p) {
          float av = ins[0][i * k + p];
          for (int j = 0; j < nn; ++j) out[i * nn + j] += av * ins[1][p * nn + j];
        }
      return 0;
    }
    case 1: for (int i = 0; i < n; ++i) out[i] = ins[0][i] + ins[1][i]; return 0;
    case 2: for (int i = 0; i < n; ++i) out[i] = ins[0][i] * ins[1][i]; return 0;
    case 3: for (int i = 0; i < n; ++i) out[i] = sigmoid_f(ins[0][i]); return 0;
    case 4: for (int i = 0; i < n; ++i) out[i] = tanh_f(ins[0][i]); return 0;
    case 5: for (int i = 0; i < n; ++i) out[i] = relu_f(ins[0][i]); return 0;
    case 6: {
      int ca = cols[0], cb = cols[1];
      for (int r = 0; r < out_rows; ++r) {
        for (int j = 0; j < ca; ++j) out[r * (ca + cb) + j] = ins[0][r * ca + j];
        for (int j = 0; j < cb; ++j) out[r * (ca + cb) + ca + j] = ins[1][r * cb + j];
      }
      return 0;
    }
    case 7: {
      int best = 0;
      for (int i = 1; i < cols[0]; ++i) if (ins[0][i] > ins[0][best]) best = i;
      out[0] = static_cast<float>(best);
      return 0;
    }
    case 8: for (int i = 0; i < n; ++i) out[i] = fill; return 0;
  }
  return -1;
}

int orc_schedule_depth(int n, const int* id, const int* phase, const int* depth, const int* sig,
                       const int* ghost, const int* nshared, const int64_t* shared_refs,
                       int* batches, int* order, long* ops) {
  struct Key {
    int phase, depth, sig;
    uint64_t shared;
    bool operator<(const Key& o) const {  // schedule.cpp:33-39 (ghost is not part of the order)
      if (phase != o.phase) return phase < o.phase;
      if (depth != o.depth) return depth < o.depth;
      if (sig != o.sig) return sig < o.sig;
      return shared < o.shared;
    }
  };
  std::map<Key, std::pair<bool, std::vector<int>>> buckets;
  const int64_t* r = shared_refs;
  for (int i = 0; i < n; ++i) {
    uint64_t h = 1469598103934665603ull;  // schedule.cpp:13-25
    auto mix = [&](uint64_t v) { h ^= v; h *= 1099511628211ull; };
    for (int s = 0; s < nshared[i]; ++s, r += 3) {
      mix(static_cast<uint64_t>(r[0] + 1));
      mix(static_cast<uint64_t>(r[1]));
      mix(static_cast<uint64_t>(r[2] + 1));
    }
    auto& b = buckets[Key{phase[i], depth[i], sig[i], h}];
    if (b.second.empty()) b.first = ghost[i] != 0;
    b.second.push_back(id[i]);
    ++*ops;
  }
  int nb = 0, k = 0;
  for (auto& [key, val] : buckets) {
    auto ids = val.second;
    std::sort(ids.begin(), ids.end());
    int* row = batches + 5 * nb++;
    row[0] = key.phase; row[1] = key.depth; row[2] = key.sig; row[3] = val.first ? 1 : 0; row[4] = int(ids.size());
    for (int x : ids) order[k++] = x;
    *ops += long(ids.size());
  }
  return nb;
}

uint64_t orc_digest_encoded(const int32_t* toks, int64_t ntok, const float* data, int64_t ndata, int count) {
  uint64_t h = 1469598103934665603ull;
  int64_t ti = 0, di = 0;
  for (int i = 0; i < count; ++i) {
    HV v;
    if (!decode(toks, ntok, ti, data, ndata, di, v)) return 0;
    digest(v, h);
  }
  return h;
}

float orc_unary(int which, float x) {
  switch (which) {
    case 0: return std::exp(x);
    case 1: return std::tanh(x);
    case 2: return sigmoid_f(x);
  }
  return 0.0f;
}

}  // extern "C"
