// ff_frontend.cpp -- RHS front end: expression parser, validator and CUDA C emitter.
//
// "The only part of the kernel that changes for different systems of equations is
// that which calculates the time derivative ... generated automatically using the definitions for
// the state variables given by the user." PAPER.md:186: no branching in user equations, so the
// grammar has no conditionals and the emitted code is straight-line.
//
// Grammar (used for interface shape only):
//   expr := term (("+"|"-") term)* ; term := factor (("*"|"/") factor)* ;
//   factor := "-" factor | power ; power := atom ("^" factor)? ;
//   atom := number | ident | ident "(" expr ("," expr)* ")" | "(" expr ")"
//
// Emission lowers the AST into a hash-consed DAG of primitive ops (MUFU-only transcendentals:
// exp -> ex2 with log2(e) folded into constant multipliers, division -> rcp, integer powers ->
// multiplications), classifies every node as uniform (parameters / constants only; `float`,
// loop-invariant) or varying (depends on the state or the swept parameter; type V = float or the
// packed pair ff2), and prints one `const` temporary per node.
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <set>
#include <sstream>
#include <unordered_map>

#include "ff_internal.hpp"

namespace ff {

// ================================================================ lexer / parser
namespace {

const std::map<std::string, int>& functions() {
  static const std::map<std::string, int> f = {
      {"exp", 1}, {"log", 1}, {"sin", 1}, {"cos", 1}, {"tan", 1}, {"tanh", 1}, {"sqrt", 1},
      {"abs", 1}, {"sigmoid", 1}, {"pow", 2}, {"min", 2}, {"max", 2}, {"vtrap", 2}};
  return f;
}

bool is_identifier(const std::string& s) {
  if (s.empty() || !(std::isalpha((unsigned char)s[0]) || s[0] == '_')) return false;
  for (char c : s)
    if (!(std::isalnum((unsigned char)c) || c == '_')) return false;
  return true;
}

struct Parser {
  const std::string& src;
  const std::string& where;  // e.g. "rhs of x"
  const std::map<std::string, int>& vars;
  const std::map<std::string, int>& params;
  size_t i = 0;

  Parser(const std::string& s, const std::string& w, const std::map<std::string, int>& v,
         const std::map<std::string, int>& p)
      : src(s), where(w), vars(v), params(p) {}

  [[noreturn]] void fail(ff_status st, const std::string& msg, size_t at) const {
    std::ostringstream o;
    o << where << ": " << msg << " at position " << at << " in \"" << src << "\"";
    throw Error(st, o.str());
  }
  void skip() {
    while (i < src.size() && std::isspace((unsigned char)src[i])) ++i;
  }
  bool peek(char c) {
    skip();
    return i < src.size() && src[i] == c;
  }
  bool accept(char c) {
    if (peek(c)) { ++i; return true; }
    return false;
  }
  void expect(char c) {
    if (!accept(c)) {
      skip();
      if (i >= src.size()) fail(FF_ERR_PARSE, std::string("expected '") + c + "' but reached end of input", i);
      fail(FF_ERR_PARSE, std::string("expected '") + c + "'", i);
    }
  }

  NodeP mk(Op op, size_t pos) {
    auto n = std::make_shared<Node>();
    n->op = op;
    n->pos = (int)pos;
    return n;
  }

  NodeP parse_all() {
    NodeP e = expr();
    skip();
    if (i != src.size()) fail(FF_ERR_PARSE, "unexpected character '" + std::string(1, src[i]) + "'", i);
    return e;
  }
  NodeP expr() {
    NodeP a = term();
    for (;;) {
      skip();
      size_t at = i;
      if (accept('+')) { auto n = mk(Op::Add, at); n->args = {a, term()}; a = n; }
      else if (accept('-')) { auto n = mk(Op::Sub, at); n->args = {a, term()}; a = n; }
      else return a;
    }
  }
  NodeP term() {
    NodeP a = factor();
    for (;;) {
      skip();
      size_t at = i;
      if (accept('*')) { auto n = mk(Op::Mul, at); n->args = {a, factor()}; a = n; }
      else if (accept('/')) { auto n = mk(Op::Div, at); n->args = {a, factor()}; a = n; }
      else return a;
    }
  }
  NodeP factor() {
    skip();
    size_t at = i;
    if (accept('-')) { auto n = mk(Op::Neg, at); n->args = {factor()}; return n; }
    return power();
  }
  NodeP power() {
    NodeP a = atom();
    skip();
    size_t at = i;
    if (accept('^')) { auto n = mk(Op::Pow, at); n->args = {a, factor()}; return n; }
    return a;
  }
  NodeP atom() {
    skip();
    size_t at = i;
    if (i >= src.size()) fail(FF_ERR_PARSE, "unexpected end of input", i);
    char c = src[i];
    if (std::isdigit((unsigned char)c) || c == '.') {
      size_t j = i;
      while (j < src.size() && std::isdigit((unsigned char)src[j])) ++j;
      if (j < src.size() && src[j] == '.') { ++j; while (j < src.size() && std::isdigit((unsigned char)src[j])) ++j; }
      if (j == i + 1 && src[i] == '.') fail(FF_ERR_PARSE, "malformed number", i);
      if (j < src.size() && (src[j] == 'e' || src[j] == 'E')) {
        size_t k = j + 1;
        if (k < src.size() && (src[k] == '+' || src[k] == '-')) ++k;
        if (k < src.size() && std::isdigit((unsigned char)src[k])) {
          while (k < src.size() && std::isdigit((unsigned char)src[k])) ++k;
          j = k;
        } else {
          fail(FF_ERR_PARSE, "malformed exponent", j);
        }
      }
      auto n = mk(Op::Num, at);
      n->value = std::strtod(src.substr(i, j - i).c_str(), nullptr);
      i = j;
      return n;
    }
    if (std::isalpha((unsigned char)c) || c == '_') {
      size_t j = i;
      while (j < src.size() && (std::isalnum((unsigned char)src[j]) || src[j] == '_')) ++j;
      std::string id = src.substr(i, j - i);
      i = j;
      if (peek('(')) {
        auto f = functions().find(id);
        if (f == functions().end()) fail(FF_ERR_PARSE, "unknown function '" + id + "'", at);
        expect('(');
        auto n = mk(Op::Call, at);
        n->name = id;
        n->args.push_back(expr());
        while (accept(',')) n->args.push_back(expr());
        expect(')');
        if ((int)n->args.size() != f->second) {
          std::ostringstream o;
          o << "function '" << id << "' takes " << f->second << " argument(s), got " << n->args.size();
          fail(FF_ERR_PARSE, o.str(), at);
        }
        return n;
      }
      if (id == "pi") { auto n = mk(Op::Num, at); n->value = 3.14159265358979323846; return n; }
      if (id == "e") { auto n = mk(Op::Num, at); n->value = 2.71828182845904523536; return n; }
      auto v = vars.find(id);
      if (v != vars.end()) { auto n = mk(Op::Var, at); n->index = v->second; n->name = id; return n; }
      auto p = params.find(id);
      if (p != params.end()) { auto n = mk(Op::Param, at); n->index = p->second; n->name = id; return n; }
      if (functions().count(id)) fail(FF_ERR_PARSE, "function '" + id + "' used without arguments", at);
      fail(FF_ERR_UNKNOWN_SYMBOL, "unknown identifier '" + id + "'", at);
    }
    if (accept('(')) {
      NodeP e = expr();
      expect(')');
      return e;
    }
    fail(FF_ERR_PARSE, "unexpected character '" + std::string(1, c) + "'", i);
  }
};

}  // namespace

// ---------------------------------------------------------------- uniform factors of components
namespace {

bool param_only(const NodeP& n, int sweep_param) {
  if (n->op == Op::Var) return false;
  if (n->op == Op::Param) return n->index != sweep_param;
  for (const NodeP& a : n->args) if (!param_only(a, sweep_param)) return false;
  return true;
}

NodeP mk(Op op, std::vector<NodeP> args, double v = 0.0) {
  NodeP n = std::make_shared<Node>();
  n->op = op;
  n->value = v;
  n->args = std::move(args);
  return n;
}

// the factors of a product tree: a * b, a / c (c a factor 1/c when it is parameter-only), -a
void factors(const NodeP& n, int sp, std::vector<NodeP>& uni, std::vector<NodeP>& var) {
  if (n->op == Op::Mul) {
    factors(n->args[0], sp, uni, var);
    factors(n->args[1], sp, uni, var);
  } else if (n->op == Op::Neg) {
    uni.push_back(mk(Op::Num, {}, -1.0));
    factors(n->args[0], sp, uni, var);
  } else if (n->op == Op::Div && param_only(n->args[1], sp)) {
    factors(n->args[0], sp, uni, var);
    uni.push_back(mk(Op::Div, {mk(Op::Num, {}, 1.0), n->args[1]}));
  } else if (param_only(n, sp)) {
    uni.push_back(n);
  } else {
    var.push_back(n);
  }
}

std::string ast_key(const NodeP& n) {  // structural key of an expression
  std::ostringstream o;
  o << (int)n->op << ':' << n->index << ':' << n->name << ':';
  {
    uint64_t bits;
    std::memcpy(&bits, &n->value, 8);
    o << bits;
  }
  o << '(';
  for (const NodeP& a : n->args) o << ast_key(a) << ',';
  o << ')';
  return o.str();
}

NodeP product(const std::vector<NodeP>& f) {
  NodeP p = f[0];
  for (size_t i = 1; i < f.size(); ++i) p = mk(Op::Mul, {p, f[i]});
  return p;
}

// ---- collecting a state variable out of a sum of driving-force terms
// Conductance equations are sums of c_i (E_i - V) (each ionic and synaptic current
// of the HH ring). Written out, every term costs a subtraction and an FFMA with three per-particle
// register operands (the slow form); collected, sum c_i (E_i - V) = sum c_i E_i -
// V sum c_i is a chain of FFMAs with uniform operands and one final product. Exact in real arithmetic.
void sum_terms(const NodeP& n, int sign, std::vector<std::pair<int, NodeP>>& out) {
  if (n->op == Op::Add) { sum_terms(n->args[0], sign, out); sum_terms(n->args[1], sign, out); }
  else if (n->op == Op::Sub) { sum_terms(n->args[0], sign, out); sum_terms(n->args[1], -sign, out); }
  else if (n->op == Op::Neg) sum_terms(n->args[0], -sign, out);
  else out.push_back({sign, n});
}
void prod_factors(const NodeP& n, int& sign, std::vector<NodeP>& out) {
  if (n->op == Op::Mul) { prod_factors(n->args[0], sign, out); prod_factors(n->args[1], sign, out); }
  else if (n->op == Op::Neg) { sign = -sign; prod_factors(n->args[0], sign, out); }
  else out.push_back(n);
}
// factor (a - V) or (V - a) with V a state variable and a free of state variables: V's index, a, and
// the orientation (+1 for a - V)
bool driving_force(const NodeP& f, int sp, int& var, NodeP& a, int& orient) {
  if (f->op != Op::Sub) return false;
  const NodeP &l = f->args[0], &r = f->args[1];
  if (r->op == Op::Var && param_only(l, sp)) { var = r->index; a = l; orient = 1; return true; }
  if (l->op == Op::Var && param_only(r, sp)) { var = l->index; a = r; orient = -1; return true; }
  return false;
}
NodeP signed_sum(const std::vector<std::pair<int, NodeP>>& t) {
  NodeP acc;
  for (const auto& e : t) {
    if (!acc) acc = e.first > 0 ? e.second : mk(Op::Neg, {e.second});
    else acc = mk(e.first > 0 ? Op::Add : Op::Sub, {acc, e.second});
  }
  return acc ? acc : mk(Op::Num, {}, 0.0);
}
NodeP collect_linear(const NodeP& root, int sp) {
  std::vector<std::pair<int, NodeP>> terms;
  sum_terms(root, 1, terms);
  std::map<int, std::vector<size_t>> by_var;
  std::vector<int> var(terms.size(), -1), orient(terms.size(), 0);
  std::vector<NodeP> a(terms.size()), c(terms.size());
  for (size_t i = 0; i < terms.size(); ++i) {
    int sign = terms[i].first;
    std::vector<NodeP> f;
    prod_factors(terms[i].second, sign, f);
    for (size_t j = 0; j < f.size(); ++j) {
      int v, o;
      NodeP av;
      if (!driving_force(f[j], sp, v, av, o)) continue;
      std::vector<NodeP> rest;
      for (size_t k = 0; k < f.size(); ++k) if (k != j) rest.push_back(f[k]);
      var[i] = v; a[i] = av; orient[i] = o * sign;   // term = orient * c * (a - V)
      c[i] = rest.empty() ? mk(Op::Num, {}, 1.0) : product(rest);
      by_var[v].push_back(i);
      break;
    }
  }
  std::vector<std::pair<int, NodeP>> out;
  std::vector<char> done(terms.size(), 0);
  for (auto& kv : by_var) {
    if (kv.second.size() < 2) continue;
    std::vector<std::pair<int, NodeP>> gsum;
    for (size_t i : kv.second) {
      out.push_back({orient[i], mk(Op::Mul, {c[i], a[i]})});   // sum c_i E_i
      gsum.push_back({orient[i], c[i]});
      done[i] = 1;
    }
    NodeP V = std::make_shared<Node>();
    V->op = Op::Var;
    V->index = kv.first;
    out.push_back({-1, mk(Op::Mul, {V, signed_sum(gsum)})});  // - V sum c_i
  }
  if (out.empty()) return root;
  for (size_t i = 0; i < terms.size(); ++i) if (!done[i]) out.push_back(terms[i]);
  return signed_sum(out);
}

}  // namespace

std::vector<int> split_scales(const System& s, int sweep_param, std::vector<NodeP>* rest, std::vector<NodeP>* scale) {
  std::vector<int> slot(s.dim, -1);
  rest->assign(s.rhs.begin(), s.rhs.end());
  scale->assign(s.dim, nullptr);
  // components with the same factor share a slot (HH ring: dV_i/dt = (...)/C for every neuron), so
  // the kernel keeps fewer loop-invariant step constants in uniform registers
  std::map<std::string, int> seen;
  for (int d = 0; d < s.dim; ++d) {
    std::vector<NodeP> uni, var;
    factors(s.rhs[d], sweep_param, uni, var);
    if (uni.empty() || var.empty()) continue;  // nothing to factor out, or a constant derivative
    // a lone -1 is left to the sign selection (free there)
    if (uni.size() == 1 && uni[0]->op == Op::Num && uni[0]->value == -1.0) continue;
    const NodeP sc = product(uni);
    const std::string key = ast_key(sc);
    auto it = seen.find(key);
    if (it == seen.end()) {
      if ((int)seen.size() >= FF_MAX_SCALED) continue;
      it = seen.emplace(key, (int)seen.size()).first;
    }
    (*rest)[d] = product(var);
    (*scale)[d] = sc;
    slot[d] = it->second;
  }
  return slot;
}

double eval_uniform(const NodeP& n, const std::vector<float>& p) {
  auto A = [&](int i) { return eval_uniform(n->args[i], p); };
  switch (n->op) {
    case Op::Num: return n->value;
    case Op::Param: return (double)p.at(n->index);
    case Op::Neg: return -A(0);
    case Op::Add: return A(0) + A(1);
    case Op::Sub: return A(0) - A(1);
    case Op::Mul: return A(0) * A(1);
    case Op::Div: return A(0) / A(1);
    case Op::Pow: return std::pow(A(0), A(1));
    case Op::Var: throw Error(FF_ERR_STATE, "internal: state variable in a uniform factor");
    case Op::Call: {
      const std::string& f = n->name;
      const double x = A(0);
      if (f == "exp") return std::exp(x);
      if (f == "log") return std::log(x);
      if (f == "sin") return std::sin(x);
      if (f == "cos") return std::cos(x);
      if (f == "tan") return std::tan(x);
      if (f == "tanh") return std::tanh(x);
      if (f == "sqrt") return std::sqrt(x);
      if (f == "abs") return std::fabs(x);
      if (f == "sigmoid") return 1.0 / (1.0 + std::exp(-x));
      const double y = A(1);
      if (f == "pow") return std::pow(x, y);
      if (f == "min") return std::fmin(x, y);
      if (f == "max") return std::fmax(x, y);
      if (f == "vtrap") {
        const double u = x / y;
        return std::fabs(u) < 0.1 ? y * (1.0 - u / 2.0 + u * u / 12.0 - u * u * u * u / 720.0) : x / std::expm1(u);
      }
      throw Error(FF_ERR_STATE, "internal: unknown function " + f);
    }
  }
  return 0.0;
}

System parse_system(const ff_system* sys) {
  if (!sys) throw Error(FF_ERR_INVALID_ARG, "system is NULL");
  if (sys->dim < 1 || sys->dim > FF_MAX_DIM)
    throw Error(FF_ERR_INVALID_ARG, "dim must be in 1.." + std::to_string(FF_MAX_DIM));
  if (sys->n_params < 0 || sys->n_params > FF_MAX_PARAMS)
    throw Error(FF_ERR_INVALID_ARG, "n_params must be in 0.." + std::to_string(FF_MAX_PARAMS));
  if (!sys->var_names || !sys->rhs) throw Error(FF_ERR_INVALID_ARG, "var_names / rhs is NULL");
  if (sys->n_params > 0 && (!sys->param_names || !sys->param_default))
    throw Error(FF_ERR_INVALID_ARG, "param_names / param_default is NULL");
  System s;
  s.dim = sys->dim;
  std::map<std::string, int> vars, params;
  std::set<std::string> reserved = {"pi", "e"};
  for (auto& f : functions()) reserved.insert(f.first);
  auto check_name = [&](const char* nm, const char* what) {
    if (!nm) throw Error(FF_ERR_INVALID_ARG, std::string(what) + " name is NULL");
    std::string n(nm);
    if (!is_identifier(n)) throw Error(FF_ERR_INVALID_ARG, std::string(what) + " name '" + n + "' is not an identifier");
    if (reserved.count(n)) throw Error(FF_ERR_INVALID_ARG, std::string(what) + " name '" + n + "' shadows a builtin");
    if (vars.count(n) || params.count(n)) throw Error(FF_ERR_INVALID_ARG, "duplicate name '" + n + "'");
    return n;
  };
  for (int i = 0; i < sys->dim; ++i) {
    std::string n = check_name(sys->var_names[i], "state variable");
    vars[n] = i;
    s.var_names.push_back(n);
  }
  for (int k = 0; k < sys->n_params; ++k) {
    std::string n = check_name(sys->param_names[k], "parameter");
    params[n] = k;
    s.param_names.push_back(n);
    const float d = sys->param_default[k];
    const float lo = sys->param_min ? sys->param_min[k] : -INFINITY;
    const float hi = sys->param_max ? sys->param_max[k] : INFINITY;
    if (!std::isfinite(d)) throw Error(FF_ERR_INVALID_ARG, "default of parameter '" + n + "' is not finite");
    if (std::isnan(lo) || std::isnan(hi) || !(lo <= d && d <= hi))
      throw Error(FF_ERR_INVALID_ARG, "parameter '" + n + "' needs min <= default <= max");
    s.param_default.push_back(d);
    s.param_min.push_back(lo);
    s.param_max.push_back(hi);
  }
  for (int i = 0; i < sys->dim; ++i) {
    if (!sys->rhs[i]) throw Error(FF_ERR_INVALID_ARG, "rhs of '" + s.var_names[i] + "' is NULL");
    std::string text(sys->rhs[i]);
    Parser p(text, "rhs of '" + s.var_names[i] + "'", vars, params);
    s.rhs_text.push_back(text);
    s.rhs.push_back(p.parse_all());
  }
  return s;
}

// ================================================================ DAG + emission
namespace {

enum class K {
  Num, Var, Param, Sweep,
  Neg, Add, Sub, Mul, Rcp, Div,
  Exp2, Log, Sin, Cos, Tan, Tanh, Sqrt, Abs, Min, Max, Pow, Sigmoid2,
  SelAbsLt  // |a0| < value ? a1 : a2 (branch-free select)
};

struct DNode {
  K k = K::Num;
  double value = 0;  // Num
  int index = -1;    // Var / Param
  std::vector<int> a;
  bool uniform = true;
};

struct Dag {
  std::vector<DNode> nodes;
  std::unordered_map<std::string, int> memo;
  int sweep_param;
  // exp sharing (see exp_): pass 1 records (signature of w, c) for every 2^(c w + d); pass 2 gets a
  // plan {signature -> base coefficient c0} and derives 2^(c w + d) = 2^d (2^(c0 w))^(c/c0).
  const std::map<std::string, double>* plan = nullptr;
  std::vector<std::pair<std::string, std::pair<double, double>>> exp_uses;
  std::unordered_map<int, std::string> sigmemo;

  explicit Dag(int sp) : sweep_param(sp) {}

  int intern(DNode n) {
    std::ostringstream key;
    key << (int)n.k << ':';
    {
      uint64_t bits;
      std::memcpy(&bits, &n.value, 8);
      key << bits;
    }
    key << ':' << n.index;
    for (int x : n.a) key << ',' << x;
    auto it = memo.find(key.str());
    if (it != memo.end()) return it->second;
    if (n.k == K::Var || n.k == K::Sweep) n.uniform = false;
    else if (n.k == K::Num || n.k == K::Param) n.uniform = true;
    else {
      n.uniform = true;
      for (int x : n.a) n.uniform = n.uniform && nodes[x].uniform;
    }
    nodes.push_back(n);
    int id = (int)nodes.size() - 1;
    memo[key.str()] = id;
    return id;
  }

  bool is_num(int x) const { return nodes[x].k == K::Num; }
  double num(int x) const { return nodes[x].value; }

  int N(double v) { DNode n; n.k = K::Num; n.value = v; return intern(n); }
  int leaf(K k, int idx) { DNode n; n.k = k; n.index = idx; return intern(n); }
  int op(K k, std::vector<int> a) { DNode n; n.k = k; n.a = std::move(a); return intern(n); }

  // ---- kinetic (gating) form: a (1 - X) -/+ b X -> a - (a +/- b) X
  // Gating variables of conductance models (dh/dt = alpha_h (1 - h) - beta_h h)
  // are written in this form; the rewrite saves the (1 - X) and one product: 2 FMA-pipe ops instead
  // of 3-4 per equation (HH ring: 72 of 813 per particle-step). Exact in real arithmetic.
  int one_minus(int n) const {  // X if node n is (1 - X) with X varying, else -1
    const DNode& d = nodes[n];
    if (d.k == K::Sub && is_num(d.a[0]) && num(d.a[0]) == 1.0 && !nodes[d.a[1]].uniform) return d.a[1];
    return -1;
  }
  // node n == alpha * (1 - X)? (also u * (alpha * (1 - X)) with u uniform)
  bool gate_form(int n, int& alpha, int& X, int depth = 0) {
    const DNode d = nodes[n];  // copy: the constructors below may grow `nodes`
    if (d.k != K::Mul || depth > 2) return false;
    for (int i = 0; i < 2; ++i) {
      const int x = one_minus(d.a[i]);
      if (x >= 0) { alpha = d.a[1 - i]; X = x; return true; }
    }
    int a2, x2;
    if (nodes[d.a[0]].uniform && gate_form(d.a[1], a2, x2, depth + 1)) { alpha = mul(d.a[0], a2); X = x2; return true; }
    return false;
  }
  // node y == rest * X (X a product factor of y)?
  bool factor_out(int y, int X, int& rest, int depth = 0) {
    if (y == X) { rest = N(1.0); return true; }
    const DNode d = nodes[y];
    if (depth > 4) return false;
    int r;
    if (d.k == K::Mul) {
      if (factor_out(d.a[1], X, r, depth + 1)) { rest = mul(d.a[0], r); return true; }
      if (factor_out(d.a[0], X, r, depth + 1)) { rest = mul(r, d.a[1]); return true; }
    }
    if (d.k == K::Div && factor_out(d.a[0], X, r, depth + 1)) { rest = div(r, d.a[1]); return true; }
    if (d.k == K::Neg && factor_out(d.a[0], X, r, depth + 1)) { rest = neg(r); return true; }
    return false;
  }
  bool gating = true;

  // ---- smart constructors with constant folding and small algebraic identities
  int neg(int x) {
    if (is_num(x)) return N(-num(x));
    if (nodes[x].k == K::Neg) return nodes[x].a[0];
    return op(K::Neg, {x});
  }
  int add(int x, int y) {
    if (is_num(x) && is_num(y)) return N(num(x) + num(y));
    if (is_num(x) && num(x) == 0.0) return y;
    if (is_num(y) && num(y) == 0.0) return x;
    if (gating) {
      int al, X, r;
      if (gate_form(x, al, X) && factor_out(y, X, r)) return add(al, mul(sub(r, al), X));  // a(1-X) + rX
      if (gate_form(y, al, X) && factor_out(x, X, r)) return add(al, mul(sub(r, al), X));
    }
    if (nodes[y].k == K::Neg && !nodes[y].uniform) return sub(x, nodes[y].a[0]);
    if (nodes[x].k == K::Neg && !nodes[x].uniform) return sub(y, nodes[x].a[0]);
    if (nodes[x].uniform && !nodes[y].uniform) std::swap(x, y);
    if (nodes[y].uniform && !nodes[x].uniform) {
      // (w + u1) + u2 -> w + (u1 + u2): uniform terms gather into one loop-invariant constant
      const DNode& nx = nodes[x];
      if (nx.k == K::Add && nodes[nx.a[1]].uniform) return add(nx.a[0], add(nx.a[1], y));
      if (nx.k == K::Add && nodes[nx.a[0]].uniform) return add(nx.a[1], add(nx.a[0], y));
      if (nx.k == K::Sub && nodes[nx.a[1]].uniform) return add(nx.a[0], sub(y, nx.a[1]));
    }
    return op(K::Add, {x, y});
  }
  int sub(int x, int y) {
    if (is_num(x) && is_num(y)) return N(num(x) - num(y));
    if (is_num(y) && num(y) == 0.0) return x;
    if (gating) {
      int al, X, r;
      if (gate_form(x, al, X) && factor_out(y, X, r)) return sub(al, mul(add(al, r), X));  // a(1-X) - rX
    }
    if (is_num(x) && num(x) == 0.0) return neg(y);
    if (nodes[y].k == K::Neg) return add(x, nodes[y].a[0]);
    if (nodes[y].uniform && !nodes[x].uniform) return add(x, neg(y));
    // x - u*w with u uniform -> x + (-u)*w: the negation moves onto the loop-invariant factor, so
    // the packed path gets one FFMA2 (FFMA2 has no operand negation).
    if (nodes[y].k == K::Mul && !nodes[y].uniform) {
      const int u = nodes[y].a[0], w = nodes[y].a[1];
      if (nodes[u].uniform) return add(x, mul(neg(u), w));
      if (nodes[w].uniform) return add(x, mul(neg(w), u));
    }
    // u - (w + v), u - (w - v), u - (v - w) with u, v uniform: gather the uniform terms
    if (nodes[x].uniform && !nodes[y].uniform && (nodes[y].k == K::Add || nodes[y].k == K::Sub)) {
      const int p = nodes[y].a[0], q = nodes[y].a[1];
      if (nodes[y].k == K::Add && nodes[q].uniform) return sub(sub(x, q), p);
      if (nodes[y].k == K::Add && nodes[p].uniform) return sub(sub(x, p), q);
      if (nodes[y].k == K::Sub && nodes[q].uniform) return sub(add(x, q), p);
      if (nodes[y].k == K::Sub && nodes[p].uniform) return add(q, sub(x, p));
    }
    return op(K::Sub, {x, y});
  }
  int mul(int x, int y) {
    if (is_num(x) && is_num(y)) return N(num(x) * num(y));
    if (is_num(y)) std::swap(x, y);  // constant first
    if (nodes[y].uniform && !nodes[x].uniform) std::swap(x, y);  // uniform first
    if (is_num(x)) {
      const double c = num(x);
      if (c == 1.0) return y;
      if (c == -1.0) return neg(y);
    }
    if (nodes[x].uniform && !nodes[y].uniform) {
      const DNode& ny = nodes[y];
      // u1 * (u2 * w) -> (u1 u2) * w
      if (ny.k == K::Mul && nodes[ny.a[0]].uniform) return mul(mul(x, ny.a[0]), ny.a[1]);
      // u * (-w) -> (-u) * w
      if (ny.k == K::Neg) return mul(neg(x), ny.a[0]);
      // u * (a / b) -> (u a) / b: u a often folds (e.g. into an existing affine node)
      if (ny.k == K::Div) return div(mul(x, ny.a[0]), ny.a[1]);
      // u * select(c, a, b) -> select(c, u a, u b): the constant folds into both branches
      if (ny.k == K::SelAbsLt) {
        DNode sn;
        sn.k = K::SelAbsLt;
        sn.value = ny.value;
        sn.a = {ny.a[0], mul(x, ny.a[1]), mul(x, ny.a[2])};
        return intern(sn);
      }
      // u * (w +- v) with one uniform term -> distribute: one FFMA instead of FADD + FMUL
      if (ny.k == K::Add || ny.k == K::Sub) {
        const int p = ny.a[0], q = ny.a[1];
        if (nodes[p].uniform || nodes[q].uniform)
          return ny.k == K::Add ? add(mul(x, p), mul(x, q)) : sub(mul(x, p), mul(x, q));
      }
    }
    return op(K::Mul, {x, y});
  }
  int rcp(int x) {
    if (is_num(x)) return N(1.0 / num(x));
    if (nodes[x].k == K::Rcp) return nodes[x].a[0];
    return op(K::Rcp, {x});
  }
  int div(int x, int y) {
    if (is_num(x) && is_num(y)) return N(num(x) / num(y));
    if (is_num(y)) return mul(N(1.0 / num(y)), x);              // x / c -> (1/c) x
    if (nodes[y].uniform) return mul(x, rcp(y));                 // uniform divisor: hoisted rcp
    if (is_num(x) && num(x) == 1.0) return rcp(y);
    return op(K::Div, {x, y});                                   // x * rcp(y) per particle
  }
  // structural signature of a subtree (stable across the two lowering passes)
  const std::string& sig(int id) {
    auto it = sigmemo.find(id);
    if (it != sigmemo.end()) return it->second;
    const DNode& n = nodes[id];
    std::ostringstream o;
    if (n.k == K::Num) {
      uint64_t bits;
      std::memcpy(&bits, &n.value, 8);
      o << 'n' << bits;
    } else {
      o << 'k' << (int)n.k << '.' << n.index << '(';
      for (int x : n.a) o << sig(x) << ',';
      o << ')';
    }
    return sigmemo[id] = o.str();
  }
  // u = c w + d with c, d literal constants and w varying?
  bool affine(int u, int& w, double& c, double& d) {
    d = 0.0;
    const DNode& n = nodes[u];
    if (n.uniform) return false;
    int m = u;
    if (n.k == K::Add && is_num(n.a[1])) { d = num(n.a[1]); m = n.a[0]; }
    const DNode& nm = nodes[m];
    if (nm.k == K::Mul && is_num(nm.a[0])) { c = num(nm.a[0]); w = nm.a[1]; }
    else { c = 1.0; w = m; }
    return c != 0.0;
  }
  int powchain(int b, long r) {
    if (r == 1) return b;
    if (r % 2 == 0) { int h = powchain(b, r / 2); return mul(h, h); }
    return mul(powchain(b, r - 1), b);
  }
  int exp_(int u) {  // e^u = 2^(log2(e) u)
    if (is_num(u)) return N(std::exp(num(u)));
    const int arg = mul(N(1.4426950408889634), u);
    int w;
    double c, d;
    if (affine(arg, w, c, d)) {
      const std::string& sw = sig(w);
      exp_uses.push_back({sw, {c, d}});
      if (plan) {
        auto it = plan->find(sw);
        if (it != plan->end()) {
          const double c0 = it->second, r = c / c0, rr = std::round(r);
          if (rr >= 1 && rr <= 16 && std::fabs(r - rr) < 1e-9 && std::fabs(d) < 64) {
            const int base = op(K::Exp2, {mul(N(c0), w)});
            const int p = powchain(base, (long)rr);
            return d == 0.0 ? p : mul(N(std::exp2(d)), p);
          }
        }
      }
    }
    return op(K::Exp2, {arg});
  }
  int powi(int x, long n) {
    if (n == 0) return N(1.0);
    if (n < 0) return rcp(powi(x, -n));
    if (n == 1) return x;
    int h = powi(x, n / 2);
    int sq = mul(h, h);
    return (n % 2) ? mul(sq, x) : sq;
  }
  int pow_(int x, int y) {
    if (is_num(x) && is_num(y)) return N(std::pow(num(x), num(y)));
    if (is_num(y)) {
      const double e = num(y);
      if (e == std::floor(e) && std::fabs(e) <= 16) return powi(x, (long)e);
      if (e == 0.5) return op(K::Sqrt, {x});
    }
    return op(K::Pow, {x, y});
  }
  int call1(K k, int x, double (*f)(double)) {
    if (is_num(x)) return N(f(num(x)));
    return op(k, {x});
  }

  int lower(const NodeP& n) {
    switch (n->op) {
      case Op::Num: return N(n->value);
      case Op::Var: return leaf(K::Var, n->index);
      case Op::Param: return n->index == sweep_param ? leaf(K::Sweep, 0) : leaf(K::Param, n->index);
      case Op::Neg: return neg(lower(n->args[0]));
      case Op::Add: return add(lower(n->args[0]), lower(n->args[1]));
      case Op::Sub: return sub(lower(n->args[0]), lower(n->args[1]));
      case Op::Mul: return mul(lower(n->args[0]), lower(n->args[1]));
      case Op::Div: return div(lower(n->args[0]), lower(n->args[1]));
      case Op::Pow: return pow_(lower(n->args[0]), lower(n->args[1]));
      case Op::Call: {
        const std::string& f = n->name;
        int x = lower(n->args[0]);
        if (f == "exp") return exp_(x);
        if (f == "log") return call1(K::Log, x, [](double v) { return std::log(v); });
        if (f == "sin") return call1(K::Sin, x, [](double v) { return std::sin(v); });
        if (f == "cos") return call1(K::Cos, x, [](double v) { return std::cos(v); });
        if (f == "tan") return call1(K::Tan, x, [](double v) { return std::tan(v); });
        if (f == "tanh") return call1(K::Tanh, x, [](double v) { return std::tanh(v); });
        if (f == "sqrt") return call1(K::Sqrt, x, [](double v) { return std::sqrt(v); });
        if (f == "abs") return call1(K::Abs, x, [](double v) { return std::fabs(v); });
        if (f == "sigmoid") {  // 1 / (1 + 2^(-log2(e) u)): MUFU.EX2 + MUFU.RCP
          if (is_num(x)) return N(1.0 / (1.0 + std::exp(-num(x))));
          return op(K::Sigmoid2, {mul(N(-1.4426950408889634), x)});
        }
        int y = lower(n->args[1]);
        if (f == "pow") return pow_(x, y);
        if (f == "min") return (is_num(x) && is_num(y)) ? N(std::fmin(num(x), num(y))) : op(K::Min, {x, y});
        if (f == "max") return (is_num(x) && is_num(y)) ? N(std::fmax(num(x), num(y))) : op(K::Max, {x, y});
        if (f == "vtrap") {
          // x / (exp(x/y) - 1), and for |x/y| < 0.1 the series y (1 - u/2 + u^2/12 - u^4/720)
          // (reading R10); lowered to primitives so its exponential can be shared (exp_)
          // Horner: y (1 - u/2 + u^2 (1/12 - u^2/720)) -- 5 FMA-pipe ops for the rarely used branch
          const int u = mul(x, rcp(y));
          const int dir = div(x, sub(exp_(u), N(1.0)));
          const int u2 = mul(u, u);
          const int inner = add(mul(N(-1.0 / 720.0), u2), N(1.0 / 12.0));
          const int ser = mul(y, add(mul(inner, u2), add(mul(N(-0.5), u), N(1.0))));
          DNode sn;
          sn.k = K::SelAbsLt;
          sn.value = 0.1;
          sn.a = {u, ser, dir};
          return intern(sn);
        }
        throw Error(FF_ERR_PARSE, "internal: unhandled function " + f);
      }
    }
    throw Error(FF_ERR_PARSE, "internal: unhandled node");
  }
};

std::string flit(double v) {
  float f = (float)v;
  if (std::isnan(f)) return "__int_as_float(0x7fc00000)";
  if (std::isinf(f)) return f > 0 ? "__int_as_float(0x7f800000)" : "__int_as_float(0xff800000)";
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.9g", (double)f);
  std::string s(buf);
  if (s.find_first_of(".eE") == std::string::npos) s += ".0";
  return s + "f";
}


template <class F>
std::string node_expr(const DNode& n, F A) {
  switch (n.k) {
    case K::Neg: return "-" + A(0);
    case K::Add: return A(0) + " + " + A(1);
    case K::Sub: return A(0) + " - " + A(1);
    case K::Mul: return A(0) + " * " + A(1);
    case K::Rcp: return "ff_rcp(" + A(0) + ")";
    case K::Div: return "ff_div(" + A(0) + ", " + A(1) + ")";
    case K::Exp2: return "ff_exp2(" + A(0) + ")";
    case K::Log: return "ff_log(" + A(0) + ")";
    case K::Sin: return "ff_sin(" + A(0) + ")";
    case K::Cos: return "ff_cos(" + A(0) + ")";
    case K::Tan: return "ff_tan(" + A(0) + ")";
    case K::Tanh: return "ff_tanh(" + A(0) + ")";
    case K::Sqrt: return "ff_sqrt(" + A(0) + ")";
    case K::Abs: return "ff_abs(" + A(0) + ")";
    case K::Min: return "ff_min(" + A(0) + ", " + A(1) + ")";
    case K::Max: return "ff_max(" + A(0) + ", " + A(1) + ")";
    case K::Pow: return "ff_pow(" + A(0) + ", " + A(1) + ")";
    case K::Sigmoid2: return "ff_rcp(1.0f + ff_exp2(" + A(0) + "))";
    case K::SelAbsLt: return "ff_sel_abs_lt(" + A(0) + ", " + A(1) + ", " + A(2) + ", " + flit(n.value) + ")";
    default: throw Error(FF_ERR_COMPILE, "internal: unexpected node in expr()");
  }
}


// ---------------------------------------------------------------- sign-aware instruction selection
// FFMA2 / FADD2 / FMUL2 (the packed pair path) have no operand negation, so every "-v" of a
// varying value costs an instruction, while negating a uniform (loop-invariant) value is free. For
// every varying node this computes the cheapest way to produce +v and -v (cost = packed FMA-pipe
// instructions, FFMA fusion of single-use products included) and emits the chosen forms. The root of
// a component may be produced negated; the integrator then uses negated step constants.
struct Operand { int node; int neg; };
struct Choice { enum Form { ADD, SUB, FMA, MUL, DIV, OTHER, NEGATE } form; Operand op[3]; };

// host-evaluated loop-invariant values shared by every emitted RHS variant: (node, negate) -> q slot
struct QTable {
  std::map<std::pair<int, int>, int> slot;
  std::vector<std::pair<int, int>> list;
};

struct SignSelect {
  const Dag& g;
  const std::vector<char>& live;
  std::vector<int> uses, addsub_uses;
  std::vector<double> c[2];
  std::map<std::pair<int, int>, std::string> memo;
  std::vector<std::string> uref;
  std::ostringstream body;
  int n_arith = 0, n_mufu = 0, tmp = 0;

  std::set<int> emul;  // exponentials computed on the FMA pipe (ff_exp2p) instead of MUFU.EX2
  static constexpr int kExp2pOps = 8;
  // sigmoid pairs sharing one reciprocal: 1/dA = dB / (dA dB), 1/dB = dA / (dA dB) (pipe balancing)
  std::map<int, int> pair_of;
  static constexpr int kPairOps = 3;   // dA dB, dB P, dA P (the clamps run on the ALU pipe)
  // the pairs' reciprocals on the FMA pipe (ff_rcpp: 6 FMA-pipe ops and the negation of the
  // denominator, which packed FFMA2 cannot fold into an operand; + 1 integer op)
  bool rcpp = false;
  static constexpr int kRcppOps = 7;
  QTable own_q;
  QTable* qt;
  SignSelect(const Dag& dag, const std::vector<char>& lv, const std::vector<int>& roots, std::set<int> em = {},
             std::map<int, int> pairs = {}, QTable* shared_q = nullptr)
      : g(dag), live(lv), uses(dag.nodes.size(), 0), uref(dag.nodes.size()), emul(std::move(em)),
        pair_of(std::move(pairs)), qt(shared_q ? shared_q : &own_q) {
    c[0].assign(g.nodes.size(), 0.0);
    c[1].assign(g.nodes.size(), 0.0);
    addsub_uses.assign(g.nodes.size(), 0);
    for (size_t id = 0; id < g.nodes.size(); ++id)
      if (live[id])
        for (int a : g.nodes[id].a) {
          ++uses[a];
          if (g.nodes[id].k == K::Add || g.nodes[id].k == K::Sub) ++addsub_uses[a];
        }
    for (int r : roots) ++uses[r];
    for (size_t id = 0; id < g.nodes.size(); ++id) {
      if (!live[id]) continue;
      Choice ch;
      c[0][id] = best((int)id, 0, ch);
      c[1][id] = best((int)id, 1, ch);
    }
  }

  double cost(int id, int s) const { return c[s][id]; }
  // An FFMA2 whose three operands are all per-particle registers runs at 87 lane-ops/clk/SM against
  // 126 with an immediate or uniform operand (register-file read bandwidth; measured on B200,
  // tools/ubench/pipes.cu): charge it ~0.45 extra issue, so a*b + u*c becomes fma(u, c, a*b)
  // rather than fma(a, b, u*c) -- the same instruction count, faster.
  double reg3(const Operand& x, const Operand& y, int z) const {
    return (!g.nodes[x.node].uniform && !g.nodes[y.node].uniform && !g.nodes[z].uniform) ? 0.45 : 0.0;
  }
  // a varying product whose every use is an addition / subtraction: each user absorbs it into an
  // FFMA (duplicating the multiply costs nothing), so it is never materialised on its own
  bool fusable(int id) const {
    const DNode& n = g.nodes[id];
    return n.k == K::Mul && !n.uniform && uses[id] == addsub_uses[id];
  }
  // cheapest factor signs (sx, sy) with sx xor sy = s for the product node m
  double prod(int m, int s, Operand& x, Operand& y) const {
    const int a = g.nodes[m].a[0], b = g.nodes[m].a[1];
    double bestc = 1e30;
    x = {a, 0};
    y = {b, s};
    for (int sa = 0; sa < 2; ++sa) {
      const int sb = sa ^ s;
      const double v = c[sa][a] + c[sb][b];
      if (v < bestc) { bestc = v; x = {a, sa}; y = {b, sb}; }
    }
    return bestc;
  }

  double best(int id, int s, Choice& ch) const {
    const DNode& n = g.nodes[id];
    if (n.uniform) return 0.0;
    const double INF = 1e30;
    double bc = INF;
    auto consider = [&](double v, Choice cand) { if (v < bc) { bc = v; ch = cand; } };
    switch (n.k) {
      case K::Var: return s ? 1.0 : 0.0;
      case K::Sweep: return 0.0;
      case K::Neg: return c[s ^ 1][n.a[0]];
      case K::Add:
      case K::Sub: {
        const int a = n.a[0], b = n.a[1];
        const int sb = n.k == K::Add ? s : (s ^ 1);  // value = (s a) + (sb b)
        consider(1 + c[s][a] + c[sb][b], {Choice::ADD, {{a, s}, {b, sb}, {}}});
        consider(1 + c[s][a] + c[sb ^ 1][b], {Choice::SUB, {{a, s}, {b, sb ^ 1}, {}}});
        consider(1 + c[sb][b] + c[s ^ 1][a], {Choice::SUB, {{b, sb}, {a, s ^ 1}, {}}});
        Operand x, y;
        if (fusable(a)) {
          double v = 1 + prod(a, s, x, y) + c[sb][b] + reg3(x, y, b);
          consider(v, {Choice::FMA, {x, y, {b, sb}}});
        }
        if (fusable(b)) {
          double v = 1 + prod(b, sb, x, y) + c[s][a] + reg3(x, y, a);
          consider(v, {Choice::FMA, {x, y, {a, s}}});
        }
        break;
      }
      case K::Mul: {
        Operand x, y;
        double v = 1 + prod(id, s, x, y);
        consider(v, {Choice::MUL, {x, y, {}}});
        break;
      }
      case K::Div: {  // a * rcp(b): rcp(-b) = -rcp(b)
        const int a = n.a[0], b = n.a[1];
        for (int sa = 0; sa < 2; ++sa)
          consider(2 + c[sa][a] + c[sa ^ s][b], {Choice::DIV, {{a, sa}, {b, sa ^ s}, {}}});
        break;
      }
      case K::Rcp:
        consider(1 + c[s][n.a[0]], {Choice::OTHER, {{n.a[0], s}, {}, {}}});
        break;
      default: {
        double v = 1;
        for (int x : n.a) v += c[0][x];
        if (s == 0) consider(v, {Choice::OTHER, {}});
        else consider(v + 1, {Choice::NEGATE, {}});
      }
    }
    return bc;
  }

  // host-evaluated loop-invariant values: (node, negate) -> q slot (table shared by the variants)
  std::string qref(int id, int s) {
    auto key = std::make_pair(id, s);
    auto it = qt->slot.find(key);
    if (it != qt->slot.end()) return "a.q[" + std::to_string(it->second) + "]";
    if ((int)qt->list.size() >= FF_MAX_DERIVED) return "";
    const int k = (int)qt->list.size();
    qt->list.push_back(key);
    qt->slot[key] = k;
    return "a.q[" + std::to_string(k) + "]";
  }

  // both sigmoids of a pair, computed together; returns the temporary holding node `id`
  std::string paired_sigmoid(int id) {
    const int a = std::min(id, pair_of.at(id)), b = std::max(id, pair_of.at(id));
    auto e = [&](int n) {
      const std::string u = get(g.nodes[n].a[0], 0);
      if (emul.count(n)) { n_arith += kExp2pOps; return "ff_exp2p(" + u + ")"; }
      ++n_mufu;
      return "ff_exp2(" + u + ")";
    };
    const std::string ea = e(a), eb = e(b);
    const std::string da = "t" + std::to_string(tmp++), db = "t" + std::to_string(tmp++);
    const std::string pr = "t" + std::to_string(tmp++), sa = "t" + std::to_string(tmp++), sb = "t" + std::to_string(tmp++);
    // exponentials clamped at 2^60 so the product stays finite (a sigmoid below 1e-18 is 0 here)
    body << "  const V " << da << " = 1.0f + ff_min(" << ea << ", 1.15292150e18f);\n";
    body << "  const V " << db << " = 1.0f + ff_min(" << eb << ", 1.15292150e18f);\n";
    body << "  const V " << pr << " = " << (rcpp ? "ff_rcpp(" : "ff_rcp(") << da << " * " << db << ");\n";
    body << "  const V " << sa << " = " << db << " * " << pr << ";\n";
    body << "  const V " << sb << " = " << da << " * " << pr << ";\n";
    n_arith += 2 + kPairOps + (rcpp ? kRcppOps : 0);
    n_mufu += rcpp ? 0 : 1;
    memo[{a, 0}] = sa;
    memo[{b, 0}] = sb;
    return memo[{id, 0}];
  }

  std::string ureference(int id) {
    if (!uref[id].empty()) return uref[id];
    const DNode& n = g.nodes[id];
    auto A = [&](int j) { return ureference(n.a[j]); };
    std::string e;
    switch (n.k) {
      case K::Num: return uref[id] = flit(n.value);
      case K::Param: return uref[id] = "a.p[" + std::to_string(n.index) + "]";
      default: e = expr(n, A); break;
    }
    std::string name = "u" + std::to_string(id);
    body << "  const float " << name << " = " << e << ";\n";
    return uref[id] = name;
  }

  template <class F>
  std::string expr(const DNode& n, F A) { return node_expr(n, A); }

  std::string get(Operand o) { return get(o.node, o.neg); }

  // reference to an expression equal to (s ? -v : v)
  std::string get(int id, int s) {
    const DNode& n = g.nodes[id];
    if (n.uniform) {
      if (n.k == K::Num) return flit(s ? -n.value : n.value);
      if (n.k == K::Param && !s) return "a.p[" + std::to_string(n.index) + "]";
      const std::string q = qref(id, s);   // computed by the host (UProgram), read from the constant bank
      if (!q.empty()) return q;
      return s ? "(-" + ureference(id) + ")" : ureference(id);
    }
    if (n.k == K::Neg) return get(n.a[0], s ^ 1);
    if (n.k == K::Sweep) return s ? "nsw" : "sw";
    if (n.k == K::Var && s == 0) return "x[" + std::to_string(n.index) + "]";
    auto key = std::make_pair(id, s);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    std::string e;
    if (n.k == K::Var) {
      e = "-x[" + std::to_string(n.index) + "]";
      ++n_arith;
    } else {
      Choice ch;
      best(id, s, ch);
      switch (ch.form) {
        case Choice::ADD: e = get(ch.op[0]) + " + " + get(ch.op[1]); ++n_arith; break;
        case Choice::SUB: e = get(ch.op[0]) + " - " + get(ch.op[1]); ++n_arith; break;
        case Choice::MUL: e = get(ch.op[0]) + " * " + get(ch.op[1]); ++n_arith; break;
        case Choice::FMA: e = "ff_fma(" + get(ch.op[0]) + ", " + get(ch.op[1]) + ", " + get(ch.op[2]) + ")"; ++n_arith; break;
        case Choice::DIV: e = "ff_div(" + get(ch.op[0]) + ", " + get(ch.op[1]) + ")"; ++n_arith; ++n_mufu; break;
        case Choice::OTHER:
          if (n.k == K::Rcp) { e = "ff_rcp(" + get(ch.op[0]) + ")"; ++n_mufu; break; }
          if (emul.count(id) && n.k == K::Exp2) {  // on the FMA pipe (pipe balancing)
            e = "ff_exp2p(" + get(n.a[0], 0) + ")";
            n_arith += kExp2pOps;
            break;
          }
          if (n.k == K::Sigmoid2 && pair_of.count(id)) return paired_sigmoid(id);
          if (emul.count(id) && n.k == K::Sigmoid2) {
            e = "ff_rcp(1.0f + ff_exp2p(" + get(n.a[0], 0) + "))";
            n_arith += kExp2pOps + 1;
            ++n_mufu;
            break;
          }
          e = expr(n, [&](int j) { return get(n.a[j], 0); });
          count(n);
          break;
        case Choice::NEGATE:
          e = "-" + get(id, 0);
          ++n_arith;
          break;
      }
    }
    std::string name = "t" + std::to_string(tmp++);
    body << "  const V " << name << " = " << e << ";\n";
    memo[key] = name;
    return name;
  }

  void count(const DNode& n) {
    switch (n.k) {
      case K::Exp2: case K::Log: case K::Sin: case K::Cos: case K::Tanh: case K::Sqrt: ++n_mufu; break;
      case K::Tan: n_mufu += 3; break;
      case K::Pow: n_mufu += 2; ++n_arith; break;
      case K::Sigmoid2: n_mufu += 2; ++n_arith; break;
      case K::SelAbsLt: n_arith += 2; break;
      default: ++n_arith;
    }
  }
};

}  // namespace

std::vector<float> eval_program(const UProgram& prog, const std::vector<float>& p) {
  std::vector<double> v(prog.ops.size());
  for (size_t i = 0; i < prog.ops.size(); ++i) {
    const UProgram::Op& o = prog.ops[i];
    auto A = [&](int j) { return v[o.a[j]]; };
    double r = 0.0;
    switch ((K)o.kind) {
      case K::Num: r = o.value; break;
      case K::Param: r = (double)p.at(o.index); break;
      case K::Neg: r = -A(0); break;
      case K::Add: r = A(0) + A(1); break;
      case K::Sub: r = A(0) - A(1); break;
      case K::Mul: r = A(0) * A(1); break;
      case K::Rcp: r = 1.0 / A(0); break;
      case K::Div: r = A(0) / A(1); break;
      case K::Exp2: r = std::exp2(A(0)); break;
      case K::Log: r = std::log(A(0)); break;
      case K::Sin: r = std::sin(A(0)); break;
      case K::Cos: r = std::cos(A(0)); break;
      case K::Tan: r = std::tan(A(0)); break;
      case K::Tanh: r = std::tanh(A(0)); break;
      case K::Sqrt: r = std::sqrt(A(0)); break;
      case K::Abs: r = std::fabs(A(0)); break;
      case K::Min: r = std::fmin(A(0), A(1)); break;
      case K::Max: r = std::fmax(A(0), A(1)); break;
      case K::Pow: r = std::pow(A(0), A(1)); break;
      case K::Sigmoid2: r = 1.0 / (1.0 + std::exp2(A(0))); break;
      case K::SelAbsLt: r = std::fabs(A(0)) < o.value ? A(1) : A(2); break;
      case K::Var:
      case K::Sweep: throw Error(FF_ERR_STATE, "internal: per-particle value in a uniform program");
    }
    v[i] = r;
  }
  std::vector<float> q;
  for (const auto& e : prog.q) q.push_back((float)(e.second ? -v[e.first] : v[e.first]));
  return q;
}

std::string emit_source(const System& s, int sweep_param, int kernel_select, UProgram* prog, bool balance,
                        bool long_launch, bool thread_redraw, int push) {
  if (sweep_param < -1 || sweep_param >= (int)s.param_names.size())
    throw Error(FF_ERR_INVALID_ARG, "sweep parameter index out of range");
  // pass 1: lower once to find exponentials sharing an affine argument c w + d
  std::map<std::string, double> plan;
  {
    Dag g1(sweep_param);
    for (int i = 0; i < s.dim; ++i) g1.lower(s.rhs[i]);
    std::map<std::string, std::set<std::pair<double, double>>> by_w;
    for (auto& e : g1.exp_uses) by_w[e.first].insert(e.second);
    for (auto& kv : by_w) {
      if (kv.second.size() < 2) continue;
      double best_c0 = 0;
      size_t best_n = 0;
      for (auto& cand : kv.second) {
        const double c0 = cand.first;
        size_t n = 0;
        for (auto& o : kv.second) {
          const double r = o.first / c0, rr = std::round(r);
          if (rr >= 1 && rr <= 16 && std::fabs(r - rr) < 1e-9) ++n;
        }
        if (n > best_n || (n == best_n && std::fabs(c0) < std::fabs(best_c0))) { best_n = n; best_c0 = c0; }
      }
      if (best_n >= 2) plan[kv.first] = best_c0;
    }
  }
  // the plain formulation's op count (no gating rewrite, no factored scales, no exponential
  // sharing): the fixed algorithmic work per evaluation that bench.py's roofline counts
  int n_arith_plain = 0, n_mufu_plain = 0, n_exp_plain = 0, n_sig_plain = 0;
  {
    Dag gp(sweep_param);
    gp.gating = false;
    std::vector<int> rp;
    for (int i = 0; i < s.dim; ++i) rp.push_back(gp.lower(s.rhs[i]));
    std::vector<char> lv(gp.nodes.size(), 0);
    std::function<void(int)> mk = [&](int x) {
      if (lv[x]) return;
      lv[x] = 1;
      for (int y : gp.nodes[x].a) mk(y);
    };
    for (int r : rp) mk(r);
    SignSelect sp(gp, lv, rp);
    for (int i = 0; i < s.dim; ++i) {
      const int r = rp[i];
      sp.get(r, (!gp.nodes[r].uniform && sp.cost(r, 1) < sp.cost(r, 0)) ? 1 : 0);
    }
    n_arith_plain = sp.n_arith;
    n_mufu_plain = sp.n_mufu;
    for (size_t id = 0; id < gp.nodes.size(); ++id)
      if (lv[id] && !gp.nodes[id].uniform && (gp.nodes[id].k == K::Exp2 || gp.nodes[id].k == K::Sigmoid2)) {
        ++n_exp_plain;
        n_sig_plain += gp.nodes[id].k == K::Sigmoid2;
      }
  }
  // pass 2: lower with the sharing plan; split components are lowered without their uniform factor
  std::vector<NodeP> rest, scale_ast;
  const std::vector<int> slot = split_scales(s, sweep_param, &rest, &scale_ast);
  Dag g(sweep_param);
  g.plan = &plan;
  std::vector<int> roots;
  for (int i = 0; i < s.dim; ++i) roots.push_back(g.lower(collect_linear(rest[i], sweep_param)));

  // reachable nodes in topological (creation) order
  std::vector<char> live(g.nodes.size(), 0);
  std::function<void(int)> mark = [&](int x) {
    if (live[x]) return;
    live[x] = 1;
    for (int y : g.nodes[x].a) mark(y);
  };
  for (int r : roots) mark(r);

  // Pipe balancing: a system bound by the MUFU pipe (16 results / clk / SM against 128 FP32 lanes)
  // moves work to the FMA pipe: (1) sigmoids in pairs share one reciprocal (1/dA = dB/(dA dB): one
  // MUFU.RCP instead of two, for 3 FMA-pipe ops), (2) K of the exponentials of a particle-step (4 RHS
  // evaluations) run as ff_exp2p (8 FMA-pipe ops each), (3) in R of the 4 RK4 stages the pairs'
  // shared reciprocals run as ff_rcpp (7 FMA-pipe ops each). K is split over the 4 RK4 stages (k or
  // k + 1 per stage: two emitted RHS variants; with R > 0 the second variant is k + FMA-pipe
  // reciprocals instead), so the balance is set per particle-step, not per evaluation. Chosen to
  // minimise max(MUFU / 16, FMA / 128) per particle-step (RK4 combination in).
  std::vector<int> cand;   // exponentials (exp / sigmoid nodes), in creation order
  std::vector<int> sigs;   // sigmoid nodes
  for (size_t id = 0; id < g.nodes.size(); ++id)
    if (live[id] && !g.nodes[id].uniform && (g.nodes[id].k == K::Exp2 || g.nodes[id].k == K::Sigmoid2)) {
      cand.push_back((int)id);
      if (g.nodes[id].k == K::Sigmoid2) sigs.push_back((int)id);
    }
  std::map<int, int> pairs;
  for (size_t i = 0; i + 1 < sigs.size(); i += 2) {
    pairs[sigs[i]] = sigs[i + 1];
    pairs[sigs[i + 1]] = sigs[i];
  }
  auto probe_counts = [&](const std::map<int, int>& pr, double& a, double& m) {
    SignSelect probe(g, live, roots, {}, pr);
    for (int i = 0; i < s.dim; ++i) {
      const int r = roots[i];
      probe.get(r, (!g.nodes[r].uniform && probe.cost(r, 1) < probe.cost(r, 0)) ? 1 : 0);
    }
    a = probe.n_arith;
    m = probe.n_mufu;
  };
  bool use_pairs = false;
  int K = 0;   // exponentials per particle-step on the FMA pipe
  // selection cost of one ff_exp2p: its 8 FMA-pipe ops plus ~4 issue slots of ALU work (clamp,
  // exponent assembly); measured on B200 (STN-GPe bifurcation, sigmoid pairs on): K = 0, 1, 2, 3 per
  // particle-step -> 3.56, 3.64, 3.35, 3.07e11 particle-steps/s, which a cost of 8 would mis-rank
  constexpr double kExp2pCost = 12.0;
  // the same for a pair reciprocal on the FMA pipe (ff_rcpp, 7 ops): measured on the STN-GPe
  // bifurcation with pairs and no exponential moved, R = 0..4 stages -> 3.58, 3.70, 3.44, 3.18,
  // 2.98e11 (tools/r01/gpu_run62.sh), which a cost of 12 ranks; ties go to fewer executed ops
  constexpr double kRcppCost = 12.0;
  int R = 0;   // stages (of 4) whose pair reciprocals run on the FMA pipe (with k_lo exponentials)
  const int n_pair_eval = (int)pairs.size() / 2;
  if (balance) {
    double best_t = 1e30, best_ops = 1e30;
    auto take = [&](double t, double ops, int k, int r, bool pv) {
      if (t < best_t - 1e-9 || (t < best_t + 1e-9 && ops < best_ops - 1e-9)) {
        best_t = t; best_ops = ops; K = k; R = r; use_pairs = pv;
      }
    };
    for (int pv = 0; pv < (pairs.empty() ? 1 : 2); ++pv) {
      double a, m;
      probe_counts(pv ? pairs : std::map<int, int>{}, a, m);
      const double A = 4 * a + 7.0 * s.dim, M = 4 * m;
      for (int k = 0; k <= 4 * (int)cand.size(); ++k)
        take(std::max((M - k) / 16.0, (A + kExp2pCost * k) / 128.0), A + SignSelect::kExp2pOps * k, k, 0, pv);
      if (pv)   // k_lo exponentials in every stage, the pair reciprocals of r stages on the FMA pipe
        for (int k = 0; k <= (int)cand.size(); ++k)
          for (int r = 1; r <= 4; ++r) {
            const double mr = M - 4 * k - r * n_pair_eval;
            const double t = std::max(mr / 16.0, (A + kExp2pCost * 4 * k + kRcppCost * r * n_pair_eval) / 128.0);
            take(t, A + SignSelect::kExp2pOps * 4 * k + SignSelect::kRcppOps * r * n_pair_eval, 4 * k, r, true);
          }
    }
    if (const char* e = std::getenv("FF_TUNE_EXP2P"))   // exponentials per evaluation, every stage
      K = 4 * std::min((int)cand.size(), std::max(0, std::atoi(e)));
    if (const char* e = std::getenv("FF_TUNE_EXP2P_STEP"))   // exponentials per particle-step
      K = std::min(4 * (int)cand.size(), std::max(0, std::atoi(e)));
    if (std::getenv("FF_TUNE_EXP2P") || std::getenv("FF_TUNE_EXP2P_STEP")) R = 0;
    if (const char* e = std::getenv("FF_TUNE_RCPP_STAGES")) {   // (K then rounds down to 4 k_lo)
      R = std::min(4, std::max(0, std::atoi(e)));
      if (R) K -= K % 4;
    }
    if (const char* e = std::getenv("FF_TUNE_RCP_PAIRS")) use_pairs = std::atoi(e) != 0 && !pairs.empty();
    if (!use_pairs) R = 0;
  }
  // stages 0 .. n_hi-1 run variant 1: k_lo + 1 exponentials on the FMA pipe, or (R > 0) k_lo and
  // their pair reciprocals on the FMA pipe
  const bool hi_rcpp = R > 0;
  const int k_lo = K / 4, n_hi = hi_rcpp ? R : K % 4;
  auto emul_set = [&](int k) {
    std::set<int> e;
    for (int i = 0; i < k && i < (int)cand.size(); ++i) e.insert(cand[i]);
    return e;
  };
  QTable qtab;
  const std::map<int, int> used_pairs = use_pairs ? pairs : std::map<int, int>{};
  SignSelect sel(g, live, roots, emul_set(k_lo), used_pairs, &qtab);
  std::vector<int> sign(s.dim, 1);
  std::vector<std::string> out(s.dim);
  for (int i = 0; i < s.dim; ++i) {
    const int r = roots[i];
    if (!g.nodes[r].uniform && sel.cost(r, 1) < sel.cost(r, 0)) sign[i] = -1;
    out[i] = sel.get(r, sign[i] < 0 ? 1 : 0);
  }
  // the second variant (one more exponential on the FMA pipe), same signs and q table
  SignSelect sel_hi(g, live, roots, emul_set(hi_rcpp ? k_lo : k_lo + 1), used_pairs, &qtab);
  sel_hi.rcpp = hi_rcpp;
  std::vector<std::string> out_hi(s.dim);
  if (n_hi)
    for (int i = 0; i < s.dim; ++i) out_hi[i] = sel_hi.get(roots[i], sign[i] < 0 ? 1 : 0);
  // per particle-step (4 evaluations)
  const int n_arith = (4 - n_hi) * sel.n_arith + n_hi * sel_hi.n_arith;
  const int n_mufu = (4 - n_hi) * sel.n_mufu + n_hi * sel_hi.n_mufu;
  if (prog) {  // the q values as a host program: every uniform node they reach, in creation order
    prog->ops.clear();
    prog->q.clear();
    prog->mufu_per_step = n_mufu;
    std::map<int, int> at;
    std::function<int(int)> put = [&](int id) -> int {
      auto it = at.find(id);
      if (it != at.end()) return it->second;
      const DNode& n = g.nodes[id];
      UProgram::Op o{(int)n.k, n.value, n.index, {0, 0, 0}};
      for (size_t j = 0; j < n.a.size() && j < 3; ++j) o.a[j] = put(n.a[j]);
      prog->ops.push_back(o);
      return at[id] = (int)prog->ops.size() - 1;
    };
    for (const auto& e : qtab.list) prog->q.push_back({put(e.first), e.second});
  }
  std::ostringstream rhs;
  rhs << "// Generated right-hand side (" << s.dim << " state variables, " << s.param_names.size()
      << " parameters, swept parameter index " << sweep_param << ").\n";
  // (user text goes into // comments: control characters -- a multi-line expression's newlines --
  // become spaces so nothing leaks out of the comment into the source)
  auto one_line = [](std::string t) {
    for (char& ch : t)
      if (static_cast<unsigned char>(ch) < 0x20 || ch == 0x7f) ch = ' ';
    return t;
  };
  for (int i = 0; i < s.dim; ++i) rhs << "//   d" << s.var_names[i] << "/dt = " << one_line(s.rhs_text[i]) << "\n";
  for (size_t k = 0; k < s.param_names.size(); ++k)
    rhs << "//   a.p[" << k << "] = " << s.param_names[k]
        << ((int)k == sweep_param ? "  (swept: the per-particle value sw is used instead)" : "") << "\n";
  rhs << "// per particle-step, 4 evaluations (front-end count): " << n_arith << " arithmetic ops, " << n_mufu
      << " MUFU ops\n";
  rhs << "// exponentials on the FMA pipe per particle-step (pipe balancing): " << K
      << "; sigmoid pairs sharing a reciprocal: " << (use_pairs ? (int)pairs.size() / 2 : 0)
      << "; stages with the pair reciprocals on the FMA pipe: " << R << "\n";
  rhs << "// plain formulation (no gating rewrite, uniform factors multiplied in every evaluation, no exponential sharing): "
      << n_arith_plain << " arithmetic ops, " << n_mufu_plain << " MUFU ops, " << n_exp_plain << " exponentials, "
      << n_sig_plain / 2 << " sigmoid pairs\n";
  auto emit_rhs = [&](const std::string& fname, SignSelect& ss, const std::vector<std::string>& o) {
    rhs << "template <class V>\n__device__ __forceinline__ void " << fname
        << "(const V* __restrict__ x, V* __restrict__ dx, const FFStepArgs& a, const V& sw) {\n";
    rhs << "  (void)a; (void)sw;\n";
    rhs << "  const V nsw = -sw; (void)nsw;\n";
    rhs << ss.body.str();
    for (int i = 0; i < s.dim; ++i) {
      const DNode& r = g.nodes[roots[i]];
      rhs << "  dx[" << i << "] = " << (r.uniform ? "ff_bcast<V>(" + o[i] + ")" : o[i]) << ";"
          << (sign[i] < 0 || slot[i] >= 0 ? "  // = d" + s.var_names[i] + "/dt" + (sign[i] < 0 ? " * (-1)" : "") +
                                                (slot[i] >= 0 ? " / scale" : "") : "")
          << "\n";
    }
    rhs << "}\n";
  };
  emit_rhs("ff_rhs_v0", sel, out);
  if (n_hi) emit_rhs("ff_rhs_v1", sel_hi, out_hi);
  // RK4 stage s evaluates variant FF_STAGE_VAR[s] (pipe balancing per particle-step)
  rhs << "__device__ constexpr int FF_STAGE_VAR[4] = {";
  for (int st = 0; st < 4; ++st) rhs << (st ? ", " : "") << (st < n_hi ? 1 : 0);
  rhs << "};\n";
  rhs << "template <int STAGE, class V>\n__device__ __forceinline__ void ff_rhs(const V* __restrict__ x, "
         "V* __restrict__ dx, const FFStepArgs& a, const V& sw) {\n";
  if (n_hi) rhs << "  if (FF_STAGE_VAR[STAGE]) ff_rhs_v1<V>(x, dx, a, sw); else ff_rhs_v0<V>(x, dx, a, sw);\n";
  else rhs << "  ff_rhs_v0<V>(x, dx, a, sw);\n";
  rhs << "}\n";
  rhs << "// dx[d] holds FF_SIGN[d] * f_d(x) / scale_d: a component computed negated saves FFMA2\n"
         "// negations, a uniform factor scale_d (slot FF_SSLOT[d] >= 0) saves a multiply; the integrator\n"
         "// uses step constants with both folded in (host-computed per launch and group: FFStepArgs hs).\n";
  rhs << "__device__ constexpr float FF_SIGN[FF_DIM] = {";
  for (int i = 0; i < s.dim; ++i) rhs << (i ? ", " : "") << (sign[i] < 0 ? "-1.0f" : "1.0f");
  rhs << "};\n";
  rhs << "__device__ constexpr int FF_SSLOT[FF_DIM] = {";
  for (int i = 0; i < s.dim; ++i) rhs << (i ? ", " : "") << slot[i];
  rhs << "};\n";
  const int dim = s.dim;
  // RK4 steps per unrolled loop iteration; small systems, measured on B200 (tools/r01/gpu_run70.sh):
  // FMA-bound Lorenz 2 > 3 > 4 (S = 100: 8.13 / 8.09 / 8.07e11), MUFU-bound STN-GPe 8 > 4 (3.74 /
  // 3.69e11: more independent MUFU work in flight per warp)
  // (HH ring, 15 variables: 2 steps per iteration 2445 -> 2391 us per 100-step frame, 3: 2627 us,
  // tools/r02/run29.sh)
  int unroll = dim <= 4 ? (n_mufu > 0 ? 8 : 2) : (dim <= 16 ? 2 : 1);
  int minb_p1 = dim <= 4 ? 4 : (dim <= 8 ? 3 : (dim <= 16 ? 2 : 1));
  // (small systems run the 256-thread packed kernel for launches of >= 50 steps: 6 blocks / <= 40
  // registers, tools/r01/gpu_run73.sh)
  int minb_p2 = dim <= 4 ? 6 : (dim <= 8 ? 2 : 1);
  // 128-thread packed kernel, small systems: 12 blocks / <= 40 registers. Launches of many steps are
  // FMA-pipe bound and run best there (measured on B200, Lorenz 8.4 M, tools/r01/gpu_run66.sh /
  // gpu_run67.sh: S = 100 7.91 -> 8.06e11, S = 1000 8.32 -> 8.46e11, S = 10 +1% over 16 blocks);
  // round 1 kept full occupancy (16 blocks, <= 32 registers) for launches of a few steps, but with
  // the packed 3-D binning and the reset rule of the bench workload the 32-register build spills and
  // 12 blocks win there too (S = 1 / 2 / 4 / 7: 93.1 -> 88.7, 120 -> 117, 136 -> 131, 164 -> 162 us,
  // tools/r02/run13.sh). tests/test_sass.py checks that the inner loops do not spill.
  int minb_p2_t128 = dim <= 4 ? 12 : (dim <= 8 ? 4 : 2);
  (void)long_launch;
  if (const char* e = std::getenv("FF_TUNE_MINB_P2_T128")) minb_p2_t128 = std::atoi(e);
  // 4 particles per thread, 128-thread blocks, 8 blocks / <= 64 registers: 1-4-step launches of small
  // systems, with or without an image (memory / L2-bound; round 1 ran them at 6 blocks: S = 1 without
  // an image 44 -> 39 us, with one 79 -> 75 us, tools/r02/run45.sh), and long launches of FMA-bound
  // small systems (two FFMA2 chains per thread: Lorenz S = 100 8.22 -> 8.41e11, tools/r01/gpu_run76.sh)
  int minb_p4 = dim <= 4 ? 8 : (dim <= 8 ? 2 : 1);
  if (const char* e = std::getenv("FF_TUNE_MINB_P4")) minb_p4 = std::atoi(e);
  // tuning knobs for experiments (not part of the ABI): FF_TUNE_MINB_P2, FF_TUNE_UNROLL
  if (const char* e = std::getenv("FF_TUNE_MINB_P2")) minb_p2 = std::atoi(e);
  if (const char* e = std::getenv("FF_TUNE_UNROLL")) unroll = std::atoi(e);
  std::ostringstream pre;
  pre << "// Fireflies kernels, generated by the libfireflies front end for sm_100a.\n";
  pre << "#define FF_DIM " << dim << "\n";
  pre << "#define FF_NP " << s.param_names.size() << "\n";
  pre << "#define FF_NP_ALLOC " << (s.param_names.empty() ? 1 : s.param_names.size()) << "\n";
  pre << "#define FF_UNROLL " << unroll << "\n";
  pre << "#define FF_MINB_P1 " << minb_p1 << "\n";
  pre << "#define FF_MINB_P2 " << minb_p2 << "\n";
  pre << "#define FF_MINB_P2_T128 " << minb_p2_t128 << "\n";
  pre << "#define FF_MINB_P4 " << minb_p4 << "\n";
  pre << "#define FF_SWEEP " << sweep_param << "\n";
  pre << "#define FF_KSEL " << kernel_select << "\n";
  // reset redraw of the 4-particles-per-thread kernel: per thread for launches of >= 50 steps (nearly
  // every reset-prone particle resets each launch), warp-cooperative otherwise (ff_reset)
  pre << "#define FF_THREAD_REDRAW " << (thread_redraw ? 1 : 0) << "\n";
  // fused (push) image exchange: where the histogram's reductions go (ff_img_add; 0 = the bound image)
  if (push) pre << "#define FF_PUSH " << push << "\n";

  std::string tmpl(kDeviceTemplate);
  const std::string marker = "#include_generated_rhs";
  size_t at = tmpl.find(marker);
  if (at == std::string::npos) throw Error(FF_ERR_COMPILE, "internal: device template marker missing");
  std::string bcast =
      "template <class V> __device__ __forceinline__ V ff_bcast(float s);\n"
      "template <> __device__ __forceinline__ float ff_bcast<float>(float s) { return s; }\n"
      "template <> __device__ __forceinline__ ff2 ff_bcast<ff2>(float s) { return ff2b(s); }\n"
      "template <> __device__ __forceinline__ ff4 ff_bcast<ff4>(float s) { return ff4b(s); }\n";
  tmpl.replace(at, marker.size(), bcast + rhs.str());
  return pre.str() + tmpl;
}

}  // namespace ff
