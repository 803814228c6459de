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
  Exp2, Log, Sin, Cos, Tan, Tanh, Sqrt, Abs, Min, Max, Pow, Sigmoid2, Vtrap
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

  explicit Dag(int sp) : sweep_param(sp) {}

  int intern(DNode n) {
    std::ostringstream key;
    key << (int)n.k << ':';
    if (n.k == K::Num) {
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
    if (nodes[y].k == K::Neg) return sub(x, nodes[y].a[0]);
    if (nodes[x].k == K::Neg) return sub(y, nodes[x].a[0]);
    return op(K::Add, {x, y});
  }
  int sub(int x, int y) {
    if (is_num(x) && is_num(y)) return N(num(x) - num(y));
    if (is_num(y) && num(y) == 0.0) return x;
    if (is_num(x) && num(x) == 0.0) return neg(y);
    if (nodes[y].k == K::Neg) return add(x, nodes[y].a[0]);
    // x - u*w with u uniform -> x + (-u)*w: the negation moves onto the loop-invariant factor, so
    // the packed path gets one FFMA2 (FFMA2 has no operand negation).
    if (nodes[y].k == K::Mul && !nodes[y].uniform) {
      const int u = nodes[y].a[0], w = nodes[y].a[1];
      if (nodes[u].uniform) return add(x, mul(neg(u), w));
      if (nodes[w].uniform) return add(x, mul(neg(w), u));
    }
    return op(K::Sub, {x, y});
  }
  int mul(int x, int y) {
    if (is_num(x) && is_num(y)) return N(num(x) * num(y));
    if (is_num(y)) std::swap(x, y);  // constant first
    if (is_num(x)) {
      const double c = num(x);
      if (c == 1.0) return y;
      if (c == -1.0) return neg(y);
      const DNode& ny = nodes[y];
      // c * (d * w) -> (c d) * w
      if (ny.k == K::Mul && is_num(ny.a[0])) return mul(N(c * num(ny.a[0])), ny.a[1]);
      // c * (-w) -> (-c) * w
      if (ny.k == K::Neg) return mul(N(-c), ny.a[0]);
      // c * (d +- w) -> c d +- c w (one FFMA instead of FADD + FMUL)
      if ((ny.k == K::Add || ny.k == K::Sub) && is_num(ny.a[0])) {
        int d = ny.a[0], w = ny.a[1];
        return ny.k == K::Add ? add(N(c * num(d)), mul(N(c), w)) : sub(N(c * num(d)), mul(N(c), w));
      }
      if ((ny.k == K::Add || ny.k == K::Sub) && is_num(ny.a[1])) {
        int w = ny.a[0], d = ny.a[1];
        return ny.k == K::Add ? add(mul(N(c), w), N(c * num(d))) : sub(mul(N(c), w), N(c * num(d)));
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
  int exp_(int u) {  // e^u = 2^(log2(e) u)
    if (is_num(u)) return N(std::exp(num(u)));
    return op(K::Exp2, {mul(N(1.4426950408889634), u)});
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
        if (f == "vtrap") return op(K::Vtrap, {x, y, rcp(y)});
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

}  // namespace

std::string emit_source(const System& s, int sweep_param) {
  if (sweep_param < -1 || sweep_param >= (int)s.param_names.size())
    throw Error(FF_ERR_INVALID_ARG, "sweep parameter index out of range");
  Dag g(sweep_param);
  std::vector<int> roots;
  for (int i = 0; i < s.dim; ++i) roots.push_back(g.lower(s.rhs[i]));

  // reachable nodes in topological (creation) order
  std::vector<char> live(g.nodes.size(), 0);
  std::function<void(int)> mark = [&](int x) {
    if (live[x]) return;
    live[x] = 1;
    for (int y : g.nodes[x].a) mark(y);
  };
  for (int r : roots) mark(r);

  std::vector<std::string> ref(g.nodes.size());
  std::ostringstream body;
  int n_mufu = 0, n_arith = 0;
  for (size_t id = 0; id < g.nodes.size(); ++id) {
    if (!live[id]) continue;
    const DNode& n = g.nodes[id];
    auto A = [&](int j) { return ref[n.a[j]]; };
    std::string e;
    switch (n.k) {
      case K::Num: ref[id] = flit(n.value); continue;
      case K::Var: ref[id] = "x[" + std::to_string(n.index) + "]"; continue;
      case K::Param: ref[id] = "a.p[" + std::to_string(n.index) + "]"; continue;
      case K::Sweep: ref[id] = "sw"; continue;
      case K::Neg: e = "-" + A(0); break;
      case K::Add: e = A(0) + " + " + A(1); ++n_arith; break;
      case K::Sub: e = A(0) + " - " + A(1); ++n_arith; break;
      case K::Mul: e = A(0) + " * " + A(1); ++n_arith; break;
      case K::Rcp: e = "ff_rcp(" + A(0) + ")"; ++n_mufu; break;
      case K::Div: e = "ff_div(" + A(0) + ", " + A(1) + ")"; ++n_mufu; ++n_arith; break;
      case K::Exp2: e = "ff_exp2(" + A(0) + ")"; ++n_mufu; break;
      case K::Log: e = "ff_log(" + A(0) + ")"; ++n_mufu; break;
      case K::Sin: e = "ff_sin(" + A(0) + ")"; ++n_mufu; break;
      case K::Cos: e = "ff_cos(" + A(0) + ")"; ++n_mufu; break;
      case K::Tan: e = "ff_tan(" + A(0) + ")"; n_mufu += 3; break;
      case K::Tanh: e = "ff_tanh(" + A(0) + ")"; ++n_mufu; break;
      case K::Sqrt: e = "ff_sqrt(" + A(0) + ")"; ++n_mufu; break;
      case K::Abs: e = "ff_abs(" + A(0) + ")"; break;
      case K::Min: e = "ff_min(" + A(0) + ", " + A(1) + ")"; break;
      case K::Max: e = "ff_max(" + A(0) + ", " + A(1) + ")"; break;
      case K::Pow: e = "ff_pow(" + A(0) + ", " + A(1) + ")"; n_mufu += 2; break;
      case K::Sigmoid2: e = "ff_rcp(1.0f + ff_exp2(" + A(0) + "))"; n_mufu += 2; ++n_arith; break;
      case K::Vtrap: e = "ff_vtrap(" + A(0) + ", " + A(1) + ", " + A(2) + ")"; n_mufu += 2; n_arith += 9; break;
    }
    // uniform nodes depend on parameters/constants only: `float`, loop-invariant (hoisted)
    const char* ty = n.uniform ? "float" : "V";
    std::string name = (n.uniform ? "u" : "t") + std::to_string(id);
    body << "  const " << ty << " " << name << " = " << e << ";\n";
    ref[id] = name;
  }
  std::ostringstream rhs;
  rhs << "// Generated right-hand side (" << s.dim << " state variables, " << s.param_names.size()
      << " parameters, swept parameter index " << sweep_param << ").\n";
  for (int i = 0; i < s.dim; ++i) rhs << "//   d" << s.var_names[i] << "/dt = " << s.rhs_text[i] << "\n";
  for (size_t k = 0; k < s.param_names.size(); ++k)
    rhs << "//   a.p[" << k << "] = " << s.param_names[k]
        << ((int)k == sweep_param ? "  (swept: the per-particle value sw is used instead)" : "") << "\n";
  rhs << "// per evaluation (front-end count): " << n_arith << " arithmetic ops, " << n_mufu << " MUFU ops\n";
  rhs << "template <class V>\n__device__ __forceinline__ void ff_rhs(const V* __restrict__ x, V* __restrict__ dx, "
         "const FFStepArgs& a, const V& sw) {\n";
  rhs << "  (void)a; (void)sw;\n";
  rhs << body.str();
  for (int i = 0; i < s.dim; ++i) {
    const DNode& r = g.nodes[roots[i]];
    rhs << "  dx[" << i << "] = " << (r.uniform ? "ff_bcast<V>(" + ref[roots[i]] + ")" : ref[roots[i]]) << ";\n";
  }
  rhs << "}\n";

  const int dim = s.dim;
  const int unroll = dim <= 4 ? 4 : (dim <= 8 ? 2 : 1);
  const int minb_p1 = dim <= 4 ? 4 : (dim <= 8 ? 3 : (dim <= 16 ? 2 : 1));
  const int minb_p2 = dim <= 4 ? 4 : (dim <= 8 ? 2 : 1);
  std::ostringstream pre;
  pre << "// Fireflies kernels, generated by the libfireflies front end for sm_100a.\n";
  pre << "#define FF_DIM " << dim << "\n";
  pre << "#define FF_NP " << s.param_names.size() << "\n";
  pre << "#define FF_NP_ALLOC " << (s.param_names.empty() ? 1 : s.param_names.size()) << "\n";
  pre << "#define FF_UNROLL " << unroll << "\n";
  pre << "#define FF_MINB_P1 " << minb_p1 << "\n";
  pre << "#define FF_MINB_P2 " << minb_p2 << "\n";
  pre << "#define FF_SWEEP " << sweep_param << "\n";

  std::string tmpl(kDeviceTemplate);
  const std::string marker = "#include_generated_rhs";
  size_t at = tmpl.find(marker);
  if (at == std::string::npos) throw Error(FF_ERR_COMPILE, "internal: device template marker missing");
  std::string bcast =
      "template <class V> __device__ __forceinline__ V ff_bcast(float s);\n"
      "template <> __device__ __forceinline__ float ff_bcast<float>(float s) { return s; }\n"
      "template <> __device__ __forceinline__ ff2 ff_bcast<ff2>(float s) { return ff2b(s); }\n";
  tmpl.replace(at, marker.size(), bcast + rhs.str());
  return pre.str() + tmpl;
}

}  // namespace ff
