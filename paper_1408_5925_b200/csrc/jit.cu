// jit.cu -- run-time generated site-expression kernels: qdp_jit_eval / qdp_jit_source.
//
// The paper's thesis (section I, sections III-IV): a QDP++
// expression over lattice fields -- products of colour and spin matrices, spinors, adjoints and
// shifts -- becomes ONE data-parallel kernel, one thread per site (the i_V = thread index mapping
// of PAPER.md:186), generated at run time from the expression's tree (Fig. 3)
// and cached for reuse, with the block size chosen by the autotuner of PAPER.md:232-238.  The
// paper walks the PETE AST and emits PTX; here a small recursive-descent parser builds the AST
// from a string, a code generator walks it (depth first, Fig. 3's order) and emits CUDA C++ for
// the library's own SoA layout, and NVRTC compiles it to an sm_100a cubin (the "compute
// compile driver" step of Fig. 2, done ahead of the launch instead of by the driver).
//
// Expression language (the operands are qdp_field handles, referenced by position):
//   $k          operand k (fermion -> spinor, colour matrix, spin matrix)
//   $k[mu]      link U_mu of a gauge operand (colour matrix; reconstruct-12 links rebuilt)
//   number      real constant
//   a + b, a - b, -a, a * b, (a)
//   adj(a)      hermitian conjugate of a colour or spin matrix
//   timesI(a)   i * a
//   gamma(mu)   gamma_mu (DeGrand-Rossi, reading R1; mu = 0..3) as a left factor of a spinor or
//   gamma5      spin matrix; gamma5 = gamma_x gamma_y gamma_z gamma_t = diag(1, 1, -1, -1)
//   shift(a, mu, s)  a(x + s mu^), s = +1 (FORWARD) or -1 (BACKWARD): PAPER.md:111-126 (R4).
//               Evaluated in place: the subexpression is computed at the neighbouring site, so a
//               shift costs no temporary and "shifts of shifts" are just diagonal
//               neighbours, periodic on the local lattice.  Along dimensions reached through
//               the halo path (multi-rank or self-halo) the displaced operand is first
//               materialised with qdp_shift, which exchanges the faces, and the
//               kernel reads that temporary (section V's face communication, not overlapped here).
// Products: colour x colour, colour x spinor, spin x spin, spin x spinor, real x anything,
// gamma x spinor / spin matrix.  Common subexpressions (same text at the same site) are
// computed once, so e.g. the hopping term can be written as
//   sum_mu  f_mu - gamma(mu)*f_mu + b_mu + gamma(mu)*b_mu,
//   f_mu = $0[mu]*shift($1,mu,+1),  b_mu = shift(adj($0[mu])*$1, mu, -1)
// and each U*psi product is formed once.
//
// Accounting (Table II convention): complex mul 6, complex add 2, real x
// complex 2 flops for every operation the kernel executes (after common-subexpression
// elimination); bytes two ways: compulsory (each distinct operand field read once + the store,
// the library's roofline numerator) and Table II's (every leaf occurrence + the store).
#include <dlfcn.h>

#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <set>
#include <sstream>

#include "internal.h"

struct qdpb::JitKernel {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  int max_threads = 1024;
  double flops = 0, bytes_all = 0, bytes_parity = 0;  // per output site (out QDP_ALL / one parity)
  long key = 0;                 // autotuner key
  // halo'd temporaries: operand temp_leaf[j] shifted by temp_dp[j] (qdp_shift chain through
  // temp_steps[j]; the last step writes temp_field[j]), allocated on first use, kept for reuse
  std::vector<int> temp_leaf;
  std::vector<std::array<int, 4>> temp_dp;
  std::vector<qdp_field> temp_field;
  std::vector<std::vector<qdp_field>> temp_steps;
  std::vector<std::pair<int, int>> leaf_disp_parity;  // (operand, parity flip) of every leaf load
};

namespace qdpb {
namespace {

enum Type { T_REAL, T_CM, T_SP, T_SM, T_GAMMA, T_CPLX };
enum NodeOp { N_NUM, N_LEAF, N_ADD, N_SUB, N_NEG, N_MUL, N_ADJ, N_SHIFT, N_GAMMA, N_TIMESI, N_TRACE, N_LNORM2, N_LINNER,
              N_REAL };

struct Node {
  NodeOp op;
  std::vector<std::unique_ptr<Node>> kid;
  double num = 0.0;
  int leaf = -1, mu = -1, sign = 0;  // leaf operand; link / shift / gamma index (gamma5 = 4)
  Type type = T_REAL;
};
using NodeP = std::unique_ptr<Node>;

const char *type_name(Type t) {
  static const char *n[] = {"real", "colour matrix", "spinor", "spin matrix", "gamma", "complex scalar"};
  return n[t];
}

// ------------------------------------------------------------------ parser
struct Parser {
  const char *s;
  size_t i = 0;
  std::string err;
  explicit Parser(const char *src) : s(src) {}

  void ws() {
    while (s[i] == ' ' || s[i] == '\t' || s[i] == '\n' || s[i] == '\r') i++;
  }
  bool eat(char c) {
    ws();
    if (s[i] == c) {
      i++;
      return true;
    }
    return false;
  }
  NodeP fail(const std::string &m) {
    if (err.empty()) err = m + " at offset " + std::to_string(i);
    return nullptr;
  }
  bool integer(int *v) {
    ws();
    size_t j = i;
    bool neg = false;
    if (s[j] == '+' || s[j] == '-') neg = s[j++] == '-';
    if (s[j] < '0' || s[j] > '9') return false;
    long x = 0;
    while (s[j] >= '0' && s[j] <= '9' && x < 1000000) x = 10 * x + (s[j++] - '0');
    i = j;
    *v = (int)(neg ? -x : x);
    return true;
  }
  std::string ident() {
    ws();
    size_t j = i;
    while ((s[j] >= 'a' && s[j] <= 'z') || (s[j] >= 'A' && s[j] <= 'Z') || (s[j] >= '0' && s[j] <= '9' && j > i)) j++;
    std::string r(s + i, s + j);
    i = j;
    return r;
  }
  static NodeP make(NodeOp op) {
    NodeP n(new Node);
    n->op = op;
    return n;
  }
  NodeP expr() {
    NodeP a = term();
    while (a) {
      ws();
      if (s[i] == '+' || s[i] == '-') {
        NodeP n = make(s[i] == '+' ? N_ADD : N_SUB);
        i++;
        NodeP b = term();
        if (!b) return nullptr;
        n->kid.push_back(std::move(a));
        n->kid.push_back(std::move(b));
        a = std::move(n);
      } else {
        break;
      }
    }
    return a;
  }
  NodeP term() {
    if (eat('-')) {  // a leading minus negates the whole product: -gamma(mu)*a = -(gamma(mu)*a)
      NodeP t = term();
      if (!t) return nullptr;
      NodeP n = make(N_NEG);
      n->kid.push_back(std::move(t));
      return n;
    }
    NodeP a = unary();
    while (a && eat('*')) {
      NodeP b = unary();
      if (!b) return nullptr;
      NodeP n = make(N_MUL);
      n->kid.push_back(std::move(a));
      n->kid.push_back(std::move(b));
      a = std::move(n);
    }
    return a;
  }
  NodeP unary() {
    if (eat('-')) {
      NodeP a = unary();
      if (!a) return nullptr;
      NodeP n = make(N_NEG);
      n->kid.push_back(std::move(a));
      return n;
    }
    return primary();
  }
  NodeP primary() {
    ws();
    const char c = s[i];
    if (c == '(') {
      i++;
      NodeP a = expr();
      if (a && !eat(')')) return fail("expected ')'");
      return a;
    }
    if (c == '$') {
      i++;
      int k;
      if (!integer(&k) || k < 0 || k >= QDP_JIT_MAX_OPERANDS) return fail("bad operand index");
      NodeP n = make(N_LEAF);
      n->leaf = k;
      if (eat('[')) {
        if (!integer(&n->mu) || n->mu < 0 || n->mu > 3) return fail("link index must be 0..3");
        if (!eat(']')) return fail("expected ']'");
      }
      return n;
    }
    if ((c >= '0' && c <= '9') || c == '.') {
      char *end = nullptr;
      const double v = strtod(s + i, &end);
      if (end == s + i) return fail("bad number");
      i = end - s;
      NodeP n = make(N_NUM);
      n->num = v;
      return n;
    }
    const std::string id = ident();
    if (id == "gamma5") {
      NodeP n = make(N_GAMMA);
      n->mu = 4;
      return n;
    }
    if (id.empty()) return fail("unexpected character");
    if (!eat('(')) return fail("expected '(' after " + id);
    NodeP n;
    if (id == "gamma") {
      n = make(N_GAMMA);
      if (!integer(&n->mu) || n->mu < 0 || n->mu > 3) return fail("gamma index must be 0..3");
    } else if (id == "adj" || id == "timesI" || id == "trace" || id == "localNorm2" || id == "real") {
      n = make(id == "adj" ? N_ADJ : id == "timesI" ? N_TIMESI : id == "trace" ? N_TRACE : id == "real" ? N_REAL : N_LNORM2);
      NodeP a = expr();
      if (!a) return nullptr;
      n->kid.push_back(std::move(a));
    } else if (id == "localInnerProduct") {
      n = make(N_LINNER);
      NodeP a = expr();
      if (!a) return nullptr;
      n->kid.push_back(std::move(a));
      if (!eat(',')) return fail("localInnerProduct needs two arguments");
      NodeP b = expr();
      if (!b) return nullptr;
      n->kid.push_back(std::move(b));
    } else if (id == "shift") {
      n = make(N_SHIFT);
      NodeP a = expr();
      if (!a) return nullptr;
      n->kid.push_back(std::move(a));
      if (!eat(',') || !integer(&n->mu) || n->mu < 0 || n->mu > 3) return fail("shift: direction must be 0..3");
      if (!eat(',') || !integer(&n->sign) || (n->sign != 1 && n->sign != -1)) return fail("shift: sign must be +1 or -1");
    } else {
      return fail("unknown function '" + id + "'");
    }
    if (!eat(')')) return fail("expected ')'");
    return n;
  }
};

// ------------------------------------------------------------------ type check
Type kind_type(int kind) {
  switch (kind) {
    case QDP_FERMION: return T_SP;
    case QDP_COLORMATRIX: return T_CM;
    case QDP_SPINMATRIX: return T_SM;
    case QDP_GAUGE:
    case QDP_GAUGE12: return T_CM;
    default: return T_GAMMA;  // not usable
  }
}

bool typecheck(Node *n, const int *kinds, int nops, std::string &err) {
  for (auto &k : n->kid)
    if (!typecheck(k.get(), kinds, nops, err)) return false;
  auto bad = [&](const std::string &m) {
    err = m;
    return false;
  };
  Type a = n->kid.size() > 0 ? n->kid[0]->type : T_REAL, b = n->kid.size() > 1 ? n->kid[1]->type : T_REAL;
  switch (n->op) {
    case N_NUM: n->type = T_REAL; return true;
    case N_GAMMA: n->type = T_GAMMA; return true;
    case N_LEAF: {
      if (n->leaf >= nops) return bad("operand $" + std::to_string(n->leaf) + " not supplied");
      const int kind = kinds[n->leaf];
      const bool g = kind == QDP_GAUGE || kind == QDP_GAUGE12;
      if (g != (n->mu >= 0)) return bad(g ? "gauge operand needs a link index [mu]" : "[mu] on a non-gauge operand");
      n->type = kind_type(kind);
      if (n->type == T_GAMMA) return bad("operand kind not usable in expressions (clover: use qdp_clover_apply)");
      return true;
    }
    case N_ADD:
    case N_SUB:
      if (a != b || a == T_GAMMA) return bad(std::string("cannot add ") + type_name(a) + " and " + type_name(b));
      n->type = a;
      return true;
    case N_NEG:
      if (a == T_GAMMA) return bad("cannot negate gamma (write -1*...)");
      n->type = a;
      return true;
    case N_TIMESI:
      if (a == T_GAMMA || a == T_REAL) return bad("timesI needs a field or complex scalar");
      n->type = a;
      return true;
    case N_ADJ:
      if (a != T_CM && a != T_SM) return bad("adj needs a colour or spin matrix");
      n->type = a;
      return true;
    case N_SHIFT:
      if (a == T_GAMMA || a == T_REAL) return bad("shift needs a field");
      n->type = a;
      return true;
    case N_TRACE:
      if (a != T_CM && a != T_SM) return bad("trace needs a colour or spin matrix");
      n->type = T_CPLX;
      return true;
    case N_LNORM2:
      if (a != T_CM && a != T_SP && a != T_SM && a != T_CPLX) return bad("localNorm2 needs a field");
      n->type = T_CPLX;
      return true;
    case N_LINNER:
      if (a != b || (a != T_CM && a != T_SP && a != T_SM && a != T_CPLX))
        return bad("localInnerProduct needs two fields of one type");
      n->type = T_CPLX;
      return true;
    case N_REAL:
      if (a != T_CPLX) return bad("real needs a complex scalar");
      n->type = T_CPLX;
      return true;
    case N_MUL:
      if (a == T_REAL && b != T_GAMMA) n->type = b;
      else if (b == T_REAL && a != T_GAMMA) n->type = a;
      else if (a == T_CM && b == T_CM) n->type = T_CM;
      else if (a == T_CM && b == T_SP) n->type = T_SP;
      else if (a == T_SM && b == T_SM) n->type = T_SM;
      else if (a == T_SM && b == T_SP) n->type = T_SP;
      else if (a == T_GAMMA && (b == T_SP || b == T_SM)) n->type = b;
      else if (a == T_CPLX && b == T_CPLX) n->type = T_CPLX;
      else return bad(std::string("cannot multiply ") + type_name(a) + " by " + type_name(b));
      return true;
  }
  return bad("internal: unknown node");
}

// ------------------------------------------------------------------ code generation
int type_reals(Type t, int kind = -1) {
  if (kind == QDP_GAUGE12) return 12;
  return t == T_CM ? 18 : t == T_SP ? 24 : t == T_SM ? 32 : t == T_CPLX ? 2 : 0;
}
const char *ctype(Type t) { return t == T_CM ? "CM" : t == T_SP ? "SP" : t == T_SM ? "SM" : t == T_CPLX ? "cx" : "R"; }
int type_complex(Type t) { return t == T_CM ? 9 : t == T_SP ? 12 : t == T_SM ? 16 : t == T_CPLX ? 1 : 0; }

// A leaf read at a displacement with components along dimensions reached through the halo path:
// the host materialises operand `leaf` shifted by `dp` (those components) with qdp_shift, which
// exchanges the faces (shifts of shifts for diagonal displacements),
// and the kernel reads that temporary at the remaining (in-kernel, periodic) displacement.
struct Temp {
  int leaf;
  int dp[4];
};

struct Gen {
  const int *kinds;
  int prec;
  int part = 0;              // dims reached through the halo path
  std::vector<Temp> temps;   // operand slots QDP_JIT_MAX_OPERANDS + j
  std::ostringstream body;
  int nv = 0;
  std::map<std::string, std::string> cse;    // canonical key -> variable
  std::map<std::string, std::string> sites;  // displacement -> "cbN" (parity in "pN")
  std::set<std::pair<int, int>> distinct;    // (operand, mu) fields read
  std::set<std::vector<int>> distinct_par;   // (operand, mu, parity flip) blocks read
  std::set<int> shift_dims;
  double flops = 0.0, table2_reals = 0.0;

  static std::string dkey(const int d[4]) {
    return std::to_string(d[0]) + "," + std::to_string(d[1]) + "," + std::to_string(d[2]) + "," + std::to_string(d[3]);
  }
  std::string site(const int d[4]) {
    const std::string k = dkey(d);
    auto it = sites.find(k);
    if (it != sites.end()) return it->second;
    const std::string v = std::to_string(sites.size());
    if (d[0] == 0 && d[1] == 0 && d[2] == 0 && d[3] == 0) {
      body << "  const int cb" << v << " = cb, p" << v << " = p;\n";
    } else {
      const int parity_flip = (std::abs(d[0]) + std::abs(d[1]) + std::abs(d[2]) + std::abs(d[3])) & 1;
      body << "  int cb" << v << ";\n  {\n    int n[4] = {c[0], c[1], c[2], c[3]};\n";
      for (int m = 0; m < 4; m++)
        if (d[m] == 1 || d[m] == -1)  // every extent is even and >= 2 (reading R6): one compare
          body << "    n[" << m << "] = " << (d[m] > 0 ? "wrap_up" : "wrap_down") << "(n[" << m << "], a.L[" << m << "]);\n";
        else if (d[m])
          body << "    n[" << m << "] = wrap(n[" << m << "] + (" << d[m] << "), a.L[" << m << "]);\n";
      body << "    cb" << v << " = (n[0] >> 1) + a.Lh0 * (n[1] + a.L[1] * (n[2] + a.L[2] * n[3]));\n  }\n";
      body << "  const int p" << v << " = p ^ " << parity_flip << ";\n";
    }
    sites[k] = v;
    return v;
  }
  std::string fresh() { return "v" + std::to_string(nv++); }

  // canonical text of n evaluated at displacement d (shift folds into d)
  static std::string key(const Node *n, const int d[4]) {
    switch (n->op) {
      case N_NUM: {
        char b[64];
        snprintf(b, sizeof b, "%.17g", n->num);
        return b;
      }
      case N_GAMMA: return "g" + std::to_string(n->mu);
      case N_LEAF: return "$" + std::to_string(n->leaf) + "[" + std::to_string(n->mu) + "]@" + dkey(d);
      case N_SHIFT: {
        int e[4] = {d[0], d[1], d[2], d[3]};
        e[n->mu] += n->sign;
        return key(n->kid[0].get(), e);
      }
      default: {
        std::string r = std::to_string((int)n->op) + "(";
        for (auto &k : n->kid) r += key(k.get(), d) + ";";
        return r + ")";
      }
    }
  }

  void count_leaves(const Node *n) {
    if (n->op == N_LEAF) table2_reals += type_reals(n->type, kinds[n->leaf]);
    for (auto &k : n->kid) count_leaves(k.get());
  }

  // cache policy: a field block (operand, mu, parity flip) read at two or more displacements is
  // reused by neighbouring threads; every other leaf is streamed
  std::map<std::vector<int>, std::set<std::string>> disp;
  std::set<std::vector<int>> reuse;
  static int flip(const int d[4]) { return (std::abs(d[0]) + std::abs(d[1]) + std::abs(d[2]) + std::abs(d[3])) & 1; }
  void collect(const Node *n, const int d[4]) {
    if (n->op == N_SHIFT) {
      int e[4] = {d[0], d[1], d[2], d[3]};
      e[n->mu] += n->sign;
      collect(n->kid[0].get(), e);
      return;
    }
    if (n->op == N_LEAF) {
      auto &ds = disp[{n->leaf, n->mu, flip(d)}];
      ds.insert(dkey(d));
      if (ds.size() > 1) reuse.insert({n->leaf, n->mu, flip(d)});
    }
    for (auto &k : n->kid) collect(k.get(), d);
  }

  // A spinor sum is flattened into signed terms; a term A and a term gamma(mu)*A (same text at the
  // same site, any grouping or order) combine into s (1 + S gamma_mu) A: spin projection.
  // When A is, after its shifts, a colour matrix times a spinor, the projector commutes with the
  // colour product, so it is applied first and U multiplies a half spinor: 12 + 132 flop instead of
  // 264 + 24.  The remaining terms are added in their written order.
  static void flatten(const Node *n, int sign, std::vector<std::pair<const Node *, int>> &terms) {
    if ((n->op == N_ADD || n->op == N_SUB) && n->type == T_SP) {
      flatten(n->kid[0].get(), sign, terms);
      flatten(n->kid[1].get(), n->op == N_ADD ? sign : -sign, terms);
    } else if (n->op == N_NEG && n->type == T_SP) {
      flatten(n->kid[0].get(), -sign, terms);
    } else {
      terms.push_back({n, sign});
    }
  }
  static bool gamma_term(const Node *n) {
    return n->op == N_MUL && n->kid[0]->op == N_GAMMA && n->kid[0]->mu <= 3;
  }
  std::string emit_projector(const Node *A, int mu, int S, const int d[4]) {
    const Node *x = A;
    int e[4] = {d[0], d[1], d[2], d[3]};
    while (x->op == N_SHIFT) {
      e[x->mu] += x->sign;
      shift_dims.insert(x->mu);
      x = x->kid[0].get();
    }
    const std::string tmpl = "<" + std::to_string(mu) + ", " + std::to_string(S) + ">";
    const std::string v = fresh();
    if (x->op == N_MUL && x->kid[0]->type == T_CM && x->kid[1]->type == T_SP) {
      const std::string u = emit(x->kid[0].get(), e), sp = emit(x->kid[1].get(), e);
      body << "  const SP " << v << " = recon" << tmpl << "(mul(" << u << ", proj" << tmpl << "(" << sp << ")));\n";
      flops += 12 + 2 * (9 * 6 + 6 * 2);
    } else {
      const std::string a = emit(A, d);
      body << "  const SP " << v << " = recon" << tmpl << "(proj" << tmpl << "(" << a << "));\n";
      flops += 12;
    }
    return v;
  }
  std::string emit_spinor_sum(const Node *n, const int d[4]) {
    std::vector<std::pair<const Node *, int>> terms;
    flatten(n, 1, terms);
    std::vector<int> used(terms.size(), 0);
    // accumulate as the terms are produced (written order), so only the running sum and the term
    // at hand are live
    std::string acc;
    auto accumulate = [&](const std::string &val, int sign) {
      if (acc.empty()) {
        if (sign > 0) {
          acc = val;
        } else {
          acc = fresh();
          body << "  const SP " << acc << " = neg(" << val << ");\n";
        }
        return;
      }
      const std::string v = fresh();
      body << "  const SP " << v << " = " << (sign > 0 ? "add(" : "sub(") << acc << ", " << val << ");\n";
      flops += 24;
      acc = v;
    };
    for (size_t i = 0; i < terms.size(); i++) {
      if (used[i]) continue;
      const Node *t = terms[i].first;
      // pair this term with a partner: t = A and a later gamma(mu)*A, or t = gamma(mu)*A and a later A
      size_t j = terms.size();
      int mu = -1;
      const Node *A = nullptr;
      for (size_t k = i + 1; k < terms.size() && j == terms.size(); k++) {
        if (used[k]) continue;
        const Node *u = terms[k].first;
        if (gamma_term(u) && !gamma_term(t) && key(u->kid[1].get(), d) == key(t, d)) {
          j = k; mu = u->kid[0]->mu; A = t;
        } else if (gamma_term(t) && !gamma_term(u) && key(t->kid[1].get(), d) == key(u, d)) {
          j = k; mu = t->kid[0]->mu; A = u;
        }
      }
      if (j < terms.size()) {
        used[j] = 1;
        const int sA = A == t ? terms[i].second : terms[j].second;  // sign of A
        const int sG = A == t ? terms[j].second : terms[i].second;  // sign of gamma(mu)*A
        accumulate(emit_projector(A, mu, sA * sG, d), sA);
      } else {
        accumulate(emit(t, d), terms[i].second);
      }
    }
    return acc;
  }

  // emit n at displacement d; returns the C++ expression naming its value
  std::string emit(const Node *n, const int d[4]) {
    if (n->op == N_NUM) {
      char b[64];
      snprintf(b, sizeof b, "R(%.17g)", n->num);
      return b;
    }
    if (n->op == N_SHIFT) {
      int e[4] = {d[0], d[1], d[2], d[3]};
      e[n->mu] += n->sign;
      shift_dims.insert(n->mu);
      return emit(n->kid[0].get(), e);
    }
    const std::string k = key(n, d);
    auto it = cse.find(k);
    if (it != cse.end()) return it->second;
    std::string v;
    if (n->op == N_LEAF) {
      int slot = n->leaf, r[4] = {d[0], d[1], d[2], d[3]};
      Temp t = {n->leaf, {0, 0, 0, 0}};
      for (int m = 0; m < 4; m++)
        if (((part >> m) & 1) && d[m]) {
          t.dp[m] = d[m];
          r[m] = 0;
        }
      if (t.dp[0] || t.dp[1] || t.dp[2] || t.dp[3]) {
        size_t j = 0;
        while (j < temps.size() && !(temps[j].leaf == t.leaf && !memcmp(temps[j].dp, t.dp, sizeof t.dp))) j++;
        if (j == temps.size()) temps.push_back(t);
        slot = QDP_JIT_MAX_OPERANDS + (int)j;
      }
      const std::string s = site(r);
      const int kind = kinds[n->leaf];
      distinct.insert({n->leaf, n->mu});
      distinct_par.insert({n->leaf, n->mu, (std::abs(d[0]) + std::abs(d[1]) + std::abs(d[2]) + std::abs(d[3])) & 1});
      v = fresh();
      const std::string base = "base(a, " + std::to_string(slot) + ", p" + s + ", " + std::to_string(n->mu) + ")";
      const char *ld = kind == QDP_FERMION ? "ld_sp" : kind == QDP_SPINMATRIX ? "ld_sm" : kind == QDP_GAUGE12 ? "ld_g12" : "ld_cm";
      const bool stream = reuse.count({n->leaf, n->mu, flip(d)}) == 0;
      body << "  const " << ctype(n->type) << " " << v << " = " << ld << (stream ? "<true>(" : "<false>(") << base
           << ", a.stride, cb" << s << ");\n";
    } else if ((n->op == N_ADD || n->op == N_SUB) && n->type == T_SP) {
      v = emit_spinor_sum(n, d);
    } else if (n->op == N_MUL && n->kid[0]->op == N_GAMMA) {
      const std::string x = emit(n->kid[1].get(), d);
      v = fresh();
      body << "  const " << ctype(n->type) << " " << v << " = gam<" << n->kid[0]->mu << ">(" << x << ");\n";
    } else {
      std::vector<std::string> xs;
      for (auto &kd : n->kid) xs.push_back(emit(kd.get(), d));
      v = fresh();
      const Type t = n->type;
      const double nc = t == T_REAL ? 0.5 : type_complex(t);  // complex numbers (real: 1 flop)
      std::string e;
      switch (n->op) {
        case N_ADD: e = "add(" + xs[0] + ", " + xs[1] + ")"; flops += 2 * nc; break;
        case N_SUB: e = "sub(" + xs[0] + ", " + xs[1] + ")"; flops += 2 * nc; break;
        case N_NEG: e = "neg(" + xs[0] + ")"; break;
        case N_ADJ: e = "adj(" + xs[0] + ")"; break;
        case N_TIMESI: e = "timesI(" + xs[0] + ")"; break;
        case N_TRACE: {
          const int nd = n->kid[0]->type == T_CM ? 3 : 4;
          e = "trace(" + xs[0] + ")";
          flops += 2 * (nd - 1);
          break;
        }
        case N_LNORM2: e = "lnorm2(" + xs[0] + ")"; flops += 4 * type_complex(n->kid[0]->type); break;
        case N_LINNER: e = "linner(" + xs[0] + ", " + xs[1] + ")"; flops += 8 * type_complex(n->kid[0]->type); break;
        case N_REAL: e = "cx{" + xs[0] + ".re, R(0)}"; break;
        case N_MUL: {
          const Type a = n->kid[0]->type, b = n->kid[1]->type;
          if (a == T_REAL && b == T_REAL) {
            e = "(" + xs[0] + " * " + xs[1] + ")";
            flops += 1;
          } else if (a == T_CPLX && b == T_CPLX) {
            e = "cmul(" + xs[0] + ", " + xs[1] + ")";
            flops += 6;
          } else if (a == T_REAL || b == T_REAL) {
            e = a == T_REAL ? "scale(" + xs[0] + ", " + xs[1] + ")" : "scale(" + xs[1] + ", " + xs[0] + ")";
            flops += 2 * nc;
          } else {
            e = "mul(" + xs[0] + ", " + xs[1] + ")";
            if (a == T_CM && b == T_CM) flops += 27 * 6 + 18 * 2;        // 198 (Table II lcm)
            else if (a == T_CM && b == T_SP) flops += 4 * (9 * 6 + 6 * 2);  // 264 (upsi)
            else if (a == T_SM && b == T_SM) flops += 64 * 6 + 48 * 2;   // 480 (spmat)
            else flops += 12 * (4 * 6 + 3 * 2);                          // spin matrix x spinor: 360
          }
          break;
        }
        default: break;
      }
      body << "  const " << ctype(t) << " " << v << " = " << e << ";\n";
    }
    cse[k] = v;
    return v;
  }
};

// device-side prelude: types, algebra and the library's SoA layouts (internal.h), per precision
const char *kPrelude = R"PRELUDE(
struct JitArgs {
  const char *op[24]; // 8 operands, then up to 16 halo'd temporaries
  char *out;
  long long blk[24];  // bytes between parity blocks (gauge: between (mu, parity) blocks)
  long long out_blk;
  int all[24];        // operand covers both parities
  int L[4];
  int Lh0, Vh, stride, parity, nblk;
};
struct cx { R re, im; };
__device__ __forceinline__ cx operator+(cx a, cx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cx operator-(cx a, cx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ cx cmul(cx a, cx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
__device__ __forceinline__ cx cmadd(cx a, cx b, cx c) {
  c.re = fma(a.re, b.re, c.re); c.re = fma(-a.im, b.im, c.re);
  c.im = fma(a.re, b.im, c.im); c.im = fma(a.im, b.re, c.im); return c;
}
__device__ __forceinline__ cx conj(cx a) { return {a.re, -a.im}; }
__device__ __forceinline__ cx ti(cx a) { return {-a.im, a.re}; }
struct CM { cx m[9]; };
struct SP { cx c[12]; };
struct SM { cx m[16]; };
template <int N> struct Arr;
#define QDPJ_ELEMENTWISE(T, N, F)                                                        \
  __device__ __forceinline__ T add(const T &a, const T &b) { T r; for (int k = 0; k < N; k++) r.F[k] = a.F[k] + b.F[k]; return r; } \
  __device__ __forceinline__ T sub(const T &a, const T &b) { T r; for (int k = 0; k < N; k++) r.F[k] = a.F[k] - b.F[k]; return r; } \
  __device__ __forceinline__ T neg(const T &a) { T r; for (int k = 0; k < N; k++) r.F[k] = {-a.F[k].re, -a.F[k].im}; return r; } \
  __device__ __forceinline__ T scale(R s, const T &a) { T r; for (int k = 0; k < N; k++) r.F[k] = {s * a.F[k].re, s * a.F[k].im}; return r; } \
  __device__ __forceinline__ T timesI(const T &a) { T r; for (int k = 0; k < N; k++) r.F[k] = ti(a.F[k]); return r; }
QDPJ_ELEMENTWISE(CM, 9, m)
QDPJ_ELEMENTWISE(SP, 12, c)
QDPJ_ELEMENTWISE(SM, 16, m)
__device__ __forceinline__ R add(R a, R b) { return a + b; }
__device__ __forceinline__ R sub(R a, R b) { return a - b; }
__device__ __forceinline__ R neg(R a) { return -a; }
__device__ __forceinline__ CM mul(const CM &x, const CM &y) {
  CM z;
  for (int r = 0; r < 3; r++)
    for (int c = 0; c < 3; c++) {
      cx acc = cmul(x.m[3 * r], y.m[c]);
      acc = cmadd(x.m[3 * r + 1], y.m[3 + c], acc);
      z.m[3 * r + c] = cmadd(x.m[3 * r + 2], y.m[6 + c], acc);
    }
  return z;
}
__device__ __forceinline__ SP mul(const CM &u, const SP &s) {
  SP o;
  for (int sp = 0; sp < 4; sp++)
    for (int a = 0; a < 3; a++) {
      cx acc = cmul(u.m[3 * a], s.c[3 * sp]);
      acc = cmadd(u.m[3 * a + 1], s.c[3 * sp + 1], acc);
      o.c[3 * sp + a] = cmadd(u.m[3 * a + 2], s.c[3 * sp + 2], acc);
    }
  return o;
}
__device__ __forceinline__ SM mul(const SM &x, const SM &y) {
  SM z;
  for (int r = 0; r < 4; r++)
    for (int c = 0; c < 4; c++) {
      cx acc = cmul(x.m[4 * r], y.m[c]);
      for (int k = 1; k < 4; k++) acc = cmadd(x.m[4 * r + k], y.m[4 * k + c], acc);
      z.m[4 * r + c] = acc;
    }
  return z;
}
__device__ __forceinline__ SP mul(const SM &m, const SP &s) {
  SP o;
  for (int sp = 0; sp < 4; sp++)
    for (int a = 0; a < 3; a++) {
      cx acc = cmul(m.m[4 * sp], s.c[a]);
      for (int t = 1; t < 4; t++) acc = cmadd(m.m[4 * sp + t], s.c[3 * t + a], acc);
      o.c[3 * sp + a] = acc;
    }
  return o;
}
__device__ __forceinline__ CM adj(const CM &u) {
  CM r;
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) r.m[3 * i + j] = conj(u.m[3 * j + i]);
  return r;
}
__device__ __forceinline__ SM adj(const SM &u) {
  SM r;
  for (int i = 0; i < 4; i++)
    for (int j = 0; j < 4; j++) r.m[4 * i + j] = conj(u.m[4 * j + i]);
  return r;
}
// complex scalars per site (trace, local norms and inner products) and their algebra
__device__ __forceinline__ cx add(cx a, cx b) { return a + b; }
__device__ __forceinline__ cx sub(cx a, cx b) { return a - b; }
__device__ __forceinline__ cx neg(cx a) { return {-a.re, -a.im}; }
__device__ __forceinline__ cx scale(R s, cx a) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ cx timesI(cx a) { return ti(a); }
__device__ __forceinline__ cx trace(const CM &u) { return u.m[0] + u.m[4] + u.m[8]; }
__device__ __forceinline__ cx trace(const SM &u) { return u.m[0] + u.m[5] + u.m[10] + u.m[15]; }
#define QDPJ_LOCAL(T, N, F)                                                                   \
  __device__ __forceinline__ cx lnorm2(const T &a) {                                           \
    R s = 0; for (int k = 0; k < N; k++) s += a.F[k].re * a.F[k].re + a.F[k].im * a.F[k].im;  \
    return {s, R(0)};                                                                          \
  }                                                                                            \
  __device__ __forceinline__ cx linner(const T &a, const T &b) {                               \
    cx s = {0, 0}; for (int k = 0; k < N; k++) s = s + cmul(conj(a.F[k]), b.F[k]); return s;   \
  }
QDPJ_LOCAL(CM, 9, m)
QDPJ_LOCAL(SP, 12, c)
QDPJ_LOCAL(SM, 16, m)
__device__ __forceinline__ cx lnorm2(cx a) { return {a.re * a.re + a.im * a.im, R(0)}; }
__device__ __forceinline__ cx linner(cx a, cx b) { return cmul(conj(a), b); }
// block sum of (v0, v1) in fp64 -> partials[2 * blockIdx.x + {0, 1}] (fixed order: deterministic)
__device__ __forceinline__ void block_partial(double v0, double v1, double *partials) {
  __shared__ double s0[32], s1[32];
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, o);
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { s0[w] = v0; s1[w] = v1; }
  __syncthreads();
  if (w == 0) {
    v0 = l < (int)(blockDim.x >> 5) ? s0[l] : 0.0;
    v1 = l < (int)(blockDim.x >> 5) ? s1[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      v0 += __shfl_xor_sync(0xffffffffu, v0, o);
      v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    }
    if (l == 0) { partials[2 * blockIdx.x] = v0; partials[2 * blockIdx.x + 1] = v1; }
  }
}
// DeGrand-Rossi gamma_mu (mu = 0..3) and gamma5 (4): row s has one entry, at column
// gcol[mu][s] with phase gph[mu][s] (0: +1, 1: +i, 2: -1, 3: -i)
__device__ __forceinline__ cx phase(int ph, cx v) {
  return ph == 0 ? v : ph == 1 ? ti(v) : ph == 2 ? cx{-v.re, -v.im} : cx{v.im, -v.re};
}
template <int MU> __device__ __forceinline__ void gtab(int s, int &col, int &ph) {
  // gamma_x: (0,3,+i) (1,2,+i) (2,1,-i) (3,0,-i);  gamma_y: (0,3,-1) (1,2,+1) (2,1,+1) (3,0,-1)
  // gamma_z: (0,2,+i) (1,3,-i) (2,0,-i) (3,1,+i);  gamma_t: (0,2,+1) (1,3,+1) (2,0,+1) (3,1,+1)
  // gamma5 : diag(+1, +1, -1, -1)
  const int cols[5][4] = {{3, 2, 1, 0}, {3, 2, 1, 0}, {2, 3, 0, 1}, {2, 3, 0, 1}, {0, 1, 2, 3}};
  const int phs[5][4] = {{1, 1, 3, 3}, {2, 0, 0, 2}, {1, 3, 3, 1}, {0, 0, 0, 0}, {0, 0, 2, 2}};
  col = cols[MU][s];
  ph = phs[MU][s];
}
template <int MU> __device__ __forceinline__ SP gam(const SP &x) {
  SP r;
#pragma unroll
  for (int s = 0; s < 4; s++) {
    int col, ph;
    gtab<MU>(s, col, ph);
#pragma unroll
    for (int a = 0; a < 3; a++) r.c[3 * s + a] = phase(ph, x.c[3 * col + a]);
  }
  return r;
}
template <int MU> __device__ __forceinline__ SM gam(const SM &x) {
  SM r;
#pragma unroll
  for (int s = 0; s < 4; s++) {
    int col, ph;
    gtab<MU>(s, col, ph);
#pragma unroll
    for (int t = 0; t < 4; t++) r.m[4 * s + t] = phase(ph, x.m[4 * col + t]);
  }
  return r;
}
// half spinor: rows 0, 1 of (1 + S gamma_mu) psi (S = +1 / -1); rows 2, 3 follow from them
// (DeGrand-Rossi, SURVEY Appendix A): index 3 * h + colour
struct HS { cx c[6]; };
template <int MU, int S> __device__ __forceinline__ HS proj(const SP &p) {
  HS h;
#pragma unroll
  for (int c = 0; c < 3; c++) {
    const cx p0 = p.c[c], p1 = p.c[3 + c], p2 = p.c[6 + c], p3 = p.c[9 + c];
    if (MU == 0) { h.c[c] = S > 0 ? p0 + ti(p3) : p0 - ti(p3); h.c[3 + c] = S > 0 ? p1 + ti(p2) : p1 - ti(p2); }
    else if (MU == 1) { h.c[c] = S > 0 ? p0 - p3 : p0 + p3; h.c[3 + c] = S > 0 ? p1 + p2 : p1 - p2; }
    else if (MU == 2) { h.c[c] = S > 0 ? p0 + ti(p2) : p0 - ti(p2); h.c[3 + c] = S > 0 ? p1 - ti(p3) : p1 + ti(p3); }
    else { h.c[c] = S > 0 ? p0 + p2 : p0 - p2; h.c[3 + c] = S > 0 ? p1 + p3 : p1 - p3; }
  }
  return h;
}
template <int MU, int S> __device__ __forceinline__ SP recon(const HS &h) {
  SP r;
#pragma unroll
  for (int c = 0; c < 3; c++) {
    const cx h0 = h.c[c], h1 = h.c[3 + c];
    const cx mh0 = {-h0.re, -h0.im}, mh1 = {-h1.re, -h1.im};
    r.c[c] = h0;
    r.c[3 + c] = h1;
    if (MU == 0) { r.c[6 + c] = ti(S > 0 ? mh1 : h1); r.c[9 + c] = ti(S > 0 ? mh0 : h0); }
    else if (MU == 1) { r.c[6 + c] = S > 0 ? h1 : mh1; r.c[9 + c] = S > 0 ? mh0 : h0; }
    else if (MU == 2) { r.c[6 + c] = ti(S > 0 ? mh0 : h0); r.c[9 + c] = ti(S > 0 ? h1 : mh1); }
    else { r.c[6 + c] = S > 0 ? h0 : mh0; r.c[9 + c] = S > 0 ? h1 : mh1; }
  }
  return r;
}
__device__ __forceinline__ HS mul(const CM &u, const HS &s) {
  HS o;
  for (int sp = 0; sp < 2; sp++)
    for (int a = 0; a < 3; a++) {
      cx acc = cmul(u.m[3 * a], s.c[3 * sp]);
      acc = cmadd(u.m[3 * a + 1], s.c[3 * sp + 1], acc);
      o.c[3 * sp + a] = cmadd(u.m[3 * a + 2], s.c[3 * sp + 2], acc);
    }
  return o;
}
__device__ __forceinline__ int wrap(int n, int L) { n %= L; return n < 0 ? n + L : n; }
__device__ __forceinline__ int wrap_up(int n, int L) { return n + 1 == L ? 0 : n + 1; }
__device__ __forceinline__ int wrap_down(int n, int L) { return n == 0 ? L - 1 : n - 1; }
__device__ __forceinline__ const char *base(const JitArgs &a, int k, int par, int mu) {
  if (mu >= 0) return a.op[k] + (long long)(2 * mu + par) * a.blk[k];
  return a.op[k] + (a.all[k] ? (long long)par * a.blk[k] : 0);
}
__device__ __forceinline__ void third_row(CM &u) {
  for (int a = 0; a < 3; a++) {
    const int b = (a + 1) % 3, c = (a + 2) % 3;
    const cx t = cmul(u.m[b], u.m[3 + c]) - cmul(u.m[c], u.m[3 + b]);
    u.m[6 + a] = conj(t);
  }
}
// Loads: S = true for a field block read at one displacement only (no reuse between threads:
// streamed past L1, like the hand-written kernels' links), false for blocks read at several
// displacements (stencil reuse through L1/L2, like the dslash's neighbour spinors).
#if QDPJ_F64
template <bool S> __device__ __forceinline__ cx ldc(const char *b, int st, int k, int cb) {
  const double2 *q = (const double2 *)b + (long long)k * st + cb;
  double2 v;
  if (S) asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(q));
  else v = __ldg(q);
  return {v.x, v.y};
}
__device__ __forceinline__ void stc(char *b, int st, int k, int cb, cx v) {
  __stcs((double2 *)b + (long long)k * st + cb, make_double2(v.re, v.im));
}
#define QDPJ_LD(T, N, F) { T r; for (int k = 0; k < N; k++) r.F[k] = ldc<S>(b, st, k, cb); return r; }
#define QDPJ_ST(N, F) { for (int k = 0; k < N; k++) stc(b, st, k, cb, x.F[k]); }
template <bool S> __device__ __forceinline__ SP ld_sp(const char *b, int st, int cb) QDPJ_LD(SP, 12, c)
template <bool S> __device__ __forceinline__ CM ld_cm(const char *b, int st, int cb) QDPJ_LD(CM, 9, m)
template <bool S> __device__ __forceinline__ SM ld_sm(const char *b, int st, int cb) QDPJ_LD(SM, 16, m)
template <bool S> __device__ __forceinline__ CM ld_g12(const char *b, int st, int cb) {
  CM u;
  for (int k = 0; k < 6; k++) u.m[k] = ldc<S>(b, st, k, cb);
  third_row(u);
  return u;
}
__device__ __forceinline__ void st_sp(char *b, int st, int cb, const SP &x) QDPJ_ST(12, c)
__device__ __forceinline__ void st_cm(char *b, int st, int cb, const CM &x) QDPJ_ST(9, m)
__device__ __forceinline__ void st_sm(char *b, int st, int cb, const SM &x) QDPJ_ST(16, m)
#else
// fp32: pairs of complex numbers per float4 plane; colour matrices 4 float4 planes + 1 float2 plane
template <bool S> __device__ __forceinline__ void ld2(const char *b, int st, int k, int cb, cx &x, cx &y) {
  const float4 *q = (const float4 *)b + (long long)k * st + cb;
  float4 v;
  if (S) asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(q));
  else v = __ldg(q);
  x = {v.x, v.y};
  y = {v.z, v.w};
}
template <bool S> __device__ __forceinline__ cx ld1(const char *b, int cb) {
  const float2 *q = (const float2 *)b + cb;
  float2 v;
  if (S) asm("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(q));
  else v = __ldg(q);
  return {v.x, v.y};
}
__device__ __forceinline__ void st2(char *b, int st, int k, int cb, cx x, cx y) {
  __stcs((float4 *)b + (long long)k * st + cb, make_float4(x.re, x.im, y.re, y.im));
}
template <bool S> __device__ __forceinline__ SP ld_sp(const char *b, int st, int cb) {
  SP r;
  for (int k = 0; k < 6; k++) ld2<S>(b, st, k, cb, r.c[2 * k], r.c[2 * k + 1]);
  return r;
}
template <bool S> __device__ __forceinline__ SM ld_sm(const char *b, int st, int cb) {
  SM r;
  for (int k = 0; k < 8; k++) ld2<S>(b, st, k, cb, r.m[2 * k], r.m[2 * k + 1]);
  return r;
}
template <bool S> __device__ __forceinline__ CM ld_cm(const char *b, int st, int cb) {
  CM r;
  for (int k = 0; k < 4; k++) ld2<S>(b, st, k, cb, r.m[2 * k], r.m[2 * k + 1]);
  r.m[8] = ld1<S>(b + (long long)64 * st, cb);
  return r;
}
template <bool S> __device__ __forceinline__ CM ld_g12(const char *b, int st, int cb) {
  CM u;
  for (int k = 0; k < 3; k++) ld2<S>(b, st, k, cb, u.m[2 * k], u.m[2 * k + 1]);
  third_row(u);
  return u;
}
__device__ __forceinline__ void st_sp(char *b, int st, int cb, const SP &x) {
  for (int k = 0; k < 6; k++) st2(b, st, k, cb, x.c[2 * k], x.c[2 * k + 1]);
}
__device__ __forceinline__ void st_sm(char *b, int st, int cb, const SM &x) {
  for (int k = 0; k < 8; k++) st2(b, st, k, cb, x.m[2 * k], x.m[2 * k + 1]);
}
__device__ __forceinline__ void st_cm(char *b, int st, int cb, const CM &x) {
  for (int k = 0; k < 4; k++) st2(b, st, k, cb, x.m[2 * k], x.m[2 * k + 1]);
  __stcs((float2 *)(b + (long long)64 * st) + cb, make_float2(x.m[8].re, x.m[8].im));
}
#endif
)PRELUDE";

struct Generated {
  std::vector<Temp> temps;
  std::string src;
  double flops = 0, table2_reals = 0;
  // compulsory reals per output site: out QDP_ALL -> each distinct field once; out one parity ->
  // each distinct (field, parity block) once (e.g. the EO hopping term reads both parities of U)
  double compulsory_all = 0, compulsory_parity = 0;
  std::set<int> shift_dims;
  std::vector<std::pair<int, int>> leaf_disp_parity;  // (operand, parity flip) of every leaf load
};

int generate(const char *expr, int out_kind, int prec, const int *kinds, int nops, int part, Generated *g,
             std::string &err) {
  if (!expr) {
    err = "null expression";
    return QDP_EINVAL;
  }
  if (nops < 0 || nops > QDP_JIT_MAX_OPERANDS) {
    err = "too many operands";
    return QDP_EINVAL;
  }
  if (prec != QDP_F64 && prec != QDP_F32) {
    err = "bad precision";
    return QDP_EPREC;
  }
  Parser P(expr);
  NodeP root = P.expr();
  P.ws();
  if (root && P.s[P.i] != '\0') root = P.fail("trailing characters");
  if (!root) {
    err = "parse error: " + P.err;
    return QDP_EINVAL;
  }
  if (!typecheck(root.get(), kinds, nops, err)) return QDP_EINVAL;
  const bool sum = out_kind == QDP_JIT_SUM;  // global sum of a complex-scalar expression
  const Type want = sum ? T_CPLX
                  : out_kind == QDP_FERMION ? T_SP : out_kind == QDP_COLORMATRIX ? T_CM : out_kind == QDP_SPINMATRIX ? T_SM
                                                                                                            : T_GAMMA;
  if (want == T_GAMMA) {
    err = "output must be a fermion, colour matrix or spin matrix field";
    return QDP_EINVAL;
  }
  if (root->type != want) {
    err = std::string("expression is a ") + type_name(root->type) + ", the output a " + type_name(want);
    return QDP_EINVAL;
  }
  Gen G;
  G.kinds = kinds;
  G.prec = prec;
  G.part = part;
  G.count_leaves(root.get());
  const int d0[4] = {0, 0, 0, 0};
  G.collect(root.get(), d0);
  G.site(d0);
  const std::string v = G.emit(root.get(), d0);
  std::ostringstream s;
  s << "// generated by qdpb jit.cu from: " << expr << "\n";
  s << (prec == QDP_F64 ? "typedef double R;\n#define QDPJ_F64 1\n" : "typedef float R;\n#define QDPJ_F64 0\n");
  s << kPrelude;
  if (sum)  // grid-stride loop, fp64 accumulation, one fixed-order partial per block
    s << "extern \"C\" __global__ void qdp_jit_kernel(const JitArgs a, double *partials) {\n"
         "  double acc_re = 0.0, acc_im = 0.0;\n"
         "  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)a.nblk * a.Vh;\n"
         "       i += (long long)gridDim.x * blockDim.x) {\n";
  else
    s << "extern \"C\" __global__ void qdp_jit_kernel(const JitArgs a) {\n"
         "  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;\n"
         "  if (i >= (long long)a.nblk * a.Vh) return;\n";
  s << "  const int bi = (int)(i / a.Vh), cb = (int)(i - (long long)bi * a.Vh);\n"
       "  const int p = a.nblk == 2 ? bi : a.parity;\n"
       "  int c[4];\n"
       "  {\n"
       "    const int xh = cb % a.Lh0, r = cb / a.Lh0;\n"
       "    c[1] = r % a.L[1];\n"
       "    const int r2 = r / a.L[1];\n"
       "    c[2] = r2 % a.L[2];\n"
       "    c[3] = r2 / a.L[2];\n"
       "    c[0] = 2 * xh + ((p + c[1] + c[2] + c[3]) & 1);\n"
       "  }\n"
       "  (void)c;\n";
  s << G.body.str();
  if (sum) {
    s << "  acc_re += (double)" << v << ".re;\n  acc_im += (double)" << v << ".im;\n  }\n"
      << "  block_partial(acc_re, acc_im, partials);\n}\n";
  } else {
    const char *st = want == T_SP ? "st_sp" : want == T_CM ? "st_cm" : "st_sm";
    s << "  " << st << "(a.out + (long long)bi * a.out_blk, a.stride, cb, " << v << ");\n}\n";
  }
  if (G.temps.size() > 16) {
    err = "more than 16 distinct operand displacements across the halo path";
    return QDP_EUNSUPPORTED;
  }
  g->temps = G.temps;
  g->src = s.str();
  g->flops = G.flops;
  g->shift_dims = G.shift_dims;
  g->compulsory_all = g->compulsory_parity = sum ? 0 : type_reals(want);
  for (const auto &f : G.distinct) g->compulsory_all += type_reals(kind_type(kinds[f.first]), kinds[f.first]);
  for (const auto &f : G.distinct_par) g->compulsory_parity += type_reals(kind_type(kinds[f[0]]), kinds[f[0]]);
  g->table2_reals = G.table2_reals + (sum ? 0 : type_reals(want));
  // parity of every leaf load relative to the output site's parity
  for (const auto &kv : G.cse) {
    const std::string &k = kv.first;
    if (k.empty() || k[0] != '$') continue;
    const int leaf = atoi(k.c_str() + 1);
    const size_t at = k.find('@');
    int d[4] = {0, 0, 0, 0};
    sscanf(k.c_str() + at + 1, "%d,%d,%d,%d", &d[0], &d[1], &d[2], &d[3]);
    g->leaf_disp_parity.push_back({leaf, (std::abs(d[0]) + std::abs(d[1]) + std::abs(d[2]) + std::abs(d[3])) & 1});
  }
  return QDP_OK;
}

// ------------------------------------------------------------------ NVRTC (dlopen'ed)
typedef int (*nvrtcCreateProgram_t)(void **, const char *, const char *, int, const char *const *, const char *const *);
typedef int (*nvrtcCompileProgram_t)(void *, int, const char *const *);
typedef int (*nvrtcGetSize_t)(void *, size_t *);
typedef int (*nvrtcGetData_t)(void *, char *);
typedef int (*nvrtcDestroyProgram_t)(void **);
struct Nvrtc {
  bool ok = false;
  std::string why;
  nvrtcCreateProgram_t create;
  nvrtcCompileProgram_t compile;
  nvrtcGetSize_t log_size, cubin_size;
  nvrtcGetData_t log, cubin;
  nvrtcDestroyProgram_t destroy;
};
const Nvrtc &nvrtc() {
  static Nvrtc n = [] {
    Nvrtc r;
    void *h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      r.why = "libnvrtc.so.12 not found";
      return r;
    }
    r.create = (nvrtcCreateProgram_t)dlsym(h, "nvrtcCreateProgram");
    r.compile = (nvrtcCompileProgram_t)dlsym(h, "nvrtcCompileProgram");
    r.log_size = (nvrtcGetSize_t)dlsym(h, "nvrtcGetProgramLogSize");
    r.log = (nvrtcGetData_t)dlsym(h, "nvrtcGetProgramLog");
    r.cubin_size = (nvrtcGetSize_t)dlsym(h, "nvrtcGetCUBINSize");
    r.cubin = (nvrtcGetData_t)dlsym(h, "nvrtcGetCUBIN");
    r.destroy = (nvrtcDestroyProgram_t)dlsym(h, "nvrtcDestroyProgram");
    r.ok = r.create && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.destroy;
    if (!r.ok) r.why = "libnvrtc.so.12 lacks a required symbol";
    return r;
  }();
  return n;
}

// source -> sm_100a cubin
int compile_cubin(const std::string &src, std::vector<char> *cubin, std::string &err) {
  const Nvrtc &N = nvrtc();
  if (!N.ok) {
    err = N.why;
    return QDP_EUNSUPPORTED;
  }
  void *prog = nullptr;
  if (N.create(&prog, src.c_str(), "qdp_jit.cu", 0, nullptr, nullptr) != 0) {
    err = "nvrtcCreateProgram failed";
    return QDP_ECUDA;
  }
  std::vector<const char *> opts = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "--fmad=true"};
  // Register budget 168 (6 x 64-thread blocks per SM, the hand-written dslash's measured optimum,
  // DESIGN.md section 6): it also makes ptxas hoist more loads.  Measured on the generated hopping
  // term: no cap 322 us, 168 -> 247 us (hand-written 242 us); profiles/r01_jit_vs_handwritten.txt.
  std::string maxreg = "--maxrregcount=168";
  if (const char *e = getenv("QDPB_JIT_MAXRREG")) maxreg = std::string("--maxrregcount=") + e;  // experiments
  opts.push_back(maxreg.c_str());
  const int rc = N.compile(prog, (int)opts.size(), opts.data());
  if (rc != 0) {
    size_t n = 0;
    N.log_size(prog, &n);
    std::string log(n, '\0');
    N.log(prog, &log[0]);
    err = "nvrtc: " + log;
    N.destroy(&prog);
    return QDP_EINVAL;
  }
  size_t n = 0;
  N.cubin_size(prog, &n);
  cubin->resize(n);
  N.cubin(prog, cubin->data());
  N.destroy(&prog);
  return QDP_OK;
}

}  // namespace

void jit_release(qdp_ctx ctx) {
  for (auto &kv : ctx->jit) {
    for (qdp_field f : kv.second->temp_field) qdp_field_free(f);
    for (auto &v : kv.second->temp_steps)
      for (qdp_field f : v) qdp_field_free(f);
    if (kv.second->lib) cudaLibraryUnload(kv.second->lib);
    delete kv.second;
  }
  ctx->jit.clear();
}

namespace {
struct HostArgs {  // mirrors JitArgs of the generated prelude
  const char *op[24];
  char *out;
  long long blk[24];
  long long out_blk;
  int all[24];
  int L[4];
  int Lh0, Vh, stride, parity, nblk;
};

// Generate / look up the kernel of (expr, operands, output kind, subset), materialise its halo'd
// temporaries and fill the launch arguments (everything but the output).
int jit_prepare(qdp_ctx ctx, const char *expr, int out_kind, int subset, int prec, const qdp_field *ops, int nops,
                JitKernel **Kout, HostArgs *a) {
  const Geom &g = ctx->geom;
  int kinds[QDP_JIT_MAX_OPERANDS];
  for (int k = 0; k < nops; k++) kinds[k] = ops[k]->kind;
  // cache key: expression text, operand kinds and subsets, output kind and subset, precision,
  // and the dims reached through the halo path (they decide which leaves become temporaries)
  std::string key = std::string(expr) + "|" + std::to_string(out_kind) + "|" + std::to_string(subset) + "|" +
                    std::to_string(prec) + "|" + std::to_string(g.part);
  for (int k = 0; k < nops; k++) key += "|" + std::to_string(kinds[k]) + "/" + std::to_string(ops[k]->subset);
  // cache first: a hit skips parsing, type checking and source generation altogether
  auto it = ctx->jit.find(key);
  JitKernel *K = it == ctx->jit.end() ? nullptr : it->second;
  int rc;
  Generated gen;
  std::string err;
  if (!K && (rc = generate(expr, out_kind, prec, kinds, nops, g.part, &gen, err)))
    return set_error(ctx, rc, "jit: %s", err.c_str());
  // operand subsets: each leaf is read at parity out_parity ^ flip; a one-parity operand must match
  for (const auto &lp : K ? K->leaf_disp_parity : gen.leaf_disp_parity) {
    const qdp_field f = ops[lp.first];
    if (is_gauge(f->kind) && f->subset != QDP_ALL)
      return set_error(ctx, QDP_EINVAL, "jit: gauge operand $%d must cover all sites", lp.first);
    if (f->subset == QDP_ALL) continue;
    if (subset == QDP_ALL || (subset ^ lp.second) != f->subset)
      return set_error(ctx, QDP_EINVAL, "jit: operand $%d is read on parity it does not hold", lp.first);
  }
  if (!K) {
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<char> cubin;
    if ((rc = compile_cubin(gen.src, &cubin, err))) return set_error(ctx, rc, "jit: %s", err.c_str());
    std::unique_ptr<JitKernel> k(new JitKernel);
    QDP_CUDA(ctx, cudaLibraryLoadData(&k->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    QDP_CUDA(ctx, cudaLibraryGetKernel(&k->kern, k->lib, "qdp_jit_kernel"));
    cudaFuncAttributes attr;
    QDP_CUDA(ctx, cudaFuncGetAttributes(&attr, (const void *)k->kern));
    k->max_threads = attr.maxThreadsPerBlock;
    k->flops = gen.flops;
    k->bytes_all = gen.compulsory_all * (prec == QDP_F64 ? 8 : 4);
    k->bytes_parity = gen.compulsory_parity * (prec == QDP_F64 ? 8 : 4);
    k->key = (1L << 62) | (long)(std::hash<std::string>()(key) & ((1L << 61) - 1));
    for (const Temp &t : gen.temps) {
      k->temp_leaf.push_back(t.leaf);
      k->temp_dp.push_back({t.dp[0], t.dp[1], t.dp[2], t.dp[3]});
    }
    k->temp_field.assign(gen.temps.size(), nullptr);
    k->temp_steps.assign(gen.temps.size(), {});
    k->leaf_disp_parity = gen.leaf_disp_parity;
    ctx->jit_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    ctx->jit_compiled++;
    K = k.release();
    ctx->jit[key] = K;
  }

  memset(a, 0, sizeof *a);
  for (int k = 0; k < nops; k++) {
    a->op[k] = (const char *)ops[k]->data;
    a->all[k] = ops[k]->subset == QDP_ALL;
    // gauge: one (mu, parity) block
    a->blk[k] = (long long)parity_block_bytes(ops[k]->kind, prec, g.stride) / (is_gauge(ops[k]->kind) ? 4 : 1);
  }
  // halo'd temporaries: operand shifted by dp, one qdp_shift per unit step (faces exchanged there)
  for (size_t j = 0; j < K->temp_leaf.size(); j++) {
    const qdp_field src = ops[K->temp_leaf[j]];
    std::vector<std::pair<int, int>> steps;  // (mu, sign)
    for (int m = 0; m < 4; m++)
      for (int i = 0; i < std::abs(K->temp_dp[j][m]); i++) steps.push_back({m, K->temp_dp[j][m] > 0 ? 1 : -1});
    auto subset_after = [&](size_t n) { return src->subset == QDP_ALL ? QDP_ALL : src->subset ^ (int)(n & 1); };
    if (!K->temp_field[j]) {
      if ((rc = qdp_field_alloc(ctx, src->kind, prec, subset_after(steps.size()), &K->temp_field[j]))) return rc;
      for (size_t i = 0; i + 1 < steps.size(); i++) {
        qdp_field f;
        if ((rc = qdp_field_alloc(ctx, src->kind, prec, subset_after(i + 1), &f))) return rc;
        K->temp_steps[j].push_back(f);
      }
    }
    qdp_field in = src;
    for (size_t i = 0; i < steps.size(); i++) {
      qdp_field o = i + 1 == steps.size() ? K->temp_field[j] : K->temp_steps[j][i];
      if ((rc = qdp_shift(o, in, steps[i].first, steps[i].second))) return rc;
      in = o;
    }
    const int slot = QDP_JIT_MAX_OPERANDS + (int)j;
    const qdp_field t = K->temp_field[j];
    a->op[slot] = (const char *)t->data;
    a->all[slot] = t->subset == QDP_ALL;
    a->blk[slot] = (long long)parity_block_bytes(t->kind, prec, g.stride) / (is_gauge(t->kind) ? 4 : 1);
  }
  for (int m = 0; m < 4; m++) a->L[m] = g.L[m];
  a->Lh0 = g.Lh0;
  a->Vh = g.Vh;
  a->stride = g.stride;
  a->nblk = subset == QDP_ALL ? 2 : 1;
  a->parity = subset == QDP_ALL ? 0 : subset;
  *Kout = K;
  return QDP_OK;
}
}  // namespace

int jit_eval(qdp_field out, const char *expr, const qdp_field *ops, int nops) {
  qdp_ctx ctx = out->ctx;
  JitKernel *K;
  HostArgs a;
  int rc = jit_prepare(ctx, expr, out->kind, out->subset, out->prec, ops, nops, &K, &a);
  if (rc) return rc;
  a.out = (char *)out->data;
  a.out_blk = (long long)parity_block_bytes(out->kind, out->prec, ctx->geom.stride);
  const long sites = (long)a.nblk * ctx->geom.Vh;
  auto go = [&](int block) -> cudaError_t {
    if (block > K->max_threads) return cudaErrorLaunchOutOfResources;
    void *args[] = {&a};
    return cudaLaunchKernel((const void *)K->kern, dim3((unsigned)((sites + block - 1) / block)), dim3(block), args, 0,
                            ctx->stream);
  };
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_BLAS, &ev);
  prof_work(ctx, QDP_PK_BLAS, K->flops * sites, (a.nblk == 2 ? K->bytes_all : K->bytes_parity) * sites);
  if ((rc = tuned_launch(ctx, K->key ^ sites, go))) {
    prof_end(ctx, &ev);
    return rc;
  }
  return prof_end(ctx, &ev);
}

int jit_sum(qdp_ctx ctx, const char *expr, const qdp_field *ops, int nops, int subset, int prec, int slot) {
  JitKernel *K;
  HostArgs a;
  int rc = jit_prepare(ctx, expr, QDP_JIT_SUM, subset, prec, ops, nops, &K, &a);
  if (rc) return rc;
  const long sites = (long)a.nblk * ctx->geom.Vh;
  // fixed launch shape (256 threads, at most 8 blocks per SM, grid-stride): the block partials and
  // therefore the rounding of the sum do not depend on tuning
  const int block = 256;
  const long want = (sites + block - 1) / block;
  const int nb = (int)(want < 148 * 8 ? want : 148 * 8);
  if (block > K->max_threads) return set_error(ctx, QDP_EUNSUPPORTED, "jit: sum kernel exceeds its register budget");
  if ((rc = ensure_reduce(ctx, nb))) return rc;
  ProfEvent ev;
  prof_begin(ctx, QDP_PK_REDUCE, &ev);
  prof_work(ctx, QDP_PK_REDUCE, K->flops * sites, (a.nblk == 2 ? K->bytes_all : K->bytes_parity) * sites);
  double *partials = ctx->red_partials;
  void *args[] = {&a, &partials};
  cudaError_t e = cudaLaunchKernel((const void *)K->kern, dim3(nb), dim3(block), args, 0, ctx->stream);
  if (e != cudaSuccess) {
    prof_end(ctx, &ev);
    return cuda_check(ctx, e, "jit sum launch");
  }
  if ((rc = prof_end(ctx, &ev))) return rc;
  if ((rc = reduce_partials(ctx, nb, slot))) return rc;
  return reduce_global(ctx, slot, 2);
}

int jit_source(const char *expr, int out_kind, int out_subset, int prec, const int *kinds, int nops, char *src,
               size_t cap, size_t *src_len, double work[3], int compile, std::string &err) {
  Generated gen;
  int rc = generate(expr, out_kind, prec, kinds, nops, 0, &gen, err);
  if (rc) return rc;
  if (work) {
    work[0] = gen.flops;
    work[1] = (out_subset == QDP_ALL ? gen.compulsory_all : gen.compulsory_parity) * (prec == QDP_F64 ? 8 : 4);
    work[2] = gen.table2_reals * (prec == QDP_F64 ? 8 : 4);
  }
  if (src_len) *src_len = gen.src.size() + 1;
  if (src && cap) {
    strncpy(src, gen.src.c_str(), cap - 1);
    src[cap - 1] = '\0';
  }
  if (compile) {
    std::vector<char> cubin;
    if ((rc = compile_cubin(gen.src, &cubin, err))) return rc;
  }
  return QDP_OK;
}

}  // namespace qdpb
