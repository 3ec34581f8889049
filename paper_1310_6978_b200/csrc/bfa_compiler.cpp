// bfa_compiler.cpp -- parser, gate DAG with Reduction, LUT3 mapping and CUDA
// code generation for libbfa.  See bfa_compiler.hpp for the pipeline.
#include "bfa_compiler.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <atomic>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <set>
#include <sstream>
#include <thread>

namespace bfa {

// ============================================================== Dag
Dag::Dag() {
  nodes.push_back(Node{NK_CONST, 0, 0, 0, 0u});  // node 0: the word 0 (literal 1 = all ones)
  word_table_[0u] = 0;
}

Lit Dag::word(uint32_t w) {
  bool neg = (w & 1u) != 0;           // normalise: stored word has bit 0 clear
  uint32_t key = neg ? ~w : w;
  auto it = word_table_.find(key);
  if (it != word_table_.end()) return mk_lit(it->second, neg);
  uint32_t id = (uint32_t)nodes.size();
  nodes.push_back(Node{NK_CONST, 0, 0, 0, key});
  word_table_[key] = id;
  return mk_lit(id, neg);
}

Lit Dag::var(uint32_t id) {
  auto it = var_table_.find(id);
  if (it != var_table_.end()) return mk_lit(it->second, false);
  uint32_t n = (uint32_t)nodes.size();
  nodes.push_back(Node{NK_VAR, 0, 0, 0, id});
  var_table_[id] = n;
  return mk_lit(n, false);
}

// Bitwise application of a 2-input truth table (bit a+2b) to two words.
static inline uint32_t apply2(uint8_t tt, uint32_t A, uint32_t B) {
  uint32_t r = 0;
  if (tt & 1) r |= ~A & ~B;
  if (tt & 2) r |= A & ~B;
  if (tt & 4) r |= ~A & B;
  if (tt & 8) r |= A & B;
  return r;
}

// Negate input a / input b of a 2-input truth table.
static inline uint8_t tt_neg_a(uint8_t tt) { return (uint8_t)(((tt & 0x5) << 1) | ((tt & 0xA) >> 1)); }
static inline uint8_t tt_neg_b(uint8_t tt) { return (uint8_t)(((tt & 0x3) << 2) | ((tt & 0xC) >> 2)); }
static inline uint8_t tt_swap(uint8_t tt) { return (uint8_t)((tt & 0x9) | ((tt & 0x2) << 1) | ((tt & 0x4) >> 1)); }

// The constructor is the Reduction step: constants are
// propagated, x op x and x op ~x are folded, NOTs are absorbed into the
// consumer's truth table, and structurally equal gates are shared.
Lit Dag::gate(uint8_t tt, Lit la, Lit lb) {
  tt &= 0xF;
  if (lit_neg(la)) tt = tt_neg_a(tt);
  if (lit_neg(lb)) tt = tt_neg_b(tt);
  uint32_t a = lit_node(la), b = lit_node(lb);
  const Node& na = nodes[a];
  const Node& nb = nodes[b];
  if (na.kind == NK_CONST && nb.kind == NK_CONST) return word(apply2(tt, na.val, nb.val));
  // a is the Boolean constant 0: f(0, b) = b ? tt[2] : tt[0]
  auto unary = [&](int f0, int f1, Lit x) -> Lit {
    if (f0 == f1) return f0 ? const1() : const0();
    return f1 ? x : (x ^ 1u);
  };
  if (na.kind == NK_CONST && na.val == 0 && a == 0) return unary(tt & 1, (tt >> 2) & 1, mk_lit(b, false));
  if (nb.kind == NK_CONST && nb.val == 0 && b == 0) return unary(tt & 1, (tt >> 1) & 1, mk_lit(a, false));
  if (a == b) return unary(tt & 1, (tt >> 3) & 1, mk_lit(a, false));
  // truth tables that ignore an input
  if ((tt & 0x3) == ((tt >> 2) & 0x3)) return unary(tt & 1, (tt >> 1) & 1, mk_lit(a, false));
  if ((tt & 0x5) == ((tt >> 1) & 0x5)) return unary(tt & 1, (tt >> 2) & 1, mk_lit(b, false));
  if (a > b) { std::swap(a, b); tt = tt_swap(tt); }
  bool neg = false;
  if (tt & 1) { tt = (uint8_t)(~tt & 0xF); neg = true; }  // normalise f(0,0) = 0
  uint64_t key = ((uint64_t)tt << 58) ^ ((uint64_t)a << 29) ^ (uint64_t)b;
  auto it = gate_table_.find(key);
  if (it != gate_table_.end()) return mk_lit(it->second, neg);
  uint32_t id = (uint32_t)nodes.size();
  nodes.push_back(Node{NK_GATE, tt, a, b, 0});
  gate_table_[key] = id;
  return mk_lit(id, neg);
}

size_t Dag::gate_count() const {
  size_t g = 0;
  for (const Node& n : nodes) g += n.kind == NK_GATE;
  return g;
}

// ============================================================== parser
// An independent recursive-descent parser for the grammar of include/bfa.h.
namespace {

enum Tok { EOF_, SEP, NOT_, AND_, XOR_, OR_, IMP_, IFF_, LP, RP, EQ, VAR, NAME, ZERO, ONE, LET };

struct Lexer {
  const std::string& s;
  size_t i = 0;
  int line = 1, col = 1, depth = 0;
  Tok tok = EOF_;
  std::string text;
  long long ival = 0;
  int tline = 1, tcol = 1;
  std::string err;

  explicit Lexer(const std::string& src) : s(src) {}

  bool fail(const std::string& msg) {
    if (err.empty()) err = std::to_string(tline) + ":" + std::to_string(tcol) + ": " + msg;
    tok = EOF_;
    return false;
  }
  char at(size_t k) const { return k < s.size() ? s[k] : '\0'; }
  void adv(size_t k) { i += k; col += (int)k; }

  bool next() {
    for (;;) {
      char c = at(i);
      if (c == '#') { while (at(i) && at(i) != '\n') adv(1); continue; }
      if (c == ' ' || c == '\t' || c == '\r') { adv(1); continue; }
      if (c == '\n' && depth > 0) { i++; line++; col = 1; continue; }
      break;
    }
    tline = line; tcol = col;
    char c = at(i);
    switch (c) {
      case '\0': tok = EOF_; return true;
      case '\n': i++; line++; col = 1; tok = SEP; return true;
      case ';': adv(1); tok = SEP; return true;
      case '~': adv(1); tok = NOT_; return true;
      case '&': adv(1); tok = AND_; return true;
      case '^': adv(1); tok = XOR_; return true;
      case '|': adv(1); tok = OR_; return true;
      case '(': adv(1); depth++; tok = LP; return true;
      case ')': adv(1); if (depth) depth--; tok = RP; return true;
      case '=': adv(1); tok = EQ; return true;
      default: break;
    }
    if (c == '-' && at(i + 1) == '>') { adv(2); tok = IMP_; return true; }
    if (c == '<' && at(i + 1) == '-' && at(i + 2) == '>') { adv(3); tok = IFF_; return true; }
    if (std::isdigit((unsigned char)c)) {
      size_t k = i;
      while (std::isdigit((unsigned char)at(k))) k++;
      std::string num = s.substr(i, k - i);
      if (num == "0") tok = ZERO;
      else if (num == "1") tok = ONE;
      else return fail("only the constants 0 and 1 are allowed");
      adv(k - i);
      return true;
    }
    if (std::isalpha((unsigned char)c) || c == '_') {
      size_t k = i;
      while (std::isalnum((unsigned char)at(k)) || at(k) == '_') k++;
      text = s.substr(i, k - i);
      adv(k - i);
      bool is_var = text.size() >= 2 && text[0] == 'x' &&
                    std::all_of(text.begin() + 1, text.end(), [](char ch) { return std::isdigit((unsigned char)ch); });
      if (is_var) {
        ival = 0;
        for (size_t q = 1; q < text.size() && ival <= 1000000; q++) ival = ival * 10 + (text[q] - '0');
        tok = VAR;
      } else {
        tok = text == "let" ? LET : NAME;
      }
      return true;
    }
    return fail(std::string("unexpected character '") + c + "'");
  }
};

struct Parser {
  Lexer lx;
  Parsed* P;
  std::unordered_map<std::string, Lit> names;

  Parser(const std::string& src, Parsed* out) : lx(src), P(out) {}
  bool ok() const { return lx.err.empty(); }

  // Balanced reduction of an operand list (n-ary & / | and the constraint conjunction).
  Lit reduce_balanced(std::vector<Lit>& v, bool is_and) {
    while (v.size() > 1) {
      std::vector<Lit> nxt;
      for (size_t k = 0; k + 1 < v.size(); k += 2)
        nxt.push_back(is_and ? P->dag.AND(v[k], v[k + 1]) : P->dag.OR(v[k], v[k + 1]));
      if (v.size() & 1) nxt.push_back(v.back());
      v.swap(nxt);
    }
    return v[0];
  }

  Lit atom() {
    Dag& d = P->dag;
    switch (lx.tok) {
      case VAR: {
        if (lx.ival > 63) { lx.fail("variable id " + std::to_string(lx.ival) + " > 63"); return 0; }
        int id = (int)lx.ival;
        P->max_var = std::max(P->max_var, id);
        P->support_mask |= 1ull << id;
        P->tree_nodes++;
        lx.next();
        return d.var((uint32_t)id);
      }
      case ZERO: P->tree_nodes++; lx.next(); return d.const0();
      case ONE: P->tree_nodes++; lx.next(); return d.const1();
      case NAME: {
        auto it = names.find(lx.text);
        if (it == names.end()) { lx.fail("name '" + lx.text + "' used before definition"); return 0; }
        P->tree_nodes++;
        lx.next();
        return it->second;
      }
      case LP: {
        lx.next();
        Lit e = expr();
        if (!ok()) return 0;
        if (lx.tok != RP) { lx.fail("expected ')'"); return 0; }
        lx.next();
        return e;
      }
      default: lx.fail("expected an operand"); return 0;
    }
  }
  Lit unary() {
    if (lx.tok == NOT_) {
      lx.next();
      Lit a = unary();
      P->tree_nodes++;
      return a ^ 1u;
    }
    return atom();
  }
  Lit chain(Tok op, bool is_and, Lit (Parser::*sub)()) {
    Lit first = (this->*sub)();
    if (!ok() || lx.tok != op) return first;
    std::vector<Lit> ops{first};
    while (ok() && lx.tok == op) {
      lx.next();
      ops.push_back((this->*sub)());
      P->tree_nodes++;
    }
    if (!ok()) return 0;
    return reduce_balanced(ops, is_and);
  }
  Lit and_() { return chain(AND_, true, &Parser::unary); }
  Lit xor_() {
    Lit a = and_();
    while (ok() && lx.tok == XOR_) { lx.next(); Lit b = and_(); P->tree_nodes++; a = P->dag.XOR(a, b); }
    return a;
  }
  Lit or_() { return chain(OR_, false, &Parser::xor_); }
  Lit imp() {
    Lit a = or_();
    if (!ok() || lx.tok != IMP_) return a;
    lx.next();
    Lit b = imp();
    P->tree_nodes++;
    return P->dag.IMP(a, b);
  }
  Lit expr() {
    Lit a = imp();
    while (ok() && lx.tok == IFF_) { lx.next(); Lit b = imp(); P->tree_nodes++; a = P->dag.IFF(a, b); }
    return a;
  }

  bool bind(const std::string& name, Lit v) {
    if (names.count(name)) return lx.fail("name '" + name + "' redefined");
    names[name] = v;
    P->lets++;
    return true;
  }

  bool program() {
    std::vector<Lit> constraints;
    lx.next();
    while (ok() && lx.tok != EOF_) {
      if (lx.tok == SEP) { lx.next(); continue; }
      if (lx.tok == LET) {
        lx.next();
        if (lx.tok != NAME) return lx.fail("expected a name after 'let'");
        std::string name = lx.text;
        lx.next();
        if (lx.tok != EQ) return lx.fail("expected '='");
        lx.next();
        Lit v = expr();
        if (!ok()) return false;
        if (!bind(name, v)) return false;
      } else if (lx.tok == NAME) {
        // one-token lookahead for NAME '=' : snapshot the lexer
        Lexer save = lx;
        std::string name = lx.text;
        lx.next();
        if (ok() && lx.tok == EQ) {
          lx.next();
          Lit v = expr();
          if (!ok()) return false;
          if (!bind(name, v)) return false;
          constraints.push_back(v);
        } else {
          if (!ok()) return false;
          lx.i = save.i; lx.line = save.line; lx.col = save.col; lx.depth = save.depth;
          lx.tok = save.tok; lx.text = save.text; lx.tline = save.tline; lx.tcol = save.tcol;
          Lit v = expr();
          if (!ok()) return false;
          constraints.push_back(v);
        }
      } else {
        Lit v = expr();
        if (!ok()) return false;
        constraints.push_back(v);
      }
      if (!ok()) return false;
      if (lx.tok != SEP && lx.tok != EOF_) return lx.fail("expected ';' or end of line");
    }
    if (!ok()) return false;
    if (constraints.empty()) {
      P->root = P->dag.const1();
    } else {
      P->tree_nodes += constraints.size() - 1;
      P->root = reduce_balanced(constraints, true);
    }
    return true;
  }
};

}  // namespace

int parse_program(const std::string& text, Parsed* out, std::string* err) {
  *out = Parsed();
  Parser ps(text, out);
  if (!ps.program()) {
    if (err) *err = ps.lx.err.empty() ? "parse error" : ps.lx.err;
    return -1;
  }
  return 0;
}

// ============================================================== rebuild (specialise)
// Rebuild the cone of `root` from `src` into `dst`, substituting every
// variable by subst[id] (a literal of dst).  dst.gate() re-runs the Reduction
// so substituted constants propagate (cofactoring).
static Lit rebuild(const Dag& src, Lit root, const std::vector<Lit>& subst, Dag& dst,
                   std::vector<Lit>& memo, std::vector<uint8_t>& done) {
  std::vector<uint32_t> stack{lit_node(root)};
  while (!stack.empty()) {
    uint32_t n = stack.back();
    if (done[n]) { stack.pop_back(); continue; }
    const Node& nd = src.nodes[n];
    if (nd.kind == NK_CONST) {
      memo[n] = n == 0 ? dst.const0() : dst.word(nd.val);
      done[n] = 1; stack.pop_back(); continue;
    }
    if (nd.kind == NK_VAR) {
      memo[n] = subst[nd.val];
      done[n] = 1; stack.pop_back(); continue;
    }
    if (!done[nd.a]) { stack.push_back(nd.a); continue; }
    if (!done[nd.b]) { stack.push_back(nd.b); continue; }
    memo[n] = dst.gate(nd.tt, memo[nd.a], memo[nd.b]);
    done[n] = 1;
    stack.pop_back();
  }
  return memo[lit_node(root)] ^ (root & 1u);
}

Parsed assume(const Parsed& src, int n, uint64_t mask, uint64_t values, std::vector<int>* free_ids) {
  Parsed out;
  out.tree_nodes = src.tree_nodes;
  out.lets = src.lets;
  std::vector<Lit> subst(64, 0);
  std::vector<int> ids;
  for (int v = 0; v < 64; v++) {
    if (v < n && ((mask >> v) & 1)) {
      subst[v] = ((values >> v) & 1) ? out.dag.const1() : out.dag.const0();
    } else {
      subst[v] = out.dag.var((uint32_t)ids.size());
      if (v < n) ids.push_back(v);
    }
  }
  std::vector<uint8_t> done(src.dag.nodes.size(), 0);
  std::vector<Lit> memo(src.dag.nodes.size(), 0);
  out.root = rebuild(src.dag, src.root, subst, out.dag, memo, done);
  // support of the reduced program
  std::vector<uint8_t> seen(out.dag.nodes.size(), 0);
  std::vector<uint32_t> st{lit_node(out.root)};
  while (!st.empty()) {
    uint32_t k = st.back(); st.pop_back();
    if (seen[k]) continue;
    seen[k] = 1;
    const Node& nd = out.dag.nodes[k];
    if (nd.kind == NK_GATE) { st.push_back(nd.a); st.push_back(nd.b); }
    if (nd.kind == NK_VAR) { out.support_mask |= 1ull << nd.val; out.max_var = std::max(out.max_var, (int)nd.val); }
  }
  if (free_ids) *free_ids = ids;
  return out;
}

uint32_t gate_count(const Parsed& p) {
  std::vector<uint8_t> seen(p.dag.nodes.size(), 0);
  std::vector<uint32_t> st{lit_node(p.root)};
  uint32_t g = 0;
  while (!st.empty()) {
    uint32_t k = st.back(); st.pop_back();
    if (seen[k]) continue;
    seen[k] = 1;
    const Node& nd = p.dag.nodes[k];
    if (nd.kind == NK_GATE) { g++; st.push_back(nd.a); st.push_back(nd.b); }
  }
  return g;
}

std::vector<int> choose_cofactor_vars(const Parsed& p, int k, int j, uint64_t* best_total, int threads) {
  std::vector<int> chosen;
  if (best_total) *best_total = UINT64_MAX;
  threads = std::max(1, std::min(threads, 64));
  for (int step = 0; step < j; step++) {
    std::vector<int> cand;
    for (int v = 0; v < k; v++)
      if (((p.support_mask >> v) & 1) && std::find(chosen.begin(), chosen.end(), v) == chosen.end()) cand.push_back(v);
    // total gates of the 2^(step+1) cofactors for each candidate (candidates
    // in parallel when threads > 1; the choice -- least total, ties to the
    // lowest variable -- does not depend on the thread count)
    std::vector<uint64_t> total(cand.size(), 0);
    auto score = [&](size_t ci) {
      const int v = cand[ci];
      uint64_t mask = 1ull << v;
      for (int c : chosen) mask |= 1ull << c;
      uint64_t t = 0;
      for (uint64_t a = 0; a < (1ull << (chosen.size() + 1)); a++) {
        uint64_t values = 0;
        int bit = 0;
        for (int c : chosen) values |= ((a >> bit++) & 1) << c;
        values |= ((a >> bit) & 1) << v;
        t += gate_count(assume(p, k, mask, values, nullptr));
      }
      total[ci] = t;
    };
    if (threads == 1 || cand.size() < 2) {
      for (size_t ci = 0; ci < cand.size(); ci++) score(ci);
    } else {
      std::atomic<size_t> next{0};
      std::vector<std::thread> th;
      for (int w = 0; w < std::min<int>(threads, (int)cand.size()); w++)
        th.emplace_back([&] {
          for (size_t ci; (ci = next.fetch_add(1)) < cand.size();) score(ci);
        });
      for (auto& x : th) x.join();
    }
    int best_v = -1;
    uint64_t best = UINT64_MAX;
    for (size_t ci = 0; ci < cand.size(); ci++)
      if (total[ci] < best) { best = total[ci]; best_v = cand[ci]; }
    if (best_v < 0) break;
    chosen.push_back(best_v);
    if (best_total) *best_total = best;
  }
  return chosen;
}

// ============================================================== LUT3 mapping
namespace {

struct Cut {
  uint32_t leaf[3];
  uint8_t n;
  uint8_t tt;   // over slots (0xF0, 0xCC, 0xAA)
  float cost;
};

constexpr uint8_t kPat[3] = {0xF0, 0xCC, 0xAA};

inline uint8_t apply3(uint8_t tt, uint8_t x, uint8_t y, uint8_t z) {
  uint8_t r = 0;
  for (int k = 0; k < 8; k++) {
    if (!((tt >> k) & 1)) continue;
    uint8_t m = (uint8_t)(((k & 4) ? x : ~x) & ((k & 2) ? y : ~y) & ((k & 1) ? z : ~z));
    r |= m;
  }
  return r;
}

// expand cut c to the slot patterns of the merged leaf list L
inline uint8_t expand(const Cut& c, const uint32_t* L, int nl) {
  uint8_t X[3] = {0, 0, 0};
  for (int j = 0; j < c.n; j++)
    for (int q = 0; q < nl; q++)
      if (L[q] == c.leaf[j]) X[j] = kPat[q];
  return apply3(c.tt, X[0], X[1], X[2]);
}

}  // namespace

// IMAD option of a gate (x, u, f0, f1); valid when u is word-uniform
struct ImadOpt {
  uint32_t x = 0, u = 0;
  uint8_t f0 = 0, f1 = 0;
  bool ok = false;
};

// unary code of f over x from (f(0), f(1)): 0:"0" 1:"~0" 2:"x" 3:"~x"
static inline uint8_t unary_code(int v0, int v1) {
  if (v0 == v1) return v0 ? 1 : 0;
  return v1 ? 2 : 3;
}

MapResult map_luts(const Dag& dag, const std::vector<Lit>& outputs,
                   const std::vector<uint8_t>& var_level, const double weights[4], double imad_cost,
                   int area_passes) {
  const size_t N = dag.nodes.size();
  MapResult res;
  res.node_level.assign(N, 0);
  std::vector<uint8_t> in_cone(N, 0);
  std::vector<uint32_t> fanout(N, 0);
  {
    std::vector<uint32_t> st;
    for (Lit o : outputs) { st.push_back(lit_node(o)); fanout[lit_node(o)]++; }
    while (!st.empty()) {
      uint32_t n = st.back(); st.pop_back();
      if (in_cone[n]) continue;
      in_cone[n] = 1;
      const Node& nd = dag.nodes[n];
      if (nd.kind == NK_GATE) {
        fanout[nd.a]++; fanout[nd.b]++;
        st.push_back(nd.a); st.push_back(nd.b);
      }
    }
  }
  for (size_t n = 0; n < N; n++) {
    const Node& nd = dag.nodes[n];
    if (nd.kind == NK_VAR) res.node_level[n] = var_level[nd.val];
    else if (nd.kind == NK_GATE) res.node_level[n] = std::max(res.node_level[nd.a], res.node_level[nd.b]);
  }
  // word-uniform nodes: 0 or ~0 in every 32-bit word (no lane mask in the cone)
  std::vector<uint8_t> uniform(N, 0);
  for (size_t n = 0; n < N; n++) {
    const Node& nd = dag.nodes[n];
    if (nd.kind == NK_VAR) uniform[n] = 1;
    else if (nd.kind == NK_CONST) uniform[n] = n == 0;
    else uniform[n] = uniform[nd.a] && uniform[nd.b];
  }
  std::vector<ImadOpt> imad(N);
  std::vector<uint8_t> use_imad(N, 0);
  // cut sets in one flat array: <= kMaxCuts priority cuts + the trivial cut
  // per node (no per-node allocation: map_luts runs inside the role search)
  constexpr int kMaxCuts = 8, kSlots = kMaxCuts + 1;
  std::vector<Cut> cutbuf(N * kSlots);
  std::vector<uint8_t> ncut(N, 0);
  auto cuts_of = [&](size_t k) { return &cutbuf[k * kSlots]; };
  std::vector<float> af(N, 0.f);
  auto leaf_share = [&](uint32_t l) -> float {
    return dag.nodes[l].kind == NK_GATE ? af[l] / (float)std::max<uint32_t>(1, fanout[l]) : 0.f;
  };
  for (size_t n = 0; n < N; n++) {
    if (!in_cone[n]) continue;
    const Node& nd = dag.nodes[n];
    Cut triv{{(uint32_t)n, 0, 0}, 1, 0xF0, 0.f};
    if (nd.kind != NK_GATE) { cuts_of(n)[0] = triv; ncut[n] = 1; continue; }
    Cut cand[kSlots * kSlots];
    int nc = 0;
    const Cut* CA = cuts_of(nd.a);
    const Cut* CB = cuts_of(nd.b);
    for (int ia = 0; ia < ncut[nd.a]; ia++) {
      const Cut& ca = CA[ia];
      for (int ib = 0; ib < ncut[nd.b]; ib++) {
        const Cut& cb = CB[ib];
        uint32_t L[6]; int nl = 0;
        for (int j = 0; j < ca.n; j++) L[nl++] = ca.leaf[j];
        for (int j = 0; j < cb.n; j++) {
          bool dup = false;
          for (int q = 0; q < nl; q++) dup |= L[q] == cb.leaf[j];
          if (!dup) L[nl++] = cb.leaf[j];
        }
        if (nl > 3) continue;
        std::sort(L, L + nl);
        Cut c{{0, 0, 0}, (uint8_t)nl, 0, 0.f};
        for (int q = 0; q < nl; q++) c.leaf[q] = L[q];
        uint8_t A = expand(ca, L, nl), B = expand(cb, L, nl);
        uint8_t r = 0;
        if (nd.tt & 1) r |= (uint8_t)(~A & ~B);
        if (nd.tt & 2) r |= (uint8_t)(A & ~B);
        if (nd.tt & 4) r |= (uint8_t)(~A & B);
        if (nd.tt & 8) r |= (uint8_t)(A & B);
        c.tt = r;
        float cost = (float)weights[res.node_level[n]];
        for (int q = 0; q < nl; q++) cost += leaf_share(L[q]);
        c.cost = cost;
        bool dup = false;
        for (int e = 0; e < nc && !dup; e++)
          dup = cand[e].n == c.n && std::equal(cand[e].leaf, cand[e].leaf + c.n, c.leaf);
        if (!dup) cand[nc++] = c;
      }
    }
    std::stable_sort(cand, cand + nc, [](const Cut& x, const Cut& y) {
      if (x.cost != y.cost) return x.cost < y.cost;
      return x.n < y.n;
    });
    nc = std::min(nc, kMaxCuts);
    af[n] = nc == 0 ? (float)weights[res.node_level[n]] : cand[0].cost;
    // IMAD cell: u ? f1(x) : f0(x) for a word-uniform input u
    if (imad_cost > 0 && (uniform[nd.a] || uniform[nd.b])) {
      ImadOpt o;
      // prefer as u the uniform input at the lower loop level (its operand
      // registers are computed less often); tie -> input b
      bool ub = uniform[nd.b] && (!uniform[nd.a] || res.node_level[nd.b] <= res.node_level[nd.a]);
      if (ub) {   // tt bit (a + 2b): x = a, u = b
        o.x = nd.a; o.u = nd.b;
        o.f0 = unary_code(nd.tt & 1, (nd.tt >> 1) & 1);
        o.f1 = unary_code((nd.tt >> 2) & 1, (nd.tt >> 3) & 1);
      } else {    // x = b, u = a
        o.x = nd.b; o.u = nd.a;
        o.f0 = unary_code(nd.tt & 1, (nd.tt >> 2) & 1);
        o.f1 = unary_code((nd.tt >> 1) & 1, (nd.tt >> 3) & 1);
      }
      o.ok = true;
      imad[n] = o;
      float c = (float)(weights[res.node_level[n]] * imad_cost) + leaf_share(o.x) + leaf_share(o.u);
      if (c < af[n]) { af[n] = c; use_imad[n] = 1; }
    }
    std::copy(cand, cand + nc, cuts_of(n));
    cuts_of(n)[nc] = triv;
    ncut[n] = (uint8_t)(nc + 1);
  }
  // exact-area recovery (the priority-cut mapper's final passes): with the
  // cover's reference counts, every referenced gate re-chooses among its
  // cuts (and its IMAD cell) the one that adds the least loop-weighted area
  // given everything else in the cover -- area flow only estimates sharing
  if (area_passes > 0) {
    std::vector<int> choice(N, 0);   // cut index, or -1 = IMAD cell
    for (size_t n = 0; n < N; n++) choice[n] = use_imad[n] ? -1 : 0;
    std::vector<uint32_t> refs(N, 0);
    auto is_gate = [&](uint32_t l) { return dag.nodes[l].kind == NK_GATE; };
    auto cell_w = [&](uint32_t n, int ch) {
      return weights[res.node_level[n]] * (ch < 0 ? imad_cost : 1.0);
    };
    auto leaves = [&](uint32_t n, int ch, uint32_t* L) -> int {
      if (ch < 0) { L[0] = imad[n].x; L[1] = imad[n].u; return 2; }
      const Cut& c = cuts_of(n)[ch];
      for (int q = 0; q < c.n; q++) L[q] = c.leaf[q];
      return c.n;
    };
    std::function<double(uint32_t, int)> ref = [&](uint32_t n, int ch) {
      double a = cell_w(n, ch);
      uint32_t L[3];
      const int k = leaves(n, ch, L);
      for (int q = 0; q < k; q++)
        if (is_gate(L[q]) && refs[L[q]]++ == 0) a += ref(L[q], choice[L[q]]);
      return a;
    };
    std::function<double(uint32_t, int)> deref = [&](uint32_t n, int ch) {
      double a = cell_w(n, ch);
      uint32_t L[3];
      const int k = leaves(n, ch, L);
      for (int q = 0; q < k; q++)
        if (is_gate(L[q]) && --refs[L[q]] == 0) a += deref(L[q], choice[L[q]]);
      return a;
    };
    for (Lit o : outputs) {
      const uint32_t r = lit_node(o);
      if (is_gate(r) && refs[r]++ == 0) ref(r, choice[r]);
    }
    for (int pass = 0; pass < area_passes; pass++) {
      for (size_t n = 0; n < N; n++) {
        if (!refs[n] || !is_gate((uint32_t)n)) continue;
        deref((uint32_t)n, choice[n]);
        int best = choice[n];
        double best_a = 1e300;
        const int nc = (int)ncut[n] - 1;  // the trivial cut last
        for (int ch = (imad[n].ok ? -1 : 0); ch < nc; ch++) {
          const double a = ref((uint32_t)n, ch);
          deref((uint32_t)n, ch);
          if (a < best_a - 1e-9 || (a <= best_a + 1e-9 && ch == choice[n])) { best_a = a; best = ch; }
        }
        choice[n] = best;
        ref((uint32_t)n, best);
      }
    }
    for (size_t n = 0; n < N; n++) {
      if (!is_gate((uint32_t)n) || !in_cone[n]) continue;
      use_imad[n] = choice[n] < 0;
      if (choice[n] > 0) std::swap(cuts_of(n)[0], cuts_of(n)[choice[n]]);
    }
  }
  // cover extraction from the outputs (reverse topological order)
  std::vector<uint8_t> req(N, 0);
  for (Lit o : outputs) req[lit_node(o)] = 1;
  for (size_t k = N; k-- > 0;) {
    if (!req[k] || dag.nodes[k].kind != NK_GATE) continue;
    if (use_imad[k]) {
      const ImadOpt& o = imad[k];
      Lut cell{};
      cell.root = (uint32_t)k;
      cell.kind = 1;
      cell.nin = 2;
      cell.in[0] = o.x; cell.in[1] = o.u; cell.in[2] = o.u;
      cell.f0 = o.f0; cell.f1 = o.f1;
      cell.level = res.node_level[k];
      res.luts.push_back(cell);
      req[o.x] = 1; req[o.u] = 1;
      continue;
    }
    const Cut& c = cuts_of(k)[0];
    Lut lut{};
    lut.root = (uint32_t)k;
    lut.nin = c.n;
    for (int q = 0; q < 3; q++) lut.in[q] = q < c.n ? c.leaf[q] : c.leaf[0];
    lut.imm = c.tt;
    lut.level = res.node_level[k];
    res.luts.push_back(lut);
    for (int q = 0; q < c.n; q++) req[c.leaf[q]] = 1;
  }
  std::reverse(res.luts.begin(), res.luts.end());
  return res;
}

// ============================================================== codegen
namespace {

constexpr uint32_t kLane[5] = {0xAAAAAAAAu, 0xCCCCCCCCu, 0xF0F0F0F0u, 0xFF00FF00u, 0xFFFF0000u};

std::string hex32(uint32_t w) {
  char b[16];
  snprintf(b, sizeof b, "0x%08xu", w);
  return b;
}

struct Emitter {
  const Dag& d;
  std::ostringstream& os;
  Emitter(const Dag& dag, std::ostringstream& o) : d(dag), os(o) {}

  std::string name(uint32_t n) const {
    const Node& nd = d.nodes[n];
    if (nd.kind == NK_CONST) return hex32(nd.val);
    if (nd.kind == NK_VAR) return "v" + std::to_string(nd.val);
    return "n" + std::to_string(n);
  }
  std::string operand(uint32_t n) const {
    const Node& nd = d.nodes[n];
    return (nd.kind == NK_CONST ? "\"n\"(" : "\"r\"(") + name(n) + ")";
  }
  std::string value(Lit l) const {
    const Node& nd = d.nodes[lit_node(l)];
    if (nd.kind == NK_CONST) return hex32(lit_neg(l) ? ~nd.val : nd.val);
    return lit_neg(l) ? "(~" + name(lit_node(l)) + ")" : name(lit_node(l));
  }
  // IMAD operand registers: (u, k, c) -> u * k + c, computed once at u's level
  std::map<uint32_t, std::set<std::pair<int, int>>> derived;
  uint64_t cells_emitted = 0;

  static void mc(uint8_t f, int* m, int* c) {  // unary f(x) = x * m + c
    switch (f) {
      case 0: *m = 0; *c = 0; break;    // 0
      case 1: *m = 0; *c = -1; break;   // ~0
      case 2: *m = 1; *c = 0; break;    // x
      default: *m = -1; *c = -1; break; // ~x
    }
  }
  static std::string dname(uint32_t u, int k, int c) {
    auto enc = [](int v) { return v < 0 ? "m" + std::to_string(-v) : std::to_string(v); };
    return "d" + std::to_string(u) + "_" + enc(k) + "_" + enc(c);
  }
  static std::string imm(int v) {
    char b[16];
    snprintf(b, sizeof b, "0x%08xu", (uint32_t)v);
    return b;
  }
  // operand of an affine function of u: k*u + c
  std::string affine(uint32_t u, int k, int c, bool record) {
    if (k == 0) return "\"n\"(" + imm(c) + ")";
    if (k == 1 && c == 0) return "\"r\"(" + name(u) + ")";
    if (record) derived[u].insert({k, c});
    return "\"r\"(" + dname(u, k, c) + ")";
  }
  // register the operand registers an IMAD cell needs (before emission)
  void plan_cell(const Lut& L) {
    if (L.kind != 1) return;
    int m0, c0, m1, c1;
    mc(L.f0, &m0, &c0);
    mc(L.f1, &m1, &c1);
    if (d.nodes[L.in[0]].kind == NK_CONST) return;
    affine(L.in[1], m0 - m1, m0, true);
    affine(L.in[1], c0 - c1, c0, true);
  }
  void emit_derived(uint32_t u, const char* indent) {
    auto it = derived.find(u);
    if (it == derived.end()) return;
    for (auto& kc : it->second)
      os << indent << "const u32 " << dname(u, kc.first, kc.second) << " = " << name(u) << " * " << imm(kc.first)
         << " + " << imm(kc.second) << ";\n";
  }
  void lut(const Lut& L, const char* indent) {
    cells_emitted++;
    if (L.kind == 1) {
      // u ? f1(x) : f0(x) = x * M + C with M = m0 + (m0 - m1) u, C = c0 + (c0 - c1) u
      // (u is 0 or ~0 = -1 in every word)
      int m0, c0, m1, c1;
      mc(L.f0, &m0, &c0);
      mc(L.f1, &m1, &c1);
      const Node& xn = d.nodes[L.in[0]];
      if (xn.kind == NK_CONST) {  // constant x: K0 + (K0 - K1) u
        uint32_t K = xn.val;
        uint32_t K0 = (uint32_t)((int)K * m0 + c0), K1 = (uint32_t)((int)K * m1 + c1);
        os << indent << "u32 " << name(L.root) << "; asm(\"mad.lo.u32 %0, %1, %2, %3;\" : \"=r\"(" << name(L.root)
           << ") : \"r\"(" << name(L.in[1]) << "), \"n\"(" << imm((int)(K0 - K1)) << "), \"n\"(" << imm((int)K0)
           << "));\n";
      } else {
        os << indent << "u32 " << name(L.root) << "; asm(\"mad.lo.u32 %0, %1, %2, %3;\" : \"=r\"(" << name(L.root)
           << ") : \"r\"(" << name(L.in[0]) << "), " << affine(L.in[1], m0 - m1, m0, false) << ", "
           << affine(L.in[1], c0 - c1, c0, false) << ");\n";
      }
    } else if (L.kind == 2) {  // x * K + C (K, C hoisted; a constant x goes in the immediate slot)
      const bool xc = d.nodes[L.in[0]].kind == NK_CONST;
      os << indent << "u32 " << name(L.root) << "; asm(\"mad.lo.u32 %0, %1, %2, %3;\" : \"=r\"(" << name(L.root)
         << ") : " << operand(xc ? L.in[1] : L.in[0]) << ", " << operand(xc ? L.in[0] : L.in[1]) << ", "
         << operand(L.in[2]) << ");\n";
    } else {
      char immb[8];
      snprintf(immb, sizeof immb, "0x%02x", L.imm);
      os << indent << "u32 " << name(L.root) << "; asm(\"lop3.b32 %0, %1, %2, %3, " << immb
         << ";\" : \"=r\"(" << name(L.root) << ") : " << operand(L.in[0]) << ", " << operand(L.in[1])
         << ", " << operand(L.in[2]) << ");\n";
    }
    emit_derived(L.root, indent);
  }
};

}  // namespace

const char* kPrelude =
    "typedef unsigned int u32;\n"
    "typedef unsigned long long u64;\n"
    "struct __align__(16) u32x4 { u32 x, y, z, w; };\n"
    "struct __align__(8) u32x2 { u32 x, y; };\n"
    "// per-warp sum, one atomic per warp (device bodies: no block barrier, no static shared memory)\n"
    "static __device__ __forceinline__ void bfa_warp_sum(u64 acc, u64* count) {\n"
    "  #pragma unroll\n"
    "  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);\n"
    "  if ((threadIdx.x & 31u) == 0 && acc) atomicAdd(count, acc);\n"
    "}\n"
    "static __device__ __forceinline__ void bfa_block_sum(u64 acc, u64* count) {\n"
    "  #pragma unroll\n"
    "  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);\n"
    "  __shared__ u64 red[32];\n"
    "  const u32 tid = threadIdx.x;\n"
    "  if ((tid & 31u) == 0) red[tid >> 5] = acc;\n"
    "  __syncthreads();\n"
    "  if (tid < 32u) {\n"
    "    u64 v = tid < (blockDim.x >> 5) ? red[tid] : 0ull;\n"
    "    #pragma unroll\n"
    "    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);\n"
    "    if (tid == 0 && v) atomicAdd(count, v);\n"
    "  }\n"
    "}\n";


// The specialised DAG of one kernel variant: the 2^s slot cofactors of f
// with lane words as constants, and the loop level of every variable from
// its bit position in the word index (spec.perm maps variable -> position;
// empty = identity).
struct Built {
  Dag D;
  std::vector<Lit> outs;
  std::vector<uint8_t> var_level;
  std::vector<int> pos;
  double w[4];
  int S = 1, s = 0, t = 8, m = 0;
};

static void build_specialised(const Parsed& prog, const KernelSpec& spec, Built* b) {
  b->S = spec.generic ? 1 : (1 << spec.slot_bits);
  b->s = spec.generic ? 0 : spec.slot_bits;
  b->t = spec.thread_bits;
  b->m = spec.inner_bits;
  const int s = b->s, t = b->t, m = b->m;
  b->pos.resize(64);
  for (int v = 0; v < 64; v++) b->pos[v] = (v < (int)spec.perm.size()) ? spec.perm[v] : v;
  if (spec.mode == KM_EVAL && !spec.generic && spec.vec_bits >= 0 && spec.vec_bits < s) {
    // eval store layout: word-index bit w of variable 5 + w holds slot bit w
    // (w < a), thread bit w - a (a <= w < a + t), slot bit w - t (a + t <= w
    // < s + t); every higher bit keeps its position
    const int a = spec.vec_bits;
    for (int w = 0; w < s + t && 5 + w < 64; w++)
      b->pos[5 + w] = 5 + (w < a ? w : w < a + t ? s + (w - a) : w - t);
  }
  // roles of word-index bit p = pos(v) - 5:
  //   generic:     every v >= 5 is level 3, read from w
  //   specialised: p < s slot (constant per slot), < s+t thread (1),
  //                < s+t+m inner (3), else outer (2)
  auto level_of = [&](int v) -> int {
    if (spec.materialised) return 3;
    const int q = b->pos[v];
    if (q < 5) return 0;
    int p = q - 5;
    if (spec.generic) return 3;
    if (p < s) return 0;
    if (p < s + t) return 1;
    if (p < s + t + m) return 3;
    return 2;
  };
  std::vector<uint8_t> done(prog.dag.nodes.size());
  std::vector<Lit> memo(prog.dag.nodes.size());
  for (int slot = 0; slot < b->S; slot++) {
    std::vector<Lit> subst(64, 0);
    for (int v = 0; v < 64; v++) {
      const int q = b->pos[v];
      if (q < 5 && !spec.materialised) subst[v] = b->D.word(kLane[q]);
      else if (!spec.generic && !spec.materialised && q - 5 < s)
        subst[v] = ((slot >> (q - 5)) & 1) ? b->D.const1() : b->D.const0();
      else subst[v] = b->D.var((uint32_t)v);
    }
    std::fill(done.begin(), done.end(), 0);
    b->outs.push_back(rebuild(prog.dag, prog.root, subst, b->D, memo, done));
  }
  b->var_level.assign(64, 0);
  for (int v = 0; v < 64; v++) b->var_level[v] = (uint8_t)level_of(v);
  const double iters_inner = (double)(1u << m);
  b->w[0] = 0.0;
  b->w[1] = 1e-4;
  b->w[2] = spec.generic ? 1.0 : 1.0 / iters_inner;
  b->w[3] = 1.0;
}

// Modelled time per thread-iteration of a cover, max(2 A, 2 F, A + F + other):
// the ALU pipe takes a LOP3 and the FMA pipe an IMAD warp-instruction every 2
// cycles per SMSP, and the scheduler issues one per cycle (bfa_peak_int
// measures 18.5 T LOP3/s, 18.5 T IMAD/s and 35.2 T/s for a 1:1 mix).
static double model_time(const Built& b, const MapResult& r, const KernelSpec& spec) {
  double A = 0, F = 0;
  // IMAD operand registers u * k + c, one per distinct (u, k, c) (as
  // Emitter::plan_cell records them), computed at u's loop level
  std::vector<uint64_t> derived;
  auto note = [&](uint32_t u, int k, int c) {
    if (k == 0 || (k == 1 && c == 0)) return;
    derived.push_back((uint64_t)u << 16 | (uint64_t)(k + 8) << 8 | (uint64_t)(c + 8));
  };
  for (const Lut& L : r.luts) {
    if (L.kind == 0) { A += b.w[L.level]; continue; }
    if (L.kind == 2) { F += b.w[L.level]; continue; }
    F += b.w[L.level];
    if (b.D.nodes[L.in[0]].kind == NK_CONST) continue;
    int m0, c0, m1, c1;
    Emitter::mc(L.f0, &m0, &c0);
    Emitter::mc(L.f1, &m1, &c1);
    note(L.in[1], m0 - m1, m0);
    note(L.in[1], c0 - c1, c0);
  }
  std::sort(derived.begin(), derived.end());
  derived.erase(std::unique(derived.begin(), derived.end()), derived.end());
  for (size_t i = 0; i < derived.size();) {   // per u: w(level of u) x its distinct (k, c)
    size_t j = i;
    while (j < derived.size() && (derived[j] >> 16) == (derived[i] >> 16)) j++;
    F += b.w[r.node_level[(uint32_t)(derived[i] >> 16)]] * (double)(j - i);
    i = j;
  }
  const double other = spec.generic ? 4.0 : b.S + b.S / 2.0 + 2.0 + 2.0 * b.m;
  double t = std::max({2 * (A + other), 2 * F, A + F + other});
  // register pressure: every thread- / outer-level value an inner cell reads
  // (and every derived IMAD operand of one) stays live across the inner
  // loop; past the register file the kernel spills (C5 at slot 7: 255
  // registers + 150-400 B of spill stores, 1.6x slower with 227 live-in
  // values; slot 5, 177 live-in values: no spill).  Each live value beyond
  // the budget costs 1 % of the iteration.
  if (!spec.generic && b.m > 0) {
    std::vector<uint64_t> live;   // hoisted nodes, and hoisted IMAD operand registers (u, k, c)
    for (const Lut& L : r.luts) {
      if (L.level != 3) continue;
      if (L.kind == 1 && b.D.nodes[L.in[0]].kind != NK_CONST) {
        const uint32_t u = L.in[1];
        if (r.node_level[u] < 3) {
          int m0, c0, m1, c1;
          Emitter::mc(L.f0, &m0, &c0);
          Emitter::mc(L.f1, &m1, &c1);
          for (auto kc : {std::make_pair(m0 - m1, m0), std::make_pair(c0 - c1, c0)})
            if (kc.first != 0 && !(kc.first == 1 && kc.second == 0))
              live.push_back(1ull << 63 | (uint64_t)u << 16 | (uint64_t)(kc.first + 8) << 8 | (uint64_t)(kc.second + 8));
            else if (kc.first == 1)
              live.push_back(u);
        }
        if (r.node_level[L.in[0]] < 3) live.push_back(L.in[0]);
        continue;
      }
      for (int q = 0; q < L.nin; q++) {
        const uint32_t x = L.in[q];
        if (b.D.nodes[x].kind != NK_CONST && r.node_level[x] < 3) live.push_back(x);
      }
    }
    std::sort(live.begin(), live.end());
    live.erase(std::unique(live.begin(), live.end()), live.end());
    const double budget = 180.0;  // of 255, leaving ~75 for the inner loop's own temporaries
    const double excess = (double)live.size() - budget;
    if (excess > 0) t *= 1.0 + 0.01 * excess;
  }
  return t;
}

// Technology mapping.  With dual_pipe, gates that have a word-uniform input
// may become IMAD cells (FMA pipe) instead of being absorbed into LOP3 cells
// (ALU pipe); sweep the IMAD:LOP3 cost ratio (or use the fixed one) and keep
// the cover with the least modelled time.
// Kind-2 IMAD cells (KernelSpec::imad_pairs).  An inner-loop LOP3 cell
// g(x, u1, u2) whose leaves u1, u2 are word-uniform (0 or ~0 in every word)
// and hoisted (thread / outer level) is, for each value of (u1, u2), one of
// the unary functions 0, ~0, x, ~x of x, i.e. x * K + C with K in {0, 1, -1}
// and C in {0, -1} functions of (u1, u2): one IMAD on the FMA pipe in the
// inner loop.  K = lop3(u1, u2, 0xFFFFFFFE) (bit 0: K != 0; bits 1..31:
// K == -1) and C = lop3(u1, u2) are cells at the hoisted level, shared
// between cells.  Cells are converted while the modelled ALU work exceeds
// the FMA work (model_time's pipe balance); the new nodes are appended to
// b.D outside the hash-consing tables.
static void imad_pairs(Built& b, MapResult& r) {
  Dag& D = b.D;
  const size_t N0 = D.nodes.size();
  std::vector<uint8_t> uniform(N0, 0);
  for (size_t n = 0; n < N0; n++) {
    const Node& nd = D.nodes[n];
    if (nd.kind == NK_VAR) uniform[n] = 1;
    else if (nd.kind == NK_CONST) uniform[n] = n == 0;
    else uniform[n] = uniform[nd.a] && uniform[nd.b];
  }
  double A = 0, F = 0;
  for (const Lut& L : r.luts) (L.kind == 0 ? A : F) += b.w[L.level];
  const double other = b.S + b.S / 2.0 + 2.0 + 2.0 * b.m;
  auto new_node = [&](NodeKind k, uint32_t a, uint32_t c, uint32_t val, uint8_t level) {
    D.nodes.push_back(Node{k, 0, a, c, val});
    r.node_level.push_back(level);
    return (uint32_t)(D.nodes.size() - 1);
  };
  std::map<std::tuple<uint32_t, uint32_t, int, int>, uint32_t> made;  // (u1, u2, K/C, tt) -> node
  uint32_t not_one = UINT32_MAX;
  std::vector<Lut> added;
  for (Lut& L : r.luts) {
    if (F + 2.0 > A + other) break;  // pipes balanced
    if (L.kind != 0 || L.level != 3 || L.nin != 3) continue;
    int ix = -1, nu = 0;
    for (int q = 0; q < 3; q++)
      if (!uniform[L.in[q]]) { ix = q; nu++; }
    if (nu != 1) continue;
    int iu[2], k = 0;
    for (int q = 0; q < 3; q++)
      if (q != ix) iu[k++] = q;
    const uint32_t u1 = L.in[iu[0]], u2 = L.in[iu[1]], x = L.in[ix];
    if (u1 == u2 || D.nodes[u1].kind == NK_CONST || D.nodes[u2].kind == NK_CONST) continue;
    const uint8_t lv = std::max(r.node_level[u1], r.node_level[u2]);
    if (lv >= 3) continue;
    int m[4], c[4];
    for (int pq = 0; pq < 4; pq++) {
      int v[2];
      for (int xv = 0; xv < 2; xv++) {
        int bits[3];
        bits[ix] = xv;
        bits[iu[0]] = pq & 1;
        bits[iu[1]] = pq >> 1;
        v[xv] = (L.imm >> (bits[0] * 4 + bits[1] * 2 + bits[2])) & 1;
      }
      Emitter::mc(unary_code(v[0], v[1]), &m[pq], &c[pq]);
    }
    const bool kconst = m[0] == m[1] && m[0] == m[2] && m[0] == m[3];
    const bool cconst = c[0] == c[1] && c[0] == c[2] && c[0] == c[3];
    const bool xconst = D.nodes[x].kind == NK_CONST;
    if (kconst && (m[0] == 0 || xconst)) continue;
    double dA = 0;
    uint32_t kn, cn;
    if (kconst) {
      kn = new_node(NK_CONST, 0, 0, (uint32_t)m[0], 0);
    } else {
      int tt = 0;
      for (int a = 0; a < 2; a++)
        for (int bb = 0; bb < 2; bb++)
          for (int cb = 0; cb < 2; cb++) {
            const int pq = a | bb << 1;
            if (cb == 0 ? m[pq] != 0 : m[pq] == -1) tt |= 1 << (a * 4 + bb * 2 + cb);
          }
      auto it = made.find({u1, u2, 0, tt});
      if (it != made.end()) {
        kn = it->second;
      } else {
        if (not_one == UINT32_MAX) not_one = new_node(NK_CONST, 0, 0, 0xFFFFFFFEu, 0);
        kn = new_node(NK_GATE, u1, u2, 0, lv);
        Lut K{};
        K.root = kn; K.nin = 3; K.in[0] = u1; K.in[1] = u2; K.in[2] = not_one; K.imm = (uint8_t)tt; K.level = lv;
        added.push_back(K);
        made[{u1, u2, 0, tt}] = kn;
        dA += b.w[lv];
      }
    }
    if (cconst) {
      cn = c[0] == 0 ? 0u : new_node(NK_CONST, 0, 0, 0xFFFFFFFFu, 0);
    } else {
      int tt = 0;
      for (int a = 0; a < 2; a++)
        for (int bb = 0; bb < 2; bb++)
          if (c[a | bb << 1] == -1) tt |= 1 << (a * 4 + bb * 2) | 1 << (a * 4 + bb * 2 + 1);
      auto it = made.find({u1, u2, 1, tt});
      if (it != made.end()) {
        cn = it->second;
      } else {
        cn = new_node(NK_GATE, u1, u2, 0, lv);
        Lut C{};
        C.root = cn; C.nin = 2; C.in[0] = u1; C.in[1] = u2; C.in[2] = u1; C.imm = (uint8_t)tt; C.level = lv;
        added.push_back(C);
        made[{u1, u2, 1, tt}] = cn;
        dA += b.w[lv];
      }
    }
    L.kind = 2;
    L.nin = 3;
    L.in[0] = x;
    L.in[1] = kn;
    L.in[2] = cn;
    A += dA - 1.0;
    F += 1.0;
  }
  for (const Lut& L : added) r.luts.push_back(L);
}

static MapResult choose_mapping(Built& b, const KernelSpec& spec, double* best_time, double* chosen) {
  MapResult mr;
  double best = 1e300, cost = 0.0;
  std::vector<double> sweep = {0.0};
  if (spec.dual_pipe && !spec.materialised) {
    if (spec.imad_cost_pct > 0) sweep = {spec.imad_cost_pct / 100.0};
    else sweep = {0.0, 0.6, 0.75, 0.9, 1.0, 1.15, 1.3, 1.6, 2.0, 3.0};
  }
  const bool pairs = spec.imad_pairs && spec.dual_pipe && spec.mode == KM_COUNT && !spec.generic && !spec.materialised;
  for (double c : sweep) {
    MapResult r = map_luts(b.D, b.outs, b.var_level, b.w, c, spec.area_passes);
    if (pairs) imad_pairs(b, r);
    double tm = model_time(b, r, spec);
    if (tm < best - 1e-9) { best = tm; mr = std::move(r); cost = c; }
  }
  if (best_time) *best_time = best;
  if (chosen) *chosen = cost;
  return mr;
}

// Emission order: depth-first post-order from the outputs (slot by slot), so
// a subtree is finished before the next starts and live ranges stay short;
// node-id order would keep e.g. every shared subterm of a big tree alive.
static void dfs_order(MapResult* mr, const std::vector<Lit>& outs) {
  std::unordered_map<uint32_t, size_t> at;
  for (size_t k = 0; k < mr->luts.size(); k++) at[mr->luts[k].root] = k;
  std::vector<uint8_t> done(mr->luts.size(), 0);
  std::vector<Lut> order;
  order.reserve(mr->luts.size());
  for (Lit o : outs) {
    auto r = at.find(lit_node(o));
    if (r == at.end()) continue;
    std::vector<std::pair<size_t, int>> st{{r->second, 0}};
    while (!st.empty()) {
      size_t k = st.back().first;
      int q = st.back().second;
      if (done[k]) { st.pop_back(); continue; }
      const Lut& L = mr->luts[k];
      const int nin = L.kind == 1 ? 2 : L.nin;
      if (q < nin) {
        st.back().second++;
        auto it = at.find(L.in[q]);
        if (it != at.end() && !done[it->second]) st.push_back({it->second, 0});
        continue;
      }
      done[k] = 1;
      order.push_back(L);
      st.pop_back();
    }
  }
  mr->luts.swap(order);
}

double model_cost(const Parsed& prog, const KernelSpec& spec) {
  KernelSpec sp = spec;
  sp.area_passes = 0;  // the search compares area-flow covers; emission refines the winner
  Built b;
  build_specialised(prog, sp, &b);
  double t = 0;
  choose_mapping(b, sp, &t, nullptr);
  return t;
}

// Constructive start of the role search: slot positions to the variables
// whose joint cofactors reduce the program most; the others ranked by forward
// cone size (gates that depend on the variable), largest first, to the lane,
// thread and outer positions; the smallest cones (variables outside the
// support first) take the inner-loop positions, so most cells hoist out of
// the inner loop.
static std::vector<int8_t> constructive_roles(const Parsed& prog, const KernelSpec& spec, int k_free, int threads) {
  const int s = spec.slot_bits, t = spec.thread_bits, m = spec.inner_bits;
  std::vector<int8_t> pm(64);
  for (int v = 0; v < 64; v++) pm[v] = (int8_t)v;
  std::vector<int> slot = choose_cofactor_vars(prog, k_free, std::max(0, std::min(s, k_free - 5)), nullptr, threads);
  const Dag& d = prog.dag;
  std::vector<uint64_t> sup(d.nodes.size(), 0);
  std::vector<uint8_t> in_cone(d.nodes.size(), 0);
  std::vector<uint32_t> st{lit_node(prog.root)};
  while (!st.empty()) {
    const uint32_t k = st.back();
    st.pop_back();
    if (in_cone[k]) continue;
    in_cone[k] = 1;
    if (d.nodes[k].kind == NK_GATE) { st.push_back(d.nodes[k].a); st.push_back(d.nodes[k].b); }
  }
  std::vector<uint32_t> cone(64, 0);
  for (size_t k = 0; k < d.nodes.size(); k++) {
    const Node& nd = d.nodes[k];
    if (nd.kind == NK_VAR) {
      sup[k] = 1ull << nd.val;
    } else if (nd.kind == NK_GATE) {
      sup[k] = sup[nd.a] | sup[nd.b];
      if (in_cone[k])
        for (uint64_t b = sup[k]; b; b &= b - 1) cone[__builtin_ctzll(b)]++;
    }
  }
  std::vector<int> rest;
  for (int v = 0; v < k_free; v++)
    if (std::find(slot.begin(), slot.end(), v) == slot.end()) rest.push_back(v);
  std::stable_sort(rest.begin(), rest.end(), [&](int x, int y) { return cone[x] > cone[y]; });
  std::vector<int> pos_order;  // positions in the order the ranked variables take them
  for (int q = 0; q < std::min(5, k_free); q++) pos_order.push_back(q);                     // lanes
  for (int q = 5 + s; q < std::min(k_free, 5 + s + t); q++) pos_order.push_back(q);         // thread
  for (int q = k_free - 1; q >= 5 + s + t + m; q--) pos_order.push_back(q);                 // outer
  for (int q = 5 + s + t; q < std::min(k_free, 5 + s + t + m); q++) pos_order.push_back(q); // inner
  std::vector<uint8_t> taken(64, 0);
  for (size_t i = 0; i < slot.size(); i++) { pm[slot[i]] = (int8_t)(5 + i); taken[5 + i] = 1; }
  size_t r = 0;
  for (int q : pos_order)
    if (!taken[q] && r < rest.size()) { pm[rest[r++]] = (int8_t)q; taken[q] = 1; }
  for (int q = 0; q < k_free && r < rest.size(); q++)  // fewer slot variables than slots
    if (!taken[q]) { pm[rest[r++]] = (int8_t)q; taken[q] = 1; }
  return pm;
}

std::vector<int8_t> search_roles(const Parsed& prog, const KernelSpec& base, int k_free, int budget, uint64_t seed,
                                 int threads) {
  // annealing temperature (fraction of the best cost) at the start of the
  // climb: C5 at slot 7, 4 seeds x 400 evaluations: mean model cost 4912
  // without, 4734 with 0.005-0.01
  const double anneal = 0.005;
  // Count mode over an aligned sub-cube of 2^k_free valuations: any
  // permutation of the variables below k_free is a bijection of the sub-cube,
  // so the count is unchanged; search the one whose cover is cheapest.
  //
  // The search is a fixed sequence of candidates drawn from one seeded
  // generator: the constructive start, random restarts, then swap hill
  // climbing between role classes (sideways moves accepted).  With
  // threads > 1 the model evaluations of consecutive candidates run
  // speculatively in parallel and are committed in sequence order, so the
  // result is the same for every thread count (and on every machine).
  k_free = std::min(k_free, 63);
  std::vector<int8_t> perm(64);
  for (int v = 0; v < 64; v++) perm[v] = (int8_t)v;
  if (k_free <= 5 || base.generic || base.materialised || base.mode != KM_COUNT) return {};
  const int s = base.slot_bits, t = base.thread_bits, m = base.inner_bits;
  // role classes for the swap moves: lane and thread positions are one class
  // (both put a cell's cost outside the loops); slot, inner and outer others
  auto role = [&](int q) { return q < 5 ? 2 : q - 5 < s ? 1 : q - 5 < s + t ? 2 : q - 5 < s + t + m ? 3 : 4; };
  auto eval = [&](const std::vector<int8_t>& pm) {
    KernelSpec spec = base;
    spec.perm = pm;
    return model_cost(prog, spec);
  };
  uint64_t rs = seed * 6364136223846793005ull + 1442695040888963407ull;
  auto rnd = [&](uint64_t n) { rs = rs * 6364136223846793005ull + 1442695040888963407ull; return (rs >> 33) % n; };
  threads = std::max(1, std::min(threads, 64));
  // evaluate a batch of candidates (in parallel when threads > 1)
  auto eval_batch = [&](const std::vector<std::vector<int8_t>>& cand, std::vector<double>* cost) {
    cost->assign(cand.size(), 0.0);
    if (threads == 1 || cand.size() == 1) {
      for (size_t i = 0; i < cand.size(); i++) (*cost)[i] = eval(cand[i]);
      return;
    }
    std::atomic<size_t> next{0};
    std::vector<std::thread> th;
    const size_t W = std::min<size_t>(cand.size(), (size_t)threads);
    for (size_t w = 0; w < W; w++)
      th.emplace_back([&] {
        for (size_t i; (i = next.fetch_add(1)) < cand.size();) (*cost)[i] = eval(cand[i]);
      });
    for (auto& x : th) x.join();
  };
  // the identity, the constructive start and random restarts (independent draws)
  std::vector<int8_t> best = perm;
  double best_c = 1e300;
  int evals = 0;
  {
    std::vector<std::vector<int8_t>> cand{perm, constructive_roles(prog, base, k_free, threads)};
    const int R = std::max(0, std::min(budget / 16, budget - 2));
    for (int r = 0; r < R; r++) {
      std::vector<int8_t> pm = perm;
      for (int i = k_free - 1; i > 0; i--) std::swap(pm[i], pm[rnd((uint64_t)i + 1)]);
      cand.push_back(std::move(pm));
    }
    std::vector<double> cost;
    eval_batch(cand, &cost);
    for (size_t r = 0; r < cand.size(); r++) {
      evals++;
      if (cost[r] < best_c) { best_c = cost[r]; best = cand[r]; }
    }
  }
  // hill climbing in rounds of kRound swap candidates (two variables of
  // different role classes) drawn from the current point and evaluated
  // together (in parallel when threads > 1): move to the best strictly
  // improving one, else to the first equal-cost one (sideways moves cross
  // plateaus).  The round size is fixed, so the result does not depend on
  // the thread count.
  constexpr int kRound = 8;
  std::vector<int8_t> cur = best;
  double cur_c = best_c;
  int stall = 0;
  while (evals < budget && stall < 100000) {
    std::vector<std::vector<int8_t>> cand;
    const int B = std::min(kRound, budget - evals);
    while ((int)cand.size() < B && stall < 100000) {
      int a = (int)rnd((uint64_t)k_free), c = (int)rnd((uint64_t)k_free);
      if (role(cur[a]) == role(cur[c])) { stall++; continue; }
      stall = 0;
      std::vector<int8_t> pm = cur;
      std::swap(pm[a], pm[c]);
      cand.push_back(std::move(pm));
    }
    if (cand.empty()) break;
    std::vector<double> cost;
    eval_batch(cand, &cost);
    evals += (int)cand.size();
    int pick = -1;
    for (size_t i = 0; i < cand.size(); i++)
      if (cost[i] < cur_c && (pick < 0 || cost[i] < cost[pick])) pick = (int)i;
    if (pick < 0)
      for (size_t i = 0; i < cand.size() && pick < 0; i++)
        if (cost[i] == cur_c) pick = (int)i;
    if (pick < 0 && anneal > 0) {
      // annealing: accept the least-worse candidate with probability
      // exp(-delta / T), T falling linearly to 0 over the budget
      size_t lw = 0;
      for (size_t i = 1; i < cand.size(); i++)
        if (cost[i] < cost[lw]) lw = i;
      const double T = anneal * best_c * (1.0 - (double)evals / budget);
      const double u = (double)rnd(1u << 30) / (double)(1u << 30);
      if (T > 0 && u < std::exp(-(cost[lw] - cur_c) / T)) pick = (int)lw;
    }
    if (pick >= 0) {
      cur = cand[pick];
      cur_c = cost[pick];
      if (cur_c < best_c) { best_c = cur_c; best = cur; }
    }
  }
  bool identity = true;
  for (int v = 0; v < 64; v++) identity &= best[v] == v;
  return identity ? std::vector<int8_t>{} : best;
}

std::string emit_kernel(const Parsed& prog, const KernelSpec& spec, KernelStats* stats) {
  KernelStats st;
  std::ostringstream os;
  os << "// generated by libbfa: " << (spec.mode == KM_COUNT ? "count" : "eval")
     << (spec.generic ? " generic" : " specialised") << " s=" << spec.slot_bits << " t=" << spec.thread_bits
     << " m=" << spec.inner_bits << (spec.perm.empty() ? "" : " (permuted roles)") << "\n";
  const bool as_body = !spec.body_name.empty() && !spec.generic;
  if (!as_body) os << kPrelude;
  Built b;
  build_specialised(prog, spec, &b);
  Dag& D = b.D;
  const std::vector<Lit>& outs = b.outs;
  const int S = b.S, s = b.s, t = b.t, m = b.m;
  const bool want_count = spec.mode == KM_COUNT || spec.fuse_count;
  auto level_of = [&](int v) { return (int)b.var_level[v]; };
  auto pos = [&](int v) { return b.pos[v]; };
  double best_t = 0;
  MapResult mr = choose_mapping(b, spec, &best_t, &st.imad_cost);
  dfs_order(&mr, outs);

  // which variables are referenced (as cell inputs or outputs)
  std::vector<uint8_t> used(64, 0);
  std::vector<uint32_t> var_node(64, 0);
  for (size_t k = 0; k < D.nodes.size(); k++)
    if (D.nodes[k].kind == NK_VAR) var_node[D.nodes[k].val] = (uint32_t)k;
  auto mark = [&](uint32_t n) { if (D.nodes[n].kind == NK_VAR) used[D.nodes[n].val] = 1; };
  for (const Lut& L : mr.luts) for (int q = 0; q < 3; q++) mark(L.in[q]);
  for (Lit o : outs) mark(lit_node(o));

  const std::string bounds = std::to_string(1 << t) + (spec.min_blocks > 0 ? ", " + std::to_string(spec.min_blocks) : "");
  Emitter E(D, os);
  for (const Lut& L : mr.luts) E.plan_cell(L);
  for (auto& kv : E.derived) {
    int lv = mr.node_level[kv.first];
    if (lv == 3) st.derived_inner += (uint32_t)kv.second.size();
    if (lv == 2) st.derived_outer += (uint32_t)kv.second.size();
  }
  auto emit_level = [&](int lvl, const char* ind) {
    for (const Lut& L : mr.luts) {
      if (L.level != lvl) continue;
      E.lut(L, ind);
      uint32_t* luts = lvl == 1 ? &st.luts_thread : lvl == 2 ? &st.luts_outer : &st.luts_inner;
      uint32_t* imads = lvl == 1 ? &st.imads_thread : lvl == 2 ? &st.imads_outer : &st.imads_inner;
      (*(L.kind != 0 ? imads : luts))++;
    }
  };
  auto declare_var = [&](int v, const std::string& expr, const char* ind) {
    os << ind << "const u32 v" << v << " = " << expr << ";\n";
    E.emit_derived(var_node[v], ind);
  };

  if (spec.generic && spec.materialised) {
    // the paper's table S in HBM: 128-bit loads of every
    // generator row the program uses, the LOP3 body in registers, 128-bit store
    os << "__device__ __forceinline__ u32 comp(const uint4& v, int c) { return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w; }\n"
       << "extern \"C\" __global__ void __launch_bounds__(" << bounds << ")\n"
       << "bfa_kernel(const u32* __restrict__ table, const u64 row_words, const u64 groups, u32* __restrict__ out, u64* __restrict__ count) {\n"
       << "  u64 acc = 0;\n"
       << "  const u64 stride = (u64)gridDim.x * blockDim.x;\n"
       << "  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < groups; k += stride) {\n";
    for (int v = 0; v < 64; v++)
      if (used[v])
        os << "    const uint4 V" << v << " = __ldcs(reinterpret_cast<const uint4*>(table + " << v
           << "ull * row_words) + k);\n";
    os << "    u32 R[4];\n"
       << "    #pragma unroll\n"
       << "    for (int c = 0; c < 4; ++c) {\n";
    for (int v = 0; v < 64; v++)
      if (used[v]) declare_var(v, "comp(V" + std::to_string(v) + ", c)", "      ");
    emit_level(3, "      ");
    os << "      R[c] = " << E.value(outs[0]) << ";\n"
       << "    }\n";
    if (spec.mode == KM_EVAL)
      os << "    __stcs(reinterpret_cast<uint4*>(out) + k, make_uint4(R[0], R[1], R[2], R[3]));\n";
    if (want_count) os << "    acc += __popc(R[0]) + __popc(R[1]) + __popc(R[2]) + __popc(R[3]);\n";
    os << "  }\n";
    if (want_count) os << "  bfa_block_sum(acc, count);\n";
    os << "}\n";
    st.words_per_iter = 4;
    for (int v = 0; v < 64; v++) st.inner_vars += used[v];
  } else if (spec.generic) {
    os << "extern \"C\" __global__ void __launch_bounds__(" << bounds << ")\n"
       << "bfa_kernel(const u64 w_begin, const u64 w_count, const u32 mask, u32* __restrict__ out, u64* __restrict__ count"
       << ") {\n"
       << "  u64 acc = 0;\n"
       << "  const u64 stride = (u64)gridDim.x * blockDim.x;\n"
       << "  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < w_count; k += stride) {\n"
       << "    const u64 w = w_begin + k;\n";
    for (int v = 0; v < 64; v++)
      if (used[v]) declare_var(v, "0u - (u32)((w >> " + std::to_string(pos(v) - 5) + ") & 1ull)", "    ");
    emit_level(3, "    ");
    os << "    const u32 r = (" << E.value(outs[0]) << ") & mask;\n";
    if (spec.mode == KM_EVAL) os << "    out[k] = r;\n";
    if (want_count) os << "    acc += __popc(r);\n";
    os << "  }\n";
    if (want_count) os << "  bfa_block_sum(acc, count);\n";
    os << "}\n";
    st.words_per_iter = 1;
    for (int v = 0; v < 64; v++) st.inner_vars += used[v];
  } else {
    const int unit = s + t + m;
    if (as_body)
      os << "extern \"C\" __device__ __noinline__ void " << spec.body_name
         << "(const u64 A, const u64 o_count, const u64 out_base_w, u32* __restrict__ out, u64* __restrict__ count"
         << ", const u32 bid_, const u32 nb_) {\n";
    else
      os << "extern \"C\" __global__ void __launch_bounds__(" << bounds << ")\n"
         << "bfa_kernel(const u64 A, const u64 o_count, const u64 out_base_w, u32* __restrict__ out, u64* __restrict__ count"
         << ") {\n";
    os << "  const u32 tid = threadIdx.x;\n"
       << (as_body ? "  const u64 q = o_count / nb_, rr = o_count % nb_, b = bid_;\n"
                   : "  const u64 q = o_count / gridDim.x, rr = o_count % gridDim.x, b = blockIdx.x;\n")
       << "  const u64 o_begin = b * q + (b < rr ? b : rr);\n"
       << "  const u64 o_end = o_begin + q + (b < rr ? 1ull : 0ull);\n";
    for (int v = 0; v < 64; v++)
      if (used[v] && level_of(v) == 1) {
        declare_var(v, "0u - ((tid >> " + std::to_string(pos(v) - 5 - s) + ") & 1u)", "  ");
        st.thread_vars++;
      }
    emit_level(1, "  ");
    os << "  u64 acc = 0;\n"
       << "  for (u64 o = o_begin; o < o_end; ++o) {\n"
       << "    const u64 wo = A + (o << " << unit << ");\n";
    for (int v = 0; v < 64; v++)
      if (used[v] && level_of(v) == 2) {
        declare_var(v, "0u - (u32)((wo >> " + std::to_string(pos(v) - 5) + ") & 1ull)", "    ");
        st.outer_vars++;
      }
    emit_level(2, "    ");
    os << "    u32 acc32 = 0;\n"
       << "    #pragma unroll 1\n"
       << "    for (u32 i = 0; i < " << (1u << m) << "u; ++i) {\n";
    for (int v = 0; v < 64; v++)
      if (used[v] && level_of(v) == 3) {
        int k = pos(v) - 5 - s - t;
        declare_var(v, "(u32)(((int)(i << " + std::to_string(31 - k) + ")) >> 31)", "      ");
        st.inner_vars++;
      }
    emit_level(3, "      ");
    for (int sl = 0; sl < S; sl++) os << "      const u32 r" << sl << " = " << E.value(outs[sl]) << ";\n";
    if (spec.mode == KM_EVAL) {
      // slot sl -> word (sl & (2^a - 1)) + (tid << a) + ((sl >> a) << (a + t))
      // of the inner iteration's 2^(s+t) words (build_specialised's layout)
      const int a = (spec.vec_bits >= 0 && spec.vec_bits < s) ? spec.vec_bits : s;
      const int V = 1 << a;
      os << "      const u64 idx = (wo - out_base_w) + ((u64)i << " << (s + t) << ") + ((u64)tid << " << a << ");\n";
      for (int g = 0; g < S; g += V) {
        const uint64_t off = (uint64_t)(g >> a) << (a + t);
        if (V == 1) os << "      out[idx + " << off << "ull] = r" << g << ";\n";
        else if (V == 2)
          os << "      *reinterpret_cast<u32x2*>(out + idx + " << off << "ull) = u32x2{r" << g << ", r" << g + 1 << "};\n";
        else
          for (int h = 0; h < V; h += 4)
            os << "      *reinterpret_cast<u32x4*>(out + idx + " << off + h << "ull) = u32x4{r" << g + h << ", r"
               << g + h + 1 << ", r" << g + h + 2 << ", r" << g + h + 3 << "};\n";
      }
    }
    if (want_count) {
      os << "      acc32 += ";
      for (int sl = 0; sl < S; sl++) os << (sl ? " + " : "") << "__popc(r" << sl << ")";
      os << ";\n";
    }
    os << "    }\n"
       << "    acc += acc32;\n"
       << "  }\n";
    const std::string acc_expr = spec.count_shift ? "acc << " + std::to_string(spec.count_shift) : "acc";
    if (want_count)
      os << (as_body ? "  bfa_warp_sum(" : "  bfa_block_sum(") << acc_expr << ", count);\n";
    os << "}\n";
    st.words_per_iter = (uint32_t)S;
  }
  if (stats) *stats = st;
  return os.str();
}

// ============================================================== PTX emission
// The count-mode specialised kernel (and the work-queue bodies) emitted as
// PTX directly and compiled by the PTX compiler alone: the same cover, the
// same schedule and the same loop structure as emit_kernel's CUDA C++ (which
// NVRTC would first have to translate to this PTX), at half the JIT time.
namespace {

constexpr const char* kPtxHeader = ".version 8.8\n.target sm_100a\n.address_size 64\n";

std::string ptx_imm(uint32_t w) {
  char b[16];
  snprintf(b, sizeof b, "0x%08X", w);
  return b;
}

struct PtxEmitter {
  const Dag& d;
  std::ostringstream& os;
  std::map<uint32_t, std::set<std::pair<int, int>>> derived;  // IMAD operand registers per u
  PtxEmitter(const Dag& dag, std::ostringstream& o) : d(dag), os(o) {}

  std::string reg(uint32_t n) const {
    const Node& nd = d.nodes[n];
    if (nd.kind == NK_VAR) return "%v" + std::to_string(nd.val);
    return "%c" + std::to_string(n);
  }
  std::string operand(uint32_t n) const {
    const Node& nd = d.nodes[n];
    return nd.kind == NK_CONST ? ptx_imm(nd.val) : reg(n);
  }
  static std::string dname(uint32_t u, int k, int c) {
    auto enc = [](int v) { return v < 0 ? "m" + std::to_string(-v) : std::to_string(v); };
    return "%d" + std::to_string(u) + "_" + enc(k) + "_" + enc(c);
  }
  std::string affine(uint32_t u, int k, int c, bool record) {
    if (k == 0) return ptx_imm((uint32_t)c);
    if (k == 1 && c == 0) return reg(u);
    if (record) derived[u].insert({k, c});
    return dname(u, k, c);
  }
  static void mc(uint8_t f, int* m, int* c) {
    switch (f) {
      case 0: *m = 0; *c = 0; break;
      case 1: *m = 0; *c = -1; break;
      case 2: *m = 1; *c = 0; break;
      default: *m = -1; *c = -1; break;
    }
  }
  void plan_cell(const Lut& L) {
    if (L.kind != 1 || d.nodes[L.in[0]].kind == NK_CONST) return;
    int m0, c0, m1, c1;
    mc(L.f0, &m0, &c0);
    mc(L.f1, &m1, &c1);
    affine(L.in[1], m0 - m1, m0, true);
    affine(L.in[1], c0 - c1, c0, true);
  }
  void emit_derived(uint32_t u) {
    auto it = derived.find(u);
    if (it == derived.end()) return;
    for (auto& kc : it->second)
      os << "\tmad.lo.u32 " << dname(u, kc.first, kc.second) << ", " << reg(u) << ", " << ptx_imm((uint32_t)kc.first)
         << ", " << ptx_imm((uint32_t)kc.second) << ";\n";
  }
  void cell(const Lut& L) {
    if (L.kind == 1) {
      int m0, c0, m1, c1;
      mc(L.f0, &m0, &c0);
      mc(L.f1, &m1, &c1);
      const Node& xn = d.nodes[L.in[0]];
      if (xn.kind == NK_CONST) {
        const uint32_t K = xn.val;
        const uint32_t K0 = (uint32_t)((int)K * m0 + c0), K1 = (uint32_t)((int)K * m1 + c1);
        os << "\tmad.lo.u32 " << reg(L.root) << ", " << reg(L.in[1]) << ", " << ptx_imm(K0 - K1) << ", "
           << ptx_imm(K0) << ";\n";
      } else {
        os << "\tmad.lo.u32 " << reg(L.root) << ", " << reg(L.in[0]) << ", " << affine(L.in[1], m0 - m1, m0, false)
           << ", " << affine(L.in[1], c0 - c1, c0, false) << ";\n";
      }
    } else if (L.kind == 2) {  // x * K + C (K, C hoisted; a constant x goes in the immediate slot)
      const bool xc = d.nodes[L.in[0]].kind == NK_CONST;
      os << "\tmad.lo.u32 " << reg(L.root) << ", " << operand(xc ? L.in[1] : L.in[0]) << ", "
         << operand(xc ? L.in[0] : L.in[1]) << ", " << operand(L.in[2]) << ";\n";
    } else {
      char imm[8];
      snprintf(imm, sizeof imm, "0x%02X", L.imm);
      os << "\tlop3.b32 " << reg(L.root) << ", " << operand(L.in[0]) << ", " << operand(L.in[1]) << ", "
         << operand(L.in[2]) << ", " << imm << ";\n";
    }
    emit_derived(L.root);
  }
};

// u64 warp sum of %acc (butterfly), leaves the total in %acc of every lane
void ptx_warp_sum(std::ostringstream& os) {
  for (int off = 16; off > 0; off >>= 1)
    os << "\tmov.b64 {%lo, %hi}, %acc;\n"
       << "\tshfl.sync.bfly.b32 %lo2, %lo, " << off << ", 31, -1;\n"
       << "\tshfl.sync.bfly.b32 %hi2, %hi, " << off << ", 31, -1;\n"
       << "\tmov.b64 %x64, {%lo2, %hi2};\n"
       << "\tadd.u64 %acc, %acc, %x64;\n";
}

}  // namespace

std::string emit_ptx(const Parsed& prog, const KernelSpec& spec, KernelStats* stats, uint64_t body_o_count) {
  KernelStats st;
  const bool as_body = !spec.body_name.empty();
  Built b;
  build_specialised(prog, spec, &b);
  const Dag& D = b.D;
  const std::vector<Lit>& outs = b.outs;
  const int S = b.S, s = b.s, t = b.t, m = b.m;
  double best_t = 0;
  MapResult mr = choose_mapping(b, spec, &best_t, &st.imad_cost);
  dfs_order(&mr, outs);
  std::vector<uint8_t> used(64, 0);
  std::vector<uint32_t> var_node(64, 0);
  for (size_t k = 0; k < D.nodes.size(); k++)
    if (D.nodes[k].kind == NK_VAR) var_node[D.nodes[k].val] = (uint32_t)k;
  auto mark = [&](uint32_t n) { if (D.nodes[n].kind == NK_VAR) used[D.nodes[n].val] = 1; };
  for (const Lut& L : mr.luts) for (int q = 0; q < 3; q++) mark(L.in[q]);
  for (Lit o : outs) mark(lit_node(o));
  std::ostringstream body;
  PtxEmitter E(D, body);
  for (const Lut& L : mr.luts) E.plan_cell(L);
  for (auto& kv : E.derived) {
    const int lv = mr.node_level[kv.first];
    if (lv == 3) st.derived_inner += (uint32_t)kv.second.size();
    if (lv == 2) st.derived_outer += (uint32_t)kv.second.size();
  }
  auto level_of = [&](int v) { return (int)b.var_level[v]; };
  // The count of one thread-iteration is sum over the 2^s slot outputs of
  // popc(output).  Per distinct output node x with k positive and j
  // complemented uses that is (k - j) popc(x) + 32 j.  Outputs computed at the
  // thread / outer level are counted once per outer iteration (x 2^m); inner
  // outputs right after the cell that defines them, so no slot output stays
  // live to the end of the body (register pressure).
  struct OutUse { int k = 0, j = 0; };
  std::map<uint32_t, OutUse> out_use;
  uint32_t const_pop = 0;
  for (int sl = 0; sl < S; sl++) {
    const Lit o = outs[sl];
    const Node& on = D.nodes[lit_node(o)];
    if (on.kind == NK_CONST) { const_pop += (uint32_t)__builtin_popcount(lit_neg(o) ? ~on.val : on.val); continue; }
    OutUse& u = out_use[lit_node(o)];
    (lit_neg(o) ? u.j : u.k)++;
  }
  auto node_level = [&](uint32_t x) {
    return D.nodes[x].kind == NK_VAR ? level_of((int)D.nodes[x].val) : (int)mr.node_level[x];
  };
  uint32_t inner_const = 0, outer_const = const_pop;
  auto count_out = [&](uint32_t x, const char* acc) {  // acc += (k - j) popc(x); constants aside
    const OutUse& u = out_use.at(x);
    (node_level(x) == 3 ? inner_const : outer_const) += 32u * (uint32_t)u.j;
    if (u.k == u.j) return;
    body << "\tpopc.b32 %t2, " << E.reg(x) << ";\n";
    if (u.k - u.j == 1) body << "\tadd.u32 " << acc << ", " << acc << ", %t2;\n";
    else body << "\tmad.lo.u32 " << acc << ", %t2, " << ptx_imm((uint32_t)(u.k - u.j)) << ", " << acc << ";\n";
  };
  auto emit_level = [&](int lvl) {
    for (const Lut& L : mr.luts) {
      if (L.level != lvl) continue;
      E.cell(L);
      uint32_t* luts = lvl == 1 ? &st.luts_thread : lvl == 2 ? &st.luts_outer : &st.luts_inner;
      uint32_t* imads = lvl == 1 ? &st.imads_thread : lvl == 2 ? &st.imads_outer : &st.imads_inner;
      (*(L.kind != 0 ? imads : luts))++;
      if (lvl == 3 && out_use.count(L.root)) count_out(L.root, "%a32");
    }
  };
  const int unit = s + t + m;
  // ---- prologue: chunk bounds and thread-level variables/cells
  body << "\tmov.u32 %tidr, %tid.x;\n";
  if (as_body) {
    body << "\tld.param.u64 %cnt, [p_count];\n\tld.param.u32 %bid, [p_bid];\n\tld.param.u32 %nb, [p_nb];\n"
         << "\tmov.u64 %A, 0;\n\tmov.u64 %O, " << body_o_count << ";\n";
  } else {
    body << "\tld.param.u64 %A, [p_A];\n\tld.param.u64 %O, [p_O];\n\tld.param.u64 %cnt, [p_count];\n"
         << "\tmov.u32 %bid, %ctaid.x;\n\tmov.u32 %nb, %nctaid.x;\n";
  }
  body << "\tcvta.to.global.u64 %cnt, %cnt;\n"
       << "\tcvt.u64.u32 %b, %bid;\n\tcvt.u64.u32 %x64, %nb;\n"
       << "\tdiv.u64 %q, %O, %x64;\n\trem.u64 %rr, %O, %x64;\n"
       << "\tmul.lo.u64 %ob, %b, %q;\n\tmin.u64 %y64, %b, %rr;\n\tadd.u64 %ob, %ob, %y64;\n"
       << "\tsetp.lt.u64 %p0, %b, %rr;\n\tselp.u64 %y64, 1, 0, %p0;\n"
       << "\tadd.u64 %oe, %ob, %q;\n\tadd.u64 %oe, %oe, %y64;\n";
  for (int v = 0; v < 64; v++)
    if (used[v] && level_of(v) == 1) {
      body << "\tbfe.u32 %t0, %tidr, " << (b.pos[v] - 5 - s) << ", 1;\n\tneg.s32 %v" << v << ", %t0;\n";
      E.emit_derived(var_node[v]);
      st.thread_vars++;
    }
  emit_level(1);
  body << "\tmov.u64 %acc, 0;\n\tmov.u64 %o, %ob;\n"
       << "\tsetp.ge.u64 %p0, %o, %oe;\n\t@%p0 bra $L_done;\n"
       << "$L_outer:\n\t.pragma \"nounroll\";\n"
       << "\tshl.b64 %wo, %o, " << unit << ";\n\tadd.u64 %wo, %wo, %A;\n";
  for (int v = 0; v < 64; v++)
    if (used[v] && level_of(v) == 2) {
      body << "\tshr.u64 %x64, %wo, " << (b.pos[v] - 5) << ";\n\tcvt.u32.u64 %t0, %x64;\n"
           << "\tand.b32 %t0, %t0, 1;\n\tneg.s32 %v" << v << ", %t0;\n";
      E.emit_derived(var_node[v]);
      st.outer_vars++;
    }
  emit_level(2);
  // thread- and outer-level outputs: counted once per outer iteration
  body << "\tmov.u32 %po, 0;\n";
  for (auto& ou : out_use)
    if (node_level(ou.first) < 3) count_out(ou.first, "%po");
  body << "\tmov.u32 %a32, 0;\n\tmov.u32 %ii, 0;\n"
       << "$L_inner:\n\t.pragma \"nounroll\";\n";
  for (int v = 0; v < 64; v++)
    if (used[v] && level_of(v) == 3) {
      const int k = b.pos[v] - 5 - s - t;
      body << "\tshl.b32 %t0, %ii, " << (31 - k) << ";\n\tshr.s32 %v" << v << ", %t0, 31;\n";
      E.emit_derived(var_node[v]);
      if (out_use.count(var_node[v])) count_out(var_node[v], "%a32");
      st.inner_vars++;
    }
  emit_level(3);
  if (inner_const) body << "\tadd.u32 %a32, %a32, " << inner_const << ";\n";
  body << "\tadd.u32 %ii, %ii, 1;\n\tsetp.lt.u32 %p1, %ii, " << (1u << m) << ";\n\t@%p1 bra $L_inner;\n";
  if (outer_const) body << "\tadd.u32 %po, %po, " << outer_const << ";\n";
  body << "\tshl.b32 %po, %po, " << m << ";\n\tadd.u32 %a32, %a32, %po;\n"
       << "\tcvt.u64.u32 %x64, %a32;\n\tadd.u64 %acc, %acc, %x64;\n"
       << "\tadd.u64 %o, %o, 1;\n\tsetp.lt.u64 %p0, %o, %oe;\n\t@%p0 bra $L_outer;\n"
       << "$L_done:\n";
  if (spec.count_shift) body << "\tshl.b64 %acc, %acc, " << spec.count_shift << ";\n";
  ptx_warp_sum(body);
  body << "\tand.b32 %t0, %tidr, 31;\n";
  if (as_body) {
    body << "\tsetp.eq.u32 %p0, %t0, 0;\n\tsetp.ne.u64 %p1, %acc, 0;\n\tand.pred %p0, %p0, %p1;\n"
         << "\t@%p0 red.global.add.u64 [%cnt], %acc;\n\tret;\n";
  } else {
    const int nw = 1 << (t - 5 > 0 ? t - 5 : 0);
    body << "\tshr.u32 %t1, %tidr, 5;\n\tmov.u32 %t2, bfa_red;\n\tshl.b32 %t1, %t1, 3;\n\tadd.u32 %t2, %t2, %t1;\n"
         << "\tsetp.eq.u32 %p0, %t0, 0;\n\t@%p0 st.shared.u64 [%t2], %acc;\n\tbar.sync 0;\n"
         << "\tsetp.ge.u32 %p0, %tidr, 32;\n\t@%p0 bra $L_end;\n"
         << "\tmov.u64 %acc, 0;\n\tsetp.lt.u32 %p1, %tidr, " << nw << ";\n"
         << "\tmov.u32 %t2, bfa_red;\n\tshl.b32 %t1, %tidr, 3;\n\tadd.u32 %t2, %t2, %t1;\n"
         << "\t@%p1 ld.shared.u64 %acc, [%t2];\n";
    ptx_warp_sum(body);
    body << "\tsetp.eq.u32 %p0, %tidr, 0;\n\tsetp.ne.u64 %p1, %acc, 0;\n\tand.pred %p0, %p0, %p1;\n"
         << "\t@%p0 red.global.add.u64 [%cnt], %acc;\n$L_end:\n\tret;\n";
  }
  // ---- declarations + signature
  std::ostringstream os;
  os << "// generated by libbfa (PTX): count specialised s=" << s << " t=" << t << " m=" << m
     << (spec.perm.empty() ? "" : " (permuted roles)") << "\n";
  const std::string bounds = "\t.maxntid " + std::to_string(1 << t) + ", 1, 1\n" +
                             (spec.min_blocks > 0 ? "\t.minnctapersm " + std::to_string(spec.min_blocks) + "\n" : "");
  if (as_body) {
    os << ".func " << spec.body_name << "(.param .b64 p_count, .param .b32 p_bid, .param .b32 p_nb)\n{\n";
  } else {
    os << kPtxHeader << ".shared .align 8 .b64 bfa_red[32];\n"
       << ".visible .entry bfa_kernel(.param .u64 p_A, .param .u64 p_O, .param .u64 p_B, .param .u64 p_out, "
          ".param .u64 p_count)\n" << bounds << "{\n";
  }
  os << "\t.reg .pred %p<2>;\n\t.reg .b32 %t<3>, %c<" << D.nodes.size() << ">, %v<64>;\n"
     << "\t.reg .b32 %tidr, %bid, %nb, %ii, %a32, %po, %lo, %hi, %lo2, %hi2;\n"
     << "\t.reg .b64 %A, %O, %cnt, %b, %q, %rr, %ob, %oe, %o, %wo, %acc, %x64, %y64;\n";
  for (auto& kv : E.derived)
    for (auto& kc : kv.second) os << "\t.reg .b32 " << PtxEmitter::dname(kv.first, kc.first, kc.second) << ";\n";
  os << body.str() << "}\n";
  st.words_per_iter = (uint32_t)S;
  if (stats) *stats = st;
  return os.str();
}

std::string emit_ptx_queue(const std::vector<std::string>& body_ptx, const std::vector<std::string>& body_name,
                           const std::vector<uint32_t>& chunks, int thread_bits, int min_blocks, int opt_level) {
  std::ostringstream os;
  const size_t nb = body_name.size();
  os << "// generated by libbfa (PTX) -O" << opt_level << ": work-queue kernel of " << nb << " programs\n"
     << kPtxHeader;
  uint64_t total = 0;
  os << ".const .align 4 .u32 bfa_qpre[" << nb + 1 << "] = {";
  for (size_t i = 0; i < nb; i++) {
    os << (i ? ", " : "") << total;
    total += chunks[i];
  }
  os << ", " << total << "};\n";
  for (const std::string& b : body_ptx) os << b;
  os << ".visible .entry bfa_kernel(.param .u64 p_count, .param .u64 p_ctr)\n"
     << "\t.maxntid " << (1 << thread_bits) << ", 1, 1\n"
     << (min_blocks > 0 ? "\t.minnctapersm " + std::to_string(min_blocks) + "\n" : "") << "{\n"
     << "\t.reg .pred %p<4>;\n\t.reg .b32 %c, %lo, %hi, %mid, %k, %tidr, %s, %qv, %sh;\n"
     << "\t.reg .b64 %cnt, %ctr, %x, %y;\n"
     << "\t.shared .align 4 .u32 s_chunk;\n"
     << "\tld.param.u64 %cnt, [p_count];\n\tld.param.u64 %ctr, [p_ctr];\n\tcvta.to.global.u64 %ctr, %ctr;\n"
     << "\tmov.u32 %tidr, %tid.x;\n\tmov.u32 %sh, s_chunk;\n"
     << "$Q_loop:\n"
     << "\tbar.sync 0;\n\tsetp.eq.u32 %p0, %tidr, 0;\n"
     << "\t@%p0 atom.global.add.u32 %c, [%ctr], 1;\n\t@%p0 st.shared.u32 [%sh], %c;\n\tbar.sync 0;\n"
     << "\tld.shared.u32 %c, [%sh];\n\tsetp.lt.u32 %p1, %c, " << total << ";\n\t@%p1 bra $Q_work;\n"
     << "\tmov.u32 %s, %nctaid.x;\n\tadd.u32 %s, %s, " << (uint32_t)(total - 1) << ";\n"
     << "\tsetp.eq.u32 %p2, %c, %s;\n\tand.pred %p2, %p2, %p0;\n\t@%p2 st.global.u32 [%ctr], 0;\n\tret;\n"
     << "$Q_work:\n\tmov.u32 %lo, 0;\n\tmov.u32 %hi, " << (nb - 1) << ";\n"
     << "$Q_bs:\n\tsetp.ge.u32 %p3, %lo, %hi;\n\t@%p3 bra $Q_found;\n"
     << "\tadd.u32 %mid, %lo, %hi;\n\tadd.u32 %mid, %mid, 1;\n\tshr.u32 %mid, %mid, 1;\n"
     << "\tmul.wide.u32 %x, %mid, 4;\n\tmov.u64 %y, bfa_qpre;\n\tadd.u64 %x, %y, %x;\n\tld.const.u32 %qv, [%x];\n"
     << "\tsetp.le.u32 %p3, %qv, %c;\n\t@%p3 mov.u32 %lo, %mid;\n\t@!%p3 sub.u32 %hi, %mid, 1;\n\tbra.uni $Q_bs;\n"
     << "$Q_found:\n\tmul.wide.u32 %x, %lo, 4;\n\tmov.u64 %y, bfa_qpre;\n\tadd.u64 %x, %y, %x;\n"
     << "\tld.const.u32 %qv, [%x];\n\tsub.u32 %k, %c, %qv;\n\tbra.uni $Q_dispatch;\n";
  for (size_t i = 0; i < nb; i++)
    os << "$Q_b" << i << ":\n\t{\n\t.param .b64 a0;\n\t.param .b32 a1;\n\t.param .b32 a2;\n"
       << "\tmov.u32 %s, " << chunks[i] << ";\n"
       << "\tst.param.b64 [a0], %cnt;\n\tst.param.b32 [a1], %k;\n\tst.param.b32 [a2], %s;\n"
       << "\tcall.uni " << body_name[i] << ", (a0, a1, a2);\n\t}\n\tbra.uni $Q_loop;\n";
  // dispatch: a balanced tree of uniform compare-and-branch on the body index
  // (an indirect `brx.idx` over a 512-entry .branchtargets table returned
  // wrong, run-to-run varying counts on sm_100a; the tree is exact)
  os << "$Q_dispatch:\n";
  std::function<void(size_t, size_t, const std::string&)> tree = [&](size_t a, size_t b, const std::string& lbl) {
    if (!lbl.empty()) os << lbl << ":\n";
    if (b - a == 1) { os << "\tbra.uni $Q_b" << a << ";\n"; return; }
    const size_t mid = (a + b) / 2;
    const std::string right = "$Q_t" + std::to_string(mid) + "_" + std::to_string(b);
    os << "\tsetp.ge.u32 %p3, %lo, " << mid << ";\n\t@%p3 bra.uni " << right << ";\n";
    tree(a, mid, "");
    tree(mid, b, right);
  };
  tree(0, nb, "");
  os << "}\n";
  return os.str();
}

SegPlan emit_segmented(const Parsed& prog, KernelMode mode, bool fuse_count, int seg_cells, int thread_bits,
                       int imad_cost_pct, int remat_cells) {
  KernelSpec spec;
  spec.mode = mode;
  spec.generic = true;
  spec.slot_bits = 0;
  spec.thread_bits = thread_bits;
  spec.inner_bits = 0;
  spec.dual_pipe = imad_cost_pct > 0;
  spec.imad_cost_pct = imad_cost_pct;
  Built b;
  build_specialised(prog, spec, &b);
  const Dag& D = b.D;
  MapResult mr = choose_mapping(b, spec, nullptr, nullptr);
  dfs_order(&mr, b.outs);
  const size_t C = mr.luts.size();
  SegPlan plan;
  const int nseg = (int)std::max<size_t>(1, (C + seg_cells - 1) / std::max(1, seg_cells));
  std::unordered_map<uint32_t, size_t> at;
  for (size_t k = 0; k < C; k++) at[mr.luts[k].root] = k;
  auto nin_of = [](const Lut& L) { return L.kind == 1 ? 2 : (int)L.nin; };
  // Rematerialisation: a cell whose whole cone (down to variables) has at
  // most kRemat cells is recomputed in every segment that needs it instead of
  // being stored -- the hash-consed DAG of a large term reuses many small
  // subterms across the whole program.
  const int kRemat = remat_cells;
  std::vector<int> cone(C, 0);
  for (size_t k = 0; k < C; k++) {
    int c = 1;
    const Lut& L = mr.luts[k];
    for (int q = 0; q < nin_of(L) && c <= kRemat; q++) {
      auto it = at.find(L.in[q]);
      if (it != at.end()) c += cone[it->second];
    }
    cone[k] = std::min(c, kRemat + 1);  // inputs precede k in DFS post-order
  }
  auto remat = [&](uint32_t n) { auto it = at.find(n); return it != at.end() && cone[it->second] <= kRemat; };
  auto seg_of = [&](size_t k) { return (int)(k / seg_cells); };
  // last segment using each stored value (the output counts as used in the last)
  std::unordered_map<uint32_t, int> last_use;
  for (size_t k = 0; k < C; k++) {
    const Lut& L = mr.luts[k];
    for (int q = 0; q < nin_of(L); q++) {
      auto it = at.find(L.in[q]);
      if (it != at.end() && !remat(L.in[q]) && seg_of(it->second) < seg_of(k))
        last_use[L.in[q]] = std::max(last_use[L.in[q]], seg_of(k));
    }
  }
  const Lit out = b.outs[0];
  {
    auto it = at.find(lit_node(out));
    if (it != at.end() && !remat(lit_node(out)) && seg_of(it->second) < nseg - 1) last_use[lit_node(out)] = nseg - 1;
  }
  // global slots, reused by liveness
  std::unordered_map<uint32_t, uint32_t> slot;
  std::vector<std::vector<uint32_t>> by_def(nseg);
  for (auto& kv : last_use) by_def[seg_of(at[kv.first])].push_back(kv.first);
  std::vector<std::pair<int, uint32_t>> busy;
  std::vector<uint32_t> free_slots;
  for (int sg = 0; sg < nseg; sg++) {
    for (size_t i = 0; i < busy.size();)
      if (busy[i].first <= sg) { free_slots.push_back(busy[i].second); busy[i] = busy.back(); busy.pop_back(); }
      else i++;
    std::sort(by_def[sg].begin(), by_def[sg].end());
    for (uint32_t v : by_def[sg]) {
      uint32_t sl;
      if (!free_slots.empty()) { sl = free_slots.back(); free_slots.pop_back(); }
      else sl = plan.n_slots++;
      slot[v] = sl;
      busy.push_back({last_use[v], sl});
    }
    plan.max_live = std::max<uint32_t>(plan.max_live, (uint32_t)busy.size());
  }
  std::unordered_map<uint32_t, std::vector<uint32_t>> var_nodes;
  for (size_t q = 0; q < D.nodes.size(); q++)
    if (D.nodes[q].kind == NK_VAR) var_nodes[D.nodes[q].val].push_back((uint32_t)q);
  const bool want_count = mode == KM_COUNT || fuse_count;
  for (int sg = 0; sg < nseg; sg++) {
    std::ostringstream os;
    os << "// generated by libbfa: segment " << sg << "/" << nseg << "\n" << kPrelude;
    Emitter E(D, os);
    for (const Lut& L : mr.luts) E.plan_cell(L);
    const size_t k0 = (size_t)sg * seg_cells, k1 = std::min(C, k0 + seg_cells);
    const bool last = sg == nseg - 1;
    os << "extern \"C\" __global__ void __launch_bounds__(" << (1 << thread_bits) << ")\n"
       << "bfa_kernel(const u64 w_begin, const u64 w_count, const u32 mask, u32* __restrict__ gbuf, const u64 stride, "
       << "u32* __restrict__ out, u64* __restrict__ count) {\n"
       << "  u64 acc = 0;\n"
       << "  const u64 gstride = (u64)gridDim.x * blockDim.x;\n"
       << "  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < w_count; k += gstride) {\n"
       << "    const u64 w = w_begin + k;\n";
    // values available in this segment; everything is emitted at first use
    std::unordered_map<uint32_t, uint8_t> avail;
    std::function<void(uint32_t)> ensure = [&](uint32_t n) {
      if (avail.count(n)) return;
      const Node& nd = D.nodes[n];
      if (nd.kind == NK_CONST) return;
      avail[n] = 1;
      if (nd.kind == NK_VAR) {
        os << "    const u32 v" << nd.val << " = 0u - (u32)((w >> " << (b.pos[nd.val] - 5) << ") & 1ull);\n";
        E.emit_derived(n, "    ");
        return;
      }
      auto it = at.find(n);
      if (it == at.end()) return;
      const size_t k = it->second;
      if ((size_t)k >= k0 && k < k1) { avail.erase(n); return; }  // defined later in this segment
      if (remat(n)) {                                            // recompute the small cone here
        const Lut& L = mr.luts[k];
        for (int q = 0; q < nin_of(L); q++) ensure(L.in[q]);
        E.lut(L, "    ");
      } else {
        os << "    const u32 " << E.name(n) << " = __ldcs(gbuf + " << slot.at(n) << "ull * stride + k);\n";
        E.emit_derived(n, "    ");
      }
    };
    for (size_t k = k0; k < k1; k++) {
      const Lut& L = mr.luts[k];
      for (int q = 0; q < nin_of(L); q++) ensure(L.in[q]);
      E.lut(L, "    ");
      avail[L.root] = 1;
      auto it = slot.find(L.root);
      if (it != slot.end()) os << "    __stcs(gbuf + " << it->second << "ull * stride + k, " << E.name(L.root) << ");\n";
    }
    if (last) {
      ensure(lit_node(out));
      os << "    const u32 r = (" << E.value(out) << ") & mask;\n";
      if (mode == KM_EVAL) os << "    out[k] = r;\n";
      if (want_count) os << "    acc += __popc(r);\n";
    }
    os << "  }\n";
    if (last && want_count) os << "  bfa_block_sum(acc, count);\n";
    os << "}\n";
    plan.sources.push_back(os.str());
    plan.cells.push_back((uint32_t)(k1 - k0));
    plan.emitted += E.cells_emitted;
  }
  return plan;
}

std::string emit_multi(const std::vector<const Parsed*>& progs, const std::vector<KernelSpec>& specs,
                       std::vector<KernelStats>* stats) {
  std::ostringstream os;
  os << "// generated by libbfa: multi-body kernel of " << progs.size() << " programs\n" << kPrelude;
  if (stats) stats->assign(progs.size(), KernelStats());
  for (size_t c = 0; c < progs.size(); c++) {
    KernelSpec sp = specs[c];
    sp.body_name = "bfa_body_" + std::to_string(c);
    KernelStats st;
    os << emit_kernel(*progs[c], sp, &st);
    if (stats) (*stats)[c] = st;
  }
  const KernelSpec& s0 = specs[0];
  const std::string bounds = std::to_string(1 << s0.thread_bits) +
                             (s0.min_blocks > 0 ? ", " + std::to_string(s0.min_blocks) : "");
  os << "extern \"C\" __global__ void __launch_bounds__(" << bounds << ")\n"
     << "bfa_kernel(const u64 A, const u64 o_count, const u64 out_base_w, u32* __restrict__ out, "
     << "u64* __restrict__ count, const u32 bpc) {\n"
     << "  const u32 c = blockIdx.x / bpc, bid = blockIdx.x - c * bpc;\n"
     << "  switch (c) {\n";
  for (size_t c = 0; c < progs.size(); c++)
    os << "    case " << c << ": bfa_body_" << c << "(A, o_count, out_base_w, out, count, bid, bpc); break;\n";
  os << "  }\n}\n";
  return os.str();
}

std::string emit_queue(const std::vector<std::string>& body_src, const std::vector<std::string>& body_name,
                       const std::vector<uint64_t>& o_count, const std::vector<uint32_t>& chunks, int thread_bits,
                       int min_blocks) {
  std::ostringstream os;
  const size_t nb = body_src.size();
  os << "// generated by libbfa: work-queue kernel of " << nb << " programs\n" << kPrelude;
  for (const std::string& b : body_src) os << b;
  uint64_t total = 0;
  os << "__constant__ u32 bfa_qpre[" << nb + 1 << "] = {";
  for (size_t i = 0; i < nb; i++) {
    os << (i ? ", " : "") << total << "u";
    total += chunks[i];
  }
  os << ", " << total << "u};\n";
  const std::string bounds = std::to_string(1 << thread_bits) + (min_blocks > 0 ? ", " + std::to_string(min_blocks) : "");
  os << "extern \"C\" __global__ void __launch_bounds__(" << bounds << ")\n"
     << "bfa_kernel(u64* __restrict__ count, u32* __restrict__ ctr) {\n"
     << "  __shared__ u32 s_chunk;\n"
     << "  for (;;) {\n"
     << "    __syncthreads();  // every thread has read the previous chunk number\n"
     << "    if (threadIdx.x == 0) s_chunk = atomicAdd(ctr, 1u);\n"
     << "    __syncthreads();\n"
     << "    const u32 c = s_chunk;\n"
     << "    if (c >= " << total << "u) {  // the last exit restores the counter for the next launch\n"
     << "      if (threadIdx.x == 0 && c == " << total << "u + gridDim.x - 1u) *ctr = 0u;\n"
     << "      return;\n"
     << "    }\n"
     << "    int lo = 0, hi = " << nb - 1 << ";\n"
     << "    while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (bfa_qpre[mid] <= c) lo = mid; else hi = mid - 1; }\n"
     << "    const u32 k = c - bfa_qpre[lo];\n"
     << "    switch (lo) {\n";
  for (size_t i = 0; i < nb; i++)
    os << "      case " << i << ": " << body_name[i] << "(0ull, " << o_count[i] << "ull, 0ull, nullptr, count, k, "
       << chunks[i] << "u); break;\n";
  os << "    }\n"
     << "  }\n"
     << "}\n";
  return os.str();
}

std::string emit_batch(const std::vector<const Parsed*>& progs, int thread_bits) {
  std::ostringstream os;
  os << "// generated by libbfa: batch of " << progs.size() << " programs\n" << kPrelude;
  KernelSpec spec;
  spec.mode = KM_COUNT;
  spec.generic = true;
  spec.slot_bits = 0;
  spec.thread_bits = thread_bits;
  spec.inner_bits = 0;
  spec.dual_pipe = 0;
  for (size_t j = 0; j < progs.size(); j++) {
    Built b;
    build_specialised(*progs[j], spec, &b);
    MapResult mr = choose_mapping(b, spec, nullptr, nullptr);
    dfs_order(&mr, b.outs);
    Emitter E(b.D, os);
    os << "__device__ __noinline__ u32 bfa_prog_" << j << "(const u64 w) {\n";
    std::vector<uint8_t> used(64, 0);
    for (const Lut& L : mr.luts)
      for (int q = 0; q < L.nin; q++)
        if (b.D.nodes[L.in[q]].kind == NK_VAR) used[b.D.nodes[L.in[q]].val] = 1;
    if (b.D.nodes[lit_node(b.outs[0])].kind == NK_VAR) used[b.D.nodes[lit_node(b.outs[0])].val] = 1;
    for (int v = 0; v < 64; v++)
      if (used[v]) os << "  const u32 v" << v << " = 0u - (u32)((w >> " << (b.pos[v] - 5) << ") & 1ull);\n";
    for (const Lut& L : mr.luts) E.lut(L, "  ");
    os << "  return " << E.value(b.outs[0]) << ";\n}\n";
  }
  os << "extern \"C\" __global__ void __launch_bounds__(" << (1 << thread_bits) << ")\n"
     << "bfa_kernel(const u64* __restrict__ start, const u32* __restrict__ masks, const u64* __restrict__ words, "
     << "const int nprog, const u64 total, u64* __restrict__ counts) {\n"
     << "  const u64 gstride = (u64)gridDim.x * blockDim.x;\n"
     << "  for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gstride) {\n"
     << "    // program of this word: warp-uniform (ranges are padded to whole warps)\n"
     << "    int lo = 0, hi = nprog - 1;\n"
     << "    while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (start[mid] <= g) lo = mid; else hi = mid - 1; }\n"
     << "    const u64 k = g - start[lo];\n"
     << "    u32 r = 0;\n"
     << "    if (k < words[lo]) {\n"
     << "      switch (lo) {\n";
  for (size_t j = 0; j < progs.size(); j++) os << "        case " << j << ": r = bfa_prog_" << j << "(k); break;\n";
  os << "      }\n"
     << "      r &= masks[lo];\n"
     << "    }\n"
     << "    u32 c = __reduce_add_sync(0xffffffffu, (u32)__popc(r));\n"
     << "    if ((threadIdx.x & 31u) == 0 && c) atomicAdd(counts + lo, (u64)c);\n"
     << "  }\n"
     << "}\n";
  return os.str();
}

InterpProgram build_interp(const Parsed& prog) {
  // the generic specialisation: lanes 0-4 as word constants, variables >= 5
  // computed from the word index; plain LUT3 cover
  Dag D;
  std::vector<Lit> subst(64);
  for (int v = 0; v < 64; v++) subst[v] = v < 5 ? D.word(kLane[v]) : D.var((uint32_t)v);
  std::vector<uint8_t> done(prog.dag.nodes.size());
  std::vector<Lit> memo(prog.dag.nodes.size());
  Lit out = rebuild(prog.dag, prog.root, subst, D, memo, done);
  std::vector<uint8_t> lv(64, 3);
  const double w[4] = {0, 1, 1, 1};
  MapResult mr = map_luts(D, {out}, lv, w);
  InterpProgram ip;
  // value list in evaluation order: used variables first, then LUT roots
  std::vector<uint32_t> order;
  std::vector<uint8_t> isvar(D.nodes.size(), 0);
  for (const Lut& L : mr.luts)
    for (int q = 0; q < 3; q++)
      if (D.nodes[L.in[q]].kind == NK_VAR && !isvar[L.in[q]]) { isvar[L.in[q]] = 1; order.push_back(L.in[q]); }
  if (D.nodes[lit_node(out)].kind == NK_VAR && !isvar[lit_node(out)]) { isvar[lit_node(out)] = 1; order.push_back(lit_node(out)); }
  std::map<uint32_t, const Lut*> lut_of;
  for (const Lut& L : mr.luts) { order.push_back(L.root); lut_of[L.root] = &L; }
  // last use (index in `order`) of every value; the output lives to the end
  std::map<uint32_t, size_t> last;
  for (size_t k = 0; k < order.size(); k++) {
    auto it = lut_of.find(order[k]);
    if (it != lut_of.end())
      for (int q = 0; q < 3; q++) last[it->second->in[q]] = k;
  }
  last[lit_node(out)] = order.size();
  std::map<uint32_t, uint32_t> constidx;
  auto cst = [&](uint32_t word) -> uint32_t {
    auto it = constidx.find(word);
    if (it != constidx.end()) return it->second;
    uint32_t i = (uint32_t)ip.consts.size();
    ip.consts.push_back(word);
    constidx[word] = i;
    return i;
  };
  std::map<uint32_t, uint32_t> slot;
  std::vector<uint32_t> free_slots;
  auto operand = [&](uint32_t n) -> uint32_t {
    if (D.nodes[n].kind == NK_CONST) return 0x80000000u | cst(D.nodes[n].val);
    return slot.at(n);
  };
  for (size_t k = 0; k < order.size(); k++) {
    const uint32_t n = order[k];
    uint32_t a = 0, b = 0, c = 0, imm = 0, kind = 1;
    auto it = lut_of.find(n);
    if (it != lut_of.end()) {
      const Lut& L = *it->second;
      kind = 0; imm = L.imm;
      a = operand(L.in[0]); b = operand(L.in[1]); c = operand(L.in[2]);
      // inputs whose last use is this op free their slots before dst is chosen
      for (int q = 0; q < 3; q++) {
        uint32_t in = L.in[q];
        if (D.nodes[in].kind != NK_CONST && last[in] == k && slot.count(in)) {
          bool dup = false;
          for (int r = 0; r < q; r++) dup |= L.in[r] == in;
          if (!dup) free_slots.push_back(slot[in]);
        }
      }
    } else {
      a = D.nodes[n].val - 5;
    }
    uint32_t dst;
    if (!free_slots.empty()) { dst = free_slots.back(); free_slots.pop_back(); }
    else dst = ip.n_slots++;
    slot[n] = dst;
    ip.ops.insert(ip.ops.end(), {dst | (imm << 16) | (kind << 24), a, b, c});
  }
  const Node& on = D.nodes[lit_node(out)];
  if (on.kind == NK_CONST) ip.out = 0x80000000u | cst(lit_neg(out) ? ~on.val : on.val);
  else { ip.out = slot.at(lit_node(out)); ip.out_neg = lit_neg(out); }
  return ip;
}

std::string to_text(const Parsed& prog) {
  // the cone of the root in node order (inputs precede their gates)
  const Dag& d = prog.dag;
  std::vector<uint8_t> in_cone(d.nodes.size(), 0);
  std::vector<uint32_t> st{lit_node(prog.root)};
  while (!st.empty()) {
    const uint32_t k = st.back();
    st.pop_back();
    if (in_cone[k]) continue;
    in_cone[k] = 1;
    if (d.nodes[k].kind == NK_GATE) { st.push_back(d.nodes[k].a); st.push_back(d.nodes[k].b); }
  }
  auto name = [&](uint32_t k) -> std::string {
    const Node& nd = d.nodes[k];
    if (nd.kind == NK_VAR) return "x" + std::to_string(nd.val);
    if (nd.kind == NK_CONST) return "0";
    return "g" + std::to_string(k);
  };
  std::ostringstream os;
  for (size_t k = 0; k < d.nodes.size(); k++) {
    if (!in_cone[k] || d.nodes[k].kind != NK_GATE) continue;
    const Node& nd = d.nodes[k];
    const std::string a = name(nd.a), b = name(nd.b);
    std::string e;
    switch (nd.tt) {   // bit (a + 2b) = f(a, b); f(0, 0) = 0 after normalisation
      case 0x2: e = a + " & ~" + b; break;
      case 0x4: e = "~" + a + " & " + b; break;
      case 0x6: e = a + " ^ " + b; break;
      case 0x8: e = a + " & " + b; break;
      case 0xE: e = a + " | " + b; break;
      default: {
        std::string t;
        for (int m = 0; m < 4; m++)
          if ((nd.tt >> m) & 1)
            t += (t.empty() ? "" : " | ") + std::string("(") + ((m & 1) ? "" : "~") + a + " & " + ((m & 2) ? "" : "~") +
                 b + ")";
        e = t.empty() ? "0" : t;
      }
    }
    os << "let " << name((uint32_t)k) << " = " << e << "\n";
  }
  const Node& rn = d.nodes[lit_node(prog.root)];
  if (rn.kind == NK_CONST) os << (lit_neg(prog.root) ? "1" : "0") << "\n";
  else os << (lit_neg(prog.root) ? "~" : "") << name(lit_node(prog.root)) << "\n";
  return os.str();
}

std::string dump_ir(const Parsed& prog, uint32_t* n_luts) {
  Dag D;
  std::vector<Lit> subst(64);
  for (int v = 0; v < 64; v++) subst[v] = D.var((uint32_t)v);
  std::vector<uint8_t> done(prog.dag.nodes.size());
  std::vector<Lit> memo(prog.dag.nodes.size());
  Lit out = rebuild(prog.dag, prog.root, subst, D, memo, done);
  std::vector<uint8_t> lv(64, 3);
  const double w[4] = {0, 1, 1, 1};
  MapResult mr = map_luts(D, {out}, lv, w);
  std::unordered_map<uint32_t, int> idx;
  std::ostringstream os;
  auto opnd = [&](uint32_t n) -> std::string {
    const Node& nd = D.nodes[n];
    if (nd.kind == NK_CONST) { char b[16]; snprintf(b, sizeof b, "0x%08x", nd.val); return b; }
    if (nd.kind == NK_VAR) return "x" + std::to_string(nd.val);
    return "L" + std::to_string(idx.at(n));
  };
  int k = 0;
  for (const Lut& L : mr.luts) {
    idx[L.root] = k;
    char imm[8];
    snprintf(imm, sizeof imm, "0x%02x", L.imm);
    os << "L" << k << " = lop3(" << opnd(L.in[0]) << ", " << opnd(L.in[1]) << ", " << opnd(L.in[2]) << ", "
       << imm << ")\n";
    k++;
  }
  os << "out = " << (lit_neg(out) ? "~" : "") << opnd(lit_node(out)) << "\n";
  if (n_luts) *n_luts = (uint32_t)mr.luts.size();
  return os.str();
}

}  // namespace bfa
