/*
 * bfa_oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously
 * correct CPU oracle for the free-Boolean-vector hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the product (paper_1310_6978_b200/, include/bfa.h):
 * it has its own tokenizer, its own parser and its own evaluator.
 *
 * What it computes (the definition the method reaches exactly):
 *   For every valuation index mu in [mu_lo, mu_hi):
 *     d[mu] = f(mu), where variable id v takes the value (mu >> v) & 1
 *   and count = sum of d[mu].
 *   - Prop 2.2 and proof: pi_mu d = t^B(mu(v1)..mu(vn))
 *   - valuations / interpretation of variables
 *   - number of models = number of 1 bits of d
 *   - connectives: ~ & | ^ with x+y = x~y v ~xy
 *   - a system e_i = phi_i is solved when every phi_i = 1
 *     so the program value is the conjunction of its constraint statements.
 *   Readings C-1..C-7 of DESIGN.md fix bit order (var id v <-> bit v of mu),
 *   vector layout (bit mu-mu_lo at u64 word (mu-mu_lo)>>6, bit (mu-mu_lo)&63),
 *   precedence  ~ > & > ^ > | > -> (right) > <-> (left), and constants.
 *
 * Evaluation is recursive descent over the AST, once per valuation, with
 * `let` definitions evaluated in order and stored per valuation, and the
 * constraints conjoined left to right with short-circuit.  No blocking, no
 * bit-parallelism, no reordering: one valuation at a time.
 *
 * Parallelism: valuations are split into 64-aligned blocks (whole output
 * words per block, so no two threads write the same word); pthreads.
 *
 * Pins: tests/test_oracle_pins.py (paper worked examples, closed forms,
 * numpy/Python-parser brute force, algebraic invariants).
 */
#include <ctype.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { K_VAR, K_CONST, K_NOT, K_AND, K_OR, K_XOR, K_IMP, K_IFF, K_REF };

typedef struct {
  int kind;
  int a, b;        /* children (binary / unary); VAR: id; CONST: value; REF: let slot */
  int first, cnt;  /* n-ary AND/OR: children list in kids[first .. first+cnt) */
} ONode;

typedef struct {
  ONode* nodes; int n_nodes, cap_nodes;
  int* kids; int n_kids, cap_kids;
  int* let_root; int n_lets, cap_lets;      /* root node of each let, in order */
  int* cons_root; int n_cons, cap_cons;     /* root node of each constraint   */
  int max_var;
  /* name table (open addressing) */
  char** names; int* name_slot; int name_cap, name_cnt;
} OProg;

/* ------------------------------------------------------------------ lexer */
enum { T_EOF, T_SEP, T_NOT, T_AND, T_XOR, T_OR, T_IMP, T_IFF, T_LP, T_RP, T_EQ,
       T_VAR, T_NAME, T_ZERO, T_ONE, T_LET };

typedef struct {
  const char* s; size_t pos; int line, col;
  int depth;                   /* paren depth: newlines separate only at depth 0 */
  int tok; long long ival; char name[256];
  int tline, tcol;
  char* err; size_t errlen; int failed;
} Lex;

static void lex_error(Lex* L, const char* fmt, ...) {
  if (L->failed) return;
  L->failed = 1;
  if (L->err && L->errlen) {
    char msg[512];
    va_list ap; va_start(ap, fmt); vsnprintf(msg, sizeof msg, fmt, ap); va_end(ap);
    snprintf(L->err, L->errlen, "%d:%d: %s", L->tline, L->tcol, msg);
  }
}

static void next(Lex* L) {
  for (;;) {
    char c = L->s[L->pos];
    if (c == '#') { while (L->s[L->pos] && L->s[L->pos] != '\n') { L->pos++; L->col++; } continue; }
    if (c == ' ' || c == '\t' || c == '\r') { L->pos++; L->col++; continue; }
    if (c == '\n' && L->depth > 0) { L->pos++; L->line++; L->col = 1; continue; }
    break;
  }
  L->tline = L->line; L->tcol = L->col;
  const char* p = L->s + L->pos;
  char c = *p;
  if (c == 0) { L->tok = T_EOF; return; }
  if (c == '\n') { L->pos++; L->line++; L->col = 1; L->tok = T_SEP; return; }
  if (c == ';') { L->pos++; L->col++; L->tok = T_SEP; return; }
  if (c == '~') { L->pos++; L->col++; L->tok = T_NOT; return; }
  if (c == '&') { L->pos++; L->col++; L->tok = T_AND; return; }
  if (c == '^') { L->pos++; L->col++; L->tok = T_XOR; return; }
  if (c == '|') { L->pos++; L->col++; L->tok = T_OR; return; }
  if (c == '(') { L->pos++; L->col++; L->depth++; L->tok = T_LP; return; }
  if (c == ')') { L->pos++; L->col++; if (L->depth > 0) L->depth--; L->tok = T_RP; return; }
  if (c == '=') { L->pos++; L->col++; L->tok = T_EQ; return; }
  if (c == '-' && p[1] == '>') { L->pos += 2; L->col += 2; L->tok = T_IMP; return; }
  if (c == '<' && p[1] == '-' && p[2] == '>') { L->pos += 3; L->col += 3; L->tok = T_IFF; return; }
  if (isdigit((unsigned char)c)) {
    size_t k = 0; while (isdigit((unsigned char)p[k])) k++;
    if (k == 1 && c == '0') { L->tok = T_ZERO; }
    else if (k == 1 && c == '1') { L->tok = T_ONE; }
    else { lex_error(L, "only the constants 0 and 1 are allowed"); L->tok = T_EOF; return; }
    L->pos += k; L->col += (int)k; return;
  }
  if (isalpha((unsigned char)c) || c == '_') {
    size_t k = 0; while (isalnum((unsigned char)p[k]) || p[k] == '_') k++;
    if (k >= sizeof L->name) { lex_error(L, "name too long"); L->tok = T_EOF; return; }
    memcpy(L->name, p, k); L->name[k] = 0;
    L->pos += k; L->col += (int)k;
    int all_digits = (k >= 2 && L->name[0] == 'x');
    for (size_t i = 1; i < k && all_digits; i++) all_digits = isdigit((unsigned char)L->name[i]);
    if (all_digits) {
      long long v = 0;
      for (size_t i = 1; i < k; i++) { v = v * 10 + (L->name[i] - '0'); if (v > 1000000) break; }
      L->ival = v; L->tok = T_VAR; return;
    }
    L->tok = strcmp(L->name, "let") == 0 ? T_LET : T_NAME;
    return;
  }
  lex_error(L, "unexpected character '%c'", c);
  L->tok = T_EOF;
}

/* ------------------------------------------------------------- program */
static void* grow(void* p, int* cap, int need, size_t elt) {
  if (need <= *cap) return p;
  int nc = *cap ? *cap : 16;
  while (nc < need) nc *= 2;
  void* q = realloc(p, (size_t)nc * elt);
  if (!q) { fprintf(stderr, "bfa_oracle: out of memory\n"); abort(); }
  *cap = nc;
  return q;
}

static int add_node(OProg* P, int kind, int a, int b) {
  P->nodes = grow(P->nodes, &P->cap_nodes, P->n_nodes + 1, sizeof(ONode));
  ONode* x = &P->nodes[P->n_nodes];
  x->kind = kind; x->a = a; x->b = b; x->first = 0; x->cnt = 0;
  return P->n_nodes++;
}

static uint64_t hash_str(const char* s) {
  uint64_t h = 1469598103934665603ull;
  while (*s) { h ^= (unsigned char)*s++; h *= 1099511628211ull; }
  return h;
}

/* returns slot or -1 */
static int name_find(const OProg* P, const char* s) {
  if (!P->name_cap) return -1;
  uint64_t h = hash_str(s) & (uint64_t)(P->name_cap - 1);
  while (P->names[h]) {
    if (strcmp(P->names[h], s) == 0) return P->name_slot[h];
    h = (h + 1) & (uint64_t)(P->name_cap - 1);
  }
  return -1;
}

static void name_insert(OProg* P, const char* s, int slot) {
  if (2 * (P->name_cnt + 1) > P->name_cap) {
    int oc = P->name_cap; char** on = P->names; int* os = P->name_slot;
    P->name_cap = oc ? oc * 2 : 64;
    P->names = calloc((size_t)P->name_cap, sizeof(char*));
    P->name_slot = calloc((size_t)P->name_cap, sizeof(int));
    P->name_cnt = 0;
    for (int i = 0; i < oc; i++) if (on[i]) { name_insert(P, on[i], os[i]); free(on[i]); }
    free(on); free(os);
  }
  uint64_t h = hash_str(s) & (uint64_t)(P->name_cap - 1);
  while (P->names[h]) h = (h + 1) & (uint64_t)(P->name_cap - 1);
  P->names[h] = strdup(s); P->name_slot[h] = slot; P->name_cnt++;
}

/* ------------------------------------------------------------- parser */
static int p_expr(Lex* L, OProg* P);

static int p_atom(Lex* L, OProg* P) {
  if (L->failed) return -1;
  switch (L->tok) {
    case T_VAR: {
      if (L->ival > 63) { lex_error(L, "variable id %lld > 63", L->ival); return -1; }
      int id = (int)L->ival;
      if (id > P->max_var) P->max_var = id;
      next(L);
      return add_node(P, K_VAR, id, 0);
    }
    case T_ZERO: next(L); return add_node(P, K_CONST, 0, 0);
    case T_ONE:  next(L); return add_node(P, K_CONST, 1, 0);
    case T_NAME: {
      int slot = name_find(P, L->name);
      if (slot < 0) { lex_error(L, "name '%s' used before definition", L->name); return -1; }
      next(L);
      return add_node(P, K_REF, slot, 0);
    }
    case T_LP: {
      next(L);
      int e = p_expr(L, P);
      if (L->failed) return -1;
      if (L->tok != T_RP) { lex_error(L, "expected ')'"); return -1; }
      next(L);
      return e;
    }
    default: lex_error(L, "expected an operand"); return -1;
  }
}

static int p_unary(Lex* L, OProg* P) {
  if (L->tok == T_NOT) { next(L); int c = p_unary(L, P); if (L->failed) return -1; return add_node(P, K_NOT, c, 0); }
  return p_atom(L, P);
}

/* n-ary AND / OR: children collected then stored contiguously in kids[] */
static int p_nary(Lex* L, OProg* P, int tok, int kind, int (*sub)(Lex*, OProg*)) {
  int first = sub(L, P);
  if (L->failed || L->tok != tok) return first;
  int cap = 8, cnt = 0; int* tmp = malloc(sizeof(int) * (size_t)cap);
  tmp[cnt++] = first;
  while (L->tok == tok) {
    next(L);
    int c = sub(L, P);
    if (L->failed) { free(tmp); return -1; }
    if (cnt == cap) { cap *= 2; tmp = realloc(tmp, sizeof(int) * (size_t)cap); }
    tmp[cnt++] = c;
  }
  int id = add_node(P, kind, 0, 0);
  P->kids = grow(P->kids, &P->cap_kids, P->n_kids + cnt, sizeof(int));
  memcpy(P->kids + P->n_kids, tmp, sizeof(int) * (size_t)cnt);
  P->nodes[id].first = P->n_kids; P->nodes[id].cnt = cnt;
  P->n_kids += cnt;
  free(tmp);
  return id;
}

static int p_and(Lex* L, OProg* P) { return p_nary(L, P, T_AND, K_AND, p_unary); }

static int p_xor(Lex* L, OProg* P) {            /* left-assoc binary */
  int a = p_and(L, P);
  while (!L->failed && L->tok == T_XOR) { next(L); int b = p_and(L, P); if (L->failed) return -1; a = add_node(P, K_XOR, a, b); }
  return a;
}

static int p_or(Lex* L, OProg* P) { return p_nary(L, P, T_OR, K_OR, p_xor); }

static int p_imp(Lex* L, OProg* P) {            /* right-assoc */
  int a = p_or(L, P);
  if (L->failed || L->tok != T_IMP) return a;
  next(L);
  int b = p_imp(L, P);
  if (L->failed) return -1;
  return add_node(P, K_IMP, a, b);
}

static int p_expr(Lex* L, OProg* P) {           /* iff: left-assoc */
  int a = p_imp(L, P);
  while (!L->failed && L->tok == T_IFF) { next(L); int b = p_imp(L, P); if (L->failed) return -1; a = add_node(P, K_IFF, a, b); }
  return a;
}

static void define_name(Lex* L, OProg* P, const char* name, int root) {
  if (name_find(P, name) >= 0) { lex_error(L, "name '%s' redefined", name); return; }
  P->let_root = grow(P->let_root, &P->cap_lets, P->n_lets + 1, sizeof(int));
  P->let_root[P->n_lets] = root;
  name_insert(P, name, P->n_lets);
  P->n_lets++;
}

static void add_constraint(OProg* P, int root) {
  P->cons_root = grow(P->cons_root, &P->cap_cons, P->n_cons + 1, sizeof(int));
  P->cons_root[P->n_cons++] = root;
}

static void free_prog(OProg* P) {
  free(P->nodes); free(P->kids); free(P->let_root); free(P->cons_root);
  for (int i = 0; i < P->name_cap; i++) free(P->names[i]);
  free(P->names); free(P->name_slot);
  memset(P, 0, sizeof *P);
}

/* program := { stmt (';' | NEWLINE) } [stmt] */
static int parse_program(const char* text, OProg* P, char* err, size_t errlen) {
  memset(P, 0, sizeof *P);
  P->max_var = -1;
  Lex L; memset(&L, 0, sizeof L);
  L.s = text; L.line = 1; L.col = 1; L.err = err; L.errlen = errlen;
  next(&L);
  while (!L.failed && L.tok != T_EOF) {
    if (L.tok == T_SEP) { next(&L); continue; }
    if (L.tok == T_LET) {
      next(&L);
      if (L.tok != T_NAME) { lex_error(&L, "expected a name after 'let'"); break; }
      char name[256]; strcpy(name, L.name);
      next(&L);
      if (L.tok != T_EQ) { lex_error(&L, "expected '='"); break; }
      next(&L);
      int r = p_expr(&L, P);
      if (L.failed) break;
      define_name(&L, P, name, r);
    } else if (L.tok == T_NAME) {
      /* NAME '=' expr (named constraint) or an expression starting with NAME */
      size_t save_pos = L.pos; int save_line = L.line, save_col = L.col, save_depth = L.depth;
      char name[256]; strcpy(name, L.name);
      int tl = L.tline, tc = L.tcol;
      next(&L);
      if (L.tok == T_EQ) {
        next(&L);
        int r = p_expr(&L, P);
        if (L.failed) break;
        define_name(&L, P, name, r);
        int ref = add_node(P, K_REF, name_find(P, name), 0);
        add_constraint(P, ref);
      } else {
        L.pos = save_pos; L.line = save_line; L.col = save_col; L.depth = save_depth;
        L.tok = T_NAME; strcpy(L.name, name); L.tline = tl; L.tcol = tc;
        int r = p_expr(&L, P);
        if (L.failed) break;
        add_constraint(P, r);
      }
    } else {
      int r = p_expr(&L, P);
      if (L.failed) break;
      add_constraint(P, r);
    }
    if (L.failed) break;
    if (L.tok != T_SEP && L.tok != T_EOF) { lex_error(&L, "expected ';' or end of line"); break; }
  }
  if (L.failed) { free_prog(P); return -1; }
  return 0;
}

/* ------------------------------------------------------------- evaluator */
/* Two-valued semantics, one valuation at a time. */
static int ev(const OProg* P, int i, uint64_t mu, const unsigned char* letval) {
  const ONode* x = &P->nodes[i];
  switch (x->kind) {
    case K_VAR:   return (int)((mu >> x->a) & 1u);
    case K_CONST: return x->a;
    case K_NOT:   return !ev(P, x->a, mu, letval);
    case K_AND:
      for (int k = 0; k < x->cnt; k++) if (!ev(P, P->kids[x->first + k], mu, letval)) return 0;
      return 1;
    case K_OR:
      for (int k = 0; k < x->cnt; k++) if (ev(P, P->kids[x->first + k], mu, letval)) return 1;
      return 0;
    case K_XOR:   return ev(P, x->a, mu, letval) != ev(P, x->b, mu, letval);     /* x+y */
    case K_IMP:   return !ev(P, x->a, mu, letval) || ev(P, x->b, mu, letval);
    case K_IFF:   return ev(P, x->a, mu, letval) == ev(P, x->b, mu, letval);
    case K_REF:   return letval[x->a];
  }
  return 0;
}

/* f(mu): lets in order, then the conjunction of the constraints. */
static int eval_mu(const OProg* P, uint64_t mu, unsigned char* letval) {
  for (int k = 0; k < P->n_lets; k++) letval[k] = (unsigned char)ev(P, P->let_root[k], mu, letval);
  for (int k = 0; k < P->n_cons; k++) if (!ev(P, P->cons_root[k], mu, letval)) return 0;
  return 1;   /* empty program: no constraints -> constant 1 */
}

typedef struct {
  const OProg* P;
  uint64_t lo, hi;          /* valuation range */
  uint64_t* out;            /* nullable; bit (mu-lo) */
  uint64_t block;           /* valuations per work item (multiple of 64) */
  uint64_t n_blocks;
  uint64_t next_block;      /* shared counter */
  pthread_mutex_t mu_lock;
  uint64_t count;
} Job;

static void* worker(void* arg) {
  Job* J = (Job*)arg;
  unsigned char* letval = malloc((size_t)(J->P->n_lets > 0 ? J->P->n_lets : 1));
  uint64_t local = 0;
  for (;;) {
    pthread_mutex_lock(&J->mu_lock);
    uint64_t b = J->next_block++;
    pthread_mutex_unlock(&J->mu_lock);
    if (b >= J->n_blocks) break;
    uint64_t s = J->lo + b * J->block;
    uint64_t e = s + J->block; if (e > J->hi || e < s) e = J->hi;
    for (uint64_t mu = s; mu < e; mu++) {
      if (eval_mu(J->P, mu, letval)) {
        local++;
        if (J->out) J->out[(mu - J->lo) >> 6] |= 1ull << ((mu - J->lo) & 63);
      }
    }
  }
  pthread_mutex_lock(&J->mu_lock);
  J->count += local;
  pthread_mutex_unlock(&J->mu_lock);
  free(letval);
  return NULL;
}

/* ---------------------------------------------------------------- API */
/* Parse only.  Returns 0 and the largest variable id (-1 if none), or -1
 * with "line:col: message" in err. */
int bfa_oracle_parse(const char* text, int* max_var_id, int* n_lets, int* n_constraints,
                     char* err, size_t errlen) {
  OProg P;
  if (!text) return -2;
  if (parse_program(text, &P, err, errlen) != 0) return -1;
  if (max_var_id) *max_var_id = P.max_var;
  if (n_lets) *n_lets = P.n_lets;
  if (n_constraints) *n_constraints = P.n_cons;
  free_prog(&P);
  return 0;
}

/* Evaluate f on every valuation mu in [mu_lo, mu_hi) of n variables.
 *   out_words: nullable; if given, ceil((mu_hi-mu_lo)/64) u64 words, zeroed
 *              here; bit (mu-mu_lo) at word (mu-mu_lo)>>6, bit (mu-mu_lo)&63.
 *   count:     number of mu with f(mu) = 1.
 *   threads:   worker threads (<=0: 1).
 * Returns 0, -1 parse error, -2 bad argument, -3 range error
 * (n > 63, a variable id >= n, mu_hi > 2^n or mu_lo > mu_hi). */
int bfa_oracle_eval(const char* text, int n, uint64_t mu_lo, uint64_t mu_hi,
                    uint64_t* out_words, uint64_t* count, int threads,
                    char* err, size_t errlen) {
  if (!text || !count) return -2;
  if (n < 0 || n > 63) { if (err && errlen) snprintf(err, errlen, "n=%d out of range [0,63]", n); return -3; }
  OProg P;
  if (parse_program(text, &P, err, errlen) != 0) return -1;
  if (P.max_var >= n) {
    if (err && errlen) snprintf(err, errlen, "variable x%d needs n > %d", P.max_var, P.max_var);
    free_prog(&P); return -3;
  }
  uint64_t full = 1ull << n;
  if (mu_lo > mu_hi || mu_hi > full) {
    if (err && errlen) snprintf(err, errlen, "bad valuation range");
    free_prog(&P); return -3;
  }
  if (out_words) memset(out_words, 0, (size_t)((mu_hi - mu_lo + 63) / 64) * 8);
  if (threads <= 0) threads = 1;
  Job J; memset(&J, 0, sizeof J);
  J.P = &P; J.lo = mu_lo; J.hi = mu_hi; J.out = out_words;
  uint64_t len = mu_hi - mu_lo;
  J.block = 1ull << 16;
  while (J.block > 64 && len / J.block < (uint64_t)threads * 8) J.block >>= 1;
  J.n_blocks = (len + J.block - 1) / J.block;
  pthread_mutex_init(&J.mu_lock, NULL);
  if (threads == 1 || J.n_blocks <= 1) {
    worker(&J);
  } else {
    pthread_t* th = malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; t++) pthread_create(&th[t], NULL, worker, &J);
    for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    free(th);
  }
  pthread_mutex_destroy(&J.mu_lock);
  *count = J.count;
  free_prog(&P);
  return 0;
}

#ifdef BFA_ORACLE_MAIN
/* bfa_oracle N file [lo hi] [threads] -- prints count */
int main(int argc, char** argv) {
  if (argc < 3) { fprintf(stderr, "usage: %s N file.bfa [lo hi] [threads]\n", argv[0]); return 1; }
  int n = atoi(argv[1]);
  FILE* f = fopen(argv[2], "rb");
  if (!f) { perror(argv[2]); return 1; }
  fseek(f, 0, SEEK_END); long sz = ftell(f); fseek(f, 0, SEEK_SET);
  char* text = malloc((size_t)sz + 1);
  if (fread(text, 1, (size_t)sz, f) != (size_t)sz) { fclose(f); return 1; }
  text[sz] = 0; fclose(f);
  uint64_t lo = 0, hi = 1ull << n;
  if (argc >= 5) { lo = strtoull(argv[3], NULL, 0); hi = strtoull(argv[4], NULL, 0); }
  int threads = argc >= 6 ? atoi(argv[5]) : 1;
  char err[512]; uint64_t c = 0;
  int rc = bfa_oracle_eval(text, n, lo, hi, NULL, &c, threads, err, sizeof err);
  if (rc) { fprintf(stderr, "error %d: %s\n", rc, err); return 2; }
  printf("%llu\n", (unsigned long long)c);
  free(text);
  return 0;
}
#endif
