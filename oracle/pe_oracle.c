/*
 * ORACLE / TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference polyeval hot path, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER. It
 * is never linked into, called by, or a fallback for the product library.
 *
 * Parity pinning: checked against (1) the reference's own known answers and
 * DOT goldens (tests/golden/, tests/test_oracle.py) and (2) the unmodified
 * reference compiled from /root/reference into oracle/_ref/ (tests/
 * test_oracle.py::test_oracle_matches_reference_*), bit-exact in every domain.
 *
 * Each function names the reference code it restates (paths relative to
 * /root/reference/proj/core).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ODOM_DOUBLE 0
#define ODOM_INTERVAL 1
#define ODOM_INT64 2

typedef struct {
  double lo, hi;
} oiv;

typedef struct otree otree;

typedef struct {
  double cf;       /* fp64 coefficient */
  int64_t ci;      /* int64 coefficient */
  otree* sub;      /* nested coefficient tree (multivariate), or NULL */
  uint32_t pd;     /* partial degree */
  uint32_t* ch;    /* children (node indices) */
  uint32_t nch, cap;
  uint32_t lh;     /* lazy height */
  int64_t parent;  /* -1 for the root */
} onode;

struct otree {
  onode* nodes;
  size_t n;
  uint32_t var;
};

typedef struct {
  uint32_t exp; /* exponent in the variable being built */
  double cf;
  int64_t ci;
  otree* sub;
} oproto;

typedef struct {
  int upper, lower;
  uint64_t cutoff;
} oscheme;

static int g_int; /* coefficient type of the polynomial being built */
static char g_err[256];

/* ---- schemes: src/scheme.cpp:10-34 ---- */
static uint64_t bit_floor64(uint64_t k) {
  uint64_t r = 1;
  while (r <= k / 2) r <<= 1;
  return k ? r : 0;
}
static uint64_t split_builtin(int id, uint64_t k) {
  switch (id) {
    case 0: return k;             /* direct */
    case 1: return 1;             /* horner */
    case 2: return bit_floor64(k); /* estrin */
    default: return (k + 1) / 2;  /* balanced, D1: ceil(k/2) */
  }
}
static uint64_t split(const oscheme* s, uint64_t k) {
  if (s->cutoff == 0) return split_builtin(s->upper, k);
  return k > s->cutoff ? split_builtin(s->upper, k) : split_builtin(s->lower, k);
}

/* ---- tree build: src/tree.cpp:30-95 ---- */
static void add_child(onode* n, uint32_t c) {
  if (n->nch == n->cap) {
    n->cap = n->cap ? 2 * n->cap : 2;
    n->ch = (uint32_t*)realloc(n->ch, n->cap * sizeof(uint32_t));
  }
  n->ch[n->nch++] = c;
}

static int build_range(const oscheme* s, oproto* t, onode* nodes, size_t first, size_t last,
                       uint32_t shift, uint32_t* root) {
  if (last - first == 1) {
    onode* nd = &nodes[first];
    nd->cf = t[first].cf;
    nd->ci = t[first].ci;
    nd->sub = t[first].sub;
    t[first].sub = NULL;
    nd->pd = t[first].exp - shift;
    *root = (uint32_t)first;
    return 0;
  }
  uint32_t degree = t[first].exp - shift;
  uint64_t e64 = split(s, degree);
  if (e64 == 0 || e64 > degree) {
    snprintf(g_err, sizeof g_err, "scheme split left the range (0, k] at k=%u", degree);
    return 1;
  }
  uint32_t e = (uint32_t)e64, threshold = shift + e;
  size_t mid = first; /* first index with exponent < threshold (lower_bound) */
  {
    size_t lo = first, hi = last;
    while (lo < hi) {
      size_t m = lo + (hi - lo) / 2;
      if (t[m].exp >= threshold) lo = m + 1; else hi = m;
    }
    mid = lo;
  }
  if (mid == last) { /* zero remainder absorbs e (tree.cpp:57-63) */
    uint32_t top;
    if (build_range(s, t, nodes, first, last, shift + e, &top)) return 1;
    nodes[top].pd += e;
    *root = top;
    return 0;
  }
  uint32_t upper, lower;
  if (build_range(s, t, nodes, first, mid, shift + e, &upper)) return 1;
  if (build_range(s, t, nodes, mid, last, shift, &lower)) return 1;
  nodes[upper].pd += e - nodes[lower].pd; /* D5, tree.cpp:66-69 */
  add_child(&nodes[lower], upper);
  *root = lower;
  return 0;
}

static otree* tree_from_proto(oproto* t, size_t n, const oscheme* s, uint32_t var) {
  otree* tr = (otree*)calloc(1, sizeof(otree));
  tr->var = var;
  tr->n = n;
  tr->nodes = (onode*)calloc(n, sizeof(onode));
  for (size_t i = 0; i < n; ++i) tr->nodes[i].parent = -1;
  uint32_t root;
  if (build_range(s, t, tr->nodes, 0, n, 0, &root)) return NULL;
  for (size_t i = 0; i < n; ++i) { /* reverse children, set parents (tree.cpp:87-93) */
    onode* nd = &tr->nodes[i];
    for (uint32_t a = 0, b = nd->nch ? nd->nch - 1 : 0; a < b; ++a, --b) {
      uint32_t x = nd->ch[a];
      nd->ch[a] = nd->ch[b];
      nd->ch[b] = x;
    }
    for (uint32_t c = 0; c < nd->nch; ++c) tr->nodes[nd->ch[c]].parent = (int64_t)i;
  }
  return tr;
}

static void free_tree(otree* t) {
  if (!t) return;
  for (size_t i = 0; i < t->n; ++i) {
    free(t->nodes[i].ch);
    free_tree(t->nodes[i].sub);
  }
  free(t->nodes);
  free(t);
}

/* ---- canonical terms: src/polynomial.cpp:13-33 ---- */
typedef struct {
  double cf;
  int64_t ci;
  uint32_t* e;
} oterm;

static uint32_t g_nv;
static int term_cmp(const void* a, const void* b) { /* decreasing lexicographic */
  const oterm* x = (const oterm*)a;
  const oterm* y = (const oterm*)b;
  for (uint32_t v = 0; v < g_nv; ++v) {
    if (x->e[v] != y->e[v]) return x->e[v] > y->e[v] ? -1 : 1;
  }
  return 0;
}

static int coef_zero(const oterm* t) { return g_int ? t->ci == 0 : t->cf == 0.0; }

/* sorts, merges like terms (stable w.r.t. input order), drops zeros; returns new count */
static size_t canonicalize(oterm* t, size_t n, uint32_t nv) {
  g_nv = nv;
  /* stable: insertion-merge sort via qsort on (exps, index) */
  for (size_t i = 1; i < n; ++i) { /* insertion sort keeps stability; n is modest */
    oterm x = t[i];
    size_t j = i;
    while (j > 0 && term_cmp(&t[j - 1], &x) > 0) {
      t[j] = t[j - 1];
      --j;
    }
    t[j] = x;
  }
  size_t m = 0;
  for (size_t i = 0; i < n; ++i) {
    if (m > 0 && term_cmp(&t[m - 1], &t[i]) == 0) {
      if (g_int) t[m - 1].ci += t[i].ci; else t[m - 1].cf += t[i].cf;
      if (coef_zero(&t[m - 1])) --m;
    } else if (!coef_zero(&t[i])) {
      t[m++] = t[i];
    }
  }
  return m;
}

/* ---- multivariate: src/tree.cpp:111-200 ---- */
static otree* build_multi_at(oterm* t, size_t n, uint32_t nv, uint32_t depth,
                             const oscheme* schemes);

static otree* zero_tree(uint32_t var) {
  otree* tr = (otree*)calloc(1, sizeof(otree));
  tr->var = var;
  tr->n = 1;
  tr->nodes = (onode*)calloc(1, sizeof(onode));
  tr->nodes[0].parent = -1;
  return tr;
}

static otree* build_multi_at(oterm* t, size_t n, uint32_t nv, uint32_t depth,
                             const oscheme* schemes) {
  if (n == 0) return zero_tree(depth);
  /* terms arrive canonical (decreasing lex) so groups by exponents[depth]
   * are NOT contiguous in general; collect distinct exponents descending */
  uint32_t* ex = (uint32_t*)malloc(n * sizeof(uint32_t));
  size_t nex = 0;
  for (size_t i = 0; i < n; ++i) {
    size_t j;
    for (j = 0; j < nex && ex[j] != t[i].e[depth]; ++j) {}
    if (j == nex) ex[nex++] = t[i].e[depth];
  }
  for (size_t i = 1; i < nex; ++i) { /* descending */
    uint32_t x = ex[i];
    size_t j = i;
    while (j > 0 && ex[j - 1] < x) { ex[j] = ex[j - 1]; --j; }
    ex[j] = x;
  }
  oproto* pr = (oproto*)calloc(nex, sizeof(oproto));
  oterm* g = (oterm*)malloc(n * sizeof(oterm));
  for (size_t k = 0; k < nex; ++k) {
    size_t m = 0;
    for (size_t i = 0; i < n; ++i) {
      if (t[i].e[depth] != ex[k]) continue;
      g[m] = t[i];
      g[m].e = (uint32_t*)malloc(nv * sizeof(uint32_t));
      memcpy(g[m].e, t[i].e, nv * sizeof(uint32_t));
      g[m].e[depth] = 0;
      ++m;
    }
    uint32_t** gown = (uint32_t**)malloc((m ? m : 1) * sizeof(uint32_t*));
    const size_t graw = m;
    for (size_t i = 0; i < m; ++i) gown[i] = g[i].e;
    m = canonicalize(g, m, nv);
    pr[k].exp = ex[k];
    int constant = m == 0;
    if (m == 1) {
      constant = 1;
      for (uint32_t v = 0; v < nv; ++v) constant &= g[0].e[v] == 0;
    }
    if (constant) {
      pr[k].cf = m ? g[0].cf : 0.0;
      pr[k].ci = m ? g[0].ci : 0;
    } else {
      pr[k].sub = build_multi_at(g, m, nv, depth + 1, schemes);
      if (!pr[k].sub) return NULL;
    }
    for (size_t i = 0; i < graw; ++i) free(gown[i]);
    free(gown);
  }
  free(g);
  otree* tr = tree_from_proto(pr, nex, &schemes[depth], depth);
  free(pr);
  free(ex);
  return tr;
}

/* ---- lazy heights with subtree usage: src/tree.cpp:202-227 (D2) ---- */
static void lazy_heights(otree* tr) {
  uint32_t* usage = (uint32_t*)calloc(tr->n, sizeof(uint32_t));
  for (size_t i = 0; i < tr->n; ++i) {
    onode* nd = &tr->nodes[i];
    if (nd->sub) lazy_heights(nd->sub);
    if (nd->nch <= 1) {
      nd->lh = 0;
    } else {
      uint32_t h = 0;
      for (uint32_t c = 1; c < nd->nch; ++c) if (usage[nd->ch[c]] > h) h = usage[nd->ch[c]];
      nd->lh = h + 1;
    }
    usage[i] = nd->lh;
    if (nd->nch && usage[nd->ch[0]] > usage[i]) usage[i] = usage[nd->ch[0]];
  }
  free(usage);
}

static uint32_t max_lh(const otree* tr) {
  uint32_t m = 0;
  for (size_t i = 0; i < tr->n; ++i) {
    if (tr->nodes[i].lh > m) m = tr->nodes[i].lh;
  }
  return m;
}

/* ---- interval primitives: src/interval.cpp:12-52 ---- */
static double endpoint_product(double a, double b) { return (a == 0.0 || b == 0.0) ? 0.0 : a * b; }
static oiv iv_add(oiv a, oiv b) {
  oiv o = {nextafter(a.lo + b.lo, -INFINITY), nextafter(a.hi + b.hi, INFINITY)};
  return o;
}
static oiv iv_mul(oiv a, oiv b) {
  double p[4] = {endpoint_product(a.lo, b.lo), endpoint_product(a.lo, b.hi),
                 endpoint_product(a.hi, b.lo), endpoint_product(a.hi, b.hi)};
  double mn = p[0], mx = p[0]; /* std::min / std::max initializer-list scan */
  for (int i = 1; i < 4; ++i) {
    if (p[i] < mn) mn = p[i];
    if (mx < p[i]) mx = p[i];
  }
  oiv o = {nextafter(mn, -INFINITY), nextafter(mx, INFINITY)};
  return o;
}

/* ---- generic value ---- */
typedef struct {
  double d;
  oiv iv;
  int64_t i;
} oval;

static int g_dom;
static int g_overflow;

static oval v_zero(void) { oval z; memset(&z, 0, sizeof z); return z; }
static oval v_add(oval a, oval b) {
  oval o = v_zero();
  if (g_dom == ODOM_DOUBLE) o.d = a.d + b.d;
  else if (g_dom == ODOM_INTERVAL) o.iv = iv_add(a.iv, b.iv);
  else if (__builtin_add_overflow(a.i, b.i, &o.i)) g_overflow = 1;
  return o;
}
static oval v_mul(oval a, oval b) {
  oval o = v_zero();
  if (g_dom == ODOM_DOUBLE) o.d = a.d * b.d;
  else if (g_dom == ODOM_INTERVAL) o.iv = iv_mul(a.iv, b.iv);
  else if (__builtin_mul_overflow(a.i, b.i, &o.i)) g_overflow = 1;
  return o;
}
/* from_integer: ring.hpp:40-48 (double), numeric.cpp:17-26 (interval) */
static oval v_coef(const onode* nd) {
  oval o = v_zero();
  if (g_dom == ODOM_INT64) {
    o.i = nd->ci;
  } else if (g_int) {
    double d = (double)nd->ci; /* RN-even */
    if (g_dom == ODOM_DOUBLE) {
      o.d = d;
    } else {
      int exact = d < 9223372036854775808.0 && d >= -9223372036854775808.0 && (int64_t)d == nd->ci;
      o.iv.lo = exact ? d : nextafter(d, -INFINITY);
      o.iv.hi = exact ? d : nextafter(d, INFINITY);
    }
  } else {
    o.d = nd->cf;
    o.iv.lo = o.iv.hi = nd->cf;
  }
  return o;
}

/* ---- power tables: include/polyeval/powers.hpp:50-72 (memoized halving) ---- */
typedef struct {
  oval* val;
  unsigned char* have;
  uint32_t max;
} opow;

static void pow_ensure(opow* t, uint32_t e) {
  if (t->have[e]) return;
  uint32_t h = e / 2;
  pow_ensure(t, h);
  pow_ensure(t, e - h);
  t->val[e] = v_mul(t->val[h], t->val[e - h]);
  t->have[e] = 1;
}

/* ---- the walk: include/polyeval/eval.hpp:208-249 ---- */
static oval walk(const otree* tr, opow* tables, oval* regs_pool, size_t pool_off) {
  uint32_t nregs = max_lh(tr) + 1;
  oval* m = regs_pool + pool_off;
  for (uint32_t r = 0; r < nregs; ++r) m[r] = v_zero();
  for (size_t i = 0; i < tr->n; ++i) {
    const onode* nd = &tr->nodes[i];
    oval v = nd->sub ? walk(nd->sub, tables, regs_pool, pool_off + nregs) : v_coef(nd);
    if (nd->nch) { /* reads_register */
      v = v_add(m[nd->lh], v);
      m[nd->lh] = v_zero();
    }
    if (nd->pd) {
      pow_ensure(&tables[tr->var], nd->pd);
      v = v_mul(v, tables[tr->var].val[nd->pd]);
    }
    if (i + 1 == tr->n) return v;
    uint32_t ps = tr->nodes[nd->parent].lh;
    m[ps] = v_add(m[ps], v);
  }
  return v_zero();
}

static uint32_t max_pd(const otree* tr, uint32_t var) {
  uint32_t m = 0;
  for (size_t i = 0; i < tr->n; ++i) {
    if (tr->var == var && tr->nodes[i].pd > m) m = tr->nodes[i].pd;
    if (tr->nodes[i].sub) {
      uint32_t s = max_pd(tr->nodes[i].sub, var);
      if (s > m) m = s;
    }
  }
  return m;
}

static size_t depth_regs(const otree* tr) {
  size_t best = 0;
  for (size_t i = 0; i < tr->n; ++i) {
    if (tr->nodes[i].sub) {
      size_t s = depth_regs(tr->nodes[i].sub);
      if (s > best) best = s;
    }
  }
  return max_lh(tr) + 1 + best;
}

/* ---------------------------------------------------------------- API */

typedef struct {
  otree* tree;
  uint32_t nvars;
  int integer;
} oprog;

const char* oracle_last_error(void) { return g_err; }

void* oracle_create(const uint32_t* exps, const void* coeffs, size_t nterms, uint32_t nvars,
                    const int* upper, const int* lower, const uint64_t* cutoff, int coeff_is_int) {
  g_err[0] = 0;
  g_int = coeff_is_int;
  oscheme* sch = (oscheme*)malloc(nvars * sizeof(oscheme));
  for (uint32_t v = 0; v < nvars; ++v) {
    sch[v].upper = upper[v];
    sch[v].lower = lower[v];
    sch[v].cutoff = cutoff[v];
  }
  oterm* t = (oterm*)malloc((nterms ? nterms : 1) * sizeof(oterm));
  for (size_t i = 0; i < nterms; ++i) {
    t[i].cf = coeff_is_int ? 0.0 : ((const double*)coeffs)[i];
    t[i].ci = coeff_is_int ? ((const int64_t*)coeffs)[i] : 0;
    t[i].e = (uint32_t*)malloc(nvars * sizeof(uint32_t));
    memcpy(t[i].e, exps + i * nvars, nvars * sizeof(uint32_t));
  }
  uint32_t** owned = (uint32_t**)malloc((nterms ? nterms : 1) * sizeof(uint32_t*));
  for (size_t i = 0; i < nterms; ++i) owned[i] = t[i].e; /* canonicalize permutes/merges */
  size_t n = canonicalize(t, nterms, nvars);
  otree* tr;
  if (nvars == 1) {
    /* build(): src/tree.cpp:159-181 */
    if (n == 0) {
      tr = zero_tree(0);
    } else {
      oproto* pr = (oproto*)calloc(n, sizeof(oproto));
      for (size_t i = 0; i < n; ++i) {
        pr[i].exp = t[i].e[0];
        pr[i].cf = t[i].cf;
        pr[i].ci = t[i].ci;
      }
      tr = tree_from_proto(pr, n, &sch[0], 0);
      free(pr);
    }
  } else {
    int constant = n == 0;
    if (n == 1) {
      constant = 1;
      for (uint32_t v = 0; v < nvars; ++v) constant &= t[0].e[v] == 0;
    }
    if (n == 0) {
      tr = zero_tree(0);
    } else if (constant) { /* tree.cpp:189-198 */
      oproto pr = {0, t[0].cf, t[0].ci, NULL};
      tr = tree_from_proto(&pr, 1, &sch[0], 0);
    } else {
      tr = build_multi_at(t, n, nvars, 0, sch);
    }
  }
  for (size_t i = 0; i < nterms; ++i) free(owned[i]);
  free(owned);
  free(t);
  free(sch);
  if (!tr) return NULL;
  lazy_heights(tr);
  oprog* p = (oprog*)calloc(1, sizeof(oprog));
  p->tree = tr;
  p->nvars = nvars;
  p->integer = coeff_is_int;
  return p;
}

void oracle_destroy(void* h) {
  oprog* p = (oprog*)h;
  if (!p) return;
  free_tree(p->tree);
  free(p);
}

/* domain: 0 double, 1 interval, 2 int64. in0/out0: values (double or int64)
 * or interval lo; in1/out1: interval hi. Returns 0, or 2 on int64 overflow. */
int oracle_eval(void* h, int domain, const void* const* in0, const void* const* in1, size_t n,
                void* out0, void* out1) {
  oprog* p = (oprog*)h;
  g_int = p->integer;
  g_dom = domain;
  g_overflow = 0;
  opow* tables = (opow*)calloc(p->nvars, sizeof(opow));
  for (uint32_t v = 0; v < p->nvars; ++v) {
    tables[v].max = max_pd(p->tree, v);
    tables[v].val = (oval*)calloc(tables[v].max + 2, sizeof(oval));
    tables[v].have = (unsigned char*)calloc(tables[v].max + 2, 1);
  }
  oval* regs = (oval*)calloc(depth_regs(p->tree) + 1, sizeof(oval));
  for (size_t i = 0; i < n; ++i) {
    for (uint32_t v = 0; v < p->nvars; ++v) { /* fresh table per point (eval.hpp:185-206) */
      memset(tables[v].have, 0, tables[v].max + 2);
      oval x = v_zero();
      if (domain == ODOM_DOUBLE) x.d = ((const double*)in0[v])[i];
      else if (domain == ODOM_INTERVAL) {
        x.iv.lo = ((const double*)in0[v])[i];
        x.iv.hi = ((const double*)in1[v])[i];
      } else x.i = ((const int64_t*)in0[v])[i];
      tables[v].val[1] = x;
      tables[v].have[1] = 1;
    }
    oval r = walk(p->tree, tables, regs, 0);
    if (domain == ODOM_DOUBLE) ((double*)out0)[i] = r.d;
    else if (domain == ODOM_INTERVAL) {
      ((double*)out0)[i] = r.iv.lo;
      ((double*)out1)[i] = r.iv.hi;
    } else ((int64_t*)out0)[i] = r.i;
  }
  for (uint32_t v = 0; v < p->nvars; ++v) {
    free(tables[v].val);
    free(tables[v].have);
  }
  free(tables);
  free(regs);
  return g_overflow ? 2 : 0;
}

/* sum over terms of |c_t| * prod |x_v|^a_tv at each point (the fp64
 * tolerance scale of the north star): out[i] */
int oracle_abs_term_sum(const uint32_t* exps, const double* coeffs, size_t nterms, uint32_t nvars,
                        const double* const* coords, size_t n, double* out) {
  for (size_t i = 0; i < n; ++i) {
    long double s = 0;
    for (size_t t = 0; t < nterms; ++t) {
      long double term = fabsl((long double)coeffs[t]);
      for (uint32_t v = 0; v < nvars; ++v) {
        long double x = fabsl((long double)coords[v][i]);
        uint32_t e = exps[t * nvars + v];
        long double pw = 1;
        while (e) {
          if (e & 1) pw *= x;
          x *= x;
          e >>= 1;
        }
        term *= pw;
      }
      s += term;
    }
    out[i] = (double)s;
  }
  return 0;
}

/* records x 5 of the root program in compile() layout (src/eval.cpp:17-48) */
int oracle_records(void* h, int32_t* out, size_t cap, size_t* count, uint32_t* register_count) {
  oprog* p = (oprog*)h;
  otree* tr = p->tree;
  /* exponent set of the root variable: all nonzero partial degrees of trees
   * over that variable, nested ones included (eval.cpp:8-15) */
  uint32_t mx = max_pd(tr, tr->var);
  unsigned char* present = (unsigned char*)calloc(mx + 2, 1);
  /* collect */
  size_t stack_cap = 64, sp = 0;
  const otree** st = (const otree**)malloc(stack_cap * sizeof(otree*));
  st[sp++] = tr;
  while (sp) {
    const otree* t = st[--sp];
    for (size_t i = 0; i < t->n; ++i) {
      if (t->var == tr->var && t->nodes[i].pd) present[t->nodes[i].pd] = 1;
      if (t->nodes[i].sub) {
        if (sp == stack_cap) {
          stack_cap *= 2;
          st = (const otree**)realloc(st, stack_cap * sizeof(otree*));
        }
        st[sp++] = t->nodes[i].sub;
      }
    }
  }
  free(st);
  uint32_t* slot = (uint32_t*)calloc(mx + 2, sizeof(uint32_t));
  uint32_t k = 0;
  for (uint32_t e = 1; e <= mx; ++e) if (present[e]) slot[e] = k++;
  *count = tr->n;
  *register_count = max_lh(tr) + 1;
  for (size_t i = 0; i < tr->n && (i + 1) * 5 <= cap; ++i) {
    const onode* nd = &tr->nodes[i];
    out[5 * i] = nd->pd ? (int32_t)slot[nd->pd] : -1;
    out[5 * i + 1] = (int32_t)nd->lh;
    out[5 * i + 2] = nd->parent >= 0 ? (int32_t)tr->nodes[nd->parent].lh : -1;
    out[5 * i + 3] = nd->nch ? 1 : 0;
    out[5 * i + 4] = nd->sub ? 1 : 0;
  }
  free(present);
  free(slot);
  return 0;
}

/* DOT of a univariate (or multivariate with scalar-only root) tree with
 * integer coefficients, reference to_dot (src/tree.cpp:290-309). */
int oracle_dot(void* h, char* buf, size_t cap, size_t* len) {
  oprog* p = (oprog*)h;
  otree* tr = p->tree;
  size_t used = 0;
  char line[160];
#define EMIT(...)                                                  \
  do {                                                             \
    int k_ = snprintf(line, sizeof line, __VA_ARGS__);             \
    if (buf && used + (size_t)k_ < cap) memcpy(buf + used, line, k_); \
    used += (size_t)k_;                                            \
  } while (0)
  EMIT("digraph evaluation_tree {\n");
  for (size_t i = 0; i < tr->n; ++i) {
    const onode* nd = &tr->nodes[i];
    if (nd->sub) return 1; /* nested labels need the renderer; not used by goldens */
    if (p->integer) EMIT("  n%zu [label=\"c=%lld d=%u lh=%u\"];\n", i, (long long)nd->ci, nd->pd, nd->lh);
    else EMIT("  n%zu [label=\"c=%.17g d=%u lh=%u\"];\n", i, nd->cf, nd->pd, nd->lh);
  }
  for (size_t i = 0; i < tr->n; ++i) {
    for (uint32_t c = 0; c < tr->nodes[i].nch; ++c) EMIT("  n%zu -> n%u;\n", i, tr->nodes[i].ch[c]);
  }
  EMIT("}\n");
#undef EMIT
  if (buf && cap) buf[used < cap ? used : cap - 1] = 0;
  *len = used;
  return 0;
}
