/*
 * bp_oracle.c -- TEST INFRASTRUCTURE ONLY (see bp_oracle.h).
 *
 * Plain-C, fp64 restatement of the reference bpsched hot path.  Each function
 * cites the reference file:line it restates (paths relative to
 * /root/reference/proj/core).  Floating-point operations are issued in the
 * reference's order so results match the reference bit for bit when both are
 * compiled with -ffp-contract=off.
 */
#define _GNU_SOURCE
#include "bp_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------ */
/* errors (errors.hpp:10-38 -> return codes)                                 */

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* mt19937_64 (std::mt19937_64) and uniform_unit (rng.hpp:11-13)             */

#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t mt[MT_N];
  int idx;
} mt64;

static void mt_seed(mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
}

static uint64_t mt_next(mt64* r) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  if (r->idx >= MT_N) {
    int i;
    for (i = 0; i < MT_N - MT_M; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    for (; i < MT_N - 1; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    uint64_t x = (r->mt[MT_N - 1] & UM) | (r->mt[0] & LM);
    r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

static double uniform_unit(mt64* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }

void orc_mt_draws(uint64_t seed, uint64_t count, uint64_t* out_raw, double* out_unit) {
  mt64 r;
  mt_seed(&r, seed);
  for (uint64_t i = 0; i < count; ++i) {
    uint64_t x = mt_next(&r);
    if (out_raw) out_raw[i] = x;
    if (out_unit) out_unit[i] = (double)(x >> 11) * 0x1.0p-53;
  }
}

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------------------ */
/* graph (mrf.hpp:31-87, mrf.cpp:25-106)                                     */

struct orc_graph {
  uint32_t V, E, D, maxq;
  uint32_t* card;
  size_t* uoff;
  double* unary;
  uint32_t* ep; /* 2E: (i, j) */
  size_t* poff;
  double* table;
  uint32_t* dsrc;
  uint32_t* dtgt;
  size_t* aoff; /* V+1 */
  uint32_t* adj;
};

void orc_graph_destroy(orc_graph* g) {
  if (!g) return;
  free(g->card);
  free(g->uoff);
  free(g->unary);
  free(g->ep);
  free(g->poff);
  free(g->table);
  free(g->dsrc);
  free(g->dtgt);
  free(g->aoff);
  free(g->adj);
  free(g);
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* check_positive_table (mrf.cpp:15-21) */
static int positive_finite(const double* t, size_t n) {
  for (size_t k = 0; k < n; ++k)
    if (!(t[k] > 0.0) || !isfinite(t[k])) return 0;
  return 1;
}

int orc_graph_create(uint32_t V, const uint32_t* cards, const double* unary, uint32_t E,
                     const uint32_t* ep, const double* tables, orc_graph** out) {
  *out = NULL;
  orc_graph* g = (orc_graph*)calloc(1, sizeof *g);
  if (!g) return fail(ORC_NOMEM, "out of memory");
  g->V = V;
  g->E = E;
  g->D = 2 * E;
  g->card = (uint32_t*)malloc(sizeof(uint32_t) * (V ? V : 1));
  g->uoff = (size_t*)malloc(sizeof(size_t) * (V + 1));
  g->uoff[0] = 0;
  for (uint32_t v = 0; v < V; ++v) {
    if (cards[v] == 0) {
      orc_graph_destroy(g);
      return fail(ORC_MODEL, "vertex %u has cardinality 0", v);
    }
    g->card[v] = cards[v];
    g->uoff[v + 1] = g->uoff[v] + cards[v];
    if (cards[v] > g->maxq) g->maxq = cards[v];
  }
  g->unary = (double*)malloc(sizeof(double) * (g->uoff[V] ? g->uoff[V] : 1));
  memcpy(g->unary, unary, sizeof(double) * g->uoff[V]);
  for (uint32_t v = 0; v < V; ++v) {
    if (!positive_finite(g->unary + g->uoff[v], cards[v])) {
      orc_graph_destroy(g);
      return fail(ORC_MODEL, "unary(%u) entries must be strictly positive and finite", v);
    }
  }
  /* mrf.cpp:55-91: endpoint checks, duplicates, tables */
  g->ep = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (E ? E : 1));
  g->poff = (size_t*)malloc(sizeof(size_t) * (E + 1));
  g->poff[0] = 0;
  for (uint32_t e = 0; e < E; ++e) {
    uint32_t i = ep[2 * e], j = ep[2 * e + 1];
    if (i >= V || j >= V) {
      orc_graph_destroy(g);
      return fail(ORC_MODEL, "edge %u references a vertex out of range", e);
    }
    if (i == j) {
      orc_graph_destroy(g);
      return fail(ORC_MODEL, "edge %u is a self-loop on vertex %u", e, i);
    }
    if (i > j) {
      orc_graph_destroy(g);
      return fail(ORC_MODEL, "edge %u endpoints must satisfy i < j", e);
    }
    g->ep[2 * e] = i;
    g->ep[2 * e + 1] = j;
    g->poff[e + 1] = g->poff[e] + (size_t)cards[i] * cards[j];
  }
  if (E > 0) {
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * E);
    for (uint32_t e = 0; e < E; ++e) keys[e] = ((uint64_t)g->ep[2 * e] << 32) | g->ep[2 * e + 1];
    qsort(keys, E, sizeof(uint64_t), cmp_u64);
    for (uint32_t e = 1; e < E; ++e) {
      if (keys[e] == keys[e - 1]) {
        uint32_t i = (uint32_t)(keys[e] >> 32), j = (uint32_t)keys[e];
        free(keys);
        orc_graph_destroy(g);
        return fail(ORC_MODEL, "duplicate edge (%u, %u)", i, j);
      }
    }
    free(keys);
  }
  g->table = (double*)malloc(sizeof(double) * (g->poff[E] ? g->poff[E] : 1));
  memcpy(g->table, tables, sizeof(double) * g->poff[E]);
  for (uint32_t e = 0; e < E; ++e) {
    if (!positive_finite(g->table + g->poff[e], g->poff[e + 1] - g->poff[e])) {
      uint32_t i = g->ep[2 * e], j = g->ep[2 * e + 1];
      orc_graph_destroy(g);
      return fail(ORC_MODEL, "pairwise(%u,%u) entries must be strictly positive and finite", i, j);
    }
  }
  /* directed edges 2e (i->j) and 2e+1 (j->i): mrf.cpp:89-90 */
  g->dsrc = (uint32_t*)malloc(sizeof(uint32_t) * (g->D ? g->D : 1));
  g->dtgt = (uint32_t*)malloc(sizeof(uint32_t) * (g->D ? g->D : 1));
  for (uint32_t e = 0; e < E; ++e) {
    g->dsrc[2 * e] = g->ep[2 * e];
    g->dtgt[2 * e] = g->ep[2 * e + 1];
    g->dsrc[2 * e + 1] = g->ep[2 * e + 1];
    g->dtgt[2 * e + 1] = g->ep[2 * e];
  }
  /* CSR of incoming directed edges in edge-id order: mrf.cpp:93-104 */
  g->aoff = (size_t*)calloc(V + 1, sizeof(size_t));
  for (uint32_t d = 0; d < g->D; ++d) g->aoff[g->dtgt[d] + 1]++;
  for (uint32_t v = 0; v < V; ++v) g->aoff[v + 1] += g->aoff[v];
  g->adj = (uint32_t*)malloc(sizeof(uint32_t) * (g->D ? g->D : 1));
  size_t* cursor = (size_t*)malloc(sizeof(size_t) * (V ? V : 1));
  for (uint32_t v = 0; v < V; ++v) cursor[v] = g->aoff[v];
  for (uint32_t d = 0; d < g->D; ++d) g->adj[cursor[g->dtgt[d]]++] = d;
  free(cursor);
  *out = g;
  return ORC_OK;
}

uint32_t orc_graph_num_vertices(const orc_graph* g) { return g->V; }
uint32_t orc_graph_num_edges(const orc_graph* g) { return g->E; }
uint64_t orc_graph_unary_size(const orc_graph* g) { return g->uoff[g->V]; }
uint64_t orc_graph_table_size(const orc_graph* g) { return g->poff[g->E]; }

void orc_graph_export(const orc_graph* g, uint32_t* cards, double* unary, uint32_t* ep,
                      double* tables) {
  if (cards) memcpy(cards, g->card, sizeof(uint32_t) * g->V);
  if (unary) memcpy(unary, g->unary, sizeof(double) * g->uoff[g->V]);
  if (ep) memcpy(ep, g->ep, sizeof(uint32_t) * 2 * g->E);
  if (tables) memcpy(tables, g->table, sizeof(double) * g->poff[g->E]);
}

void orc_graph_incoming(const orc_graph* g, uint64_t* offsets, uint32_t* adjacency) {
  for (uint32_t v = 0; v <= g->V; ++v) offsets[v] = g->aoff[v];
  memcpy(adjacency, g->adj, sizeof(uint32_t) * g->D);
}

/* ------------------------------------------------------------------------ */
/* generators (generators.cpp:9-71) + new Potts / Erdos-Renyi definitions     */

/* unit_open: generators.cpp:9-14 */
static double unit_open(mt64* r) {
  double u = uniform_unit(r);
  while (u == 0.0) u = uniform_unit(r);
  return u;
}

int orc_generate_ising(uint32_t n, double c, uint64_t seed, orc_graph** out) {
  mt64 r;
  mt_seed(&r, seed);
  const uint32_t V = n * n;
  uint32_t* cards = (uint32_t*)malloc(sizeof(uint32_t) * (V ? V : 1));
  double* un = (double*)malloc(sizeof(double) * 2 * (V ? V : 1));
  for (uint32_t v = 0; v < V; ++v) {
    cards[v] = 2;
    un[2 * v] = unit_open(&r); /* generators.cpp:35: {unit_open, unit_open} */
    un[2 * v + 1] = unit_open(&r);
  }
  const uint32_t E = n ? 2 * n * (n - 1) : 0;
  uint32_t* ep = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (E ? E : 1));
  uint32_t e = 0;
  for (uint32_t row = 0; row < n; ++row) /* generators.cpp:37-43 */
    for (uint32_t col = 0; col < n; ++col) {
      const uint32_t v = row * n + col;
      if (col + 1 < n) { ep[2 * e] = v; ep[2 * e + 1] = v + 1; ++e; }
      if (row + 1 < n) { ep[2 * e] = v; ep[2 * e + 1] = v + n; ++e; }
    }
  double* tb = (double*)malloc(sizeof(double) * 4 * (E ? E : 1));
  for (uint32_t k = 0; k < E; ++k) { /* generators.cpp:44-48, ising_edge_table :18-22 */
    const double lambda = uniform_unit(&r) - 0.5;
    const double agree = exp(lambda * c), disagree = exp(-lambda * c);
    tb[4 * k] = agree; tb[4 * k + 1] = disagree; tb[4 * k + 2] = disagree; tb[4 * k + 3] = agree;
  }
  int rc = orc_graph_create(V, cards, un, E, ep, tb, out);
  free(cards); free(un); free(ep); free(tb);
  return rc;
}

int orc_generate_chain(uint32_t n, double c, uint64_t seed, orc_graph** out) {
  mt64 r;
  mt_seed(&r, seed);
  uint32_t* cards = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  double* un = (double*)malloc(sizeof(double) * 2 * (n ? n : 1));
  for (uint32_t v = 0; v < n; ++v) {
    cards[v] = 2;
    un[2 * v] = unit_open(&r);
    un[2 * v + 1] = unit_open(&r);
  }
  const uint32_t E = n > 0 ? n - 1 : 0;
  uint32_t* ep = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (E ? E : 1));
  double* tb = (double*)malloc(sizeof(double) * 4 * (E ? E : 1));
  for (uint32_t v = 0; v + 1 < n; ++v) { /* generators.cpp:63-67 */
    const double lambda = uniform_unit(&r) - 0.5;
    const double agree = exp(lambda * c), disagree = exp(-lambda * c);
    ep[2 * v] = v; ep[2 * v + 1] = v + 1;
    tb[4 * v] = agree; tb[4 * v + 1] = disagree; tb[4 * v + 2] = disagree; tb[4 * v + 3] = agree;
  }
  int rc = orc_graph_create(n, cards, un, E, ep, tb, out);
  free(cards); free(un); free(ep); free(tb);
  return rc;
}

/* Potts n x n, q states (new): q unit_open unaries per
 * vertex in vertex order, grid edges in Ising order, then one lambda per edge;
 * table = exp(lambda c) on the diagonal, exp(-lambda c) off it. */
int orc_generate_potts(uint32_t n, uint32_t q, double c, uint64_t seed, orc_graph** out) {
  mt64 r;
  mt_seed(&r, seed);
  const uint32_t V = n * n;
  uint32_t* cards = (uint32_t*)malloc(sizeof(uint32_t) * (V ? V : 1));
  double* un = (double*)malloc(sizeof(double) * (size_t)q * (V ? V : 1));
  for (uint32_t v = 0; v < V; ++v) {
    cards[v] = q;
    for (uint32_t x = 0; x < q; ++x) un[(size_t)q * v + x] = unit_open(&r);
  }
  const uint32_t E = n ? 2 * n * (n - 1) : 0;
  uint32_t* ep = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (E ? E : 1));
  uint32_t e = 0;
  for (uint32_t row = 0; row < n; ++row)
    for (uint32_t col = 0; col < n; ++col) {
      const uint32_t v = row * n + col;
      if (col + 1 < n) { ep[2 * e] = v; ep[2 * e + 1] = v + 1; ++e; }
      if (row + 1 < n) { ep[2 * e] = v; ep[2 * e + 1] = v + n; ++e; }
    }
  const size_t qq = (size_t)q * q;
  double* tb = (double*)malloc(sizeof(double) * qq * (E ? E : 1));
  for (uint32_t k = 0; k < E; ++k) {
    const double lambda = uniform_unit(&r) - 0.5;
    const double agree = exp(lambda * c), disagree = exp(-lambda * c);
    for (uint32_t a = 0; a < q; ++a)
      for (uint32_t b = 0; b < q; ++b) tb[qq * k + (size_t)a * q + b] = a == b ? agree : disagree;
  }
  int rc = orc_graph_create(V, cards, un, E, ep, tb, out);
  free(cards); free(un); free(ep); free(tb);
  return rc;
}

/* Erdos-Renyi G(n, m), binary, Ising-style potentials (new; DESIGN.md
 * section 3): 2 unit_open unaries per vertex; then endpoint pairs
 * a = floor(u n), b = floor(u n) drawn until a != b and {a,b} is new; pairs are
 * stored (min,max) and sorted lexicographically; then one lambda per edge in
 * sorted order. */
int orc_generate_er(uint32_t n, uint32_t m, double c, uint64_t seed, orc_graph** out) {
  if (n < 2 && m > 0) return fail(ORC_INVALID_ARGUMENT, "er: need n >= 2");
  if ((uint64_t)m > (uint64_t)n * (n - 1) / 2) return fail(ORC_INVALID_ARGUMENT, "er: too many edges");
  mt64 r;
  mt_seed(&r, seed);
  uint32_t* cards = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  double* un = (double*)malloc(sizeof(double) * 2 * (n ? n : 1));
  for (uint32_t v = 0; v < n; ++v) {
    cards[v] = 2;
    un[2 * v] = unit_open(&r);
    un[2 * v + 1] = unit_open(&r);
  }
  /* open-addressing set of 64-bit keys */
  size_t cap = 16;
  while (cap < (size_t)m * 2 + 16) cap <<= 1;
  uint64_t* set = (uint64_t*)malloc(sizeof(uint64_t) * cap);
  memset(set, 0xff, sizeof(uint64_t) * cap);
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (m ? m : 1));
  uint32_t got = 0;
  while (got < m) {
    uint32_t a = (uint32_t)(uniform_unit(&r) * (double)n);
    uint32_t b = (uint32_t)(uniform_unit(&r) * (double)n);
    if (a == b) continue;
    if (a > b) { uint32_t t = a; a = b; b = t; }
    uint64_t key = ((uint64_t)a << 32) | b;
    size_t h = (size_t)((key * 0x9E3779B97F4A7C15ULL) >> 20) & (cap - 1);
    int dup = 0;
    while (set[h] != UINT64_MAX) {
      if (set[h] == key) { dup = 1; break; }
      h = (h + 1) & (cap - 1);
    }
    if (dup) continue;
    set[h] = key;
    keys[got++] = key;
  }
  free(set);
  qsort(keys, m, sizeof(uint64_t), cmp_u64);
  uint32_t* ep = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (m ? m : 1));
  double* tb = (double*)malloc(sizeof(double) * 4 * (m ? m : 1));
  for (uint32_t k = 0; k < m; ++k) {
    ep[2 * k] = (uint32_t)(keys[k] >> 32);
    ep[2 * k + 1] = (uint32_t)keys[k];
    const double lambda = uniform_unit(&r) - 0.5;
    const double agree = exp(lambda * c), disagree = exp(-lambda * c);
    tb[4 * k] = agree; tb[4 * k + 1] = disagree; tb[4 * k + 2] = disagree; tb[4 * k + 3] = agree;
  }
  free(keys);
  int rc = orc_graph_create(n, cards, un, m, ep, tb, out);
  free(cards); free(un); free(ep); free(tb);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* config (schedulers.cpp:78-90), select_parallelism (:218-224)              */

int orc_validate_config(const orc_config* c) {
  if (!(c->epsilon > 0.0) || !isfinite(c->epsilon))
    return fail(ORC_INVALID_ARGUMENT, "epsilon must be positive");
  if (!(c->p > 0.0) || c->p > 1.0) return fail(ORC_INVALID_ARGUMENT, "p must be in (0, 1]");
  if (!(c->low_p > 0.0) || c->low_p > c->high_p || c->high_p > 1.0)
    return fail(ORC_INVALID_ARGUMENT, "parallelism settings must satisfy 0 < low_p <= high_p <= 1");
  if (!(c->edge_ratio_threshold > 0.0) || c->edge_ratio_threshold > 1.0)
    return fail(ORC_INVALID_ARGUMENT, "edge_ratio_threshold must be in (0, 1]");
  if (!(c->time_limit > 0.0)) return fail(ORC_INVALID_ARGUMENT, "time_limit must be positive");
  if (c->kind < ORC_LBP || c->kind > ORC_RNBP) return fail(ORC_INVALID_ARGUMENT, "unknown scheduler");
  return ORC_OK;
}

double orc_select_parallelism(uint32_t prev, uint32_t now, const orc_config* c) {
  if (prev == 0) return c->high_p;
  const double ratio = (double)now / (double)prev;
  return ratio > c->edge_ratio_threshold ? c->low_p : c->high_p;
}

/* ------------------------------------------------------------------------ */
/* engine: MessageStore + ResidualTracker + EngineState                      */

struct orc_engine {
  const orc_graph* g;
  orc_config cfg;
  size_t* moff; /* D+1, message offsets (messages.cpp:23-39) */
  double* msg;
  double* shadow;
  double* cand;
  double* res;
  uint32_t unconverged;
  uint64_t iteration;
  int has_prev;
  uint32_t prev;
  mt64 rng;
  uint32_t* touched;
  double* scratch;
  /* splash overlay: written[d] == stamp means written in the current splash */
  uint64_t* written;
  uint64_t stamp;
};

/* normalize_in_place: messages.cpp:41-49 */
static int normalize_in_place(double* v, uint32_t n) {
  double sum = 0.0;
  for (uint32_t k = 0; k < n; ++k) sum += v[k];
  if (!(sum >= 1e-300) || !isfinite(sum))
    return fail(ORC_NUMERIC, "probability vector collapsed: total mass %f", sum);
  const double inv = 1.0 / sum;
  for (uint32_t k = 0; k < n; ++k) v[k] *= inv;
  return ORC_OK;
}

/* residual: messages.cpp:56-65 */
static double residual(const double* a, const double* b, uint32_t n) {
  double worst = 0.0;
  for (uint32_t k = 0; k < n; ++k) {
    const double d = fabs(a[k] - b[k]);
    worst = worst < d ? d : worst; /* std::max(worst, d) */
  }
  return worst;
}

/* message view: live store, or the shadow for edges written in the current
 * splash (SplashOverlayView, schedulers.cpp:47-54) */
static inline const double* view(const orc_engine* e, uint32_t d, int overlay) {
  if (overlay && e->written[d] == e->stamp) return e->shadow + e->moff[d];
  return e->msg + e->moff[d];
}

/* detail::update_message_into: messages.hpp:114-151 */
static int update_message_into(const orc_engine* e, uint32_t d, double* out, double* prod,
                               int overlay) {
  const orc_graph* g = e->g;
  const uint32_t src = g->dsrc[d], tgt = g->dtgt[d];
  const uint32_t ci = g->card[src], cj = g->card[tgt];
  const double* un = g->unary + g->uoff[src];
  for (uint32_t x = 0; x < ci; ++x) prod[x] = un[x];
  const uint32_t excluded = d ^ 1u;
  for (size_t a = g->aoff[src]; a < g->aoff[src + 1]; ++a) {
    const uint32_t in = g->adj[a];
    if (in == excluded) continue;
    const double* m = view(e, in, overlay);
    for (uint32_t x = 0; x < ci; ++x) prod[x] *= m[x];
  }
  const double* table = g->table + g->poff[d >> 1];
  if ((d & 1u) == 0) {
    for (uint32_t xj = 0; xj < cj; ++xj) {
      double acc = 0.0;
      for (uint32_t xi = 0; xi < ci; ++xi) acc += table[(size_t)xi * cj + xj] * prod[xi];
      out[xj] = acc;
    }
  } else {
    for (uint32_t xj = 0; xj < cj; ++xj) {
      double acc = 0.0;
      const double* row = table + (size_t)xj * ci;
      for (uint32_t xi = 0; xi < ci; ++xi) acc += row[xi] * prod[xi];
      out[xj] = acc;
    }
  }
  return normalize_in_place(out, cj);
}

/* refresh_residuals: residuals.cpp:26-59 (serial; the reference sums integer
 * per-chunk deltas, so chunking does not change the result) */
static int refresh(orc_engine* e, const uint32_t* touched, size_t n) {
  int64_t delta = 0;
  const double eps = e->cfg.epsilon;
  for (size_t k = 0; k < n; ++k) {
    const uint32_t d = touched[k];
    const int was = e->res[d] >= eps;
    double* cand = e->cand + e->moff[d];
    int rc = update_message_into(e, d, cand, e->scratch, 0);
    if (rc) return rc;
    e->res[d] = residual(cand, e->msg + e->moff[d], (uint32_t)(e->moff[d + 1] - e->moff[d]));
    const int now = e->res[d] >= eps;
    delta += (int64_t)now - (int64_t)was;
  }
  e->unconverged = (uint32_t)((int64_t)e->unconverged + delta);
  return ORC_OK;
}

void orc_engine_destroy(orc_engine* e) {
  if (!e) return;
  free(e->moff);
  free(e->msg);
  free(e->shadow);
  free(e->cand);
  free(e->res);
  free(e->touched);
  free(e->scratch);
  free(e->written);
  free(e);
}

/* EngineState ctor: schedulers.cpp:92-97 = init_messages (messages.cpp:23-39)
 * + ResidualTracker ctor (residuals.cpp:9-24) + rng(seed) */
int orc_engine_create(const orc_graph* g, const orc_config* cfg, orc_engine** out) {
  *out = NULL;
  orc_engine* e = (orc_engine*)calloc(1, sizeof *e);
  if (!e) return fail(ORC_NOMEM, "out of memory");
  e->g = g;
  e->cfg = *cfg;
  const uint32_t D = g->D;
  e->moff = (size_t*)malloc(sizeof(size_t) * (D + 1));
  e->moff[0] = 0;
  for (uint32_t d = 0; d < D; ++d) e->moff[d + 1] = e->moff[d] + g->card[g->dtgt[d]];
  const size_t total = e->moff[D] ? e->moff[D] : 1;
  e->msg = (double*)malloc(sizeof(double) * total);
  e->shadow = (double*)malloc(sizeof(double) * total);
  e->cand = (double*)malloc(sizeof(double) * total);
  e->res = (double*)calloc(D ? D : 1, sizeof(double));
  e->touched = (uint32_t*)malloc(sizeof(uint32_t) * (D ? D : 1));
  e->scratch = (double*)malloc(sizeof(double) * (g->maxq ? g->maxq : 1));
  e->written = (uint64_t*)calloc(D ? D : 1, sizeof(uint64_t));
  e->stamp = 0;
  for (uint32_t d = 0; d < D; ++d) {
    const size_t len = e->moff[d + 1] - e->moff[d];
    const double u = 1.0 / (double)len;
    for (size_t k = e->moff[d]; k < e->moff[d + 1]; ++k) e->msg[k] = u;
  }
  memcpy(e->shadow, e->msg, sizeof(double) * e->moff[D]);
  for (uint32_t d = 0; d < D; ++d) e->touched[d] = d;
  int rc = refresh(e, e->touched, D);
  if (rc) {
    orc_engine_destroy(e);
    return rc;
  }
  mt_seed(&e->rng, cfg->seed);
  *out = e;
  return ORC_OK;
}

uint32_t orc_engine_unconverged(const orc_engine* e) { return e->unconverged; }
uint64_t orc_engine_iteration(const orc_engine* e) { return e->iteration; }
void orc_engine_advance(orc_engine* e) { e->iteration++; }
void orc_engine_messages(const orc_engine* e, double* out) {
  memcpy(out, e->msg, sizeof(double) * e->moff[e->g->D]);
}
void orc_engine_candidates(const orc_engine* e, double* out) {
  memcpy(out, e->cand, sizeof(double) * e->moff[e->g->D]);
}
void orc_engine_residuals(const orc_engine* e, double* out) {
  memcpy(out, e->res, sizeof(double) * e->g->D);
}

/* Load a message state into the engine (test aid, no reference counterpart):
 * live messages <- msgs (MessageStore layout), then the ResidualTracker is
 * rebuilt from scratch as in its ctor (residuals.cpp:9-24) -- candidates
 * f(m), residuals r(m) and the unconverged count of that state, in fp64 with
 * the reference's arithmetic.  Used to check that a device run's converged
 * state is a converged state of the reference's update rule. */
int orc_engine_set_messages(orc_engine* e, const double* msgs) {
  const uint32_t D = e->g->D;
  memcpy(e->msg, msgs, sizeof(double) * e->moff[D]);
  memcpy(e->shadow, e->msg, sizeof(double) * e->moff[D]);
  for (uint32_t d = 0; d < D; ++d) {
    e->res[d] = 0.0;
    e->touched[d] = d;
  }
  e->unconverged = 0;
  return refresh(e, e->touched, D);
}

int orc_engine_update_message(const orc_engine* e, uint32_t d, double* out) {
  if (d >= e->g->D) return fail(ORC_INVALID_ARGUMENT, "directed edge out of range");
  double* scratch = (double*)malloc(sizeof(double) * (e->g->maxq ? e->g->maxq : 1));
  int rc = update_message_into(e, d, out, scratch, 0);
  free(scratch);
  return rc;
}

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

/* collect_touched: schedulers.cpp:31-42 */
static size_t collect_touched(const orc_engine* e, const uint32_t* frontier, size_t n,
                              uint32_t** buf) {
  const orc_graph* g = e->g;
  size_t cap = n, len = 0;
  for (size_t k = 0; k < n; ++k) {
    const uint32_t t = g->dtgt[frontier[k]];
    cap += g->aoff[t + 1] - g->aoff[t];
  }
  uint32_t* t = (uint32_t*)malloc(sizeof(uint32_t) * (cap ? cap : 1));
  for (size_t k = 0; k < n; ++k) {
    const uint32_t d = frontier[k];
    t[len++] = d;
    const uint32_t tgt = g->dtgt[d];
    for (size_t a = g->aoff[tgt]; a < g->aoff[tgt + 1]; ++a) t[len++] = g->adj[a] ^ 1u;
  }
  qsort(t, len, sizeof(uint32_t), cmp_u32);
  size_t u = 0;
  for (size_t k = 0; k < len; ++k)
    if (u == 0 || t[k] != t[u - 1]) t[u++] = t[k];
  *buf = t;
  return u;
}

/* apply_frontier: schedulers.cpp:226-251 */
int orc_engine_apply_frontier(orc_engine* e, const uint32_t* frontier, uint64_t n) {
  if (n == 0) return ORC_OK;
  for (uint64_t k = 0; k < n; ++k) {
    const uint32_t d = frontier[k];
    memcpy(e->msg + e->moff[d], e->cand + e->moff[d], sizeof(double) * (e->moff[d + 1] - e->moff[d]));
  }
  if (n == e->g->D) return refresh(e, frontier, n);
  uint32_t* t;
  size_t len = collect_touched(e, frontier, n, &t);
  int rc = refresh(e, t, len);
  free(t);
  return rc;
}

/* frontier_lbp: schedulers.cpp:99-103 */
void orc_engine_frontier_lbp(const orc_engine* e, uint32_t* out, uint64_t* n) {
  for (uint32_t d = 0; d < e->g->D; ++d) out[d] = d;
  *n = e->g->D;
}

/* select_top_k: schedulers.cpp:105-116 (the k best by (residual desc, id asc);
 * returned ascending by that order -- the reference's order is unspecified) */
static const double* g_sort_keys;
static int cmp_best_first(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  const double rx = g_sort_keys[x], ry = g_sort_keys[y];
  if (rx != ry) return rx > ry ? -1 : 1;
  return x < y ? -1 : x > y;
}

void orc_select_top_k(const double* residuals, uint64_t m, uint64_t k, uint32_t* out, uint64_t* n) {
  for (uint64_t d = 0; d < m; ++d) out[d] = (uint32_t)d;
  if (k >= m) {
    *n = m;
    return;
  }
  g_sort_keys = residuals;
  qsort(out, m, sizeof(uint32_t), cmp_best_first);
  *n = k;
}

/* rbp_frontier: schedulers.cpp:122-126 (k = max(1, llround(p * 2|E|))) */
void orc_engine_rbp_frontier(const orc_engine* e, double p, uint32_t* out, uint64_t* n) {
  const uint64_t m = e->g->D;
  long long k = llround(p * (double)m);
  uint64_t kk = k < 1 ? 1 : (uint64_t)k;
  orc_select_top_k(e->res, m, kk, out, n);
}

/* rnbp_frontier: schedulers.cpp:194-216 */
void orc_engine_rnbp_frontier(orc_engine* e, double p, uint32_t* out, uint64_t* n) {
  const uint32_t D = e->g->D;
  const double eps = e->cfg.epsilon;
  uint32_t* surv = (uint32_t*)malloc(sizeof(uint32_t) * (D ? D : 1));
  size_t s = 0;
  for (uint32_t d = 0; d < D; ++d)
    if (e->res[d] >= eps) surv[s++] = d;
  *n = 0;
  if (s == 0) {
    free(surv);
    return;
  }
  for (int attempt = 0; attempt < 2; ++attempt) {
    uint64_t f = 0;
    for (size_t k = 0; k < s; ++k)
      if (uniform_unit(&e->rng) < p) out[f++] = surv[k];
    if (f > 0) {
      *n = f;
      free(surv);
      return;
    }
  }
  size_t pick = (size_t)(uniform_unit(&e->rng) * (double)s);
  if (pick > s - 1) pick = s - 1;
  out[0] = surv[pick];
  *n = 1;
  free(surv);
}

/* vertex_residual: schedulers.cpp:128-134 */
static double vertex_residual(const orc_engine* e, uint32_t v) {
  double worst = 0.0;
  for (size_t a = e->g->aoff[v]; a < e->g->aoff[v + 1]; ++a) {
    const double r = e->res[e->g->adj[a]];
    worst = worst < r ? r : worst;
  }
  return worst;
}

/* build_splash: schedulers.cpp:136-167. Appends the splash's edges to
 * edges[*ne...]; claimed[] holds the root id or UINT32_MAX. */
static void build_splash(const orc_engine* e, uint32_t root, uint32_t h, uint32_t* claimed,
                         uint32_t* queue_v, uint32_t* queue_d, uint32_t* edges, uint64_t* ne) {
  const orc_graph* g = e->g;
  size_t head = 0, tail = 0;
  claimed[root] = root;
  queue_v[tail] = root;
  queue_d[tail++] = 0;
  while (head < tail) {
    const uint32_t v = queue_v[head], depth = queue_d[head];
    ++head; /* visited order == queue order */
    if (depth < h) {
      for (size_t a = g->aoff[v]; a < g->aoff[v + 1]; ++a) {
        const uint32_t nb = g->dsrc[g->adj[a]];
        if (claimed[nb] == UINT32_MAX) {
          claimed[nb] = root;
          queue_v[tail] = nb;
          queue_d[tail++] = depth + 1;
        }
      }
    }
  }
  for (size_t k = 0; k < tail; ++k) {
    const uint32_t v = queue_v[k];
    for (size_t a = g->aoff[v]; a < g->aoff[v + 1]; ++a) edges[(*ne)++] = g->adj[a] ^ 1u;
  }
}

int orc_engine_build_splash(const orc_engine* e, uint32_t root, uint32_t h, uint32_t* claimed,
                            uint32_t* edges, uint64_t* n) {
  const uint32_t V = e->g->V;
  if (root >= V) return fail(ORC_INVALID_ARGUMENT, "root out of range");
  if (claimed[root] != UINT32_MAX) return fail(ORC_INVALID_ARGUMENT, "splash root %u is already claimed", root);
  uint32_t* qv = (uint32_t*)malloc(sizeof(uint32_t) * V);
  uint32_t* qd = (uint32_t*)malloc(sizeof(uint32_t) * V);
  *n = 0;
  build_splash(e, root, h, claimed, qv, qd, edges, n);
  free(qv);
  free(qd);
  return ORC_OK;
}

/* rs_frontier: schedulers.cpp:169-192 */
int orc_engine_rs_frontier(orc_engine* e, double p, uint32_t h, uint32_t* roots,
                           uint64_t* eoff, uint32_t* edges, uint64_t* num) {
  const orc_graph* g = e->g;
  const uint32_t V = g->V;
  *num = 0;
  eoff[0] = 0;
  if (V == 0) return ORC_OK;
  long long kr = llround(p * (double)V);
  const uint64_t k = kr < 1 ? 1 : (uint64_t)kr;
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * V);
  double* vres = (double*)malloc(sizeof(double) * V);
  for (uint32_t v = 0; v < V; ++v) {
    order[v] = v;
    vres[v] = vertex_residual(e, v);
  }
  g_sort_keys = vres;
  qsort(order, V, sizeof(uint32_t), cmp_best_first);
  uint32_t* claimed = (uint32_t*)malloc(sizeof(uint32_t) * V);
  for (uint32_t v = 0; v < V; ++v) claimed[v] = UINT32_MAX;
  uint32_t* qv = (uint32_t*)malloc(sizeof(uint32_t) * V);
  uint32_t* qd = (uint32_t*)malloc(sizeof(uint32_t) * V);
  uint64_t ne = 0, ns = 0;
  for (uint32_t idx = 0; idx < V; ++idx) {
    if (ns >= k) break;
    const uint32_t root = order[idx];
    if (claimed[root] != UINT32_MAX) continue;
    build_splash(e, root, h, claimed, qv, qd, edges, &ne);
    roots[ns] = root;
    eoff[++ns] = ne;
  }
  *num = ns;
  free(order); free(vres); free(claimed); free(qv); free(qd);
  return ORC_OK;
}

/* apply_splash_frontier: schedulers.cpp:253-291 */
int orc_engine_apply_splashes(orc_engine* e, uint64_t ns, const uint32_t* roots,
                              const uint64_t* eoff, const uint32_t* edges) {
  (void)roots;
  const uint64_t total = eoff[ns];
  if (total == 0) return ORC_OK;
  {
    uint32_t* check = (uint32_t*)malloc(sizeof(uint32_t) * total);
    memcpy(check, edges, sizeof(uint32_t) * total);
    qsort(check, total, sizeof(uint32_t), cmp_u32);
    for (uint64_t k = 1; k < total; ++k)
      if (check[k] == check[k - 1]) {
        free(check);
        return fail(ORC_MODEL, "overlapping splashes: an edge is updated by two splashes");
      }
    free(check);
  }
  for (uint64_t s = 0; s < ns; ++s) {
    e->stamp++; /* fresh `written` set per splash */
    for (uint64_t k = eoff[s]; k < eoff[s + 1]; ++k) {
      const uint32_t d = edges[k];
      int rc = update_message_into(e, d, e->shadow + e->moff[d], e->scratch, 1);
      if (rc) return rc;
      e->written[d] = e->stamp;
    }
  }
  e->stamp++;
  for (uint64_t k = 0; k < total; ++k) { /* commit_shadow: messages.cpp:15-21 */
    const uint32_t d = edges[k];
    memcpy(e->msg + e->moff[d], e->shadow + e->moff[d], sizeof(double) * (e->moff[d + 1] - e->moff[d]));
  }
  uint32_t* t;
  size_t len = collect_touched(e, edges, total, &t);
  int rc = refresh(e, t, len);
  free(t);
  return rc;
}

/* compute_beliefs: messages.cpp:82-105 */
int orc_engine_beliefs(const orc_engine* e, double* out) {
  const orc_graph* g = e->g;
  for (uint32_t v = 0; v < g->V; ++v) {
    double* b = out + g->uoff[v];
    const uint32_t q = g->card[v];
    for (uint32_t x = 0; x < q; ++x) b[x] = g->unary[g->uoff[v] + x];
    for (size_t a = g->aoff[v]; a < g->aoff[v + 1]; ++a) {
      const double* m = e->msg + e->moff[g->adj[a]];
      for (uint32_t x = 0; x < q; ++x) b[x] *= m[x];
    }
    int rc = normalize_in_place(b, q);
    if (rc) return rc;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* serial RBP (serial_rbp.cpp:30-82): indexed binary max-heap with the same
 * strict order as PqLess (serial_rbp.cpp:19-24), so pops are identical.    */

typedef struct {
  uint32_t* heap; /* heap[pos] = edge */
  uint32_t* pos;  /* pos[edge] */
  double* key;    /* key[edge]: the residual as last pushed (PqItem::res) */
  uint32_t n;
} iheap;

static inline int better(const iheap* h, uint32_t a, uint32_t b) {
  if (h->key[a] != h->key[b]) return h->key[a] > h->key[b];
  return a < b;
}
static void sift_up(iheap* h, uint32_t i) {
  while (i > 0) {
    uint32_t p = (i - 1) / 2;
    if (!better(h, h->heap[i], h->heap[p])) break;
    uint32_t t = h->heap[i]; h->heap[i] = h->heap[p]; h->heap[p] = t;
    h->pos[h->heap[i]] = i; h->pos[h->heap[p]] = p;
    i = p;
  }
}
static void sift_down(iheap* h, uint32_t i) {
  for (;;) {
    uint32_t l = 2 * i + 1, r = l + 1, b = i;
    if (l < h->n && better(h, h->heap[l], h->heap[b])) b = l;
    if (r < h->n && better(h, h->heap[r], h->heap[b])) b = r;
    if (b == i) break;
    uint32_t t = h->heap[i]; h->heap[i] = h->heap[b]; h->heap[b] = t;
    h->pos[h->heap[i]] = i; h->pos[h->heap[b]] = b;
    i = b;
  }
}

static int run_serial_rbp(const orc_graph* g, const orc_config* cfg, orc_result* res,
                          double* beliefs, orc_record* trace, uint64_t trace_cap) {
  const double t0 = now_seconds();
  orc_engine* e;
  int rc = orc_engine_create(g, cfg, &e);
  if (rc) return rc;
  const uint32_t D = g->D;
  iheap h;
  h.heap = (uint32_t*)malloc(sizeof(uint32_t) * (D ? D : 1));
  h.pos = (uint32_t*)malloc(sizeof(uint32_t) * (D ? D : 1));
  h.key = (double*)malloc(sizeof(double) * (D ? D : 1));
  h.n = D;
  for (uint32_t d = 0; d < D; ++d) { h.heap[d] = d; h.pos[d] = d; h.key[d] = e->res[d]; }
  for (int64_t i = (int64_t)D / 2 - 1; i >= 0; --i) sift_down(&h, (uint32_t)i);
  uint64_t updates = 0, tl = 0;
  while (h.n > 0) {
    const uint32_t top = h.heap[0];
    if (e->res[top] < cfg->epsilon) break;
    if (updates >= cfg->max_iterations || now_seconds() - t0 >= cfg->time_limit) break;
    const uint32_t d = top;
    memcpy(e->msg + e->moff[d], e->cand + e->moff[d], sizeof(double) * (e->moff[d + 1] - e->moff[d]));
    uint32_t* t;
    size_t len = collect_touched(e, &d, 1, &t);
    rc = refresh(e, t, len);
    if (rc) { free(t); break; }
    for (size_t k = 0; k < len; ++k) { /* heap.update, one key at a time */
      h.key[t[k]] = e->res[t[k]];
      sift_up(&h, h.pos[t[k]]);
      sift_down(&h, h.pos[t[k]]);
    }
    free(t);
    ++updates;
    if (trace && tl < trace_cap) {
      trace[tl].iteration = updates - 1;
      trace[tl].frontier_size = 1;
      trace[tl].unconverged = e->unconverged;
      trace[tl].elapsed_seconds = now_seconds() - t0;
    }
    ++tl;
  }
  if (!rc) {
    res->converged = e->unconverged == 0;
    res->iterations = updates;
    res->messages_updated_total = updates;
    res->trace_len = tl;
    if (beliefs) rc = orc_engine_beliefs(e, beliefs);
    res->wall_time = now_seconds() - t0;
  }
  free(h.heap);
  free(h.pos);
  free(h.key);
  orc_engine_destroy(e);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* run: schedulers.cpp:293-353                                                */

int orc_run(const orc_graph* g, const orc_config* cfg, orc_result* res, double* beliefs,
            orc_record* trace, uint64_t trace_cap) {
  memset(res, 0, sizeof *res);
  int rc = orc_validate_config(cfg);
  if (rc) return rc;
  if (cfg->kind == ORC_SRBP) return run_serial_rbp(g, cfg, res, beliefs, trace, trace_cap);
  const double t0 = now_seconds();
  orc_engine* e;
  rc = orc_engine_create(g, cfg, &e);
  if (rc) return rc;
  const uint32_t D = g->D;
  uint32_t* frontier = (uint32_t*)malloc(sizeof(uint32_t) * (D ? D : 1));
  uint32_t* roots = (uint32_t*)malloc(sizeof(uint32_t) * (g->V ? g->V : 1));
  uint64_t* eoff = (uint64_t*)malloc(sizeof(uint64_t) * (g->V + 1));
  uint64_t tl = 0;
  for (;;) {
    const uint32_t unconverged = e->unconverged;
    if (unconverged == 0) {
      res->converged = 1;
      break;
    }
    if (e->iteration >= cfg->max_iterations || now_seconds() - t0 >= cfg->time_limit) break;
    uint64_t fsize = 0, n = 0;
    switch (cfg->kind) {
      case ORC_LBP:
        orc_engine_frontier_lbp(e, frontier, &n);
        fsize = n;
        rc = orc_engine_apply_frontier(e, frontier, n);
        break;
      case ORC_RBP:
        orc_engine_rbp_frontier(e, cfg->p, frontier, &n);
        fsize = n;
        rc = orc_engine_apply_frontier(e, frontier, n);
        break;
      case ORC_RNBP: {
        const double p_now =
            orc_select_parallelism(e->has_prev ? e->prev : 0, unconverged, cfg);
        e->prev = unconverged;
        e->has_prev = 1;
        orc_engine_rnbp_frontier(e, p_now, frontier, &n);
        fsize = n;
        rc = orc_engine_apply_frontier(e, frontier, n);
        break;
      }
      case ORC_RS: {
        uint64_t ns = 0;
        orc_engine_rs_frontier(e, cfg->p, cfg->splash_depth, roots, eoff, frontier, &ns);
        fsize = eoff[ns];
        rc = orc_engine_apply_splashes(e, ns, roots, eoff, frontier);
        break;
      }
      default:
        break;
    }
    if (rc) break;
    res->messages_updated_total += fsize;
    if (trace && tl < trace_cap) {
      trace[tl].iteration = e->iteration;
      trace[tl].frontier_size = fsize;
      trace[tl].unconverged = e->unconverged;
      trace[tl].elapsed_seconds = now_seconds() - t0;
    }
    ++tl;
    e->iteration++;
  }
  if (!rc) {
    res->iterations = e->iteration;
    res->trace_len = tl;
    if (beliefs) rc = orc_engine_beliefs(e, beliefs);
    res->wall_time = now_seconds() - t0;
  }
  free(frontier);
  free(roots);
  free(eoff);
  orc_engine_destroy(e);
  return rc;
}
