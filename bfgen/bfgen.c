/*
 * bfgen.c -- seeded synthetic bipartite-graph generators.
 *
 * This module is shared by the oracle side (tests) and the product side
 * (bench.py, GPU tests).  It holds NONE of the butterfly-counting arithmetic:
 * it only draws edges.  The recipe is DESIGN.md "Input recipe", which follows
 * SURVEY.md 8(d) (the choices marked there as choices are fixed here):
 *
 *   RNG        splitmix64 over a counter, keyed by (seed, stream id).
 *              uniform double = (r >> 11) * 2^-53.
 *   ids        per side, a seeded Fisher-Yates permutation maps
 *              weight-index -> vertex id (degree uncorrelated with id).
 *   distinct   candidate pairs are drawn in batches until >= m distinct keys
 *              k = u*|V| + v exist; the m keys with the smallest
 *              splitmix64(k ^ seed) are kept (planted keys always kept).
 *   order      edges are emitted sorted by splitmix64(k ^ seed).
 *   Chung-Lu   side weight w_i = (i+1)^(-1/(gamma-1)), sampled with a Vose
 *              alias table (same distribution as the survey's prefix-sum
 *              binary search; O(1) per draw).
 *   geo-Zipf   user degree D = 1 + floor(ln(U)/ln(1-p)) (Geometric on
 *              {1,2,...}, mean 1/p), capped at |V|; items i.i.d.
 *              Zipf(s) over |V| ranks with per-user rejection of repeats.
 *
 * The paper measures on KONECT graphs (Table
 * table-graphs); these generators stand in for them.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t sm64_mix(uint64_t z) {
  z += GOLDEN;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return sm64_mix(sm64_mix(seed) ^ (stream * 0xD1B54A32D192ED03ULL));
}
/* i-th draw of a stream: splitmix64 over a counter */
static inline uint64_t rnd(uint64_t key, uint64_t i) { return sm64_mix(key + i * GOLDEN); }
static inline double u01(uint64_t r) { return (double)(r >> 11) * 0x1.0p-53; }
static inline uint32_t bounded(uint64_t r, uint64_t n) {
  return (uint32_t)(((r >> 32) * n) >> 32);
}

uint64_t bfgen_splitmix64(uint64_t x) { return sm64_mix(x); }

/* ---------------- LSD radix sort of (u64 key, u64 payload) -------------- */
static void radix_sort_kv(uint64_t* k, uint64_t* v, size_t n, int bits) {
  if (n < 2 || bits <= 0) return;
  uint64_t* tk = (uint64_t*)malloc(n * 8);
  uint64_t* tv = v ? (uint64_t*)malloc(n * 8) : NULL;
  const int D = 11;
  size_t cnt[1 << D];
  for (int sh = 0; sh < bits; sh += D) {
    memset(cnt, 0, sizeof(cnt));
    for (size_t i = 0; i < n; i++) cnt[(k[i] >> sh) & ((1 << D) - 1)]++;
    size_t s = 0;
    for (int d = 0; d < (1 << D); d++) { size_t c = cnt[d]; cnt[d] = s; s += c; }
    for (size_t i = 0; i < n; i++) {
      size_t p = cnt[(k[i] >> sh) & ((1 << D) - 1)]++;
      tk[p] = k[i];
      if (v) tv[p] = v[i];
    }
    memcpy(k, tk, n * 8);
    if (v) memcpy(v, tv, n * 8);
  }
  free(tk);
  free(tv);
}
static int bits_for(uint64_t maxv) { int b = 0; while (b < 64 && (maxv >> b)) b++; return b; }

/* sort + unique in place; returns new length */
static size_t sort_unique(uint64_t* k, size_t n, uint64_t maxkey) {
  radix_sort_kv(k, NULL, n, bits_for(maxkey));
  size_t w = 0;
  for (size_t i = 0; i < n; i++)
    if (w == 0 || k[i] != k[w - 1]) k[w++] = k[i];
  return w;
}
/* merge two sorted unique arrays into out (unique); returns length */
static size_t merge_unique(const uint64_t* a, size_t na, const uint64_t* b, size_t nb, uint64_t* out) {
  size_t i = 0, j = 0, w = 0;
  while (i < na || j < nb) {
    uint64_t x;
    if (j >= nb || (i < na && a[i] < b[j])) x = a[i++];
    else if (i >= na || b[j] < a[i]) x = b[j++];
    else { x = a[i++]; j++; }
    out[w++] = x;
  }
  return w;
}

/* Fisher-Yates permutation of [0,n) with stream key */
static void permutation(uint32_t* p, uint32_t n, uint64_t key) {
  for (uint32_t i = 0; i < n; i++) p[i] = i;
  for (uint32_t i = n; i > 1; i--) {
    uint32_t j = bounded(rnd(key, i), i);
    uint32_t t = p[i - 1]; p[i - 1] = p[j]; p[j] = t;
  }
}

/* ---------------- Vose alias table ---------------- */
typedef struct { double* prob; uint32_t* alias; uint32_t n; } alias_t;
static void alias_build(alias_t* a, const double* w, uint32_t n) {
  a->n = n;
  a->prob = (double*)malloc(sizeof(double) * n);
  a->alias = (uint32_t*)malloc(sizeof(uint32_t) * n);
  double sum = 0;
  for (uint32_t i = 0; i < n; i++) sum += w[i];
  double* sc = (double*)malloc(sizeof(double) * n);
  uint32_t* small = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* large = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t ns = 0, nl = 0;
  for (uint32_t i = 0; i < n; i++) {
    sc[i] = w[i] * n / sum;
    if (sc[i] < 1.0) small[ns++] = i; else large[nl++] = i;
  }
  while (ns && nl) {
    uint32_t s = small[--ns], l = large[--nl];
    a->prob[s] = sc[s]; a->alias[s] = l;
    sc[l] = (sc[l] + sc[s]) - 1.0;
    if (sc[l] < 1.0) small[ns++] = l; else large[nl++] = l;
  }
  while (nl) { uint32_t l = large[--nl]; a->prob[l] = 1.0; a->alias[l] = l; }
  while (ns) { uint32_t s = small[--ns]; a->prob[s] = 1.0; a->alias[s] = s; }
  free(sc); free(small); free(large);
}
static inline uint32_t alias_draw(const alias_t* a, uint64_t r1, uint64_t r2) {
  uint32_t i = bounded(r1, a->n);
  return (u01(r2) < a->prob[i]) ? i : a->alias[i];
}
static void alias_free(alias_t* a) { free(a->prob); free(a->alias); }

/* ---------------- selection of m keys by hash, emission ---------------- */
/* keys: sorted unique candidate keys (n of them, n >= m).  planted: sorted
 * unique keys that must be kept (np of them, all present in keys).
 * Writes m edges (u,v) to out in splitmix64(k ^ seed) order. */
static void select_and_emit(const uint64_t* keys, size_t n, const uint64_t* planted, size_t np,
                            uint64_t m, uint32_t nV, uint64_t seed, uint32_t* out) {
  uint64_t* h = (uint64_t*)malloc(n * 8);
  uint64_t* kk = (uint64_t*)malloc(n * 8);
  #pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; i++) { h[i] = sm64_mix(keys[i] ^ seed); kk[i] = keys[i]; }
  radix_sort_kv(h, kk, n, 64);
  uint64_t keep_free = m - np, taken_free = 0, w = 0;
  for (size_t i = 0; i < n && w < m; i++) {
    uint64_t k = kk[i];
    int is_planted = 0;
    if (np) { /* binary search */
      size_t lo = 0, hi = np;
      while (lo < hi) { size_t mid = (lo + hi) / 2; if (planted[mid] < k) lo = mid + 1; else hi = mid; }
      is_planted = (lo < np && planted[lo] == k);
    }
    if (!is_planted) { if (taken_free >= keep_free) continue; taken_free++; }
    out[2 * w] = (uint32_t)(k / nV);
    out[2 * w + 1] = (uint32_t)(k % nV);
    w++;
  }
  free(h); free(kk);
}

/* Draw candidate pair keys until >= m distinct (including the planted set).
 * draw(i) produces the i-th candidate key.  Returns sorted unique array. */
typedef uint64_t (*draw_fn)(const void* ctx, uint64_t i);
static uint64_t* draw_distinct(const void* ctx, draw_fn draw, uint64_t m, const uint64_t* planted,
                               size_t np, uint64_t maxkey, size_t* n_out) {
  size_t cap = np;
  uint64_t* have = (uint64_t*)malloc((np ? np : 1) * 8);
  if (np) memcpy(have, planted, np * 8);
  size_t nh = np;
  uint64_t next = 0;
  int round = 0;
  while (nh < m) {
    uint64_t need = m - nh;
    uint64_t batch = round == 0 ? m + m / 16 + 1024 : need * 2 + 1024;
    uint64_t* b = (uint64_t*)malloc(batch * 8);
    #pragma omp parallel for schedule(static)
    for (uint64_t i = 0; i < batch; i++) b[i] = draw(ctx, next + i);
    next += batch;
    size_t nb = sort_unique(b, batch, maxkey);
    uint64_t* merged = (uint64_t*)malloc((nh + nb) * 8);
    nh = merge_unique(have, nh, b, nb, merged);
    free(have); free(b);
    have = merged;
    cap = nh;
    round++;
    if (round > 200) break; /* saturated distribution; caller checks */
  }
  (void)cap;
  *n_out = nh;
  return have;
}

/* ---------------- uniform (config 1) ---------------- */
typedef struct { uint32_t nU, nV; uint64_t ku, kv; } uni_ctx;
static uint64_t uni_draw(const void* c, uint64_t i) {
  const uni_ctx* x = (const uni_ctx*)c;
  uint64_t u = bounded(rnd(x->ku, i), x->nU), v = bounded(rnd(x->kv, i), x->nV);
  return u * x->nV + v;
}
/* returns 0 on success, -1 if m > |U||V| */
int bfgen_uniform(uint32_t nU, uint32_t nV, uint64_t m, uint64_t seed, uint32_t* out) {
  if ((uint64_t)nU * nV < m) return -1;
  if (m == 0) return 0;
  uni_ctx c = {nU, nV, stream_key(seed, 1), stream_key(seed, 2)};
  size_t n;
  uint64_t* keys = draw_distinct(&c, uni_draw, m, NULL, 0, (uint64_t)nU * nV, &n);
  if (n < m) { free(keys); return -2; }
  select_and_emit(keys, n, NULL, 0, m, nV, seed, out);
  free(keys);
  return 0;
}

/* ---------------- Chung-Lu (configs 2, 3, 5) ---------------- */
typedef struct { alias_t au, av; uint32_t *pu, *pv; uint32_t nV; uint64_t ku, kv; } cl_ctx;
static uint64_t cl_draw(const void* c, uint64_t i) {
  const cl_ctx* x = (const cl_ctx*)c;
  uint32_t iu = alias_draw(&x->au, rnd(x->ku, 2 * i), rnd(x->ku, 2 * i + 1));
  uint32_t iv = alias_draw(&x->av, rnd(x->kv, 2 * i), rnd(x->kv, 2 * i + 1));
  return (uint64_t)x->pu[iu] * x->nV + x->pv[iv];
}
static void powerlaw_weights(double* w, uint32_t n, double gamma) {
  double e = -1.0 / (gamma - 1.0);
  for (uint32_t i = 0; i < n; i++) w[i] = pow((double)(i + 1), e);
}
/* planted_a x planted_b biclique on uniformly chosen distinct vertices
 * (0 = none).  returns 0 on success, <0 on failure. */
int bfgen_chung_lu(uint32_t nU, uint32_t nV, uint64_t m, double gU, double gV,
                   uint32_t planted_a, uint32_t planted_b, uint64_t seed, uint32_t* out,
                   uint32_t* planted_u_out, uint32_t* planted_v_out) {
  if ((uint64_t)nU * nV < m || nU == 0 || nV == 0) return -1;
  if (planted_a > nU || planted_b > nV) return -1;
  cl_ctx c;
  double* w = (double*)malloc(sizeof(double) * (nU > nV ? nU : nV));
  powerlaw_weights(w, nU, gU); alias_build(&c.au, w, nU);
  powerlaw_weights(w, nV, gV); alias_build(&c.av, w, nV);
  free(w);
  c.pu = (uint32_t*)malloc(4ull * nU); c.pv = (uint32_t*)malloc(4ull * nV);
  permutation(c.pu, nU, stream_key(seed, 3));
  permutation(c.pv, nV, stream_key(seed, 4));
  c.nV = nV; c.ku = stream_key(seed, 5); c.kv = stream_key(seed, 6);
  /* planted biclique: first planted_a entries of a fresh permutation */
  size_t np = (size_t)planted_a * planted_b;
  uint64_t* planted = NULL;
  if (np) {
    uint32_t* qu = (uint32_t*)malloc(4ull * nU);
    uint32_t* qv = (uint32_t*)malloc(4ull * nV);
    permutation(qu, nU, stream_key(seed, 7));
    permutation(qv, nV, stream_key(seed, 8));
    planted = (uint64_t*)malloc(np * 8);
    size_t t = 0;
    for (uint32_t a = 0; a < planted_a; a++)
      for (uint32_t b = 0; b < planted_b; b++) planted[t++] = (uint64_t)qu[a] * nV + qv[b];
    if (planted_u_out) memcpy(planted_u_out, qu, 4ull * planted_a);
    if (planted_v_out) memcpy(planted_v_out, qv, 4ull * planted_b);
    free(qu); free(qv);
    np = sort_unique(planted, np, (uint64_t)nU * nV);
  }
  int rc = 0;
  if (np > m) rc = -1;
  else {
    size_t n;
    uint64_t* keys = draw_distinct(&c, cl_draw, m, planted, np, (uint64_t)nU * nV, &n);
    if (n < m) rc = -2;
    else select_and_emit(keys, n, planted, np, m, nV, seed, out);
    free(keys);
  }
  free(planted);
  alias_free(&c.au); alias_free(&c.av); free(c.pu); free(c.pv);
  return rc;
}

/* ---------------- geometric users x Zipf items (config 4) ---------------- */
/* Two calls: out == NULL returns m (= sum of user degrees); then call again
 * with out sized 2*m.  Deterministic for (nU, nV, p, s, seed). */
static uint32_t geo_degree(uint64_t key, uint32_t u, double p, uint32_t cap) {
  double x = u01(rnd(key, u));
  if (x <= 0.0) x = 0x1.0p-53;
  double d = 1.0 + floor(log(x) / log(1.0 - p));
  if (d > cap) d = cap;
  return (uint32_t)d;
}
int64_t bfgen_geo_zipf(uint32_t nU, uint32_t nV, double p, double s, uint64_t seed, uint32_t* out) {
  if (nU == 0 || nV == 0 || !(p > 0 && p <= 1)) return -1;
  uint64_t kdeg = stream_key(seed, 11);
  uint64_t* off = (uint64_t*)malloc(8ull * ((uint64_t)nU + 1));
  off[0] = 0;
  for (uint32_t u = 0; u < nU; u++) off[u + 1] = off[u] + geo_degree(kdeg, u, p, nV);
  uint64_t m = off[nU];
  if (!out) { free(off); return (int64_t)m; }
  double* w = (double*)malloc(sizeof(double) * nV);
  for (uint32_t i = 0; i < nV; i++) w[i] = pow((double)(i + 1), -s);
  alias_t a; alias_build(&a, w, nV); free(w);
  uint32_t* perm = (uint32_t*)malloc(4ull * nV);
  permutation(perm, nV, stream_key(seed, 12));
  uint32_t* uperm = (uint32_t*)malloc(4ull * nU);
  permutation(uperm, nU, stream_key(seed, 13));
  uint64_t kit = stream_key(seed, 14);
  uint64_t* keys = (uint64_t*)malloc(8 * m);
  #pragma omp parallel for schedule(dynamic, 4096)
  for (uint32_t u = 0; u < nU; u++) {
    uint64_t ku = sm64_mix(kit ^ ((uint64_t)u * GOLDEN));
    uint64_t b = off[u], d = off[u + 1] - b, got = 0, t = 0;
    uint32_t uid = uperm[u];
    while (got < d) {
      uint32_t it = perm[alias_draw(&a, rnd(ku, 2 * t), rnd(ku, 2 * t + 1))];
      t++;
      int dup = 0;
      for (uint64_t j = 0; j < got; j++) if ((uint32_t)(keys[b + j] % nV) == it) { dup = 1; break; }
      if (!dup) keys[b + got++] = (uint64_t)uid * nV + it;
    }
  }
  select_and_emit(keys, m, NULL, 0, m, nV, seed, out); /* keys need not be sorted here */
  free(keys); free(off); alias_free(&a); free(perm); free(uperm);
  return (int64_t)m;
}
