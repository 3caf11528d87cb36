/*
 * oracle.c -- plain, slow, single-threaded CPU oracle for exact butterfly
 * counting.  TEST INFRASTRUCTURE ONLY: it may be called by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg,
 * never by the product path.  It shares no code, header, table or helper with
 * the CUDA library (paper_1907_08607_b200/csrc) and neither includes the other.
 *
 * What it computes is the plain definition, not the paper's
 * ranked wedge algorithm:
 *
 *   c(x,x')  = |N(x) ∩ N(x')| for x != x' on the same side
 *   b(x)     = Σ_{x' != x} C(c(x,x'), 2)                  Eq. (1)
 *   b(u,v)   = Σ_{u' ∈ N(v) \ {u}} (c(u,u') - 1)          Eq. (2)
 *   T        = Σ_{x∈X} b(x) / 2                           (butterfly = pair of same-side
 *                                                          vertices + 2 common nbrs)
 *   centre   b(y) += Σ_{x'∈N(y), x'>x} (c(x,x') - 1)      (each unordered endpoint pair once;
 *                                                          every centre of a d-wedge group gets
 *                                                          d-1: Fig. fig-count-ex Step 4,
 *                                                          P:349-356; Alg. 3 l.6)
 *
 * Pairs with c <= 1 contribute 0, so visiting only pairs reachable through a
 * common neighbour is the same sum.  All sums are taken in
 * unsigned __int128 and checked against 2^64 (reading Z9).
 *
 * It also holds the paper's rankings (readings Z1-Z4) and the
 * wedge count W = Σ_x Σ_{y∈N_x(x)} deg_x(y) (Alg. 2 loop
 * bounds P:739-744, reading Z6) written straight from the definitions, for
 * the work metric and its pins.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

enum { ORC_OK = 0, ORC_ERANGE = 1, ORC_EDUP = 2, ORC_ENOMEM = 3, ORC_EOVERFLOW = 4, ORC_EINVAL = 5 };

typedef struct {
  uint32_t n[2];     /* n[0] = |U|, n[1] = |V| */
  uint64_t m;
  uint64_t* off[2];  /* off[s][x] .. off[s][x+1]: neighbours of side-s vertex x */
  uint32_t* adj[2];  /* neighbour ids (other side), ascending */
  uint32_t* eid[2];  /* input edge index of each adjacency entry */
  uint32_t* cnt;     /* scratch dense counters, size max(n) */
  uint32_t* touched; /* scratch touched list */
} orc_graph;

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

void orc_free(orc_graph* g) {
  if (!g) return;
  for (int s = 0; s < 2; s++) { free(g->off[s]); free(g->adj[s]); free(g->eid[s]); }
  free(g->cnt); free(g->touched); free(g);
}

/* Per-side sorted adjacency.  Rejects out-of-range ids
 * and repeated (u,v) pairs (reading Z8). */
int orc_build(uint32_t nU, uint32_t nV, const uint32_t* edges, uint64_t m, orc_graph** out) {
  *out = NULL;
  orc_graph* g = (orc_graph*)calloc(1, sizeof(orc_graph));
  if (!g) return ORC_ENOMEM;
  g->n[0] = nU; g->n[1] = nV; g->m = m;
  for (uint64_t e = 0; e < m; e++)
    if (edges[2 * e] >= nU || edges[2 * e + 1] >= nV) { free(g); return ORC_ERANGE; }
  for (int s = 0; s < 2; s++) {
    uint32_t n = g->n[s];
    g->off[s] = (uint64_t*)calloc((size_t)n + 1, 8);
    g->adj[s] = (uint32_t*)malloc(m ? m * 4 : 4);
    g->eid[s] = (uint32_t*)malloc(m ? m * 4 : 4);
    if (!g->off[s] || !g->adj[s] || !g->eid[s]) { orc_free(g); return ORC_ENOMEM; }
    for (uint64_t e = 0; e < m; e++) g->off[s][edges[2 * e + s] + 1]++;
    for (uint32_t x = 0; x < n; x++) g->off[s][x + 1] += g->off[s][x];
    uint64_t* fill = (uint64_t*)malloc(((size_t)n + 1) * 8);
    memcpy(fill, g->off[s], ((size_t)n + 1) * 8);
    for (uint64_t e = 0; e < m; e++) {
      uint32_t x = edges[2 * e + s], y = edges[2 * e + 1 - s];
      uint64_t p = fill[x]++;
      g->adj[s][p] = y;
      g->eid[s][p] = (uint32_t)e;
    }
    free(fill);
    /* sort each neighbour list ascending (pack (y, eid) into one u64) */
    uint64_t* tmp = NULL; size_t tcap = 0;
    for (uint32_t x = 0; x < n; x++) {
      uint64_t a = g->off[s][x], b = g->off[s][x + 1], d = b - a;
      if (d < 2) continue;
      if (d > tcap) { free(tmp); tcap = d; tmp = (uint64_t*)malloc(tcap * 8); }
      for (uint64_t i = 0; i < d; i++) tmp[i] = ((uint64_t)g->adj[s][a + i] << 32) | g->eid[s][a + i];
      qsort(tmp, d, 8, cmp_u64);
      for (uint64_t i = 0; i < d; i++) {
        g->adj[s][a + i] = (uint32_t)(tmp[i] >> 32);
        g->eid[s][a + i] = (uint32_t)tmp[i];
        if (i && g->adj[s][a + i] == g->adj[s][a + i - 1]) { free(tmp); orc_free(g); return ORC_EDUP; }
      }
    }
    free(tmp);
  }
  uint32_t nmax = nU > nV ? nU : nV;
  g->cnt = (uint32_t*)calloc(nmax ? nmax : 1, 4);
  g->touched = (uint32_t*)malloc((nmax ? nmax : 1) * 4);
  if (!g->cnt || !g->touched) { orc_free(g); return ORC_ENOMEM; }
  *out = g;
  return ORC_OK;
}

uint32_t orc_degree(const orc_graph* g, int side, uint32_t x) {
  return (uint32_t)(g->off[side][x + 1] - g->off[side][x]);
}

/* cnt[x'] = c(x,x') for every x' != x on x's side reachable in two hops;
 * returns the number of touched x'. */
static uint32_t common_neighbour_counts(orc_graph* g, int X, uint32_t x) {
  int Y = 1 - X;
  uint32_t nt = 0;
  for (uint64_t i = g->off[X][x]; i < g->off[X][x + 1]; i++) {
    uint32_t y = g->adj[X][i];
    for (uint64_t j = g->off[Y][y]; j < g->off[Y][y + 1]; j++) {
      uint32_t x2 = g->adj[Y][j];
      if (x2 == x) continue;
      if (g->cnt[x2]++ == 0) g->touched[nt++] = x2;
    }
  }
  return nt;
}
static void reset_counts(orc_graph* g, uint32_t nt) {
  for (uint32_t t = 0; t < nt; t++) g->cnt[g->touched[t]] = 0;
}
static inline u128 choose2(uint64_t c) { return (u128)c * (c - (c > 0)) / 2; }

/*
 * Enumerate x in [x_lo, x_hi) of side X (0 = U, 1 = V), following SURVEY
 * 8(c) step 3.  Outputs (each may be NULL, and each is ADDED to, so shards
 * can be summed):
 *   bx   [n_X]  b(x) for x in range (Eq. 1)
 *   by   [n_Y]  centre-rule partial sums (equal to Eq. 1 once all x are done)
 *   be   [m]    b(e) for edges whose X-endpoint is in range (Eq. 2)
 *   sum_bx      Σ b(x) over the range (= 2T when the range is all of X)
 * Returns ORC_EOVERFLOW if any value reaches 2^64.
 */
int orc_count(orc_graph* g, int X, uint32_t x_lo, uint32_t x_hi,
              uint64_t* bx, uint64_t* by, uint64_t* be, uint64_t* sum_bx) {
  if (X < 0 || X > 1 || x_hi > g->n[X] || x_lo > x_hi) return ORC_EINVAL;
  int Y = 1 - X;
  const u128 LIM = (u128)1 << 64;
  u128 total2 = 0;
  for (uint32_t x = x_lo; x < x_hi; x++) {
    uint32_t nt = common_neighbour_counts(g, X, x);
    /* Eq. (1) for x */
    u128 b = 0;
    for (uint32_t t = 0; t < nt; t++) b += choose2(g->cnt[g->touched[t]]);
    if (bx) { u128 s = (u128)bx[x] + b; if (s >= LIM) { reset_counts(g, nt); return ORC_EOVERFLOW; } bx[x] = (uint64_t)s; }
    total2 += b;
    for (uint64_t i = g->off[X][x]; i < g->off[X][x + 1]; i++) {
      uint32_t y = g->adj[X][i];
      u128 e_sum = 0, c_sum = 0;
      for (uint64_t j = g->off[Y][y]; j < g->off[Y][y + 1]; j++) {
        uint32_t x2 = g->adj[Y][j];
        if (x2 == x) continue;
        uint64_t c = g->cnt[x2]; /* >= 1: y is a common neighbour */
        e_sum += c - 1;                 /* Eq. (2) */
        if (x2 > x) c_sum += c - 1;     /* centre rule */
      }
      if (be) { u128 s = (u128)be[g->eid[X][i]] + e_sum; if (s >= LIM) { reset_counts(g, nt); return ORC_EOVERFLOW; } be[g->eid[X][i]] = (uint64_t)s; }
      if (by) { u128 s = (u128)by[y] + c_sum; if (s >= LIM) { reset_counts(g, nt); return ORC_EOVERFLOW; } by[y] = (uint64_t)s; }
    }
    reset_counts(g, nt);
  }
  if (total2 >= LIM) return ORC_EOVERFLOW;
  if (sum_bx) *sum_bx = (uint64_t)total2;
  return ORC_OK;
}

/* Enumeration-side choice: X = U if Σ_V deg² <= Σ_U deg²,
 * else V.  Only selects which symmetric identity is evaluated (cost). */
int orc_cheap_side(const orc_graph* g) {
  u128 s[2] = {0, 0};
  for (int side = 0; side < 2; side++)
    for (uint32_t x = 0; x < g->n[side]; x++) { uint64_t d = orc_degree(g, side, x); s[side] += (u128)d * d; }
  return s[1] <= s[0] ? 0 : 1;
}

/* Eq. (1) for one vertex (sampled parity at full size). */
int orc_vertex(orc_graph* g, int side, uint32_t x, uint64_t* out) {
  if (side < 0 || side > 1 || x >= g->n[side]) return ORC_EINVAL;
  uint32_t nt = common_neighbour_counts(g, side, x);
  u128 b = 0;
  for (uint32_t t = 0; t < nt; t++) b += choose2(g->cnt[g->touched[t]]);
  reset_counts(g, nt);
  if (b >> 64) return ORC_EOVERFLOW;
  *out = (uint64_t)b;
  return ORC_OK;
}

/* Eq. (2) for one input edge e = (u,v): Σ_{u'∈N(v)\{u}} (c(u,u') - 1). */
int orc_edge(orc_graph* g, const uint32_t* edges, uint64_t e, uint64_t* out) {
  if (e >= g->m) return ORC_EINVAL;
  uint32_t u = edges[2 * e], v = edges[2 * e + 1];
  uint32_t nt = common_neighbour_counts(g, 0, u);
  u128 b = 0;
  for (uint64_t j = g->off[1][v]; j < g->off[1][v + 1]; j++) {
    uint32_t u2 = g->adj[1][j];
    if (u2 == u) continue;
    b += (u128)g->cnt[u2] - 1;
  }
  reset_counts(g, nt);
  if (b >> 64) return ORC_EOVERFLOW;
  *out = (uint64_t)b;
  return ORC_OK;
}

/* ------------------------------------------------------------------------
 * Rankings (§3.1.1) over global ids gid = u (U) or nU+v (V).
 * rank_out[gid] = position in the order (0 = first = processed as the
 * lowest-ranked endpoint; reading Z4).
 *   kind 0 side:    the side whose vertices, as endpoints, give fewer
 *                   wedges goes first: U first iff Σ_{v∈V} C(deg v,2) <=
 *                   Σ_{u∈U} C(deg u,2) (reading Z1; tie -> U); gid order
 *                   inside a side.
 *   kind 1 approx:  decreasing floor(log2 deg) (deg 0 -> -1), ties by gid
 *                   (readings Z2, Z3).
 *   kind 2 degree:  decreasing degree, ties by gid (reading Z2).
 *   kind 3 explicit: rank_out is an input (a permutation), left as is.
 *   kind 4 approximate complement degeneracy:
 *                   "repeatedly removes vertices of largest log-degree" --
 *                   each round removes ALL remaining vertices whose
 *                   floor(log2 of the degree in the subgraph induced on the
 *                   remaining vertices) equals the current maximum (deg 0 ->
 *                   -1), then lowers their remaining neighbours' degrees;
 *                   vertices removed in earlier rounds rank first, ties by
 *                   gid (readings Z2, Z3, Z16).
 * --------------------------------------------------------------------- */
static int64_t floor_log2(uint64_t d) { int64_t l = -1; while (d) { l++; d >>= 1; } return l; }
static int rank_approx_codegen(const orc_graph* g, uint32_t* rank_out) {
  uint64_t nU = g->n[0], n = nU + g->n[1];
  uint64_t* cur = (uint64_t*)malloc((n ? n : 1) * 8);
  uint8_t* alive = (uint8_t*)malloc(n ? n : 1);
  uint8_t* dying = (uint8_t*)malloc(n ? n : 1);
  if (!cur || !alive || !dying) { free(cur); free(alive); free(dying); return ORC_ENOMEM; }
  for (uint64_t z = 0; z < n; z++) {
    cur[z] = z < nU ? orc_degree(g, 0, (uint32_t)z) : orc_degree(g, 1, (uint32_t)(z - nU));
    alive[z] = 1;
  }
  uint64_t next = 0, left = n;
  while (left) {
    int64_t B = -2;
    for (uint64_t z = 0; z < n; z++)
      if (alive[z] && floor_log2(cur[z]) > B) B = floor_log2(cur[z]);
    for (uint64_t z = 0; z < n; z++) {  /* this round's vertices, in gid order */
      dying[z] = alive[z] && floor_log2(cur[z]) == B;
      if (dying[z]) rank_out[z] = (uint32_t)next++;
    }
    for (uint64_t z = 0; z < n; z++) {
      if (!dying[z]) continue;
      alive[z] = 0;
      left--;
    }
    for (uint64_t z = 0; z < n; z++) {  /* remaining neighbours lose the removed vertices */
      if (!dying[z]) continue;
      int X = z < nU ? 0 : 1, Y = 1 - X;
      uint32_t x = (uint32_t)(X ? z - nU : z);
      for (uint64_t i = g->off[X][x]; i < g->off[X][x + 1]; i++) {
        uint64_t gy = Y ? nU + g->adj[X][i] : g->adj[X][i];
        if (alive[gy]) cur[gy]--;
      }
    }
  }
  free(cur); free(alive); free(dying);
  return ORC_OK;
}
static int64_t* g_sort_key; /* qsort comparator context (single-threaded) */
static int cmp_by_key(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  if (g_sort_key[x] != g_sort_key[y]) return g_sort_key[x] > g_sort_key[y] ? -1 : 1; /* decreasing key */
  return x < y ? -1 : x > y; /* ties: increasing gid */
}

int orc_rank(const orc_graph* g, int kind, uint32_t* rank_out) {
  uint64_t nU = g->n[0], n = (uint64_t)g->n[0] + g->n[1];
  if (kind == 3) return ORC_OK;
  if (kind == 4) return rank_approx_codegen(g, rank_out);
  if (kind < 0 || kind > 4) return ORC_EINVAL;
  int64_t* key = (int64_t*)malloc((n ? n : 1) * 8);
  uint32_t* order = (uint32_t*)malloc((n ? n : 1) * 4);
  if (kind == 0) {
    u128 wU = 0, wV = 0; /* wedges with U endpoints are centred in V, and vice versa */
    for (uint32_t v = 0; v < g->n[1]; v++) wU += choose2(orc_degree(g, 1, v));
    for (uint32_t u = 0; u < g->n[0]; u++) wV += choose2(orc_degree(g, 0, u));
    int u_first = wU <= wV;
    for (uint64_t z = 0; z < n; z++) key[z] = (z < nU) == u_first ? 1 : 0;
  } else {
    for (uint64_t z = 0; z < n; z++) {
      uint64_t d = z < nU ? orc_degree(g, 0, (uint32_t)z) : orc_degree(g, 1, (uint32_t)(z - nU));
      key[z] = kind == 2 ? (int64_t)d : floor_log2(d);
    }
  }
  for (uint64_t z = 0; z < n; z++) order[z] = (uint32_t)z;
  g_sort_key = key;
  qsort(order, n, 4, cmp_by_key);
  for (uint64_t i = 0; i < n; i++) rank_out[order[i]] = (uint32_t)i;
  free(key); free(order);
  return ORC_OK;
}

/* Wedges processed under a ranking: for every x1, every neighbour y with
 * rank(y) > rank(x1), every neighbour x2 of y with rank(x2) > rank(x1)
 * (Alg. 2; W = Σ_x Σ_{y∈N_x(x)} deg_x(y)).
 * w_out[gid] (may be NULL) receives the per-start-vertex count. */
int orc_wedges(const orc_graph* g, const uint32_t* rank, uint64_t* w_out, uint64_t* total) {
  uint64_t nU = g->n[0], n = nU + g->n[1];
  u128 W = 0;
  for (uint64_t z = 0; z < n; z++) {
    int X = z < nU ? 0 : 1, Y = 1 - X;
    uint32_t x = (uint32_t)(X ? z - nU : z);
    uint64_t rx = rank[z], w = 0;
    for (uint64_t i = g->off[X][x]; i < g->off[X][x + 1]; i++) {
      uint32_t y = g->adj[X][i];
      uint64_t gy = Y ? nU + y : y;
      if (rank[gy] <= rx) continue;
      for (uint64_t j = g->off[Y][y]; j < g->off[Y][y + 1]; j++) {
        uint32_t x2 = g->adj[Y][j];
        uint64_t g2 = X ? nU + x2 : x2;
        if (rank[g2] > rx) w++;
      }
    }
    if (w_out) w_out[z] = w;
    W += w;
  }
  if (W >> 64) return ORC_EOVERFLOW;
  *total = (uint64_t)W;
  return ORC_OK;
}

/* ------------------------------------------------------------------------
 * Sparsification (§4.4), written out from the
 * definition for the approximate-counting pins; the counter-based generator
 * is the published splitmix64 step, restated here (not shared with the CUDA
 * path): h(s, x) = mix(s + (x+1)*0x9E3779B97F4A7C15).
 *   method 0 (edge):   keep edge e iff h(seed, e) < p*2^64 (keep_all: p = 1)
 *   method 1 (colour): colour(z) = h(seed ^ 0xD1B54A32D192ED03, gid z) mod c;
 *                      keep an edge iff both endpoints have the same colour
 * keep[e] receives 0/1.
 */
static uint64_t splitmix_out(uint64_t state) {
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t orc_h64(uint64_t seed, uint64_t x) { return splitmix_out(seed + (x + 1) * 0x9E3779B97F4A7C15ull); }

int orc_sparsify(uint32_t nU, const uint32_t* edges, uint64_t m, int method, uint64_t thr, int keep_all,
                 uint32_t colors, uint64_t seed, uint8_t* keep) {
  if (method != 0 && method != 1) return ORC_EINVAL;
  if (method == 1 && colors == 0) return ORC_EINVAL;
  for (uint64_t e = 0; e < m; e++) {
    if (method == 0) {
      keep[e] = keep_all || orc_h64(seed, e) < thr;
    } else {
      uint64_t s2 = seed ^ 0xD1B54A32D192ED03ull;
      uint64_t cu = orc_h64(s2, edges[2 * e]) % colors;
      uint64_t cv = orc_h64(s2, (uint64_t)nU + edges[2 * e + 1]) % colors;
      keep[e] = cu == cv;
    }
  }
  return ORC_OK;
}
