/*
 * crosscheck.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * An independent, fast CPU computation of the full per-edge table of the
 * reference's _micro_edge (census.py:190-256; columns RAW_MICRO_FIELDS,
 * census.py:95-97) and of the 13 CensusSums of _census_batch
 * (census.py:437-466), for graphs where the literal restatement
 * (census_oracle.c, cost sum_e d(lo) + S(lo): 2e13 reads at R-MAT-20, 5e14 at
 * the 4M-vertex Chung-Lu graph) cannot finish.
 *
 * It shares no code with the B200 kernels and uses different enumerations:
 *   pass 1  degree-oriented triangle / 4-clique listing with two mark arrays
 *           (each triangle a<x<y and each 4-clique a<x<y<z exactly once):
 *           t(e), cl(e), T(x);
 *   pass 2  the same triangle listing again: per edge (u, v) the sums over its
 *           triangle set Tri_e of t(u, w), t(v, w) and d(w);
 *   pass 3  per centre vertex c a dense common-neighbour array c(c, x)
 *           (cost sum_v d(v)^2); per edge (lo, c) the 4-cycles through it
 *           C4(e) = sum_{x in N(lo) - c} (c(c, x) - 1);
 *   pass 4  the ten fields from the reference's own per-edge formulas
 *           (census.py:246-250: ti = tdeg - 2t - 2cl - ts,
 *           si = sdeg - su - sv - ts - 2(uu + vv) - 2cy) and the marks
 *           identities  ts_u = sum t(u,w) - 2cl - t,  uu = T(u) - t - cl - ts_u,
 *           cy = C4(e) - ts - 2cl  (DESIGN.md section 2 derives them).
 * Pinned against the literal oracle (itself pinned to the reference) by
 * tests/test_crosscheck.py on the dense / C1 / C2 cases and on the C3 samples.
 */
#include <omp.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

typedef struct {
  int64_t n, m;
  int64_t* ip;    /* [n+1] full CSR */
  int32_t* adj;   /* [2m] ascending */
  int32_t* deg;   /* [n] */
  int64_t* op;    /* [n+1] oriented CSR: higher (degree, id) neighbours */
  int32_t* oadj;  /* [m] */
  int32_t* oeid;  /* [m] canonical edge id of each oriented slot */
} XG;

static int cmp_pair(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

static inline int higher(const XG* g, int32_t a, int32_t b) { /* b above a */
  return g->deg[b] > g->deg[a] || (g->deg[b] == g->deg[a] && b > a);
}

static int xg_build(XG* g, const int64_t* edges, int64_t m, int64_t n) {
  memset(g, 0, sizeof(*g));
  g->n = n;
  g->m = m;
  g->ip = calloc((size_t)n + 1, 8);
  g->adj = malloc(4 * (size_t)(2 * m + 1));
  g->deg = calloc((size_t)n + 1, 4);
  g->op = calloc((size_t)n + 1, 8);
  g->oadj = malloc(4 * (size_t)(m + 1));
  g->oeid = malloc(4 * (size_t)(m + 1));
  int64_t* pos = malloc(8 * (size_t)(n + 1));
  int64_t* tmp = malloc(8 * (size_t)(2 * m + 1));
  if (!g->ip || !g->adj || !g->deg || !g->op || !g->oadj || !g->oeid || !pos || !tmp) return -1;
  for (int64_t e = 0; e < m; e++) {
    int64_t u = edges[2 * e], v = edges[2 * e + 1];
    if (u < 0 || v < 0 || u >= n || v >= n || u >= v) return -2;
    g->deg[u]++;
    g->deg[v]++;
  }
  for (int64_t v = 0; v < n; v++) g->ip[v + 1] = g->ip[v] + g->deg[v];
  memcpy(pos, g->ip, 8 * (size_t)n);
  for (int64_t e = 0; e < m; e++) {
    int32_t u = (int32_t)edges[2 * e], v = (int32_t)edges[2 * e + 1];
    g->adj[pos[u]++] = v;
    g->adj[pos[v]++] = u;
  }
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < n; v++) {
    int64_t b = g->ip[v], d = g->ip[v + 1] - b;
    for (int64_t i = 0; i < d; i++) tmp[b + i] = g->adj[b + i];
    qsort(tmp + b, (size_t)d, 8, cmp_pair);
    for (int64_t i = 0; i < d; i++) g->adj[b + i] = (int32_t)tmp[b + i];
  }
  /* oriented rows, (neighbour << 32 | edge id) sorted by neighbour id */
  for (int64_t e = 0; e < m; e++) {
    int32_t u = (int32_t)edges[2 * e], v = (int32_t)edges[2 * e + 1];
    int32_t lo = higher(g, u, v) ? u : v;
    g->op[lo + 1]++;
  }
  for (int64_t v = 0; v < n; v++) g->op[v + 1] += g->op[v];
  memcpy(pos, g->op, 8 * (size_t)n);
  for (int64_t e = 0; e < m; e++) {
    int32_t u = (int32_t)edges[2 * e], v = (int32_t)edges[2 * e + 1];
    int32_t lo = higher(g, u, v) ? u : v, hi = lo == u ? v : u;
    tmp[pos[lo]++] = ((int64_t)hi << 32) | e;
  }
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < n; v++) {
    int64_t b = g->op[v], d = g->op[v + 1] - b;
    qsort(tmp + b, (size_t)d, 8, cmp_pair);
    for (int64_t i = 0; i < d; i++) {
      g->oadj[b + i] = (int32_t)(tmp[b + i] >> 32);
      g->oeid[b + i] = (int32_t)(tmp[b + i] & 0xffffffff);
    }
  }
  free(pos);
  free(tmp);
  return 0;
}

static void xg_free(XG* g) {
  free(g->ip);
  free(g->adj);
  free(g->deg);
  free(g->op);
  free(g->oadj);
  free(g->oeid);
}

#define ADD(p, v) __atomic_fetch_add((p), (v), __ATOMIC_RELAXED)

/* pass 1 (sums == NULL): t, cl, T.  pass 2: per-edge triangle-set sums. */
static void triangle_pass(const XG* g, const int64_t* edges, int64_t* t, int64_t* cl, int64_t* T,
                          int64_t* sum_u, int64_t* sum_v, int64_t* tdeg, int threads) {
  const int64_t n = g->n;
  const int second = sum_u != NULL;
#pragma omp parallel num_threads(threads)
  {
    int32_t* mk1 = malloc(4 * (size_t)n);  /* edge id + 1 of (a, x), x in N+(a) */
    int32_t* mk2 = malloc(4 * (size_t)n);  /* edge id + 1 of (x, y), y in N+(a) & N+(x) */
    int32_t* L = malloc(4 * (size_t)n);
    /* membership bitmaps in front of mk1 / mk2: n bits stay cache-resident
       where the n-int arrays do not (most probes are misses) */
    uint64_t* bm1 = calloc((size_t)(n >> 6) + 1, 8);
    uint64_t* bm2 = calloc((size_t)(n >> 6) + 1, 8);
    memset(mk1, 0, 4 * (size_t)n);
    memset(mk2, 0, 4 * (size_t)n);
#pragma omp for schedule(dynamic, 64)
    for (int64_t a = 0; a < n; a++) {
      const int64_t b = g->op[a], e_ = g->op[a + 1];
      if (e_ - b < 2) continue;
      for (int64_t i = b; i < e_; i++) {
        mk1[g->oadj[i]] = g->oeid[i] + 1;
        bm1[g->oadj[i] >> 6] |= 1ull << (g->oadj[i] & 63);
      }
      for (int64_t i = b; i < e_; i++) {
        const int32_t x = g->oadj[i], eax = g->oeid[i];
        int64_t nl = 0;
        for (int64_t j = g->op[x]; j < g->op[x + 1]; j++) {
          const int32_t y = g->oadj[j];
          if (!((bm1[y >> 6] >> (y & 63)) & 1)) continue;
          const int32_t exy = g->oeid[j], eay = mk1[y] - 1;
          /* triangle {a, x, y} */
          if (!second) {
            ADD(&t[eax], 1);
            ADD(&t[eay], 1);
            ADD(&t[exy], 1);
            ADD(&T[a], 1);
            ADD(&T[x], 1);
            ADD(&T[y], 1);
            mk2[y] = exy + 1;
            bm2[y >> 6] |= 1ull << (y & 63);
            L[nl++] = y;
          } else {
            /* edge (p, q) with third vertex r: t(p, r) to p's side,
               t(q, r) to q's side, d(r) to tdeg */
            const int32_t P_[3] = {(int32_t)a, (int32_t)a, x};
            const int32_t R_[3] = {y, x, (int32_t)a};
            const int32_t E_[3] = {eax, eay, exy};
            const int32_t EPR[3] = {eay, eax, eax};
            const int32_t EQR[3] = {exy, exy, eay};
            for (int k = 0; k < 3; k++) {
              const int32_t e = E_[k];
              const int64_t tp = t[EPR[k]], tq = t[EQR[k]];
              const int p_is_u = edges[2 * (int64_t)e] == P_[k];
              ADD(&sum_u[e], p_is_u ? tp : tq);
              ADD(&sum_v[e], p_is_u ? tq : tp);
              ADD(&tdeg[e], (int64_t)g->deg[R_[k]]);
            }
          }
        }
        if (second) continue;
        /* 4-cliques {a, x, y, z}: z in N+(y) with z in N+(a) & N+(x) */
        for (int64_t li = 0; li < nl; li++) {
          const int32_t y = L[li];
          const int32_t eay = mk1[y] - 1, exy = mk2[y] - 1;
          for (int64_t j = g->op[y]; j < g->op[y + 1]; j++) {
            const int32_t z = g->oadj[j];
            if (!((bm2[z >> 6] >> (z & 63)) & 1)) continue;
            ADD(&cl[eax], 1);
            ADD(&cl[eay], 1);
            ADD(&cl[mk1[z] - 1], 1);
            ADD(&cl[exy], 1);
            ADD(&cl[mk2[z] - 1], 1);
            ADD(&cl[g->oeid[j]], 1);
          }
        }
        for (int64_t li = 0; li < nl; li++) {
          mk2[L[li]] = 0;
          bm2[L[li] >> 6] = 0;
        }
      }
      for (int64_t i = b; i < e_; i++) {
        mk1[g->oadj[i]] = 0;
        bm1[g->oadj[i] >> 6] = 0;
      }
    }
    free(mk1);
    free(mk2);
    free(bm1);
    free(bm2);
    free(L);
  }
}

/* pass 3: C4(e) for every edge, from the higher endpoint's common-neighbour
 * counts c(c, x).  Centres with a small 2-hop volume S(c) use one dense
 * n-sized array; for the rest the x range is cut into tiles of 2^18 counters
 * (1 MB, cache-resident) walked with per-row cursors -- the same counts, but
 * a 4M-vertex graph's 1.4e12 increments no longer each miss the cache. */
static void cycle_pass(const XG* g, int64_t* c4, int threads) {
  const int64_t n = g->n;
  /* tile size and the S(c) above which a centre is tiled (tests shrink both) */
  const char* ev = getenv("XC_TILE");
  const int64_t XT_TILE = ev ? atoll(ev) : (1 << 18);
  ev = getenv("XC_TILE_S");
  const int64_t XT_S = ev ? atoll(ev) : 4 * XT_TILE;
#pragma omp parallel num_threads(threads)
  {
    uint32_t* cnt = calloc((size_t)n, 4);
    uint32_t* tile = calloc((size_t)XT_TILE, 4);
    int64_t* curw = NULL;
    int64_t* curl = NULL;
    int64_t* acc = NULL;
    int32_t* lows = NULL;
    int64_t cap = 0;
#pragma omp for schedule(dynamic, 16)
    for (int64_t c = 0; c < n; c++) {
      const int64_t b = g->ip[c], e_ = g->ip[c + 1], dc = e_ - b;
      int64_t nlow = 0, S = 0;
      for (int64_t i = b; i < e_; i++) {
        nlow += higher(g, g->adj[i], (int32_t)c);
        S += g->deg[g->adj[i]];
      }
      if (!nlow) continue;
      if (S <= XT_S) {
        for (int64_t i = b; i < e_; i++) {
          const int32_t w = g->adj[i];
          for (int64_t j = g->ip[w]; j < g->ip[w + 1]; j++) cnt[g->adj[j]]++;
        }
      }
      if (dc > cap) {
        cap = dc;
        curw = realloc(curw, 8 * (size_t)cap);
        curl = realloc(curl, 8 * (size_t)cap);
        acc = realloc(acc, 8 * (size_t)cap);
        lows = realloc(lows, 4 * (size_t)cap);
      }
      nlow = 0;
      for (int64_t i = b; i < e_; i++)
        if (higher(g, g->adj[i], (int32_t)c)) lows[nlow++] = g->adj[i];
      if (S <= XT_S) {
        for (int64_t k = 0; k < nlow; k++) {
          const int32_t lo = lows[k];
          int64_t s = 0;
          for (int64_t j = g->ip[lo]; j < g->ip[lo + 1]; j++) {
            const int32_t x = g->adj[j];
            if (x != c) s += (int64_t)cnt[x] - 1;
          }
          acc[k] = s;
        }
        for (int64_t i = b; i < e_; i++) {
          const int32_t w = g->adj[i];
          for (int64_t j = g->ip[w]; j < g->ip[w + 1]; j++) cnt[g->adj[j]] = 0;
        }
      } else {
        for (int64_t i = 0; i < dc; i++) curw[i] = g->ip[g->adj[b + i]];
        for (int64_t k = 0; k < nlow; k++) {
          curl[k] = g->ip[lows[k]];
          acc[k] = 0;
        }
        for (int64_t x0 = 0; x0 < n; x0 += XT_TILE) {
          const int64_t x1 = x0 + XT_TILE;
          for (int64_t i = 0; i < dc; i++) {
            const int32_t w = g->adj[b + i];
            int64_t p = curw[i];
            const int64_t pe = g->ip[w + 1];
            for (; p < pe && g->adj[p] < x1; p++) tile[g->adj[p] - x0]++;
            curw[i] = p;
          }
          for (int64_t k = 0; k < nlow; k++) {
            const int32_t lo = lows[k];
            int64_t p = curl[k], s = 0;
            const int64_t pe = g->ip[lo + 1];
            for (; p < pe && g->adj[p] < x1; p++) {
              const int32_t x = g->adj[p];
              if (x != c) s += (int64_t)tile[x - x0] - 1;
            }
            curl[k] = p;
            acc[k] += s;
          }
          memset(tile, 0, 4 * (size_t)XT_TILE);
        }
      }
      for (int64_t k = 0; k < nlow; k++) {
        /* edge id of (lo, c): lo's oriented row holds c */
        const int32_t lo = lows[k];
        int64_t a = g->op[lo], z = g->op[lo + 1];
        while (a < z) {
          int64_t mid = (a + z) >> 1;
          if (g->oadj[mid] < c) a = mid + 1; else z = mid;
        }
        c4[g->oeid[a]] = acc[k];
      }
    }
    free(cnt);
    free(tile);
    free(curw);
    free(curl);
    free(acc);
    free(lows);
  }
}

/*
 * Full per-edge table (rows int64 [m][10], canonical edge order, columns
 * RAW_MICRO_FIELDS) and the 13 CensusSums (u64 [13][2]) of a canonical
 * (lexicographic, u < v) edge list.
 */
int crosscheck_table(const int64_t* edges, int64_t m, int64_t n, int threads, int64_t* rows,
                     uint64_t* sums) {
  XG g;
  int rc = xg_build(&g, edges, m, n);
  if (rc) {
    xg_free(&g);
    return rc;
  }
  const int T_ = threads > 0 ? threads : omp_get_max_threads();
  int64_t* t = calloc((size_t)m + 1, 8);
  int64_t* cl = calloc((size_t)m + 1, 8);
  int64_t* su = calloc((size_t)m + 1, 8);
  int64_t* sv = calloc((size_t)m + 1, 8);
  int64_t* td = calloc((size_t)m + 1, 8);
  int64_t* c4 = calloc((size_t)m + 1, 8);
  int64_t* T = calloc((size_t)n + 1, 8);
  int64_t* S = calloc((size_t)n + 1, 8);
  u128* acc = calloc((size_t)T_ * 13, sizeof(u128));
  if (!t || !cl || !su || !sv || !td || !c4 || !T || !S || !acc) return -1;
  const int verbose = getenv("XC_VERBOSE") != NULL;
  double t0 = omp_get_wtime();
  triangle_pass(&g, edges, t, cl, T, NULL, NULL, NULL, T_);
  if (verbose) fprintf(stderr, "crosscheck: triangles + 4-cliques %.1f s\n", omp_get_wtime() - t0);
  triangle_pass(&g, edges, t, cl, T, su, sv, td, T_);
  if (verbose) fprintf(stderr, "crosscheck: triangle-set sums %.1f s\n", omp_get_wtime() - t0);
  cycle_pass(&g, c4, T_);
  if (verbose) fprintf(stderr, "crosscheck: 4-cycles %.1f s\n", omp_get_wtime() - t0);
#pragma omp parallel for num_threads(T_) schedule(static, 4096)
  for (int64_t v = 0; v < n; v++) {
    int64_t s = 0;
    for (int64_t i = g.ip[v]; i < g.ip[v + 1]; i++) s += g.deg[g.adj[i]];
    S[v] = s;
  }
#pragma omp parallel num_threads(T_)
  {
    u128* a = acc + 13 * omp_get_thread_num();
#pragma omp for schedule(static, 8192)
    for (int64_t e = 0; e < m; e++) {
      const int64_t u = edges[2 * e], v = edges[2 * e + 1];
      const int64_t du = g.deg[u], dv = g.deg[v];
      const int64_t te = t[e], c = cl[e];
      const int64_t s_u = du - 1 - te, s_v = dv - 1 - te;
      const int64_t tsu = su[e] - 2 * c - te, tsv = sv[e] - 2 * c - te, ts = tsu + tsv;
      const int64_t uu = T[u] - te - c - tsu, vv = T[v] - te - c - tsv;
      const int64_t cy = c4[e] - ts - 2 * c;
      const int64_t sdeg = S[u] - dv + S[v] - du - 2 * td[e];
      const int64_t ti = td[e] - 2 * te - 2 * c - ts;
      const int64_t si = sdeg - s_u - s_v - ts - 2 * (uu + vv) - 2 * cy;
      int64_t* r = rows + 10 * e;
      r[0] = te; r[1] = s_u; r[2] = s_v; r[3] = c; r[4] = cy;
      r[5] = uu; r[6] = vv; r[7] = ts; r[8] = ti; r[9] = si;
      /* _census_batch (census.py:449-462) */
      const int64_t i3 = n - 2 - te - s_u - s_v;
      a[0] += (u128)te;
      a[1] += (u128)(s_u + s_v);
      a[2] += (u128)i3;
      a[3] += (u128)c;
      a[4] += (u128)cy;
      a[5] += (u128)(te * (te - 1) / 2);
      a[6] += (u128)s_u * (u128)s_v;
      a[7] += (u128)te * (u128)(s_u + s_v);
      a[8] += (u128)(s_u * (s_u - 1) / 2 + s_v * (s_v - 1) / 2);
      a[9] += (u128)te * (u128)i3;
      a[10] += (u128)(s_u + s_v) * (u128)i3;
      a[11] += (u128)i3 * (u128)(i3 - 1) / 2;
      a[12] += (u128)(m + 1 - (te + s_u + 1) - (te + s_v + 1));
    }
  }
  for (int k = 0; k < 13; k++) {
    u128 s = 0;
    for (int i = 0; i < T_; i++) s += acc[13 * i + k];
    sums[2 * k] = (uint64_t)s;
    sums[2 * k + 1] = (uint64_t)(s >> 64);
  }
  free(t); free(cl); free(su); free(sv); free(td); free(c4); free(T); free(S); free(acc);
  xg_free(&g);
  return 0;
}
