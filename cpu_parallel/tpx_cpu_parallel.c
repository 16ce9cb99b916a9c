/*
 * tpx_cpu_parallel.c -- the paper's multi-core CPU clustering, as a
 * comparator for the GPU path.  Not the oracle (which is
 * the plain single-threaded definition, oracle/) and not the product (the
 * sm_100a library): a stronger CPU baseline, timed beside them in bench.py.
 * It shares no code with either.
 *
 * Method (§3.2 "Data-based parallelization", §3.2.3 "Temporal
 * splitting" l.117-119, §3.3 "Merging split clusters" l.121-139, Alg. 1
 * "High-level data-driven clustering" l.75-87):
 *   1. temporal splitting: hits are partitioned into time windows of
 *      window_ticks by their ToA (counting sort, input order kept inside a
 *      window); windows go to the worker threads round-robin (l.117);
 *   2. per window: time sorting (l.99-101; the window's hits by (toa, index))
 *      and Alg. 1 with the per-pixel reference matrix of the latest hit
 *      ("store references ... for each pixel in the matrix", l.71): a hit
 *      joins the clusters of the latest hits on its 9 pixels that are within
 *      dt_max (reading R2: same pixel included) and merges them;
 *   3. border clusters (within dt_max of a window border, l.123) are merged
 *      per border time by parallel merge workers (l.135-139) with the
 *      three-step cascade (l.127-133): (1) temporal distance <= dt_max,
 *      (2) bounding boxes (grown by one pixel) intersect, (3) the larger
 *      cluster's hits in the box intersection go into a 2D array and every
 *      hit of the smaller cluster is checked against its 9 neighbour pixels;
 *   4. labels (smallest input index of the merged cluster, reading R6) and the
 *      64-byte feature records in ascending label order (reading R7), the
 *      same output contract as tpx_cluster_run.
 * The latest-hit-per-pixel rule gives exactly the connected components of
 * definition (iii)(a): an older hit g on pixel p within dt_max of h is
 * connected to h through the latest hit on p before h (same pixel, between
 * them in time).  So the result is bit-identical to the oracle
 * (tests/test_cpu_parallel.py).
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct phit {
  uint64_t toa;
  uint16_t x, y, tot, reserved;
} phit;

typedef struct pfeat {
  uint32_t label, size;
  uint64_t toa_min, toa_max, tot_sum, sum_x, sum_y, sum_tot_x, sum_tot_y;
} pfeat;

typedef struct pstats {
  uint64_t windows, clusters, border_clusters, border_checks, bbox_checks, full_checks, merges;
} pstats;

enum { P_OK = 0, P_ERR_ARG = -1, P_ERR_COORD = -3, P_ERR_OOM = -6 };

/* ------------------------------------------------------- thread helpers */
typedef struct job {
  void (*fn)(void* ctx, int tid, int nthreads);
  void* ctx;
  int tid, nthreads;
} job;

static void* job_main(void* a) {
  job* j = (job*)a;
  j->fn(j->ctx, j->tid, j->nthreads);
  return NULL;
}

static void parallel(int nthreads, void (*fn)(void*, int, int), void* ctx) {
  pthread_t th[256];
  job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (job){fn, ctx, t, nthreads};
    if (t) pthread_create(&th[t], NULL, job_main, &jobs[t]);
  }
  job_main(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------- shared state */
typedef struct run {
  const phit* h;
  uint64_t n, dt, wticks;
  uint32_t W, H;
  int nthreads;
  uint64_t toa_min;
  uint64_t nw;            /* number of time windows                          */
  uint64_t* wcount;       /* [nthreads][nw] per-thread window histograms     */
  uint64_t* wstart;       /* [nw + 1] window offsets into order              */
  uint32_t* order;        /* hit indices grouped by window, then (toa, index) */
  uint32_t* cl_of;        /* [n] by position in order: global cluster id     */
  uint32_t* parent;       /* [n] by position: window-local union-find        */
  /* clusters, allocated per window at [wstart[w], wstart[w] + count)        */
  pfeat* rec;             /* features; label = smallest input index          */
  uint16_t* bbox;         /* [n][4] x_min, x_max, y_min, y_max               */
  uint32_t* mstart;       /* [n + 1] member offsets (by position)            */
  uint32_t* members;      /* [n] positions in order, grouped by cluster      */
  uint32_t* ncl;          /* [nw] clusters of window w                       */
  uint8_t* border;        /* [n] cluster touches a window border             */
  /* merge results */
  uint32_t** pairs;       /* per border worker: (cluster, cluster) pairs     */
  uint64_t* npairs;
  uint64_t* capairs;
  pstats* tstats;         /* [nthreads]                                      */
  int err;
  /* output */
  uint32_t* labels;
  pfeat* feats;
  uint64_t k;
  uint32_t* final_of;     /* [n] merged cluster -> root cluster id            */
  uint64_t* bits;         /* [ceil(n/64)] label bitmap                        */
  uint64_t* wbase;        /* [ceil(n/64) + 1] prefix of set bits              */
} run;

static uint64_t win_of(const run* r, uint64_t toa) { return (toa - r->toa_min) / r->wticks; }

/* 1a. min ToA + coordinate check */
typedef struct minmax_ctx {
  run* r;
  uint64_t mn[256], mx[256];
  int bad[256];
} minmax_ctx;

static void k_minmax(void* c, int t, int T) {
  minmax_ctx* m = (minmax_ctx*)c;
  const run* r = m->r;
  uint64_t a = r->n * t / T, b = r->n * (t + 1) / T, mn = ~0ull, mx = 0;
  int bad = 0;
  for (uint64_t i = a; i < b; ++i) {
    const phit* p = r->h + i;
    if (p->toa < mn) mn = p->toa;
    if (p->toa > mx) mx = p->toa;
    bad |= p->x >= r->W || p->y >= r->H;
  }
  m->mn[t] = mn;
  m->mx[t] = mx;
  m->bad[t] = bad;
}

/* 1b. per-thread window histograms, 1c. scatter (input order kept) */
static void k_hist(void* c, int t, int T) {
  run* r = (run*)c;
  uint64_t a = r->n * t / T, b = r->n * (t + 1) / T;
  uint64_t* cnt = r->wcount + (uint64_t)t * r->nw;
  for (uint64_t i = a; i < b; ++i) cnt[win_of(r, r->h[i].toa)]++;
}

static void k_scatter(void* c, int t, int T) {
  run* r = (run*)c;
  uint64_t a = r->n * t / T, b = r->n * (t + 1) / T;
  uint64_t* cur = r->wcount + (uint64_t)t * r->nw; /* holds this thread's offsets */
  for (uint64_t i = a; i < b; ++i) r->order[cur[win_of(r, r->h[i].toa)]++] = (uint32_t)i;
}

/* 2. per window: time sort + Alg. 1 + cluster records + members */
static __thread const phit* t_cmp_h;
static int cmp_pos(const void* a, const void* b) {
  uint32_t i = *(const uint32_t*)a, j = *(const uint32_t*)b;
  uint64_t ti = t_cmp_h[i].toa, tj = t_cmp_h[j].toa;
  if (ti != tj) return ti < tj ? -1 : 1;
  return (i > j) - (i < j);
}

static uint32_t uf_find(uint32_t* par, uint32_t x) {
  while (par[x] != x) {
    par[x] = par[par[x]];
    x = par[x];
  }
  return x;
}

static void k_windows(void* c, int t, int T) {
  run* r = (run*)c;
  const phit* h = r->h;
  t_cmp_h = h;
  const uint64_t npix = (uint64_t)r->W * r->H;
  /* per-pixel reference matrix: position (in order) of the latest hit, +1 (0 = none) */
  uint64_t* last = (uint64_t*)calloc(npix, sizeof(uint64_t));
  uint32_t* tmp = NULL;
  uint64_t tmp_cap = 0;
  if (!last) {
    r->err = P_ERR_OOM;
    return;
  }
  pstats* st = r->tstats + t;
  for (uint64_t w = (uint64_t)t; w < r->nw; w += (uint64_t)T) {
    const uint64_t a = r->wstart[w], b = r->wstart[w + 1], m = b - a;
    if (!m) continue;
    st->windows++;
    uint32_t* ord = r->order + a;
    qsort(ord, m, sizeof(uint32_t), cmp_pos);  /* time sorting (l.99-101) */
    uint32_t* par = r->parent + a;             /* local positions 0..m-1 */
    for (uint64_t p = 0; p < m; ++p) par[p] = (uint32_t)p;
    /* Alg. 1: findNeighborClusters through the latest hit of each of the 9 pixels */
    for (uint64_t p = 0; p < m; ++p) {
      const phit* hp = h + ord[p];
      for (int dy = -1; dy <= 1; ++dy) {
        const int y = (int)hp->y + dy;
        if (y < 0 || y >= (int)r->H) continue;
        for (int dx = -1; dx <= 1; ++dx) {
          const int x = (int)hp->x + dx;
          if (x < 0 || x >= (int)r->W) continue;
          const uint64_t q1 = last[(uint64_t)y * r->W + x];
          if (q1 <= a) continue; /* none, or a hit of an earlier window */
          const uint64_t q = q1 - 1 - a;
          if (hp->toa - h[ord[q]].toa > r->dt) continue;
          uint32_t ra = uf_find(par, (uint32_t)p), rb = uf_find(par, (uint32_t)q);
          if (ra != rb) { /* addHitToCluster / mergeClusters */
            if (ra < rb) par[rb] = ra; else par[ra] = rb;
          }
        }
      }
      last[(uint64_t)hp->y * r->W + hp->x] = a + p + 1;
    }
    /* clusters of the window: records at [a, a + ncl) */
    uint32_t nc = 0;
    for (uint64_t p = 0; p < m; ++p) {
      const uint32_t root = uf_find(par, (uint32_t)p);
      if (root == p) r->cl_of[a + p] = (uint32_t)(a + nc++);
      else r->cl_of[a + p] = r->cl_of[a + root];  /* root < p: already set */
    }
    r->ncl[w] = nc;
    st->clusters += nc;
    for (uint32_t k = 0; k < nc; ++k) {
      pfeat* f = r->rec + a + k;
      memset(f, 0, sizeof(*f));
      f->label = 0xffffffffu;
      f->toa_min = ~0ull;
      uint16_t* bb = r->bbox + 4 * (a + k);
      bb[0] = bb[2] = 0xffff;
      bb[1] = bb[3] = 0;
      r->mstart[a + k] = 0;
    }
    for (uint64_t p = 0; p < m; ++p) {
      const uint32_t id = r->cl_of[a + p];
      const phit* hp = h + ord[p];
      pfeat* f = r->rec + id;
      if (ord[p] < f->label) f->label = ord[p];
      f->size++;
      if (hp->toa < f->toa_min) f->toa_min = hp->toa;
      if (hp->toa > f->toa_max) f->toa_max = hp->toa;
      f->tot_sum += hp->tot;
      f->sum_x += hp->x;
      f->sum_y += hp->y;
      f->sum_tot_x += (uint64_t)hp->tot * hp->x;
      f->sum_tot_y += (uint64_t)hp->tot * hp->y;
      uint16_t* bb = r->bbox + 4 * (uint64_t)id;
      if (hp->x < bb[0]) bb[0] = hp->x;
      if (hp->x > bb[1]) bb[1] = hp->x;
      if (hp->y < bb[2]) bb[2] = hp->y;
      if (hp->y > bb[3]) bb[3] = hp->y;
      r->mstart[id]++;
    }
    /* member lists (exclusive offsets within the window's range) */
    uint32_t s = 0;
    for (uint32_t k = 0; k < nc; ++k) {
      const uint32_t c0 = r->mstart[a + k];
      r->mstart[a + k] = (uint32_t)a + s;
      s += c0;
    }
    if (tmp_cap < nc) {
      free(tmp);
      tmp_cap = nc * 2;
      tmp = (uint32_t*)malloc(tmp_cap * sizeof(uint32_t));
      if (!tmp) {
        r->err = P_ERR_OOM;
        free(last);
        return;
      }
    }
    for (uint32_t k = 0; k < nc; ++k) tmp[k] = r->mstart[a + k];
    for (uint64_t p = 0; p < m; ++p) r->members[tmp[r->cl_of[a + p] - a]++] = (uint32_t)(a + p);
    /* border clusters (l.123): within dt_max of the window's lower or upper time border */
    const uint64_t lo = r->toa_min + w * r->wticks, hi = lo + r->wticks;
    for (uint32_t k = 0; k < nc; ++k) {
      const pfeat* f = r->rec + a + k;
      const uint8_t bl = f->toa_min < lo + r->dt, bu = f->toa_max + r->dt >= hi;
      r->border[a + k] = (uint8_t)(bl | (bu << 1));
      st->border_clusters += (bl | bu) != 0;
    }
  }
  free(tmp);
  free(last);
}

/* 3. merge workers, one border time each (l.135-139), with the cascade */
typedef struct grid2d {
  uint32_t* head;   /* [gw * gh] first entry + 1 (0 = none)  */
  uint32_t* next;   /* per entry: next + 1                    */
  uint64_t* toa;    /* per entry                              */
  uint64_t cap_cells, cap_entries;
} grid2d;

static int grid_reserve(grid2d* g, uint64_t cells, uint64_t entries) {
  if (cells > g->cap_cells) {
    free(g->head);
    g->head = (uint32_t*)calloc(cells, sizeof(uint32_t));
    g->cap_cells = g->head ? cells : 0;
    if (!g->head) return P_ERR_OOM;
  }
  if (entries > g->cap_entries) {
    free(g->next);
    free(g->toa);
    g->next = (uint32_t*)malloc(entries * sizeof(uint32_t));
    g->toa = (uint64_t*)malloc(entries * sizeof(uint64_t));
    g->cap_entries = (g->next && g->toa) ? entries : 0;
    if (!g->next || !g->toa) return P_ERR_OOM;
  }
  return P_OK;
}

/* cascade steps 2-3 for clusters A and B (step 1 done by the caller) */
static int mergeable(const run* r, uint32_t A, uint32_t B, grid2d* g, pstats* st) {
  const uint16_t* ba = r->bbox + 4 * (uint64_t)A;
  const uint16_t* bb = r->bbox + 4 * (uint64_t)B;
  /* 2. bounding boxes, grown by one pixel (8-neighbourhood), must intersect */
  st->bbox_checks++;
  const int x0 = (int)(ba[0] > bb[0] ? ba[0] : bb[0]) - 1, x1 = (int)(ba[1] < bb[1] ? ba[1] : bb[1]) + 1;
  const int y0 = (int)(ba[2] > bb[2] ? ba[2] : bb[2]) - 1, y1 = (int)(ba[3] < bb[3] ? ba[3] : bb[3]) + 1;
  if (x0 > x1 || y0 > y1) return 0;
  /* 3. larger cluster's hits inside the (grown) intersection -> 2D array;
   * every hit of the smaller one checks its 9 neighbour pixels */
  st->full_checks++;
  const uint32_t sa = r->rec[A].size, sb = r->rec[B].size;
  const uint32_t L = sa >= sb ? A : B, S = sa >= sb ? B : A;
  const int gx0 = x0 - 1, gy0 = y0 - 1, gw = x1 - x0 + 3, gh = y1 - y0 + 3;
  if (grid_reserve(g, (uint64_t)gw * gh, r->rec[L].size)) return -1;
  memset(g->head, 0, (size_t)gw * gh * sizeof(uint32_t));
  uint32_t ne = 0;
  for (uint32_t k = 0; k < r->rec[L].size; ++k) {
    const phit* p = r->h + r->order[r->members[r->mstart[L] + k]];
    if ((int)p->x < x0 || (int)p->x > x1 || (int)p->y < y0 || (int)p->y > y1) continue;
    const uint64_t cell = (uint64_t)((int)p->y - gy0) * gw + ((int)p->x - gx0);
    g->toa[ne] = p->toa;
    g->next[ne] = g->head[cell];
    g->head[cell] = ++ne;
  }
  int found = 0;
  for (uint32_t k = 0; k < r->rec[S].size && !found; ++k) {
    const phit* p = r->h + r->order[r->members[r->mstart[S] + k]];
    if ((int)p->x < x0 || (int)p->x > x1 || (int)p->y < y0 || (int)p->y > y1) continue;
    for (int dy = -1; dy <= 1 && !found; ++dy)
      for (int dx = -1; dx <= 1 && !found; ++dx) {
        const int cx = (int)p->x + dx - gx0, cy = (int)p->y + dy - gy0;
        for (uint32_t e = g->head[(uint64_t)cy * gw + cx]; e; e = g->next[e - 1]) {
          const uint64_t t = g->toa[e - 1];
          const uint64_t d = t > p->toa ? t - p->toa : p->toa - t;
          if (d <= r->dt) {
            found = 1;
            break;
          }
        }
      }
  }
  return found;
}

static void add_pair(run* r, int t, uint32_t a, uint32_t b) {
  if (r->npairs[t] == r->capairs[t]) {
    uint64_t nc = r->capairs[t] ? 2 * r->capairs[t] : 1024;
    uint32_t* np = (uint32_t*)realloc(r->pairs[t], nc * 2 * sizeof(uint32_t));
    if (!np) {
      r->err = P_ERR_OOM;
      return;
    }
    r->pairs[t] = np;
    r->capairs[t] = nc;
  }
  r->pairs[t][2 * r->npairs[t]] = a;
  r->pairs[t][2 * r->npairs[t] + 1] = b;
  r->npairs[t]++;
}

static void k_merge(void* c, int t, int T) {
  run* r = (run*)c;
  grid2d g = {0};
  pstats* st = r->tstats + t;
  uint32_t *lo_set = NULL, *up_set = NULL;
  uint64_t cap = 0;
  for (uint64_t b = (uint64_t)t; b + 1 < r->nw; b += (uint64_t)T) {
    /* border time between window b and b+1 */
    const uint64_t a0 = r->wstart[b], a1 = r->wstart[b + 1];
    const uint32_t n0 = r->ncl[b], n1 = r->ncl[b + 1];
    if (!n0 || !n1) continue;
    if (cap < (uint64_t)n0 + n1) {
      free(lo_set);
      free(up_set);
      cap = 2 * ((uint64_t)n0 + n1);
      lo_set = (uint32_t*)malloc(cap * sizeof(uint32_t));
      up_set = (uint32_t*)malloc(cap * sizeof(uint32_t));
      if (!lo_set || !up_set) {
        r->err = P_ERR_OOM;
        break;
      }
    }
    uint32_t nl = 0, nu = 0;
    for (uint32_t k = 0; k < n0; ++k)
      if (r->border[a0 + k] & 2u) lo_set[nl++] = (uint32_t)(a0 + k);
    for (uint32_t k = 0; k < n1; ++k)
      if (r->border[a1 + k] & 1u) up_set[nu++] = (uint32_t)(a1 + k);
    for (uint32_t i = 0; i < nl; ++i)
      for (uint32_t j = 0; j < nu; ++j) {
        const pfeat* fa = r->rec + lo_set[i];
        const pfeat* fb = r->rec + up_set[j];
        st->border_checks++;
        /* 1. temporal distance (l.127) */
        uint64_t d = 0;
        if (fb->toa_min > fa->toa_max) d = fb->toa_min - fa->toa_max;
        if (fa->toa_min > fb->toa_max) d = fa->toa_min - fb->toa_max;
        if (d > r->dt) continue;
        const int m = mergeable(r, lo_set[i], up_set[j], &g, st);
        if (m < 0) {
          r->err = P_ERR_OOM;
          break;
        }
        if (m) {
          add_pair(r, t, lo_set[i], up_set[j]);
          st->merges++;
        }
      }
  }
  free(lo_set);
  free(up_set);
  free(g.head);
  free(g.next);
  free(g.toa);
}

/* 4. labels and records */
static void k_labels(void* c, int t, int T) {
  run* r = (run*)c;
  for (uint64_t w = (uint64_t)t; w < r->nw; w += (uint64_t)T)
    for (uint64_t p = r->wstart[w]; p < r->wstart[w + 1]; ++p)
      r->labels[r->order[p]] = r->rec[r->final_of[r->cl_of[p]]].label;
}

static void k_bits(void* c, int t, int T) {
  run* r = (run*)c;
  for (uint64_t w = (uint64_t)t; w < r->nw; w += (uint64_t)T)
    for (uint64_t k = 0; k < r->ncl[w]; ++k) {
      const uint64_t id = r->wstart[w] + k;
      if (r->final_of[id] != id) continue;
      const uint32_t L = r->rec[id].label;
      __atomic_fetch_or(r->bits + (L >> 6), 1ull << (L & 63), __ATOMIC_RELAXED);
    }
}

static void k_emit(void* c, int t, int T) {
  run* r = (run*)c;
  for (uint64_t w = (uint64_t)t; w < r->nw; w += (uint64_t)T)
    for (uint64_t k = 0; k < r->ncl[w]; ++k) {
      const uint64_t id = r->wstart[w] + k;
      if (r->final_of[id] != id) continue;
      const uint32_t L = r->rec[id].label;
      const uint64_t ord = r->wbase[L >> 6] + __builtin_popcountll(r->bits[L >> 6] & ((1ull << (L & 63)) - 1));
      r->feats[ord] = r->rec[id];
    }
}

static uint32_t root_of(uint32_t* f, uint32_t x) {
  while (f[x] != x) {
    f[x] = f[f[x]];
    x = f[x];
  }
  return x;
}

int cpu_parallel_cluster(const phit* h, uint64_t n, uint64_t dt, uint32_t W, uint32_t H, uint64_t window_ticks,
                         int nthreads, uint32_t* labels, pfeat* feats, uint64_t* n_clusters, pstats* stats_out) {
  if (!n_clusters || W == 0 || H == 0 || (n && (!h || !labels || !feats)) || n >= 0xffffffffull) return P_ERR_ARG;
  *n_clusters = 0;
  if (stats_out) memset(stats_out, 0, sizeof(*stats_out));
  if (n == 0) return P_OK;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  run R;
  memset(&R, 0, sizeof(R));
  run* r = &R;
  r->h = h;
  r->n = n;
  r->dt = dt;
  r->W = W;
  r->H = H;
  r->nthreads = nthreads;
  r->labels = labels;
  r->feats = feats;
  minmax_ctx* mm = (minmax_ctx*)calloc(1, sizeof(minmax_ctx));
  if (!mm) return P_ERR_OOM;
  mm->r = r;
  parallel(nthreads, k_minmax, mm);
  uint64_t mn = ~0ull, mx = 0;
  int bad = 0;
  for (int t = 0; t < nthreads; ++t) {
    if (mm->mn[t] < mn) mn = mm->mn[t];
    if (mm->mx[t] > mx) mx = mm->mx[t];
    bad |= mm->bad[t];
  }
  free(mm);
  if (bad) return P_ERR_COORD;
  /* windows must be wider than dt_max (edges only between neighbouring windows) */
  uint64_t wt = window_ticks ? window_ticks : 100 * (dt ? dt : 1);
  if (wt <= dt) wt = dt + 1;
  if ((mx - mn) / wt > 50000000ull) wt = (mx - mn) / 50000000ull + 1; /* bound the window count */
  r->wticks = wt;
  r->toa_min = mn;
  r->nw = (mx - mn) / wt + 1;
  int rc = P_OK;
  r->wcount = (uint64_t*)calloc((size_t)nthreads * r->nw, sizeof(uint64_t));
  r->wstart = (uint64_t*)malloc((r->nw + 1) * sizeof(uint64_t));
  r->order = (uint32_t*)malloc(n * sizeof(uint32_t));
  r->cl_of = (uint32_t*)malloc(n * sizeof(uint32_t));
  r->parent = (uint32_t*)malloc(n * sizeof(uint32_t));
  r->rec = (pfeat*)malloc(n * sizeof(pfeat));
  r->bbox = (uint16_t*)malloc(n * 4 * sizeof(uint16_t));
  r->mstart = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
  r->members = (uint32_t*)malloc(n * sizeof(uint32_t));
  r->ncl = (uint32_t*)calloc(r->nw, sizeof(uint32_t));
  r->border = (uint8_t*)calloc(n, 1);
  r->pairs = (uint32_t**)calloc(nthreads, sizeof(uint32_t*));
  r->npairs = (uint64_t*)calloc(nthreads, sizeof(uint64_t));
  r->capairs = (uint64_t*)calloc(nthreads, sizeof(uint64_t));
  r->tstats = (pstats*)calloc(nthreads, sizeof(pstats));
  r->final_of = (uint32_t*)malloc(n * sizeof(uint32_t));
  const uint64_t nwords = (n + 63) / 64;
  r->bits = (uint64_t*)calloc(nwords, sizeof(uint64_t));
  r->wbase = (uint64_t*)malloc((nwords + 1) * sizeof(uint64_t));
  if (!r->wcount || !r->wstart || !r->order || !r->cl_of || !r->parent || !r->rec || !r->bbox || !r->mstart ||
      !r->members || !r->ncl || !r->border || !r->pairs || !r->npairs || !r->capairs || !r->tstats ||
      !r->final_of || !r->bits || !r->wbase) {
    rc = P_ERR_OOM;
    goto done;
  }
  /* 1. temporal splitting: counting sort of the hits by window */
  parallel(nthreads, k_hist, r);
  {
    uint64_t s = 0;
    for (uint64_t w = 0; w < r->nw; ++w) {
      r->wstart[w] = s;
      for (int t = 0; t < nthreads; ++t) {
        const uint64_t c = r->wcount[(uint64_t)t * r->nw + w];
        r->wcount[(uint64_t)t * r->nw + w] = s;
        s += c;
      }
    }
    r->wstart[r->nw] = s;
  }
  parallel(nthreads, k_scatter, r);
  /* 2. windows: time sort + Alg. 1 */
  parallel(nthreads, k_windows, r);
  if (r->err) {
    rc = r->err;
    goto done;
  }
  /* 3. border merges */
  parallel(nthreads, k_merge, r);
  if (r->err) {
    rc = r->err;
    goto done;
  }
  /* merged sets: smallest label of the set wins (reading R6) */
  for (uint64_t i = 0; i < n; ++i) r->final_of[i] = (uint32_t)i;
  for (int t = 0; t < nthreads; ++t)
    for (uint64_t p = 0; p < r->npairs[t]; ++p) {
      const uint32_t a = root_of(r->final_of, r->pairs[t][2 * p]), b = root_of(r->final_of, r->pairs[t][2 * p + 1]);
      if (a == b) continue;
      /* the root keeps the record with the smaller label */
      if (r->rec[a].label < r->rec[b].label) r->final_of[b] = a; else r->final_of[a] = b;
    }
  for (int t = 0; t < nthreads; ++t)
    for (uint64_t p = 0; p < r->npairs[t]; ++p)
      for (int e = 0; e < 2; ++e) {
        const uint32_t x = r->pairs[t][2 * p + e];
        const uint32_t root = root_of(r->final_of, x);
        if (root == x) continue;
        /* fold x's record into the root's, once per merged record */
        pfeat* f = r->rec + x;
        if (f->size == 0) continue;
        pfeat* d = r->rec + root;
        d->size += f->size;
        if (f->toa_min < d->toa_min) d->toa_min = f->toa_min;
        if (f->toa_max > d->toa_max) d->toa_max = f->toa_max;
        d->tot_sum += f->tot_sum;
        d->sum_x += f->sum_x;
        d->sum_y += f->sum_y;
        d->sum_tot_x += f->sum_tot_x;
        d->sum_tot_y += f->sum_tot_y;
        f->size = 0;
      }
  for (uint64_t i = 0; i < n; ++i) r->final_of[i] = root_of(r->final_of, (uint32_t)i);
  /* 4. labels, records in label order (bitmap rank) */
  parallel(nthreads, k_labels, r);
  parallel(nthreads, k_bits, r);
  {
    uint64_t s = 0;
    for (uint64_t w = 0; w < nwords; ++w) {
      r->wbase[w] = s;
      s += (uint64_t)__builtin_popcountll(r->bits[w]);
    }
    r->wbase[nwords] = s;
    r->k = s;
  }
  parallel(nthreads, k_emit, r);
  *n_clusters = r->k;
  if (stats_out)
    for (int t = 0; t < nthreads; ++t) {
      stats_out->windows += r->tstats[t].windows;
      stats_out->clusters += r->tstats[t].clusters;
      stats_out->border_clusters += r->tstats[t].border_clusters;
      stats_out->border_checks += r->tstats[t].border_checks;
      stats_out->bbox_checks += r->tstats[t].bbox_checks;
      stats_out->full_checks += r->tstats[t].full_checks;
      stats_out->merges += r->tstats[t].merges;
    }
done:
  free(r->wcount);
  free(r->wstart);
  free(r->order);
  free(r->cl_of);
  free(r->parent);
  free(r->rec);
  free(r->bbox);
  free(r->mstart);
  free(r->members);
  free(r->ncl);
  free(r->border);
  if (r->pairs)
    for (int t = 0; t < nthreads; ++t) free(r->pairs[t]);
  free(r->pairs);
  free(r->npairs);
  free(r->capairs);
  free(r->tstats);
  free(r->final_of);
  free(r->bits);
  free(r->wbase);
  return rc;
}
