/*
 * tpx_oracle.c -- plain, slow, single-threaded CPU oracle for Timepix3 hit
 * clustering.  TEST INFRASTRUCTURE ONLY: it is linked and called only by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs.  It shares no code, header, table or helper with the CUDA
 * path (paper_2412_11809_b200/), and it never reads anything produced by it.
 *
 * What it computes (the plain definition, written out):
 *   Graph G = (hits, E) -- PAPER.md §2.1 lines 61-62 ("each detected hit ... is
 *   a node ... If two hits are adjacent in space and time, they are connected
 *   with an edge ... finding connected components in the graph G ... graph
 *   traversal").  Adjacency in space = 8-neighbouring pixels (§2 (ii),
 *   line 35) plus the pixel itself (§4.1, reading R2);
 *   adjacency in time = |toa_i - toa_j| <= dt_max (§2 (iii)(a), line 39,
 *   inclusive, reading R3).  Clusters = connected components (reading R1).
 *   label(i) = smallest input index of i's component (reading R6); feature
 *   records in ascending label order (reading R7); fields per reading R8.
 *
 * Algorithm (no blocking or fusion beyond the definition):
 *   1. bucket hits by pixel id y*W + x (counting sort), each bucket sorted by
 *      (toa, input index);
 *   2. for each pixel p and each of its 9 neighbour pixels q, a two-pointer
 *      sweep over the two ToA-sorted buckets emits every j != i with
 *      |toa_i - toa_j| <= dt  -> explicit CSR adjacency (count, then fill);
 *   3. BFS from every unvisited hit in ascending input index: the seed is the
 *      component's smallest index, i.e. its label; features accumulate in the
 *      same traversal and records are appended in label order.
 *
 * Oracle-only extras: the streaming conventions for variants (iii)(b) and
 * (iii)(c) (§2 lines 40-41; SPEC.md serial_clusterer notes) used
 * only for the "definitions coincide for large dt_max" invariant (line 45),
 * and a single-component BFS over an implicit-neighbour pixel index for
 * sampled parity at sizes where the CSR graph does not fit.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct ohit {       /* 16-byte input record (same layout as the ABI) */
  uint64_t toa;
  uint16_t x, y, tot, reserved;
} ohit;

typedef struct ofeat {      /* 64-byte feature record */
  uint32_t label, size;
  uint64_t toa_min, toa_max, tot_sum, sum_x, sum_y, sum_tot_x, sum_tot_y;
} ofeat;

enum { O_OK = 0, O_ERR_ARG = -1, O_ERR_UNSUPPORTED = -2, O_ERR_COORD = -3, O_ERR_OOM = -6 };

/* ------------------------------------------------------- pixel index */
typedef struct pix_index {
  const ohit* h;
  uint64_t n;
  uint32_t W, H;
  uint64_t* start;   /* W*H+1 bucket offsets                     */
  uint32_t* order;   /* hit ids, bucketed, (toa, id)-sorted       */
} pix_index;

static _Thread_local const ohit* g_sort_hits; /* qsort context (one per calling thread) */
static int cmp_toa_id(const void* a, const void* b) {
  uint32_t i = *(const uint32_t*)a, j = *(const uint32_t*)b;
  uint64_t ti = g_sort_hits[i].toa, tj = g_sort_hits[j].toa;
  if (ti != tj) return ti < tj ? -1 : 1;
  return (i > j) - (i < j);
}

static int index_build(pix_index* ix, const ohit* h, uint64_t n, uint32_t W, uint32_t H) {
  ix->h = h; ix->n = n; ix->W = W; ix->H = H;
  size_t np = (size_t)W * H;
  ix->start = (uint64_t*)calloc(np + 1, sizeof(uint64_t));
  ix->order = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  if (!ix->start || !ix->order) return O_ERR_OOM;
  for (uint64_t i = 0; i < n; ++i) ix->start[(size_t)h[i].y * W + h[i].x + 1]++;
  for (size_t p = 0; p < np; ++p) ix->start[p + 1] += ix->start[p];
  uint64_t* fill = (uint64_t*)malloc((np ? np : 1) * sizeof(uint64_t));
  if (!fill) return O_ERR_OOM;
  memcpy(fill, ix->start, np * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) ix->order[fill[(size_t)h[i].y * W + h[i].x]++] = (uint32_t)i;
  free(fill);
  g_sort_hits = h;
  for (size_t p = 0; p < np; ++p) {
    uint64_t a = ix->start[p], b = ix->start[p + 1];
    if (b - a > 1) qsort(ix->order + a, b - a, sizeof(uint32_t), cmp_toa_id);
  }
  return O_OK;
}

static void index_free(pix_index* ix) {
  free(ix->start); free(ix->order);
  ix->start = NULL; ix->order = NULL;
}

static int check_coords(const ohit* h, uint64_t n, uint32_t W, uint32_t H) {
  for (uint64_t i = 0; i < n; ++i)
    if (h[i].x >= W || h[i].y >= H) return O_ERR_COORD;
  return O_OK;
}

/* first position in bucket [a,b) with toa >= t */
static uint64_t lower_toa(const pix_index* ix, uint64_t a, uint64_t b, uint64_t t) {
  while (a < b) {
    uint64_t m = a + (b - a) / 2;
    if (ix->h[ix->order[m]].toa < t) a = m + 1; else b = m;
  }
  return a;
}

/* ------------------------------------------------------- main oracle */
/* Cluster n hits; labels[n] (input order) and feats[] (ascending label,
 * capacity n) are caller-allocated.  Returns O_OK / O_ERR_*. */
int oracle_cluster_local(const ohit* h, uint64_t n, uint64_t dt, uint32_t W, uint32_t H,
                         uint32_t* labels, ofeat* feats, uint64_t* n_clusters) {
  if (!n_clusters || W == 0 || H == 0 || (n && (!h || !labels || !feats))) return O_ERR_ARG;
  *n_clusters = 0;
  if (n == 0) return O_OK;
  if (check_coords(h, n, W, H)) return O_ERR_COORD;
  pix_index ix;
  int rc = index_build(&ix, h, n, W, H);
  if (rc) { index_free(&ix); return rc; }

  /* step 2: explicit CSR adjacency, count pass then fill pass */
  uint64_t* off = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
  if (!off) { index_free(&ix); return O_ERR_OOM; }
  for (int pass = 0; pass < 2; ++pass) {
    uint32_t* adj = NULL;
    uint64_t* cur = NULL;
    if (pass == 1) {
      for (uint64_t i = 0; i < n; ++i) off[i + 1] += off[i];
      adj = (uint32_t*)malloc((off[n] ? off[n] : 1) * sizeof(uint32_t));
      cur = (uint64_t*)malloc(n * sizeof(uint64_t));
      if (!adj || !cur) { free(adj); free(cur); free(off); index_free(&ix); return O_ERR_OOM; }
      memcpy(cur, off, n * sizeof(uint64_t));
    }
    for (uint32_t py = 0; py < H; ++py)
      for (uint32_t px = 0; px < W; ++px) {
        size_t p = (size_t)py * W + px;
        uint64_t pa = ix.start[p], pb = ix.start[p + 1];
        if (pa == pb) continue;
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            int qx = (int)px + dx, qy = (int)py + dy;
            if (qx < 0 || qy < 0 || qx >= (int)W || qy >= (int)H) continue; /* no wraparound, R5 */
            size_t q = (size_t)qy * W + (size_t)qx;
            uint64_t qa = ix.start[q], qb = ix.start[q + 1];
            if (qa == qb) continue;
            /* two pointers over the window [toa_i - dt, toa_i + dt] in q */
            uint64_t lo = qa, hi = qa;
            for (uint64_t a = pa; a < pb; ++a) {
              uint32_t i = ix.order[a];
              uint64_t ti = h[i].toa;
              while (lo < qb && h[ix.order[lo]].toa + dt < ti) ++lo;      /* toa_j < ti - dt */
              if (hi < lo) hi = lo;
              while (hi < qb && h[ix.order[hi]].toa <= ti + dt) ++hi;     /* toa_j <= ti + dt */
              for (uint64_t b = lo; b < hi; ++b) {
                uint32_t j = ix.order[b];
                if (j == i) continue;
                if (pass == 0) off[i + 1]++;
                else adj[cur[i]++] = j;
              }
            }
          }
      }
    if (pass == 1) {
      free(cur);
      /* step 3: BFS in ascending input index; seed = label */
      uint8_t* seen = (uint8_t*)calloc(n, 1);
      uint32_t* queue = (uint32_t*)malloc(n * sizeof(uint32_t));
      if (!seen || !queue) { free(seen); free(queue); free(adj); free(off); index_free(&ix); return O_ERR_OOM; }
      uint64_t k = 0;
      for (uint64_t s = 0; s < n; ++s) {
        if (seen[s]) continue;
        ofeat f;
        memset(&f, 0, sizeof f);
        f.label = (uint32_t)s;
        f.toa_min = UINT64_MAX;
        uint64_t qh = 0, qt = 0;
        queue[qt++] = (uint32_t)s;
        seen[s] = 1;
        while (qh < qt) {
          uint32_t u = queue[qh++];
          labels[u] = (uint32_t)s;
          f.size += 1;
          if (h[u].toa < f.toa_min) f.toa_min = h[u].toa;
          if (h[u].toa > f.toa_max) f.toa_max = h[u].toa;
          f.tot_sum += h[u].tot;
          f.sum_x += h[u].x;
          f.sum_y += h[u].y;
          f.sum_tot_x += (uint64_t)h[u].tot * h[u].x;
          f.sum_tot_y += (uint64_t)h[u].tot * h[u].y;
          for (uint64_t e = off[u]; e < off[u + 1]; ++e) {
            uint32_t v = adj[e];
            if (!seen[v]) { seen[v] = 1; queue[qt++] = v; }
          }
        }
        feats[k++] = f;
      }
      *n_clusters = k;
      free(seen); free(queue); free(adj);
    }
  }
  free(off);
  index_free(&ix);
  return O_OK;
}

/* Number of edges of G (each unordered pair once) -- for tests/diagnostics. */
int64_t oracle_count_edges(const ohit* h, uint64_t n, uint64_t dt, uint32_t W, uint32_t H) {
  if (n == 0) return 0;
  if (!h || check_coords(h, n, W, H)) return -1;
  pix_index ix;
  if (index_build(&ix, h, n, W, H)) { index_free(&ix); return -1; }
  int64_t m = 0;
  for (uint64_t i = 0; i < n; ++i) {
    int x = h[i].x, y = h[i].y;
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int qx = x + dx, qy = y + dy;
        if (qx < 0 || qy < 0 || qx >= (int)W || qy >= (int)H) continue;
        size_t q = (size_t)qy * W + (size_t)qx;
        uint64_t lo_t = h[i].toa > dt ? h[i].toa - dt : 0;
        uint64_t a = lower_toa(&ix, ix.start[q], ix.start[q + 1], lo_t);
        for (uint64_t b = a; b < ix.start[q + 1] && h[ix.order[b]].toa <= h[i].toa + dt; ++b)
          if (ix.order[b] > i) ++m;
      }
  }
  index_free(&ix);
  return m;
}

/* ------------------------------------------- sampled single component */
/* BFS from `seed` over implicit neighbours (same edge predicate, pixel index
 * built once).  Returns the component size, writes its members (unsorted)
 * into members[0..cap) when members != NULL and its feature record into *f.
 * The handle is created by oracle_index_new and freed by oracle_index_delete. */
typedef struct oracle_index {
  pix_index ix;
  uint64_t dt;
  uint8_t* seen;
  uint32_t* queue;
} oracle_index;

void* oracle_index_new(const ohit* h, uint64_t n, uint64_t dt, uint32_t W, uint32_t H) {
  if (!h || n == 0 || check_coords(h, n, W, H)) return NULL;
  oracle_index* o = (oracle_index*)calloc(1, sizeof(oracle_index));
  if (!o) return NULL;
  if (index_build(&o->ix, h, n, W, H)) { index_free(&o->ix); free(o); return NULL; }
  o->dt = dt;
  o->seen = (uint8_t*)calloc(n, 1);
  o->queue = (uint32_t*)malloc(n * sizeof(uint32_t));
  if (!o->seen || !o->queue) { free(o->seen); free(o->queue); index_free(&o->ix); free(o); return NULL; }
  return o;
}

void oracle_index_delete(void* p) {
  oracle_index* o = (oracle_index*)p;
  if (!o) return;
  free(o->seen); free(o->queue); index_free(&o->ix); free(o);
}

int64_t oracle_index_component(void* p, uint32_t seed, uint32_t* members, uint64_t cap, ofeat* f) {
  oracle_index* o = (oracle_index*)p;
  if (!o || seed >= o->ix.n || !f) return -1;
  const ohit* h = o->ix.h;
  uint64_t dt = o->dt;
  uint64_t qh = 0, qt = 0;
  o->queue[qt++] = seed;
  o->seen[seed] = 1;
  memset(f, 0, sizeof *f);
  f->label = UINT32_MAX;
  f->toa_min = UINT64_MAX;
  while (qh < qt) {
    uint32_t u = o->queue[qh++];
    if (u < f->label) f->label = u;
    f->size += 1;
    if (h[u].toa < f->toa_min) f->toa_min = h[u].toa;
    if (h[u].toa > f->toa_max) f->toa_max = h[u].toa;
    f->tot_sum += h[u].tot;
    f->sum_x += h[u].x;
    f->sum_y += h[u].y;
    f->sum_tot_x += (uint64_t)h[u].tot * h[u].x;
    f->sum_tot_y += (uint64_t)h[u].tot * h[u].y;
    int x = h[u].x, y = h[u].y;
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int qx = x + dx, qy = y + dy;
        if (qx < 0 || qy < 0 || qx >= (int)o->ix.W || qy >= (int)o->ix.H) continue;
        size_t q = (size_t)qy * o->ix.W + (size_t)qx;
        uint64_t lo_t = h[u].toa > dt ? h[u].toa - dt : 0;
        uint64_t a = lower_toa(&o->ix, o->ix.start[q], o->ix.start[q + 1], lo_t);
        for (uint64_t b = a; b < o->ix.start[q + 1]; ++b) {
          uint32_t v = o->ix.order[b];
          if (h[v].toa > h[u].toa + dt) break;
          if (!o->seen[v]) { o->seen[v] = 1; o->queue[qt++] = v; }
        }
      }
  }
  if (members) for (uint64_t i = 0; i < qt && i < cap; ++i) members[i] = o->queue[i];
  for (uint64_t i = 0; i < qt; ++i) o->seen[o->queue[i]] = 0;   /* reset for the next call */
  return (int64_t)qt;
}

/* ------------------------------------------- streaming variants (oracle only) */
/* Hits in (toa, index) order; a hit joins every existing cluster that has a
 * member on one of its 9 neighbour pixels and satisfies the variant's time
 * predicate (SPEC.md serial_clusterer notes):
 *   0 LOCAL : |toa(hit) - toa(member)| <= dt for some such member
 *   1 GLOBAL: toa(hit) - cluster.maxToa <= dt   (§2 (iii)(b) l.40)
 *   2 STATIC: toa(hit) - cluster.minToa <= dt   (§2 (iii)(c) l.41)
 * All joinable clusters are merged.  O(n^2): small inputs only.
 * labels[i] = smallest input index of the final cluster. */
int oracle_cluster_streaming(const ohit* h, uint64_t n, uint64_t dt, uint32_t W, uint32_t H,
                             int variant, uint32_t* labels) {
  if (n && (!h || !labels)) return O_ERR_ARG;
  if (variant < 0 || variant > 2) return O_ERR_UNSUPPORTED;
  if (n == 0) return O_OK;
  if (check_coords(h, n, W, H)) return O_ERR_COORD;
  uint32_t* ord = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* cl = (uint32_t*)malloc(n * sizeof(uint32_t));      /* hit -> cluster id (by first hit) */
  uint64_t* cmin = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint64_t* cmax = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint8_t* hit_cand = (uint8_t*)malloc(n);
  if (!ord || !cl || !cmin || !cmax || !hit_cand) {
    free(ord); free(cl); free(cmin); free(cmax); free(hit_cand); return O_ERR_OOM;
  }
  for (uint64_t i = 0; i < n; ++i) ord[i] = (uint32_t)i;
  g_sort_hits = h;
  qsort(ord, n, sizeof(uint32_t), cmp_toa_id);
  for (uint64_t a = 0; a < n; ++a) {
    uint32_t i = ord[a];
    memset(hit_cand, 0, n);
    /* which clusters are joinable? */
    for (uint64_t b = 0; b < a; ++b) {
      uint32_t j = ord[b];
      int ddx = (int)h[i].x - (int)h[j].x, ddy = (int)h[i].y - (int)h[j].y;
      if (ddx < -1 || ddx > 1 || ddy < -1 || ddy > 1) continue;
      uint32_t c = cl[j];
      int ok;
      if (variant == 0) ok = h[i].toa - h[j].toa <= dt;
      else if (variant == 1) ok = h[i].toa - cmax[c] <= dt;
      else ok = h[i].toa - cmin[c] <= dt;
      if (ok) hit_cand[c] = 1;
    }
    uint32_t target = i;
    int any = 0;
    for (uint64_t b = 0; b < a; ++b) {   /* smallest candidate cluster id among members */
      uint32_t c = cl[ord[b]];
      if (hit_cand[c]) { if (!any || c < target) target = c; any = 1; }
    }
    if (!any) {
      cl[i] = i; cmin[i] = h[i].toa; cmax[i] = h[i].toa;
      continue;
    }
    uint64_t mn = h[i].toa, mx = h[i].toa;
    for (uint64_t b = 0; b < a; ++b) {
      uint32_t c = cl[ord[b]];
      if (hit_cand[c]) {
        if (cmin[c] < mn) mn = cmin[c];
        if (cmax[c] > mx) mx = cmax[c];
      }
    }
    for (uint64_t b = 0; b < a; ++b) {
      uint32_t j = ord[b];
      if (hit_cand[cl[j]]) cl[j] = target;
    }
    cl[i] = target;
    cmin[target] = mn; cmax[target] = mx;
  }
  /* canonical label = smallest input index per cluster */
  uint32_t* mn = (uint32_t*)malloc(n * sizeof(uint32_t));
  for (uint64_t i = 0; i < n; ++i) mn[i] = UINT32_MAX;
  for (uint64_t i = 0; i < n; ++i) if ((uint32_t)i < mn[cl[i]]) mn[cl[i]] = (uint32_t)i;
  for (uint64_t i = 0; i < n; ++i) labels[i] = mn[cl[i]];
  free(mn); free(ord); free(cl); free(cmin); free(cmax); free(hit_cand);
  return O_OK;
}

/* ------------------------------------------------ cluster shape records */
/* Per cluster, in the order of feats[] (ascending label): the bounding box
 * "smallest rectangle (aligned with the sensor) enclosing the cluster"
 * (§3.3) and the unweighted second moments sum x^2, sum x*y,
 * sum y^2 (shape features, §1 line 15; reading R19).  Plain
 * definition: one pass over the hits, each hit added to the record of its
 * label (label -> record position by a direct map). */
typedef struct oshape {     /* 32-byte shape record */
  uint16_t x_min, x_max, y_min, y_max;
  uint64_t sum_xx, sum_xy, sum_yy;
} oshape;

int oracle_shapes(const ohit* h, uint64_t n, const uint32_t* labels, const ofeat* feats, uint64_t k,
                  oshape* out) {
  if (n && (!h || !labels || !feats || !out)) return O_ERR_ARG;
  uint32_t* pos = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  if (!pos) return O_ERR_OOM;
  for (uint64_t i = 0; i < n; ++i) pos[i] = UINT32_MAX;
  for (uint64_t c = 0; c < k; ++c) {
    pos[feats[c].label] = (uint32_t)c;
    out[c].x_min = out[c].y_min = UINT16_MAX;
    out[c].x_max = out[c].y_max = 0;
    out[c].sum_xx = out[c].sum_xy = out[c].sum_yy = 0;
  }
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t c = pos[labels[i]];
    if (c == UINT32_MAX) { free(pos); return O_ERR_ARG; }
    uint64_t x = h[i].x, y = h[i].y;
    if (h[i].x < out[c].x_min) out[c].x_min = h[i].x;
    if (h[i].x > out[c].x_max) out[c].x_max = h[i].x;
    if (h[i].y < out[c].y_min) out[c].y_min = h[i].y;
    if (h[i].y > out[c].y_max) out[c].y_max = h[i].y;
    out[c].sum_xx += x * x;
    out[c].sum_xy += x * y;
    out[c].sum_yy += y * y;
  }
  free(pos);
  return O_OK;
}

/* --------------------------------------------- cluster-contiguous output */
/* Alg. "High-level GPU clustering" Step 6 (§4): "Sort
 * clusters by their minimum time of arrival, causing the hits from the same
 * cluster to form adjacent memory blocks".  Reading R18: hits are ordered by
 * (toa, input index); a cluster's position is that of its earliest hit in
 * this order (ties in minimum ToA broken by that hit's input index); inside a
 * block, hits keep the (toa, input index) order.
 *   order[n]       input indices, cluster blocks one after another
 *   offsets[k+1]   block g is order[offsets[g] .. offsets[g+1])
 *   cluster_of[k]  block g holds the cluster feats[cluster_of[g]]            */
static _Thread_local const uint64_t* g_sort_keys;
static int cmp_key_u32(const void* a, const void* b) {
  uint32_t i = *(const uint32_t*)a, j = *(const uint32_t*)b;
  uint64_t ki = g_sort_keys[i], kj = g_sort_keys[j];
  if (ki != kj) return ki < kj ? -1 : 1;
  return (i > j) - (i < j);
}

int oracle_group(const ohit* h, uint64_t n, const uint32_t* labels, const ofeat* feats, uint64_t k,
                 uint32_t* order, uint64_t* offsets, uint32_t* cluster_of) {
  if ((n && (!h || !labels || !feats || !order)) || !offsets || (k && !cluster_of)) return O_ERR_ARG;
  uint32_t* S = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t* pos = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  uint64_t* first = (uint64_t*)malloc((k ? k : 1) * sizeof(uint64_t));
  uint32_t* cl = (uint32_t*)malloc((k ? k : 1) * sizeof(uint32_t));
  uint64_t* cursor = (uint64_t*)malloc((k ? k : 1) * sizeof(uint64_t));
  uint32_t* block_of = (uint32_t*)malloc((k ? k : 1) * sizeof(uint32_t));
  if (!S || !pos || !first || !cl || !cursor || !block_of) {
    free(S); free(pos); free(first); free(cl); free(cursor); free(block_of);
    return O_ERR_OOM;
  }
  /* 1. the (toa, input index) order of all hits */
  for (uint64_t i = 0; i < n; ++i) S[i] = (uint32_t)i;
  g_sort_hits = h;
  qsort(S, n, sizeof(uint32_t), cmp_toa_id);
  /* 2. label -> record position; each cluster's earliest position in S */
  for (uint64_t i = 0; i < n; ++i) pos[i] = UINT32_MAX;
  for (uint64_t c = 0; c < k; ++c) { pos[feats[c].label] = (uint32_t)c; first[c] = UINT64_MAX; }
  for (uint64_t p = 0; p < n; ++p) {
    uint32_t c = pos[labels[S[p]]];
    if (c == UINT32_MAX) { n = 0; k = 0; break; }
    if (first[c] == UINT64_MAX) first[c] = p;
  }
  /* 3. clusters in the order of their earliest hit */
  for (uint64_t c = 0; c < k; ++c) cl[c] = (uint32_t)c;
  g_sort_keys = first;
  qsort(cl, k, sizeof(uint32_t), cmp_key_u32);
  /* 4. block offsets from the cluster sizes */
  offsets[0] = 0;
  for (uint64_t g = 0; g < k; ++g) {
    cluster_of[g] = cl[g];
    block_of[cl[g]] = (uint32_t)g;
    offsets[g + 1] = offsets[g] + feats[cl[g]].size;
  }
  /* 5. hits in S order appended to their cluster's block */
  for (uint64_t g = 0; g < k; ++g) cursor[g] = offsets[g];
  for (uint64_t p = 0; p < n; ++p) {
    uint32_t g = block_of[pos[labels[S[p]]]];
    order[cursor[g]++] = S[p];
  }
  int rc = (k && offsets[k] != n) ? O_ERR_ARG : O_OK;
  free(S); free(pos); free(first); free(cl); free(cursor); free(block_of);
  return rc;
}

/* ------------------------------------------------------------ centroid */
/* cx = sum_tot_x / tot_sum, cy = sum_tot_y / tot_sum (one IEEE division each);
 * tot_sum == 0 -> unweighted sum_x / size (reading R8). */
void oracle_centroids(const ofeat* f, uint64_t k, double* cxy) {
  for (uint64_t i = 0; i < k; ++i) {
    if (f[i].tot_sum) {
      cxy[2 * i] = (double)f[i].sum_tot_x / (double)f[i].tot_sum;
      cxy[2 * i + 1] = (double)f[i].sum_tot_y / (double)f[i].tot_sum;
    } else {
      cxy[2 * i] = (double)f[i].sum_x / (double)f[i].size;
      cxy[2 * i + 1] = (double)f[i].sum_y / (double)f[i].size;
    }
  }
}
