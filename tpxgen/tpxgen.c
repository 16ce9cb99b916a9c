/*
 * tpxgen.c -- deterministic synthetic Timepix3/Timepix4 hit-stream generator.
 *
 * INPUT INFRASTRUCTURE shared by the oracle tests and the CUDA path: it draws
 * hits and holds none of the clustering method's arithmetic (no adjacency
 * test, no union-find, no feature reduction).
 *
 * Shape of the workload:
 *  - Poisson cluster arrivals at lambda = rate / E[size] (§1 l.13:
 *    "data rates can surpass 40 million hits per second").
 *  - Cluster size laws moment-matched to the dataset table (§5,
 *    lines 240-264): lognormal for gamma dots (2.46 +- 2.15) and pion tracks
 *    at 0/45/75 deg (7.22 +- 27.35, 23.33 +- 33.47, 60.27 +- 64.33); log-uniform
 *    sizes for heavy-ion blobs (Pb subsets, lines 258-262).
 *  - Shapes: 8-connected random growth (dots), rasterised line segments
 *    (tracks), filled discs / 2:1 ellipses with a ToT core (blobs).
 *  - Pixel dead time: a pixel hit at toa t with ToT k is dead until
 *    t + 16 k + 300 ticks.
 *  - Readout disorder: hits are emitted in order of e = toa + 16 ToT + U[0,J),
 *    so the stream is t-ordered (§3.1 lines 99-100), not sorted.
 *
 * Determinism: the time axis is cut into fixed segments (length derived from
 * the rate only); segment s draws from its own xoshiro256** stream seeded by
 * SplitMix64(seed, s), with its own dead-time map.  Output = concatenation of
 * segments in order, truncated to n hits; independent of thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct gen_hit {
  uint64_t toa;
  uint16_t x, y, tot, reserved;
} gen_hit;

typedef struct tpxgen_config {
  uint64_t n_hits;
  uint32_t width, height;
  double rate_hz;          /* hit rate                                      */
  double frac_dot, frac_track, frac_blob; /* mix by cluster count           */
  uint32_t dot_min, dot_max;
  uint32_t track_min, track_max;
  uint32_t blob_min, blob_max;
  uint64_t disorder_ticks; /* J                                             */
  uint64_t toa_origin;     /* added to every ToA                            */
  uint64_t seed;
  int32_t n_threads;       /* 0 = OpenMP default                            */
  int32_t pad;
} tpxgen_config;

/* ------------------------------------------------------------------ RNG */
static uint64_t splitmix64(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
typedef struct { uint64_t s[4]; } rng_t;
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static inline uint64_t rng_next(rng_t* r) {
  uint64_t* s = r->s;
  uint64_t result = rotl(s[1] * 5, 7) * 9;
  uint64_t t = s[1] << 17;
  s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
  s[2] ^= t; s[3] = rotl(s[3], 45);
  return result;
}
static void rng_seed(rng_t* r, uint64_t seed, uint64_t stream) {
  uint64_t sm = seed * 0xD1B54A32D192ED03ull ^ (stream + 0x632BE59BD9B4E019ull);
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&sm);
}
static inline double rng_u01(rng_t* r) { return (rng_next(r) >> 11) * (1.0 / 9007199254740992.0); }
static inline uint64_t rng_below(rng_t* r, uint64_t n) { return n ? rng_next(r) % n : 0; }
static inline int rng_int(rng_t* r, int lo, int hi) { return lo + (int)rng_below(r, (uint64_t)(hi - lo + 1)); }
static double rng_normal(rng_t* r) {
  double u1 = rng_u01(r), u2 = rng_u01(r);
  if (u1 < 1e-300) u1 = 1e-300;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
static double rng_exp(rng_t* r, double mean) {
  double u = rng_u01(r);
  return -mean * log1p(-u);
}

/* ------------------------------------------------------------ size laws */
typedef struct { double mu, sigma; uint32_t lo, hi; } lognorm_t;
static lognorm_t lognorm_make(double mean, double sd, uint32_t lo, uint32_t hi) {
  lognorm_t l;
  l.sigma = sqrt(log(1.0 + (sd * sd) / (mean * mean)));
  l.mu = log(mean) - 0.5 * l.sigma * l.sigma;
  l.lo = lo < 1 ? 1 : lo;
  l.hi = hi < l.lo ? l.lo : hi;
  return l;
}
static uint32_t lognorm_draw(rng_t* r, const lognorm_t* l) {
  double x = exp(l->mu + l->sigma * rng_normal(r));
  double k = floor(x + 0.5);
  if (k < l->lo) k = l->lo;
  if (k > l->hi) k = l->hi;
  return (uint32_t)k;
}
static double phi(double z) { return 0.5 * erfc(-z / sqrt(2.0)); }
static double lognorm_mean(const lognorm_t* l) {
  double e = 0.0;
  for (uint32_t k = l->lo; k <= l->hi; ++k) {
    double a = (k == l->lo) ? 0.0 : phi((log(k - 0.5) - l->mu) / l->sigma);
    double b = (k == l->hi) ? 1.0 : phi((log(k + 0.5) - l->mu) / l->sigma);
    e += k * (b - a);
  }
  return e;
}

/* --------------------------------------------------------- event shapes */
typedef struct { int x, y; uint32_t tot; uint32_t dtoa; } px_t;

static inline uint32_t timewalk(rng_t* r, uint32_t tot) {
  uint32_t tw = 48u / (tot ? tot : 1u);
  if (tw > 32u) tw = 32u;
  return tw + (uint32_t)rng_below(r, 2);
}

static int has_px(const px_t* p, int m, int x, int y) {
  for (int i = 0; i < m; ++i) if (p[i].x == x && p[i].y == y) return 1;
  return 0;
}

/* X-ray / gamma dot: random 8-connected growth from a seed pixel. */
static int make_dot(rng_t* r, uint32_t m, int cx, int cy, px_t* out) {
  int n = 0;
  out[n].x = cx; out[n].y = cy; out[n].tot = (uint32_t)rng_int(r, 20, 60); n++;
  for (uint32_t k = 1; k < m; ++k) {
    for (int tries = 0; tries < 16; ++tries) {
      int b = (int)rng_below(r, (uint64_t)n);
      int d = (int)rng_below(r, 8);
      static const int DX[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
      static const int DY[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
      int x = out[b].x + DX[d], y = out[b].y + DY[d];
      if (!has_px(out, n, x, y)) {
        out[n].x = x; out[n].y = y; out[n].tot = (uint32_t)rng_int(r, 1, 20); n++;
        break;
      }
    }
  }
  for (int i = 0; i < n; ++i) out[i].dtoa = timewalk(r, out[i].tot);
  return n;
}

/* MIP track: rasterised 8-connected segment, width 1-2 px, drift along it. */
static int make_track(rng_t* r, uint32_t m, int cx, int cy, px_t* out) {
  double th = 6.283185307179586 * rng_u01(r);
  double c = cos(th), s = sin(th);
  double mx = fabs(c) > fabs(s) ? fabs(c) : fabs(s);
  double sx = c / mx, sy = s / mx;
  int wide = rng_below(r, 2) == 0;
  int perp_x = fabs(c) > fabs(s) ? 0 : 1, perp_y = 1 - perp_x;
  int n = 0;
  double px = cx, py = cy;
  for (uint32_t k = 0; n < (int)m; ++k) {
    int x = (int)floor(px + 0.5), y = (int)floor(py + 0.5);
    out[n].x = x; out[n].y = y; out[n].tot = (uint32_t)rng_int(r, 5, 40);
    out[n].dtoa = (uint32_t)((16ull * k) / (m > 1 ? m - 1 : 1));
    n++;
    if (wide && n < (int)m && rng_below(r, 100) < 35) {
      out[n].x = x + perp_x; out[n].y = y + perp_y; out[n].tot = (uint32_t)rng_int(r, 5, 40);
      out[n].dtoa = out[n - 1].dtoa;
      n++;
    }
    px += sx; py += sy;
  }
  for (int i = 0; i < n; ++i) out[i].dtoa += timewalk(r, out[i].tot);
  return n;
}

/* Heavy-ion blob: filled disc (50%) or 2:1 ellipse (50%) with a ToT core. */
static int make_blob(rng_t* r, uint32_t m, int cx, int cy, px_t* out, int cap) {
  double rad = sqrt((double)m / 3.141592653589793);
  double a = rad, b = rad;
  if (rng_below(r, 2)) { a = rad * 1.4142135623730951; b = rad / 1.4142135623730951; }
  double phi_ = 3.141592653589793 * rng_u01(r);
  double c = cos(phi_), s = sin(phi_);
  int R = (int)ceil(a) + 1;
  uint32_t core = (uint32_t)rng_int(r, 400, 1023);
  double tmean = 20.0 + 60.0 * rng_u01(r);
  int n = 0;
  for (int dy = -R; dy <= R && n < cap; ++dy)
    for (int dx = -R; dx <= R && n < cap; ++dx) {
      double u = dx * c + dy * s, v = -dx * s + dy * c;
      double rho2 = (u * u) / (a * a) + (v * v) / (b * b);
      if (rho2 > 1.0) continue;
      uint32_t rim = (uint32_t)rng_int(r, 1, 20);
      double t = rim + (core - rim) * (1.0 - rho2);
      uint32_t tot = (uint32_t)(t * (0.9 + 0.2 * rng_u01(r)));
      if (tot < 1) tot = 1;
      if (tot > 1023) tot = 1023;
      double off = rng_exp(r, tmean) * (0.5 + sqrt(rho2));
      if (off > 256.0) off = 256.0;
      out[n].x = cx + dx; out[n].y = cy + dy; out[n].tot = tot; out[n].dtoa = (uint32_t)off;
      n++;
    }
  return n;
}

/* -------------------------------------------------------------- segments */
typedef struct {
  gen_hit* hits;
  uint32_t* truth;   /* event index local to the segment */
  uint64_t n;
  uint64_t n_events;
} segment_t;

typedef struct { uint64_t key; uint32_t idx; uint32_t pad; } skey_t;
static int cmp_skey(const void* a, const void* b) {
  const skey_t* x = (const skey_t*)a; const skey_t* y = (const skey_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return (x->idx > y->idx) - (x->idx < y->idx);
}

typedef struct {
  tpxgen_config c;
  lognorm_t dot, trk[3];
  double lambda_per_tick;   /* cluster arrivals per tick */
  uint64_t seg_len;         /* ticks */
  double p_dot, p_track;    /* cumulative mix */
} gen_state;

#define SEG_TARGET_HITS 262144.0
#define TICK_S 1.5625e-9

static void gen_segment(const gen_state* g, uint64_t sidx, segment_t* seg) {
  const tpxgen_config* c = &g->c;
  rng_t r;
  rng_seed(&r, c->seed, sidx);
  uint64_t cap = (uint64_t)(SEG_TARGET_HITS * 1.5) + 16384;
  gen_hit* h = (gen_hit*)malloc(cap * sizeof(gen_hit));
  uint32_t* tr = (uint32_t*)malloc(cap * sizeof(uint32_t));
  uint64_t* ekey = (uint64_t*)malloc(cap * sizeof(uint64_t));
  uint32_t mx = c->blob_max > c->track_max ? c->blob_max : c->track_max;
  if (c->dot_max > mx) mx = c->dot_max;
  size_t npx_cap = (size_t)mx * 2 + 64;
  if (npx_cap < 64) npx_cap = 64;
  px_t* px = (px_t*)malloc(npx_cap * sizeof(px_t));
  size_t npix = (size_t)c->width * c->height;
  uint64_t* dead = (uint64_t*)calloc(npix, sizeof(uint64_t));
  uint64_t n = 0, nev = 0;
  double t = (double)(sidx * g->seg_len);
  double tend = (double)((sidx + 1) * g->seg_len);
  for (;;) {
    t += rng_exp(&r, 1.0 / g->lambda_per_tick);
    if (t >= tend) break;
    uint64_t t0 = (uint64_t)t;
    double u = rng_u01(&r);
    int cx = (int)rng_below(&r, c->width), cy = (int)rng_below(&r, c->height);
    int m;
    if (u < g->p_dot) {
      uint32_t sz = lognorm_draw(&r, &g->dot);
      m = make_dot(&r, sz, cx, cy, px);
    } else if (u < g->p_track) {
      int which = (int)rng_below(&r, 3);
      uint32_t sz = lognorm_draw(&r, &g->trk[which]);
      m = make_track(&r, sz, cx, cy, px);
    } else {
      double lo = c->blob_min, hi = c->blob_max;
      uint32_t sz = (uint32_t)floor(lo * exp(rng_u01(&r) * log(hi / lo)));
      m = make_blob(&r, sz, cx, cy, px, (int)npx_cap);
    }
    for (int i = 0; i < m; ++i) {
      if (px[i].x < 0 || px[i].y < 0 || px[i].x >= (int)c->width || px[i].y >= (int)c->height) continue;
      size_t p = (size_t)px[i].y * c->width + (size_t)px[i].x;
      uint64_t toa = t0 + px[i].dtoa;
      if (toa < dead[p]) continue;
      uint64_t d = toa + 16ull * px[i].tot + 300ull;
      if (d > dead[p]) dead[p] = d;
      if (n == cap) {
        cap *= 2;
        h = (gen_hit*)realloc(h, cap * sizeof(gen_hit));
        tr = (uint32_t*)realloc(tr, cap * sizeof(uint32_t));
        ekey = (uint64_t*)realloc(ekey, cap * sizeof(uint64_t));
      }
      h[n].toa = toa + c->toa_origin;
      h[n].x = (uint16_t)px[i].x; h[n].y = (uint16_t)px[i].y;
      h[n].tot = (uint16_t)px[i].tot; h[n].reserved = 0;
      tr[n] = (uint32_t)nev;
      ekey[n] = toa + 16ull * px[i].tot + (c->disorder_ticks ? rng_below(&r, c->disorder_ticks) : 0);
      n++;
    }
    nev++;
  }
  /* emission order: (e, generation order) */
  skey_t* k = (skey_t*)malloc((n ? n : 1) * sizeof(skey_t));
  for (uint64_t i = 0; i < n; ++i) { k[i].key = ekey[i]; k[i].idx = (uint32_t)i; k[i].pad = 0; }
  qsort(k, n, sizeof(skey_t), cmp_skey);
  seg->hits = (gen_hit*)malloc((n ? n : 1) * sizeof(gen_hit));
  seg->truth = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  for (uint64_t i = 0; i < n; ++i) { seg->hits[i] = h[k[i].idx]; seg->truth[i] = tr[k[i].idx]; }
  seg->n = n;
  seg->n_events = nev;
  free(k); free(h); free(tr); free(ekey); free(px); free(dead);
}

/* Expected hits per cluster of the configured mix (before edge/dead-time loss). */
double tpxgen_expected_cluster_size(const tpxgen_config* c) {
  double s = c->frac_dot + c->frac_track + c->frac_blob;
  if (s <= 0) return 1.0;
  lognorm_t dot = lognorm_make(2.46, 2.15, c->dot_min, c->dot_max);
  lognorm_t t0 = lognorm_make(7.22, 27.35, c->track_min, c->track_max);
  lognorm_t t1 = lognorm_make(23.33, 33.47, c->track_min, c->track_max);
  lognorm_t t2 = lognorm_make(60.27, 64.33, c->track_min, c->track_max);
  double e_trk = (lognorm_mean(&t0) + lognorm_mean(&t1) + lognorm_mean(&t2)) / 3.0;
  double lo = c->blob_min, hi = c->blob_max;
  double e_blob = hi > lo ? (hi - lo) / log(hi / lo) : lo;
  return (c->frac_dot * lognorm_mean(&dot) + c->frac_track * e_trk + c->frac_blob * e_blob) / s;
}

/* Generate exactly cfg->n_hits hits into hits_out (16-B records) and, when
 * truth_out != NULL, the generator's event id per hit.  Returns 0 on success,
 * -1 on bad arguments, -2 on allocation failure. */
int tpxgen_generate(const tpxgen_config* cfg, void* hits_out, uint32_t* truth_out) {
  if (!cfg || (!hits_out && cfg->n_hits) || cfg->width == 0 || cfg->height == 0 ||
      cfg->width > 65535 || cfg->height > 65535 || !(cfg->rate_hz > 0))
    return -1;
  if (cfg->n_hits == 0) return 0;
  gen_state g;
  g.c = *cfg;
  if (g.c.dot_min < 1) g.c.dot_min = 1;
  if (g.c.track_min < 1) g.c.track_min = 1;
  if (g.c.blob_min < 1) g.c.blob_min = 1;
  if (g.c.dot_max < g.c.dot_min) g.c.dot_max = g.c.dot_min;
  if (g.c.track_max < g.c.track_min) g.c.track_max = g.c.track_min;
  if (g.c.blob_max < g.c.blob_min) g.c.blob_max = g.c.blob_min;
  double fs = g.c.frac_dot + g.c.frac_track + g.c.frac_blob;
  if (!(fs > 0)) return -1;
  g.p_dot = g.c.frac_dot / fs;
  g.p_track = (g.c.frac_dot + g.c.frac_track) / fs;
  g.dot = lognorm_make(2.46, 2.15, g.c.dot_min, g.c.dot_max);
  g.trk[0] = lognorm_make(7.22, 27.35, g.c.track_min, g.c.track_max);
  g.trk[1] = lognorm_make(23.33, 33.47, g.c.track_min, g.c.track_max);
  g.trk[2] = lognorm_make(60.27, 64.33, g.c.track_min, g.c.track_max);
  double es = tpxgen_expected_cluster_size(&g.c);
  double hits_per_tick = g.c.rate_hz * TICK_S;
  g.lambda_per_tick = hits_per_tick / es;
  g.seg_len = (uint64_t)ceil(SEG_TARGET_HITS / hits_per_tick);
  if (g.seg_len < 1) g.seg_len = 1;

  gen_hit* out = (gen_hit*)hits_out;
  uint64_t filled = 0, ev_base = 0, sidx = 0;
  int nthr = 1;
#ifdef _OPENMP
  nthr = cfg->n_threads > 0 ? cfg->n_threads : omp_get_max_threads();
#endif
  int batch = nthr * 2;
  segment_t* segs = (segment_t*)calloc((size_t)batch, sizeof(segment_t));
  if (!segs) return -2;
  while (filled < cfg->n_hits) {
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthr)
#endif
    for (int b = 0; b < batch; ++b) gen_segment(&g, sidx + (uint64_t)b, &segs[b]);
    for (int b = 0; b < batch; ++b) {
      uint64_t take = segs[b].n;
      if (filled < cfg->n_hits) {
        if (take > cfg->n_hits - filled) take = cfg->n_hits - filled;
        memcpy(out + filled, segs[b].hits, take * sizeof(gen_hit));
        if (truth_out)
          for (uint64_t i = 0; i < take; ++i) truth_out[filled + i] = (uint32_t)(ev_base + segs[b].truth[i]);
        filled += take;
      }
      ev_base += segs[b].n_events;
      free(segs[b].hits); free(segs[b].truth);
      segs[b].hits = NULL; segs[b].truth = NULL;
    }
    sidx += (uint64_t)batch;
  }
  free(segs);
  return 0;
}
