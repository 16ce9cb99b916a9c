/*
 * tpx_cluster.h -- C ABI of the B200-native Timepix3 hit-clustering hot path.
 *
 * What is computed (the problem statement, §2 "Preliminaries --
 * clustering", lines 29-45, variant (iii)(a) "dynamic local-time-neighborhood",
 * line 39; graph reading of §2.1, lines 61-62; union-find over "the 8 neighboring
 * pixels plus the pixel itself", §4.1):
 *
 *   Hits h_0 .. h_{n-1} (§1 line 11: x, y, ToA, ToT) are the nodes of a
 *   graph. Hits i != j are joined by an edge iff
 *        max(|x_i - x_j|, |y_i - y_j|) <= 1        (8-neighbouring or same pixel)
 *    and |toa_i - toa_j| <= dt_max                 (integer ToA ticks, inclusive).
 *   A cluster is a connected component of that graph (reading R1: the
 *   "exists a path" reading of (iii)(a); R2: same-pixel hits are neighbours;
 *   R3: the bound is inclusive).
 *
 *   labels_out[i]  = the smallest input index of the cluster containing hit i.
 *   features_out[] = one record per cluster, in ascending label order.
 *
 * Units (reading R4): ToA in 1.5625 ns ticks, ToT in 25 ns ticks,
 * dt_max in ToA ticks (100/200/500 ns = 64/128/320 ticks).
 *
 * Everything here is plain C: pointers are either HOST or DEVICE as stated
 * per argument, sizes are element counts unless named *_bytes.  No entry
 * point throws; each returns a tpx_status (0 = TPX_OK).  A context is not
 * thread-safe: use one context per host thread / stream.
 */
#ifndef TPX_CLUSTER_H
#define TPX_CLUSTER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPX_ABI_VERSION 1

/* One pixel hit, 16 bytes, arrays must be 16-byte aligned (§1 l.11).
 * toa < 2^48.  0 <= x < width, 0 <= y < height (create-time sensor size).
 * `reserved` is ignored on input. */
typedef struct tpx_hit {
  uint64_t toa;      /* time of arrival, 1.5625 ns ticks                     */
  uint16_t x;        /* pixel column                                         */
  uint16_t y;        /* pixel row                                            */
  uint16_t tot;      /* time over threshold, 25 ns ticks                     */
  uint16_t reserved;
} tpx_hit;

/* Per-cluster integer features, 64 bytes (motivated by PAPER.md §1 l.17 and
 * §6 l.320; field list from BASELINE.json north_star; reading R8).
 * Coordinates are pixel indices.  The ToT-weighted centroid is
 * (sum_tot_x / tot_sum, sum_tot_y / tot_sum), see tpx_cluster_centroids(). */
typedef struct tpx_cluster_features {
  uint32_t label;    /* smallest input index in the cluster                  */
  uint32_t size;     /* number of hits                                       */
  uint64_t toa_min;  /* earliest ToA (ticks); span = toa_max - toa_min       */
  uint64_t toa_max;
  uint64_t tot_sum;  /* sum of ToT (ticks)                                   */
  uint64_t sum_x;
  uint64_t sum_y;
  uint64_t sum_tot_x;
  uint64_t sum_tot_y;
} tpx_cluster_features;

/* PAPER.md §2 (iii)(a) l.39, (iii)(b) l.40, (iii)(c) l.41.  Only LOCAL is
 * implemented on the GPU path; the others return TPX_ERR_UNSUPPORTED. */
enum {
  TPX_VARIANT_LOCAL = 0,
  TPX_VARIANT_GLOBAL = 1,
  TPX_VARIANT_STATIC = 2
};

enum {
  TPX_OK = 0,
  TPX_ERR_INVALID_ARG = -1,   /* null pointer, bad size, bad variant value     */
  TPX_ERR_UNSUPPORTED = -2,   /* variant != LOCAL                              */
  TPX_ERR_COORD_RANGE = -3,   /* some hit has x >= width or y >= height, or
                                 toa >= 2^48; outputs are unspecified          */
  TPX_ERR_TOO_MANY_HITS = -4, /* n >= 2^32 - 1 (labels are u32)                */
  TPX_ERR_CAPACITY = -5,      /* n_clusters > capacity: labels_out is valid,
                                 *n_clusters_out holds the required count,
                                 features_out holds the first `capacity`       */
  TPX_ERR_OOM = -6,           /* workspace too small                           */
  TPX_ERR_CUDA = -7,          /* a CUDA runtime call failed                    */
  TPX_ERR_NCCL = -8           /* an NCCL call failed (sharded path)            */
};

typedef struct tpx_cluster tpx_cluster;

/* Build-time ABI version (TPX_ABI_VERSION). */
int tpx_abi_version(void);

/* Static English text for a status code; never NULL. */
const char* tpx_status_string(int status);

/* Create a context.  dt_max_ticks: Delta t_max in ToA ticks (0 allowed: only
 * equal ToAs connect).  variant: TPX_VARIANT_*.  width/height: sensor size in
 * pixels, 1..32768 (256x256 Timepix3, 448x512 Timepix4).  *out receives the
 * context (host memory owned by the library, freed by tpx_cluster_destroy).
 * Errors: INVALID_ARG, UNSUPPORTED (variant != LOCAL), CUDA. */
int tpx_cluster_create(uint64_t dt_max_ticks, int variant, uint32_t width,
                       uint32_t height, tpx_cluster** out);

/* Destroy a context (NULL is a no-op).  Caller-owned buffers are untouched. */
void tpx_cluster_destroy(tpx_cluster* ctx);

/* Device workspace needed by tpx_cluster_run for n hits (bytes, >= 256). */
int tpx_cluster_workspace_bytes(const tpx_cluster* ctx, uint64_t n,
                                size_t* bytes);

/* Cluster n hits already resident in device memory.
 *   hits         DEVICE, n records, arrival order (any order is accepted;
 *                near-ToA-ordered input takes the fast sort path).
 *   labels_out   DEVICE, n u32, written in input order.
 *   features_out DEVICE, `capacity` records, ascending label; capacity = n is
 *                always enough.
 *   n_clusters_out HOST, receives the cluster count.
 *   workspace    DEVICE, >= tpx_cluster_workspace_bytes(n), 256-B aligned.
 *   stream       cudaStream_t (NULL = legacy default stream).
 * All work is stream-ordered on `stream`; the call returns after the cluster
 * count has been read back (one small device->host copy + stream sync).
 * n = 0 returns TPX_OK with 0 clusters.  The caller owns every buffer. */
int tpx_cluster_run(tpx_cluster* ctx, const tpx_hit* hits, uint64_t n,
                    uint32_t* labels_out, tpx_cluster_features* features_out,
                    uint64_t capacity, uint64_t* n_clusters_out,
                    void* workspace, size_t workspace_bytes, void* stream);

/* Device workspace needed by tpx_cluster_run_host: device staging for the
 * hits, labels and `capacity` feature records plus tpx_cluster_run's own. */
int tpx_cluster_host_workspace_bytes(const tpx_cluster* ctx, uint64_t n,
                                     uint64_t capacity, size_t* bytes);

/* End-to-end variant with HOST buffers (pinned memory recommended): copies
 * the hits host->device, runs tpx_cluster_run on device staging carved from
 * `workspace`, and copies labels (n u32) and the n_clusters feature records
 * back to host.  Same semantics and errors as tpx_cluster_run. */
int tpx_cluster_run_host(tpx_cluster* ctx, const tpx_hit* hits_host,
                         uint64_t n, uint32_t* labels_host,
                         tpx_cluster_features* features_host,
                         uint64_t capacity, uint64_t* n_clusters_out,
                         void* workspace, size_t workspace_bytes,
                         void* stream);

/* fp64 ToT-weighted centroids from feature records (north_star: "integer
 * moment sums for the centroid"; reading R8):
 *   cxy[2k]   = sum_tot_x / tot_sum,  cxy[2k+1] = sum_tot_y / tot_sum
 * (one IEEE-754 round-to-nearest division each); when tot_sum == 0 the
 * unweighted sum_x / size, sum_y / size is used.
 *   features DEVICE, n_clusters records; cxy DEVICE, 2*n_clusters doubles.
 * Stream-ordered, asynchronous (no sync). */
int tpx_cluster_centroids(const tpx_cluster_features* features,
                          uint64_t n_clusters, double* cxy, void* stream);

/* Diagnostics of the last run on this context (HOST struct). */
typedef struct tpx_run_stats {
  uint64_t n_hits;
  uint64_t n_clusters;
  uint32_t sort_path;      /* 0 = windowed bounded-disorder sort,
                              1 = global radix fallback                      */
  uint32_t sort_retries;   /* windowed attempts that failed verification     */
  uint64_t cross_pairs;    /* tile-border union pairs processed              */
  uint32_t kernel_launches;/* kernels launched by the last run               */
  uint32_t n_stages;       /* valid entries in stage_ms / stage names        */
  float stage_ms[16];      /* per-stage device time (only when profiling)    */
  uint64_t open_hits;      /* hits of tile-border-crossing components        */
  uint64_t overflow_hits;  /* hits whose ToA window left the staged halo     */
  uint64_t tile_phase_cycles[16]; /* tile-kernel phase clocks, summed over
                              CTAs (only when profiling; diagnostics)        */
} tpx_run_stats;

int tpx_cluster_last_stats(const tpx_cluster* ctx, tpx_run_stats* out);

/* Enable (1) / disable (0) per-stage CUDA-event timing inside tpx_cluster_run
 * (events are recorded on the run stream; adds no synchronisation beyond the
 * run's own final sync). */
int tpx_cluster_set_profiling(tpx_cluster* ctx, int enable);

/* Static name of stage i (0 <= i < 16) as reported in stage_ms; "" if unused. */
const char* tpx_cluster_stage_name(int i);

#ifdef __cplusplus
}
#endif

#endif /* TPX_CLUSTER_H */
