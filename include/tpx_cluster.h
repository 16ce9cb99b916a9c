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

/* PAPER.md §2 (iii)(a) l.39, (iii)(b) l.40, (iii)(c) l.41.  LOCAL is the
 * connected-component definition above.  GLOBAL and STATIC follow the
 * streaming convention (R11, R21): hits in (toa, index) order; a
 * hit joins every existing cluster that has a member on one of its 9
 * neighbouring pixels and satisfies toa - cluster.maxToA <= dt_max (GLOBAL)
 * or toa - cluster.minToA <= dt_max (STATIC); all joinable clusters merge.
 * Labels and records are defined as for LOCAL.  GLOBAL/STATIC contexts need
 * a larger workspace (tpx_cluster_workspace_bytes) and support neither
 * run_partial with n_owned < n nor the stream API. */
enum {
  TPX_VARIANT_LOCAL = 0,
  TPX_VARIANT_GLOBAL = 1,
  TPX_VARIANT_STATIC = 2
};

enum {
  TPX_OK = 0,
  TPX_ERR_INVALID_ARG = -1,   /* null pointer, bad size, bad variant value     */
  TPX_ERR_UNSUPPORTED = -2,   /* operation not available for this variant      */
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
 * Errors: INVALID_ARG, CUDA. */
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
 * count has been read back (a one-block kernel stores it into mapped pinned
 * memory, then a stream sync -- no copy-engine transfer, so a run never waits
 * behind another buffer's bulk copy; a second read-back after the sort carries
 * its verification and the window-density probe).  The windowed sort is
 * verified before any clustering work; when its displacement bound fails the
 * run retries with wider windows (D = 1024, 2560, 3072), then the global
 * radix sort, and the context starts later runs at the attempt that succeeded
 * (results are identical on every path; tpx_run_stats reports the path).
 * n = 0 returns TPX_OK with 0 clusters.  The caller owns every buffer.
 * Not thread-safe per context (one context per stream). */
int tpx_cluster_run(tpx_cluster* ctx, const tpx_hit* hits, uint64_t n,
                    uint32_t* labels_out, tpx_cluster_features* features_out,
                    uint64_t capacity, uint64_t* n_clusters_out,
                    void* workspace, size_t workspace_bytes, void* stream);

/* tpx_cluster_run for a sharded rank: the first n_owned hits are this rank's
 * own, the remaining n - n_owned are a halo borrowed from the next rank.
 * Connectivity uses all n hits; features count only the owned hits, and
 * records are produced only for clusters whose label (smallest input index)
 * is < n_owned (the halo must be stored after the owned hits).  labels_out
 * covers all n hits.  Same buffers, errors and synchronisation as
 * tpx_cluster_run (which is run_partial with n_owned = n). */
int tpx_cluster_run_partial(tpx_cluster* ctx, const tpx_hit* hits, uint64_t n,
                            uint64_t n_owned, uint32_t* labels_out,
                            tpx_cluster_features* features_out,
                            uint64_t capacity, uint64_t* n_clusters_out,
                            void* workspace, size_t workspace_bytes,
                            void* stream);

/* Per-cluster shape record, 32 bytes: the bounding box, "the smallest
 * rectangle (aligned with the sensor) enclosing the cluster" (§3.3
 * l.132), and the unweighted second moments sum x^2, sum x*y, sum y^2 (shape
 * features, §1 l.15; reading R19).  Coordinates are pixel indices. */
typedef struct tpx_cluster_shape {
  uint16_t x_min, x_max, y_min, y_max;
  uint64_t sum_xx;
  uint64_t sum_xy;
  uint64_t sum_yy;
} tpx_cluster_shape;

/* tpx_cluster_run plus the cluster-contiguous hit order of Alg. "High-level
 * GPU clustering" Step 6 (§4 l.175: "Sort clusters by their minimum
 * time of arrival, causing the hits from the same cluster to form adjacent
 * memory blocks"; reading R18: hits are ordered by (toa, input
 * index), a cluster is placed by its earliest hit in that order, and inside
 * its block the hits keep that order).  Uses tpx_cluster_workspace_bytes(n).
 *   labels_out, features_out, capacity, n_clusters_out: as tpx_cluster_run;
 *                  capacity must be >= n_clusters (else TPX_ERR_CAPACITY with
 *                  valid labels and no grouping outputs).
 *   shapes_out     DEVICE, `capacity` records in features_out order, or NULL.
 *   order_out      DEVICE, n u32 input indices: block g is
 *                  order_out[offsets_out[g] .. offsets_out[g+1]).
 *   offsets_out    DEVICE, n_clusters + 1 u32 (offsets_out[n_clusters] = n).
 *   cluster_of_out DEVICE, n_clusters u32: block g holds the cluster
 *                  features_out[cluster_of_out[g]].
 * Returns after the whole pass completed on `stream` (stream sync). */
int tpx_cluster_run_grouped(tpx_cluster* ctx, const tpx_hit* hits, uint64_t n,
                            uint32_t* labels_out,
                            tpx_cluster_features* features_out,
                            tpx_cluster_shape* shapes_out, uint64_t capacity,
                            uint64_t* n_clusters_out, uint32_t* order_out,
                            uint32_t* offsets_out, uint32_t* cluster_of_out,
                            void* workspace, size_t workspace_bytes,
                            void* stream);

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
  uint32_t sort_retries;   /* windowed attempts that failed verification in
                              this run (grouped runs: + 1 if the windowed
                              key sort of the grouping fell back)            */
  uint64_t cross_pairs;    /* tile-border union pairs processed              */
  uint32_t kernel_launches;/* kernels launched by the last run               */
  uint32_t n_stages;       /* valid entries in stage_ms / stage names        */
  float stage_ms[16];      /* per-stage device time (only when profiling)    */
  uint64_t open_hits;      /* hits of tile-border-crossing components        */
  uint64_t overflow_hits;  /* hits whose ToA window left the staged halo     */
  uint64_t tile_phase_cycles[16]; /* tile-kernel phase clocks, summed over
                              CTAs (only when profiling; diagnostics)        */
  uint32_t tile_dense;     /* 1 if the dense (large-halo) tile configuration
                              ran (window-density probe)                     */
  uint32_t reserved0;
} tpx_run_stats;

int tpx_cluster_last_stats(const tpx_cluster* ctx, tpx_run_stats* out);

/* 0: off.  1: per-stage CUDA-event timing inside tpx_cluster_run (events are
 * recorded on the run stream; adds no synchronisation beyond the run's own
 * final sync).  2: also per-phase clock counters inside the tile kernel
 * (diagnostics; slows the kernel).  Errors: INVALID_ARG. */
int tpx_cluster_set_profiling(tpx_cluster* ctx, int enable);

/* Tile configuration of the clustering kernel: TPX_TILE_AUTO (default) lets
 * a window-density probe on the sorted stream choose; TPX_TILE_SPARSE (2048-hit
 * tiles, counting-sorted 2x2-pixel cell index with backward hooking for
 * sensors up to 1024 x 1024, else the linked-list cell index) /
 * TPX_TILE_DENSE (pixel hash, large halo) force one; TPX_TILE_CELL forces the
 * linked-list cell kernel (kept for comparison and wide sensors).
 * TPX_TILE_COLUMN (round 1's column-bucket kernel) is no longer available:
 * INVALID_ARG.  Results are identical; only speed differs -- the parity
 * tests cover every mode.  Errors: INVALID_ARG. */
enum { TPX_TILE_AUTO = 0, TPX_TILE_SPARSE = 1, TPX_TILE_DENSE = 2, TPX_TILE_COLUMN = 3, TPX_TILE_CELL = 4 };
int tpx_cluster_set_tile_mode(tpx_cluster* ctx, int mode);

/* Static name of stage i (0 <= i < 16) as reported in stage_ms; "" if unused. */
const char* tpx_cluster_stage_name(int i);

/* ------------------------------------------------------------------------
 * Host-buffer pipeline (copy/compute overlap across buffers).
 *
 * The paper's GPU driver copies a filled host buffer to the device, clusters
 * it and copies the result back, with buffers cycling "in use" / "reusable"
 * (Alg. "High-level GPU clustering") and copies hidden
 * behind compute with CUDA streams (l.310).  A pipeline has `depth` slots,
 * each with its own context, stream and slice of one caller-provided DEVICE
 * workspace; one native worker thread per slot runs tpx_cluster_run_host on
 * the buffers submitted to it (round robin), so H2D / D2H of one buffer
 * overlap the kernels of another.  Every buffer is an independent closed
 * stream (results identical to tpx_cluster_run_host).  Host buffers are
 * owned by the caller and must stay valid (pinned recommended) until
 * tpx_pipeline_wait returns for their ticket.
 * ---------------------------------------------------------------------- */
typedef struct tpx_pipeline tpx_pipeline;

/* Device workspace for a pipeline of `depth` (1..16) slots, each able to hold
 * max_hits hits and `capacity` feature records. */
int tpx_pipeline_workspace_bytes(const tpx_cluster* proto, uint64_t max_hits,
                                 uint64_t capacity, int depth, size_t* bytes);

/* Create a pipeline on the current device (contexts as tpx_cluster_create).
 * workspace: DEVICE, 256-B aligned, >= tpx_pipeline_workspace_bytes. */
int tpx_pipeline_create(uint64_t dt_max_ticks, int variant, uint32_t width,
                        uint32_t height, uint64_t max_hits, uint64_t capacity,
                        int depth, void* workspace, size_t workspace_bytes,
                        tpx_pipeline** out);

/* Queue one HOST buffer (n <= max_hits, capacity <= the pipeline's);
 * *ticket identifies it for tpx_pipeline_wait.  Non-blocking. */
int tpx_pipeline_submit(tpx_pipeline* p, const tpx_hit* hits_host, uint64_t n,
                        uint32_t* labels_host,
                        tpx_cluster_features* features_host,
                        uint64_t capacity, uint64_t* ticket);

/* Block until buffer `ticket` is done; returns its tpx_cluster_run_host
 * status and cluster count (HOST). Each ticket can be waited on once. */
int tpx_pipeline_wait(tpx_pipeline* p, uint64_t ticket,
                      uint64_t* n_clusters_out);

/* Device timing across the slot streams: mark(0) records a start event on
 * every slot stream, mark(1) a stop event; elapsed_ms = latest stop minus
 * earliest start (CUDA events; synchronises on the stop events). */
int tpx_pipeline_mark(tpx_pipeline* p, int which);
int tpx_pipeline_elapsed_ms(tpx_pipeline* p, float* ms);

/* Stop the workers (after finishing queued buffers) and free the slots. */
void tpx_pipeline_destroy(tpx_pipeline* p);

/* ------------------------------------------------------------------------
 * ToA-sharded multi-GPU clustering; one process per
 * GPU, one rank per process.
 *
 * Method: temporal splitting (§3.2.3 l.117-119: "we only need to
 * examine the dt_max-time neighborhood around each border") with the GPU's
 * border stitching (§4 l.173).  Rank r owns the contiguous input-index block
 * [o_r, o_r + n_r) of the t-ordered stream (§3.1 l.99-100), o_r = n_0 + ... +
 * n_{r-1}.  Edges only join hits within dt_max in ToA (§2 (iii)(a) l.39), so
 * every edge between ranks r and r+1 has its rank-(r+1) end among the hits
 * with toa <= maxToA(r) + dt_max (the "halo" rank r+1 lends to rank r),
 * provided no edge skips a rank: minToA(r+2) > maxToA(r) + dt_max for every r
 * (checked; TPX_ERR_UNSUPPORTED otherwise).  One run:
 *   1. all-gather [n_r, minToA, maxToA] (+ halo counts); rank r+1 selects and
 *      sends its halo to rank r (NCCL send/recv);
 *   2. each rank clusters [owned | halo] (the tpx_cluster_run kernels; only
 *      owned hits contribute features), labels written as global indices;
 *   3. rank r+1 returns its labels of the lent hits; each (label on r, label
 *      on r+1) pair of a halo hit is all-gathered, every rank unites all
 *      pairs (smallest label wins = label of the merged cluster, reading R6);
 *   4. owned labels are relabelled; records of clusters whose final label is
 *      elsewhere are all-gathered as partials and folded (integer add / min /
 *      max: exact, order independent) by the rank owning the final label.
 * Output: labels of the owned hits (global input indices) and the records of
 * the clusters whose label falls in [o_r, o_r + n_r), ascending -- so the
 * ranks' outputs concatenated in rank order equal tpx_cluster_run on the
 * whole stream byte for byte.  Variant (iii)(a) only.
 * ---------------------------------------------------------------------- */

typedef struct tpx_comm tpx_comm;

/* NCCL bootstrap (multi-GPU product path).  Rank 0 calls tpx_nccl_unique_id
 * and distributes the 128 bytes to every rank (e.g. over the torch process
 * group); every rank then calls tpx_nccl_comm_init on its own CUDA device
 * (the current device of the calling thread).  The communicator is owned by
 * the library (tpx_comm_destroy frees it).  libnccl.so.2 is loaded with
 * dlopen on first use.  Errors: NCCL (library missing or an NCCL call
 * failed), INVALID_ARG. */
int tpx_nccl_unique_id(uint8_t id_out[128]);
int tpx_nccl_comm_init(int rank, int world, const uint8_t id[128],
                       tpx_comm** out);

/* Host-callback transport (functional runs where NCCL cannot be used:
 * in-process virtual ranks, gloo process groups, several ranks on one GPU).
 * Device buffers are staged through pinned host memory.  Callbacks return 0
 * on success; HOST pointers:
 *   allgather(user, send, recv, bytes): recv[r*bytes .. (r+1)*bytes) =
 *       rank r's send (bytes each, world ranks);
 *   sendrecv(user, to, send, send_bytes, from, recv, recv_bytes): send to
 *       rank `to` and receive from rank `from` (-1: none) concurrently. */
typedef int (*tpx_allgather_fn)(void* user, const void* send, void* recv,
                                size_t bytes);
typedef int (*tpx_sendrecv_fn)(void* user, int to, const void* send,
                               size_t send_bytes, int from, void* recv,
                               size_t recv_bytes);
int tpx_comm_create_host(int rank, int world, tpx_allgather_fn allgather,
                         tpx_sendrecv_fn sendrecv, void* user, tpx_comm** out);

void tpx_comm_destroy(tpx_comm* comm);
int tpx_comm_rank(const tpx_comm* comm, int* rank, int* world);

/* Host-buffer self test of a communicator (no GPU needed for host
 * transports): every rank all-gathers `bytes` bytes of a rank-dependent
 * pattern and exchanges a pattern with its neighbours (to r-1, from r+1);
 * returns TPX_OK iff every received byte is as expected. */
int tpx_comm_selftest(tpx_comm* comm, size_t bytes);

/* Device workspace of tpx_cluster_run_sharded for n_local owned hits on a
 * communicator of `world` ranks (bytes). */
int tpx_cluster_sharded_workspace_bytes(const tpx_cluster* ctx, uint64_t n_local,
                                        int world, size_t* bytes);

/* Halo capacity: hits one rank may lend to the previous one per run
 * (TPX_ERR_UNSUPPORTED beyond; ~ rate x (readout disorder + dt_max)). */
#define TPX_SHARD_HALO_CAP (1u << 18)

/* The sharded run (every rank calls it, collectively, on its own stream).
 *   local_hits        DEVICE, n_local >= 1 owned hits (the block), 16-B aligned
 *   labels_out_local  DEVICE, n_local entries: global labels of owned hits
 *   features_out_local DEVICE, capacity records: clusters whose label is in
 *                     this rank's block, ascending label
 *   n_local_clusters_out HOST: number of those records (> capacity: CAPACITY,
 *                     labels valid, records truncated)
 *   global_offset_out HOST, may be NULL: o_r
 * Total hits < 2^32 - 1.  Host synchronisations: 3 (counts after the halo
 * exchange, the sort status, the final count).  Errors: INVALID_ARG,
 * UNSUPPORTED (variant, sensor wider than 1024 px, a rank-skipping edge, halo
 * above TPX_SHARD_HALO_CAP), COORD_RANGE, TOO_MANY_HITS, CAPACITY, OOM, CUDA,
 * NCCL -- the same status on every rank. */
int tpx_cluster_run_sharded(tpx_cluster* ctx, tpx_comm* comm,
                            const tpx_hit* local_hits, uint64_t n_local,
                            uint32_t* labels_out_local,
                            tpx_cluster_features* features_out_local,
                            uint64_t capacity, uint64_t* n_local_clusters_out,
                            uint64_t* global_offset_out, void* workspace,
                            size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Streaming ingest: Alg. "Hit buffer filling" (PAPER.md
 * §4 l.184-213) feeding Alg. "High-level GPU clustering" (l.160-182) with
 * exact carry-over of clusters open at a buffer border.
 *
 * Hits are pushed in readout (arrival) order; arrival index a = number of
 * hits pushed before.  A buffer is sent when storeHit says so; its cut is
 * C = toa_max + t_closing, and since the stream is t-ordered (l.99-100) every
 * later hit has toa >= C.  A cluster with a hit within dt_max of C stays open:
 * its hits are kept on the device and clustered again with the next buffer;
 * every other cluster is final and is emitted in a batch.  The union of all
 * batches equals tpx_cluster_run on the whole stream, with
 *   label = the smallest ARRIVAL index of the cluster (u64),
 * and in each batch clusters in Step-6 order (l.175, reading R18: by earliest
 * hit in (toa, arrival index) order), each cluster's hits contiguous in
 * (toa, arrival index) order (Step 8: "Transfer hits and labels").  Hits that
 * violate t-orderedness (toa < the last sent cut) are counted in late_hits;
 * results are then not guaranteed exact.  Device memory: caller workspace.
 * Not thread-safe.  Buffers are clustered synchronously inside push/flush on
 * `cuda_stream`.
 */
typedef struct tpx_stream tpx_stream;

typedef struct tpx_stream_config {
  uint64_t dt_max_ticks;     /* Delta t_max (ToA ticks)                       */
  uint32_t width, height;    /* sensor size, as tpx_cluster_create            */
  uint64_t buffer_hits;      /* b: maximum buffer size                        */
  uint64_t reserve_hits;     /* b_t < b: hits that can arrive in t + t_closing */
  uint64_t disorder_ticks;   /* t: the stream is t-ordered                    */
  uint64_t closing_ticks;    /* t_closing (expected cluster duration)         */
  uint64_t max_device_hits;  /* >= b + b_t: device room per buffer including
                                the carried hits of open clusters (< 2^32-1) */
} tpx_stream_config;

/* One emitted cluster, 80 bytes.  Hits: batch.hits[offset .. offset+size). */
typedef struct tpx_stream_cluster {
  uint64_t label;            /* smallest arrival index in the cluster         */
  uint64_t offset;           /* first hit of the cluster in the batch         */
  uint32_t size;
  uint32_t reserved;
  uint64_t toa_min, toa_max, tot_sum, sum_x, sum_y, sum_tot_x, sum_tot_y;
} tpx_stream_cluster;

typedef struct tpx_stream_batch {
  uint64_t seq;                        /* buffer sequence number             */
  uint64_t n_clusters, n_hits;
  const tpx_stream_cluster* clusters;  /* HOST, owned by the stream, valid
                                          until the next pop or destroy      */
  const tpx_hit* hits;                 /* HOST, n_hits, cluster blocks       */
  const uint64_t* hit_index;           /* HOST, n_hits arrival indices       */
} tpx_stream_batch;

typedef struct tpx_stream_stats {
  uint64_t hits_in, hits_out, clusters_out, buffers;
  uint64_t carried_max, carried_last;  /* hits of open clusters kept on device */
  uint64_t late_hits;                  /* t-orderedness violations           */
  double device_ms;                    /* summed per-buffer H2D..D2H time    */
} tpx_stream_stats;

/* Errors: INVALID_ARG (b <= b_t, max_device_hits < b + b_t or >= 2^32-1). */
int tpx_stream_workspace_bytes(const tpx_stream_config* cfg, size_t* bytes);
/* workspace: DEVICE, 256-B aligned, >= tpx_stream_workspace_bytes.  *out is
 * owned by the library (tpx_stream_destroy).  Errors: INVALID_ARG, OOM, CUDA. */
int tpx_stream_create(const tpx_stream_config* cfg, void* workspace,
                      size_t workspace_bytes, void* cuda_stream,
                      tpx_stream** out);
/* hits_host: HOST, n records in arrival order (copied; pinned not required).
 * Clusters every buffer that becomes full.  Errors: INVALID_ARG (after
 * flush), CAPACITY (a buffer plus carried hits exceeds max_device_hits), OOM,
 * CUDA, COORD_RANGE. */
int tpx_stream_push(tpx_stream* s, const tpx_hit* hits_host, uint64_t n);
/* End of stream: sends what is buffered; every cluster is closed. */
int tpx_stream_flush(tpx_stream* s);
/* Returns 1 and fills *out with the oldest unread batch, 0 if none (<0 on
 * error).  The previous batch's memory is recycled by this call. */
int tpx_stream_pop(tpx_stream* s, tpx_stream_batch* out);
int tpx_stream_get_stats(const tpx_stream* s, tpx_stream_stats* out);
void tpx_stream_destroy(tpx_stream* s);

/* One-shot host-to-host run of a whole stream held in host memory -- the
 * paper's GPU benchmark clock (§5 l.278-280: from a populated host
 * buffer until the clustered data is back on the host).  Same BufFill
 * decisions, carry and results as tpx_stream_push + flush, without host-side
 * copies of the input (runs go to the device straight from hits_host, which
 * should be pinned), and with copy/compute overlap across buffers (l.310).
 *   hits_host     HOST, n < 2^32 - 1 hits in arrival order.
 *   order_out     HOST, n u32: arrival indices, cluster blocks back to back
 *                 (buffer after buffer, Step-6 order inside a buffer).
 *   clusters_out  HOST, `capacity` records; offset = position in order_out.
 *   n_clusters_out HOST: number of clusters (TPX_ERR_CAPACITY if > capacity;
 *                 the first `capacity` records are written).
 *   workspace     DEVICE, >= tpx_stream_run_host_workspace_bytes(cfg).
 *   stats_out     HOST, may be NULL; device_ms = first H2D to last D2H.
 * Synchronous: returns when every result is in host memory. */
int tpx_stream_run_host_workspace_bytes(const tpx_stream_config* cfg,
                                        size_t* bytes);
int tpx_stream_run_host(const tpx_stream_config* cfg, const tpx_hit* hits_host,
                        uint64_t n, uint32_t* order_out,
                        tpx_stream_cluster* clusters_out, uint64_t capacity,
                        uint64_t* n_clusters_out, void* workspace,
                        size_t workspace_bytes, void* cuda_stream,
                        tpx_stream_stats* stats_out);

/* Host-only helper (no GPU): the buffer each hit is sent in by Alg. "Hit
 * buffer filling" (buffer_id_out[n], HOST) and each buffer's cut (cuts_out,
 * HOST, cuts_cap entries; the final buffer's cut is UINT64_MAX), exactly as
 * tpx_stream_push/flush assign them.  Errors: INVALID_ARG, CAPACITY
 * (more than cuts_cap buffers; *n_buffers_out holds the count). */
int tpx_buffill_assign(const tpx_hit* hits, uint64_t n, uint64_t b,
                       uint64_t b_t, uint64_t t, uint64_t t_closing,
                       uint32_t* buffer_id_out, uint64_t* cuts_out,
                       uint64_t cuts_cap, uint64_t* n_buffers_out);

#ifdef __cplusplus
}
#endif

#endif /* TPX_CLUSTER_H */
