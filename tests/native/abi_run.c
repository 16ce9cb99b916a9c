/*
 * abi_run.c -- a plain C caller of the C ABI (include/tpx_cluster.h), no
 * PyTorch, no Python: test infrastructure for tests/test_gpu_sanitizer.py.
 * It reads n 16-byte tpx_hit records from a file, copies them to the device,
 * runs tpx_cluster_run once (or tpx_cluster_run_grouped), and writes the
 * labels (u32[n]) and feature records (64 B each) to files.  Running it under
 * compute-sanitizer checks the library's kernels (memcheck / racecheck /
 * synccheck / initcheck) without any other kernel in the process.
 *
 *   abi_run hits.bin dt width height labels.out feats.out [tile_mode] [variant]
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "tpx_cluster.h"

static void die(const char* what, int rc) {
  fprintf(stderr, "abi_run: %s: %d (%s)\n", what, rc, rc < 0 ? tpx_status_string(rc) : "");
  exit(2);
}

int main(int argc, char** argv) {
  if (argc < 7) {
    fprintf(stderr, "usage: %s hits.bin dt width height labels.out feats.out [tile_mode] [variant]\n", argv[0]);
    return 1;
  }
  const unsigned long long dt = strtoull(argv[2], 0, 10);
  const unsigned W = (unsigned)atoi(argv[3]), H = (unsigned)atoi(argv[4]);
  const int tile_mode = argc > 7 ? atoi(argv[7]) : 0;
  const int variant = argc > 8 ? atoi(argv[8]) : 0;
  FILE* f = fopen(argv[1], "rb");
  if (!f) die("open hits", -1);
  fseek(f, 0, SEEK_END);
  const long bytes = ftell(f);
  fseek(f, 0, SEEK_SET);
  const uint64_t n = (uint64_t)bytes / sizeof(tpx_hit);
  tpx_hit* h = (tpx_hit*)malloc(bytes ? bytes : 16);
  if (bytes && fread(h, 1, bytes, f) != (size_t)bytes) die("read hits", -1);
  fclose(f);

  tpx_cluster* c = NULL;
  int rc = tpx_cluster_create(dt, variant, W, H, &c);
  if (rc) die("create", rc);
  if (tile_mode && (rc = tpx_cluster_set_tile_mode(c, tile_mode))) die("tile mode", rc);
  size_t ws_bytes = 0;
  if ((rc = tpx_cluster_workspace_bytes(c, n, &ws_bytes))) die("workspace", rc);
  void *d_hits = NULL, *d_labels = NULL, *d_feats = NULL, *d_ws = NULL;
  const uint64_t nn = n ? n : 1;
  if (cudaMalloc(&d_hits, nn * 16) || cudaMalloc(&d_labels, nn * 4) || cudaMalloc(&d_feats, nn * 64) ||
      cudaMalloc(&d_ws, ws_bytes))
    die("cudaMalloc", -7);
  if (n && cudaMemcpy(d_hits, h, n * 16, cudaMemcpyHostToDevice)) die("H2D", -7);
  cudaStream_t s;
  cudaStreamCreate(&s);
  uint64_t k = 0;
  rc = tpx_cluster_run(c, (const tpx_hit*)d_hits, n, (uint32_t*)d_labels, (tpx_cluster_features*)d_feats, n, &k,
                       d_ws, ws_bytes, s);
  if (rc) die("run", rc);
  if (cudaStreamSynchronize(s)) die("sync", -7);
  uint32_t* labels = (uint32_t*)malloc(nn * 4);
  tpx_cluster_features* feats = (tpx_cluster_features*)malloc((k ? k : 1) * 64);
  if (n && cudaMemcpy(labels, d_labels, n * 4, cudaMemcpyDeviceToHost)) die("D2H labels", -7);
  if (k && cudaMemcpy(feats, d_feats, k * 64, cudaMemcpyDeviceToHost)) die("D2H feats", -7);
  FILE* fl = fopen(argv[5], "wb");
  FILE* ff = fopen(argv[6], "wb");
  if (!fl || !ff) die("open outputs", -1);
  fwrite(labels, 4, n, fl);
  fwrite(feats, 64, k, ff);
  fclose(fl);
  fclose(ff);
  tpx_run_stats st;
  tpx_cluster_last_stats(c, &st);
  printf("abi_run ok: n=%llu k=%llu launches=%u dense=%d sort_path=%d\n", (unsigned long long)n,
         (unsigned long long)k, (unsigned)st.kernel_launches, (int)st.tile_dense, (int)st.sort_path);
  tpx_cluster_destroy(c);
  cudaFree(d_hits);
  cudaFree(d_labels);
  cudaFree(d_feats);
  cudaFree(d_ws);
  cudaStreamDestroy(s);
  free(h);
  free(labels);
  free(feats);
  return 0;
}
