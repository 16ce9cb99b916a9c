// common.cuh -- shared device types and helpers of the CUDA path (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "tpx_cluster.h"

// Bounds checks of the checked build (build.py --checked: -DTPX_CHECKED, a
// separate lib/checked/libtpxcluster.so used only by tests/test_gpu_checked.py):
// a failing check is a device-side assert (file, line, failing index printed;
// the launch reports cudaErrorAssert).  The product build compiles them out.
#ifdef TPX_CHECKED
#undef NDEBUG
#include <cassert>
#define TPX_BOUND(i, n) assert((unsigned long long)(i) < (unsigned long long)(n))
#else
#define TPX_BOUND(i, n) ((void)0)
#endif

// Sorted records gathered per thread and step (their loads in flight
// together) at the end of the window sort and of the last radix pass.
// Measured (A/B of builds, one box): window sort 1 / 2 / 4 -> mixed 200M
// 4.037 / 4.07 / 4.041 ms (Timepix4 6.716 / 6.649 / 6.679); radix 1 / 2 / 4
// -> heavy-ion 50M sort 2.411 / 2.327 / 2.303 ms.
#ifndef TPX_WSORT_GATHER_U
#define TPX_WSORT_GATHER_U 1
#endif
#ifndef TPX_RADIX_GATHER_U
#define TPX_RADIX_GATHER_U 4
#endif

namespace tpx {

constexpr unsigned kFull = 0xffffffffu;

// Sorted hit record, 16 B, the in-HBM layout after the ToA sort (DESIGN.md
// "HBM layout"): tt = toa << 16 | tot (toa < 2^48), xy = y << 16 | x,
// idx = input index.  One 128-bit load gives everything the window search,
// the union-find and the feature reductions need.
struct __align__(16) srec {
  uint64_t tt;
  uint32_t xy;
  uint32_t idx;
};
static_assert(sizeof(srec) == 16, "srec is 16 bytes");

__device__ __forceinline__ uint64_t srec_toa(const srec& r) { return r.tt >> 16; }
__device__ __forceinline__ uint32_t srec_tot(const srec& r) { return (uint32_t)(r.tt & 0xffffu); }
__device__ __forceinline__ uint32_t srec_x(const srec& r) { return r.xy & 0xffffu; }
__device__ __forceinline__ uint32_t srec_y(const srec& r) { return r.xy >> 16; }

__device__ __forceinline__ srec load_srec(const srec* p) {
  uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
  srec r;
  r.tt = (uint64_t)v.x | ((uint64_t)v.y << 32);
  r.xy = v.z;
  r.idx = v.w;
  return r;
}

__device__ __forceinline__ void store_srec(srec* p, const srec& r) {
  uint4 v;
  v.x = (uint32_t)r.tt;
  v.y = (uint32_t)(r.tt >> 32);
  v.z = r.xy;
  v.w = r.idx;
  *reinterpret_cast<uint4*>(p) = v;
}

// Input hit (tpx_hit) as one 128-bit load.
struct hit4 {
  uint64_t toa;
  uint32_t x, y, tot;
};
__device__ __forceinline__ hit4 load_hit(const tpx_hit* h) {
  uint4 v = __ldg(reinterpret_cast<const uint4*>(h));
  hit4 r;
  r.toa = (uint64_t)v.x | ((uint64_t)v.y << 32);
  r.x = v.z & 0xffffu;
  r.y = v.z >> 16;
  r.tot = v.w & 0xffffu;
  return r;
}

// L2 eviction-priority hints (createpolicy + ld/st .L2::cache_hint): the
// window sort loads its window "evict last" so the record gather at the end
// of the CTA finds the lines still in L2, and gathers / stores the records it
// will not touch again "evict first".
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ldg_v4_hint(const void* ptr, uint64_t pol) {
  uint4 v;
  asm("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ void stg_v4_hint(void* ptr, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ hit4 load_hit_hint(const tpx_hit* h, uint64_t pol) {
  const uint4 v = ldg_v4_hint(h, pol);
  hit4 r;
  r.toa = (uint64_t)v.x | ((uint64_t)v.y << 32);
  r.x = v.z & 0xffffu;
  r.y = v.z >> 16;
  r.tot = v.w & 0xffffu;
  return r;
}

// Input of the sort kernels: one array, or two concatenated segments (the
// sharded path sorts [owned hits | halo received from the next rank] without
// copying the caller's owned hits): element i is a[i] for i < na, else
// b[i - na].  Implicit from a plain pointer (one segment).
struct hit_src {
  const tpx_hit* a;
  const tpx_hit* b;
  uint64_t na;
  __host__ __device__ hit_src(const tpx_hit* p = nullptr) : a(p), b(nullptr), na(~0ull) {}
  __host__ __device__ hit_src(const tpx_hit* p, uint64_t n1, const tpx_hit* q) : a(p), b(q), na(n1) {}
  __device__ __forceinline__ const tpx_hit* operator+(uint64_t i) const { return i < na ? a + i : b + (i - na); }
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Coherent (L2) load: parent pointers are written concurrently by other CTAs.
__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) { return __ldcg(p); }

// ---------------------------------------------------------------- union-find
// Parent forest over sorted positions (§4.1 l.215).  Links always go
// from the larger root index to the smaller one, so parent(v) <= v, roots are
// the earliest hit of their tree in (ToA, input index) order and the paper's
// time-invariant toa(h) >= toa(parent(h)) (l.219-221) holds by construction.
// find() compresses paths by halving (l.221, "path compression").
__device__ __forceinline__ uint32_t uf_find(uint32_t* parent, uint32_t v) {
  uint32_t cur = ld_cg(parent + v);
  if (cur != v) {
    uint32_t prev = v, next;
    while (cur > (next = ld_cg(parent + cur))) {
      parent[prev] = next;   // benign race: next is an ancestor of prev
      prev = cur;
      cur = next;
    }
  }
  return cur;
}

// Read-only find for the flatten pass: path-halving stores from other threads
// could otherwise overwrite a root another thread has just stored.
__device__ __forceinline__ uint32_t uf_root(const uint32_t* parent, uint32_t v) {
  uint32_t cur = ld_cg(parent + v), next;
  while (cur != (next = ld_cg(parent + cur))) cur = next;
  return cur;
}

// Lock-free union by atomicCAS on the larger root (ECL-CC style hooking).
__device__ __forceinline__ void uf_unite(uint32_t* parent, uint32_t a, uint32_t b) {
  uint32_t ra = uf_find(parent, a), rb = uf_find(parent, b);
  while (ra != rb) {
    if (ra < rb) {
      uint32_t old = atomicCAS(parent + rb, rb, ra);
      if (old == rb) break;
      rb = old;
    } else {
      uint32_t old = atomicCAS(parent + ra, ra, rb);
      if (old == ra) break;
      ra = old;
    }
  }
}

// The same union with both walks climbing in lockstep (the two parent loads
// of a step are independent, so the L2 round trips overlap) and stopping as
// soon as they meet.  A climb step halves the path (benign race as above).
__device__ __forceinline__ void uf_unite_il(uint32_t* parent, uint32_t a, uint32_t b) {
  for (;;) {
    if (a == b) return;
    const uint32_t pa = ld_cg(parent + a), pb = ld_cg(parent + b);
    if (pa == pb) return;
    if (pa == a && pb == b) {  // two roots: larger under smaller
      const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
      const uint32_t old = atomicCAS(parent + hi, hi, lo);
      if (old == hi) return;
      a = lo;
      b = old;
      continue;
    }
    if (pa != a) {
      const uint32_t ga = ld_cg(parent + pa);
      if (ga != pa) parent[a] = ga;
      a = ga;
    }
    if (pb != b) {
      const uint32_t gb = ld_cg(parent + pb);
      if (gb != pb) parent[b] = gb;
      b = gb;
    }
  }
}

// Small device -> host read-backs (run header, counts, probe samples) are
// stored by a one-block kernel into mapped pinned memory instead of a
// cudaMemcpyAsync: a D2H copy would queue on the copy engine behind whatever
// bulk D2H another buffer has in flight (the host-buffer pipeline and the
// streaming path overlap exactly those), stalling this run until it drains.
__global__ void k_readback(const unsigned char* __restrict__ src, unsigned char* dst, uint32_t bytes) {
  for (uint32_t i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}
// host_mapped: memory from cudaHostAlloc(..., cudaHostAllocMapped)
inline cudaError_t readback_async(void* host_mapped, const void* dev, size_t bytes, cudaStream_t s) {
  void* dptr = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&dptr, host_mapped, 0);
  if (e != cudaSuccess) return e;
  k_readback<<<1, 256, 0, s>>>((const unsigned char*)dev, (unsigned char*)dptr, (uint32_t)bytes);
  return cudaGetLastError();
}

}  // namespace tpx
