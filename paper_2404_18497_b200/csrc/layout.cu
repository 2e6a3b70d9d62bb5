// K2 layout: per-partition counts -> key offsets, offset deltas and the
// two layout statistics the later stages size themselves by.
//
// Replaces partitioning.partition_arrays' cumsum / expected_offset loop
// (partitioning.py:96-108) and delta_width (partitioning.py:125-128).
// nparts is at most ~400k (n = 1e9, P = 2500): one persistent CTA scans it
// in a few microseconds, so no multi-pass device scan is needed.
#include "common.cuh"
#include "phobic_internal.h"

namespace phb {

constexpr int LT = 1024;

__device__ __forceinline__ uint64_t block_incl_scan(uint64_t v, uint64_t* sh) {
  // Hillis-Steele over a warp, then over the 32 warp totals
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    uint64_t w = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    sh[lane] = w;
  }
  __syncthreads();
  uint64_t add = wid ? sh[wid - 1] : 0;
  __syncthreads();
  return v + add;
}

__global__ void __launch_bounds__(LT) k_layout(const uint32_t* __restrict__ counts, int64_t nparts,
                                               int64_t key_base, int64_t part_base,
                                               int64_t global_n, int64_t global_nparts,
                                               int64_t* __restrict__ key_off,
                                               int64_t* __restrict__ deltas,
                                               int64_t* __restrict__ stats) {
  __shared__ uint64_t sh[32];
  __shared__ unsigned long long s_maxd, s_maxc;
  if (threadIdx.x == 0) s_maxd = 0, s_maxc = 0;
  __syncthreads();
  // each thread owns a contiguous run of partitions
  const int64_t per = (nparts + LT - 1) / LT;
  const int64_t a = threadIdx.x * per;
  const int64_t b = min(a + per, nparts);
  uint64_t local = 0;
  uint32_t maxc = 0;
  for (int64_t j = a; j < b; ++j) {
    local += counts[j];
    maxc = max(maxc, counts[j]);
  }
  uint64_t incl = block_incl_scan(local, sh);
  uint64_t run = incl - local;
  uint64_t maxd = 0;
  for (int64_t j = a; j <= b && j <= nparts; ++j) {
    if (j == b && b != nparts) break;  // boundary j belongs to the next thread
    int64_t off = (int64_t)run;
    key_off[j] = off;
    int64_t d = (key_base + off) - expected_offset(part_base + j, global_n, global_nparts);
    deltas[j] = d;
    uint64_t ad = d < 0 ? (uint64_t)(-d) : (uint64_t)d;
    maxd = max(maxd, ad);
    if (j < b) run += counts[j];
  }
  if (a >= b && threadIdx.x == LT - 1 && nparts == 0) {
    key_off[0] = 0;
  }
  atomicMax(&s_maxd, (unsigned long long)maxd);
  atomicMax(&s_maxc, (unsigned long long)maxc);
  __syncthreads();
  if (threadIdx.x == 0) {
    stats[0] = (int64_t)s_maxd;
    stats[1] = (int64_t)s_maxc;
  }
}

size_t layout_temp_bytes(int64_t) { return 0; }

int launch_layout(const uint32_t* counts, int64_t nparts, int64_t key_base, int64_t part_base,
                  int64_t global_n, int64_t global_nparts, int64_t* key_off, int64_t* deltas,
                  int64_t* stats, void*, size_t, cudaStream_t st) {
  if (nparts < 1) return 1003;  // PHB_E_ARGS
  k_layout<<<1, LT, 0, st>>>(counts, nparts, key_base, part_base, global_n, global_nparts,
                             key_off, deltas, stats);
  return (int)cudaGetLastError();
}

}  // namespace phb
