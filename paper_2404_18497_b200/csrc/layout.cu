// K2 layout: per-partition counts -> key offsets, offset deltas and the
// two layout statistics the later stages size themselves by.
//
// Replaces partitioning.partition_arrays' cumsum / expected_offset loop
// (partitioning.py:96-108) and delta_width (partitioning.py:125-128).
// nparts is at most ~400k (n = 1e9, P = 2500): one persistent CTA scans it
// in a few microseconds, so no multi-pass device scan is needed.
#include <algorithm>
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
  note_launch(), k_layout<<<1, LT, 0, st>>>(counts, nparts, key_base, part_base, global_n, global_nparts,
                             key_off, deltas, stats);
  return (int)cudaGetLastError();
}

}  // namespace phb

// ---- multi-GPU regroup (distributed.py step 5) ------------------------
// The destination rank receives G chunks (one per source rank), each holding
// the records of its owned partitions [0, np) grouped by partition, with
// C[s][j] records of partition j from source s. Merge them into one
// partition-grouped array: partition j occupies [off[j], off[j+1]) with the
// sources' records in rank order (the order inside a partition is
// irrelevant to the result, SURVEY.md §0 finding 2; rank order keeps the
// merge deterministic).
namespace phb {

// One CTA: row scans (source-local offsets), column prefix sums and the
// partition offsets. G * np is at most a few hundred thousand.
__global__ void __launch_bounds__(LT) k_regroup_plan(const int32_t* __restrict__ C, int64_t G,
                                                     int64_t np, int64_t* __restrict__ srcoff,
                                                     int64_t* __restrict__ dstoff,
                                                     int64_t* __restrict__ key_off) {
  __shared__ uint64_t sh[32];
  // partition totals -> key_off (exclusive scan over j)
  const int64_t per = (np + LT - 1) / LT;
  const int64_t a = threadIdx.x * per, b = min(a + per, np);
  uint64_t local = 0;
  for (int64_t j = a; j < b; ++j)
    for (int64_t s = 0; s < G; ++s) local += (uint64_t)C[s * np + j];
  uint64_t incl = block_incl_scan(local, sh);
  uint64_t run = incl - local;
  for (int64_t j = a; j < b; ++j) {
    key_off[j] = (int64_t)run;
    uint64_t col = run;
    for (int64_t s = 0; s < G; ++s) {
      dstoff[s * np + j] = (int64_t)col;
      col += (uint64_t)C[s * np + j];
    }
    run = col;
  }
  if (b == np && a < b) key_off[np] = (int64_t)run;
  if (np == 0 && threadIdx.x == 0) key_off[0] = 0;
  // source rows: srcoff[s][j] = base[s] + sum_{j' < j} C[s][j']
  uint64_t base = 0;
  for (int64_t s = 0; s < G; ++s) {
    uint64_t loc = 0;
    for (int64_t j = a; j < b; ++j) loc += (uint64_t)C[s * np + j];
    uint64_t inc = block_incl_scan(loc, sh);
    uint64_t r = base + inc - loc;
    for (int64_t j = a; j < b; ++j) {
      srcoff[s * np + j] = (int64_t)r;
      r += (uint64_t)C[s * np + j];
    }
    // row total from the last thread's inclusive value
    __shared__ uint64_t tot;
    if (threadIdx.x == LT - 1) tot = inc;
    __syncthreads();
    base += tot;
    __syncthreads();
  }
}

// One warp per partition: copy each source's segment into place.
__global__ void __launch_bounds__(256) k_regroup_copy(const uint64_t* __restrict__ lo_in,
                                                      const uint16_t* __restrict__ aux_in,
                                                      const int32_t* __restrict__ C, int64_t G,
                                                      int64_t np,
                                                      const int64_t* __restrict__ srcoff,
                                                      const int64_t* __restrict__ dstoff,
                                                      uint64_t* __restrict__ lo_out,
                                                      uint16_t* __restrict__ aux_out) {
  const int lane = threadIdx.x & 31;
  for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < np;
       j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    for (int64_t s = 0; s < G; ++s) {
      const int64_t c = C[s * np + j], so = srcoff[s * np + j], dst_o = dstoff[s * np + j];
      for (int64_t t = lane; t < c; t += 32) {
        lo_out[dst_o + t] = lo_in[so + t];
        aux_out[dst_o + t] = aux_in[so + t];
      }
    }
  }
}

int launch_regroup(const uint64_t* lo_in, const uint16_t* aux_in, const int32_t* C, int64_t G,
                   int64_t np, uint64_t* lo_out, uint16_t* aux_out, int64_t* key_off,
                   cudaStream_t st) {
  if (G < 1 || np < 0) return 1003;
  int64_t* scratch = nullptr;
  const size_t cells = (size_t)(G * np > 0 ? G * np : 1);
  PHB_CUDA_TRY(cudaMallocAsync(&scratch, 2 * cells * sizeof(int64_t), st));
  note_launch(), k_regroup_plan<<<1, LT, 0, st>>>(C, G, np, scratch, scratch + cells, key_off);
  PHB_CUDA_TRY(cudaGetLastError());
  if (np > 0) {
    int64_t warps = np;
    int grid = (int)std::min<int64_t>((warps * 32 + 255) / 256, (int64_t)num_sms() * 16);
    note_launch(), k_regroup_copy<<<grid, 256, 0, st>>>(lo_in, aux_in, C, G, np, scratch, scratch + cells,
                                         lo_out, aux_out);
    PHB_CUDA_TRY(cudaGetLastError());
  }
  PHB_CUDA_TRY(cudaFreeAsync(scratch, st));
  return 0;
}

}  // namespace phb
