// K2 layout: per-partition counts -> key offsets, offset deltas and the
// two layout statistics the later stages size themselves by.
//
// Replaces partitioning.partition_arrays' cumsum / expected_offset loop
// (partitioning.py:96-108) and delta_width (partitioning.py:125-128).
//
// Multi-CTA single-pass scan with decoupled look-back: each CTA takes the
// next tile of LT * PER partitions (tile ids from an atomic counter, so a
// tile's predecessors are already running), publishes its aggregate, then
// sums predecessor aggregates until it meets an inclusive prefix. The
// expected offsets round(j n / nparts) walk incrementally within a thread's
// run (one 64-bit division per run, then quotient/remainder steps) instead
// of a 128-bit division per partition.
#include <algorithm>
#include "common.cuh"
#include "phobic_internal.h"

namespace phb {

constexpr int LT = 1024;
constexpr int PER = 4;  // partitions per thread per tile

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

// tile status word: bits 62-63 flag (1 aggregate, 2 inclusive prefix), value below.
// It is stored over the tile's first two counts (consumed by then): two
// counts < 2^30 read as a word with flag bits 0, i.e. "not published".
constexpr uint64_t ST_AGG = 1ull << 62, ST_INC = 2ull << 62, ST_VAL = (1ull << 62) - 1;

__global__ void __launch_bounds__(LT) k_layout(uint32_t* __restrict__ counts, int64_t nparts,
                                               int64_t key_base, int64_t part_base,
                                               int64_t global_n, int64_t global_nparts,
                                               int64_t* __restrict__ key_off,
                                               int64_t* __restrict__ deltas,
                                               unsigned long long* __restrict__ stats) {
  __shared__ uint64_t sh[32];
  __shared__ uint64_t s_prefix;
  __shared__ unsigned long long s_tile;
  // tile ids in arrival order (deltas[nparts] is the counter until the
  // owner of j = nparts, in the last tile, overwrites it)
  auto* ctr = reinterpret_cast<unsigned long long*>(deltas + nparts);
  auto* tstat = reinterpret_cast<unsigned long long*>(counts);  // word t at counts[t * LT * PER]
  if (threadIdx.x == 0) s_tile = atomicAdd(ctr, 1ull);
  __syncthreads();
  const int64_t tile = (int64_t)s_tile;
  const int64_t tsz = (int64_t)(LT * PER);
  const int64_t a = tile * tsz + (int64_t)threadIdx.x * PER;
  const int64_t b = min(a + PER, nparts);
  uint32_t c[PER];
  uint64_t local = 0;
  uint32_t maxc = 0;
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    c[e] = a + e < b ? counts[a + e] : 0u;
    local += c[e];
    maxc = max(maxc, c[e]);
  }
  const uint64_t incl = block_incl_scan(local, sh);  // syncs: every count of the tile is read
  // ---- decoupled look-back over the tile aggregates
  if (threadIdx.x == LT - 1) {
    const uint64_t agg = incl;  // the tile's total
    unsigned long long* const mine = tstat + (tile * tsz) / 2;
    if (tile == 0) s_prefix = 0;
    if (tile * tsz + 1 < nparts)  // the tile owns two count slots for its word
      atomicExch(mine, (tile == 0 ? ST_INC : ST_AGG) | agg);
    if (tile > 0) {
      uint64_t excl = 0;
      int64_t t = tile - 1;
      for (;;) {
        const uint64_t w = atomicAdd(tstat + (t * tsz) / 2, 0ull);  // L2-coherent read
        if (w & ST_INC) {
          excl += w & ST_VAL;
          break;
        }
        if (w & ST_AGG) {
          excl += w & ST_VAL;
          --t;
        }  // else: predecessor not published yet, spin
      }
      if (tile * tsz + 1 < nparts) atomicExch(mine, ST_INC | (excl + agg));
      s_prefix = excl;
    }
  }
  __syncthreads();
  uint64_t run = s_prefix + incl - local;
  // ---- offsets, deltas: expected(j) = round-half-up(j n / nparts)
  //      = floor((2 j n + nparts) / (2 nparts)), walked incrementally
  uint64_t maxd = 0;
  const bool owns_end = a <= nparts && nparts < a + PER;  // writes j = nparts
  const int64_t last = owns_end ? nparts : b - 1;
  if (a <= last) {
    const uint64_t D = 2ull * (uint64_t)global_nparts;
    const uint64_t step = 2ull * (uint64_t)global_n;
    const uint64_t sq = step / D, sr = step % D;
    const uint64_t num0 = 2ull * (uint64_t)(part_base + a) * (uint64_t)global_n + (uint64_t)global_nparts;
    uint64_t q = num0 / D, r = num0 % D;
    for (int64_t j = a; j <= last; ++j) {
      const int64_t off = (int64_t)run;
      key_off[j] = off;
      const int64_t d = (key_base + off) - (int64_t)q;
      deltas[j] = d;
      maxd = max(maxd, (uint64_t)(d < 0 ? -d : d));
      if (j < b) run += c[j - a];
      q += sq;
      r += sr;
      if (r >= D) r -= D, ++q;
    }
  }
  // block maxima, then one atomic per warp
  for (int o = 16; o > 0; o >>= 1) {
    maxd = max(maxd, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)maxd, o));
    maxc = max(maxc, __shfl_xor_sync(0xffffffffu, maxc, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(stats, (unsigned long long)maxd);
    atomicMax(stats + 1, (unsigned long long)maxc);
  }
}

size_t layout_temp_bytes(int64_t) { return 0; }

int launch_layout(uint32_t* counts, int64_t nparts, int64_t key_base, int64_t part_base,
                  int64_t global_n, int64_t global_nparts, int64_t* key_off, int64_t* deltas,
                  int64_t* stats, void*, size_t, cudaStream_t st) {
  if (nparts < 1) return 1003;  // PHB_E_ARGS
  if (reinterpret_cast<uintptr_t>(counts) & 7) return 1003;  // tile words live over counts
  // tiles cover the nparts + 1 offsets; no scratch: the tile counter is
  // deltas[nparts], the tile states overwrite the tiles' first counts
  const int64_t tiles = nparts / (LT * PER) + 1;
  PHB_CUDA_TRY(cudaMemsetAsync(stats, 0, 2 * sizeof(int64_t), st));
  PHB_CUDA_TRY(cudaMemsetAsync(deltas + nparts, 0, sizeof(int64_t), st));
  note_launch(), k_layout<<<(unsigned)tiles, LT, 0, st>>>(
      counts, nparts, key_base, part_base, global_n, global_nparts,
      key_off, deltas, reinterpret_cast<unsigned long long*>(stats));
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
  PHB_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&scratch), 2 * cells * sizeof(int64_t), st));
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
