// Decode of an encoded seed section back to the seed matrix, on device.
//
// Replaces CompactVector.decode_all (encoders.py:101-102, _unpack_fields
// :53-63), RiceVector.decode_all (encoders.py:232-235, scan_ones :157-162)
// and the two decode_matrix layouts (InterleavedSeeds :309-311,
// MonoSeeds :337-338). Used for structures loaded with Mphf.deserialize,
// whose query path needs the seed matrix (mphf.py:114-117).
//
// Rice highs: word popcounts -> per-column exclusive scan (chunked) ->
// every set bit writes its position at its rank -> high_r = pos_r -
// pos_{r-1} - 1.
#include <algorithm>
#include "common.cuh"
#include "phobic_internal.h"

namespace phb {

constexpr int DT = 256;
constexpr int DWPT = 16;            // highs words per thread
constexpr int DCH = DT * DWPT;      // highs words per chunk

struct DCol {
  int64_t kind, param, count, pay_byte, highs_byte, highs_nbits, pad0, pad1;
};

__device__ __forceinline__ uint64_t get_bits(const uint8_t* __restrict__ blob, uint64_t addr,
                                             int nbits) {
  if (nbits <= 0) return 0;
  // read 16 bytes covering [addr, addr + 64 + 7) bytewise-safe via aligned words
  const uint64_t byte = addr >> 3;
  const int sh = (int)(addr & 7);
  uint64_t lo = 0, hi = 0;
  const uint8_t* p = blob + byte;
  const int need = (sh + nbits + 7) >> 3;  // <= 9
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < need) lo |= (uint64_t)p[i] << (8 * i);
  if (need > 8) hi = p[8];
  uint64_t v = (lo >> sh) | (sh ? (hi << (64 - sh)) : 0ull);
  return nbits >= 64 ? v : (v & ((1ull << nbits) - 1));
}

__device__ __forceinline__ void store_val(uint64_t* seeds, int mono, int64_t c, int64_t t,
                                          int64_t nparts, uint32_t B, uint64_t v) {
  if (!mono) {
    seeds[c * nparts + t] = v;
  } else {
    int64_t j = t / B, i = t - j * B;
    seeds[i * nparts + j] = v;
  }
}

// Compact columns, and the low parts of Rice columns.
__global__ void k_decode_fields(const uint8_t* __restrict__ blob, const DCol* __restrict__ cols,
                                int64_t ncols, int64_t per_col, int64_t nparts, uint32_t B,
                                int mono, uint64_t* __restrict__ seeds) {
  const int64_t total = ncols * per_col;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / per_col, t = i - c * per_col;
    const DCol d = cols[c];
    if (t >= d.count) continue;
    const int w = (int)d.param;
    uint64_t v = w ? get_bits(blob, 8ull * d.pay_byte + (uint64_t)t * w, w) : 0ull;
    store_val(seeds, mono, c, t, nparts, B, v);
  }
}

__device__ __forceinline__ uint32_t highs_word(const uint8_t* blob, const DCol& d, int64_t w) {
  const int64_t nb = d.highs_nbits - 32 * w;
  if (nb <= 0) return 0;
  return (uint32_t)get_bits(blob, 8ull * d.highs_byte + 32ull * w, nb < 32 ? (int)nb : 32);
}

__global__ void __launch_bounds__(DT) k_highs_chunks(const uint8_t* __restrict__ blob,
                                                     const DCol* __restrict__ cols,
                                                     int64_t nch,
                                                     unsigned long long* __restrict__ csum) {
  __shared__ unsigned long long s;
  const int64_t c = blockIdx.x / nch, q = blockIdx.x - c * nch;
  const DCol d = cols[c];
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  unsigned long long acc = 0;
  if (d.kind == 1) {
    const int64_t nw = (d.highs_nbits + 31) / 32;
    for (int64_t w = q * DCH + threadIdx.x; w < min(nw, (q + 1) * (int64_t)DCH); w += DT)
      acc += __popc(highs_word(blob, d, w));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&s, acc);
  __syncthreads();
  if (threadIdx.x == 0) csum[blockIdx.x] = s;
}

__global__ void k_highs_scan(int64_t ncols, int64_t nch, unsigned long long* __restrict__ csum) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  unsigned long long run = 0;
  for (int64_t q = 0; q < nch; ++q) {
    unsigned long long v = csum[c * nch + q];
    csum[c * nch + q] = run;
    run += v;
  }
}

__global__ void __launch_bounds__(DT) k_highs_emit(const uint8_t* __restrict__ blob,
                                                   const DCol* __restrict__ cols, int64_t nch,
                                                   const unsigned long long* __restrict__ cpre,
                                                   int64_t per_col,
                                                   uint64_t* __restrict__ pos) {
  __shared__ unsigned long long sh[DT / 32];
  const int64_t c = blockIdx.x / nch, q = blockIdx.x - c * nch;
  const DCol d = cols[c];
  if (d.kind != 1) return;
  const int64_t nw = (d.highs_nbits + 31) / 32;
  const int64_t w0 = q * DCH + (int64_t)threadIdx.x * DWPT;
  uint32_t words[DWPT];
  unsigned long long local = 0;
#pragma unroll
  for (int e = 0; e < DWPT; ++e) {
    words[e] = (w0 + e < nw) ? highs_word(blob, d, w0 + e) : 0u;
    local += __popc(words[e]);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long v = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    unsigned long long x = lane < DT / 32 ? sh[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane < DT / 32) sh[lane] = x;
  }
  __syncthreads();
  unsigned long long rank = cpre[blockIdx.x] + (wid ? sh[wid - 1] : 0ull) + v - local;
#pragma unroll
  for (int e = 0; e < DWPT; ++e) {
    uint32_t x = words[e];
    while (x) {
      int bit = __ffs(x) - 1;
      x &= x - 1;
      if ((int64_t)rank < d.count) pos[c * per_col + rank] = 32ull * (w0 + e) + bit;
      ++rank;
    }
  }
}

__global__ void k_highs_apply(const DCol* __restrict__ cols, int64_t ncols, int64_t per_col,
                              const uint64_t* __restrict__ pos, int64_t nparts, uint32_t B,
                              int mono, uint64_t* __restrict__ seeds) {
  const int64_t total = ncols * per_col;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / per_col, t = i - c * per_col;
    const DCol d = cols[c];
    if (d.kind != 1 || t >= d.count) continue;
    const uint64_t p = pos[c * per_col + t];
    const uint64_t prev = t ? pos[c * per_col + t - 1] : ~0ull;  // -1
    const uint64_t high = p - prev - 1;
    const int b = (int)d.param;
    uint64_t low;
    if (!mono)
      low = seeds[c * nparts + t];
    else {
      int64_t j = t / B, ii = t - j * B;
      low = seeds[ii * nparts + j];
    }
    uint64_t v = b >= 64 ? low : ((high << b) | low);
    store_val(seeds, mono, c, t, nparts, B, v);
  }
}

int launch_decode(const uint8_t* blob, int64_t ncols, const int64_t* host_info, int64_t nparts,
                  uint32_t B, int mono, uint64_t* seeds, cudaStream_t st) {
  if (ncols <= 0) return 0;
  const int64_t per_col = mono ? nparts * (int64_t)B : nparts;
  int64_t max_words = 1;
  bool any_rice = false;
  for (int64_t c = 0; c < ncols; ++c) {
    const int64_t* ci = host_info + 8 * c;
    if (ci[0] == 1) {
      any_rice = true;
      int64_t nw = (ci[5] + 31) / 32;
      if (nw > max_words) max_words = nw;
    }
  }
  const int64_t nch = (max_words + DCH - 1) / DCH;
  DCol* dcols = nullptr;
  unsigned long long* csum = nullptr;
  uint64_t* pos = nullptr;
  PHB_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&dcols), sizeof(DCol) * ncols, st));
  PHB_CUDA_TRY(cudaMemcpyAsync(dcols, host_info, sizeof(DCol) * ncols, cudaMemcpyHostToDevice, st));
  const int64_t total = ncols * per_col;
  int g = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
  if (g < 1) g = 1;
  note_launch(), k_decode_fields<<<g, 256, 0, st>>>(blob, dcols, ncols, per_col, nparts, B, mono, seeds);
  PHB_CUDA_TRY(cudaGetLastError());
  if (any_rice) {
    PHB_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&csum), sizeof(unsigned long long) * ncols * nch, st));
    PHB_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&pos), sizeof(uint64_t) * ncols * per_col, st));
    note_launch(), k_highs_chunks<<<(unsigned)(ncols * nch), DT, 0, st>>>(blob, dcols, nch, csum);
    note_launch(), k_highs_scan<<<(unsigned)((ncols + 255) / 256), 256, 0, st>>>(ncols, nch, csum);
    note_launch(), k_highs_emit<<<(unsigned)(ncols * nch), DT, 0, st>>>(blob, dcols, nch, csum, per_col, pos);
    note_launch(), k_highs_apply<<<g, 256, 0, st>>>(dcols, ncols, per_col, pos, nparts, B, mono, seeds);
    PHB_CUDA_TRY(cudaGetLastError());
    PHB_CUDA_TRY(cudaFreeAsync(csum, st));
    PHB_CUDA_TRY(cudaFreeAsync(pos, st));
  }
  PHB_CUDA_TRY(cudaFreeAsync(dcols, st));
  return 0;
}

}  // namespace phb
