// K5/K6 encode: interleaved (and mono) Compact / Golomb-Rice seed encoding
// and the device-assembled serialized body.
//
// Replaces, in the reference:
//   InterleavedSeeds.build   encoders.py:291-299  (column i = seed of bucket
//                            i+1 from every partition, partition order)
//   MonoSeeds.build          encoders.py:322-327  (one column, row-major)
//   CompactVector.encode     encoders.py:83-87    (width = bitlen(max))
//   _pack_fields             encoders.py:35-50    (LSB-first fields)
//   rice_parameter           encoders.py:165-183  (exact argmin, ties low)
//   RiceVector.encode        encoders.py:195-222  (lows + unary highs)
//   Select.from_ones         encoders.py:121-123  (every 1024th one)
//   _encoder_block           encoders.py:245-255  (block byte layout)
//   serialize_seeds          encoders.py:353-355
//   pack_deltas              partitioning.py:131-142 (bias 2^(w-1), w bits)
//   Mphf.serialize body      mphf.py:156-175      (everything after the
//                            57-byte fixed header, before the checksum)
//
// Every output bit is placed with atomicOr into a zeroed, 4-byte aligned
// blob at its absolute bit address, so fields that straddle byte or block
// boundaries need no special casing. Rice unary positions come from a
// per-column chunked exclusive scan of (high + 1).
#include "common.cuh"
#include "phobic_internal.h"
#include "phobic_encode.h"
#include <algorithm>

namespace phb {

constexpr int ET = 256;      // threads per CTA
constexpr int EPT = 16;      // values per thread
constexpr int ECH = ET * EPT;  // values per chunk (4096)

__device__ __forceinline__ void put_bits(uint32_t* __restrict__ words, uint64_t addr, uint64_t v,
                                         int nbits) {
  if (nbits <= 0 || v == 0) return;
  const uint64_t w = addr >> 5;
  const int sh = (int)(addr & 31);
  const uint64_t x0 = v << sh;
  const uint64_t x1 = sh ? (v >> (64 - sh)) : 0ull;
  uint32_t p0 = (uint32_t)x0, p1 = (uint32_t)(x0 >> 32), p2 = (uint32_t)x1;
  if (p0) atomicOr(words + w, p0);
  if (p1) atomicOr(words + w + 1, p1);
  if (p2) atomicOr(words + w + 2, p2);
}

__device__ __forceinline__ int bitlen64(uint64_t v) { return v ? 64 - __clzll(v) : 0; }

struct Cols {
  const uint64_t* seeds;  // column-major [B][nparts]
  int64_t nparts;
  uint32_t B;
  int mono;
  int64_t t_off;          // global index of this shard's value 0 in every column
  __device__ __forceinline__ int64_t ncols() const { return mono ? 1 : B; }
  __device__ __forceinline__ int64_t count() const { return mono ? nparts * (int64_t)B : nparts; }
  // value t of column c in the reference's order
  __device__ __forceinline__ uint64_t at(int64_t c, int64_t t) const {
    if (!mono) return seeds[c * nparts + t];
    int64_t j = t / B, i = t - j * B;
    return seeds[i * nparts + j];
  }
};

// E1: per-column max and per-bit population counts (Rice cost vector).
// Compact columns (c < compact_prefix) need only the max (C2, IC-C:
// 0.22 -> 0.08 ms for the plan). (Warp-wide ballot + popc bit counts measured
// slower than the per-thread counters for Rice columns.)
__global__ void __launch_bounds__(ET) k_col_stats(Cols cols, int64_t nchunks_per_col,
                                                  unsigned long long* __restrict__ colstat,
                                                  int compact_prefix) {
  __shared__ unsigned long long s_bits[64];
  __shared__ unsigned long long s_max;
  const int64_t c = blockIdx.x / nchunks_per_col;
  const int64_t q = blockIdx.x - c * nchunks_per_col;
  if (threadIdx.x < 64) s_bits[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  const int64_t cnt = cols.count();
  const int64_t t0 = q * ECH;
  const int64_t t1 = min(t0 + (int64_t)ECH, cnt);
  const int lane = threadIdx.x & 31;
  uint64_t mx = 0;
  if (c < compact_prefix) {
    for (int64_t t = t0 + threadIdx.x; t < t1; t += ET)
      mx = max(mx, cols.mono ? cols.seeds[t] : cols.seeds[c * cols.nparts + t]);
  } else {
    uint32_t bits[64];
#pragma unroll
    for (int b = 0; b < 64; ++b) bits[b] = 0;
    for (int64_t t = t0 + threadIdx.x; t < t1; t += ET) {
      // mono stats are order-free: read storage linearly
      uint64_t v = cols.mono ? cols.seeds[t] : cols.seeds[c * cols.nparts + t];
      mx = max(mx, v);
#pragma unroll
      for (int b = 0; b < 64; ++b) bits[b] += (uint32_t)((v >> b) & 1ull);
    }
    // warp-reduce the bit counters, one shared atomic per warp and bit
#pragma unroll
    for (int b = 0; b < 64; ++b) {
      uint32_t x = bits[b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0 && x) atomicAdd(&s_bits[b], (unsigned long long)x);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) atomicMax(&s_max, (unsigned long long)mx);
  __syncthreads();
  unsigned long long* out = colstat + c * 65;
  if (threadIdx.x < 64 && s_bits[threadIdx.x]) atomicAdd(out + 1 + threadIdx.x, s_bits[threadIdx.x]);
  if (threadIdx.x == 0) atomicMax(out, s_max);
}

// Sum over values of (v >> b), from the bit population counts (exact mod 2^64,
// like the reference's uint64 sum).
__device__ __forceinline__ uint64_t shifted_sum(const unsigned long long* st, int b) {
  uint64_t s = 0;
  for (int p = b; p < 64; ++p) s += (uint64_t)st[1 + p] << (p - b);
  return s;
}

// E1b: status / trials reduction over the partitions, multi-CTA: trials
// summed into sum->trials_total, the first failing partition j kept as
// max(nparts - j) in sum->first_bad (0 = none; k_plan decodes it).
// sum->trials_total and sum->first_bad are zeroed before the launch.
__global__ void __launch_bounds__(256) k_status_reduce(const int64_t* __restrict__ part_trials,
                                                       const uint8_t* __restrict__ status,
                                                       int64_t nparts,
                                                       EncodeSummary* __restrict__ sum) {
  unsigned long long tr = 0, bad = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nparts;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (part_trials) tr += (unsigned long long)part_trials[j];
    if (status && status[j]) bad = max(bad, (unsigned long long)(nparts - j));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    tr += __shfl_xor_sync(0xffffffffu, tr, o);
    bad = max(bad, __shfl_xor_sync(0xffffffffu, bad, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (tr) atomicAdd(reinterpret_cast<unsigned long long*>(&sum->trials_total), tr);
    if (bad) atomicMax(reinterpret_cast<unsigned long long*>(&sum->first_bad), bad);
  }
}

// E2: per-column parameters, block sizes and byte offsets; seed-section
// geometry. One CTA (the partition-wide reduction is k_status_reduce).
__global__ void __launch_bounds__(1024) k_plan(EncodeArgs a, const unsigned long long* colstat,
                                               ColInfo* __restrict__ info,
                                               EncodeSummary* __restrict__ sum) {
  __shared__ unsigned long long sh[32];
  const int ncols = a.mono ? 1 : (int)a.bcount;
  const int64_t cnt = a.count_global ? a.count_global
                                     : (a.mono ? a.nparts * (int64_t)a.bcount : a.nparts);

  // delta width (partitioning.py:125-128): bitlen(max |delta|) + 1
  const int w = bitlen64((uint64_t)a.layout_stats[0]) + 1;
  const uint64_t delta_bytes = ((uint64_t)(a.nparts_global + 1) * w + 7) / 8;
  const uint64_t sec0 = HEADER_FIXED + 1 + delta_bytes + 4;  // u32 num_encoders at sec0

  // per-column block sizes; each thread a contiguous run of columns
  const int per = (ncols + blockDim.x - 1) / blockDim.x;
  const int c0 = threadIdx.x * per, c1 = min(c0 + per, ncols);
  uint64_t local = 0;
  for (int c = c0; c < c1; ++c) {
    const unsigned long long* st = colstat + (int64_t)c * 65;
    const uint64_t mx = st[0];
    ColInfo ci;
    ci.count = (uint64_t)cnt;
    const bool compact = c < a.compact_prefix;
    if (compact) {
      ci.kind = 0;
      ci.param = (uint8_t)bitlen64(mx);
      ci.highs_nbits = 0;
      ci.nsamples = 0;
      ci.block_bytes = 10 + (ci.count * ci.param + 7) / 8;
    } else {
      // rice_parameter: b in [0, min(64, bitlen(max) + 1)], ties -> smaller b
      int top = bitlen64(mx);
      int bmax = min(64, top + 1);
      int best_b = 0;
      unsigned __int128 best = 0;
      for (int b = 0; b <= bmax; ++b) {
        uint64_t ssum = b >= 64 ? 0ull : shifted_sum(st, b);
        unsigned __int128 cost = (unsigned __int128)ci.count * (b + 1) + ssum;
        if (b == 0 || cost < best) best = cost, best_b = b;
      }
      if (cnt == 0) best_b = 0;
      ci.kind = 1;
      ci.param = (uint8_t)best_b;
      uint64_t hsum = best_b >= 64 ? 0ull : shifted_sum(st, best_b);
      ci.highs_nbits = cnt ? hsum + ci.count : 0;
      ci.nsamples = (uint32_t)((ci.count + 1023) / 1024);
      ci.block_bytes = 10 + 12 + 8ull * ci.nsamples + (ci.count * best_b + 7) / 8 +
                       (ci.highs_nbits + 7) / 8;
    }
    info[c] = ci;
    local += ci.block_bytes;
  }
  __syncthreads();
  // exclusive scan of block sizes -> byte offsets
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t v = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    uint64_t x = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    sh[lane] = x;
  }
  __syncthreads();
  uint64_t run = (wid ? sh[wid - 1] : 0) + v - local;
  for (int c = c0; c < c1; ++c) {
    ColInfo& ci = info[c];
    ci.block_off = sec0 + 4 + run;
    const uint64_t body = ci.block_off + 10;
    if (ci.kind == 0) {
      ci.pay_bit = 8 * body;
      ci.samples_byte = 0;
      ci.highs_bit = 0;
    } else {
      ci.samples_byte = body + 12;
      ci.pay_bit = 8 * (ci.samples_byte + 8ull * ci.nsamples);
      ci.highs_bit = ci.pay_bit + 8 * ((ci.count * ci.param + 7) / 8);
    }
    run += ci.block_bytes;
  }
  if (threadIdx.x == blockDim.x - 1) {
    sum->total_bytes = sec0 + 4 + run;  // body length without checksum
    sum->delta_width = w;
    sum->seed_section = sec0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t v = sum->first_bad;  // max(nparts - j) from k_status_reduce, 0 = none
    const int64_t bad = v ? a.nparts - v : -1;
    sum->first_bad = bad;
    sum->bad_code = (bad < 0 || !a.status) ? 0 : a.status[bad];
    sum->ncols = ncols;
  }
}

// R1: per-chunk sums of (high + 1) for Rice columns.
__global__ void __launch_bounds__(ET) k_rice_chunks(Cols cols, int64_t nchunks_per_col,
                                                    const ColInfo* __restrict__ info,
                                                    unsigned long long* __restrict__ chunk_sum) {
  __shared__ unsigned long long s;
  const int64_t c = blockIdx.x / nchunks_per_col;
  const int64_t q = blockIdx.x - c * nchunks_per_col;
  const ColInfo ci = info[c];
  if (ci.kind != 1) return;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  const int64_t t0 = q * ECH, t1 = min(t0 + (int64_t)ECH, cols.count());
  unsigned long long acc = 0;
  const int b = ci.param;
  for (int64_t t = t0 + threadIdx.x; t < t1; t += ET) {
    uint64_t v = cols.at(c, t);
    acc += (b >= 64 ? 0ull : (v >> b)) + 1;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&s, acc);
  __syncthreads();
  if (threadIdx.x == 0) chunk_sum[blockIdx.x] = s;
}

// R2: exclusive scan of chunk sums inside each column (thread per column).
__global__ void k_rice_chunk_scan(int64_t ncols, int64_t nchunks_per_col,
                                  unsigned long long* __restrict__ chunk_sum,
                                  unsigned long long* __restrict__ col_total) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  unsigned long long run = 0;
  for (int64_t q = 0; q < nchunks_per_col; ++q) {
    unsigned long long v = chunk_sum[c * nchunks_per_col + q];
    chunk_sum[c * nchunks_per_col + q] = run;
    run += v;
  }
  if (col_total) col_total[c] = run;  // this shard's unary bits (sharded encode)
}

// E3: headers, deltas and every payload bit.
__global__ void k_headers(EncodeArgs a, const ColInfo* __restrict__ info,
                          const EncodeSummary* __restrict__ sum, uint32_t* __restrict__ blob) {
  const int64_t ncols = sum->ncols;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int w = sum->delta_width;
  if (tid == 0) {
    put_bits(blob, 8ull * HEADER_FIXED, (uint64_t)w, 8);
    put_bits(blob, 8ull * (sum->seed_section - 4), (uint64_t)a.bcount, 32);
    put_bits(blob, 8ull * sum->seed_section, (uint64_t)ncols, 32);
  }
  if (tid < ncols) {
    const ColInfo ci = info[tid];
    const uint64_t at = 8ull * ci.block_off;
    put_bits(blob, at, ci.kind, 8);
    put_bits(blob, at + 8, ci.param, 8);
    put_bits(blob, at + 16, ci.count, 64);
    if (ci.kind == 1) {
      put_bits(blob, at + 80, ci.highs_nbits, 64);
      put_bits(blob, at + 144, ci.nsamples, 32);
    }
  }
}

__global__ void k_deltas(const int64_t* __restrict__ deltas, int64_t count,
                         const EncodeSummary* __restrict__ sum, uint32_t* __restrict__ blob) {
  const int w = sum->delta_width;
  const uint64_t base = 8ull * (HEADER_FIXED + 1);
  const uint64_t bias = 1ull << (w - 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t v = (uint64_t)deltas[i] + bias;
    if (w < 64) v &= (1ull << w) - 1;
    put_bits(blob, base + (uint64_t)i * w, v, w);
  }
}

__global__ void __launch_bounds__(ET) k_payload(Cols cols, int64_t nchunks_per_col,
                                                const ColInfo* __restrict__ info,
                                                const unsigned long long* __restrict__ chunk_pre,
                                                const unsigned long long* __restrict__ rice_base,
                                                uint32_t* __restrict__ blob) {
  __shared__ unsigned long long sh[ET / 32];
  const int64_t c = blockIdx.x / nchunks_per_col;
  const int64_t q = blockIdx.x - c * nchunks_per_col;
  const ColInfo ci = info[c];
  const int64_t t0 = q * ECH;
  const int64_t t1 = min(t0 + (int64_t)ECH, cols.count());
  if (t0 >= t1) return;
  const int b = ci.param;
  const uint64_t toff = (uint64_t)cols.t_off;  // global index = local + toff
  if (ci.kind == 0) {
    for (int64_t t = t0 + threadIdx.x; t < t1; t += ET)
      put_bits(blob, ci.pay_bit + ((uint64_t)t + toff) * b, cols.at(c, t), b);
    return;
  }
  // Rice: thread owns EPT consecutive values so the unary scan is local
  const uint64_t lmask = b >= 64 ? ~0ull : ((1ull << b) - 1);
  const int64_t mine0 = t0 + (int64_t)threadIdx.x * EPT;
  uint64_t vals[EPT];
  unsigned long long local = 0;
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    int64_t t = mine0 + e;
    vals[e] = t < t1 ? cols.at(c, t) : 0ull;
    if (t < t1) local += (b >= 64 ? 0ull : (vals[e] >> b)) + 1;
  }
  // block exclusive scan of local sums
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
    unsigned long long x = lane < ET / 32 ? sh[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane < ET / 32) sh[lane] = x;
  }
  __syncthreads();
  unsigned long long run = (rice_base ? rice_base[c] : 0ull) + chunk_pre[blockIdx.x] +
                           (wid ? sh[wid - 1] : 0ull) + v - local;
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    int64_t t = mine0 + e;
    if (t < t1) {
      const uint64_t tg = (uint64_t)t + toff;
      const uint64_t hv = b >= 64 ? 0ull : (vals[e] >> b);
      const uint64_t one = run + hv;  // position of this value's terminating 1
      put_bits(blob, ci.highs_bit + one, 1ull, 1);
      if (b > 0) put_bits(blob, ci.pay_bit + tg * b, vals[e] & lmask, b);
      if ((tg & 1023) == 0) put_bits(blob, 8ull * ci.samples_byte + 64ull * (tg >> 10), one, 64);
      run += hv + 1;
    }
  }
}

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

size_t encode_workspace_bytes(int64_t nparts, uint32_t bcount, int mono) {
  int64_t ncols = mono ? 1 : bcount;
  int64_t cnt = mono ? nparts * (int64_t)bcount : nparts;
  int64_t nch = cdiv(cnt, ECH);
  if (nch < 1) nch = 1;
  size_t bytes = 0;
  bytes += (size_t)ncols * 65 * 8;        // colstat
  bytes += (size_t)ncols * sizeof(ColInfo);
  bytes += (size_t)ncols * nch * 8;       // chunk sums
  bytes += sizeof(EncodeSummary) + 256;
  return bytes + 1024;
}

static inline char* align_up(char* p, size_t a) {
  return (char*)(((uintptr_t)p + a - 1) & ~(uintptr_t)(a - 1));
}

struct WsLayout {
  unsigned long long* colstat;
  ColInfo* info;
  unsigned long long* chunks;
  EncodeSummary* sum;
};

static WsLayout carve(void* ws, int64_t ncols, int64_t nch) {
  WsLayout L;
  char* p = align_up((char*)ws, 256);
  L.colstat = (unsigned long long*)p;
  p = align_up(p + (size_t)ncols * 65 * 8, 256);
  L.info = (ColInfo*)p;
  p = align_up(p + (size_t)ncols * sizeof(ColInfo), 256);
  L.chunks = (unsigned long long*)p;
  p = align_up(p + (size_t)ncols * nch * 8, 256);
  L.sum = (EncodeSummary*)p;
  return L;
}

int launch_encode_plan(const EncodeArgs& a, void* ws, EncodeSummary* host_sum, cudaStream_t st) {
  const int64_t ncols = a.mono ? 1 : a.bcount;
  const int64_t cnt = a.mono ? a.nparts * (int64_t)a.bcount : a.nparts;
  int64_t nch = cdiv(cnt, ECH);
  if (nch < 1) nch = 1;
  WsLayout L = carve(ws, ncols, nch);
  Cols cols{a.seeds, a.nparts, a.bcount, a.mono, a.row0 * (a.mono ? (int64_t)a.bcount : 1)};
  if (a.colstat_in) {  // sharded: statistics already reduced over all shards
    PHB_CUDA_TRY(cudaMemcpyAsync(L.colstat, a.colstat_in, (size_t)ncols * 65 * 8,
                                 cudaMemcpyDeviceToDevice, st));
  } else {
    PHB_CUDA_TRY(cudaMemsetAsync(L.colstat, 0, (size_t)ncols * 65 * 8, st));
    note_launch(), k_col_stats<<<(unsigned)(ncols * nch), ET, 0, st>>>(cols, nch, L.colstat,
                                                                        a.compact_prefix);
    PHB_CUDA_TRY(cudaGetLastError());
  }
  PHB_CUDA_TRY(cudaMemsetAsync(L.sum, 0, sizeof(EncodeSummary), st));
  if (a.nparts > 0 && (a.part_trials || a.status)) {
    const int64_t g = std::min<int64_t>(cdiv(a.nparts, 256), (int64_t)num_sms() * 4);
    note_launch(), k_status_reduce<<<(unsigned)g, 256, 0, st>>>(a.part_trials, a.status,
                                                                a.nparts, L.sum);
    PHB_CUDA_TRY(cudaGetLastError());
  }
  note_launch(), k_plan<<<1, 1024, 0, st>>>(a, L.colstat, L.info, L.sum);
  PHB_CUDA_TRY(cudaGetLastError());
  note_launch(), k_rice_chunks<<<(unsigned)(ncols * nch), ET, 0, st>>>(cols, nch, L.info, L.chunks);
  PHB_CUDA_TRY(cudaGetLastError());
  note_launch(), k_rice_chunk_scan<<<(unsigned)cdiv(ncols, 256), 256, 0, st>>>(ncols, nch, L.chunks,
                                                               a.rice_totals_out);
  PHB_CUDA_TRY(cudaGetLastError());
  if (host_sum) {
    PHB_CUDA_TRY(cudaMemcpyAsync(host_sum, L.sum, sizeof(EncodeSummary), cudaMemcpyDeviceToHost,
                                 st));
    PHB_CUDA_TRY(cudaStreamSynchronize(st));
  }
  return 0;
}

int launch_encode_write(const EncodeArgs& a, void* ws, uint8_t* blob, size_t blob_bytes,
                        cudaStream_t st) {
  const int64_t ncols = a.mono ? 1 : a.bcount;
  const int64_t cnt = a.mono ? a.nparts * (int64_t)a.bcount : a.nparts;
  int64_t nch = cdiv(cnt, ECH);
  if (nch < 1) nch = 1;
  if (((uintptr_t)blob & 3) != 0) return 1003;
  WsLayout L = carve(ws, ncols, nch);
  PHB_CUDA_TRY(cudaMemsetAsync(blob, 0, blob_bytes, st));
  uint32_t* words = reinterpret_cast<uint32_t*>(blob);
  if (a.write_headers) {
    note_launch(), k_headers<<<(unsigned)cdiv(ncols, 256), 256, 0, st>>>(a, L.info, L.sum, words);
    PHB_CUDA_TRY(cudaGetLastError());
  }
  int64_t nd = a.nparts_global + 1;
  if (a.deltas && a.write_headers) {
    note_launch(), k_deltas<<<(unsigned)std::min<int64_t>(cdiv(nd, 256), 4096), 256, 0, st>>>(a.deltas, nd, L.sum,
                                                                        words);
    PHB_CUDA_TRY(cudaGetLastError());
  }
  Cols cols{a.seeds, a.nparts, a.bcount, a.mono, a.row0 * (a.mono ? (int64_t)a.bcount : 1)};
  note_launch(), k_payload<<<(unsigned)(ncols * nch), ET, 0, st>>>(cols, nch, L.info, L.chunks, a.rice_base,
                                                    words);
  return (int)cudaGetLastError();
}

int launch_encode_stats(const EncodeArgs& a, void* ws, unsigned long long* colstat_out,
                        cudaStream_t st) {
  const int64_t ncols = a.mono ? 1 : a.bcount;
  const int64_t cnt = a.mono ? a.nparts * (int64_t)a.bcount : a.nparts;
  int64_t nch = cdiv(cnt, ECH);
  if (nch < 1) nch = 1;
  (void)ws;
  PHB_CUDA_TRY(cudaMemsetAsync(colstat_out, 0, (size_t)ncols * 65 * 8, st));
  Cols cols{a.seeds, a.nparts, a.bcount, a.mono, 0};
  if (cnt > 0)
    note_launch(), k_col_stats<<<(unsigned)(ncols * nch), ET, 0, st>>>(cols, nch, colstat_out,
                                                                        a.compact_prefix);
  return (int)cudaGetLastError();
}

}  // namespace phb
