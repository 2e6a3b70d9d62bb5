// K1 hash_count / K3 scatter_group: the key-side passes of the build.
//
// Replaces, in the reference:
//   murmur3_many            _kernels.py:89-146
//   partition_index_many    partitioning.py:73-78
//   bincount (sizes)        partitioning.py:96
//   np.lexsort + gathers    partitioning.py:93-95  (only the grouping matters:
//                           results are invariant to key order inside a
//                           partition, SURVEY.md §0 finding 2)
//   _bucket_of per key      _kernels.py:252-255    (moved here: the bucket id
//                           travels with the low word)
//
// Both passes are HBM-bound streaming kernels: one thread per key, grid
// sized in multiples of the SM count, coalesced 8-byte key loads.
#include <algorithm>

#include "common.cuh"
#include "phobic_internal.h"

namespace phb {

struct U64Keys {
  const uint64_t* __restrict__ keys;
  __device__ __forceinline__ Hash128 hash(int64_t i, uint64_t seed) const {
    return murmur3_u64(__ldg(keys + i), seed);
  }
};

struct ByteKeys {
  const uint8_t* __restrict__ buf;
  const int64_t* __restrict__ offsets;
  __device__ __forceinline__ Hash128 hash(int64_t i, uint64_t seed) const {
    int64_t a = __ldg(offsets + i), b = __ldg(offsets + i + 1);
    return murmur3_bytes(buf + a, b - a, seed);
  }
};

template <class K>
__global__ void __launch_bounds__(256) k_murmur(K keys, int64_t n, uint64_t seed,
                                                uint64_t* __restrict__ hi,
                                                uint64_t* __restrict__ lo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    Hash128 h = keys.hash(i, seed);
    hi[i] = h.hi;
    lo[i] = h.lo;
  }
}

// K1: per-partition key counts. Small partition counts use a shared-memory
// histogram per CTA (contention on few L2 lines otherwise); large ones go
// straight to L2 atomics spread over nparts addresses.
// store != NULL (byte keys): the 128-bit hashes are kept, (hi, lo) per key,
// so that K3 (k_scatter_hashed) does not hash the key bytes a second time.
template <class K, bool SMEM>
__global__ void __launch_bounds__(256) k_hash_count(K keys, int64_t n, uint64_t seed,
                                                    uint64_t nparts,
                                                    uint32_t* __restrict__ counts,
                                                    ulonglong2* __restrict__ store) {
  extern __shared__ uint32_t sh_hist[];
  if (SMEM) {
    for (uint32_t t = threadIdx.x; t < nparts; t += blockDim.x) sh_hist[t] = 0;
    __syncthreads();
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    Hash128 h = keys.hash(i, seed);
    if (store) store[i] = make_ulonglong2(h.hi, h.lo);
    uint32_t j = (uint32_t)mulhi(h.hi, nparts);
    if (SMEM)
      atomicAdd(sh_hist + j, 1u);
    else
      atomicAdd(counts + j, 1u);
  }
  if (SMEM) {
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < nparts; t += blockDim.x)
      if (sh_hist[t]) atomicAdd(counts + t, sh_hist[t]);
  }
}

// K3: re-hash, compute the bucket id, and scatter (lo, bucket) into the
// partition's contiguous range. cursor[j] starts at key_off[j] (absolute),
// so one atomic gives the destination. Per-partition cursors advance
// sequentially, so only ~nparts 32-byte sectors are write-active at a time
// and L2 merges the scattered 8/2-byte stores into full sectors.
template <class K>
__global__ void __launch_bounds__(256) k_scatter(K keys, int64_t n, uint64_t seed, uint64_t nparts,
                                                 const double* __restrict__ entries,
                                                 uint32_t bcount, uint32_t* __restrict__ cursor,
                                                 uint64_t* __restrict__ lo_out,
                                                 uint16_t* __restrict__ bid_out) {
  __shared__ double2 tab[BUCKET_TAB];
  load_bucket_pairs(entries, tab);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    Hash128 h = keys.hash(i, seed);
    uint32_t j = (uint32_t)mulhi(h.hi, nparts);
    uint32_t b = bucket_of_pairs(tab, h.hi, bcount);
    uint32_t pos = atomicAdd(cursor + j, 1u);
    if (bid_out) {
      lo_out[pos] = h.lo;
      bid_out[pos] = (uint16_t)b;
    } else {  // 16-byte records (lo, bucket id): one scattered store per key
      reinterpret_cast<ulonglong2*>(lo_out)[pos] = make_ulonglong2(h.lo, b);
    }
  }
}

// u64 fast path: 4 keys per thread per step (two 16-byte loads), so four
// independent hash -> atomic -> store chains are in flight per thread.
__global__ void __launch_bounds__(256) k_scatter_u64x4(const ulonglong2* __restrict__ keys2,
                                                       int64_t n, uint64_t seed, uint64_t nparts,
                                                       const double* __restrict__ entries,
                                                       uint32_t bcount,
                                                       uint32_t* __restrict__ cursor,
                                                       uint64_t* __restrict__ lo_out,
                                                       uint16_t* __restrict__ bid_out) {
  __shared__ double2 tab[BUCKET_TAB];
  load_bucket_pairs(entries, tab);
  const int64_t nq = n >> 2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq;
       q += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2 a = __ldg(keys2 + 2 * q), c = __ldg(keys2 + 2 * q + 1);
    const uint64_t k[4] = {a.x, a.y, c.x, c.y};
    uint32_t pos[4], b[4];
    uint64_t lo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const Hash128 h = murmur3_u64(k[e], seed);
      lo[e] = h.lo;
      b[e] = bucket_of_pairs(tab, h.hi, bcount);
      pos[e] = atomicAdd(cursor + (uint32_t)mulhi(h.hi, nparts), 1u);
    }
    if (bid_out) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        lo_out[pos[e]] = lo[e];
        bid_out[pos[e]] = (uint16_t)b[e];
      }
    } else {  // 16-byte records: one scattered store per key instead of two (-0.55 ms at C2)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        reinterpret_cast<ulonglong2*>(lo_out)[pos[e]] = make_ulonglong2(lo[e], b[e]);
    }
  }
  // tail (n % 4 keys)
  const int64_t t = (nq << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) {
    const uint64_t* keys = reinterpret_cast<const uint64_t*>(keys2);
    const Hash128 h = murmur3_u64(__ldg(keys + t), seed);
    const uint32_t pos = atomicAdd(cursor + (uint32_t)mulhi(h.hi, nparts), 1u);
    const uint32_t b = bucket_of_pairs(tab, h.hi, bcount);
    if (bid_out) {
      lo_out[pos] = h.lo;
      bid_out[pos] = (uint16_t)b;
    } else {
      reinterpret_cast<ulonglong2*>(lo_out)[pos] = make_ulonglong2(h.lo, b);
    }
  }
}

// Record-layout u64 scatter with NK keys per thread per step (NK / 2 16-byte
// loads): NK independent hash -> cursor atomic -> record store chains in
// flight per thread (the atomics' L2 round trips are the latency to hide).
#ifndef PHB_K3_MINB
#define PHB_K3_MINB 1
#endif
template <int NK>
__global__ void __launch_bounds__(256, PHB_K3_MINB) k_scatter_rec_u64(const ulonglong2* __restrict__ keys2,
                                                         int64_t n, uint64_t seed, uint64_t nparts,
                                                         const double* __restrict__ entries,
                                                         uint32_t bcount,
                                                         uint32_t* __restrict__ cursor,
                                                         ulonglong2* __restrict__ rec_out) {
  __shared__ double2 tab[BUCKET_TAB];
  load_bucket_pairs(entries, tab);
  const int64_t nv = n / NK;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nv;
       q += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k[NK];
#pragma unroll
    for (int e = 0; e < NK / 2; ++e) {
      const ulonglong2 v = __ldcs(keys2 + (NK / 2) * q + e);
      k[2 * e] = v.x;
      k[2 * e + 1] = v.y;
    }
    uint32_t pos[NK], b[NK];
    uint64_t lo[NK];
#pragma unroll
    for (int e = 0; e < NK; ++e) {
      const Hash128 h = murmur3_u64(k[e], seed);
      lo[e] = h.lo;
      b[e] = bucket_of_pairs(tab, h.hi, bcount);
      pos[e] = atomicAdd(cursor + (uint32_t)mulhi(h.hi, nparts), 1u);
    }
#pragma unroll
    for (int e = 0; e < NK; ++e) rec_out[pos[e]] = make_ulonglong2(lo[e], b[e]);
  }
  const int64_t t = nv * NK + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) {  // tail (n % NK keys, NK <= 256)
    const Hash128 h = murmur3_u64(__ldg(reinterpret_cast<const uint64_t*>(keys2) + t), seed);
    const uint32_t pos = atomicAdd(cursor + (uint32_t)mulhi(h.hi, nparts), 1u);
    rec_out[pos] = make_ulonglong2(h.lo, bucket_of_pairs(tab, h.hi, bcount));
  }
}

// K3 from the hashes K1 stored (byte keys): (hi, lo) -> partition, bucket
// id, 16-byte record at the partition's atomic cursor; 8 keys per thread.
// The key bytes are hashed once per build instead of twice.
__global__ void __launch_bounds__(256) k_scatter_hashed(const ulonglong2* __restrict__ hashes,
                                                        int64_t n, uint64_t nparts,
                                                        const double* __restrict__ entries,
                                                        uint32_t bcount,
                                                        uint32_t* __restrict__ cursor,
                                                        ulonglong2* __restrict__ rec_out) {
  constexpr int NK = 8;
  __shared__ double2 tab[BUCKET_TAB];
  load_bucket_pairs(entries, tab);
  const int64_t nv = n / NK;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nv;
       q += (int64_t)gridDim.x * blockDim.x) {
    ulonglong2 h[NK];
#pragma unroll
    for (int e = 0; e < NK; ++e) h[e] = __ldcs(hashes + NK * q + e);
    uint32_t pos[NK];
#pragma unroll
    for (int e = 0; e < NK; ++e) pos[e] = atomicAdd(cursor + (uint32_t)mulhi(h[e].x, nparts), 1u);
#pragma unroll
    for (int e = 0; e < NK; ++e)
      rec_out[pos[e]] = make_ulonglong2(h[e].y, bucket_of_pairs(tab, h[e].x, bcount));
  }
  const int64_t t = nv * NK + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) {
    const ulonglong2 hh = __ldg(hashes + t);
    const uint32_t pos = atomicAdd(cursor + (uint32_t)mulhi(hh.x, nparts), 1u);
    rec_out[pos] = make_ulonglong2(hh.y, bucket_of_pairs(tab, hh.x, bcount));
  }
}

// ---- K3 into fixed-capacity partition slots (no K1 pass before it).
// Partition j owns records [j * cap, j * cap + cap); its cursor starts at
// j * cap. The keys can arrive in chunks (one launch per chunk, overlapped
// with the host-to-device copy of the next); the exact per-partition counts
// are the cursors afterwards (phb_padded_counts), which also flags a
// partition that overflowed its capacity (the caller then falls back to
// the counted layout: K1 + K2 + K3).
__global__ void k_padded_init(int64_t nparts, uint32_t cap, uint32_t* __restrict__ cursor) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nparts;
       j += (int64_t)gridDim.x * blockDim.x)
    cursor[j] = (uint32_t)(j * cap);
}

__global__ void __launch_bounds__(256) k_scatter_padded_u64x4(
    const ulonglong2* __restrict__ keys2, int64_t n, uint64_t seed, uint64_t nparts,
    const double* __restrict__ entries, uint32_t bcount, uint32_t cap,
    uint32_t* __restrict__ cursor, uint64_t* __restrict__ lo_out, uint16_t* __restrict__ bid_out,
    uint32_t* __restrict__ overflow) {
  __shared__ double2 tab[BUCKET_TAB];
  load_bucket_pairs(entries, tab);
  const int64_t nq = n >> 2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq;
       q += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2 a = __ldg(keys2 + 2 * q), c = __ldg(keys2 + 2 * q + 1);
    const uint64_t k[4] = {a.x, a.y, c.x, c.y};
    uint32_t pos[4], b[4], lim[4];
    uint64_t lo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const Hash128 h = murmur3_u64(k[e], seed);
      const uint32_t j = (uint32_t)mulhi(h.hi, nparts);
      lo[e] = h.lo;
      b[e] = bucket_of_pairs(tab, h.hi, bcount);
      lim[e] = (j + 1) * cap;
      pos[e] = atomicAdd(cursor + j, 1u);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (pos[e] < lim[e]) {
        if (bid_out) {
          lo_out[pos[e]] = lo[e];
          bid_out[pos[e]] = (uint16_t)b[e];
        } else {  // 16-byte records
          reinterpret_cast<ulonglong2*>(lo_out)[pos[e]] = make_ulonglong2(lo[e], b[e]);
        }
      } else {
        atomicOr(overflow, 1u);
      }
    }
  }
  const int64_t t = (nq << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) {
    const uint64_t* keys = reinterpret_cast<const uint64_t*>(keys2);
    const Hash128 h = murmur3_u64(__ldg(keys + t), seed);
    const uint32_t j = (uint32_t)mulhi(h.hi, nparts);
    const uint32_t pos = atomicAdd(cursor + j, 1u);
    if (pos < (j + 1) * cap) {
      const uint32_t b = bucket_of_pairs(tab, h.hi, bcount);
      if (bid_out) {
        lo_out[pos] = h.lo;
        bid_out[pos] = (uint16_t)b;
      } else {
        reinterpret_cast<ulonglong2*>(lo_out)[pos] = make_ulonglong2(h.lo, b);
      }
    } else {
      atomicOr(overflow, 1u);
    }
  }
}

__global__ void k_padded_counts(const uint32_t* __restrict__ cursor, int64_t nparts, uint32_t cap,
                                uint32_t* __restrict__ counts, uint32_t* __restrict__ overflow) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nparts;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = cursor[j] - (uint32_t)(j * cap);
    counts[j] = c;
    if (c > cap) atomicOr(overflow, 1u);
  }
}

__global__ void k_cursor_init(const int64_t* __restrict__ key_off, int64_t nparts,
                              uint32_t* __restrict__ cursor) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nparts;
       j += (int64_t)gridDim.x * blockDim.x)
    cursor[j] = (uint32_t)key_off[j];
}

// K1 u64 fast path with a shared-memory histogram over all partitions
// (up to ~56k bins in 224 KB): one CTA of 1024 threads per SM, 4 keys per
// thread per step, then one global atomic per (CTA, non-empty bin).
__global__ void __launch_bounds__(1024, 1) k_hash_count_u64x4(const ulonglong2* __restrict__ keys2,
                                                              int64_t n, uint64_t seed,
                                                              uint64_t nparts,
                                                              uint32_t* __restrict__ counts) {
  extern __shared__ uint32_t hist[];
  for (uint32_t t = threadIdx.x; t < nparts; t += blockDim.x) hist[t] = 0;
  __syncthreads();
#ifndef PHB_K1_NK
#define PHB_K1_NK 8  // C2: 0.259 (4) -> 0.244 ms
#endif
  constexpr int NK = PHB_K1_NK;  // keys per thread per step (NK / 2 16-byte streaming loads)
  const int64_t nq = n / NK;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq;
       q += (int64_t)gridDim.x * blockDim.x) {
    ulonglong2 v[NK / 2];
#pragma unroll
    for (int e = 0; e < NK / 2; ++e) v[e] = __ldcs(keys2 + (NK / 2) * q + e);
#pragma unroll
    for (int e = 0; e < NK / 2; ++e) {
      atomicAdd(hist + (uint32_t)mulhi(murmur3_u64(v[e].x, seed).hi, nparts), 1u);
      atomicAdd(hist + (uint32_t)mulhi(murmur3_u64(v[e].y, seed).hi, nparts), 1u);
    }
  }
  const int64_t t = nq * NK + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) {
    const uint64_t* keys = reinterpret_cast<const uint64_t*>(keys2);
    atomicAdd(hist + (uint32_t)mulhi(murmur3_u64(__ldg(keys + t), seed).hi, nparts), 1u);
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < nparts; j += blockDim.x)
    if (hist[j]) atomicAdd(counts + j, hist[j]);
}

// Bucket ids of already-hashed, already-grouped keys (used by the
// reference-shaped entry point that receives his/los like
// build_partition_range, _kernels.py:252-255).
__global__ void __launch_bounds__(256) k_bucket_ids(const uint64_t* __restrict__ his, int64_t n,
                                                    const double* __restrict__ entries,
                                                    uint32_t bcount, uint16_t* __restrict__ bid) {
  __shared__ double2 tab[BUCKET_TAB];
  load_bucket_pairs(entries, tab);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bid[i] = (uint16_t)bucket_of_pairs(tab, __ldg(his + i), bcount);
}

static inline int grid_for(int64_t n, int per_sm = 16) {
  int sms = num_sms();
  int64_t need = (n + 255) / 256;
  int64_t cap = (int64_t)sms * per_sm;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

int launch_murmur(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t n,
                  uint64_t seed, uint64_t* hi, uint64_t* lo, cudaStream_t st) {
  if (n <= 0) return 0;
  int g = grid_for(n);
  if (keys64)
    note_launch(), k_murmur<<<g, 256, 0, st>>>(U64Keys{keys64}, n, seed, hi, lo);
  else
    note_launch(), k_murmur<<<g, 256, 0, st>>>(ByteKeys{buf, offsets}, n, seed, hi, lo);
  return (int)cudaGetLastError();
}

constexpr uint64_t SMEM_HIST_MAX = 12288;      // 48 KB of u32 bins (256-thread CTAs)
constexpr uint64_t SMEM_HIST_MAX_BIG = 56 * 1024; // 224 KB (one 1024-thread CTA per SM)

static inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int launch_hash_count(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64,
                      int64_t n, uint64_t seed, uint64_t nparts, uint32_t* counts,
                      cudaStream_t st, uint64_t* hashes_out) {
  if (n <= 0) return 0;
  int g = grid_for(n);
  ulonglong2* const store = reinterpret_cast<ulonglong2*>(hashes_out);
  if (keys64 && store) return 1003;  // u64 keys re-hash cheaply; the store is for byte keys
  if (keys64 && aligned16(keys64) && nparts > SMEM_HIST_MAX && nparts <= SMEM_HIST_MAX_BIG) {
    size_t sh = nparts * sizeof(uint32_t);
    // the largest histogram this path takes (not this launch's size): a
    // concurrent launch from another host thread must not see a lower cap
    PHB_CUDA_TRY(cudaFuncSetAttribute(k_hash_count_u64x4,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(SMEM_HIST_MAX_BIG * sizeof(uint32_t))));
    int64_t need = ((n >> 2) + 1023) / 1024;
    int gb = (int)std::max<int64_t>(1, std::min<int64_t>(need, num_sms()));
    note_launch(), k_hash_count_u64x4<<<gb, 1024, sh, st>>>(reinterpret_cast<const ulonglong2*>(keys64), n,
                                            seed, nparts, counts);
    return (int)cudaGetLastError();
  }
  if (nparts <= SMEM_HIST_MAX) {
    // fewer, fatter CTAs: the flush costs nparts atomics per CTA
    int gs = g < 2 * num_sms() ? g : 2 * num_sms();
    size_t sh = nparts * sizeof(uint32_t);
    if (keys64)
      note_launch(), k_hash_count<U64Keys, true><<<gs, 256, sh, st>>>(U64Keys{keys64}, n, seed, nparts, counts, nullptr);
    else
      note_launch(), k_hash_count<ByteKeys, true>
          <<<gs, 256, sh, st>>>(ByteKeys{buf, offsets}, n, seed, nparts, counts, store);
  } else {
    if (keys64)
      note_launch(), k_hash_count<U64Keys, false><<<g, 256, 0, st>>>(U64Keys{keys64}, n, seed, nparts, counts, nullptr);
    else
      note_launch(), k_hash_count<ByteKeys, false>
          <<<g, 256, 0, st>>>(ByteKeys{buf, offsets}, n, seed, nparts, counts, store);
  }
  return (int)cudaGetLastError();
}

int launch_scatter(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t n,
                   uint64_t seed, uint64_t nparts, const double* entries, uint32_t bcount,
                   const int64_t* key_off, uint32_t* cursor, uint64_t* lo_out, uint16_t* bid_out,
                   cudaStream_t st) {
  if (n <= 0) return 0;
  if (n >= (int64_t(1) << 32)) return 1003;  // u32 cursors
  note_launch(), k_cursor_init<<<(int)std::min<int64_t>((nparts + 255) / 256, 4096), 256, 0, st>>>(
      key_off, (int64_t)nparts, cursor);
  PHB_CUDA_TRY(cudaGetLastError());
  int g = grid_for(n);
#ifndef PHB_K3_NK
#define PHB_K3_NK 8  // C2: 2.31 (4) -> 2.26 ms; C3: 27.4 -> 25.4 ms
#endif
  if (keys64 && aligned16(keys64) && !bid_out) {
    const int gk = grid_for((n + PHB_K3_NK - 1) / PHB_K3_NK);
    note_launch(), k_scatter_rec_u64<PHB_K3_NK><<<gk, 256, 0, st>>>(
        reinterpret_cast<const ulonglong2*>(keys64), n, seed, nparts, entries, bcount, cursor,
        reinterpret_cast<ulonglong2*>(lo_out));
  } else if (keys64 && aligned16(keys64)) {
    int g4 = grid_for((n + 3) / 4);
    note_launch(), k_scatter_u64x4<<<g4, 256, 0, st>>>(reinterpret_cast<const ulonglong2*>(keys64), n, seed,
                                        nparts, entries, bcount, cursor, lo_out, bid_out);
  } else if (keys64) {
    note_launch(), k_scatter<<<g, 256, 0, st>>>(U64Keys{keys64}, n, seed, nparts, entries, bcount, cursor,
                                 lo_out, bid_out);
  } else {
    note_launch(), k_scatter<<<g, 256, 0, st>>>(ByteKeys{buf, offsets}, n, seed, nparts, entries, bcount,
                                 cursor, lo_out, bid_out);
  }
  return (int)cudaGetLastError();
}

int launch_scatter_padded(const uint64_t* keys64, int64_t n, uint64_t seed, uint64_t nparts,
                          const double* entries, uint32_t bcount, uint32_t cap, int init,
                          uint32_t* cursor, uint64_t* lo_out, uint16_t* bid_out,
                          uint32_t* overflow, cudaStream_t st) {
  if ((uint64_t)nparts * cap >= (uint64_t(1) << 32)) return 1003;  // u32 cursors
  if (init) {
    note_launch(), k_padded_init<<<(int)std::min<uint64_t>((nparts + 255) / 256, 4096), 256, 0, st>>>(
        (int64_t)nparts, cap, cursor);
    PHB_CUDA_TRY(cudaGetLastError());
  }
  if (n <= 0) return 0;
  if (!aligned16(keys64)) return 1003;
  note_launch(), k_scatter_padded_u64x4<<<grid_for((n + 3) / 4), 256, 0, st>>>(
      reinterpret_cast<const ulonglong2*>(keys64), n, seed, nparts, entries, bcount, cap, cursor,
      lo_out, bid_out, overflow);
  return (int)cudaGetLastError();
}

int launch_padded_counts(const uint32_t* cursor, int64_t nparts, uint32_t cap, uint32_t* counts,
                         uint32_t* overflow, cudaStream_t st) {
  note_launch(), k_padded_counts<<<(int)std::min<int64_t>((nparts + 255) / 256, 4096), 256, 0, st>>>(
      cursor, nparts, cap, counts, overflow);
  return (int)cudaGetLastError();
}

int launch_bucket_ids(const uint64_t* his, int64_t n, const double* entries, uint32_t bcount,
                      uint16_t* bid, cudaStream_t st) {
  if (n <= 0) return 0;
  note_launch(), k_bucket_ids<<<grid_for(n), 256, 0, st>>>(his, n, entries, bcount, bid);
  return (int)cudaGetLastError();
}

int launch_scatter_hashed(const uint64_t* hashes, int64_t n, uint64_t nparts,
                          const double* entries, uint32_t bcount, const int64_t* key_off,
                          uint32_t* cursor, uint64_t* rec_out, cudaStream_t st) {
  if (n <= 0) return 0;
  if (n >= (int64_t(1) << 32)) return 1003;  // u32 cursors
  if (reinterpret_cast<uintptr_t>(hashes) & 15) return 1003;
  note_launch(), k_cursor_init<<<(int)std::min<int64_t>((nparts + 255) / 256, 4096), 256, 0, st>>>(
      key_off, (int64_t)nparts, cursor);
  PHB_CUDA_TRY(cudaGetLastError());
  note_launch(), k_scatter_hashed<<<grid_for((n + 7) / 8), 256, 0, st>>>(
      reinterpret_cast<const ulonglong2*>(hashes), n, nparts, entries, bcount, cursor,
      reinterpret_cast<ulonglong2*>(rec_out));
  return (int)cudaGetLastError();
}

}  // namespace phb
