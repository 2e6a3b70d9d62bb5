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
template <class K, bool SMEM>
__global__ void __launch_bounds__(256) k_hash_count(K keys, int64_t n, uint64_t seed,
                                                    uint64_t nparts,
                                                    uint32_t* __restrict__ counts) {
  extern __shared__ uint32_t sh_hist[];
  if (SMEM) {
    for (uint32_t t = threadIdx.x; t < nparts; t += blockDim.x) sh_hist[t] = 0;
    __syncthreads();
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    Hash128 h = keys.hash(i, seed);
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
// partition's contiguous range. Per-partition cursors advance
// sequentially, so only ~nparts 32-byte sectors are write-active at a time
// and L2 merges the scattered 8/2-byte stores into full sectors.
template <class K>
__global__ void __launch_bounds__(256) k_scatter(K keys, int64_t n, uint64_t seed, uint64_t nparts,
                                                 const double* __restrict__ entries,
                                                 uint32_t bcount,
                                                 const int64_t* __restrict__ key_off,
                                                 uint32_t* __restrict__ cursor,
                                                 uint64_t* __restrict__ lo_out,
                                                 uint16_t* __restrict__ bid_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    Hash128 h = keys.hash(i, seed);
    uint32_t j = (uint32_t)mulhi(h.hi, nparts);
    uint32_t b = bucket_of(entries, h.hi, bcount);
    int64_t pos = __ldg(key_off + j) + atomicAdd(cursor + j, 1u);
    lo_out[pos] = h.lo;
    bid_out[pos] = (uint16_t)b;
  }
}

// Bucket ids of already-hashed, already-grouped keys (used by the
// reference-shaped entry point that receives his/los like
// build_partition_range, _kernels.py:252-255).
__global__ void __launch_bounds__(256) k_bucket_ids(const uint64_t* __restrict__ his, int64_t n,
                                                    const double* __restrict__ entries,
                                                    uint32_t bcount, uint16_t* __restrict__ bid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bid[i] = (uint16_t)bucket_of(entries, __ldg(his + i), bcount);
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
    k_murmur<<<g, 256, 0, st>>>(U64Keys{keys64}, n, seed, hi, lo);
  else
    k_murmur<<<g, 256, 0, st>>>(ByteKeys{buf, offsets}, n, seed, hi, lo);
  return (int)cudaGetLastError();
}

constexpr uint64_t SMEM_HIST_MAX = 12288;  // 48 KB of u32 bins

int launch_hash_count(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64,
                      int64_t n, uint64_t seed, uint64_t nparts, uint32_t* counts,
                      cudaStream_t st) {
  if (n <= 0) return 0;
  int g = grid_for(n);
  if (nparts <= SMEM_HIST_MAX) {
    // fewer, fatter CTAs: the flush costs nparts atomics per CTA
    int gs = g < 2 * num_sms() ? g : 2 * num_sms();
    size_t sh = nparts * sizeof(uint32_t);
    if (keys64)
      k_hash_count<U64Keys, true><<<gs, 256, sh, st>>>(U64Keys{keys64}, n, seed, nparts, counts);
    else
      k_hash_count<ByteKeys, true>
          <<<gs, 256, sh, st>>>(ByteKeys{buf, offsets}, n, seed, nparts, counts);
  } else {
    if (keys64)
      k_hash_count<U64Keys, false><<<g, 256, 0, st>>>(U64Keys{keys64}, n, seed, nparts, counts);
    else
      k_hash_count<ByteKeys, false>
          <<<g, 256, 0, st>>>(ByteKeys{buf, offsets}, n, seed, nparts, counts);
  }
  return (int)cudaGetLastError();
}

int launch_scatter(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t n,
                   uint64_t seed, uint64_t nparts, const double* entries, uint32_t bcount,
                   const int64_t* key_off, uint32_t* cursor, uint64_t* lo_out, uint16_t* bid_out,
                   cudaStream_t st) {
  if (n <= 0) return 0;
  int g = grid_for(n);
  if (keys64)
    k_scatter<<<g, 256, 0, st>>>(U64Keys{keys64}, n, seed, nparts, entries, bcount, key_off,
                                 cursor, lo_out, bid_out);
  else
    k_scatter<<<g, 256, 0, st>>>(ByteKeys{buf, offsets}, n, seed, nparts, entries, bcount,
                                 key_off, cursor, lo_out, bid_out);
  return (int)cudaGetLastError();
}

int launch_bucket_ids(const uint64_t* his, int64_t n, const double* entries, uint32_t bcount,
                      uint16_t* bid, cudaStream_t st) {
  if (n <= 0) return 0;
  k_bucket_ids<<<grid_for(n), 256, 0, st>>>(his, n, entries, bcount, bid);
  return (int)cudaGetLastError();
}

}  // namespace phb
