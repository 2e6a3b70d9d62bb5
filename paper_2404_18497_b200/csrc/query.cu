// K7 query / K8 verify.
//
// K7 replaces query_many_kernel (_kernels.py:379-397) and the scalar
// Mphf.query (mphf.py:119-128):
//   j = mulhi(hi, nparts); off_j = key_off[j] (= expected(j) + delta[j]);
//   m = off_{j+1} - off_j; m <= 0 -> off_j if off_j < n else n - 1;
//   b = bucket(hi); p = seed[j, b-1];
//   out = off_j + (mulhi(mix64(lo ^ mix64((p / m) ^ SALT)), m) + p) mod m.
// Hashing is fused (u64 or byte keys), or precomputed (his, los) are read,
// matching the reference kernel's own signature.
//
// K8 replaces is_bijection_on (mphf.py:147-151): instead of sorting the n
// outputs it sets one bit per output in an n-bit map; a repeated bit or an
// out-of-range output flags failure. n outputs, no repeats <=> bijection.
#include "common.cuh"
#include "phobic_internal.h"

namespace phb {

template <int MODE>  // 0: u64 keys, 1: byte keys, 2: precomputed his/los
__global__ void __launch_bounds__(256)
    k_query(const uint8_t* __restrict__ buf, const int64_t* __restrict__ offsets,
            const uint64_t* __restrict__ keys64, const uint64_t* __restrict__ his,
            const uint64_t* __restrict__ los, int64_t nq, uint64_t seed, int64_t n,
            uint64_t nparts, const int64_t* __restrict__ key_off,
            const double* __restrict__ entries, uint32_t bcount,
            const uint64_t* __restrict__ seeds, int64_t s_sj, int64_t s_sb,
            int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq;
       i += (int64_t)gridDim.x * blockDim.x) {
    Hash128 h;
    if (MODE == 0) {
      h = murmur3_u64(__ldg(keys64 + i), seed);
    } else if (MODE == 1) {
      int64_t a = __ldg(offsets + i), b = __ldg(offsets + i + 1);
      h = murmur3_bytes(buf + a, b - a, seed);
    } else {
      h.hi = __ldg(his + i);
      h.lo = __ldg(los + i);
    }
    const uint64_t j = mulhi(h.hi, nparts);
    const int64_t offj = __ldg(key_off + j);
    const int64_t m = __ldg(key_off + j + 1) - offj;
    int64_t r;
    if (m <= 0) {
      r = offj < n ? offj : n - 1;
    } else {
      const uint32_t b = bucket_of(entries, h.hi, bcount);
      const uint64_t p = __ldg(seeds + (int64_t)j * s_sj + (int64_t)(b - 1) * s_sb);
      const uint64_t mu = (uint64_t)m;
      const uint64_t s = p / mu;
      const uint64_t d = p - s * mu;
      const uint64_t g = mix64(s ^ POSITION_SALT);
      uint64_t pos = mulhi(mix64(h.lo ^ g), mu) + d;  // (base + p) mod m == (base + d) mod m
      if (pos >= mu) pos -= mu;
      r = offj + (int64_t)pos;
    }
    out[i] = r;
  }
}

__global__ void __launch_bounds__(256) k_verify(const int64_t* __restrict__ out, int64_t nq,
                                                int64_t n, uint32_t* __restrict__ bitmap,
                                                uint32_t* __restrict__ bad) {
  uint32_t local_bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = out[i];
    if (v < 0 || v >= n) {
      local_bad = 1;
      continue;
    }
    uint32_t bit = 1u << (v & 31);
    if (atomicOr(bitmap + (v >> 5), bit) & bit) local_bad = 1;
  }
  if (__any_sync(0xffffffffu, local_bad) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

static inline int qgrid(int64_t n) {
  int64_t need = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms() * 16;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

int launch_query(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64,
                 const uint64_t* his, const uint64_t* los, int64_t nq, uint64_t seed, int64_t n,
                 int64_t nparts, const int64_t* key_off, const double* entries, uint32_t bcount,
                 const uint64_t* seeds, int64_t s_sj, int64_t s_sb, int64_t* out,
                 cudaStream_t st) {
  if (nq <= 0) return 0;
  const int g = qgrid(nq);
  if (his)
    k_query<2><<<g, 256, 0, st>>>(buf, offsets, keys64, his, los, nq, seed, n, (uint64_t)nparts,
                                  key_off, entries, bcount, seeds, s_sj, s_sb, out);
  else if (keys64)
    k_query<0><<<g, 256, 0, st>>>(buf, offsets, keys64, his, los, nq, seed, n, (uint64_t)nparts,
                                  key_off, entries, bcount, seeds, s_sj, s_sb, out);
  else
    k_query<1><<<g, 256, 0, st>>>(buf, offsets, keys64, his, los, nq, seed, n, (uint64_t)nparts,
                                  key_off, entries, bcount, seeds, s_sj, s_sb, out);
  return (int)cudaGetLastError();
}

int launch_verify(const int64_t* out, int64_t nq, int64_t n, uint32_t* bitmap, uint32_t* bad,
                  cudaStream_t st) {
  if (nq <= 0) return 0;
  k_verify<<<qgrid(nq), 256, 0, st>>>(out, nq, n, bitmap, bad);
  return (int)cudaGetLastError();
}

}  // namespace phb
