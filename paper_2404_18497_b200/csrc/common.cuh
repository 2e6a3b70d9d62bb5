// Shared device primitives for the PHOBIC construction engine (sm_100a).
//
// Every function here restates one arithmetic step of the reference
// (`pilothash`, /root/reference/pkg/src/pilothash) bit for bit:
//   mix64            _kernels.py:40-47   (splitmix64 finalizer)
//   mulhi            _kernels.py:50-55   (exact floor(z*m / 2^64), m < 2^32)
//   fmix64 / rotl    _kernels.py:58-70
//   murmur3 u64/bytes _kernels.py:89-146 (canonical MurmurHash3_x64_128)
//   bucket_of        _kernels.py:149-167 (FP64, separately rounded, no FMA)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace phb {

constexpr uint64_t MIX1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t MIX2 = 0x94D049BB133111EBull;
constexpr uint64_t BUCKET_SALT = 0xC2B2AE3D27D4EB4Full;    // _kernels.py:29
constexpr uint64_t POSITION_SALT = 0x9E3779B97F4A7C15ull;  // _kernels.py:30
constexpr uint64_t MM_C1 = 0x87C37B91114253D5ull;
constexpr uint64_t MM_C2 = 0x4CF5AD432745937Full;
constexpr uint64_t MM_F1 = 0xFF51AFD7ED558CCDull;
constexpr uint64_t MM_F2 = 0xC4CEB9FE1A85EC53ull;
constexpr int GRID = 2048;  // assignment.py:26

__host__ __device__ constexpr uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= MIX1;
  z ^= z >> 27;
  z *= MIX2;
  z ^= z >> 31;
  return z;
}

__device__ __forceinline__ uint64_t mulhi(uint64_t z, uint64_t m) { return __umul64hi(z, m); }

__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) {
#ifdef __CUDA_ARCH__
  // two 32-bit funnel shifts (the generic 64-bit form compiles to ~4 ops)
  const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  uint32_t nhi, nlo;
  if (r < 32) {
    nhi = __funnelshift_l(lo, hi, r);
    nlo = __funnelshift_l(hi, lo, r);
  } else {
    nhi = __funnelshift_l(hi, lo, r - 32);
    nlo = __funnelshift_l(lo, hi, r - 32);
  }
  return ((uint64_t)nhi << 32) | nlo;
#else
  return (x << r) | (x >> (64 - r));
#endif
}

__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z ^= z >> 33;
  z *= MM_F1;
  z ^= z >> 33;
  z *= MM_F2;
  z ^= z >> 33;
  return z;
}

struct Hash128 {
  uint64_t hi, lo;
};

// murmur3 finalisation shared by both key paths (_kernels.py:137-146).
__device__ __forceinline__ Hash128 mm_final(uint64_t h1, uint64_t h2, uint64_t len) {
  h1 ^= len;
  h2 ^= len;
  h1 += h2;
  h2 += h1;
  h1 = fmix64(h1);
  h2 = fmix64(h2);
  h1 += h2;
  h2 += h1;
  return {h1, h2};
}

__device__ __forceinline__ uint64_t mm_k1(uint64_t k1) {
  k1 *= MM_C1;
  k1 = rotl64(k1, 31);
  k1 *= MM_C2;
  return k1;
}
__device__ __forceinline__ uint64_t mm_k2(uint64_t k2) {
  k2 *= MM_C2;
  k2 = rotl64(k2, 33);
  k2 *= MM_C1;
  return k2;
}

// Fast path: a u64 key == its 8-byte little-endian string. nblocks = 0,
// tail k1 = the word, k2 = 0 (_kernels.py:118-136). Mixing a zero k1 is a
// no-op, so the `if k1 != 0` guard needs no branch.
__device__ __forceinline__ Hash128 murmur3_u64(uint64_t key, uint64_t seed) {
  uint64_t h1 = seed ^ mm_k1(key);
  return mm_final(h1, seed, 8ull);
}

// Little-endian bytes [p, p + nbytes), 1 <= nbytes <= 8, from the aligned
// 8-byte words that contain them: the second word is read only when the
// bytes spill into it, so no word without a key byte is touched.
__device__ __forceinline__ uint64_t load_le_words(const uint8_t* __restrict__ p, int nbytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint64_t* w = reinterpret_cast<const uint64_t*>(a & ~uintptr_t(7));
  const int sh = int(a & 7);
  uint64_t v = __ldg(w) >> (8 * sh);
  if (sh + nbytes > 8) v |= __ldg(w + 1) << (64 - 8 * sh);
  return nbytes >= 8 ? v : (v & ((1ull << (8 * nbytes)) - 1));
}

// Variable-length path over a byte buffer (_kernels.py:89-146); the key may
// be arbitrarily aligned: bytes are assembled from aligned 8-byte words.
__device__ __forceinline__ Hash128 murmur3_bytes(const uint8_t* __restrict__ key, int64_t len,
                                                 uint64_t seed) {
  uint64_t h1 = seed, h2 = seed;
  const int64_t nblocks = len >> 4;
  if (nblocks > 0) {
    // 16-byte blocks from consecutive aligned words: word i+1 of one block
    // is word 0 of the next (one load per 8 bytes when the key is unaligned)
    const uintptr_t a = reinterpret_cast<uintptr_t>(key);
    const uint64_t* w = reinterpret_cast<const uint64_t*>(a & ~uintptr_t(7));
    const int sh = int(a & 7) * 8;
    uint64_t w0 = __ldg(w);
    for (int64_t blk = 0; blk < nblocks; ++blk) {
      uint64_t k1, k2;
      if (sh == 0) {
        k1 = w0;
        k2 = __ldg(w + 2 * blk + 1);
        if (blk + 1 < nblocks) w0 = __ldg(w + 2 * blk + 2);
      } else {
        const uint64_t w1 = __ldg(w + 2 * blk + 1), w2 = __ldg(w + 2 * blk + 2);
        k1 = (w0 >> sh) | (w1 << (64 - sh));
        k2 = (w1 >> sh) | (w2 << (64 - sh));
        w0 = w2;
      }
      h1 ^= mm_k1(k1);
      h1 = rotl64(h1, 27);
      h1 += h2;
      h1 = h1 * 5 + 0x52DCE729ull;
      h2 ^= mm_k2(k2);
      h2 = rotl64(h2, 31);
      h2 += h1;
      h2 = h2 * 5 + 0x38495AB5ull;
    }
  }
  const uint8_t* tail = key + nblocks * 16;
  const int rem = int(len - nblocks * 16);
  uint64_t k1 = 0, k2 = 0;
  if (rem > 8) {
    k1 = load_le_words(tail, 8);
    k2 = load_le_words(tail + 8, rem - 8);
  } else if (rem > 0) {
    k1 = load_le_words(tail, rem);
  }
  h2 ^= mm_k2(k2);
  h1 ^= mm_k1(k1);
  return mm_final(h1, h2, (uint64_t)len);
}

// Bucket of a high word (_kernels.py:158-167, assignment.py:124-161).
// x = (f64(mix64(hi ^ SALT)) + 1) * 2^-64; t = 2048 x; k = int(t);
// gamma = e[2048] if k >= 2048 else e[k] + (t - k) * (e[k+1] - e[k]);
// b = clamp(ceil(gamma * B), 1, B). Each operation rounds on its own:
// the explicit _rn intrinsics forbid FMA contraction.
//
// Default: the direct conversions (I2F / F2I / FRND on the XU pipe).
// PHB_BUCKET_FP64 builds an XU-free form, bit-identical (edge cases in
// tools/bucket_edge.py): an integer below 2^32 becomes a double as
// (2^52 + v) - 2^52 on the FP64 pipe, a u64 is rounded once by an FMA of its
// two exact halves, int(t) and ceil(y) come from the 2^52
// round-to-integer trick with a one-step correction. Measured slower in
// the query (1.42 vs 1.14 ms at C2: a longer dependent chain; the XU pipe
// was at 10%, not the limit) and neutral in the scatter, so it is off.
__device__ __forceinline__ double f64_of_u32(uint32_t v) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)v), 0x1p52);
}
__device__ __forceinline__ double f64_rn_of_u64(uint64_t v) {  // == __ull2double_rn(v)
  return __fma_rn(f64_of_u32((uint32_t)(v >> 32)), 0x1p32, f64_of_u32((uint32_t)v));
}

struct BucketT {
  double t, kd;  // t = 2048 x and (double)k
  int k;         // k = int(t), t in [0, 2048]
};
#ifndef PHB_BUCKET_FP64
__device__ __forceinline__ BucketT bucket_t(uint64_t hi) {
  const uint64_t xb = mix64(hi ^ BUCKET_SALT);
  const double x = __dmul_rn(__dadd_rn(__ull2double_rn(xb), 1.0), 0x1p-64);
  const double t = __dmul_rn(x, 2048.0);
  const int k = __double2int_rz(t);
  return {t, (double)k, k};
}
__device__ __forceinline__ uint32_t bucket_finish(double g, uint32_t bcount) {
  double y = __dmul_rn(g, (double)bcount);
  double c = ceil(y);
  if (c < 1.0) return 1u;
  if (c > (double)bcount) return bcount;
  return (uint32_t)c;
}
#else
__device__ __forceinline__ BucketT bucket_t(uint64_t hi) {
  const uint64_t xb = mix64(hi ^ BUCKET_SALT);
  const double x = __dmul_rn(__dadd_rn(f64_rn_of_u64(xb), 1.0), 0x1p-64);
  const double t = __dmul_rn(x, 2048.0);
  const double r = __dadd_rn(t, 0x1p52);  // 2^52 + round-to-nearest-even(t)
  double kd = __dsub_rn(r, 0x1p52);
  int k = __double2loint(r);
  if (kd > t) {  // rounded up: truncate
    kd = __dsub_rn(kd, 1.0);
    k -= 1;
  }
  return {t, kd, k};
}
__device__ __forceinline__ uint32_t bucket_finish(double g, uint32_t bcount) {
  const double y = __dmul_rn(g, f64_of_u32(bcount));  // y in [0, B]
  const double r = __dadd_rn(y, 0x1p52);
  uint32_t c = (uint32_t)__double2loint(r);  // round-to-nearest-even(y)
  if (__dsub_rn(r, 0x1p52) < y) c += 1;      // ceil
  if (c < 1u) return 1u;
  if (c > bcount) return bcount;
  return c;
}
#endif

__device__ __forceinline__ uint32_t bucket_of(const double* __restrict__ e, uint64_t hi,
                                              uint32_t bcount) {
  const BucketT b = bucket_t(hi);
  double g;
  if (b.k >= GRID) {
    g = __ldg(e + GRID);
  } else {
    const double ek = __ldg(e + b.k), ek1 = __ldg(e + b.k + 1);
    g = __dadd_rn(ek, __dmul_rn(__dsub_rn(b.t, b.kd), __dsub_rn(ek1, ek)));
  }
  return bucket_finish(g, bcount);
}

// bucket_of over a shared-memory copy of the table as adjacent pairs
// tab[k] = (e[k], e[k+1]) for k < GRID and tab[GRID] = (e[GRID], e[GRID]):
// one 16-byte shared load instead of two random L1 gathers per key.
constexpr int BUCKET_TAB = GRID + 1;  // double2 entries (32 KB)

__device__ __forceinline__ void load_bucket_pairs(const double* __restrict__ entries,
                                                  double2* tab) {
  for (int k = threadIdx.x; k <= GRID; k += blockDim.x)
    tab[k] = make_double2(__ldg(entries + k), __ldg(entries + (k < GRID ? k + 1 : k)));
  __syncthreads();
}

__device__ __forceinline__ uint32_t bucket_of_pairs(const double2* tab, uint64_t hi,
                                                    uint32_t bcount) {
  const BucketT b = bucket_t(hi);
  const double2 e = tab[b.k < GRID ? b.k : GRID];
  const double g = b.k >= GRID ? e.x : __dadd_rn(e.x, __dmul_rn(__dsub_rn(b.t, b.kd),
                                                                  __dsub_rn(e.y, e.x)));
  return bucket_finish(g, bcount);
}

__device__ __forceinline__ uint32_t position(uint64_t lo, uint64_t g, uint32_t m) {
  return (uint32_t)mulhi(mix64(lo ^ g), (uint64_t)m);
}

// expected offset: round-half-up of j*n/nparts (partitioning.py:68-70)
__host__ __device__ __forceinline__ int64_t expected_offset(int64_t j, int64_t n, int64_t nparts) {
  unsigned __int128 num = (unsigned __int128)(2 * (uint64_t)j) * (uint64_t)n + (uint64_t)nparts;
  return (int64_t)(num / (unsigned __int128)(2 * (uint64_t)nparts));
}

}  // namespace phb

#define PHB_CUDA_TRY(expr)                   \
  do {                                       \
    cudaError_t _e = (expr);                 \
    if (_e != cudaSuccess) return (int)_e;   \
  } while (0)
