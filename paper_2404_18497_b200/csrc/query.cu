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
      h = murmur3_u64(__ldcs(keys64 + i), seed);  // streaming: keep the tables in L2
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
    __stcs(out + i, r);
  }
}

// ---- K7q: the same query over compact tables, for structures where every
// seed and every key offset fits 32 bits (far beyond the BASELINE sizes:
// the largest C3 seed is ~2^24, n < 2^32):
//   * seeds32 [B][nparts] u32 = (s << 16) | d for p = s m + d: half the
//     gather footprint of the u64 matrix (44 MB at C2, L2-resident) and no
//     division per query (needs s < 2^16; the C2 maximum is ~3,500);
//   * part2 [nparts] (offset, end) u32 pairs: one 8-byte gather per query
//     instead of two 8-byte key_off loads;
//   * the bucket table as (e[k], e[k+1]) pairs in shared memory: one
//     16-byte shared load instead of two random L1 gathers per query (those
//     queued behind the global loads: lg_throttle in the profile);
//   * u64 keys: four per thread, so four independent gather chains overlap.
__device__ __forceinline__ int64_t finish_query(uint64_t lo, uint2 pe, int64_t n, uint32_t sd) {
  const int64_t offj = pe.x;
  if (pe.y <= pe.x) return offj < n ? offj : n - 1;
  const uint32_t mu = pe.y - pe.x;
  const uint32_t sq = sd >> 16, d = sd & 0xffffu;  // p = sq * m + d, split once at table build
  const uint64_t g = mix64((uint64_t)sq ^ POSITION_SALT);
  uint32_t pos = (uint32_t)mulhi(mix64(lo ^ g), (uint64_t)mu) + d;  // (base + p) mod m
  if (pos >= mu) pos -= mu;
  return offj + (int64_t)pos;
}

__global__ void __launch_bounds__(256)
    k_query32_u64x4(const ulonglong2* __restrict__ keys2, int64_t nq, uint64_t seed, int64_t n,
                    uint64_t nparts, const uint2* __restrict__ part2,
                    const double* __restrict__ entries, uint32_t bcount,
                    const uint32_t* __restrict__ seeds32, longlong2* __restrict__ out2) {
  __shared__ double2 tab[BUCKET_TAB];
  load_bucket_pairs(entries, tab);
  const int64_t nv = nq >> 2;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv;
       v += (int64_t)gridDim.x * blockDim.x) {
    // streaming keys / outputs are marked evict-first so the tables stay in L2
    const ulonglong2 ka = __ldcs(keys2 + 2 * v), kc = __ldcs(keys2 + 2 * v + 1);
    const uint64_t k[4] = {ka.x, ka.y, kc.x, kc.y};
    uint64_t hi[4], lo[4], j[4];
    uint2 pe[4];
    uint32_t p[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const Hash128 h = murmur3_u64(k[e], seed);
      hi[e] = h.hi;
      lo[e] = h.lo;
      j[e] = mulhi(h.hi, nparts);
      pe[e] = __ldg(part2 + j[e]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t b = bucket_of_pairs(tab, hi[e], bcount);
      p[e] = __ldg(seeds32 + (int64_t)(b - 1) * (int64_t)nparts + (int64_t)j[e]);
    }
    int64_t r[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) r[e] = finish_query(lo[e], pe[e], n, p[e]);
    __stcs(out2 + 2 * v, make_longlong2(r[0], r[1]));
    __stcs(out2 + 2 * v + 1, make_longlong2(r[2], r[3]));
  }
  // tail (nq % 4 keys)
  const int64_t t = (nv << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < nq) {
    const Hash128 h = murmur3_u64(__ldg(reinterpret_cast<const uint64_t*>(keys2) + t), seed);
    const uint64_t jj = mulhi(h.hi, nparts);
    const uint2 q = __ldg(part2 + jj);
    const uint32_t b = bucket_of_pairs(tab, h.hi, bcount);
    const uint32_t pp = __ldg(seeds32 + (int64_t)(b - 1) * (int64_t)nparts + (int64_t)jj);
    reinterpret_cast<int64_t*>(out2)[t] = finish_query(h.lo, q, n, pp);
  }
}

__global__ void __launch_bounds__(256)
    k_query32_bytes(const uint8_t* __restrict__ buf, const int64_t* __restrict__ offsets,
                    int64_t nq, uint64_t seed, int64_t n, uint64_t nparts,
                    const uint2* __restrict__ part2, const double* __restrict__ entries,
                    uint32_t bcount, const uint32_t* __restrict__ seeds32,
                    int64_t* __restrict__ out) {
  __shared__ double2 tab[BUCKET_TAB];
  load_bucket_pairs(entries, tab);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = __ldg(offsets + i), e = __ldg(offsets + i + 1);
    const Hash128 h = murmur3_bytes(buf + a, e - a, seed);
    const uint64_t j = mulhi(h.hi, nparts);
    const uint2 q = __ldg(part2 + j);
    const uint32_t b = bucket_of_pairs(tab, h.hi, bcount);
    const uint32_t p = __ldg(seeds32 + (int64_t)(b - 1) * (int64_t)nparts + (int64_t)j);
    out[i] = finish_query(h.lo, q, n, p);
  }
}

// K7s: K7q with the partition offsets in shared memory (u32 key_off[0..nparts],
// 4 B per partition: up to ~49k partitions next to the 32 KB bucket table,
// i.e. C2's 40k). A query then makes ONE random global gather (its seed),
// not two: the random gathers are what the L1 tag stage serialises (32
// distinct lines per warp instruction). One 1024-thread CTA per SM, the
// tables loaded once per CTA.
#ifndef PHB_Q_NK
#define PHB_Q_NK 4
#endif
// Byte-key master hashes as (hi, lo) pairs, for the two-pass string query.
__global__ void __launch_bounds__(256) k_hash_pairs(const uint8_t* __restrict__ buf,
                                                    const int64_t* __restrict__ offsets, int64_t n,
                                                    uint64_t seed, ulonglong2* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = __ldg(offsets + i), b = __ldg(offsets + i + 1);
    const Hash128 h = murmur3_bytes(buf + a, b - a, seed);
    out[i] = make_ulonglong2(h.hi, h.lo);
  }
}

// Seed hashes mix64(s ^ POSITION_SALT) of seeds s < QGT_N, for the
// encoded-section kernel's shared table (K7es); the matrix kernel K7s keeps
// the 64-bit mix (a table there measured 3% slower).
constexpr int QGT_N = 256;

// HASHED: keys2 holds (hi, lo) master-hash pairs (byte keys, hashed by
// k_hash_pairs first) instead of u64 keys.
template <bool HASHED>
__global__ void __launch_bounds__(1024, 1)
    k_query32s_u64x4(const ulonglong2* __restrict__ keys2, int64_t nq, uint64_t seed, int64_t n,
                     uint64_t nparts, const int64_t* __restrict__ key_off,
                     const double* __restrict__ entries, uint32_t bcount,
                     const uint32_t* __restrict__ seeds32, longlong2* __restrict__ out2) {
  constexpr int NK = PHB_Q_NK;  // keys per thread per step
  extern __shared__ __align__(16) unsigned char q_smem[];
  double2* const tab = reinterpret_cast<double2*>(q_smem);
  uint32_t* const koff = reinterpret_cast<uint32_t*>(tab + BUCKET_TAB);
  for (int64_t j = threadIdx.x; j <= (int64_t)nparts; j += blockDim.x)
    koff[j] = (uint32_t)__ldg(key_off + j);
  load_bucket_pairs(entries, tab);  // ends with __syncthreads
  const int64_t nv = nq / NK;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv;
       v += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k[NK];
    ulonglong2 hk[HASHED ? NK : 1];
    if (HASHED) {
#pragma unroll
      for (int e = 0; e < NK; ++e) hk[e] = __ldcs(keys2 + NK * v + e);
    } else {
#pragma unroll
      for (int e = 0; e < NK / 2; ++e) {
        // streaming keys / outputs are marked evict-first so the seed table stays in L2
        const ulonglong2 kv = __ldcs(keys2 + (NK / 2) * v + e);
        k[2 * e] = kv.x;
        k[2 * e + 1] = kv.y;
      }
    }
    uint64_t lo[NK];
    uint2 pe[NK];
    uint32_t p[NK];
#pragma unroll
    for (int e = 0; e < NK; ++e) {
      const Hash128 h = HASHED ? Hash128{hk[e].x, hk[e].y} : murmur3_u64(k[e], seed);
      lo[e] = h.lo;
      const uint32_t j = (uint32_t)mulhi(h.hi, nparts);
      const uint32_t b = bucket_of_pairs(tab, h.hi, bcount);
      p[e] = __ldg(seeds32 + (int64_t)(b - 1) * (int64_t)nparts + j);
      pe[e] = make_uint2(koff[j], koff[j + 1]);
    }
#pragma unroll
    for (int e = 0; e < NK / 2; ++e)
      __stcs(out2 + (NK / 2) * v + e, make_longlong2(finish_query(lo[2 * e], pe[2 * e], n, p[2 * e]),
                                                     finish_query(lo[2 * e + 1], pe[2 * e + 1], n,
                                                                  p[2 * e + 1])));
  }
  const int64_t t = nv * NK + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < nq) {
    const Hash128 h = HASHED ? Hash128{__ldg(keys2 + t).x, __ldg(keys2 + t).y}
                             : murmur3_u64(__ldg(reinterpret_cast<const uint64_t*>(keys2) + t), seed);
    const uint32_t j = (uint32_t)mulhi(h.hi, nparts);
    const uint32_t b = bucket_of_pairs(tab, h.hi, bcount);
    const uint32_t pp = __ldg(seeds32 + (int64_t)(b - 1) * (int64_t)nparts + j);
    reinterpret_cast<int64_t*>(out2)[t] = finish_query(h.lo, make_uint2(koff[j], koff[j + 1]), n, pp);
  }
}

// key_off (int64 [nparts + 1]) -> (offset, end) u32 pairs
__global__ void k_part_table32(const int64_t* __restrict__ key_off, int64_t nparts,
                               uint2* __restrict__ part2) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nparts;
       j += (int64_t)gridDim.x * blockDim.x)
    part2[j] = make_uint2((uint32_t)key_off[j], (uint32_t)key_off[j + 1]);
}

// u64 seed matrix [B][nparts] -> the (s << 16) | d table of K7q; *overflow
// = 1 if some entry does not fit (s >= 2^16 or m > 2^16: the caller keeps
// the u64 path then).
__global__ void k_seed_table32(const uint64_t* __restrict__ seeds, const int64_t* __restrict__ key_off,
                               int64_t nparts, int64_t count, uint32_t* __restrict__ out,
                               uint32_t* __restrict__ overflow) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i % nparts;
    const int64_t m = key_off[j + 1] - key_off[j];
    const uint64_t p = seeds[i];
    uint32_t v = 0;
    if (m > 0) {
      const uint64_t sq = p / (uint64_t)m, d = p - sq * (uint64_t)m;
      if (sq >= 65536u || m > 65536) atomicOr(overflow, 1u);
      v = (uint32_t)((sq << 16) | d);
    }
    out[i] = v;
  }
}

// ---- K7e: query straight from the encoded seed section (no decoded matrix).
// Replaces CompactVector.get (encoders.py:89-99), RiceVector.get
// (encoders.py:224-230) with Select.select1 / next_one (encoders.py:129-154),
// and InterleavedSeeds.seed_at / MonoSeeds index maps (encoders.py:305-341)
// inside query_many_kernel. The section stays in HBM/L2 at its serialized
// size (~bits/key * n / 8), e.g. 27 MB at C2 instead of a 89 MB matrix.
struct ECol {  // one encoder of the section, byte offsets relative to the section blob
  int64_t kind, param, count, pay_byte, highs_byte, highs_nbits, samples_byte, nsamples;
};

#ifndef PHB_EBITS_BYTES
#define PHB_EBITS_BYTES 0
#endif
// little-endian bit field [addr, addr + nbits), nbits <= 64. Default: two
// aligned 64-bit loads (the section blob is 8-byte aligned and zero padded);
// PHB_EBITS_BYTES: byte loads.
__device__ __forceinline__ uint64_t ebits(const uint8_t* __restrict__ blob, uint64_t addr,
                                          int nbits) {
  if (nbits <= 0) return 0;
#if PHB_EBITS_BYTES
  const uint8_t* p = blob + (addr >> 3);
  const int sh = (int)(addr & 7);
  const int need = (sh + nbits + 7) >> 3;  // <= 9
  uint64_t lo = 0, hi = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < need) lo |= (uint64_t)__ldg(p + i) << (8 * i);
  if (need > 8) hi = __ldg(p + 8);
  const uint64_t v = (lo >> sh) | (sh ? (hi << (64 - sh)) : 0ull);
#else
  const uint64_t* w = reinterpret_cast<const uint64_t*>(blob) + (addr >> 6);
  const int sh = (int)(addr & 63);
  uint64_t v = __ldg(w) >> sh;
  if (sh + nbits > 64) v |= __ldg(w + 1) << (64 - sh);
#endif
  return nbits >= 64 ? v : (v & ((1ull << nbits) - 1));
}

__device__ __forceinline__ uint32_t ehigh_word(const uint8_t* blob, const ECol& d, int64_t w) {
  const int64_t nb = d.highs_nbits - 32 * w;
  if (nb <= 0) return 0;
  return (uint32_t)ebits(blob, 8ull * d.highs_byte + 32ull * w, nb < 32 ? (int)nb : 32);
}

// Dense select directory (built on the device once per loaded structure):
// dsel[c * stride + r] = position of the (64 r)-th one of Rice column c, so
// a select scans at most 63 ones instead of up to 1023 from the serialized
// every-1024th samples. One CTA per column.
constexpr int DS_STEP = 64;
__global__ void __launch_bounds__(256) k_select_index(const uint8_t* __restrict__ sec,
                                                      const ECol* __restrict__ cols,
                                                      int64_t stride, uint32_t* __restrict__ dsel) {
  __shared__ uint32_t wsum[8];
  __shared__ uint64_t carry;
  const ECol d = cols[blockIdx.x];
  if (d.kind != 1 || d.param >= 64) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int64_t nw = (d.highs_nbits + 31) / 32;
  constexpr int WPT = 8;
  uint32_t* row = dsel + (int64_t)blockIdx.x * stride;
  for (int64_t w0 = 0; w0 < nw; w0 += 256 * WPT) {
    const int64_t wb = w0 + (int64_t)threadIdx.x * WPT;
    uint32_t words[WPT], local = 0;
#pragma unroll
    for (int e = 0; e < WPT; ++e) {
      words[e] = wb + e < nw ? ehigh_word(sec, d, wb + e) : 0u;
      local += __popc(words[e]);
    }
    uint32_t inc = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      uint32_t x = lane < 8 ? wsum[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
      }
      if (lane < 8) wsum[lane] = x;
    }
    __syncthreads();
    uint64_t rank = carry + (wid ? wsum[wid - 1] : 0u) + inc - local;
#pragma unroll
    for (int e = 0; e < WPT; ++e) {
      uint32_t x = words[e];
      const uint32_t c = __popc(x);
      // ones with rank r = 0 (mod 64) inside this word
      uint64_t r = (rank + DS_STEP - 1) / DS_STEP * DS_STEP;
      while (r < rank + c) {
        uint32_t y = x;
        for (uint64_t q = rank; q < r; ++q) y &= y - 1;
        row[r / DS_STEP] = (uint32_t)(32 * (wb + e) + (__ffs(y) - 1));
        r += DS_STEP;
      }
      rank += c;
    }
    __syncthreads();
    if (threadIdx.x == 255) carry = rank;
    __syncthreads();
  }
}

// Select.select1: position of the (k+1)-th one (k >= 0); from the dense
// directory when there is one, else from the serialized samples
__device__ int64_t eselect1(const uint8_t* blob, const ECol& d, int64_t k,
                            const uint32_t* __restrict__ drow) {
  int64_t spos;
  int need;
  if (drow) {
    spos = __ldg(drow + (k >> 6));
    need = (int)(k & 63) + 1;
  } else {
    spos = (int64_t)ebits(blob, 8ull * d.samples_byte + 64ull * (k >> 10), 64);
    need = (int)(k & 1023) + 1;
  }
  int64_t w = spos >> 5;
  uint32_t word = ehigh_word(blob, d, w) & (0xffffffffu << (spos & 31));
  for (;;) {
    const int c = __popc(word);
    if (c >= need) {
      for (int r = 1; r < need; ++r) word &= word - 1;
      return 32 * w + (__ffs(word) - 1);
    }
    need -= c;
    word = ehigh_word(blob, d, ++w);
  }
}

// Select.next_one: first one at index >= pos
__device__ int64_t enext_one(const uint8_t* blob, const ECol& d, int64_t pos) {
  int64_t w = pos >> 5;
  uint32_t word = ehigh_word(blob, d, w) & (0xffffffffu << (pos & 31));
  while (!word) word = ehigh_word(blob, d, ++w);
  return 32 * w + (__ffs(word) - 1);
}

__device__ __forceinline__ uint64_t eget(const uint8_t* blob, const ECol* dp, int64_t i,
                                         const uint32_t* drow) {
  // only {kind, param} and {count, payload} are read for Compact columns
  const longlong2 kp = __ldg(reinterpret_cast<const longlong2*>(dp));
  const int64_t pay = __ldg(&dp->pay_byte);
  if (kp.x == 0) {  // CompactVector.get
    const int w = (int)kp.y;
    return w ? ebits(blob, 8ull * pay + (uint64_t)i * w, w) : 0ull;
  }
  const int b = (int)kp.y;  // RiceVector.get
  const uint64_t low = b ? ebits(blob, 8ull * pay + (uint64_t)i * b, b) : 0ull;
  if (b >= 64) return low;
  const ECol d = *dp;
  const int64_t prev = i > 0 ? eselect1(blob, d, i - 1, drow) : -1;
  const int64_t pos = enext_one(blob, d, prev + 1);
  return ((uint64_t)(pos - prev - 1) << b) | low;
}

template <int MODE>
__global__ void __launch_bounds__(256)
    k_query_enc(const uint8_t* __restrict__ buf, const int64_t* __restrict__ offsets,
                const uint64_t* __restrict__ keys64, int64_t nq, uint64_t seed, int64_t n,
                uint64_t nparts, const int64_t* __restrict__ key_off,
                const double* __restrict__ entries, uint32_t bcount,
                const uint8_t* __restrict__ sec, const ECol* __restrict__ cols, int mono,
                const uint32_t* __restrict__ dsel, int64_t dstride, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq;
       i += (int64_t)gridDim.x * blockDim.x) {
    Hash128 h;
    if (MODE == 0) {
      h = murmur3_u64(__ldcs(keys64 + i), seed);  // streaming: keep the section in L2
    } else {
      int64_t a = __ldg(offsets + i), b = __ldg(offsets + i + 1);
      h = murmur3_bytes(buf + a, b - a, seed);
    }
    const uint64_t j = mulhi(h.hi, nparts);
    const int64_t offj = __ldg(key_off + j);
    const int64_t m = __ldg(key_off + j + 1) - offj;
    int64_t r;
    if (m <= 0) {
      r = offj < n ? offj : n - 1;
    } else {
      const uint32_t b = bucket_of(entries, h.hi, bcount);
      const uint64_t p =
          mono ? eget(sec, cols, (int64_t)j * bcount + (b - 1), dsel)
               : eget(sec, cols + (b - 1), (int64_t)j, dsel ? dsel + (int64_t)(b - 1) * dstride : nullptr);
      const uint64_t mu = (uint64_t)m;
      const uint64_t s = (p >> 32) ? p / mu : (uint64_t)((uint32_t)p / (uint32_t)mu);
      const uint64_t d = p - s * mu;
      uint64_t pos = mulhi(mix64(h.lo ^ mix64(s ^ POSITION_SALT)), mu) + d;
      if (pos >= mu) pos -= mu;
      r = offj + (int64_t)pos;
    }
    __stcs(out + i, r);
  }
}

// K7es: K7e for large u64 batches of an interleaved structure, the K7s way:
// partition offsets (u32), bucket pairs and the Compact columns' (payload bit,
// width) in shared memory, four keys per thread, streaming keys / outputs.
// A Compact query then makes one random access into the section (its field);
// Rice columns take eget's select path (global descriptors).
// C32 (sections below 4 GB): the column descriptors as 8-byte (payload byte,
// kind | width) pairs and the seed hashes of seeds < QGT_N in shared memory,
// which keeps the C2 footprint under the 196 KB carveout step (16-byte
// descriptors put it at 197.6 KB -> 228 KB carveout, L1 60 -> 28 KB).
template <bool C32>
__global__ void __launch_bounds__(1024, 1)
    k_query_enc_s(const ulonglong2* __restrict__ keys2, int64_t nq, uint64_t seed, int64_t n,
                  uint64_t nparts, const int64_t* __restrict__ key_off,
                  const double* __restrict__ entries, uint32_t bcount,
                  const uint8_t* __restrict__ sec, const ECol* __restrict__ cols,
                  const uint32_t* __restrict__ dsel, int64_t dstride,
                  longlong2* __restrict__ out2) {
  extern __shared__ __align__(16) unsigned char q_smem[];
  double2* const tab = reinterpret_cast<double2*>(q_smem);
  ulonglong2* const cdesc = reinterpret_cast<ulonglong2*>(tab + BUCKET_TAB);  // (pay bit, kind|width)
  uint2* const cdesc32 = reinterpret_cast<uint2*>(tab + BUCKET_TAB);          // (pay byte, kind<<31|width)
  uint64_t* const gt = C32 ? reinterpret_cast<uint64_t*>(cdesc32 + ((bcount + 1) & ~1u)) : nullptr;
  uint32_t* const koff = C32 ? reinterpret_cast<uint32_t*>(gt + QGT_N)
                             : reinterpret_cast<uint32_t*>(cdesc + bcount);
  for (uint32_t c = threadIdx.x; c < bcount; c += blockDim.x) {
    const ECol d = cols[c];
    if (C32)
      cdesc32[c] = make_uint2((uint32_t)d.pay_byte,
                              ((uint32_t)(d.kind != 0) << 31) | (uint32_t)d.param);
    else
      cdesc[c] = make_ulonglong2(8ull * (uint64_t)d.pay_byte,
                                 ((uint64_t)(d.kind != 0) << 32) | (uint64_t)d.param);
  }
  if (C32)
    for (int t = threadIdx.x; t < QGT_N; t += blockDim.x) gt[t] = mix64((uint64_t)t ^ POSITION_SALT);
  for (int64_t j = threadIdx.x; j <= (int64_t)nparts; j += blockDim.x)
    koff[j] = (uint32_t)__ldg(key_off + j);
  load_bucket_pairs(entries, tab);  // ends with __syncthreads
  const int64_t nv = nq >> 2;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv;
       v += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2 ka = __ldcs(keys2 + 2 * v), kc = __ldcs(keys2 + 2 * v + 1);
    const uint64_t k[4] = {ka.x, ka.y, kc.x, kc.y};
    int64_t r[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const Hash128 h = murmur3_u64(k[e], seed);
      const uint32_t j = (uint32_t)mulhi(h.hi, nparts);
      const uint32_t b = bucket_of_pairs(tab, h.hi, bcount);
      const int64_t offj = koff[j];
      const int64_t m = (int64_t)koff[j + 1] - offj;
      if (m <= 0) {
        r[e] = offj < n ? offj : n - 1;
        continue;
      }
      uint64_t pbit, kw;
      if (C32) {
        const uint2 cd = cdesc32[b - 1];
        pbit = 8ull * cd.x;
        kw = cd.y;
      } else {
        const ulonglong2 cd = cdesc[b - 1];
        pbit = cd.x;
        kw = (cd.y >> 32) ? (1u << 31) | (uint32_t)cd.y : (uint32_t)cd.y;
      }
      uint64_t p;
      if ((kw >> 31) == 0) {  // CompactVector.get: one field
        const int w = (int)(kw & 0x7fffffffu);
        p = w ? ebits(sec, pbit + (uint64_t)j * w, w) : 0ull;
      } else {
        p = eget(sec, cols + (b - 1), (int64_t)j, dsel ? dsel + (int64_t)(b - 1) * dstride : nullptr);
      }
      const uint64_t mu = (uint64_t)m;
      const uint64_t sq = (p >> 32) ? p / mu : (uint64_t)((uint32_t)p / (uint32_t)mu);
      const uint64_t d = p - sq * mu;
      const uint64_t g = C32 && sq < (uint64_t)QGT_N ? gt[sq] : mix64(sq ^ POSITION_SALT);
      uint64_t pos = mulhi(mix64(h.lo ^ g), mu) + d;
      if (pos >= mu) pos -= mu;
      r[e] = offj + (int64_t)pos;
    }
    __stcs(out2 + 2 * v, make_longlong2(r[0], r[1]));
    __stcs(out2 + 2 * v + 1, make_longlong2(r[2], r[3]));
  }
  const int64_t t = (nv << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < nq) {
    const Hash128 h = murmur3_u64(__ldg(reinterpret_cast<const uint64_t*>(keys2) + t), seed);
    const uint32_t j = (uint32_t)mulhi(h.hi, nparts);
    const uint32_t b = bucket_of_pairs(tab, h.hi, bcount);
    const int64_t offj = koff[j];
    const int64_t m = (int64_t)koff[j + 1] - offj;
    int64_t rr;
    if (m <= 0) {
      rr = offj < n ? offj : n - 1;
    } else {
      const uint64_t p = eget(sec, cols + (b - 1), (int64_t)j,
                              dsel ? dsel + (int64_t)(b - 1) * dstride : nullptr);
      const uint64_t mu = (uint64_t)m;
      const uint64_t sq = p / mu, d = p - sq * mu;
      uint64_t pos = mulhi(mix64(h.lo ^ mix64(sq ^ POSITION_SALT)), mu) + d;
      if (pos >= mu) pos -= mu;
      rr = offj + (int64_t)pos;
    }
    reinterpret_cast<int64_t*>(out2)[t] = rr;
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
    note_launch(), k_query<2><<<g, 256, 0, st>>>(buf, offsets, keys64, his, los, nq, seed, n, (uint64_t)nparts,
                                  key_off, entries, bcount, seeds, s_sj, s_sb, out);
  else if (keys64)
    note_launch(), k_query<0><<<g, 256, 0, st>>>(buf, offsets, keys64, his, los, nq, seed, n, (uint64_t)nparts,
                                  key_off, entries, bcount, seeds, s_sj, s_sb, out);
  else
    note_launch(), k_query<1><<<g, 256, 0, st>>>(buf, offsets, keys64, his, los, nq, seed, n, (uint64_t)nparts,
                                  key_off, entries, bcount, seeds, s_sj, s_sb, out);
  return (int)cudaGetLastError();
}

int launch_query32(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t nq,
                   uint64_t seed, int64_t n, int64_t nparts, const int64_t* key_off,
                   const uint2* part2,
                   const double* entries, uint32_t bcount, const uint32_t* seeds32, int64_t* out,
                   cudaStream_t st) {
  if (nq <= 0) return 0;
  if (keys64) {
    if ((reinterpret_cast<uintptr_t>(keys64) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
      return 1003;  // PHB_E_ARGS: the 4-key vector path needs 16-byte alignment
    const size_t sh = sizeof(double2) * BUCKET_TAB + sizeof(uint32_t) * (size_t)(nparts + 1);
    int dev = 0, optin = 0;
    PHB_CUDA_TRY(cudaGetDevice(&dev));
    PHB_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (key_off && sh <= (size_t)optin && nq >= (int64_t)num_sms() * 4096) {
      // the largest shared footprint this path takes (concurrent launches
      // from other host threads must not see a lower cap)
      PHB_CUDA_TRY(cudaFuncSetAttribute(k_query32s_u64x4<false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
      note_launch(), k_query32s_u64x4<false><<<num_sms(), 1024, sh, st>>>(
          reinterpret_cast<const ulonglong2*>(keys64), nq, seed, n, (uint64_t)nparts, key_off,
          entries, bcount, seeds32, reinterpret_cast<longlong2*>(out));
    } else {
      note_launch(), k_query32_u64x4<<<qgrid((nq + 3) / 4), 256, 0, st>>>(
          reinterpret_cast<const ulonglong2*>(keys64), nq, seed, n, (uint64_t)nparts, part2,
          entries, bcount, seeds32, reinterpret_cast<longlong2*>(out));
    }
  } else {
    // large batches: hash all keys first (the fused kernel's per-thread byte
    // loads thrash L1/L2 next to the seed gathers: 8.9 GB of DRAM reads for
    // 5.5 GB of key bytes at C5), then the shared-table query over the hashes
    const size_t sh = sizeof(double2) * BUCKET_TAB + sizeof(uint32_t) * (size_t)(nparts + 1);
    int dev = 0, optin = 0;
    PHB_CUDA_TRY(cudaGetDevice(&dev));
    PHB_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
#ifndef PHB_NO_Q2PASS
    if (key_off && sh <= (size_t)optin && nq >= (int64_t)num_sms() * 4096 &&
        (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
      // chunks of QCH keys: a pooled 512 MB scratch (the pool keeps 1 GB)
      constexpr int64_t QCH = 32ll << 20;
      const int64_t ch = nq < QCH ? nq : QCH;
      ulonglong2* hp = nullptr;
      PHB_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&hp), sizeof(ulonglong2) * (size_t)ch, st));
      PHB_CUDA_TRY(cudaFuncSetAttribute(k_query32s_u64x4<true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
      for (int64_t c0 = 0; c0 < nq; c0 += ch) {
        const int64_t c = nq - c0 < ch ? nq - c0 : ch;
        note_launch(), k_hash_pairs<<<qgrid(c), 256, 0, st>>>(buf, offsets + c0, c, seed, hp);
        PHB_CUDA_TRY(cudaGetLastError());
        note_launch(), k_query32s_u64x4<true><<<num_sms(), 1024, sh, st>>>(
            hp, c, seed, n, (uint64_t)nparts, key_off, entries, bcount, seeds32,
            reinterpret_cast<longlong2*>(out + c0));
        PHB_CUDA_TRY(cudaGetLastError());
      }
      PHB_CUDA_TRY(cudaFreeAsync(hp, st));
      return 0;
    }
#endif
    note_launch(), k_query32_bytes<<<qgrid(nq), 256, 0, st>>>(buf, offsets, nq, seed, n,
                                                              (uint64_t)nparts, part2, entries,
                                                              bcount, seeds32, out);
  }
  return (int)cudaGetLastError();
}

int launch_part_table32(const int64_t* key_off, int64_t nparts, uint2* part2, cudaStream_t st) {
  if (nparts <= 0) return 0;
  note_launch(), k_part_table32<<<qgrid(nparts), 256, 0, st>>>(key_off, nparts, part2);
  return (int)cudaGetLastError();
}

int launch_seed_table32(const uint64_t* seeds, const int64_t* key_off, int64_t nparts,
                        int64_t count, uint32_t* out, uint32_t* overflow, cudaStream_t st) {
  if (count <= 0) return 0;
  note_launch(), k_seed_table32<<<qgrid(count), 256, 0, st>>>(seeds, key_off, nparts, count, out,
                                                              overflow);
  return (int)cudaGetLastError();
}

int launch_query_encoded(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64,
                         int64_t nq, uint64_t seed, int64_t n, int64_t nparts,
                         const int64_t* key_off, const double* entries, uint32_t bcount,
                         const uint8_t* section, const int64_t* cols, int mono,
                         const uint32_t* dsel, int64_t dstride, int64_t* out, cudaStream_t st) {
  if (nq <= 0) return 0;
  const int g = qgrid(nq);
  const ECol* c = reinterpret_cast<const ECol*>(cols);
  const size_t sh = sizeof(double2) * BUCKET_TAB + sizeof(ulonglong2) * bcount +
                    sizeof(uint32_t) * (size_t)(nparts + 1);
  // compact descriptors: payload byte offsets below 2^32 (n < 2^29 keys bounds
  // the section by 8 bytes per seed entry, i.e. below 4 GB)
  const size_t sh32 = sizeof(double2) * BUCKET_TAB + sizeof(uint2) * ((bcount + 1) & ~1u) +
                      sizeof(uint64_t) * QGT_N + sizeof(uint32_t) * (size_t)(nparts + 1);
  int dev = 0, optin = 0;
  PHB_CUDA_TRY(cudaGetDevice(&dev));
  PHB_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
#ifdef PHB_NO_C32
  const bool c32 = false;
#else
  const bool c32 = n < ((int64_t)1 << 29) && sh32 <= (size_t)optin;
#endif
  // large u64 batches of an interleaved section without a select directory
  // (no Rice column: IC-C) take the shared-table kernel; Rice selects keep
  // the many-CTA kernel, whose occupancy hides their scan latency better
  if (keys64 && !mono && !dsel && n < ((int64_t)1 << 32) && (c32 || sh <= (size_t)optin) &&
      nq >= (int64_t)num_sms() * 4096 && (reinterpret_cast<uintptr_t>(keys64) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    if (c32) {
      PHB_CUDA_TRY(cudaFuncSetAttribute(k_query_enc_s<true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
      note_launch(), k_query_enc_s<true><<<num_sms(), 1024, sh32, st>>>(
          reinterpret_cast<const ulonglong2*>(keys64), nq, seed, n, (uint64_t)nparts, key_off,
          entries, bcount, section, c, dsel, dstride, reinterpret_cast<longlong2*>(out));
    } else {
      PHB_CUDA_TRY(cudaFuncSetAttribute(k_query_enc_s<false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
      note_launch(), k_query_enc_s<false><<<num_sms(), 1024, sh, st>>>(
          reinterpret_cast<const ulonglong2*>(keys64), nq, seed, n, (uint64_t)nparts, key_off,
          entries, bcount, section, c, dsel, dstride, reinterpret_cast<longlong2*>(out));
    }
  } else if (keys64)
    note_launch(), k_query_enc<0><<<g, 256, 0, st>>>(buf, offsets, keys64, nq, seed, n, (uint64_t)nparts, key_off,
                                      entries, bcount, section, c, mono, dsel, dstride, out);
  else
    note_launch(), k_query_enc<1><<<g, 256, 0, st>>>(buf, offsets, keys64, nq, seed, n, (uint64_t)nparts, key_off,
                                      entries, bcount, section, c, mono, dsel, dstride, out);
  return (int)cudaGetLastError();
}

int launch_select_index(const uint8_t* section, const int64_t* cols, int64_t ncols,
                        int64_t stride, uint32_t* dsel, cudaStream_t st) {
  if (ncols <= 0) return 0;
  note_launch(), k_select_index<<<(unsigned)ncols, 256, 0, st>>>(section, reinterpret_cast<const ECol*>(cols),
                                                  stride, dsel);
  return (int)cudaGetLastError();
}

int launch_verify(const int64_t* out, int64_t nq, int64_t n, uint32_t* bitmap, uint32_t* bad,
                  cudaStream_t st) {
  if (nq <= 0) return 0;
  note_launch(), k_verify<<<qgrid(nq), 256, 0, st>>>(out, nq, n, bitmap, bad);
  return (int)cudaGetLastError();
}

}  // namespace phb
