// K4 search: per-partition bucket grouping, bucket ordering and the seed
// search, one warp per partition.
//
// Replaces build_partition_range (_kernels.py:221-371) and its oracle
// build_partition (builder.py:199-221). The result is the reference's
// sequential first-fit, bit for bit: for every bucket (in the order of
// _kernels.py:268-282) the smallest p = s*m + d such that the bucket's keys
// land on pairwise distinct free slots, plus the reference's trial count
// (one unit per key per tested (s, d) candidate, _kernels.py:330-369).
//
// Design (B200):
//  * One warp owns one partition; partitions come from a global atomic
//    work queue, so heavy-tailed partitions (bucket 1 birthday searches,
//    SURVEY.md §0 finding 7) load-balance dynamically across the resident
//    warps. No __syncthreads anywhere: warps are independent.
//  * Per-warp shared memory holds only bitmaps and bucket metadata
//    (~5 KB at lambda = 9): a doubled occupancy bitmap (2m bits, so a cyclic
//    window is one funnel shift), an m-bit self-collision scratch map,
//    bucket sizes / offsets, the processing order and the current bucket's
//    base positions. Keys stay in L1/L2 (bucket-grouped scratch `glo`).
//  * Displacement search is bit-parallel: valid(d) = AND_i free(p_i + d).
//    A lane owns consecutive 32-bit words of the valid mask (single-seed
//    steps: 3 words per lane, 96 words = 3072 displacements per pass); keys
//    are swept in pairs, both windows OR-ed into the accumulator with one
//    3-input LOP3 per word (2 funnel shifts + 1 LOP3 per pair-word); a
//    ballot + ffs picks the smallest d. No early exit on saturated windows
//    (measured: the check costs more than it saves at every lambda).
//  * Small buckets test G seeds per step (G = 4 for k <= 8 with 88-word
//    windows, 2 for k <= 16 with 96-word windows), one lane group per seed;
//    the batched instantiations are lean (seeds >= 1 below the cap,
//    closed-form resolution in 32-bit arithmetic), the single-seed one keeps
//    seed 0's duplicate check and the cap. Per-seed hashes of the first 4096
//    seeds come from a compile-time table.
//  * Self-collision of a candidate s: __match_any_sync on positions for
//    k <= 32, shared-memory atomicOr test-and-set for larger buckets.
//  * Trials use the closed form k * (S_self + sum_fail(dmax+1) + d* + 1),
//    identical to the reference's per-candidate counting.
//  * Bound: SM issue (74%), with the shared LSU (78%) and the ALU pipe (68%)
//    next, not HBM (profiles/search_sm_c2.json); measured alternatives in
//    DESIGN.md §3.
#include <cstdio>
#include "common.cuh"
#include "phobic_internal.h"

namespace phb {

// Register budget: CTAs of 4 warps per SM (8 -> 64 registers, 32 warps/SM).
// Variants measured at C2 (tools/variant_bench.py) are listed with their
// times in DESIGN.md §3.
#ifndef PHB_MINB
#define PHB_MINB 8
#endif
// The per-seed hash mix64(s ^ POSITION_SALT) (_kernels.py:330) for the first
// GTAB_N seeds, computed at compile time: one L1-resident load per batch
// lane instead of a 64-bit mix (seeds at C2 stay below ~3,500).
constexpr int GTAB_N = 4096;
struct SeedHashTable {
  uint64_t v[GTAB_N];
};
constexpr SeedHashTable make_seed_hashes() {
  SeedHashTable t{};
  for (int s = 0; s < GTAB_N; ++s) t.v[s] = mix64((uint64_t)s ^ POSITION_SALT);
  return t;
}
__device__ const SeedHashTable g_seed_hash = make_seed_hashes();

__device__ __forceinline__ uint64_t seed_hash(int64_t s) {
  return s < GTAB_N ? __ldg(&g_seed_hash.v[s]) : mix64((uint64_t)s ^ POSITION_SALT);
}

// window words of the batched seed steps (multiples of 8 / 16 lanes; a
// partition takes the G = 4 / G = 2 step only if its m bits fit the window)
#ifndef PHB_W4
#define PHB_W4 88  // C2 search 23.26 -> 23.00 ms (m_max ~2,700 < 2,816 bits)
#endif
#ifndef PHB_W2
#define PHB_W2 96
#endif
constexpr int W4 = PHB_W4, W2 = PHB_W2;
#ifndef PHB_PRO_D
#define PHB_PRO_D 4  // prologue records in flight per lane
#endif
constexpr int PRO_D = PHB_PRO_D;
constexpr int SH = 256;     // size classes of the counting-sort bucket order
constexpr int PMAX = 256;   // bucket sizes whose base positions are staged in smem
#ifndef PHB_WARPS
#define PHB_WARPS 4
#endif
constexpr int WARPS = PHB_WARPS;  // warps (= partitions in flight) per CTA
constexpr unsigned FULL = 0xffffffffu;

// Per-warp shared-memory plan, in 32-bit words.
struct SmemPlan {
  int occ_w, scr_w, cnt_w, ord_w, sh_w, pos_w, total_w;
};

__host__ __device__ inline SmemPlan smem_plan(int64_t m_max, uint32_t bcount) {
  SmemPlan p;
  // reads reach word (m-1)/32 + 3*31 + 3 of a pass, marks reach bit 2m - 1
  p.occ_w = (int)((2 * m_max) / 32 + 104);
  p.scr_w = (int)((m_max / 32 + 3) & ~1);  // even: 8-byte aligned sweep entries follow
  p.cnt_w = (int)bcount + 1;  // cnt and endp each
  p.ord_w = (int)(bcount + 2) / 2;
  p.sh_w = SH;       // shist + srun as u16
  p.pos_w = PMAX / 2;  // u16 base positions (generic) or u32 sweep entries (k <= 32)
  p.occ_w = (p.occ_w + 3) & ~3;  // keep the mask table that follows 16-byte aligned
  // the bucket-order scratch (shist/srun) is dead before the search state
  // (mask table, collision map, positions) is written: they share one region
  const int search_w = 96 + p.scr_w + p.pos_w;
  // the mask table (first word of the search union) 16-byte aligned for vector loads
  p.ord_w = ((p.occ_w + 2 * p.cnt_w + p.ord_w + 3) & ~3) - p.occ_w - 2 * p.cnt_w;
  p.total_w = p.occ_w + 2 * p.cnt_w + p.ord_w + (p.sh_w > search_w ? p.sh_w : search_w);
  p.total_w = (p.total_w + 3) & ~3;  // 16-byte aligned warp regions (LDS.128)
  return p;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

__device__ __forceinline__ uint32_t warp_max(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

extern __shared__ uint32_t smem[];

#ifdef PHB_STATS
// [0] G=1 batches [1] G=2 batches [2] G=4 batches [3] small key-steps
// [4] generic s-iterations [5] generic key-rounds [6] singletons [7] buckets k>=2
// [8] early exits [9] generic d-searches
// [10] cycles: prologue (histogram, grouping, order) [11] singletons
// [12] small k (<= 32) [13] generic (k > 32 or m > 3072) [14] queue + output
// [16..18] cycles for k in 2..8 / 9..16 / 17..32, [19..21] their bucket counts,
// [22..24] their seeds tested (s* + 1)
// Counters live per warp in shared memory (lane 0 only, no contention) and
// are flushed to g_stats once per warp at kernel exit, so the counting does
// not perturb the timings it records.
__device__ unsigned long long g_stats[32];
__shared__ unsigned long long s_stats[4][32];
#define STAT(i, v) do { if ((threadIdx.x & 31) == 0) s_stats[threadIdx.x >> 5][i] += (unsigned long long)(v); } while (0)
#define TSTAMP(t) const long long t = clock64()
#define TACC(i, t0) STAT(i, clock64() - (t0))
#else
#define STAT(i, v) do { } while (0)
#define TSTAMP(t) do { } while (0)
#define TACC(i, t0) do { } while (0)
#endif

__device__ __forceinline__ void mark(uint32_t occ, uint32_t slot, uint32_t m, int tag = 0) {
#ifdef PHB_DEBUG
  if (slot >= m) { printf("mark: slot %u m %u tag %d\n", slot, m, tag); __trap(); }
  if (smem[occ + (slot >> 5)] & (1u << (slot & 31))) { printf("mark: slot %u already taken (m %u) tag %d\n", slot, m, tag); __trap(); }
#endif
  atomicOr(&smem[occ + (slot >> 5)], 1u << (slot & 31));
  const uint32_t s2 = slot + m;
  atomicOr(&smem[occ + (s2 >> 5)], 1u << (s2 & 31));
}

// Processing order of the non-empty buckets (_kernels.py:268-282):
// size descending, ties by `tie` descending where tie = b ("asc-expected",
// tie_desc = 1) or B - b. Returns the number of non-empty buckets.
__device__ uint32_t bucket_order(uint32_t cnt, uint32_t B, int tie_desc, uint32_t maxsz,
                                 uint16_t* order, uint16_t* shist, uint16_t* srun, int lane) {
  if (maxsz < (uint32_t)SH) {
#pragma unroll 1
    for (int s = lane; s < SH; s += 32) shist[s] = 0, srun[s] = 0;
    __syncwarp();
#pragma unroll 1
    for (uint32_t c0 = 1; c0 <= B; c0 += 32) {
      uint32_t b = c0 + lane;
      uint32_t sz = b <= B ? smem[cnt + b] : 0u;
      uint32_t peers = __match_any_sync(FULL, sz);
      if (sz > 0 && lane == __ffs(peers) - 1) shist[sz] += (uint16_t)__popc(peers);
      __syncwarp();
    }
    // base[s] = number of buckets with size > s
    uint32_t run = 0;
#pragma unroll 1
    for (int c = 0; c < SH / 32; ++c) {
      int s = SH - 1 - (c * 32 + lane);
      uint32_t v = shist[s];
      uint32_t inc = warp_incl_scan(v, lane);
      __syncwarp();
      shist[s] = (uint16_t)(run + inc - v);
      run += __shfl_sync(FULL, inc, 31);
    }
    __syncwarp();
#pragma unroll 1
    for (uint32_t c0 = 0; c0 < B; c0 += 32) {
      uint32_t idx = c0 + lane;
      uint32_t b = tie_desc ? (B - idx) : (idx + 1);
      uint32_t sz = idx < B ? smem[cnt + b] : 0u;
      uint32_t peers = __match_any_sync(FULL, sz);
      if (sz > 0) order[shist[sz] + srun[sz] + __popc(peers & lanemask_lt())] = (uint16_t)b;
      __syncwarp();
      if (sz > 0 && lane == __ffs(peers) - 1) srun[sz] += (uint16_t)__popc(peers);
      __syncwarp();
    }
    return run;
  }
  // general path (some bucket holds >= SH keys): rank by direct comparison
  uint32_t nb = 0;
#pragma unroll 1
  for (uint32_t c0 = 1; c0 <= B; c0 += 32) {
    uint32_t b = c0 + lane;
    uint32_t sz = b <= B ? smem[cnt + b] : 0u;
    if (sz > 0) {
      uint64_t key = (uint64_t)sz * (B + 1) + (tie_desc ? b : B - b);
      uint32_t rank = 0;
#pragma unroll 1
      for (uint32_t b2 = 1; b2 <= B; ++b2) {
        uint32_t s2 = smem[cnt + b2];
        uint64_t k2 = (uint64_t)s2 * (B + 1) + (tie_desc ? b2 : B - b2);
        rank += (s2 > 0 && k2 > key);
      }
      order[rank] = (uint16_t)b;
    }
    nb += __popc(__ballot_sync(FULL, sz > 0));
  }
  __syncwarp();
  return nb;
}

// First displacement d in [0, dmax] with every key's slot free, or -1.
// Base positions come from the staged u16 list (k <= PMAX) or are re-derived
// from the key scratch (larger buckets).
__device__ int64_t find_d(uint32_t occ, const uint16_t* pos16, uint32_t k,
                                          int64_t dmax, const uint64_t* kl, uint64_t g,
                                          uint32_t m, int lane) {
  const uint32_t nwd = (uint32_t)((dmax + 32) >> 5);  // words of the valid mask
#pragma unroll 1
  for (uint32_t g0 = 0; g0 < nwd; g0 += 96) {
    const uint32_t wb = g0 + 3u * lane;
    uint32_t a0 = 0, a1 = 0, a2 = 0;
#pragma unroll 1
    for (uint32_t i = 0; i < k; ++i) {
      const uint32_t p = k <= (uint32_t)PMAX ? (uint32_t)pos16[i] : position(kl[i], g, m);
      const uint32_t W = occ + (p >> 5) + wb;
      const uint32_t sh = p & 31;
      const uint32_t x0 = smem[W], x1 = smem[W + 1], x2 = smem[W + 2], x3 = smem[W + 3];
      a0 |= __funnelshift_r(x0, x1, sh);
      a1 |= __funnelshift_r(x1, x2, sh);
      a2 |= __funnelshift_r(x2, x3, sh);
      if ((i & 3) == 3 && __all_sync(FULL, (a0 & a1 & a2) == FULL)) break;
    }
    // restrict to d <= dmax; lanes past the end contribute nothing
    uint32_t v0 = ~a0, v1 = ~a1, v2 = ~a2;
    const int64_t lim = dmax - 32 * (int64_t)wb;  // last valid bit index in word wb
    if (lim < 95) {
      v0 = lim < 0 ? 0u : (lim < 31 ? v0 & ((2u << lim) - 1u) : v0);
      v1 = lim < 32 ? 0u : (lim < 63 ? v1 & ((2u << (lim - 32)) - 1u) : v1);
      v2 = lim < 64 ? 0u : (lim < 95 ? v2 & ((2u << (lim - 64)) - 1u) : v2);
    }
    const uint32_t bal = __ballot_sync(FULL, (v0 | v1 | v2) != 0);
    if (bal) {
      const int l = __ffs(bal) - 1;
      const uint32_t t = v0 ? 0u : (v1 ? 1u : 2u);
      const uint32_t vv = v0 ? v0 : (v1 ? v1 : v2);
      const uint32_t word = __shfl_sync(FULL, t, l);
      const uint32_t bits = __shfl_sync(FULL, vv, l);
      return 32 * (int64_t)(g0 + 3u * l + word) + (__ffs(bits) - 1);
    }
  }
  return -1;
}


// find_d for buckets of k >= 2 keys, keys swept in pairs: both windows are
// OR-ed into the accumulators with one 3-input LOP3 per word (as in
// small_bucket); an odd k repeats its last key (OR is idempotent).
__device__ int64_t find_d_pairs(uint32_t occ, const uint16_t* pos16, uint32_t k, int64_t dmax,
                                const uint64_t* kl, uint64_t g, uint32_t m, int lane) {
  const uint32_t nwd = (uint32_t)((dmax + 32) >> 5);
#pragma unroll 1
  for (uint32_t g0 = 0; g0 < nwd; g0 += 96) {
    const uint32_t wb = g0 + 3u * lane;
    uint32_t a0 = 0, a1 = 0, a2 = 0;
#pragma unroll 1
    for (uint32_t i = 0; i < k; i += 2) {
      const uint32_t i2 = i + 1 < k ? i + 1 : i;
      const uint32_t pa = k <= (uint32_t)PMAX ? (uint32_t)pos16[i] : position(kl[i], g, m);
      const uint32_t pb = k <= (uint32_t)PMAX ? (uint32_t)pos16[i2] : position(kl[i2], g, m);
      const uint32_t Wa = occ + (pa >> 5) + wb, Wb = occ + (pb >> 5) + wb;
      const uint32_t sa = pa & 31, sb = pb & 31;
      const uint32_t x0 = smem[Wa], x1 = smem[Wa + 1], x2 = smem[Wa + 2], x3 = smem[Wa + 3];
      const uint32_t y0 = smem[Wb], y1 = smem[Wb + 1], y2 = smem[Wb + 2], y3 = smem[Wb + 3];
      a0 |= __funnelshift_r(x0, x1, sa) | __funnelshift_r(y0, y1, sb);
      a1 |= __funnelshift_r(x1, x2, sa) | __funnelshift_r(y1, y2, sb);
      a2 |= __funnelshift_r(x2, x3, sa) | __funnelshift_r(y2, y3, sb);
      // (no saturation exit: measured 1.5% slower with it, like the batched sweeps)
    }
    uint32_t v0 = ~a0, v1 = ~a1, v2 = ~a2;
    const int64_t lim = dmax - 32 * (int64_t)wb;
    if (lim < 95) {
      v0 = lim < 0 ? 0u : (lim < 31 ? v0 & ((2u << lim) - 1u) : v0);
      v1 = lim < 32 ? 0u : (lim < 63 ? v1 & ((2u << (lim - 32)) - 1u) : v1);
      v2 = lim < 64 ? 0u : (lim < 95 ? v2 & ((2u << (lim - 64)) - 1u) : v2);
    }
    const uint32_t bal = __ballot_sync(FULL, (v0 | v1 | v2) != 0);
    if (bal) {
      const int l = __ffs(bal) - 1;
      const uint32_t t = v0 ? 0u : (v1 ? 1u : 2u);
      const uint32_t vv = v0 ? v0 : (v1 ? v1 : v2);
      const uint32_t word = __shfl_sync(FULL, t, l);
      const uint32_t bits = __shfl_sync(FULL, vv, l);
      return 32 * (int64_t)(g0 + 3u * l + word) + (__ffs(bits) - 1);
    }
  }
  return -1;
}

// Outcome of one bucket's search.
struct BucketResult {
  int64_t seed, trials;
  int status;  // 0 found, 1 duplicate low words, 2 seed cap
};

// Generic single-s search (any k, any m): the reference loop of
// _kernels.py:312-369 with each s tested by the whole warp.
__device__ BucketResult generic_bucket(uint32_t occ, uint32_t scr, uint16_t* pos16, uint32_t k,
                                       const uint64_t* kl, uint32_t m, int64_t cap,
                                       int64_t s_begin, int64_t trials, int lane) {
  const uint32_t R = (k + 31) >> 5;
  const uint32_t amask = k >= 32 ? FULL : ((1u << k) - 1u);
  const uint64_t key0 = (uint32_t)lane < k ? kl[lane] : 0ull;
  const uint32_t scr_used = m / 32 + 2;
  uint32_t p0 = 0;  // this lane's base position (k <= 32)
#pragma unroll 1
  for (int64_t s = s_begin;; ++s) {
    STAT(4, 1);
    STAT(5, (k + 31) / 32);
    const int64_t pbase = s * (int64_t)m;
    if (s > 0 && pbase > cap) return {0, trials, 2};  // _kernels.py:324-328
    const uint64_t g = seed_hash(s);
    bool coll = false;
    uint32_t cmask = 0;  // per-round collision flags (s = 0 duplicate check)
    __syncwarp();  // the previous candidate's find_d reads of pos16 precede this seed's writes
    if (k <= 32) {
      p0 = position(key0, g, m);
      const uint32_t peers = __match_any_sync(FULL, p0) & amask;
      coll = __any_sync(FULL, (uint32_t)lane < k && __popc(peers) > 1);
      if (!coll && (uint32_t)lane < k) pos16[lane] = (uint16_t)p0;
    } else {
#pragma unroll 1
      for (uint32_t r = 0; r < R; ++r) {
        const uint32_t i = 32u * r + lane;
        bool c = false;
        if (i < k) {
          const uint32_t p = position(kl[i], g, m);
          const uint32_t bit = 1u << (p & 31);
          c = (atomicOr(&smem[scr + (p >> 5)], bit) & bit) != 0;
          if (i < (uint32_t)PMAX) pos16[i] = (uint16_t)p;
        }
        if (r < 32) cmask |= (uint32_t)c << r;
        if (__any_sync(FULL, c)) {
          coll = true;
          if (s > 0) break;  // s = 0 inserts every key for the dup check
        }
      }
      __syncwarp();
#pragma unroll 1
      for (uint32_t w = lane; w < scr_used; w += 32) smem[scr + w] = 0;
    }
    __syncwarp();
    if (s == 0) {
      // duplicate low words collide at every s, so they can only exist if
      // s = 0 collides (_kernels.py:312-319)
      if (coll) {
        bool dup = false;
        if (k <= 32) {
          const uint32_t peers = __match_any_sync(FULL, key0) & amask;
          dup = (uint32_t)lane < k && __popc(peers) > 1;
        } else if (R <= 32) {
          // a duplicate pair's later key found its slot taken: compare every
          // key that collided against the whole bucket
#pragma unroll 1
          for (uint32_t r = 0; r < R; ++r) {
            uint32_t bal = __ballot_sync(FULL, (cmask >> r) & 1u);
            while (bal) {
              const uint32_t src = 32u * r + (__ffs(bal) - 1);
              bal &= bal - 1;
              const uint64_t v = kl[src];
#pragma unroll 1
              for (uint32_t i2 = lane; i2 < k; i2 += 32)
                if (i2 != src && kl[i2] == v) dup = true;
            }
          }
        } else {
#pragma unroll 1
          for (uint32_t i = 0; i < k; ++i) {
            const uint64_t v = kl[i];
#pragma unroll 1
            for (uint32_t i2 = lane; i2 < k; i2 += 32)
              if (i2 != i && kl[i2] == v) dup = true;
          }
        }
        if (__any_sync(FULL, dup)) return {0, trials, 1};
      }
      if (pbase > cap) return {0, trials, 2};
    }
    if (coll) {
      trials += k;
      continue;
    }
    int64_t dmax = cap - pbase;
    if (dmax > (int64_t)m - 1) dmax = (int64_t)m - 1;
    const int64_t d = find_d_pairs(occ, pos16, k, dmax, kl, g, m, lane);
    if (d >= 0) {
      trials += (int64_t)k * (d + 1);
#pragma unroll 1
      for (uint32_t i = lane; i < k; i += 32) {
        const uint32_t p =
            k <= 32 ? p0 : (i < (uint32_t)PMAX ? (uint32_t)pos16[i] : position(kl[i], g, m));
        uint32_t slot = p + (uint32_t)d;
        if (slot >= m) slot -= m;
        mark(occ, slot, m, 2000 + (int)k);
      }
      return {pbase + d, trials, 0};
    }
    trials += (int64_t)k * (dmax + 1);
  }
}

// A key's sweep entry (u32, in the position area): bits 0-4 the funnel shift
// p & 31 (SHF.R.W reads only those bits), bits 7 and up the byte offset of
// its first bitmap word, 4 (p >> 5), shifted left by 5. The word address is
// then one LEA.HI off the lane's base and the shift needs no mask; a pair of
// entries is one LDS.64 (C2 search 22.1 -> 21.7 ms: 5 fewer instructions per
// key pair against u16 base positions).
__device__ __forceinline__ uint32_t sweep_entry(uint32_t p) { return ((p >> 5) << 7) | (p & 31u); }

// One pair of keys OR-ed into a lane's WPL accumulator words: word t gets
// funnel(occ[r + wb + t], occ[r + wb + t + 1], p & 31) of both keys
// (r = p >> 5, ob = the byte address of occ[wb]). Keys in pairs: both windows
// go into the accumulator with one 3-input LOP3 per word (2 funnel shifts +
// 1 LOP3 per pair-word instead of 2 shifts + 2 ORs).
template <int WPL>
__device__ __forceinline__ void sweep_pair(uint32_t (&acc)[WPL], const char* ob, uint32_t ea,
                                           uint32_t eb) {
  const uint32_t* const Wa = reinterpret_cast<const uint32_t*>(ob + (ea >> 5));
  const uint32_t* const Wb = reinterpret_cast<const uint32_t*>(ob + (eb >> 5));
  uint32_t xa = Wa[0], xb = Wb[0];
#pragma unroll
  for (int t = 0; t < WPL; ++t) {
    const uint32_t ya = Wa[t + 1], yb = Wb[t + 1];
    acc[t] |= __funnelshift_r(xa, ya, ea) | __funnelshift_r(xb, yb, eb);
    xa = ya;
    xb = yb;
  }
}

// Batched search for small buckets (k <= 32 / G) in partitions with
// m <= 3072: G consecutive seeds s are tested per step, one group of
// L = 32 / G lanes per seed, each lane owning WPL = 96 / L consecutive
// words of that seed's valid mask (WPL + 1 shared loads per key). The
// groups are then resolved in seed order exactly like the sequential loop,
// so seeds and trials are unchanged. G = 1 steps resolve seed by seed
// (seed 0's duplicate check, the seed cap); G > 1 batches only ever run on
// seeds >= 1 whose whole displacement range is below the cap, and resolve in
// closed form (a lean instantiation: -6% search time at C2 against the
// generic resolution); anything else is left to G = 1 steps. Returns
// status -1 when max_batches ran out (or the batch would need the generic
// resolution) without a decision; the caller continues.
template <int G, int W = 96>
__device__ BucketResult small_bucket(uint32_t occ, uint32_t dmask, uint16_t* pos16, uint32_t k,
                                     const uint64_t* kl, uint32_t m, int64_t cap,
                                     int64_t& s_next, int64_t trials, int max_batches,
                                     int lane) {
  constexpr int L = 32 / G, WPL = W / L;  // W: window words per seed (W >= (m + 31) / 32)
  static_assert(W % L == 0 && W <= 96, "window");
  constexpr uint32_t LMASK = L == 32 ? FULL : ((1u << L) - 1u);
  const int grp = lane / L, gl = lane % L;
  const bool act = (uint32_t)gl < k;
  const uint64_t key = act ? kl[gl] : 0ull;
  uint32_t* const mye = reinterpret_cast<uint32_t*>(pos16) + grp * L;  // sweep entries
  const uint32_t wb = (uint32_t)gl * WPL;
  const char* const ob = reinterpret_cast<const char*>(smem + occ + wb);
#pragma unroll 1
  for (int bt = 0; bt < max_batches; ++bt) {
    if constexpr (G > 1) {
      // batches never see seed 0 or the seed cap: those go to the
      // single-seed instantiation, which keeps the seed-by-seed resolution
      // (a gate that let batches start at seed 0 measured 9% slower)
      if (s_next < 1 || (s_next + G) * (int64_t)m - 1 > cap) return {0, trials, -1};
    }
    STAT(G == 1 ? 0 : (G == 2 ? 1 : 2), 1);
    const int64_t s = s_next + grp;
    const uint64_t g = seed_hash(s);
    const uint32_t p = position(key, g, m);
    const uint32_t tag = act ? (((uint32_t)grp << 16) | p) : (0x80000000u | (uint32_t)lane);
    // every lane must execute the vote (no short-circuit around it)
    const uint32_t tpeers = __match_any_sync(FULL, tag);
    const uint32_t cball = __ballot_sync(FULL, act && __popc(tpeers) > 1);
    if (act) mye[gl] = sweep_entry(p);
    // keys are swept in pairs: an odd k repeats its last key (OR is idempotent)
    if ((k & 1u) && (uint32_t)gl == k - 1) mye[k] = sweep_entry(p);
    __syncwarp();
    const bool gcoll = ((cball >> (grp * L)) & LMASK) != 0;
    const int64_t pbase = s * (int64_t)m;
    int64_t dmax = cap - pbase;
    if (dmax > (int64_t)m - 1) dmax = (int64_t)m - 1;
    const bool dead_group = gcoll || pbase > cap;
    // start from "displacements past dmax are occupied": the partition's
    // mask table (dmax = m - 1) or, near the seed cap, computed here
    uint32_t acc[WPL];
    if (G > 1) {
      // a self-colliding group (rare) is masked out after the sweep instead
      // vector loads of the mask table (3 LDS.128 instead of 12 LDS at G = 4)
      if constexpr (WPL % 4 == 0) {
        const uint4* src = reinterpret_cast<const uint4*>(smem + dmask + wb);
#pragma unroll
        for (int t = 0; t < WPL / 4; ++t) {
          const uint4 v = src[t];
          acc[4 * t] = v.x, acc[4 * t + 1] = v.y, acc[4 * t + 2] = v.z, acc[4 * t + 3] = v.w;
        }
      } else if constexpr (WPL % 2 == 0) {
        const uint2* src = reinterpret_cast<const uint2*>(smem + dmask + wb);
#pragma unroll
        for (int t = 0; t < WPL / 2; ++t) {
          const uint2 v = src[t];
          acc[2 * t] = v.x, acc[2 * t + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int t = 0; t < WPL; ++t) acc[t] = smem[dmask + wb + t];
      }
    } else if (dmax == (int64_t)m - 1) {
#pragma unroll
      for (int t = 0; t < WPL; ++t) acc[t] = dead_group ? FULL : smem[dmask + wb + t];
    } else {
      const int64_t lim = dmax - 32 * (int64_t)wb;
#pragma unroll
      for (int t = 0; t < WPL; ++t) {
        const int64_t lt = lim - 32 * t;
        acc[t] = (dead_group || lt < 0) ? FULL : (lt < 31 ? ~((2u << lt) - 1u) : 0u);
      }
    }
    // Keys in pairs (sweep_pair); the next pair's entries are loaded one
    // iteration ahead.
    // No early exit on saturated windows: buckets of k <= 32 keys rarely
    // saturate every lane before their last pair, and the check (an AND over
    // the window plus a vote every other pair) cost more than it saved
    // (C2 search: lambda = 9 -1%, lambda = 7 -5% without it).
    const uint2* const me2 = reinterpret_cast<const uint2*>(mye);
    uint2 ee = me2[0];
#pragma unroll 1
    for (uint32_t i = 0; i < k; i += 2) {
      STAT(3, 2);
      const uint32_t ea = ee.x, eb = ee.y;
      // the next pair's entries; past the last pair this reads a spare
      // entry of the (128-entry) position area, never used
      ee = me2[(i >> 1) + 1];
      sweep_pair<WPL>(acc, ob, ea, eb);
    }
    // this lane's first valid displacement (d <= dmax), or -1
    uint32_t sat = FULL;
#pragma unroll
    for (int t = 0; t < WPL; ++t) sat &= acc[t];
    const bool hv = sat != FULL && !(G > 1 && gcoll);
    const uint32_t fball = __ballot_sync(FULL, hv);
    // this lane's first free displacement, 32-bit (only a lane with hv is read)
    uint32_t myd = 0;
    if (fball) {
      uint32_t tw = 0, vv = FULL;
#pragma unroll
      for (int t = WPL - 1; t >= 0; --t)
        if (acc[t] != FULL) tw = (uint32_t)t, vv = acc[t];
      myd = 32u * (wb + tw) + (uint32_t)(__ffs(~vv) - 1);
    }
    if constexpr (G > 1) {
      // closed form of the sequential loop: seeds before the first group with
      // a valid displacement self-collided (k trials) or swept m (k*m)
      // one bit per self-collided group, without a loop of compares (-1.7%)
      uint32_t collg;
      if constexpr (G == 4)
        collg = ((__vcmpne4(cball, 0u) & 0x01010101u) * 0x01020408u) >> 24;
      else
        collg = (uint32_t)((cball & 0xffffu) != 0u) | ((uint32_t)((cball >> 16) != 0u) << 1);
      const int src = __ffs(fball) - 1;  // first lane with a valid d lies in the first found group
      const int gw = fball ? (int)((uint32_t)src / (uint32_t)L) : G;
      const int ncoll = __popc(collg & ((1u << gw) - 1u));
      // k <= 16, m <= 3072, gw <= 4: every term fits 32 bits
      const uint32_t tr = k * ((uint32_t)ncoll + m * (uint32_t)(gw - ncoll));
      if (src >= 0) {
        const uint32_t d = __shfl_sync(FULL, myd, src);
        trials += (int64_t)(tr + k * (d + 1u));
        if (grp == gw && act) {
          uint32_t slot = p + (uint32_t)d;
          if (slot >= m) slot -= m;
          mark(occ, slot, m, 100 * G + (int)k);
        }
        return {(s_next + gw) * (int64_t)m + d, trials, 0};
      }
      trials += (int64_t)tr;
      s_next += G;
      __syncwarp();
    } else {
      // single-seed step (G = 1): seed 0's duplicate check and the seed cap
      const int64_t si = s_next;
      const int64_t pb = si * (int64_t)m;
      const bool ci = cball != 0;
      if (si > 0 && pb > cap) return {0, trials, 2};
      if (si == 0) {
        if (ci) {
          const uint32_t peers = __match_any_sync(FULL, key) & __ballot_sync(FULL, act);
          const bool dup = act && __popc(peers) > 1;
          if (__any_sync(FULL, dup)) return {0, trials, 1};
        }
        if (pb > cap) return {0, trials, 2};
      }
      if (ci) {
        trials += k;
      } else {
        int64_t dmi = cap - pb;
        if (dmi > (int64_t)m - 1) dmi = (int64_t)m - 1;
        if (fball) {
          const int64_t d = __shfl_sync(FULL, myd, __ffs(fball) - 1);
          trials += (int64_t)k * (d + 1);
          if (act) {
            uint32_t slot = p + (uint32_t)d;
            if (slot >= m) slot -= m;
            mark(occ, slot, m, 100 + (int)k);
          }
          return {pb + d, trials, 0};
        }
        trials += (int64_t)k * (dmi + 1);
      }
      s_next += 1;
      __syncwarp();
    }
  }
  return {0, trials, -1};
}

// Speculative seed-0 step for up to four consecutive small buckets
// (2 <= k <= 8) of the processing order, one 8-lane group each (the
// small_bucket<4> layout: 12 words of the valid mask per lane). Every group
// sweeps seed 0 against the occupancy before the step; the groups are then
// accepted in order: group g keeps its first-fit displacement d_g if it has
// one (and no self-collision) and none of its slots was taken by the
// groups accepted before it in this step. That is exactly the sequential
// result: displacements below d_g were invalid on the old occupancy and
// stay invalid with more slots taken (_kernels.py:312-369; trials k (d + 1)).
// The first group that fails ends the step; its bucket (and the rest) go
// on through the regular path. Returns the number of buckets placed and
// writes their seeds / trials; *tr_out accumulates their trials.
__device__ uint32_t multi_bucket0(const SearchArgs& a, int64_t row, uint32_t occ, uint32_t dmask,
                                  uint16_t* pos16, const uint16_t* order, uint32_t oi, uint32_t nG,
                                  uint32_t cnt, uint32_t endp, const uint64_t* kbase, uint32_t m,
                                  uint64_t g0, int64_t& tr_out, uint32_t& placed, int lane) {
#ifndef PHB_MB_WPL
#define PHB_MB_WPL 11  // 88-word windows like the 4-seed batches (lambda = 5: -1.6%)
#endif
  constexpr int L = 8, WPL = PHB_MB_WPL;  // 8 lanes x WPL words of the seed-0 window
  const int grp = lane >> 3, gl = lane & 7;
  const bool ing = (uint32_t)grp < nG;
  const uint32_t bg = ing ? order[oi + grp] : 0u;
  const uint32_t kg = ing ? smem[cnt + bg] : 0u;
  const bool act = (uint32_t)gl < kg;
  const uint64_t key = act ? kbase[smem[endp + bg] - kg + gl] : 0ull;
  const uint32_t p = position(key, g0, m);
  const uint32_t tag = act ? (((uint32_t)grp << 16) | p) : (0x80000000u | (uint32_t)lane);
  const uint32_t tpeers = __match_any_sync(FULL, tag);
  const uint32_t cball = __ballot_sync(FULL, act && __popc(tpeers) > 1);
  // base positions, every group padded to the largest k (pairs) with its last key
  const uint32_t kmax = __reduce_max_sync(FULL, kg);
  const uint32_t kpad = (kmax + 1u) & ~1u;
  const uint32_t from = kg ? (uint32_t)(grp * L) + min((uint32_t)gl, kg - 1u) : (uint32_t)lane;
  const uint32_t pfill = __shfl_sync(FULL, p, from);
  uint32_t* const mye = reinterpret_cast<uint32_t*>(pos16) + grp * L;  // sweep entries
  if ((uint32_t)gl < kpad) mye[gl] = sweep_entry(pfill);
  __syncwarp();
  const uint32_t wb = (uint32_t)gl * WPL;
  uint32_t acc[WPL];
#pragma unroll
  for (int t = 0; t < WPL; ++t) acc[t] = smem[dmask + wb + t];
  const uint2* const me2 = reinterpret_cast<const uint2*>(mye);
  const char* const ob = reinterpret_cast<const char*>(smem + occ + wb);
#pragma unroll 1
  for (uint32_t i = 0; i < kpad; i += 2) {
    const uint2 ee = me2[i >> 1];
    sweep_pair<WPL>(acc, ob, ee.x, ee.y);
  }
  uint32_t sat = FULL;
#pragma unroll
  for (int t = 0; t < WPL; ++t) sat &= acc[t];
  const bool gcoll = ((cball >> (grp * L)) & 0xffu) != 0;
  const uint32_t fball = __ballot_sync(FULL, ing && sat != FULL && !gcoll);
  uint32_t myd = 0;
  if (fball) {
    uint32_t tw = 0, vv = FULL;
#pragma unroll
    for (int t = WPL - 1; t >= 0; --t)
      if (acc[t] != FULL) tw = (uint32_t)t, vv = acc[t];
    myd = 32u * (wb + tw) + (uint32_t)(__ffs(~vv) - 1);
  }
  // Acceptance of all groups at once: a group's first fit (free before the
  // step) stands unless one of its slots equals a slot of an earlier group of
  // this step (match on the slots); the step accepts groups 0 .. A-1, A the
  // first group without a fit or with such a repeat. (A group-by-group loop
  // of shuffles, shared reads and votes cost 7-13% of the low-lambda search.)
  const uint32_t gbm = (fball >> (grp * L)) & 0xffu;
  const uint32_t dm = __shfl_sync(FULL, myd, gbm ? grp * L + __ffs(gbm) - 1 : lane);
  const bool cand = act && gbm != 0u;
  uint32_t slot = p + dm;
  if (slot >= m) slot -= m;
  const uint32_t stag = cand ? slot : (0x80000000u | (uint32_t)lane);
  const uint32_t speers = __match_any_sync(FULL, stag);
  const bool rep = cand && (speers & ((1u << (grp * L)) - 1u)) != 0u;  // an earlier group's slot
  const uint32_t repb = __ballot_sync(FULL, rep);
  uint32_t stopg = 0;  // groups that stop the step: no fit, or a repeat
#pragma unroll
  for (uint32_t g = 0; g < 4; ++g)
    if (g < nG && (((fball >> (g * L)) & 0xffu) == 0u || ((repb >> (g * L)) & 0xffu) != 0u))
      stopg |= 1u << g;
  const uint32_t accepted = stopg ? (uint32_t)(__ffs(stopg) - 1) : nG;
  const bool acc_g = (uint32_t)grp < accepted;
  if (acc_g && act) mark(occ, slot, m, 500 + (int)kg);
  const int64_t trg = acc_g && gl == 0 ? (int64_t)kg * ((int64_t)dm + 1) : 0;
  if (acc_g && gl == 0) {
    a.seeds[row * a.s_sj + (int64_t)(bg - 1) * a.s_sb] = (uint64_t)dm;
    if (a.trials) a.trials[row * a.s_sj + (int64_t)(bg - 1) * a.s_sb] = trg;
  }
  tr_out += (int64_t)__reduce_add_sync(FULL, (uint32_t)trg);
  placed += __reduce_add_sync(FULL, acc_g && gl == 0 ? kg : 0u);
  __syncwarp();  // the sweep's reads of the base positions precede the next writer's
  return accepted;
}

// The trailing singletons (k = 1 buckets come last in the size-descending
// order), up to 32 per step: a singleton takes the first free slot
// cyclically from its seed-0 base (_kernels.py:300-310), in order. The
// lanes hash the keys in parallel; lane 0 then places them one after the
// other with word scans of the doubled bitmap (a singleton costs ~15
// instructions: the few issue slots of this latency-bound loop leave the
// SM to the other warps). Seeds and trials are written by the lanes.
__device__ void singles0(const SearchArgs& a, int64_t row, uint32_t occ, uint16_t* pos16,
                         const uint16_t* order, uint32_t oi, uint32_t nS, uint32_t endp,
                         const uint64_t* kbase, uint32_t m, uint64_t g0, int64_t& tr_out,
                         int lane) {
  const bool act = (uint32_t)lane < nS;
  const uint32_t b = act ? order[oi + lane] : 0u;
  const uint64_t key = act ? kbase[smem[endp + b] - 1] : 0ull;
  const uint32_t p = position(key, g0, m);
  if (act) pos16[lane] = (uint16_t)p;
  __syncwarp();
  if (lane == 0) {
#pragma unroll 1
    for (uint32_t i = 0; i < nS; ++i) {
      const uint32_t q = pos16[i];
      // first free bit at or after q in the doubled bitmap (one exists in [q, q + m))
      uint32_t w = q >> 5;
      uint32_t bits = ~smem[occ + w] & (FULL << (q & 31));
#pragma unroll 1
      while (!bits) bits = ~smem[occ + (++w)];
      uint32_t slot = 32u * w + (uint32_t)(__ffs(bits) - 1);
      if (slot >= m) slot -= m;
      smem[occ + (slot >> 5)] |= 1u << (slot & 31);  // one writer: plain stores
      const uint32_t s2 = slot + m;
      smem[occ + (s2 >> 5)] |= 1u << (s2 & 31);
      pos16[i] = (uint16_t)(slot >= q ? slot - q : slot + m - q);  // d
    }
  }
  __syncwarp();
  const uint32_t d = act ? (uint32_t)pos16[lane] : 0u;
  if (act) {
    a.seeds[row * a.s_sj + (int64_t)(b - 1) * a.s_sb] = (uint64_t)d;
    if (a.trials) a.trials[row * a.s_sj + (int64_t)(b - 1) * a.s_sb] = (int64_t)d + 1;
  }
  tr_out += (int64_t)__reduce_add_sync(FULL, act ? d + 1u : 0u);
  __syncwarp();
}

// LOWL (low lambda, average bucket below ~7 keys): most buckets fit at seed 0,
// so the per-bucket fixed cost dominates; the trailing singletons go 32 per
// step (singles0) and runs of small buckets 4 per speculative seed-0 step
// (multi_bucket0). A separate instantiation, so the high-lambda kernel keeps
// its instruction footprint (measured: both paths cost ~3% at lambda = 9).
template <bool LOWL>
__global__ void __launch_bounds__(WARPS * 32, PHB_MINB) k_search(SearchArgs a, SmemPlan plan) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t B = a.bcount;
  const uint32_t occ = wid * plan.total_w;
  const uint32_t cnt = occ + plan.occ_w;
  const uint32_t endp = cnt + plan.cnt_w;
  uint16_t* const sm16 = reinterpret_cast<uint16_t*>(smem);
  uint16_t* const order = sm16 + 2 * (endp + plan.cnt_w);
  const uint32_t shared_x = endp + plan.cnt_w + plan.ord_w;  // bucket-order / search union
  uint16_t* const shist = sm16 + 2 * shared_x;
  uint16_t* const srun = shist + SH;
  const uint32_t dmask = shared_x;      // 96-word "past dmax" table for dmax = m - 1
  const uint32_t scr = dmask + 96;      // self-collision map (m bits)
  uint16_t* const pos16 = sm16 + 2 * (scr + plan.scr_w);
  const int64_t nrange = a.p_hi - a.p_lo;
  const uint64_t g0 = mix64(POSITION_SALT);  // s = 0
  const int64_t cap = a.seed_cap;
#ifdef PHB_STATS
  if (lane == 0)
    for (int i = 0; i < 32; ++i) s_stats[wid][i] = 0;
#endif

#pragma unroll 1
  for (;;) {
    TSTAMP(tq);
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(a.queue, 1u);
    t = __shfl_sync(FULL, t, 0);
    if ((int64_t)t >= nrange) {
#ifdef PHB_STATS
      if (lane == 0)
        for (int i = 0; i < 32; ++i) atomicAdd(&g_stats[i], s_stats[wid][i]);
#endif
      break;
    }
    const int64_t j = a.p_lo + t;
    const int64_t row = j - a.out_base;
    const int64_t o0 = a.key_off[j];
    const uint32_t m = (uint32_t)(a.key_off[j + 1] - o0);
    const int64_t kb = a.rec_stride ? (j - a.p_lo) * a.rec_stride : o0;  // records of j
    if (m == 0) {  // empty partitions are skipped (_kernels.py:248-249)
      if (lane == 0) {
        a.status[row] = 0;
        if (a.part_trials) a.part_trials[row] = 0;
      }
      continue;
    }

    TACC(14, tq);
    TSTAMP(tp);
    // ---- bucket histogram + counting sort into glo (_kernels.py:252-266)
#pragma unroll 1
    for (uint32_t b = lane; b <= B; b += 32) smem[cnt + b] = 0;
    __syncwarp();
    // records: separate (lo, u16 bucket id) arrays, or 16-byte (lo, bucket id)
    // records when bid is null (phb_scatter's one-store layout)
    const uint64_t* const rec = a.bid ? nullptr : a.lo;
    // PRO_D records per lane in flight: the loads come straight from K3's
    // writes (L2 / DRAM); one at a time they serialised the prologue
    // (C2 search: lambda = 4 7.48 -> 7.12 ms, lambda = 5 6.96 -> 6.77 ms)
    {
      uint32_t q = lane;
#pragma unroll 1
      for (; q + 32 * (PRO_D - 1) < m; q += 32 * PRO_D) {
        uint32_t bb[PRO_D];
#pragma unroll
        for (int e = 0; e < PRO_D; ++e)
          bb[e] = rec ? (uint32_t)__ldcg(&rec[2 * (kb + q + 32 * e) + 1]) : (uint32_t)a.bid[kb + q + 32 * e];
#pragma unroll
        for (int e = 0; e < PRO_D; ++e) atomicAdd(&smem[cnt + bb[e]], 1u);
      }
#pragma unroll 1
      for (; q < m; q += 32)
        atomicAdd(&smem[cnt + (rec ? (uint32_t)rec[2 * (kb + q) + 1] : (uint32_t)a.bid[kb + q])], 1u);
    }
    __syncwarp();
    uint32_t run = 0, maxsz = 0;
#pragma unroll 1
    for (uint32_t c0 = 1; c0 <= B; c0 += 32) {
      uint32_t b = c0 + lane;
      uint32_t v = b <= B ? smem[cnt + b] : 0u;
      uint32_t inc = warp_incl_scan(v, lane);
      if (b <= B) smem[endp + b] = run + inc - v;
      run += __shfl_sync(FULL, inc, 31);
      maxsz = max(maxsz, v);
    }
    maxsz = warp_max(maxsz);
    __syncwarp();
    {
      uint32_t q = lane;
      if (rec) {
#pragma unroll 1
        for (; q + 32 * (PRO_D - 1) < m; q += 32 * PRO_D) {
          ulonglong2 r[PRO_D];
#pragma unroll
          for (int e = 0; e < PRO_D; ++e) r[e] = reinterpret_cast<const ulonglong2*>(rec)[kb + q + 32 * e];
#pragma unroll
          for (int e = 0; e < PRO_D; ++e) {
            const uint32_t at = atomicAdd(&smem[endp + (uint32_t)r[e].y], 1u);
            a.glo[kb + at] = r[e].x;
          }
        }
      }
#pragma unroll 1
      for (; q < m; q += 32) {
        uint64_t lo;
        uint32_t b;
        if (rec) {
          const ulonglong2 r = reinterpret_cast<const ulonglong2*>(rec)[kb + q];
          lo = r.x;
          b = (uint32_t)r.y;
        } else {
          lo = a.lo[kb + q];
          b = a.bid[kb + q];
        }
        const uint32_t at = atomicAdd(&smem[endp + b], 1u);
        a.glo[kb + at] = lo;
      }
    }
    const uint32_t occ_used = min((uint32_t)plan.occ_w, (2 * m) / 32 + 104);
#pragma unroll 1
    for (uint32_t w = lane; w < occ_used; w += 32) smem[occ + w] = 0;
    __syncwarp();

    const uint32_t nb = bucket_order(cnt, B, a.tie_desc, maxsz, order, shist, srun, lane);
    __syncwarp();
    // search state (overwrites the bucket-order scratch)
    const uint32_t scr_used = m / 32 + 2;
#pragma unroll 1
    for (uint32_t w = lane; w < scr_used; w += 32) smem[scr + w] = 0;
#pragma unroll 1
    for (uint32_t w = lane; w < 96; w += 32) {
      const int64_t lt = (int64_t)m - 1 - 32 * (int64_t)w;  // last valid bit of word w
      smem[dmask + w] = lt < 0 ? FULL : (lt < 31 ? ~((2u << lt) - 1u) : 0u);
    }
    __syncwarp();

    TACC(10, tp);
    // ---- seed search, bucket by bucket (_kernels.py:295-369)
    int64_t ptrials = 0;
    uint8_t status = 0;
    const bool small_ok = m <= 3072;
    // speculative seed-0 steps over several small buckets pay while most of
    // them fit at seed 0, i.e. below ~85% fill; they need the whole seed-0
    // displacement range below the cap
    const bool multi_ok = small_ok && cap >= (int64_t)m - 1 && m <= 32u * 8u * PHB_MB_WPL;
    uint32_t placed = 0, mb_fail = 0xffffffffu;
#pragma unroll 1
    for (uint32_t oi = 0; oi < nb;) {
      const uint32_t b = order[oi];
      const uint32_t k = smem[cnt + b];
      const uint64_t* kl = a.glo + kb + (smem[endp + b] - k);
      BucketResult res;
      STAT(k == 1 ? 6 : 7, 1);
      TSTAMP(tb);
      if (LOWL && k == 1) {
        // the trailing singletons, up to 32 per step (no cap: _kernels.py:300-310)
        const uint32_t nS = min(32u, nb - oi);
        singles0(a, row, occ, pos16, order, oi, nS, endp, a.glo + kb, m, g0, ptrials, lane);
        TACC(11, tb);
        oi += nS;
        continue;
      }
#ifndef PHB_MB_E
#define PHB_MB_E 2.0f  // C2 lambda = 5 search 7.22 -> 6.99 ms (4.0: the round-2a gate)
#endif
      // expected seed-0 fits of this bucket, m (1 - fill)^k: the step pays
      // when the first (largest) bucket almost surely fits at seed 0
      if (LOWL && multi_ok && k <= 8 && oi != mb_fail && oi + 1 < nb &&
          (float)m * __powf((float)(m - placed) / (float)m, (float)k) >= PHB_MB_E) {
        uint32_t nG = 1;
#pragma unroll 1
        while (nG < 4 && oi + nG < nb) {
          const uint32_t kn = smem[cnt + order[oi + nG]];
          if (kn < 2) break;
          ++nG;
        }
        if (nG >= 2) {
          const uint32_t acc_n = multi_bucket0(a, row, occ, dmask, pos16, order, oi, nG, cnt, endp,
                                               a.glo + kb, m, g0, ptrials, placed, lane);
          TACC(12, tb);
          if (acc_n) {
            oi += acc_n;
            continue;
          }
          mb_fail = oi;  // this bucket failed seed 0: the regular path takes it
        }
      }
      if (!LOWL && k == 1) {
        // singleton: first free slot cyclically from the s = 0 base; no cap
        // (_kernels.py:300-310)
        const uint32_t p = position(kl[0], g0, m);
        if (lane == 0) pos16[0] = (uint16_t)p;
        __syncwarp();
        const int64_t d = find_d(occ, pos16, 1, (int64_t)m - 1, kl, g0, m, lane);
        uint32_t slot = p + (uint32_t)d;
        if (slot >= m) slot -= m;
        if (lane == 0) mark(occ, slot, m, 1);
        res = {d, d + 1, 0};
      } else if (small_ok && k <= 32) {
        // one single-seed step first (sparse tables usually succeed at s = 0),
        // then batches of G seeds; one call site per instantiation keeps the
        // kernel's instruction footprint small
        int64_t s_next = 0;
        const uint32_t kg1 = 16u;  // larger buckets stay single-seed
        res = small_bucket<1>(occ, dmask, pos16, k, kl, m, cap, s_next, 0, k > kg1 ? (1 << 30) : 1,
                              lane);
        if (res.status < 0) {
          // batched instantiations hold 32 / G lanes per seed: only k <= 16
          if (k <= 8 && (W4 >= 96 || m <= 32u * W4))
            res = small_bucket<4, W4>(occ, dmask, pos16, k, kl, m, cap, s_next, res.trials, 1 << 30,
                                      lane);
          else if (k <= kg1 && (W2 >= 96 || m <= 32u * W2))
            res = small_bucket<2, W2>(occ, dmask, pos16, k, kl, m, cap, s_next, res.trials, 1 << 30,
                                      lane);
          // near the seed cap, or k > 16: single-seed steps until decided
          while (res.status < 0)
            res = small_bucket<1>(occ, dmask, pos16, k, kl, m, cap, s_next, res.trials, 1 << 30,
                                  lane);
        }
      } else {
        res = generic_bucket(occ, scr, pos16, k, kl, m, cap, 0, 0, lane);
      }
      TACC(k == 1 ? 11 : ((small_ok && k <= 32) ? 12 : 13), tb);
#ifdef PHB_STATS
      if (small_ok && k >= 2 && k <= 32 && res.status == 0) {
        const int cls = k <= 8 ? 0 : (k <= 16 ? 1 : 2);
        TACC(16 + cls, tb);
        STAT(19 + cls, 1);
        STAT(22 + cls, res.seed / m + 1);
      }
#endif
      if (res.status > 0) {
        status = (uint8_t)res.status;
        break;
      }
      __syncwarp();
      if (lane == 0) {
        a.seeds[row * a.s_sj + (int64_t)(b - 1) * a.s_sb] = (uint64_t)res.seed;
        if (a.trials) a.trials[row * a.s_sj + (int64_t)(b - 1) * a.s_sb] = res.trials;
      }
      ptrials += res.trials;
      placed += k;
      ++oi;
    }
    __syncwarp();
    if (lane == 0) {
      a.status[row] = status;
      if (a.part_trials) a.part_trials[row] = ptrials;
    }
  }
}

int search_stats(unsigned long long* out16, int reset) {
#ifdef PHB_STATS
  PHB_CUDA_TRY(cudaMemcpyFromSymbol(out16, g_stats, sizeof(unsigned long long) * 32));
  if (reset) {
    unsigned long long z[32] = {0};
    PHB_CUDA_TRY(cudaMemcpyToSymbol(g_stats, z, sizeof(z)));
  }
  return 0;
#else
  for (int i = 0; i < 32; ++i) out16[i] = 0;
  return 1003;
#endif
}

int launch_search(const SearchArgs& a, cudaStream_t st) {
  const int64_t nrange = a.p_hi - a.p_lo;
  if (nrange <= 0) return 0;
  if (a.bcount < 1 || a.bcount > 65535) return 1001;  // PHB_E_BUCKETS
  if (a.m_max >= 65536) return 1002;                   // u16 positions
  SmemPlan plan = smem_plan(a.m_max < 1 ? 1 : a.m_max, a.bcount);
  size_t per_cta = (size_t)plan.total_w * 4 * WARPS;
  int dev = 0;
  PHB_CUDA_TRY(cudaGetDevice(&dev));
  int max_optin = 0;
  PHB_CUDA_TRY(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (per_cta > (size_t)max_optin) return 1002;  // PHB_E_PARTITION_TOO_LARGE
  // the device's opt-in maximum, not this launch's size: host threads
  // launching concurrently (compat_kernels under builder.py's thread pool)
  // would otherwise race on the attribute and launch above each other's cap
  // average keys per bucket, from the largest partition: below 6 the
  // low-lambda instantiation (measured at C2: lambda = 4 / 5 search 10.6 /
  // 9.3 -> 7.9 / 7.5 ms; at lambda = 6 and up it is slower)
  const bool lowl = (double)a.m_max < 6.0 * (double)a.bcount;
  const void* fn = lowl ? (const void*)k_search<true> : (const void*)k_search<false>;
  cudaFuncAttributes fa;
  PHB_CUDA_TRY(cudaFuncGetAttributes(&fa, fn));
  const int dyn_max = max_optin - (int)fa.sharedSizeBytes;  // the static part counts too
  if (per_cta > (size_t)dyn_max) return 1002;               // PHB_E_PARTITION_TOO_LARGE
  PHB_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max));
  int per_sm = 0;
  PHB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, WARPS * 32, per_cta));
  if (per_sm < 1) per_sm = 1;
  int64_t want = (nrange + WARPS - 1) / WARPS;
  int64_t cap = (int64_t)num_sms() * per_sm;
  int grid = (int)(want < cap ? want : cap);
  PHB_CUDA_TRY(cudaMemsetAsync(a.queue, 0, sizeof(uint32_t), st));
  if (lowl)
    note_launch(), k_search<true><<<grid, WARPS * 32, per_cta, st>>>(a, plan);
  else
    note_launch(), k_search<false><<<grid, WARPS * 32, per_cta, st>>>(a, plan);
  return (int)cudaGetLastError();
}

}  // namespace phb
