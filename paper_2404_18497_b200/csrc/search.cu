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
//    SURVEY.md §0 finding 7) load-balance dynamically across ~40 resident
//    warps per SM. No __syncthreads anywhere: warps are independent.
//  * Per-warp shared memory holds only bitmaps and bucket metadata
//    (~4-6 KB): a doubled occupancy bitmap (2m bits, so a cyclic window is
//    one funnel shift), an m-bit self-collision scratch map, bucket sizes /
//    offsets and the processing order. Keys stay in L1/L2 (bucket-grouped
//    scratch `glo`) and in registers (<= 256 keys per bucket).
//  * Displacement search is bit-parallel: valid(d) = AND_i free(p_i + d).
//    Lane l evaluates d in [1024c + 32l, +32) as one u32 word; a ballot +
//    ffs picks the smallest d. 32 lanes x 32 bits = 1024 displacements per
//    step, with an early exit once every lane's word is saturated.
//  * Self-collision of a candidate s: __match_any_sync on positions for
//    k <= 32, shared-memory atomicOr test-and-set for larger buckets.
//  * Trials use the closed form k * (S_self + sum_fail(dmax+1) + d* + 1),
//    identical to the reference's per-candidate counting.
#include "common.cuh"
#include "phobic_internal.h"

namespace phb {

constexpr int KREG = 8;    // key rounds held in registers: buckets up to 256 keys
constexpr int SH = 256;    // size classes of the counting-sort bucket order
constexpr int WARPS = 4;   // warps (= partitions in flight) per CTA
constexpr unsigned FULL = 0xffffffffu;

struct SmemPlan {
  int occ_w, scr_w, cnt_w, ord_w, sh_w, total_w;
};

__host__ __device__ inline SmemPlan smem_plan(int64_t m_max, uint32_t bcount) {
  SmemPlan p;
  p.occ_w = (int)((2 * m_max + 64) / 32 + 2);
  p.scr_w = (int)(m_max / 32 + 2);
  p.cnt_w = (int)bcount + 1;  // cnt and endp each
  p.ord_w = (int)(bcount + 2) / 2;
  p.sh_w = SH;  // shist + srun as u16
  p.total_w = p.occ_w + p.scr_w + 2 * p.cnt_w + p.ord_w + p.sh_w;
  p.total_w += p.total_w & 1;
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

__device__ __forceinline__ uint32_t window(const uint32_t* occ, uint32_t q) {
  uint32_t w = q >> 5;
  return __funnelshift_r(occ[w], occ[w + 1], q & 31);
}

__device__ __forceinline__ void mark(uint32_t* occ, uint32_t slot, uint32_t m) {
  atomicOr(occ + (slot >> 5), 1u << (slot & 31));
  uint32_t s2 = slot + m;
  atomicOr(occ + (s2 >> 5), 1u << (s2 & 31));
}

// Processing order of the non-empty buckets (_kernels.py:268-282):
// size descending, ties by `tie` descending where tie = b ("asc-expected",
// tie_desc = 1) or B - b. Returns the number of non-empty buckets.
__device__ uint32_t bucket_order(const uint32_t* cnt, uint32_t B, int tie_desc, uint32_t maxsz,
                                 uint16_t* order, uint16_t* shist, uint16_t* srun, int lane) {
  if (maxsz < (uint32_t)SH) {
    for (int s = lane; s < SH; s += 32) shist[s] = 0, srun[s] = 0;
    __syncwarp();
    for (uint32_t c0 = 1; c0 <= B; c0 += 32) {
      uint32_t b = c0 + lane;
      uint32_t sz = b <= B ? cnt[b] : 0u;
      uint32_t peers = __match_any_sync(FULL, sz);
      if (sz > 0 && lane == __ffs(peers) - 1) shist[sz] += (uint16_t)__popc(peers);
      __syncwarp();
    }
    // base[s] = number of buckets with size > s
    uint32_t run = 0;
    for (int c = 0; c < SH / 32; ++c) {
      int s = SH - 1 - (c * 32 + lane);
      uint32_t v = shist[s];
      uint32_t inc = warp_incl_scan(v, lane);
      __syncwarp();
      shist[s] = (uint16_t)(run + inc - v);
      run += __shfl_sync(FULL, inc, 31);
    }
    __syncwarp();
    for (uint32_t c0 = 0; c0 < B; c0 += 32) {
      uint32_t idx = c0 + lane;
      uint32_t b = tie_desc ? (B - idx) : (idx + 1);
      uint32_t sz = idx < B ? cnt[b] : 0u;
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
  for (uint32_t c0 = 1; c0 <= B; c0 += 32) {
    uint32_t b = c0 + lane;
    uint32_t sz = b <= B ? cnt[b] : 0u;
    if (sz > 0) {
      uint64_t key = (uint64_t)sz * (B + 1) + (tie_desc ? b : B - b);
      uint32_t rank = 0;
      for (uint32_t b2 = 1; b2 <= B; ++b2) {
        uint32_t s2 = cnt[b2];
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
// pos[r] holds the base positions of key 32r + lane (registers, r < KREG);
// rounds beyond KREG re-derive positions from the key scratch.
__device__ __forceinline__ int64_t first_valid(const uint32_t* occ, const uint32_t (&pos)[KREG],
                                               uint32_t k, int64_t dmax, const uint64_t* kl,
                                               uint64_t g, uint32_t m, int lane) {
  const uint32_t R = (k + 31) >> 5;
  const uint32_t nch = (uint32_t)((dmax + 1024) >> 10);
  for (uint32_t c = 0; c < nch; ++c) {
    const int64_t dbase = (int64_t)c * 1024 + lane * 32;
    const bool live = dbase <= dmax;
    const uint32_t db = (uint32_t)dbase;
    uint32_t acc = live ? 0u : FULL;
    bool dead = false;
#pragma unroll
    for (int r = 0; r < KREG; ++r) {
      if ((uint32_t)r < R && !dead) {
        const uint32_t kr = min(32u, k - 32u * r);
        for (uint32_t src = 0; src < kr; ++src) {
          uint32_t p = __shfl_sync(FULL, pos[r], src);
          if (live) acc |= window(occ, p + db);
          if ((src & 7) == 7 && __all_sync(FULL, acc == FULL)) {
            dead = true;
            break;
          }
        }
      }
    }
    for (uint32_t r = KREG; r < R && !dead; ++r) {
      const uint32_t kr = min(32u, k - 32u * r);
      uint32_t mine = lane < kr ? position(kl[32 * r + lane], g, m) : 0u;
      for (uint32_t src = 0; src < kr; ++src) {
        uint32_t p = __shfl_sync(FULL, mine, src);
        if (live) acc |= window(occ, p + db);
        if ((src & 7) == 7 && __all_sync(FULL, acc == FULL)) {
          dead = true;
          break;
        }
      }
    }
    uint32_t valid = ~acc;
    if (live) {
      int64_t rem = dmax - dbase;
      if (rem < 31) valid &= (2u << rem) - 1u;
    }
    uint32_t bal = __ballot_sync(FULL, valid != 0);
    if (bal) {
      int l = __ffs(bal) - 1;
      uint32_t vv = __shfl_sync(FULL, valid, l);
      return (int64_t)c * 1024 + l * 32 + (__ffs(vv) - 1);
    }
  }
  return -1;
}

__global__ void __launch_bounds__(WARPS * 32) k_search(SearchArgs a, SmemPlan plan) {
  extern __shared__ uint32_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t B = a.bcount;
  uint32_t* occ = smem + wid * plan.total_w;
  uint32_t* scr = occ + plan.occ_w;
  uint32_t* cnt = scr + plan.scr_w;
  uint32_t* endp = cnt + plan.cnt_w;
  uint16_t* order = reinterpret_cast<uint16_t*>(endp + plan.cnt_w);
  uint16_t* shist = order + 2 * plan.ord_w;
  uint16_t* srun = shist + SH;
  const int64_t nrange = a.p_hi - a.p_lo;
  const uint64_t g0 = mix64(POSITION_SALT);  // s = 0
  const int64_t cap = a.seed_cap;

  for (;;) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(a.queue, 1u);
    t = __shfl_sync(FULL, t, 0);
    if ((int64_t)t >= nrange) break;
    const int64_t j = a.p_lo + t;
    const int64_t row = j - a.out_base;
    const int64_t kb = a.key_off[j];
    const uint32_t m = (uint32_t)(a.key_off[j + 1] - kb);
    if (m == 0) {  // empty partitions are skipped (_kernels.py:248-249)
      if (lane == 0) {
        a.status[row] = 0;
        if (a.part_trials) a.part_trials[row] = 0;
      }
      continue;
    }

    // ---- bucket histogram + stable-free counting sort (_kernels.py:252-266)
    for (uint32_t b = lane; b <= B; b += 32) cnt[b] = 0;
    __syncwarp();
    for (uint32_t q = lane; q < m; q += 32) atomicAdd(cnt + a.bid[kb + q], 1u);
    __syncwarp();
    uint32_t run = 0, maxsz = 0;
    for (uint32_t c0 = 1; c0 <= B; c0 += 32) {
      uint32_t b = c0 + lane;
      uint32_t v = b <= B ? cnt[b] : 0u;
      uint32_t inc = warp_incl_scan(v, lane);
      if (b <= B) endp[b] = run + inc - v;
      run += __shfl_sync(FULL, inc, 31);
      maxsz = max(maxsz, v);
    }
    maxsz = warp_max(maxsz);
    __syncwarp();
    for (uint32_t q = lane; q < m; q += 32) {
      uint32_t b = a.bid[kb + q];
      uint32_t at = atomicAdd(endp + b, 1u);
      a.glo[kb + at] = a.lo[kb + q];
    }
    const uint32_t occ_used = (2 * m + 64) / 32 + 2;
    for (uint32_t w = lane; w < occ_used; w += 32) occ[w] = 0;
    const uint32_t scr_used = m / 32 + 2;
    for (uint32_t w = lane; w < scr_used; w += 32) scr[w] = 0;
    __syncwarp();

    const uint32_t nb = bucket_order(cnt, B, a.tie_desc, maxsz, order, shist, srun, lane);
    __syncwarp();

    // ---- seed search, bucket by bucket (_kernels.py:295-369)
    int64_t ptrials = 0;
    uint8_t status = 0;
    for (uint32_t oi = 0; oi < nb; ++oi) {
      const uint32_t b = order[oi];
      const uint32_t k = cnt[b];
      const uint64_t* kl = a.glo + kb + (endp[b] - k);
      int64_t seed = 0, trials = 0;
      if (k == 1) {
        // singleton: first free slot cyclically from the s = 0 base; no cap
        // (_kernels.py:300-310). Same first_valid machinery with one key.
        const uint32_t p = position(kl[0], g0, m);
        uint32_t pos[KREG] = {};
        pos[0] = p;
        int64_t d = first_valid(occ, pos, 1, (int64_t)m - 1, kl, g0, m, lane);
        uint32_t slot = p + (uint32_t)d;
        if (slot >= m) slot -= m;
        if (lane == 0) mark(occ, slot, m);
        seed = d;
        trials = d + 1;
      } else {
        const uint32_t R = (k + 31) >> 5;
        const uint32_t amask = k >= 32 ? FULL : ((1u << k) - 1u);
        uint64_t key[KREG];
        uint32_t pos[KREG];
#pragma unroll
        for (int r = 0; r < KREG; ++r) {
          uint32_t i = 32u * r + lane;
          key[r] = ((uint32_t)r < R && i < k) ? kl[i] : 0ull;
          pos[r] = 0;
        }
        for (int64_t s = 0;; ++s) {
          const int64_t pbase = s * (int64_t)m;
          if (s > 0 && pbase > cap) {  // _kernels.py:324-328
            status = 2;
            break;
          }
          const uint64_t g = mix64((uint64_t)s ^ POSITION_SALT);
          bool coll = false;
          if (k <= 32) {
            pos[0] = position(key[0], g, m);
            uint32_t peers = __match_any_sync(FULL, pos[0]) & amask;
            coll = __any_sync(FULL, lane < (int)k && __popc(peers) > 1);
          } else {
#pragma unroll
            for (int r = 0; r < KREG; ++r) {
              if ((uint32_t)r < R && !coll) {
                uint32_t i = 32u * r + lane;
                pos[r] = position(key[r], g, m);
                bool c = false;
                if (i < k) {
                  uint32_t bit = 1u << (pos[r] & 31);
                  c = (atomicOr(scr + (pos[r] >> 5), bit) & bit) != 0;
                }
                coll = __any_sync(FULL, c);
              }
            }
            for (uint32_t r = KREG; r < R && !coll; ++r) {
              uint32_t i = 32u * r + lane;
              bool c = false;
              if (i < k) {
                uint32_t p = position(kl[i], g, m);
                uint32_t bit = 1u << (p & 31);
                c = (atomicOr(scr + (p >> 5), bit) & bit) != 0;
              }
              coll = __any_sync(FULL, c);
            }
            __syncwarp();
            for (uint32_t w = lane; w < scr_used; w += 32) scr[w] = 0;
            __syncwarp();
          }
          if (s == 0) {
            // duplicate low words collide at every s, so they can only
            // exist if s = 0 collides (_kernels.py:312-319)
            if (coll) {
              bool dup = false;
              if (k <= 32) {
                uint32_t peers = __match_any_sync(FULL, key[0]) & amask;
                dup = lane < (int)k && __popc(peers) > 1;
              } else if (R <= (uint32_t)KREG) {
#pragma unroll
                for (int r1 = 0; r1 < KREG; ++r1) {
                  if ((uint32_t)r1 < R) {
                    const uint32_t kr = min(32u, k - 32u * r1);
                    for (uint32_t src = 0; src < kr; ++src) {
                      uint64_t v = __shfl_sync(FULL, key[r1], src);
#pragma unroll
                      for (int r2 = 0; r2 < KREG; ++r2) {
                        uint32_t i2 = 32u * r2 + lane;
                        if ((uint32_t)r2 < R && i2 < k && i2 != 32u * r1 + src && key[r2] == v)
                          dup = true;
                      }
                    }
                  }
                }
              } else {
                for (uint32_t i = 0; i < k; ++i) {
                  uint64_t v = kl[i];
                  for (uint32_t i2 = lane; i2 < k; i2 += 32)
                    if (i2 != i && kl[i2] == v) dup = true;
                }
              }
              if (__any_sync(FULL, dup)) {
                status = 1;
                break;
              }
            }
            if (pbase > cap) {
              status = 2;
              break;
            }
          }
          if (coll) {
            trials += k;
            continue;
          }
          int64_t dmax = cap - pbase;
          if (dmax > (int64_t)m - 1) dmax = (int64_t)m - 1;
          int64_t d = first_valid(occ, pos, k, dmax, kl, g, m, lane);
          if (d >= 0) {
            trials += (int64_t)k * (d + 1);
            seed = pbase + d;
#pragma unroll
            for (int r = 0; r < KREG; ++r) {
              uint32_t i = 32u * r + lane;
              if ((uint32_t)r < R && i < k) {
                uint32_t slot = pos[r] + (uint32_t)d;
                if (slot >= m) slot -= m;
                mark(occ, slot, m);
              }
            }
            for (uint32_t r = KREG; r < R; ++r) {
              uint32_t i = 32u * r + lane;
              if (i < k) {
                uint32_t slot = position(kl[i], g, m) + (uint32_t)d;
                if (slot >= m) slot -= m;
                mark(occ, slot, m);
              }
            }
            break;
          }
          trials += (int64_t)k * (dmax + 1);
        }
        if (status) break;
      }
      __syncwarp();
      if (lane == 0) {
        a.seeds[row * a.s_sj + (int64_t)(b - 1) * a.s_sb] = (uint64_t)seed;
        if (a.trials) a.trials[row * a.s_sj + (int64_t)(b - 1) * a.s_sb] = trials;
      }
      ptrials += trials;
    }
    __syncwarp();
    if (lane == 0) {
      a.status[row] = status;
      if (a.part_trials) a.part_trials[row] = ptrials;
    }
  }
}

int launch_search(const SearchArgs& a, cudaStream_t st) {
  const int64_t nrange = a.p_hi - a.p_lo;
  if (nrange <= 0) return 0;
  if (a.bcount < 1 || a.bcount > 65535) return 1001;  // PHB_E_BUCKETS
  SmemPlan plan = smem_plan(a.m_max < 1 ? 1 : a.m_max, a.bcount);
  size_t per_cta = (size_t)plan.total_w * 4 * WARPS;
  int dev = 0;
  PHB_CUDA_TRY(cudaGetDevice(&dev));
  int max_optin = 0;
  PHB_CUDA_TRY(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (per_cta > (size_t)max_optin) return 1002;  // PHB_E_PARTITION_TOO_LARGE
  PHB_CUDA_TRY(cudaFuncSetAttribute(k_search, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)per_cta));
  int per_sm = 0;
  PHB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_search, WARPS * 32,
                                                             per_cta));
  if (per_sm < 1) per_sm = 1;
  int64_t want = (nrange + WARPS - 1) / WARPS;
  int64_t cap = (int64_t)num_sms() * per_sm;
  int grid = (int)(want < cap ? want : cap);
  PHB_CUDA_TRY(cudaMemsetAsync(a.queue, 0, sizeof(uint32_t), st));
  k_search<<<grid, WARPS * 32, per_cta, st>>>(a, plan);
  return (int)cudaGetLastError();
}

}  // namespace phb
