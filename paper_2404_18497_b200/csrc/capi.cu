// extern "C" boundary of libphobic_b200.so (declared in include/phobic.h).
// Thin argument marshalling around the launchers; no state survives a call.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "../../include/phobic.h"
#include "common.cuh"
#include "phobic_encode.h"
#include "phobic_internal.h"

namespace phb {

unsigned long long g_launch_count = 0;

// Stream-ordered scratch for the library's short-lived buffers (layout
// tile states, decode temporaries, ...). The device's default memory pool
// keeps freed blocks (release threshold raised once per device), so these
// allocations do not go back to the driver at every synchronisation;
// PyTorch's own allocator does not use this pool.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st) {
  static int configured[64] = {0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < 64 && !__atomic_load_n(&configured[dev], __ATOMIC_ACQUIRE)) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = 1ull << 30;  // up to 1 GiB of freed blocks stay in the pool
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    __atomic_store_n(&configured[dev], 1, __ATOMIC_RELEASE);
  }
  return cudaMallocAsync(p, bytes, st);
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1)
      v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

int search_stats(unsigned long long* out16, int reset);

int launch_decode(const uint8_t* blob, int64_t ncols, const int64_t* host_info, int64_t nparts,
                  uint32_t B, int mono, uint64_t* seeds, cudaStream_t st);

__global__ void k_range_max(const int64_t* __restrict__ key_off, int64_t p_lo, int64_t p_hi,
                            unsigned long long* __restrict__ out) {
  unsigned long long mx = 0;
  for (int64_t j = p_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < p_hi;
       j += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, (unsigned long long)(key_off[j + 1] - key_off[j]));
  atomicMax(out, mx);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[1] = (unsigned long long)key_off[p_lo];
    out[2] = (unsigned long long)key_off[p_hi];
  }
}

__global__ void k_offsets_from_deltas(const int64_t* __restrict__ deltas, int64_t n,
                                      int64_t nparts, int64_t* __restrict__ key_off) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= nparts;
       j += (int64_t)gridDim.x * blockDim.x)
    key_off[j] = expected_offset(j, n, nparts) + deltas[j];
}

__global__ void k_synth(uint64_t* __restrict__ out, int64_t n, uint64_t offset) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = mix64(offset + (uint64_t)i);
}

}  // namespace phb

using namespace phb;

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

const char* phb_version(void) { return "phobic-b200 0.1.0 (sm_100a)"; }

const char* phb_error_string(int code) {
  switch (code) {
    case PHB_OK:
      return "ok";
    case PHB_E_BUCKETS:
      return "bucket count outside [1, 65535]";
    case PHB_E_PARTITION_TOO_LARGE:
      return "partition search state exceeds shared memory";
    case PHB_E_ARGS:
      return "invalid arguments";
    default:
      if (code > 0 && code < 1000) return cudaGetErrorString((cudaError_t)code);
      return "unknown error";
  }
}

int phb_device_sms(void) { return num_sms(); }

unsigned long long phb_launch_count(void) { return __atomic_load_n(&g_launch_count, __ATOMIC_RELAXED); }

int phb_murmur3_many(const uint8_t* buf, const int64_t* offsets, int64_t n, uint64_t seed,
                     uint64_t* out_hi, uint64_t* out_lo, void* stream) {
  if (n < 0 || (n > 0 && !offsets)) return PHB_E_ARGS;
  return launch_murmur(buf, offsets, nullptr, n, seed, out_hi, out_lo, S(stream));
}

int phb_murmur3_u64(const uint64_t* keys, int64_t n, uint64_t seed, uint64_t* out_hi,
                    uint64_t* out_lo, void* stream) {
  if (n < 0 || (n > 0 && !keys)) return PHB_E_ARGS;
  return launch_murmur(nullptr, nullptr, keys, n, seed, out_hi, out_lo, S(stream));
}

int phb_bucket_ids(const uint64_t* his, int64_t n, const double* entries, int32_t bcount,
                   uint16_t* out, void* stream) {
  if (bcount < 1 || bcount > 65535) return PHB_E_BUCKETS;
  if (n < 0) return PHB_E_ARGS;
  return launch_bucket_ids(his, n, entries, (uint32_t)bcount, out, S(stream));
}

int phb_hash_count(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t n,
                   uint64_t seed, int64_t nparts, uint32_t* counts, void* stream) {
  if (n < 0 || nparts < 1 || nparts >= (int64_t(1) << 32)) return PHB_E_ARGS;
  return launch_hash_count(buf, offsets, keys64, n, seed, (uint64_t)nparts, counts, S(stream));
}

int phb_hash_count_store(const uint8_t* buf, const int64_t* offsets, int64_t n, uint64_t seed,
                         int64_t nparts, uint32_t* counts, uint64_t* hashes_out, void* stream) {
  if (n < 0 || nparts < 1 || nparts >= (int64_t(1) << 32) || !hashes_out) return PHB_E_ARGS;
  if (n > 0 && (!buf || !offsets)) return PHB_E_ARGS;
  return launch_hash_count(buf, offsets, nullptr, n, seed, (uint64_t)nparts, counts, S(stream),
                           hashes_out);
}

int phb_scatter_hashed(const uint64_t* hashes, int64_t n, int64_t nparts, const double* entries,
                       int32_t bcount, const int64_t* key_off, uint32_t* cursor, uint64_t* rec_out,
                       void* stream) {
  if (bcount < 1 || bcount > 65535) return PHB_E_BUCKETS;
  if (n < 0 || nparts < 1) return PHB_E_ARGS;
  return launch_scatter_hashed(hashes, n, (uint64_t)nparts, entries, (uint32_t)bcount, key_off,
                               cursor, rec_out, S(stream));
}

int phb_layout(uint32_t* counts, int64_t nparts, int64_t key_base, int64_t part_base,
               int64_t global_n, int64_t global_nparts, int64_t* key_off, int64_t* deltas,
               int64_t* stats, void* stream) {
  return launch_layout(counts, nparts, key_base, part_base, global_n, global_nparts, key_off,
                       deltas, stats, nullptr, 0, S(stream));
}

int phb_scatter(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t n,
                uint64_t seed, int64_t nparts, const double* entries, int32_t bcount,
                const int64_t* key_off, uint32_t* cursor, uint64_t* lo_out, uint16_t* bid_out,
                void* stream) {
  if (bcount < 1 || bcount > 65535) return PHB_E_BUCKETS;
  if (n < 0 || nparts < 1) return PHB_E_ARGS;
  return launch_scatter(buf, offsets, keys64, n, seed, (uint64_t)nparts, entries,
                        (uint32_t)bcount, key_off, cursor, lo_out, bid_out, S(stream));
}

int phb_search(const uint64_t* lo, const uint16_t* bid, const int64_t* key_off, int64_t p_lo,
               int64_t p_hi, int64_t out_base, int32_t bcount, int64_t seed_cap, int32_t tie_desc,
               int64_t m_max, uint64_t* seeds, int64_t s_sj, int64_t s_sb, int64_t* trials,
               int64_t* part_trials, uint8_t* status, uint64_t* glo, uint32_t* queue,
               void* stream) {
  if (bcount < 1 || bcount > 65535) return PHB_E_BUCKETS;
  SearchArgs a;
  a.lo = lo;
  a.bid = bid;
  a.key_off = key_off;
  a.p_lo = p_lo;
  a.p_hi = p_hi;
  a.out_base = out_base;
  a.bcount = (uint32_t)bcount;
  a.seed_cap = seed_cap;
  a.tie_desc = tie_desc;
  a.seeds = seeds;
  a.s_sj = s_sj;
  a.s_sb = s_sb;
  a.trials = trials;
  a.part_trials = part_trials;
  a.status = status;
  a.glo = glo;
  a.queue = queue;
  a.m_max = m_max;
  return launch_search(a, S(stream));
}

int phb_search_strided(const uint64_t* lo, const uint16_t* bid, const int64_t* key_off,
                       int64_t p_lo, int64_t p_hi, int64_t out_base, int32_t bcount,
                       int64_t seed_cap, int32_t tie_desc, int64_t m_max, uint64_t* seeds,
                       int64_t s_sj, int64_t s_sb, int64_t* trials, int64_t* part_trials,
                       uint8_t* status, uint64_t* glo, uint32_t* queue, int64_t rec_stride,
                       void* stream) {
  if (bcount < 1 || bcount > 65535) return PHB_E_BUCKETS;
  if (rec_stride < 0 || (rec_stride > 0 && m_max > rec_stride)) return PHB_E_ARGS;
  SearchArgs a;
  a.lo = lo;
  a.bid = bid;
  a.key_off = key_off;
  a.p_lo = p_lo;
  a.p_hi = p_hi;
  a.out_base = out_base;
  a.bcount = (uint32_t)bcount;
  a.seed_cap = seed_cap;
  a.tie_desc = tie_desc;
  a.seeds = seeds;
  a.s_sj = s_sj;
  a.s_sb = s_sb;
  a.trials = trials;
  a.part_trials = part_trials;
  a.status = status;
  a.glo = glo;
  a.queue = queue;
  a.m_max = m_max;
  a.rec_stride = rec_stride;
  return launch_search(a, S(stream));
}

int phb_scatter_padded(const uint64_t* keys64, int64_t n, uint64_t seed, int64_t nparts,
                       const double* entries, int32_t bcount, int32_t cap, int32_t init,
                       uint32_t* cursor, uint64_t* lo_out, uint16_t* bid_out,
                       uint32_t* overflow, void* stream) {
  if (bcount < 1 || bcount > 65535) return PHB_E_BUCKETS;
  if (n < 0 || nparts < 1 || cap < 1 || !cursor || !overflow || (n > 0 && !keys64))
    return PHB_E_ARGS;
  return launch_scatter_padded(keys64, n, seed, (uint64_t)nparts, entries, (uint32_t)bcount,
                               (uint32_t)cap, init, cursor, lo_out, bid_out, overflow, S(stream));
}

int phb_padded_counts(const uint32_t* cursor, int64_t nparts, int32_t cap, uint32_t* counts,
                      uint32_t* overflow, void* stream) {
  if (nparts < 1 || cap < 1 || !cursor || !counts || !overflow) return PHB_E_ARGS;
  return launch_padded_counts(cursor, nparts, (uint32_t)cap, counts, overflow, S(stream));
}

int phb_build_partition_range(const uint64_t* his, const uint64_t* los, const int64_t* key_off,
                              int64_t p_lo, int64_t p_hi, const double* entries, int32_t bcount,
                              int64_t seed_cap, int32_t tie_desc, uint64_t* seeds_out,
                              int64_t* trials_out, uint8_t* status_out, void* stream) {
  if (bcount < 1 || bcount > 65535) return PHB_E_BUCKETS;
  if (p_hi <= p_lo) return 0;
  cudaStream_t st = S(stream);
  unsigned long long* d_stat = nullptr;
  unsigned long long h_stat[3] = {0, 0, 0};
  PHB_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&d_stat), 3 * sizeof(unsigned long long), st));
  PHB_CUDA_TRY(cudaMemsetAsync(d_stat, 0, 3 * sizeof(unsigned long long), st));
  int g = (int)std::min<int64_t>((p_hi - p_lo + 255) / 256, 1024);
  note_launch(), k_range_max<<<g, 256, 0, st>>>(key_off, p_lo, p_hi, d_stat);
  PHB_CUDA_TRY(cudaGetLastError());
  PHB_CUDA_TRY(cudaMemcpyAsync(h_stat, d_stat, sizeof(h_stat), cudaMemcpyDeviceToHost, st));
  PHB_CUDA_TRY(cudaStreamSynchronize(st));
  const int64_t k0 = (int64_t)h_stat[1], k1 = (int64_t)h_stat[2];
  const int64_t nk = k1 - k0;
  uint16_t* bid = nullptr;
  uint64_t* glo = nullptr;
  uint32_t* queue = nullptr;
  PHB_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&bid), sizeof(uint16_t) * (nk > 0 ? nk : 1), st));
  PHB_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&glo), sizeof(uint64_t) * (nk > 0 ? nk : 1), st));
  PHB_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&queue), sizeof(uint32_t), st));
  int rc = launch_bucket_ids(his + k0, nk, entries, (uint32_t)bcount, bid, st);
  if (rc == 0) {
    SearchArgs a;
    a.lo = los;
    a.bid = bid - k0;   // absolute indexing by key_off
    a.key_off = key_off;
    a.p_lo = p_lo;
    a.p_hi = p_hi;
    a.out_base = 0;
    a.bcount = (uint32_t)bcount;
    a.seed_cap = seed_cap;
    a.tie_desc = tie_desc;
    a.seeds = seeds_out;
    a.s_sj = bcount;
    a.s_sb = 1;
    a.trials = trials_out;
    a.part_trials = nullptr;
    a.status = status_out;
    a.glo = glo - k0;
    a.queue = queue;
    a.m_max = (int64_t)h_stat[0];
    rc = launch_search(a, st);
  }
  cudaFreeAsync(bid, st);
  cudaFreeAsync(glo, st);
  cudaFreeAsync(queue, st);
  cudaFreeAsync(d_stat, st);
  return rc;
}

int phb_offsets_from_deltas(const int64_t* deltas, int64_t n, int64_t nparts, int64_t* key_off,
                            void* stream) {
  if (nparts < 1) return PHB_E_ARGS;
  int g = (int)std::min<int64_t>((nparts + 256) / 256, 4096);
  note_launch(), k_offsets_from_deltas<<<g, 256, 0, S(stream)>>>(deltas, n, nparts, key_off);
  return (int)cudaGetLastError();
}

int phb_query_many(const uint64_t* his, const uint64_t* los, int64_t nq, int64_t n,
                   int64_t nparts, const int64_t* deltas, const double* entries, int32_t bcount,
                   const uint64_t* seed_mat, int64_t* out, void* stream) {
  if (bcount < 1 || bcount > 65535) return PHB_E_BUCKETS;
  if (nparts < 1) return PHB_E_ARGS;
  cudaStream_t st = S(stream);
  int64_t* key_off = nullptr;
  PHB_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&key_off), sizeof(int64_t) * (nparts + 1), st));
  int rc = phb_offsets_from_deltas(deltas, n, nparts, key_off, stream);
  if (rc == 0)
    rc = launch_query(nullptr, nullptr, nullptr, his, los, nq, 0, n, nparts, key_off, entries,
                      (uint32_t)bcount, seed_mat, bcount, 1, out, st);
  cudaFreeAsync(key_off, st);
  return rc;
}

size_t phb_encode_workspace_bytes(int64_t nparts, int32_t bcount, int32_t mono) {
  return encode_workspace_bytes(nparts, (uint32_t)bcount, mono);
}

static EncodeArgs make_enc(const uint64_t* seeds, int64_t nparts, int32_t bcount, int32_t mono,
                           int32_t compact_prefix, const int64_t* deltas, int64_t nparts_global,
                           const int64_t* layout_stats, const uint8_t* status,
                           const int64_t* part_trials) {
  EncodeArgs a;
  a.seeds = seeds;
  a.nparts = nparts;
  a.bcount = (uint32_t)bcount;
  a.mono = mono;
  a.compact_prefix = compact_prefix;
  a.deltas = deltas;
  a.nparts_global = nparts_global;
  a.layout_stats = layout_stats;
  a.status = status;
  a.part_trials = part_trials;
  return a;
}

int phb_encode_plan(const uint64_t* seeds, int64_t nparts, int32_t bcount, int32_t mono,
                    int32_t compact_prefix, const int64_t* deltas, int64_t nparts_global,
                    const int64_t* layout_stats, const uint8_t* status,
                    const int64_t* part_trials, void* workspace, int64_t* summary_out,
                    void* stream) {
  if (bcount < 1 || nparts < 1 || !layout_stats || !workspace) return PHB_E_ARGS;
  EncodeArgs a = make_enc(seeds, nparts, bcount, mono, compact_prefix, deltas, nparts_global,
                          layout_stats, status, part_trials);
  EncodeSummary s;
  int rc = launch_encode_plan(a, workspace, summary_out ? &s : nullptr, S(stream));
  if (rc == 0 && summary_out) {
    summary_out[0] = (int64_t)s.total_bytes;
    summary_out[1] = (int64_t)s.seed_section;
    summary_out[2] = (int64_t)s.trials_total;
    summary_out[3] = s.first_bad;
    summary_out[4] = s.bad_code;
    summary_out[5] = s.delta_width;
    summary_out[6] = s.ncols;
    summary_out[7] = 0;
  }
  return rc;
}

int phb_encode_write(const uint64_t* seeds, int64_t nparts, int32_t bcount, int32_t mono,
                     int32_t compact_prefix, const int64_t* deltas, int64_t nparts_global,
                     const int64_t* layout_stats, void* workspace, uint8_t* blob,
                     size_t blob_bytes, void* stream) {
  if (bcount < 1 || nparts < 1 || !workspace || !blob) return PHB_E_ARGS;
  EncodeArgs a = make_enc(seeds, nparts, bcount, mono, compact_prefix, deltas, nparts_global,
                          layout_stats, nullptr, nullptr);
  return launch_encode_write(a, workspace, blob, blob_bytes, S(stream));
}

// ---- sharded encode (multi-GPU, distributed.py step 7)
int phb_encode_shard_stats(const uint64_t* seeds, int64_t nparts, int32_t bcount, int32_t mono,
                           unsigned long long* colstat_out, void* stream) {
  if (bcount < 1 || nparts < 0 || !colstat_out) return PHB_E_ARGS;
  EncodeArgs a = make_enc(seeds, nparts, bcount, mono, 0, nullptr, nparts, nullptr, nullptr,
                          nullptr);
  return launch_encode_stats(a, nullptr, colstat_out, S(stream));
}

int phb_encode_shard_plan(const uint64_t* seeds, int64_t nparts, int64_t row0,
                          int64_t nparts_global, int32_t bcount, int32_t mono,
                          int32_t compact_prefix, const int64_t* layout_stats,
                          const unsigned long long* colstat_global, void* workspace,
                          unsigned long long* rice_totals_out, int64_t* summary_out,
                          void* stream) {
  if (bcount < 1 || nparts < 0 || row0 < 0 || row0 + nparts > nparts_global || !layout_stats ||
      !workspace || !colstat_global || !rice_totals_out)
    return PHB_E_ARGS;
  EncodeArgs a = make_enc(seeds, nparts, bcount, mono, compact_prefix, nullptr, nparts_global,
                          layout_stats, nullptr, nullptr);
  a.row0 = row0;
  a.count_global = mono ? nparts_global * (int64_t)bcount : nparts_global;
  a.colstat_in = colstat_global;
  a.rice_totals_out = rice_totals_out;
  EncodeSummary s;
  int rc = launch_encode_plan(a, workspace, summary_out ? &s : nullptr, S(stream));
  if (rc == 0 && summary_out) {
    summary_out[0] = (int64_t)s.total_bytes;
    summary_out[1] = (int64_t)s.seed_section;
    summary_out[2] = 0;
    summary_out[3] = -1;
    summary_out[4] = 0;
    summary_out[5] = s.delta_width;
    summary_out[6] = s.ncols;
    summary_out[7] = 0;
  }
  return rc;
}

int phb_encode_shard_write(const uint64_t* seeds, int64_t nparts, int64_t row0,
                           int64_t nparts_global, int32_t bcount, int32_t mono,
                           int32_t compact_prefix, const int64_t* deltas,
                           const int64_t* layout_stats, const unsigned long long* rice_base,
                           int32_t write_headers, void* workspace, uint8_t* blob,
                           size_t blob_bytes, void* stream) {
  if (bcount < 1 || nparts < 0 || !workspace || !blob || !layout_stats) return PHB_E_ARGS;
  EncodeArgs a = make_enc(seeds, nparts, bcount, mono, compact_prefix, deltas, nparts_global,
                          layout_stats, nullptr, nullptr);
  a.row0 = row0;
  a.count_global = mono ? nparts_global * (int64_t)bcount : nparts_global;
  a.rice_base = rice_base;
  a.write_headers = write_headers;
  return launch_encode_write(a, workspace, blob, blob_bytes, S(stream));
}

int phb_decode_seeds(const uint8_t* blob, int64_t ncols, const int64_t* col_info, int64_t nparts,
                     int32_t bcount, int32_t mono, uint64_t* seeds, void* stream) {
  if (bcount < 1 || nparts < 1 || !col_info) return PHB_E_ARGS;
  return launch_decode(blob, ncols, col_info, nparts, (uint32_t)bcount, mono, seeds, S(stream));
}

int phb_query(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t nq,
              uint64_t seed, int64_t n, int64_t nparts, const int64_t* key_off,
              const double* entries, int32_t bcount, const uint64_t* seeds, int64_t s_sj,
              int64_t s_sb, int64_t* out, void* stream) {
  if (bcount < 1 || bcount > 65535) return PHB_E_BUCKETS;
  if (nparts < 1) return PHB_E_ARGS;
  return launch_query(buf, offsets, keys64, nullptr, nullptr, nq, seed, n, nparts, key_off,
                      entries, (uint32_t)bcount, seeds, s_sj, s_sb, out, S(stream));
}

int phb_query32(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t nq,
                uint64_t seed, int64_t n, int64_t nparts, const int64_t* key_off,
                const uint32_t* part2, const double* entries, int32_t bcount,
                const uint32_t* seeds32, int64_t* out, void* stream) {
  if (bcount < 1 || bcount > 65535) return PHB_E_BUCKETS;
  if (nparts < 1 || !seeds32 || !part2 || n >= (int64_t)1 << 32) return PHB_E_ARGS;
  return launch_query32(buf, offsets, keys64, nq, seed, n, nparts, key_off,
                        reinterpret_cast<const uint2*>(part2), entries, (uint32_t)bcount, seeds32,
                        out, S(stream));
}

int phb_part_table32(const int64_t* key_off, int64_t nparts, uint32_t* part2, void* stream) {
  if (nparts < 0 || (nparts > 0 && (!key_off || !part2))) return PHB_E_ARGS;
  return launch_part_table32(key_off, nparts, reinterpret_cast<uint2*>(part2), S(stream));
}

int phb_seed_table32(const uint64_t* seeds, const int64_t* key_off, int64_t nparts, int64_t count,
                     uint32_t* out, uint32_t* overflow, void* stream) {
  if (count < 0 || nparts < 1 || (count > 0 && (!seeds || !key_off || !out || !overflow)))
    return PHB_E_ARGS;
  return launch_seed_table32(seeds, key_off, nparts, count, out, overflow, S(stream));
}

int phb_query_encoded(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64,
                      int64_t nq, uint64_t seed, int64_t n, int64_t nparts,
                      const int64_t* key_off, const double* entries, int32_t bcount,
                      const uint8_t* section, const int64_t* col_info, int32_t num_enc,
                      int32_t mono, const uint32_t* select_dir, int64_t select_stride,
                      int64_t* out, void* stream) {
  if (bcount < 1 || bcount > 65535) return PHB_E_BUCKETS;
  if (nparts < 1 || !section || !col_info) return PHB_E_ARGS;
  if (mono ? num_enc != 1 : num_enc != bcount) return PHB_E_ARGS;
  return launch_query_encoded(buf, offsets, keys64, nq, seed, n, nparts, key_off, entries,
                              (uint32_t)bcount, section, col_info, mono, select_dir,
                              select_stride, out, S(stream));
}

int phb_select_index(const uint8_t* section, const int64_t* col_info, int64_t num_enc,
                     int64_t stride, uint32_t* select_dir, void* stream) {
  if (num_enc < 0 || stride < 1 || (num_enc > 0 && (!section || !col_info || !select_dir)))
    return PHB_E_ARGS;
  return launch_select_index(section, col_info, num_enc, stride, select_dir, S(stream));
}

int phb_verify(const int64_t* out, int64_t nq, int64_t n, uint32_t* bitmap, uint32_t* bad_flag,
               void* stream) {
  return launch_verify(out, nq, n, bitmap, bad_flag, S(stream));
}

int phb_regroup(const uint64_t* lo_in, const uint16_t* aux_in, const int32_t* counts, int64_t G,
                int64_t np, uint64_t* lo_out, uint16_t* aux_out, int64_t* key_off, void* stream) {
  return launch_regroup(lo_in, aux_in, counts, G, np, lo_out, aux_out, key_off, S(stream));
}

int phb_scatter_p2p(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t n,
                    uint64_t seed, int64_t nparts, const double* entries, int32_t bcount,
                    const int64_t* part_base, const uint8_t* owner, uint64_t* const* lo_dst,
                    uint16_t* const* bid_dst, int32_t G, uint32_t* cursor, void* stream) {
  if (bcount < 1 || bcount > 65535) return PHB_E_BUCKETS;
  if (!lo_dst) return PHB_E_ARGS;  // bid_dst NULL: 16-byte records in lo_dst
  return launch_scatter_p2p(buf, offsets, keys64, n, seed, nparts, entries, (uint32_t)bcount,
                            part_base, owner, lo_dst, bid_dst, G, cursor, S(stream));
}

int phb_ipc_alloc(size_t bytes, void** dptr) {
  if (!dptr) return PHB_E_ARGS;
  return (int)cudaMalloc(dptr, bytes ? bytes : 16);
}

int phb_ipc_free(void* dptr) { return (int)cudaFree(dptr); }

int phb_ipc_handle(void* dptr, uint8_t* handle64) {
  cudaIpcMemHandle_t h;
  PHB_CUDA_TRY(cudaIpcGetMemHandle(&h, dptr));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle64, &h, 64);
  return 0;
}

int phb_ipc_open(const uint8_t* handle64, void** dptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  return (int)cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess);
}

int phb_ipc_close(void* dptr) { return (int)cudaIpcCloseMemHandle(dptr); }

int phb_sync(void* stream) { return (int)cudaStreamSynchronize(S(stream)); }

int phb_search_stats(unsigned long long* out16, int reset) {
  return search_stats(out16, reset);
}

int phb_synth_keys(uint64_t* out, int64_t n, uint64_t offset, void* stream) {
  if (n < 0) return PHB_E_ARGS;
  if (n == 0) return 0;
  int g = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  note_launch(), k_synth<<<g, 256, 0, S(stream)>>>(out, n, offset);
  return (int)cudaGetLastError();
}

}  // extern "C"
