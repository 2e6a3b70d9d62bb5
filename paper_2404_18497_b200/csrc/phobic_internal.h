// Internal launchers shared between the kernel translation units and the
// C-ABI layer (capi.cu). Not part of the public interface (include/phobic.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace phb {

// Process-wide count of kernel launches issued by this library (every
// <<<>>> site is written `note_launch(), kernel<<<...>>>(...)`); exported as
// phb_launch_count() so bench.py reports launches it counted, not a constant.
extern unsigned long long g_launch_count;
inline int note_launch() {
  __atomic_fetch_add(&g_launch_count, 1ull, __ATOMIC_RELAXED);
  return 0;
}

int num_sms();
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st);

int launch_murmur(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t n,
                  uint64_t seed, uint64_t* hi, uint64_t* lo, cudaStream_t st);
int launch_hash_count(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64,
                      int64_t n, uint64_t seed, uint64_t nparts, uint32_t* counts,
                      cudaStream_t st, uint64_t* hashes_out = nullptr);
int launch_scatter_hashed(const uint64_t* hashes, int64_t n, uint64_t nparts,
                          const double* entries, uint32_t bcount, const int64_t* key_off,
                          uint32_t* cursor, uint64_t* rec_out, cudaStream_t st);
int launch_scatter_padded(const uint64_t* keys64, int64_t n, uint64_t seed, uint64_t nparts,
                          const double* entries, uint32_t bcount, uint32_t cap, int init,
                          uint32_t* cursor, uint64_t* lo_out, uint16_t* bid_out,
                          uint32_t* overflow, cudaStream_t st);
int launch_padded_counts(const uint32_t* cursor, int64_t nparts, uint32_t cap, uint32_t* counts,
                         uint32_t* overflow, cudaStream_t st);
int launch_scatter(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t n,
                   uint64_t seed, uint64_t nparts, const double* entries, uint32_t bcount,
                   const int64_t* key_off, uint32_t* cursor, uint64_t* lo_out, uint16_t* bid_out,
                   cudaStream_t st);
int launch_bucket_ids(const uint64_t* his, int64_t n, const double* entries, uint32_t bcount,
                      uint16_t* bid, cudaStream_t st);

// layout.cu
size_t layout_temp_bytes(int64_t nparts);
// counts[nparts] -> key_off[nparts+1], deltas[nparts+1] (relative to
// expected offsets of the global layout: global_n / global_nparts, shifted
// by part_base / key_base for sharded builds), stats[0] = max |delta|,
// stats[1] = max partition size.
int launch_layout(uint32_t* counts, int64_t nparts, int64_t key_base, int64_t part_base,
                  int64_t global_n, int64_t global_nparts, int64_t* key_off, int64_t* deltas,
                  int64_t* stats, void* temp, size_t temp_bytes, cudaStream_t st);

int launch_regroup(const uint64_t* lo_in, const uint16_t* aux_in, const int32_t* C, int64_t G,
                   int64_t np, uint64_t* lo_out, uint16_t* aux_out, int64_t* key_off,
                   cudaStream_t st);

int launch_scatter_p2p(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64,
                       int64_t n, uint64_t seed, int64_t nparts, const double* entries,
                       uint32_t bcount, const int64_t* part_base, const uint8_t* owner,
                       uint64_t* const* lo_dst, uint16_t* const* bid_dst, int32_t G,
                       uint32_t* cursor, cudaStream_t st);

// search.cu
struct SearchArgs {
  const uint64_t* lo;
  const uint16_t* bid;
  const int64_t* key_off;  // absolute offsets into lo/bid/glo
  int64_t p_lo, p_hi;      // partition range [p_lo, p_hi)
  int64_t out_base;        // output row of partition j is j - out_base
  uint32_t bcount;
  int64_t seed_cap;
  int tie_desc;            // reference flag: 1 for "asc-expected"
  uint64_t* seeds;         // seeds[(j-out_base)*s_sj + (b-1)*s_sb]
  int64_t s_sj, s_sb;
  int64_t* trials;         // optional per-bucket trials, same strides
  int64_t* part_trials;    // optional per-partition totals [(j-out_base)]
  uint8_t* status;         // status[(j-out_base)]: 0 ok, 1 dup, 2 cap
  uint64_t* glo;           // scratch, indexed like lo
  uint32_t* queue;         // zeroed work counter
  int64_t m_max;           // largest partition size in the range
  int64_t rec_stride = 0;  // >0: partition j's records start at (j - p_lo) * rec_stride
};
int launch_search(const SearchArgs& a, cudaStream_t st);


// query.cu
int launch_query(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64,
                 const uint64_t* his, const uint64_t* los, int64_t nq, uint64_t seed, int64_t n,
                 int64_t nparts, const int64_t* key_off, const double* entries, uint32_t bcount,
                 const uint64_t* seeds, int64_t s_sj, int64_t s_sb, int64_t* out,
                 cudaStream_t st);
int launch_query32(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t nq,
                   uint64_t seed, int64_t n, int64_t nparts, const int64_t* key_off,
                   const uint2* part2,
                   const double* entries, uint32_t bcount, const uint32_t* seeds32, int64_t* out,
                   cudaStream_t st);
int launch_part_table32(const int64_t* key_off, int64_t nparts, uint2* part2, cudaStream_t st);
int launch_seed_table32(const uint64_t* seeds, const int64_t* key_off, int64_t nparts,
                        int64_t count, uint32_t* out, uint32_t* overflow, cudaStream_t st);
int launch_query_encoded(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64,
                         int64_t nq, uint64_t seed, int64_t n, int64_t nparts,
                         const int64_t* key_off, const double* entries, uint32_t bcount,
                         const uint8_t* section, const int64_t* cols, int mono,
                         const uint32_t* dsel, int64_t dstride, int64_t* out, cudaStream_t st);
int launch_select_index(const uint8_t* section, const int64_t* cols, int64_t ncols,
                        int64_t stride, uint32_t* dsel, cudaStream_t st);
int launch_verify(const int64_t* out, int64_t nq, int64_t n, uint32_t* bitmap, uint32_t* bad,
                  cudaStream_t st);

}  // namespace phb
