// Encoder plan structures shared by encode.cu and the C-ABI layer.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace phb {

// Bytes of the fixed Mphf header before the delta-width byte
// (mphf.py:158-168): "PHOB" u32 u64 u64 f64 f64 u8 f64 u64.
constexpr uint64_t HEADER_FIXED = 57;

struct EncodeArgs {
  const uint64_t* seeds;        // column-major [bcount][nparts]
  int64_t nparts;               // rows (partitions) in `seeds`
  uint32_t bcount;
  int mono;                     // 1: MonoSeeds (one column, row-major order)
  int compact_prefix;           // columns [0, t) Compact, the rest Rice
  const int64_t* deltas;        // [nparts_global + 1] or null (no delta section write)
  int64_t nparts_global;
  const int64_t* layout_stats;  // device: [0] = max |delta|
  const uint8_t* status;        // optional [nparts]
  const int64_t* part_trials;   // optional [nparts]
  // sharded (multi-GPU) encoding: this shard holds rows [row0, row0 + nparts)
  // of a column of count_global values; 0 / null = a whole-matrix encode
  int64_t row0 = 0;
  int64_t count_global = 0;            // values per column over all shards
  const unsigned long long* colstat_in = nullptr;   // reduced stats [ncols][65]
  unsigned long long* rice_totals_out = nullptr;    // this shard's sum(high + 1) per column
  const unsigned long long* rice_base = nullptr;    // unary bits of earlier shards per column
  int write_headers = 1;               // headers + deltas (one shard writes them)
};

struct ColInfo {
  uint64_t count, block_off, block_bytes, pay_bit, highs_bit, samples_byte, highs_nbits;
  uint32_t nsamples;
  uint8_t kind, param;
};

struct EncodeSummary {
  uint64_t total_bytes;   // serialized body length, checksum excluded
  uint64_t seed_section;  // byte offset of u32 num_encoders
  uint64_t trials_total;
  int64_t first_bad;      // first partition with status != 0, or -1
  int32_t bad_code;
  int32_t delta_width;
  int64_t ncols;
};

size_t encode_workspace_bytes(int64_t nparts, uint32_t bcount, int mono);
int launch_encode_stats(const EncodeArgs& a, void* ws, unsigned long long* colstat_out,
                        cudaStream_t st);
int launch_encode_plan(const EncodeArgs& a, void* ws, EncodeSummary* host_sum, cudaStream_t st);
int launch_encode_write(const EncodeArgs& a, void* ws, uint8_t* blob, size_t blob_bytes,
                        cudaStream_t st);

}  // namespace phb
