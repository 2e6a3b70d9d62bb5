/*
 * phobic.h — C-ABI of the B200-native PHOBIC construction engine
 * (libphobic_b200.so, built from paper_2404_18497_b200/csrc/).
 *
 * Conventions (mirroring the reference operator layer, pilothash._kernels,
 * /root/reference/pkg/src/pilothash/_kernels.py:1-9):
 *   - every pointer argument is a DEVICE pointer (cudaMalloc / torch CUDA
 *     memory) unless documented as host memory;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *   - the caller allocates and, where the reference zero-fills
 *     (builder.py:238-240), zero-fills every output; kernels write in place
 *     and keep no allocation across calls;
 *   - every function returns 0 on success, a cudaError_t value (1..999) for
 *     CUDA / launch errors, or one of the PHB_E_* codes below. Per-partition
 *     search failures are DATA (status_out), exactly as in the reference.
 *
 * Key ABI: a 64-bit key is its 8-byte little-endian string (SURVEY.md §0
 * finding 4); byte keys are a flat buffer plus int64 offsets[n+1]
 * (keygen.KeyCorpus, keygen.py:25-57).
 */
#ifndef PHOBIC_B200_H
#define PHOBIC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PHB_OK 0
#define PHB_E_BUCKETS 1001             /* bucket count outside [1, 65535] */
#define PHB_E_PARTITION_TOO_LARGE 1002 /* a partition's search state exceeds shared memory */
#define PHB_E_ARGS 1003                /* invalid sizes / misaligned buffers */

const char* phb_version(void);
const char* phb_error_string(int code);
int phb_device_sms(void);
/* Kernel launches this library has issued in this process (all entry
 * points; relaxed atomic counter). Host-only, no CUDA context needed. */
unsigned long long phb_launch_count(void);

/* ---------------------------------------------------------------------
 * Reference-shaped operators: one-for-one replacements of the three
 * pilothash._kernels entry points (same argument meaning and layout).
 * ------------------------------------------------------------------- */

/* replaces _kernels.murmur3_many(buf, offsets, seed, out_hi, out_lo)
 * (_kernels.py:89-146), called by hashing.master_hash_many (hashing.py:65-76).
 * offsets has n+1 entries. */
int phb_murmur3_many(const uint8_t* buf, const int64_t* offsets, int64_t n, uint64_t seed,
                     uint64_t* out_hi, uint64_t* out_lo, void* stream);

/* u64 fast path of the same hash: keys[i] hashed as its 8-byte LE string. */
int phb_murmur3_u64(const uint64_t* keys, int64_t n, uint64_t seed, uint64_t* out_hi,
                    uint64_t* out_lo, void* stream);

/* replaces _kernels.build_partition_range(his, los, key_off, p_lo, p_hi,
 * entries, bcount, seed_cap, tie_desc, seeds_out, trials_out, status_out)
 * (_kernels.py:221-371), called by builder.build_all_partitions
 * (builder.py:244-258). Keys must arrive grouped by partition (any order
 * inside a partition). entries: the 2049 f64 table built on the host
 * (assignment.tabulate, assignment.py:115-121). tie_desc follows the
 * reference flag (1 for "asc-expected", builder.py:241). Outputs:
 * seeds_out[j*bcount + b-1] (u64), trials_out (i64, same index, may be
 * NULL), status_out[j] (0 ok, 1 duplicate low words, 2 seed cap). */
int phb_build_partition_range(const uint64_t* his, const uint64_t* los, const int64_t* key_off,
                              int64_t p_lo, int64_t p_hi, const double* entries, int32_t bcount,
                              int64_t seed_cap, int32_t tie_desc, uint64_t* seeds_out,
                              int64_t* trials_out, uint8_t* status_out, void* stream);

/* replaces _kernels.query_many_kernel(his, los, n, nparts, deltas, entries,
 * bcount, seed_mat, out) (_kernels.py:379-397), called by Mphf.query_many
 * (mphf.py:130-145). seed_mat is row-major [nparts, bcount] u64. */
int phb_query_many(const uint64_t* his, const uint64_t* los, int64_t nq, int64_t n,
                   int64_t nparts, const int64_t* deltas, const double* entries, int32_t bcount,
                   const uint64_t* seed_mat, int64_t* out, void* stream);

/* Bucket ids of master-hash high words: clamp(ceil(gamma(x) * B), 1, B) with
 * x = (f64(mix64(hi ^ SALT)) + 1) 2^-64 (_kernels._bucket_of, _kernels.py:158-167;
 * assignment.bucket_many, assignment.py:146-149). out: u16[n]. */
int phb_bucket_ids(const uint64_t* his, int64_t n, const double* entries, int32_t bcount,
                   uint16_t* out, void* stream);

/* ---------------------------------------------------------------------
 * Staged build pipeline (what pilothash.mphf.build, mphf.py:236-290,
 * becomes on B200). keys64 != NULL selects the u64 path, otherwise
 * (buf, offsets) byte keys.
 * ------------------------------------------------------------------- */

/* K1: murmur3 + partition index + per-partition counts (counts zeroed by
 * caller). Replaces master_hash_many + partition_index_many + bincount
 * (partitioning.py:73-96). */
int phb_hash_count(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t n,
                   uint64_t seed, int64_t nparts, uint32_t* counts, void* stream);

/* K1 for byte keys that also keeps the 128-bit hashes: hashes_out[2i] = hi,
 * hashes_out[2i+1] = lo (16-byte aligned, 2n u64), so K3 can run from them
 * (phb_scatter_hashed) instead of hashing the key bytes again. */
int phb_hash_count_store(const uint8_t* buf, const int64_t* offsets, int64_t n, uint64_t seed,
                         int64_t nparts, uint32_t* counts, uint64_t* hashes_out, void* stream);

/* K3 from stored hashes: the same 16-byte {lo, bucket id} records as
 * phb_scatter with bid_out == NULL (rec_out: 2n u64). */
int phb_scatter_hashed(const uint64_t* hashes, int64_t n, int64_t nparts, const double* entries,
                       int32_t bcount, const int64_t* key_off, uint32_t* cursor, uint64_t* rec_out,
                       void* stream);

/* K2: counts[nparts] -> key_off[nparts+1] (local, from 0) and
 * deltas[nparts+1] = key_base + key_off[j] - expected(part_base + j,
 * global_n, global_nparts) (partitioning.py:101-108); stats[0] = max |delta|,
 * stats[1] = max partition size. For a single-GPU build pass key_base =
 * part_base = 0, global_n = n, global_nparts = nparts. counts (8-byte
 * aligned) is CLOBBERED: the multi-CTA scan keeps its tile states over the
 * tiles' first counts (no scratch allocation). */
int phb_layout(uint32_t* counts, int64_t nparts, int64_t key_base, int64_t part_base,
               int64_t global_n, int64_t global_nparts, int64_t* key_off, int64_t* deltas,
               int64_t* stats, void* stream);

/* K3: re-hash and scatter (lo, bucket id) into partition ranges (cursor:
 * nparts u32 of scratch, contents ignored; n < 2^32). Replaces the lexsort grouping (partitioning.py:93-95)
 * and _bucket_of (_kernels.py:252-255). bid_out == NULL: 16-byte records
 * {lo, bucket id} into lo_out (2n u64), one scattered store per key. */
int phb_scatter(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t n,
                uint64_t seed, int64_t nparts, const double* entries, int32_t bcount,
                const int64_t* key_off, uint32_t* cursor, uint64_t* lo_out, uint16_t* bid_out,
                void* stream);

/* K4: bucket order + seed search for partitions [p_lo, p_hi) over records
 * grouped by partition (separate lo / bid arrays, or bid == NULL: lo holds
 * the 16-byte {lo, bucket id} records of phb_scatter). Seeds land at seeds[(j-out_base)*s_sj + (b-1)*s_sb];
 * trials (may be NULL) at the same index; part_trials[(j-out_base)] (may be
 * NULL); status[(j-out_base)]. glo: scratch indexed like lo. queue: one
 * device u32. m_max: largest partition size in the range (layout stats[1]). */
int phb_search(const uint64_t* lo, const uint16_t* bid, const int64_t* key_off, int64_t p_lo,
               int64_t p_hi, int64_t out_base, int32_t bcount, int64_t seed_cap, int32_t tie_desc,
               int64_t m_max, uint64_t* seeds, int64_t s_sj, int64_t s_sb, int64_t* trials,
               int64_t* part_trials, uint8_t* status, uint64_t* glo, uint32_t* queue,
               void* stream);

/* K3 into fixed-capacity partition slots, for u64 keys arriving in chunks
 * (no counting pass first): partition j's records go to [j*cap, j*cap + cap)
 * of lo_out / bid_out (bid_out == NULL: 16-byte records in lo_out, as for
 * phb_scatter) through cursor[j] (init != 0 on the first chunk sets
 * cursor[j] = j*cap; nparts*cap < 2^32). phb_padded_counts then turns the
 * cursors into the exact per-partition counts (input of phb_layout) and sets
 * *overflow if any partition exceeded cap (records past it are dropped: the
 * caller falls back to phb_hash_count + phb_layout + phb_scatter). keys64
 * must be 16-byte aligned. */
int phb_scatter_padded(const uint64_t* keys64, int64_t n, uint64_t seed, int64_t nparts,
                       const double* entries, int32_t bcount, int32_t cap, int32_t init,
                       uint32_t* cursor, uint64_t* lo_out, uint16_t* bid_out,
                       uint32_t* overflow, void* stream);
int phb_padded_counts(const uint32_t* cursor, int64_t nparts, int32_t cap, uint32_t* counts,
                      uint32_t* overflow, void* stream);

/* K4 over records laid out with a fixed stride (phb_scatter_padded): the
 * records of partition j start at (j - p_lo) * rec_stride; key_off still
 * gives the exact offsets (sizes m = key_off[j+1] - key_off[j]). */
int phb_search_strided(const uint64_t* lo, const uint16_t* bid, const int64_t* key_off,
                       int64_t p_lo, int64_t p_hi, int64_t out_base, int32_t bcount,
                       int64_t seed_cap, int32_t tie_desc, int64_t m_max, uint64_t* seeds,
                       int64_t s_sj, int64_t s_sb, int64_t* trials, int64_t* part_trials,
                       uint8_t* status, uint64_t* glo, uint32_t* queue, int64_t rec_stride,
                       void* stream);

/* K5/K6: interleaved / mono Compact-Rice encoding of a column-major seed
 * matrix seeds[bcount][nparts] plus the packed deltas, into the serialized
 * body of Mphf.serialize (mphf.py:156-175) from byte 57 on (the fixed header
 * and the blake2b checksum are host work). Two phases: plan (sizes; writes
 * 8 int64 to HOST summary_out: total_bytes, seed_section, trials_total,
 * first_bad, bad_code, delta_width, ncols, 0; synchronizes `stream`) and
 * write (blob: device, 4-byte aligned, >= total_bytes + 16 bytes). */
size_t phb_encode_workspace_bytes(int64_t nparts, int32_t bcount, int32_t mono);
int phb_encode_plan(const uint64_t* seeds, int64_t nparts, int32_t bcount, int32_t mono,
                    int32_t compact_prefix, const int64_t* deltas, int64_t nparts_global,
                    const int64_t* layout_stats, const uint8_t* status,
                    const int64_t* part_trials, void* workspace, int64_t* summary_out,
                    void* stream);
int phb_encode_write(const uint64_t* seeds, int64_t nparts, int32_t bcount, int32_t mono,
                     int32_t compact_prefix, const int64_t* deltas, int64_t nparts_global,
                     const int64_t* layout_stats, void* workspace, uint8_t* blob,
                     size_t blob_bytes, void* stream);

/* Sharded K5 (multi-GPU, one call sequence per rank; distributed.py step 7).
 * A rank holds the seed rows [row0, row0 + nparts) of the global matrix
 * (column-major [bcount][nparts] locally, nparts may be 0):
 *   1. phb_encode_shard_stats: per-column max + 64 bit-population counts
 *      of the local rows -> colstat_out (DEVICE u64[ncols][65]); the caller
 *      reduces them over ranks (MAX of [c][0], SUM of [c][1..64]);
 *   2. phb_encode_shard_plan: the global plan from the reduced stats (same
 *      geometry, sizes and summary on every rank) and this rank's Rice unary
 *      totals per column -> rice_totals_out (DEVICE u64[ncols]);
 *   3. phb_encode_shard_write: this rank's fields at their global bit
 *      addresses into a zeroed body; rice_base (DEVICE u64[ncols]) = the
 *      unary totals of lower ranks; write_headers on exactly one rank.
 * Every bit of the body is written by exactly one rank, so a byte-wise SUM
 * over ranks (ncclAllReduce, uint8) is their OR: the single-GPU body.
 * workspace: phb_encode_workspace_bytes(nparts, bcount, mono). */
int phb_encode_shard_stats(const uint64_t* seeds, int64_t nparts, int32_t bcount, int32_t mono,
                           unsigned long long* colstat_out, void* stream);
int phb_encode_shard_plan(const uint64_t* seeds, int64_t nparts, int64_t row0,
                          int64_t nparts_global, int32_t bcount, int32_t mono,
                          int32_t compact_prefix, const int64_t* layout_stats,
                          const unsigned long long* colstat_global, void* workspace,
                          unsigned long long* rice_totals_out, int64_t* summary_out,
                          void* stream);
int phb_encode_shard_write(const uint64_t* seeds, int64_t nparts, int64_t row0,
                           int64_t nparts_global, int32_t bcount, int32_t mono,
                           int32_t compact_prefix, const int64_t* deltas,
                           const int64_t* layout_stats, const unsigned long long* rice_base,
                           int32_t write_headers, void* workspace, uint8_t* blob,
                           size_t blob_bytes, void* stream);

/* Decode an encoded seed section (device copy of a serialized body) back to
 * the column-major matrix seeds[bcount][nparts] (decode_matrix,
 * encoders.py:309-311 / :337-338). col_info: HOST array of 8 int64 per
 * encoder (kind, param, count, payload_byte, highs_byte, highs_nbits, 0, 0)
 * as parsed by the host from the block headers. */
int phb_decode_seeds(const uint8_t* blob, int64_t ncols, const int64_t* col_info, int64_t nparts,
                     int32_t bcount, int32_t mono, uint64_t* seeds, void* stream);

/* K7: batched query with fused hashing; key_off[nparts+1] absolute offsets
 * (expected + delta). seeds indexed [j*s_sj + (b-1)*s_sb]. */
int phb_query(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t nq,
              uint64_t seed, int64_t n, int64_t nparts, const int64_t* key_off,
              const double* entries, int32_t bcount, const uint64_t* seeds, int64_t s_sj,
              int64_t s_sb, int64_t* out, void* stream);

/* K7e: batched query reading seeds straight from the encoded seed section
 * (Compact fields, Rice lows + sampled select over the unary highs:
 * CompactVector.get / RiceVector.get, encoders.py:89-99, :224-230, :129-154),
 * no decoded matrix. section: DEVICE copy of the serialized seed section's
 * encoder blocks; col_info: DEVICE int64[num_enc][8] = {kind (0 Compact,
 * 1 Rice), width or b, count, payload byte, highs byte, highs_nbits,
 * samples byte, nsamples}, byte offsets relative to section. Interleaved:
 * num_enc == bcount, encoder b-1 indexed by partition; mono: one encoder
 * indexed j*bcount + b-1. */
/* Batched query over compact tables (seeds32 = phb_seed_table32 of the
 * column-major [B][nparts] u64 matrix; part2 = phb_part_table32 of key_off,
 * requires n < 2^32): same outputs as phb_query with half the gather
 * footprint, one 8-byte partition gather and no division, four u64 keys
 * per thread. key_off (int64 [nparts + 1], may be NULL): large u64 batches
 * whose u32 offsets fit in shared memory (~49k partitions) read them there
 * and make a single random gather per query. u64 keys and out must be 16-byte aligned (PHB_E_ARGS
 * otherwise; use phb_query). Replaces query_many_kernel (_kernels.py:379-397). */
int phb_query32(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t nq,
                uint64_t seed, int64_t n, int64_t nparts, const int64_t* key_off,
                const uint32_t* part2, const double* entries, int32_t bcount,
                const uint32_t* seeds32, int64_t* out, void* stream);
/* key_off (int64 [nparts + 1]) -> part2 (u32 (offset, end) pairs [nparts]). */
int phb_part_table32(const int64_t* key_off, int64_t nparts, uint32_t* part2, void* stream);
/* u64 seeds [B][nparts] -> u32 (s << 16) | d with p = s m + d (m from
 * key_off); *overflow (device u32, zeroed by the caller) becomes 1 if some
 * entry does not fit (s >= 2^16 or m > 2^16). */
int phb_seed_table32(const uint64_t* seeds, const int64_t* key_off, int64_t nparts, int64_t count,
                     uint32_t* out, uint32_t* overflow, void* stream);

int phb_query_encoded(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64,
                      int64_t nq, uint64_t seed, int64_t n, int64_t nparts,
                      const int64_t* key_off, const double* entries, int32_t bcount,
                      const uint8_t* section, const int64_t* col_info, int32_t num_enc,
                      int32_t mono, const uint32_t* select_dir, int64_t select_stride,
                      int64_t* out, void* stream);

/* Dense select directory for the Rice encoders of a section (optional input
 * of phb_query_encoded; NULL there = use the serialized every-1024th
 * samples): select_dir[e * stride + r] = bit position, within encoder e's
 * unary highs, of its (64 r)-th one; stride >= ceil(count / 64) of every
 * Rice encoder. Built once per loaded structure. */
int phb_select_index(const uint8_t* section, const int64_t* col_info, int64_t num_enc,
                     int64_t stride, uint32_t* select_dir, void* stream);

/* K8: bijection check onto [0, n): bitmap (ceil(n/32) u32, zeroed by
 * caller) and bad_flag (one u32, zeroed) set to 1 on a repeat or an
 * out-of-range output. Bijection <=> nq == n and bad_flag == 0. */
int phb_verify(const int64_t* out, int64_t nq, int64_t n, uint32_t* bitmap, uint32_t* bad_flag,
               void* stream);

/* key_off[j] = expected(j, n, nparts) + deltas[j], j in [0, nparts]
 * (partitioning.offset, partitioning.py:119-122). */
int phb_offsets_from_deltas(const int64_t* deltas, int64_t n, int64_t nparts, int64_t* key_off,
                            void* stream);

/* Multi-GPU regroup (paper_2404_18497_b200/distributed.py): merge the G
 * chunks received from the all-to-all, each grouped by the owned partitions
 * [0, np) with C[s*np + j] records of partition j from source s (int32,
 * row-major [G][np]), into one partition-grouped array; key_off[np+1] gets
 * the partition offsets. No reference counterpart (the reference is single
 * process). */
int phb_regroup(const uint64_t* lo_in, const uint16_t* aux_in, const int32_t* counts, int64_t G,
                int64_t np, uint64_t* lo_out, uint16_t* aux_out, int64_t* key_off, void* stream);

/* Fused multi-GPU route (distributed.py, transport="p2p"): K3 scatter and the
 * all-to-all in one kernel. Each local key's (lo, bucket id) is stored
 * directly into its owner rank's receive buffer over NVLink peer memory, at
 * part_base[j] + (rank of the key among this source's keys of partition j).
 * part_base: device i64[nparts]; owner: device u8[nparts] (owner rank of
 * partition j); lo_dst / bid_dst: HOST arrays of G device pointers (peer
 * buffers mapped with phb_ipc_open, the local one for g == rank; bid_dst
 * NULL: lo_dst buffers take 16-byte {lo, bucket id} records, one peer store
 * per key, the layout phb_search reads with bid NULL); cursor:
 * device u32[nparts] scratch. The caller orders the kernel before the
 * owners' reads (stream sync + group barrier). */
int phb_scatter_p2p(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64, int64_t n,
                    uint64_t seed, int64_t nparts, const double* entries, int32_t bcount,
                    const int64_t* part_base, const uint8_t* owner, uint64_t* const* lo_dst,
                    uint16_t* const* bid_dst, int32_t G, uint32_t* cursor, void* stream);

/* CUDA IPC plumbing for the peer buffers (64-byte cudaIpcMemHandle_t). */
int phb_ipc_alloc(size_t bytes, void** dptr);
int phb_ipc_free(void* dptr);
int phb_ipc_handle(void* dptr, uint8_t* handle64);
int phb_ipc_open(const uint8_t* handle64, void** dptr);
int phb_ipc_close(void* dptr);
int phb_sync(void* stream);

/* Search work counters (only in builds with -DPHB_STATS; else returns
 * PHB_E_ARGS): 32 u64 to HOST out16; reset != 0 clears them. */
int phb_search_stats(unsigned long long* out16, int reset);

/* Synthetic distinct 64-bit keys for benchmarks: out[i] = mix64(offset + i)
 * (mix64 is a bijection on u64, so keys are distinct for distinct i). The
 * host restatement is keygen.synth_u64. Not a reference interface: bench
 * input generation. */
int phb_synth_keys(uint64_t* out, int64_t n, uint64_t offset, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PHOBIC_B200_H */
