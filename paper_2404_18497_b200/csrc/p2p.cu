// Fused multi-GPU route: K3 scatter + all-to-all in one kernel over NVLink
// peer memory (distributed.py, transport="p2p").
//
// Every source rank knows, from the all-gathered per-partition counts, the
// exact slot range its records of partition j occupy inside the owner
// rank's receive buffer (rank order inside a partition). The kernel hashes
// each local key once, computes its bucket id, and stores (lo, bucket id)
// -- one 16-byte record per key when bid_dst is NULL, the layout the build
// uses -- straight into the owner's buffer through a CUDA-IPC-mapped peer pointer:
// the records land partition-grouped, so the owner runs K4 on them with no
// receive-side regroup and no staging copy. Peer stores over NVLink 5 /
// NVSwitch overlap the hashing of the next keys; the host orders the
// kernel before the owners' reads with a stream sync + group barrier.
#include <algorithm>

#include "common.cuh"
#include "phobic_internal.h"

namespace phb {

struct PeerTable {
  uint64_t* lo[64];
  uint16_t* bid[64];
};

template <class K, bool REC>
__global__ void __launch_bounds__(256)
    k_scatter_p2p(K keys, int64_t n, uint64_t seed, uint64_t nparts,
                  const double* __restrict__ entries, uint32_t bcount,
                  const uint8_t* __restrict__ owner, uint32_t* __restrict__ cursor, PeerTable peers) {
  __shared__ double2 tab[BUCKET_TAB];
  load_bucket_pairs(entries, tab);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Hash128 h = keys.hash(i, seed);
    const uint32_t j = (uint32_t)mulhi(h.hi, nparts);
    const uint32_t b = bucket_of_pairs(tab, h.hi, bcount);
    const uint32_t g = __ldg(owner + j);
    const uint32_t pos = atomicAdd(cursor + j, 1u);
    if (REC) {  // one 16-byte peer store per key: {lo, bucket id}
      reinterpret_cast<ulonglong2*>(peers.lo[g])[pos] = make_ulonglong2(h.lo, b);
    } else {
      peers.lo[g][pos] = h.lo;
      peers.bid[g][pos] = (uint16_t)b;
    }
  }
}

struct U64KeysP {
  const uint64_t* __restrict__ keys;
  __device__ __forceinline__ Hash128 hash(int64_t i, uint64_t seed) const {
    return murmur3_u64(__ldg(keys + i), seed);
  }
};
struct ByteKeysP {
  const uint8_t* __restrict__ buf;
  const int64_t* __restrict__ offsets;
  __device__ __forceinline__ Hash128 hash(int64_t i, uint64_t seed) const {
    int64_t a = __ldg(offsets + i), b = __ldg(offsets + i + 1);
    return murmur3_bytes(buf + a, b - a, seed);
  }
};

__global__ void k_cursor_from_i64(const int64_t* __restrict__ base, int64_t nparts,
                                  uint32_t* __restrict__ cursor) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nparts;
       j += (int64_t)gridDim.x * blockDim.x)
    cursor[j] = (uint32_t)base[j];
}

int launch_scatter_p2p(const uint8_t* buf, const int64_t* offsets, const uint64_t* keys64,
                       int64_t n, uint64_t seed, int64_t nparts, const double* entries,
                       uint32_t bcount, const int64_t* part_base, const uint8_t* owner,
                       uint64_t* const* lo_dst, uint16_t* const* bid_dst, int32_t G,
                       uint32_t* cursor, cudaStream_t st) {
  if (G < 1 || G > 64 || nparts < 1) return 1003;
  PeerTable t;
  const bool rec = bid_dst == nullptr;  // 16-byte records in lo_dst
  for (int g = 0; g < G; ++g) t.lo[g] = lo_dst[g], t.bid[g] = rec ? nullptr : bid_dst[g];
  note_launch(), k_cursor_from_i64<<<(int)std::min<int64_t>((nparts + 255) / 256, 4096), 256, 0, st>>>(
      part_base, nparts, cursor);
  PHB_CUDA_TRY(cudaGetLastError());
  if (n <= 0) return 0;
  int64_t need = (n + 255) / 256;
  int grid = (int)std::min<int64_t>(need, (int64_t)num_sms() * 16);
  if (keys64 && rec)
    note_launch(), k_scatter_p2p<U64KeysP, true><<<grid, 256, 0, st>>>(
        U64KeysP{keys64}, n, seed, (uint64_t)nparts, entries, bcount, owner, cursor, t);
  else if (keys64)
    note_launch(), k_scatter_p2p<U64KeysP, false><<<grid, 256, 0, st>>>(
        U64KeysP{keys64}, n, seed, (uint64_t)nparts, entries, bcount, owner, cursor, t);
  else if (rec)
    note_launch(), k_scatter_p2p<ByteKeysP, true><<<grid, 256, 0, st>>>(
        ByteKeysP{buf, offsets}, n, seed, (uint64_t)nparts, entries, bcount, owner, cursor, t);
  else
    note_launch(), k_scatter_p2p<ByteKeysP, false><<<grid, 256, 0, st>>>(
        ByteKeysP{buf, offsets}, n, seed, (uint64_t)nparts, entries, bcount, owner, cursor, t);
  return (int)cudaGetLastError();
}

}  // namespace phb
