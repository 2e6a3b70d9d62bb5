// K3 with cluster-shared cursors (distributed shared memory), standalone at
// C2 size. A cluster of CS CTAs owns a contiguous key range; partition j's
// counter / cursor lives in CTA (j % CS)'s shared memory. K1c counts per
// cluster with remote shared-memory atomics; a prefix over clusters gives
// every cluster its own base per partition; K3c places keys with remote
// returning atomics (no global atomics) -> one write stream per (cluster,
// partition) instead of per (CTA, partition). Checks per-partition sums.
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
#include "../../paper_2404_18497_b200/csrc/common.cuh"
namespace cg = cooperative_groups;
using namespace phb;

__global__ void k_keys(uint64_t* k, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    k[i] = mix64((uint64_t)i * 0x9E3779B97F4A7C15ull + 1);
}
__global__ void k_count(const uint64_t* k, int64_t n, uint64_t np, uint32_t* c) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(c + mulhi(murmur3_u64(k[i], 0).hi, np), 1u);
}
__global__ void __launch_bounds__(256) k_v0(const uint64_t* k, int64_t n, uint64_t np, uint32_t* cur, ulonglong2* out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n / 8; q += (int64_t)gridDim.x * blockDim.x) {
    uint32_t pos[8]; uint64_t lo[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      Hash128 h = murmur3_u64(__ldcs(k + 8 * q + e), 0);
      lo[e] = h.lo;
      pos[e] = atomicAdd(cur + mulhi(h.hi, np), 1u);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) out[pos[e]] = make_ulonglong2(lo[e], 7);
  }
}
// key range of this CTA: cluster c owns [c n / NC, (c+1) n / NC), its CTAs split it
__device__ __forceinline__ void my_range(int64_t n, int64_t& a, int64_t& b) {
  const int cs = (int)cg::this_cluster().num_blocks();
  const int64_t c = blockIdx.x / cs, r = blockIdx.x % cs, nc = gridDim.x / cs;
  const int64_t ca = n * c / nc, cb = n * (c + 1) / nc;
  a = ca + (cb - ca) * r / cs;
  b = ca + (cb - ca) * (r + 1) / cs;
}
__global__ void __launch_bounds__(1024, 1) k_count_cl(const uint64_t* k, int64_t n, uint64_t np, uint32_t* cc) {
  extern __shared__ uint32_t h[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t cs = cl.num_blocks(), rank = cl.block_rank();
  const uint32_t slice = (uint32_t)((np + cs - 1) / cs);
  for (uint32_t t = threadIdx.x; t < slice; t += blockDim.x) h[t] = 0;
  cl.sync();
  int64_t a, b; my_range(n, a, b);
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
    const uint32_t j = (uint32_t)mulhi(murmur3_u64(__ldcs(k + i), 0).hi, np);
    atomicAdd(cl.map_shared_rank(h, j % cs) + j / cs, 1u);
  }
  cl.sync();
  const int64_t c = blockIdx.x / cs;
  for (uint32_t t = threadIdx.x; t < slice; t += blockDim.x) {
    const uint64_t j = (uint64_t)t * cs + rank;
    if (j < np) cc[c * np + j] = h[t];
  }
}
__global__ void k_prefix(const uint32_t* off, int64_t np, int nc, uint32_t* cc) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= np) return;
  uint32_t run = off[j];
  for (int c = 0; c < nc; ++c) { uint32_t v = cc[(int64_t)c * np + j]; cc[(int64_t)c * np + j] = run; run += v; }
}
__global__ void __launch_bounds__(1024, 1) k_scatter_cl(const uint64_t* k, int64_t n, uint64_t np, const uint32_t* cc, ulonglong2* out) {
  extern __shared__ uint32_t cur[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t cs = cl.num_blocks(), rank = cl.block_rank();
  const uint32_t slice = (uint32_t)((np + cs - 1) / cs);
  const int64_t c = blockIdx.x / cs;
  for (uint32_t t = threadIdx.x; t < slice; t += blockDim.x) {
    const uint64_t j = (uint64_t)t * cs + rank;
    cur[t] = j < np ? cc[c * np + j] : 0;
  }
  cl.sync();
  int64_t a, b; my_range(n, a, b);
  for (int64_t i0 = a + 4 * threadIdx.x; i0 < b; i0 += 4 * blockDim.x) {
    uint32_t pos[4]; uint64_t lo[4]; bool ok[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      ok[e] = i0 + e < b;
      if (ok[e]) {
        Hash128 h = murmur3_u64(__ldcs(k + i0 + e), 0);
        const uint32_t j = (uint32_t)mulhi(h.hi, np);
        lo[e] = h.lo;
        pos[e] = atomicAdd(cl.map_shared_rank(cur, j % cs) + j / cs, 1u);
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) if (ok[e]) out[pos[e]] = make_ulonglong2(lo[e], 7);
  }
  cl.sync();  // remote cursors stay alive until every CTA of the cluster is done
}
__global__ void k_sums(const ulonglong2* out, const uint32_t* off, int64_t np, unsigned long long* sums) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= np) return;
  unsigned long long s = 0;
  for (uint32_t q = off[j]; q < off[j + 1]; ++q) s += out[q].x * 0x9E3779B97F4A7C15ull + out[q].y;
  sums[j] = s;
}

int main(int argc, char** argv) {
  const int64_t n = 100000000; const uint64_t np = 40000;
  uint64_t* keys; ulonglong2 *out0, *out1; uint32_t *cnt, *cur, *off, *cc; unsigned long long *s0, *s1;
  cudaMalloc(&keys, n * 8); cudaMalloc(&out0, n * 16); cudaMalloc(&out1, n * 16);
  cudaMalloc(&cnt, np * 4); cudaMalloc(&cur, np * 4); cudaMalloc(&off, (np + 1) * 4);
  cudaMalloc(&cc, 64 * np * 4); cudaMalloc(&s0, np * 8); cudaMalloc(&s1, np * 8);
  k_keys<<<4096, 256>>>(keys, n);
  cudaMemset(cnt, 0, np * 4);
  k_count<<<4096, 256>>>(keys, n, np, cnt);
  std::vector<uint32_t> h(np), o(np + 1);
  cudaMemcpy(h.data(), cnt, np * 4, cudaMemcpyDeviceToHost);
  uint32_t run = 0; for (uint64_t j = 0; j < np; ++j) { o[j] = run; run += h[j]; } o[np] = run;
  cudaMemcpy(off, o.data(), (np + 1) * 4, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1, e2, e3; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3);
  float best = 1e9;
  for (int r = 0; r < 4; ++r) {
    cudaMemcpy(cur, off, np * 4, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0); k_v0<<<sms * 16, 256>>>(keys, n, np, cur, out0); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
  }
  printf("atomic K3 %.3f ms\n", best);
  k_sums<<<(np + 255) / 256, 256>>>(out0, off, np, s0);
  std::vector<unsigned long long> h0(np), h1(np);
  cudaMemcpy(h0.data(), s0, np * 8, cudaMemcpyDeviceToHost);
  for (int cs : {4, 8, 16}) {
    const size_t sh = ((np + cs - 1) / cs) * 4;
    cudaFuncSetAttribute(k_count_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_scatter_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_count_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);
    cudaFuncSetAttribute(k_scatter_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = sh;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cfg.gridDim = dim3(cs);
    int ncl = 0;
    cudaError_t oe = cudaOccupancyMaxActiveClusters(&ncl, (void*)k_scatter_cl, &cfg);
    if (oe != cudaSuccess || ncl < 1) { printf("cs %d: no cluster occupancy (%s)\n", cs, cudaGetErrorString(oe)); cudaGetLastError(); continue; }
    cfg.gridDim = dim3(ncl * cs);
    float bc = 1e9, bs = 1e9;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, k_count_cl, (const uint64_t*)keys, n, np, cc);
      cudaEventRecord(e1);
      k_prefix<<<(np + 255) / 256, 256>>>(off, np, ncl, cc);
      cudaEventRecord(e2);
      cudaLaunchKernelEx(&cfg, k_scatter_cl, (const uint64_t*)keys, n, np, (const uint32_t*)cc, out1);
      cudaEventRecord(e3); cudaEventSynchronize(e3);
      float a, b; cudaEventElapsedTime(&a, e0, e1); cudaEventElapsedTime(&b, e2, e3);
      bc = std::min(bc, a); bs = std::min(bs, b);
    }
    k_sums<<<(np + 255) / 256, 256>>>(out1, off, np, s1);
    cudaMemcpy(h1.data(), s1, np * 8, cudaMemcpyDeviceToHost);
    int bad = 0; for (uint64_t j = 0; j < np; ++j) bad += h0[j] != h1[j];
    printf("cluster %2d x %d clusters: count %.3f ms  scatter %.3f ms  differing partitions %d  %s\n", cs, ncl, bc, bs, bad,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
