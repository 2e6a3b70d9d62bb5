// K3 grouping-pass variants at C2 size (100M u64 keys, 40k partitions):
// where does the scatter's time go? Standalone (nvcc -I csrc), timed with
// CUDA events; run under ncu for DRAM bytes per variant.
//   V0 global atomic cursors, 16-byte records (the build's K3)
//   V1 CTA-private cursors (shared-memory atomics), 16-byte records
//   V2 CTA-private cursors, 32-byte records (one full sector per key)
//   V3 global atomic cursors, 32-byte records
//   V4 atomics only (RED, result unused), coalesced 16-byte stores
#include <cstdio>
#include <vector>
#include "../../paper_2404_18497_b200/csrc/common.cuh"
using namespace phb;

__global__ void k_keys(uint64_t* k, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    k[i] = mix64((uint64_t)i * 0x9E3779B97F4A7C15ull + 1);
}
__global__ void k_count(const uint64_t* k, int64_t n, uint64_t np, uint32_t* c) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(c + mulhi(murmur3_u64(k[i], 0).hi, np), 1u);
}
// per-CTA histograms with the same contiguous split as the CTA scatter
__global__ void k_count_cta(const uint64_t* k, int64_t n, uint64_t np, uint32_t* cc) {
  extern __shared__ uint32_t h[];
  for (uint32_t j = threadIdx.x; j < np; j += blockDim.x) h[j] = 0;
  __syncthreads();
  int64_t a = n * blockIdx.x / gridDim.x, b = n * (blockIdx.x + 1) / gridDim.x;
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) atomicAdd(h + mulhi(murmur3_u64(k[i], 0).hi, np), 1u);
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < np; j += blockDim.x) cc[(uint64_t)blockIdx.x * np + j] = h[j];
}
template <int REC>
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
    for (int e = 0; e < 8; ++e) out[(uint64_t)pos[e] * REC] = make_ulonglong2(lo[e], 7);
  }
}
template <int REC>
__global__ void __launch_bounds__(1024, 1) k_v1(const uint64_t* k, int64_t n, uint64_t np, const uint32_t* base, ulonglong2* out) {
  extern __shared__ uint32_t cur[];
  for (uint32_t j = threadIdx.x; j < np; j += blockDim.x) cur[j] = base[(uint64_t)blockIdx.x * np + j];
  __syncthreads();
  int64_t a = n * blockIdx.x / gridDim.x, b = n * (blockIdx.x + 1) / gridDim.x;
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
    Hash128 h = murmur3_u64(__ldcs(k + i), 0);
    uint32_t pos = atomicAdd(cur + mulhi(h.hi, np), 1u);
    out[(uint64_t)pos * REC] = make_ulonglong2(h.lo, 7);
  }
}
__global__ void __launch_bounds__(256) k_v4(const uint64_t* k, int64_t n, uint64_t np, uint32_t* cur, ulonglong2* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    Hash128 h = murmur3_u64(__ldcs(k + i), 0);
    atomicAdd(cur + mulhi(h.hi, np), 1u);
    out[i] = make_ulonglong2(h.lo, 7);
  }
}
// per-partition prefix over CTAs -> absolute bases
__global__ void k_prefix(const uint32_t* cnt, int64_t np, int g, uint32_t* cc) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= np) return;
  uint32_t run = 0;
  for (int c = 0; c < g; ++c) { uint32_t v = cc[(int64_t)c * np + j]; cc[(int64_t)c * np + j] = run; run += v; }
}
__global__ void k_add_off(const uint32_t* off, int64_t np, int g, uint32_t* cc) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= np) return;
  for (int c = 0; c < g; ++c) cc[(int64_t)c * np + j] += off[j];
}

int main() {
  const int64_t n = 100000000; const uint64_t np = 40000;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint64_t* keys; ulonglong2* out; uint32_t *cnt, *cur, *cc, *off;
  cudaMalloc(&keys, n * 8); cudaMalloc(&out, (size_t)n * 32); cudaMalloc(&cnt, np * 4); cudaMalloc(&cur, np * 4);
  cudaMalloc(&cc, (size_t)sms * np * 4); cudaMalloc(&off, np * 4);
  k_keys<<<4096, 256>>>(keys, n);
  cudaMemset(cnt, 0, np * 4);
  k_count<<<4096, 256>>>(keys, n, np, cnt);
  std::vector<uint32_t> h(np), o(np);
  cudaMemcpy(h.data(), cnt, np * 4, cudaMemcpyDeviceToHost);
  uint32_t run = 0; for (uint64_t j = 0; j < np; ++j) { o[j] = run; run += h[j]; }
  cudaMemcpy(off, o.data(), np * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_count_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k_v1<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k_v1<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  k_count_cta<<<sms, 1024, np * 4>>>(keys, n, np, cc);
  k_prefix<<<(np + 255) / 256, 256>>>(cnt, np, sms, cc);
  k_add_off<<<(np + 255) / 256, 256>>>(off, np, sms, cc);
  uint32_t* ccb; cudaMalloc(&ccb, (size_t)sms * np * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"V0 global atomics, 16 B rec", "V1 CTA cursors, 16 B rec", "V2 CTA cursors, 32 B rec",
                         "V3 global atomics, 32 B rec", "V4 atomics only + coalesced stores"};
  int gk = sms * 16;
  for (int v = 0; v < 5; ++v) {
    float best = 1e9;
    for (int r = 0; r < 4; ++r) {
      cudaMemcpy(cur, off, np * 4, cudaMemcpyDeviceToDevice);
      cudaMemcpy(ccb, cc, (size_t)sms * np * 4, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      if (v == 0) k_v0<1><<<gk, 256>>>(keys, n, np, cur, out);
      if (v == 1) k_v1<1><<<sms, 1024, np * 4>>>(keys, n, np, ccb, out);
      if (v == 2) k_v1<2><<<sms, 1024, np * 4>>>(keys, n, np, ccb, out);
      if (v == 3) k_v0<2><<<gk, 256>>>(keys, n, np, cur, out);
      if (v == 4) k_v4<<<gk, 256>>>(keys, n, np, cur, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("%-40s %7.3f ms  %s\n", names[v], best, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
