// scan.cuh -- hand-written CTA scan and stream compaction of byte flags (ascending,
// deterministic), shared by the encoder (row partitions) and the distributed plan (halo
// rows).  Kernels have internal linkage: each including translation unit gets its copy.
#pragma once
#include <cstdint>

#include "gse_internal.cuh"

namespace gse {

// ---- stream compaction of row flags (hand-written; ascending, deterministic): 3 kernels,
// 4096 flags per CTA -- counts, one-CTA exclusive scan of the counts, ordered scatter.
constexpr int CMP_THREADS = 256, CMP_ITEMS = 16, CMP_TILE = CMP_THREADS * CMP_ITEMS;

// exclusive scan of one value per thread over the CTA (blockDim.x <= 1024); *total gets the sum
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t wsum[32], wtot;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  uint32_t inc = v;
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
    if (lane >= d) inc += o;
  }
  __syncthreads();  // wsum reuse across calls
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < nw ? wsum[lane] : 0u, wi = w;
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, wi, d);
      if (lane >= d) wi += o;
    }
    if (lane < nw) wsum[lane] = wi - w;
    if (lane == 31) wtot = wi;  // lanes >= nw add 0: lane 31 holds the CTA total
  }
  __syncthreads();
  *total = wtot;
  return wsum[warp] + inc - v;
}

static __global__ void __launch_bounds__(CMP_THREADS) k_cmp_count(const uint8_t* __restrict__ f,
                                                            int64_t n, uint32_t* __restrict__ cnt) {
  const int64_t base = (int64_t)blockIdx.x * CMP_TILE + (int64_t)threadIdx.x * CMP_ITEMS;
  uint32_t c = 0;
  for (int i = 0; i < CMP_ITEMS; ++i) c += (base + i < n && f[base + i]) ? 1u : 0u;
  uint32_t tot;
  block_excl_scan(c, &tot);
  if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

static __global__ void __launch_bounds__(1024) k_cmp_scan(uint32_t* __restrict__ cnt, int64_t nb,
                                                   int* __restrict__ total) {
  uint32_t run = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += 1024) {
    const int64_t i = b0 + threadIdx.x;
    const uint32_t v = i < nb ? cnt[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(v, &tot);
    if (i < nb) cnt[i] = run + ex;
    run += tot;
  }
  if (threadIdx.x == 0) *total = (int)run;
}

static __global__ void __launch_bounds__(CMP_THREADS) k_cmp_scatter(const uint8_t* __restrict__ f,
                                                              int64_t n,
                                                              const uint32_t* __restrict__ off,
                                                              uint32_t* __restrict__ out) {
  const int64_t base = (int64_t)blockIdx.x * CMP_TILE + (int64_t)threadIdx.x * CMP_ITEMS;
  uint32_t c = 0;
  for (int i = 0; i < CMP_ITEMS; ++i) c += (base + i < n && f[base + i]) ? 1u : 0u;
  uint32_t tot;
  uint32_t o = off[blockIdx.x] + block_excl_scan(c, &tot);
  for (int i = 0; i < CMP_ITEMS; ++i)
    if (base + i < n && f[base + i]) out[o++] = (uint32_t)(base + i);
}

// indices of the set flags, ascending, into out[]; the count lands in *d_count (device)
static inline gse_status compact_flags(const uint8_t* flags, int64_t n, uint32_t* out, int* d_count,
                                cudaStream_t s) {
  const int64_t nb = (n + CMP_TILE - 1) / CMP_TILE;
  if (nb == 0) return cuda_status(cudaMemsetAsync(d_count, 0, sizeof(int), s), "memset");
  uint32_t* cnt = dev_alloc_n<uint32_t>((size_t)nb, s);
  if (!cnt) return GSE_ERR_OOM;
  k_cmp_count<<<(unsigned)nb, CMP_THREADS, 0, s>>>(flags, n, cnt);
  k_cmp_scan<<<1, 1024, 0, s>>>(cnt, nb, d_count);
  k_cmp_scatter<<<(unsigned)nb, CMP_THREADS, 0, s>>>(flags, n, cnt, out);
  GSE_CUDA_TRY(cudaGetLastError());
  dev_free(cnt, s);
  return GSE_OK;
}


}  // namespace gse
