// Microbenchmark (developer tool, not product): which part of the window kernel's plane ring
// (spmv_win.cu RING experiment) costs streaming bandwidth.  Stages of the
// level-1 shape: 8 KB + 4 KB + 256 B + 48 B copies; 2 CTAs/SM, producer warp + 8 consumers.
//  mode 0: stages interleaved across CTAs (stage s -> CTA s % grid)
//  mode 1: tiles of 8 stages, tile t owned by CTA t % grid (each CTA streams its own region)
//  mode 2: mode 1 + a 16 KB x window per tile (double-buffered, consumers wait at tile start)
//  mode 3: mode 2 + per-stage records folded by producer lane 0 (record barrier per stage)
//  mode 4: mode 1 with one copy per stage (12 KB) instead of four
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mexp(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void marr(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  uint32_t d = 0;
  while (!d) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n" : "=r"(d) : "r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b, int keep) {
  uint64_t pol;
  if (keep) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(su(dst)), "l"(src), "r"(n), "r"(su(b)), "l"(pol) : "memory");
}
constexpr uint32_t STB = 12672, D = 4, TS = 8, WIN = 16448;
__global__ void __launch_bounds__(288, 2) k(const unsigned char* col, const unsigned char* head,
    const unsigned char* rb, const unsigned char* cp, const unsigned char* x, size_t nst, int mode,
    unsigned* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* win = sm;                 // 2 windows
  unsigned char* ring = sm + 2 * WIN;
  __shared__ __align__(8) uint64_t full[D], empty[D], wfull[2], rec[2 * D];
  __shared__ uint32_t recv[2 * D][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < D; ++i) { minit(&full[i], 1); minit(&empty[i], 8); }
    for (uint32_t i = 0; i < 2 * D; ++i) minit(&rec[i], 8);
    minit(&wfull[0], 1); minit(&wfull[1], 1);
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncthreads();
  const size_t ntiles = nst / TS;
  // stage sequence of this CTA
  auto stage_of = [&](size_t q, size_t& s, bool& tile_start, size_t& tile) {
    if (mode == 0) { s = blockIdx.x + q * gridDim.x; tile_start = false; tile = 0; return s < nst; }
    tile = blockIdx.x + (q / TS) * gridDim.x; s = tile * TS + q % TS; tile_start = (q % TS) == 0;
    return tile < ntiles;
  };
  if (warp == 8) {
    uint32_t sf = 0, acc = 0;
    size_t q = 0, s, tile; bool ts; uint32_t it = 0;
    for (; stage_of(q, s, ts, tile); ++q) {
      if (ts && mode >= 2 && lane == 0) {
        mexp(&wfull[it & 1], WIN);
        bulk(win + (it & 1) * WIN, x + (tile * 7919 % 4096) * WIN, WIN, &wfull[it & 1], 1);
      }
      if (ts) ++it;
      const uint32_t slot = q % D;
      if (q >= D) mwait(&empty[slot], ((q / D) - 1) & 1);
      if (mode == 3) {
        while (sf + 2 * D <= q) {
          mwait(&rec[sf % (2 * D)], (sf / (2 * D)) & 1);
          if (lane == 0) for (int w = 0; w < 8; ++w) acc += recv[sf % (2 * D)][w];
          __syncwarp(); ++sf;
        }
      }
      unsigned char* sb = ring + slot * STB;
      if (lane == 0) mexp(&full[slot], mode == 4 ? 12288u : 8192u + 4096u + 256u + 48u);
      __syncwarp();
      if (mode == 4) { if (lane == 0) bulk(sb, col + s * 12288, 12288, &full[slot], 0); }
      else {
        if (lane == 0) bulk(sb, col + s * 8192, 8192, &full[slot], 0);
        if (lane == 1) bulk(sb + 8192, head + s * 4096, 4096, &full[slot], 0);
        if (lane == 2) bulk(sb + 12288, rb + s * 256, 256, &full[slot], 0);
        if (lane == 3) bulk(sb + 12544, cp + (s & ~3ull) * 4, 48, &full[slot], 0);
      }
    }
    if (mode == 3) while (sf < q) { mwait(&rec[sf % (2 * D)], (sf / (2 * D)) & 1); ++sf; }
    if (acc == 0x12345678) *sink = acc;
    return;
  }
  uint32_t acc = 0, it = 0;
  size_t q = 0, s, tile; bool ts;
  for (; stage_of(q, s, ts, tile); ++q) {
    if (ts && mode >= 2) { mwait(&wfull[it & 1], (it >> 1) & 1); acc += *(const uint32_t*)(win + (it & 1) * WIN + lane * 4); }
    if (ts) ++it;
    const uint32_t slot = q % D;
    mwait(&full[slot], (q / D) & 1);
    acc += *(const uint32_t*)(ring + slot * STB + warp * 1024 + lane * 32);
    __syncwarp();
    if (lane == 0) marr(&empty[slot]);
    if (mode == 3 && lane == 0) { recv[q % (2 * D)][warp] = acc; marr(&rec[q % (2 * D)]); }
  }
  if (acc == 0x12345678) *sink = acc;
}
int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const size_t nst = 98304;  // 200M nnz / 2048
  unsigned char *col, *head, *rb, *cp, *x; unsigned* sink;
  cudaMalloc(&col, nst * 12288 + 4096); cudaMalloc(&head, nst * 4096); cudaMalloc(&rb, nst * 256);
  cudaMalloc(&cp, nst * 4 + 64); cudaMalloc(&x, (size_t)4096 * WIN); cudaMalloc(&sink, 4);
  cudaMemset(col, 1, nst * 12288 + 4096); cudaMemset(head, 1, nst * 4096); cudaMemset(rb, 1, nst * 256);
  cudaMemset(cp, 1, nst * 4 + 64); cudaMemset(x, 1, (size_t)4096 * WIN);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 2 * WIN + D * STB;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode <= 4; ++mode) {
    k<<<2 * sms, 288, smem>>>(col, head, rb, cp, x, nst, mode, sink);
    cudaEventRecord(a);
    k<<<2 * sms, 288, smem>>>(col, head, rb, cp, x, nst, mode, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)nst * (mode == 4 ? 12288 : 12592) + (mode >= 2 ? (double)nst / TS * WIN : 0);
    printf("mode %d: %.1f us  %.0f GB/s  %s\n", mode, ms * 1e3, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
