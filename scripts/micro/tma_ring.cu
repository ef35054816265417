// Microbenchmark (developer tool, not product): TMA bulk-copy ring throughput.
// grid = 2 CTAs/SM; warp 8 = producer (lane-parallel copies of PIECE bytes per stage of
// STAGE bytes), warps 0..7 = consumers that wait for each stage, read one 16B word per lane
// and release.  Prints GB/s for each (stage, piece, depth).
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
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b, int hint) {
  uint64_t pol;
  if (hint) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(su(dst)), "l"(src), "r"(n), "r"(su(b)), "l"(pol) : "memory");
}
__global__ void __launch_bounds__(288, 2) k(const unsigned char* src, size_t total, uint32_t stage,
                                             uint32_t piece, uint32_t D, int hint, unsigned* sink) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[8], empty[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (uint32_t i = 0; i < D; ++i) { minit(&full[i], 1); minit(&empty[i], 8); } asm volatile("fence.proxy.async.shared::cta;"); }
  __syncthreads();
  const size_t nst = total / stage;
  if (warp == 8) {
    uint32_t si = 0;
    for (size_t s = blockIdx.x; s < nst; s += gridDim.x, ++si) {
      const uint32_t slot = si % D;
      if (si >= D) mwait(&empty[slot], ((si / D) - 1) & 1);
      if (lane == 0) mexp(&full[slot], stage);
      __syncwarp();
      const uint32_t np = stage / piece;
      for (uint32_t i = lane; i < np; i += 32)
        bulk(ring + (size_t)slot * stage + i * piece, src + s * stage + i * piece, piece, &full[slot], hint);
    }
    return;
  }
  uint32_t si = 0, acc = 0;
  for (size_t s = blockIdx.x; s < nst; s += gridDim.x, ++si) {
    const uint32_t slot = si % D;
    mwait(&full[slot], (si / D) & 1);
    acc += *(const uint32_t*)(ring + (size_t)slot * stage + ((threadIdx.x * 16) % stage));
    __syncwarp();
    if (lane == 0) marr(&empty[slot]);
  }
  if (acc == 0x12345678) *sink = acc;
}
int main() {
  setvbuf(stdout, NULL, _IONBF, 0); size_t total = (size_t)1 << 30;
  unsigned char* src; cudaMalloc(&src, total); cudaMemset(src, 1, total);
  unsigned* sink; cudaMalloc(&sink, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  uint32_t stages[] = {4096, 8192, 12288, 16384, 24576, 32768};
  uint32_t pieces[] = {512, 1024, 2048, 4096, 8192, 16384};
  for (int hint = 1; hint < 2; ++hint)
  for (uint32_t st : stages) for (uint32_t pc : pieces) for (uint32_t D : {2u, 3u, 4u, 6u}) {
    if (pc > st || st / pc > 64) continue;
    size_t sm = (size_t)st * D; if (sm > 100 * 1024) continue;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<2 * sms, 288, sm>>>(src, total, st, pc, D, hint, sink);
    cudaEventRecord(a);
    k<<<2 * sms, 288, sm>>>(src, total, st, pc, D, hint, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("hint=%d stage=%u piece=%u D=%u  %.0f GB/s %s\n", hint, st, pc, D, (double)(total / st * st) / ms / 1e6, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
