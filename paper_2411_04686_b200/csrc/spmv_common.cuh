// spmv_common.cuh -- shared pieces of the two SpMV kernels (spmv_sp.cu: strided products
// for irregular rows; spmv_rw.cu: row walk over staged planes for regular rows).
#pragma once
#include <cuda_fp16.h>

#include <cstdint>

#include "decode.cuh"
#include "gse_internal.cuh"

namespace gse {

// Matrix planes are streamed once per SpMV: every plane load carries an L2 evict-first
// policy so the 126 MB L2 keeps the solver vectors (x, r, p, q) resident instead
// (DESIGN.md "L2 residency").
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// x (the SpMV operand) is re-read by every tile window and by the far gathers: its lines
// carry evict-last so the streamed planes do not push it out of L2
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint32_t ld_nc_u32(const uint32_t* p) {
  uint32_t r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
      : "=r"(r)
      : "l"(p), "l"(l2_evict_first()));
  return r;
}
__device__ __forceinline__ uint32_t ld_nc_u16(const uint16_t* p) {
  unsigned short r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;"
      : "=h"(r)
      : "l"(p), "l"(l2_evict_first()));
  return r;
}
__device__ __forceinline__ uint32_t ld_nc_u8(const uint8_t* p) {
  unsigned short r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;"
      : "=h"(r)
      : "l"(p), "l"(l2_evict_first()));
  return r;
}
__device__ __forceinline__ double ld_nc_f64(const double* p) {
  double r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
      : "=d"(r)
      : "l"(p), "l"(l2_evict_first()));
  return r;
}
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "l"(l2_evict_first()));
  return r;
}
__device__ __forceinline__ uint2 ld_nc_v2(const void* p) {
  uint2 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
      : "=r"(r.x), "=r"(r.y)
      : "l"(p), "l"(l2_evict_first()));
  return r;
}

// ---- mbarrier + TMA bulk-copy helpers (row-walk stages, window-kernel x windows)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(l2_evict_first())
      : "memory");
}
// the same with an evict-last hint (x windows: re-read by neighbouring tiles and gathers)
__device__ __forceinline__ void bulk_g2s_keep(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(l2_evict_last())
      : "memory");
}

// Kernel "levels": 0 = FP64 CSR (a6), 1..3 = GSE segments (a5), and the 16-bit storage
// baselines of P:406 (FP16 / BF16 codes in the head plane, converted exactly to FP64).
constexpr int L_FP16 = 4, L_BF16 = 5;
template <int L>
__host__ __device__ constexpr bool has_head() { return L >= 1; }
template <int L>
__host__ __device__ constexpr bool has_t1() { return L == 2 || L == 3; }
template <int L>
__host__ __device__ constexpr bool has_t2() { return L == 3; }
template <int L>
__host__ __device__ constexpr bool is_half() { return L == L_FP16 || L == L_BF16; }

// exact FP64 value of a 16-bit code (binary16: via FP32, which holds every binary16 value;
// bfloat16: the top half of an FP32)
template <int L>
__device__ __forceinline__ double half_value(uint32_t h) {
  if constexpr (L == L_FP16)
    return (double)__half2float(__ushort_as_half((unsigned short)h));
  else
    return (double)__uint_as_float(h << 16);
}

template <class T>
struct SpmvParams {
  const BlockDesc* __restrict__ blocks;
  const uint32_t* __restrict__ row_ptr;
  const uint32_t* __restrict__ col_ei;
  const uint8_t* __restrict__ side;
  const uint16_t* __restrict__ head;
  const uint16_t* __restrict__ tail1;
  const uint32_t* __restrict__ tail2;
  const double* __restrict__ val;
  uint32_t n_blocks;  // SP warp blocks
  uint32_t rows;
  uint32_t n_groups;  // RW 32-row groups
  uint32_t rw_stage;  // RW: elements per staging buffer (>= max group span, multiple of 16)
  uint32_t rw_stage2;  // the same for 64-row groups
  int ei_shift;       // 32 - ei_bits
  uint32_t col_mask;  // (1 << (32 - ei_bits)) - 1, or ~0u
  const T* __restrict__ x;
  const T* __restrict__ xd;  // x of the launch's rows for the fused dot (x + first row)
  T* __restrict__ y;
  double* partials;
  unsigned* ticket;
  double* dot_result;
  const int* stop;    // optional: skip the launch when *stop != 0 (GMRES cycle graphs)
  // window mode (spmv_win.cu)
  const BlockDesc* __restrict__ tiles;
  const uint8_t* __restrict__ rowbits;
  const uint32_t* __restrict__ chunk_prev;
  uint32_t n_tiles;
  uint32_t nnz_pad;   // allocated (padded) plane length: bulk copies never read past it
  uint32_t cols;
  int win_on;         // x is 16-byte aligned: windows staged by TMA (else every gather is global)
  long long d64[64];  // decode deltas of the launched level (integer form, FP64)
  int d32[64];        // (integer form, FP32)
  double sc64[64];    // multiply-form scales when the table allows it (FAST)
  float sc32[64];
};

// Level-L value of one element.  FAST: |v| = D_L * scale -- exact and never underflowing
// for this table (build_decode_table), so it equals the bit-exact integer form of
// decode.cuh on every value except the sign of a zero significand (+0 vs -0), which cannot
// change a row sum that has a nonzero term.
template <int L, bool FAST>
__device__ __forceinline__ double dec64(uint32_t h, uint32_t t1, uint32_t t2,
                                        const long long* sd, const double* sc, uint32_t ei) {
  if constexpr (FAST) {
    const uint32_t neg = h & 0x8000u;
    double m;
    if constexpr (L == 1) {
      const int D = (int)(h & 0x7FFFu);
      m = (double)(neg ? -D : D);
    } else if constexpr (L == 2) {
      const int D = (int)(((h & 0x7FFFu) << 16) | t1);
      m = (double)(neg ? -D : D);
    } else {
      const uint64_t D = ((uint64_t)(h & 0x7FFFu) << 48) | ((uint64_t)t1 << 32) | t2;
      m = __ull2double_rz(D);
      m = neg ? -m : m;
    }
    return m * sc[ei];
  } else {
    if constexpr (L == 1)
      return decode_l1(h, sd[ei]);
    else if constexpr (L == 2)
      return decode_l2(h, t1, sd[ei]);
    else
      return decode_l3(h, t1, t2, sd[ei]);
  }
}

template <int L, bool FAST>
__device__ __forceinline__ float dec32(uint32_t h, uint32_t t1, uint32_t t2, const int* sd,
                                       const float* sc, uint32_t ei) {
  if constexpr (FAST) {
    float m;
    if constexpr (L == 1)
      m = (float)(int)(h & 0x7FFFu);
    else if constexpr (L == 2)
      m = __uint2float_rz(((h & 0x7FFFu) << 16) | t1);
    else
      m = __ull2float_rz(((uint64_t)(h & 0x7FFFu) << 48) | ((uint64_t)t1 << 32) | t2);
    m = (h & 0x8000u) ? -m : m;
    return m * sc[ei];
  } else {
    if constexpr (L == 1)
      return decode_f32_u32(h & 0x7FFFu, sd[ei], h);
    else if constexpr (L == 2)
      return decode_f32_u32(((h & 0x7FFFu) << 16) | t1, sd[ei], h);
    else
      return decode_f32(((uint64_t)(h & 0x7FFFu) << 48) | ((uint64_t)t1 << 32) | t2, sd[ei], h);
  }
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
  return v;  // lane 0 holds the sum (fixed tree)
}

// CTA-wide sum of one value per warp (lane 0's), fixed order; then the last CTA to arrive
// sums all CTA partials in index order -> deterministic scalar.
__device__ __forceinline__ void finalize_dot(double wsum, double* partials, unsigned* ticket,
                                             double* result) {
  __shared__ double red[SPMV_WARPS];
  __shared__ unsigned s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = wsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < SPMV_WARPS; ++i) s += red[i];
    partials[blockIdx.x] = s;
    __threadfence();
    s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double acc = 0.0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) acc += __ldcg(partials + i);
  acc = warp_sum(acc);
  __syncthreads();
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < SPMV_WARPS; ++i) s += red[i];
    *result = s;
    *ticket = 0u;
  }
}

// stage the per-EI decode constants into shared memory (once per CTA)
template <int L, class T>
__device__ __forceinline__ void stage_tables(const SpmvParams<T>& p, long long* sd64, int* sd32,
                                             double* sc64, float* sc32) {
  if constexpr (L >= 1) {
    const int t = threadIdx.x;
    if (t < 64) {
      if constexpr (sizeof(T) == 8) {
        sd64[t] = p.d64[t];
        sc64[t] = p.sc64[t];
      } else {
        sd32[t] = p.d32[t];
        sc32[t] = p.sc32[t];
      }
    }
    __syncthreads();
  }
}

// launchers (spmv_sp.cu / spmv_rw.cu)
template <class T>
void launch_sp(const Matrix& M, int level, bool dot, bool fast, const SpmvParams<T>& p,
               cudaStream_t s);
template <class T>
void launch_rw(const Matrix& M, int level, bool dot, bool fast, const SpmvParams<T>& p,
               cudaStream_t s);
template <class T>
void launch_win(const Matrix& M, int level, bool dot, bool fast, const SpmvParams<T>& p,
                cudaStream_t s);

// persistent grid size for a kernel: resident CTAs per SM x SMs, capped by the work units
template <class K>
inline int persistent_grid(K kernel, int device, int64_t units_per_cta_work, int* cache) {
  const int dev = device < 64 ? device : 0;
  if (!cache[dev]) {
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, SPMV_THREADS, 0);
    cache[dev] = (blocks < 1 ? 1 : blocks) * num_sms(device);
  }
  const int64_t want = (units_per_cta_work + SPMV_WARPS - 1) / SPMV_WARPS;
  int g = (int)(want < cache[dev] ? want : cache[dev]);
  return g < 1 ? 1 : g;
}

}  // namespace gse
