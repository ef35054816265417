// spmv_rw.cu -- "row walk" SpMV kernel for regular row lengths (stencils: configs 1, 2, 4,
// 5).  SURVEY 8(a) a4-a6; paper Alg. spmv -- a row per thread group -- and
// P:212 for levels 2-3.
//
//  * persistent CTAs of 8 independent warps; a warp owns groups of 32 consecutive rows
//    (lane = row) with a fixed grid stride;
//  * the planes of the NEXT group (only the requested ones) are fetched into a
//    warp-private shared-memory stage by TMA bulk copies (cp.async.bulk, one elected lane,
//    completion on a per-stage mbarrier) while the warp computes the current group: DRAM
//    latency leaves the dependent chain and no registers hold data in flight;
//  * lane = row: a lane walks its row in storage order (the oracle's summation order) with
//    8 x-gathers in flight, branch-free (slots past the row end contribute exact zeros).
//    For stencil rows the j-th element of 32 consecutive rows lies on one diagonal, so a
//    warp-wide gather touches ~2 cache lines;
//  * decode in multiply form with the sign folded into a shared scale table
//    (|v| = D_L * scale[EI], exact for the tables that allow it, see build_decode_table);
//  * chosen at encode when every group's span fits RW_TILE and the row lengths of a group
//    are close (Matrix::rw_efficiency >= 0.6); otherwise spmv_sp.cu runs.
#include "spmv_common.cuh"

#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

namespace gse {

// bytes per staged element at level L (col_ei + requested planes; L = 0: FP64 values)
template <int L>
__host__ __device__ constexpr uint32_t rw_elem_bytes() {
  return 4u + (L == 0 ? 8u : 0u) + (has_head<L>() ? 2u : 0u) + (has_t1<L>() ? 2u : 0u) +
         (has_t2<L>() ? 4u : 0u);
}

// views of one staging buffer (rebuilt from the dynamic shared array each time, so the
// compiler keeps them in the shared window and emits LDS; pointer structs indexed at run
// time decay to generic 64-bit loads)
template <int L>
struct Stage {
  uint32_t* col;
  double* val;
  uint16_t* head;
  uint16_t* tail1;
  uint32_t* tail2;
  __device__ Stage(unsigned char* base, uint32_t N) {
    unsigned char* q = base;
    col = reinterpret_cast<uint32_t*>(q);
    q += 4 * N;
    val = reinterpret_cast<double*>(q);
    if (L == 0) q += 8 * N;
    head = reinterpret_cast<uint16_t*>(q);
    if (has_head<L>()) q += 2 * N;
    tail1 = reinterpret_cast<uint16_t*>(q);
    if (has_t1<L>()) q += 2 * N;
    tail2 = reinterpret_cast<uint32_t*>(q);
  }
};

template <int L, class T>
__device__ __forceinline__ void issue_stage(const SpmvParams<T>& p, const Stage<L>& st,
                                            uint64_t* bar, uint32_t s, uint32_t e) {
  const uint32_t base = s & ~7u;
  // 8-element units, plus 8 more: row walks read 8 slots unconditionally, and the over-copied
  // elements are real stored entries (or the zero padding after nnz), so every gathered
  // column stays in bounds; their products are masked to exact zeros
  const uint32_t n = (e > base) ? ((e - base + 7u) & ~7u) + 8u : 0u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads -> async writes
  mbar_arrive_expect_tx(bar, n * rw_elem_bytes<L>());
  if (n == 0) return;
  bulk_g2s(st.col, p.col_ei + base, 4 * n, bar);
  if constexpr (L == 0) bulk_g2s(st.val, p.val + base, 8 * n, bar);
  if constexpr (has_head<L>()) bulk_g2s(st.head, p.head + base, 2 * n, bar);
  if constexpr (has_t1<L>()) bulk_g2s(st.tail1, p.tail1 + base, 2 * n, bar);
  if constexpr (has_t2<L>()) bulk_g2s(st.tail2, p.tail2 + base, 4 * n, bar);
}

// index of the zero entry of the sign-folded scale tables: masked slots decode to exact 0
constexpr uint32_t SSC_ZERO = 128;

#ifndef GSE_RW_PAIR
#define GSE_RW_PAIR 1
#endif

template <class T>
struct Chunk8 {
  uint32_t c[8], h[8], t1[8], t2[8];
  double v0[8];
  T xv[8];
};

// the 8 staged slots from j on and their gathered operands (all gathers issued here)
template <int L, class T>
__device__ __forceinline__ void load_chunk(const SpmvParams<T>& p, const Stage<L>& st,
                                           uint32_t j, Chunk8<T>& K) {
  uint32_t* c = K.c;
  uint32_t* h = K.h;
  uint32_t* t1 = K.t1;
  uint32_t* t2 = K.t2;
  double* v0 = K.v0;
  T* xv = K.xv;
  // 8 slots read unconditionally at immediate offsets: the stage holds >= 8 over-copied
  // stored entries past every row (issue_stage), so the columns are valid; slots past
  // the row end are masked to exact zeros below
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    c[q] = st.col[j + q];
    if constexpr (L == 0) v0[q] = st.val[j + q];
    if constexpr (has_head<L>()) h[q] = st.head[j + q];
    if constexpr (has_t1<L>()) t1[q] = st.tail1[j + q];
    if constexpr (has_t2<L>()) t2[q] = st.tail2[j + q];
  }
  // all 8 gathers issued before any product (ld.global.nc, volatile asm keeps the order)
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const T* a = p.x + (c[q] & p.col_mask);
    if constexpr (sizeof(T) == 8) {
      double v;
      asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(a));
      xv[q] = v;
    } else {
      float v;
      asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(a));
      xv[q] = v;
    }
  }
}

// sum += the chunk's products in slot order (slots q >= nrem lie past the row end)
template <int L, bool FAST, class T>
__device__ __forceinline__ T sum_chunk(const SpmvParams<T>& p, const Chunk8<T>& K,
                                       uint32_t nrem, T sum, const double* ssc64,
                                       const float* ssc32, const long long* sd64,
                                       const int* sd32, const double* sc64, const float* sc32) {
  const uint32_t* c = K.c;
  const uint32_t* h = K.h;
  const uint32_t* t1 = K.t1;
  const uint32_t* t2 = K.t2;
  const double* v0 = K.v0;
  const T* xv = K.xv;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const bool ok = (uint32_t)q < nrem;
    // slots past the row end take x = 0 (their decoded values are finite stored entries or
    // the zero padding), so a NaN / Inf in x reaches only the rows that reference it
    const T xq = ok ? xv[q] : (T)0;
    T prod;
    if constexpr (L == 0) {
      prod = (T)__dmul_rn(ok ? v0[q] : 0.0, (double)xq);  // (FP64 kind: values unchecked)
    } else if constexpr (is_half<L>()) {  // P:406 baselines: exact code value x x in FP64
      prod = (T)__dmul_rn(ok ? half_value<L>(h[q]) : 0.0, (double)xq);  // (codes may be +-Inf)
    } else if constexpr (FAST) {
      // scale index = EI | sign << ei_bits in one funnel shift (col's top bits are EI)
      const uint32_t idx = __funnelshift_rc(c[q], h[q] >> 15, p.ei_shift);
      if constexpr (L == 1) {
        const uint32_t D = h[q] & 0x7FFFu;
        if constexpr (sizeof(T) == 8)
          prod = __dmul_rn(__dmul_rn((double)D, ssc64[idx]), xq);
        else
          prod = __fmul_rn(__fmul_rn((float)D, ssc32[idx]), xq);
      } else if constexpr (L == 2) {
        const uint32_t D = ((h[q] & 0x7FFFu) << 16) | t1[q];
        if constexpr (sizeof(T) == 8)
          prod = __dmul_rn(__dmul_rn((double)D, ssc64[idx]), xq);
        else
          prod = __fmul_rn(__fmul_rn(__uint2float_rz(D), ssc32[idx]), xq);
      } else {
        const uint64_t D = ((uint64_t)(h[q] & 0x7FFFu) << 48) | ((uint64_t)t1[q] << 32) | t2[q];
        if constexpr (sizeof(T) == 8)
          prod = __dmul_rn(__dmul_rn(__ull2double_rz(D), ssc64[idx]), xq);
        else
          prod = __fmul_rn(__fmul_rn(__ull2float_rz(D), ssc32[idx]), xq);
      }
    } else {
      const uint32_t ei = __funnelshift_rc(c[q], 0u, p.ei_shift);
      const uint32_t tt1 = L >= 2 ? t1[q] : 0u, tt2 = L == 3 ? t2[q] : 0u;
      if constexpr (sizeof(T) == 8) {
        const double a = dec64<L, false>(h[q], tt1, tt2, sd64, sc64, ei);
        prod = __dmul_rn(a, xq);
      } else {
        const float a = dec32<L, false>(h[q], tt1, tt2, sd32, sc32, ei);
        prod = __fmul_rn(a, xq);
      }
    }
    sum += prod;
  }
  return sum;
}

// sum of one row, elements [j0, j1) of the stage, in storage order
template <int L, bool FAST, class T>
__device__ __forceinline__ T walk_row(const SpmvParams<T>& p, const Stage<L>& st, uint32_t j0,
                                      uint32_t j1, const double* ssc64, const float* ssc32,
                                      const long long* sd64, const int* sd32,
                                      const double* sc64, const float* sc32) {
  T sum = 0;
  for (uint32_t j = j0; j < j1; j += 8) {
    Chunk8<T> K;
    load_chunk<L, T>(p, st, j, K);
    sum = sum_chunk<L, FAST, T>(p, K, j1 - j, sum, ssc64, ssc32, sd64, sd32, sc64, sc32);
  }
  return sum;
}

// RPL = rows per lane: a group is 32 * RPL consecutive rows staged by one set of bulk
// copies and walked in RPL passes of lane = row (RPL = 2 halves the per-group overhead:
// row bounds, copy issue, barrier wait)
// register budget: 3 resident CTAs per SM (measured: capping at 64 registers for 4 CTAs
// gains 6 % on the plain level-1 SpMV at 256^3 but loses 6 % on the 128^3 CG's fused-dot
// variant and 1-7 % at levels 2/3); GSE_RW_MINB overrides (A/B builds)
#ifdef GSE_RW_MINB
#define RW_MINB(L) GSE_RW_MINB
#else
#define RW_MINB(L) 3
#endif
template <int L, int RPL, bool DOT, bool FAST, class T>
__global__ void __launch_bounds__(SPMV_THREADS, RW_MINB(L)) k_spmv_rw(const SpmvParams<T> p) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t bars[SPMV_WARPS][2];
  __shared__ long long sd64[64];
  __shared__ int sd32[64];
  __shared__ double sc64[64];
  __shared__ float sc32[64];
  // sign-folded scales: [EI | sign << ei_bits] = (sign ? -1 : 1) scale; [SSC_ZERO] = 0
  __shared__ double ssc64[SSC_ZERO + 1];
  __shared__ float ssc32[SSC_ZERO + 1];
  if (threadIdx.x <= SSC_ZERO) {
    const uint32_t t = threadIdx.x, eb = 32u - (uint32_t)p.ei_shift;
    const uint32_t sign = t >> eb, ei = t & ((1u << eb) - 1u);
    const bool live = t < SSC_ZERO && sign <= 1u;
    if constexpr (sizeof(T) == 8)
      ssc64[t] = live ? (sign ? -p.sc64[ei] : p.sc64[ei]) : 0.0;
    else
      ssc32[t] = live ? (sign ? -p.sc32[ei] : p.sc32[ei]) : 0.0f;
  }
  stage_tables<L>(p, sd64, sd32, sc64, sc32);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t N = RPL == 1 ? p.rw_stage : p.rw_stage2;
  const uint32_t SB = N * rw_elem_bytes<L>();
  unsigned char* wbase = dsm + (size_t)warp * 2 * SB;
  if (lane == 0) {
    mbar_init(&bars[warp][0], 1);
    mbar_init(&bars[warp][1], 1);
    // make the initialised barriers visible to the async (TMA) proxy; a cluster-scope
    // fence.mbarrier_init would also invalidate L1 (CCTL.IVALL)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();

  constexpr uint32_t GR = RW_ROWS * RPL;  // rows per group
  double dacc = 0.0;
  const uint32_t rows = p.rows, ng = (rows + GR - 1) / GR;
  const uint32_t W = gridDim.x * SPMV_WARPS;
  uint32_t g = blockIdx.x * SPMV_WARPS + warp;
  // row bounds of a group: a[k] = rp[r0 + 32 k + lane], c = rp[r0 + GR] (indices clamped to
  // rows: rows past the end are empty); a row's end is the next row's start
  struct Bounds {
    uint32_t a[RPL];
    uint32_t c;
  };
  auto bounds = [&](uint32_t grp) {
    Bounds B;
#pragma unroll
    for (int k = 0; k < RPL; ++k) B.a[k] = 0;
    B.c = 0;
    if (grp < ng) {
      const uint32_t r0 = grp * GR;
#pragma unroll
      for (int k = 0; k < RPL; ++k) B.a[k] = p.row_ptr[min(r0 + 32 * k + lane, rows)];
      B.c = p.row_ptr[min(r0 + GR, rows)];
    }
    return B;
  };
  // prologue on constant data (tables, row pointers, the first tile of planes) overlaps
  // the previous kernel's drain under programmatic dependent launch
  Bounds cur_b = bounds(g), nxt_b = bounds(g + W);
  if (g < ng && lane == 0)
    issue_stage<L>(p, Stage<L>(wbase, N), &bars[warp][0], cur_b.a[0], cur_b.c);
  pdl_wait();
  if (p.stop && *p.stop) {  // drain the issued copy before the CTA exits
    if (g < ng) mbar_wait(&bars[warp][0], 0);
    return;
  }
  pdl_trigger();
  uint32_t it = 0;
  for (; g < ng; g += W, ++it) {
    const uint32_t cur = it & 1u;
    const Bounds n2_b = bounds(g + 2 * W);  // two groups ahead
    if (g + W < ng) {                       // planes of the next group -> the other stage
      const uint32_t s = __shfl_sync(0xFFFFFFFFu, nxt_b.a[0], 0);
      if (lane == 0)
        issue_stage<L>(p, Stage<L>(wbase + (cur ^ 1u) * SB, N), &bars[warp][cur ^ 1u], s,
                       nxt_b.c);
    }
    const uint32_t r0 = g * GR;
    const uint32_t base = __shfl_sync(0xFFFFFFFFu, cur_b.a[0], 0) & ~7u;
    uint32_t ea[RPL];
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      ea[k] = __shfl_down_sync(0xFFFFFFFFu, cur_b.a[k], 1);
      const uint32_t last = (k + 1 < RPL) ? __shfl_sync(0xFFFFFFFFu, cur_b.a[k + 1 < RPL ? k + 1 : k], 0)
                                          : cur_b.c;
      if (lane == 31) ea[k] = last;
    }
    mbar_wait(&bars[warp][cur], (it >> 1) & 1u);
    const Stage<L> st(wbase + cur * SB, N);
    T sums[RPL];
    bool paired = false;
#if GSE_RW_PAIR
    if constexpr (RPL == 2 && sizeof(T) == 4) {
      // both rows of the lane fit one 8-slot chunk (stencils): issue the 16 gathers of the
      // two rows before any product.  FP32 accumulation only: C2 level-1 cold 4221 -> 4566
      // GB/s; with FP64 accumulation it lost (steady 5253 -> 4855 GB/s, CG 46.0 -> 49.9 us
      // per iteration; profiles/ab_rw_pair_r01.txt)
      const uint32_t n0 = ea[0] - cur_b.a[0], n1 = ea[1] - cur_b.a[1];
      if (__all_sync(0xFFFFFFFFu, n0 <= 8u && n1 <= 8u)) {
        Chunk8<T> K0, K1;
        load_chunk<L, T>(p, st, cur_b.a[0] - base, K0);
        load_chunk<L, T>(p, st, cur_b.a[1] - base, K1);
        sums[0] = n0 ? sum_chunk<L, FAST, T>(p, K0, n0, T(0), ssc64, ssc32, sd64, sd32, sc64,
                                             sc32)
                     : T(0);
        sums[1] = n1 ? sum_chunk<L, FAST, T>(p, K1, n1, T(0), ssc64, ssc32, sd64, sd32, sc64,
                                             sc32)
                     : T(0);
        paired = true;
      }
    }
#endif
    if (!paired) {
#pragma unroll
      for (int k = 0; k < RPL; ++k)
        sums[k] = walk_row<L, FAST, T>(p, st, cur_b.a[k] - base, ea[k] - base, ssc64, ssc32,
                                       sd64, sd32, sc64, sc32);
    }
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const T sa = sums[k];
      const uint32_t row = r0 + 32 * k + lane;
      if (row < rows) {
        p.y[row] = sa;
        if constexpr (DOT) dacc += (double)p.xd[row] * (double)sa;
      }
    }
    __syncwarp();
    cur_b = nxt_b;
    nxt_b = n2_b;
  }
  if constexpr (DOT) finalize_dot(warp_sum(dacc), p.partials, p.ticket, p.dot_result);
}

// Launch configuration of one kernel instantiation.  The dynamic shared-memory attribute
// is per function and process-wide, while matrices (and host threads -- one per rank in the
// thread backend) launch it with different stage sizes: the attribute only ever grows
// (under a lock), and the occupancy is cached per stage size.
struct RwLaunchCache {
  std::mutex mu;
  int max_smem[64] = {0};
  std::map<std::pair<int, size_t>, int> grid;  // (device, smem) -> resident CTAs x SMs
};

template <int L, int RPL, bool DOT, bool FAST, class T>
static void go_rpl(const Matrix& M, const SpmvParams<T>& p, cudaStream_t s) {
  static RwLaunchCache lc;
  const int dev = M.device < 64 ? M.device : 0;
  const uint32_t N = RPL == 1 ? p.rw_stage : p.rw_stage2;
  const size_t smem = (size_t)SPMV_WARPS * 2 * N * rw_elem_bytes<L>();
  auto kern = k_spmv_rw<L, RPL, DOT, FAST, T>;
  int cap = 0;
  {
    std::lock_guard<std::mutex> lk(lc.mu);
    if ((int)smem > lc.max_smem[dev]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      lc.max_smem[dev] = (int)smem;
    }
    auto it = lc.grid.find({dev, smem});
    if (it == lc.grid.end()) {
      int blocks = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, SPMV_THREADS, smem);
      cap = (blocks < 1 ? 1 : blocks) * num_sms(M.device);
      lc.grid[{dev, smem}] = cap;
    } else {
      cap = it->second;
    }
  }
  const int64_t ng = (M.rows + RW_ROWS * RPL - 1) / (RW_ROWS * RPL);
  const int64_t want = (ng + SPMV_WARPS - 1) / SPMV_WARPS;
  int g = (int)(want < cap ? want : cap);
  if (g < 1) g = 1;
  launch_k(kern, g, SPMV_THREADS, smem, s, p);
}

// rows per lane (measured): 2 for level 1 (its per-group overhead
// is the largest share of the walk) and, for the other levels, when every warp gets >= 32
// groups (fewer: the +-1 group tail imbalance of the static schedule costs more than the
// overhead saved); 1 when the doubled stages do not fit 3 CTAs per SM
template <int L>
static int rw_rpl(const Matrix& M, uint32_t rw_stage2) {
  const char* e = getenv("GSE_RW_RPL");  // A/B and test override: 1 or 2 (read per launch)
  const int forced = e ? atoi(e) : 0;
  if (forced == 1 || forced == 2) return forced;
  const size_t two = (size_t)SPMV_WARPS * 2 * rw_stage2 * rw_elem_bytes<L>();
  if (two * 3 > 200 * 1024) return 1;
  if (L == 1) return 2;
  const int64_t warps = (int64_t)num_sms(M.device) * 3 * SPMV_WARPS;
  return (M.rows + 2 * RW_ROWS - 1) / (2 * RW_ROWS) >= 32 * warps ? 2 : 1;
}

template <int L, bool DOT, bool FAST, class T>
static void go(const Matrix& M, const SpmvParams<T>& p, cudaStream_t s) {
  if (rw_rpl<L>(M, p.rw_stage2) == 2)
    go_rpl<L, 2, DOT, FAST, T>(M, p, s);
  else
    go_rpl<L, 1, DOT, FAST, T>(M, p, s);
}

template <int L, bool DOT, class T>
static void go_l(const Matrix& M, bool fast, const SpmvParams<T>& p, cudaStream_t s) {
  if (fast)
    go<L, DOT, true, T>(M, p, s);
  else
    go<L, DOT, false, T>(M, p, s);
}

template <bool DOT, class T>
static void go_dot(const Matrix& M, int level, bool fast, const SpmvParams<T>& p,
                   cudaStream_t s) {
  if (M.kind == GSE_KIND_FP64) {
    go<0, DOT, false, T>(M, p, s);
  } else if (M.kind == GSE_KIND_FP16 || M.kind == GSE_KIND_BF16) {
    if constexpr (sizeof(T) == 8) {  // FP64 accumulation only
      if (M.kind == GSE_KIND_FP16)
        go<L_FP16, DOT, false, T>(M, p, s);
      else
        go<L_BF16, DOT, false, T>(M, p, s);
    }
  } else if (level == 1) {
    go_l<1, DOT, T>(M, fast, p, s);
  } else if (level == 2) {
    go_l<2, DOT, T>(M, fast, p, s);
  } else {
    go_l<3, DOT, T>(M, fast, p, s);
  }
}

template <>
void launch_rw<double>(const Matrix& M, int level, bool dot, bool fast,
                       const SpmvParams<double>& p, cudaStream_t s) {
  if (dot)
    go_dot<true, double>(M, level, fast, p, s);
  else
    go_dot<false, double>(M, level, fast, p, s);
}

template <>
void launch_rw<float>(const Matrix& M, int level, bool dot, bool fast,
                      const SpmvParams<float>& p, cudaStream_t s) {
  (void)dot;
  go_dot<false, float>(M, level, fast, p, s);
}

}  // namespace gse
