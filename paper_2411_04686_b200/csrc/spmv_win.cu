// spmv_win.cu -- "window" SpMV kernel for irregular row lengths (the power-law config C3,
// any matrix the row walk does not take).  SURVEY 8(a) a4-a6; paper Alg. spmv
// and P:212 for levels 2-3: y_i = sum_j dec_L(a_ij) x_j with FP64 (or FP32) accumulation.
//
// Why this shape: on the power-law matrix the previous strided-products
// kernel was bound by the L1 data pipe -- each warp-wide x gather touched ~13 distinct
// 128-byte lines and the row sums went through a shared-memory products tile.  Here:
//  * the encoder cuts the rows into row-aligned TILES of ~WIN_TNNZ non-zeros (<= WIN_RMAX
//    rows); a persistent CTA takes tiles round robin and, one tile ahead, stages the x
//    window x[R0 - WIN_HALF, R1 + WIN_HALF) in shared memory with ONE TMA bulk copy
//    (double-buffered).  SuiteSparse-like matrices keep most partners near the diagonal
//    (C3: 91 % within 512 columns), so those gathers become shared-memory loads (cost: the
//    bank conflicts of one random 8-byte access per lane, not one line per lane); the rest
//    are predicated global gathers that skip L1;
//  * lane l of a warp owns 8 CONSECUTIVE non-zeros of a 256-element chunk: its planes are
//    three to six 128-bit loads (only the requested planes), and it sums its own row
//    pieces in registers;
//  * row starts come from an encode-time bitmap (1 bit per non-zero, instead of reading
//    row_ptr) plus the row holding each chunk's first element; a lane's row index is an
//    exclusive warp scan of popcounts;
//  * rows that span lanes are closed by one segmented warp scan (shuffles) per chunk; rows
//    that span warps of a tile by a fixed-order pass of one thread at the tile end.
// Summation order differs from the oracle's sequential one (R25: parity by tolerance);
// it is fixed, so results and the fused dot are bitwise reproducible.
// Matrices with empty rows take a slower row-lookup path (EMPTY): their rows are found by
// binary search in row_ptr and their y entries zeroed per tile.
#include "spmv_common.cuh"

#include <map>
#include <mutex>
#include <utility>

namespace gse {

constexpr int WIN_THREADS = 256;
constexpr int WIN_WARPS = WIN_THREADS / 32;
static_assert(WIN_EPT == 8, "the plane loads below are written for 8 non-zeros per lane");

// predicated y store
__device__ __forceinline__ void stg_y(double* a, double v, uint32_t pred) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.global.f64 [%0], %1;\n}\n" ::"l"(a),
      "d"(v), "r"(pred)
      : "memory");
}
__device__ __forceinline__ void stg_y(float* a, float v, uint32_t pred) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.global.f32 [%0], %1;\n}\n" ::"l"(a),
      "f"(v), "r"(pred)
      : "memory");
}

// x operand: from the staged window when o < wlen (shared memory), else from global (no L1
// allocation); exactly one of the two predicated loads executes
__device__ __forceinline__ void x_near_or_far(double& v, uint32_t o, uint32_t wlen,
                                              uint32_t saddr, const double* g) {
  asm volatile(
      "{\n .reg .pred q;\n setp.lt.u32 q, %1, %2;\n @q ld.shared.f64 %0, [%3];\n"
      " @!q ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%4], %5;\n}\n"
      : "=d"(v)
      : "r"(o), "r"(wlen), "r"(saddr), "l"(g), "l"(l2_evict_last()));
}
__device__ __forceinline__ void x_near_or_far(float& v, uint32_t o, uint32_t wlen,
                                              uint32_t saddr, const float* g) {
  asm volatile(
      "{\n .reg .pred q;\n setp.lt.u32 q, %1, %2;\n @q ld.shared.f32 %0, [%3];\n"
      " @!q ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%4], %5;\n}\n"
      : "=f"(v)
      : "r"(o), "r"(wlen), "r"(saddr), "l"(g), "l"(l2_evict_last()));
}
// the same for a possibly masked element (ok = 0: neither load, v keeps its value)
__device__ __forceinline__ void x_near_or_far_masked(double& v, uint32_t o, uint32_t wlen,
                                                     uint32_t saddr, const double* g,
                                                     uint32_t ok) {
  asm volatile(
      "{\n .reg .pred q, k, n, f;\n setp.lt.u32 q, %1, %2;\n setp.ne.u32 k, %5, 0;\n"
      " and.pred n, q, k;\n not.pred q, q;\n and.pred f, q, k;\n"
      " @n ld.shared.f64 %0, [%3];\n @f ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%4], %6;\n}\n"
      : "+d"(v)
      : "r"(o), "r"(wlen), "r"(saddr), "l"(g), "r"(ok), "l"(l2_evict_last()));
}
__device__ __forceinline__ void x_near_or_far_masked(float& v, uint32_t o, uint32_t wlen,
                                                     uint32_t saddr, const float* g,
                                                     uint32_t ok) {
  asm volatile(
      "{\n .reg .pred q, k, n, f;\n setp.lt.u32 q, %1, %2;\n setp.ne.u32 k, %5, 0;\n"
      " and.pred n, q, k;\n not.pred q, q;\n and.pred f, q, k;\n"
      " @n ld.shared.f32 %0, [%3];\n @f ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%4], %6;\n}\n"
      : "+f"(v)
      : "r"(o), "r"(wlen), "r"(saddr), "l"(g), "r"(ok), "l"(l2_evict_last()));
}
// h += a b when in_h, else t += a b: two predicated FMAs, no selects
__device__ __forceinline__ void fma_split(double& h, double& t, bool in_h, double a, double b) {
  asm("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q fma.rn.f64 %0, %3, %4, %0;\n"
      " @!q fma.rn.f64 %1, %3, %4, %1;\n}\n"
      : "+d"(h), "+d"(t)
      : "r"((uint32_t)in_h), "d"(a), "d"(b));
}
__device__ __forceinline__ void fma_split(float& h, float& t, bool in_h, float a, float b) {
  asm("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q fma.rn.f32 %0, %3, %4, %0;\n"
      " @!q fma.rn.f32 %1, %3, %4, %1;\n}\n"
      : "+f"(h), "+f"(t)
      : "r"((uint32_t)in_h), "f"(a), "f"(b));
}
__device__ __forceinline__ double fma_t(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fma_t(float a, float b, float c) { return __fmaf_rn(a, b, c); }

__device__ __forceinline__ void unpack16(uint4 v, uint32_t* o) {
  o[0] = v.x & 0xFFFFu;
  o[1] = v.x >> 16;
  o[2] = v.y & 0xFFFFu;
  o[3] = v.y >> 16;
  o[4] = v.z & 0xFFFFu;
  o[5] = v.z >> 16;
  o[6] = v.w & 0xFFFFu;
  o[7] = v.w >> 16;
}

// row of the tile holding non-zero q: the last r in [R0, R1) with rp[r] <= q (empty rows
// share their start with the next row, so the last one is the non-empty row); q outside
// the tile maps to a row outside [R0, R1), whose writes are suppressed
__device__ __forceinline__ uint32_t row_of(const uint32_t* __restrict__ rp, uint32_t R0,
                                           uint32_t R1, uint32_t s, uint32_t e, uint32_t q,
                                           bool before_start) {
  if (before_start || q < s) return R0 - 1u;
  if (q >= e) return R1;
  uint32_t lo = R0, hi = R1;
  while (hi - lo > 1u) {
    const uint32_t mid = (lo + hi) >> 1;
    if (rp[mid] <= q)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

template <class T>
struct WinStash {  // per warp, double-buffered across tiles
  T head_val[2][WIN_WARPS], tail_val[2][WIN_WARPS];
  uint32_t head_row[2][WIN_WARPS], tail_row[2][WIN_WARPS];
  int state[2][WIN_WARPS];  // bit 0: warp had chunks, bit 1: warp closed a row
};

// resident CTAs per SM the register budget is sized for: 4 (64 registers) where the lane's
// planes fit, 3 for the 8-byte planes of level 3 / FP64 CSR (GSE_WIN_MINB: A/B knob)
#ifndef GSE_WIN_HIADD
#define GSE_WIN_HIADD 1
#endif
#ifndef GSE_WIN_HIADD3  // the same at level 3 (A/B)
#define GSE_WIN_HIADD3 1
#endif
#ifndef GSE_WIN_MINB_LO
#define GSE_WIN_MINB_LO 3
#endif
#ifndef GSE_WIN_MINB_HI
#define GSE_WIN_MINB_HI 3
#endif
#define WIN_MINB(L) ((L) == 3 || (L) == 0 ? GSE_WIN_MINB_HI : GSE_WIN_MINB_LO)
// 4 resident CTAs (64 registers) where that measured faster on C3: level 1 (FP64: 550 ->
// 526 us, FP32 428 -> 401 us) and level 2 with FP32 accumulation (447 -> 419 us); level 2
// FP64 and the fused-dot variants spill more at 64 registers and keep 3
// (profiles/r02k/win_c3_minb4.json vs win_c3_base_same_run_as_minb4.json)
#ifndef GSE_WIN_MINB4
#define GSE_WIN_MINB4 1
#endif
template <int L, bool DOT, class T>
constexpr int win_minb() {
  return (GSE_WIN_MINB4 && !DOT && (L == 1 || (L == 2 && sizeof(T) == 4))) ? 4 : WIN_MINB(L);
}

template <int L, bool SIDE, bool DOT, bool FAST, bool EMPTY, class T>
__global__ void __launch_bounds__(WIN_THREADS, (win_minb<L, DOT, T>())) k_spmv_win(const SpmvParams<T> p) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ long long sd64[64];
  __shared__ int sd32[64];
  __shared__ double sc64[64];
  __shared__ float sc32[64];
  // sign-folded scales (FAST): [EI | sign << ei_bits] = (sign ? -1 : 1) * scale[EI]
  // FP64: {ssc, -2^52 ssc} pairs (levels 1-2 decode as one FMA, one 16-byte table load)
  __shared__ __align__(16) T ssc2[256];
#if GSE_WIN_HIADD
  // FP64 levels 1-2: [EI | sign << ei_bits] = (k_EI << 20) + (sign << 31), added to the hi
  // word of the exactly converted D_L (|v| = D_L 2^k; FAST excludes under/overflow)
  __shared__ uint32_t shadd[128];
#endif
  __shared__ WinStash<T> stash;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t eb = 32u - (uint32_t)p.ei_shift;
  if constexpr (L >= 1 && L <= 3 && FAST) {
    if (threadIdx.x < 128) {
      const uint32_t t = threadIdx.x, sign = t >> eb, ei = t & ((1u << eb) - 1u);
      T v = (T)0;
      if (sign <= 1u) {
        if constexpr (sizeof(T) == 8)
          v = sign ? -p.sc64[ei] : p.sc64[ei];
        else
          v = sign ? -p.sc32[ei] : p.sc32[ei];
      }
      if constexpr (sizeof(T) == 8) {
        ssc2[2 * t] = v;
        ssc2[2 * t + 1] = -4503599627370496.0 * (double)v;
#if GSE_WIN_HIADD
        shadd[t] = sign <= 1u ? (uint32_t)(__double2hiint(p.sc64[ei]) - (1023 << 20)) + (sign << 31)
                              : 0u;
#endif
      } else {
        ssc2[t] = v;
      }
    }
  }
  stage_tables<L>(p, sd64, sd32, sc64, sc32);  // (includes a __syncthreads for L >= 1)
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  if (p.stop && *p.stop) return;
  pdl_trigger();

  T* const wbuf = reinterpret_cast<T*>(dsm);
  constexpr uint32_t A = 16u / sizeof(T);  // elements per 16 bytes (TMA granule)
  const uint32_t nt = p.n_tiles;
  auto window = [&](uint32_t t, uint32_t& wb, uint32_t& wlen) {
    const uint32_t R0 = p.tiles[t].row0, R1 = p.tiles[t + 1].row0;
    wb = R0 > WIN_HALF ? ((R0 - WIN_HALF) & ~(A - 1u)) : 0u;
    uint32_t we = R1 + WIN_HALF;
    we = we > p.cols ? p.cols : we;
    wlen = (p.win_on && we > wb) ? ((we - wb) & ~(A - 1u)) : 0u;
    wlen = wlen > WIN_CAP ? (WIN_CAP & ~(A - 1u)) : wlen;
  };
  auto issue = [&](uint32_t t, uint32_t buf) {
    uint32_t wb, wlen;
    window(t, wb, wlen);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect_tx(&bars[buf], wlen * (uint32_t)sizeof(T));
    if (wlen) bulk_g2s_keep(wbuf + (size_t)buf * WIN_CAP, p.x + wb, wlen * (uint32_t)sizeof(T),
                            &bars[buf]);
  };

  double dacc = 0.0;
  uint32_t t = blockIdx.x, it = 0;
  if (t < nt && threadIdx.x == 0) issue(t, 0);
  for (; t < nt; t += gridDim.x, ++it) {
    const uint32_t cur = it & 1u;
    if (t + gridDim.x < nt && threadIdx.x == 0) issue(t + gridDim.x, cur ^ 1u);
    const uint32_t R0 = p.tiles[t].row0, R1 = p.tiles[t + 1].row0;
    const uint32_t s = p.tiles[t].nnz0, e = p.tiles[t + 1].nnz0;
    const uint32_t nrows = R1 - R0;
    uint32_t wb, wlen;
    window(t, wb, wlen);
    const T* win = wbuf + (size_t)cur * WIN_CAP;
    if constexpr (EMPTY) {  // y = 0 on the tile's empty rows (no bit marks them)
      for (uint32_t r = R0 + threadIdx.x; r < R1; r += WIN_THREADS)
        if (p.row_ptr[r] == p.row_ptr[r + 1]) p.y[r] = (T)0;
    }
    // the tile's 256-element chunks, split into contiguous ranges per warp
    const uint32_t cA = s / WIN_CH, cB = (e + WIN_CH - 1u) / WIN_CH, nch = cB - cA;
    const uint32_t w0 = cA + (uint32_t)(((uint64_t)nch * warp) / WIN_WARPS);
    const uint32_t w1 = cA + (uint32_t)(((uint64_t)nch * (warp + 1)) / WIN_WARPS);
    mbar_wait(&bars[cur], (it >> 1) & 1u);

    const uint32_t win_s = smem_u32(win);
    // x of a row (the fused dot): staged when inside the window
    auto xrow = [&](uint32_t r) -> double {
      const uint32_t o = r - wb;
      return o < wlen ? (double)win[o] : (double)p.x[r];
    };
    auto write_row = [&](uint32_t r, T v) {
      if (r - R0 < nrows) {
        p.y[r] = v;
        if constexpr (DOT) {
          const uint32_t o = r - wb;
          const double xr = o < wlen ? (double)win[o] : (double)p.x[r];
          dacc += xr * (double)v;
        }
      }
    };

    T carry = (T)0;
    bool need_head = true;
    uint32_t last_row = 0;
    for (uint32_t c = w0; c < w1; ++c) {
      const uint32_t p0 = c * WIN_CH + (uint32_t)lane * WIN_EPT;
      const bool act = p0 < e && p0 + WIN_EPT > s;
      const uint32_t Mb = ld_nc_u8(p.rowbits + (p0 >> 3));  // row starts among the 8
      uint32_t cprev = 0;
      if constexpr (!EMPTY) cprev = __ldg(p.chunk_prev + c);
      // ---- planes (only the requested ones), 128-bit loads, evict-first in L2
      uint4 ca = make_uint4(0u, 0u, 0u, 0u), cb = ca, hq = ca, t1q = ca, t2a = ca, t2b = ca;
      uint2 sv = make_uint2(0u, 0u);
      uint4 vq[4] = {ca, ca, ca, ca};
      if (act) {
        ca = ld_nc_v4(p.col_ei + p0);
        cb = ld_nc_v4(p.col_ei + p0 + 4);
        if constexpr (L == 0) {
#pragma unroll
          for (int q = 0; q < 4; ++q) vq[q] = ld_nc_v4(p.val + p0 + 2 * q);
        }
        if constexpr (has_head<L>()) hq = ld_nc_v4(p.head + p0);
        if constexpr (has_t1<L>()) t1q = ld_nc_v4(p.tail1 + p0);
        if constexpr (has_t2<L>()) {
          t2a = ld_nc_v4(p.tail2 + p0);
          t2b = ld_nc_v4(p.tail2 + p0 + 4);
        }
        if constexpr (SIDE && L >= 1 && L <= 3) sv = ld_nc_v2(p.side + p0);
      }
      const uint32_t cw[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
      // level-L value of element j (masked elements: x = 0 below, so their finite value
      // contributes an exact zero; FP64 / 16-bit kinds select 0 since they may hold +-Inf)
      auto value = [&](int j) -> T {
        const uint32_t hw = j < 2 ? hq.x : j < 4 ? hq.y : j < 6 ? hq.z : hq.w;
        const uint32_t h = (j & 1) ? (hw >> 16) : (hw & 0xFFFFu);
        if constexpr (L == 0) {
          const uint4 v = vq[j >> 1];
          return (T)((j & 1) ? __hiloint2double((int)v.w, (int)v.z)
                             : __hiloint2double((int)v.y, (int)v.x));
        } else if constexpr (is_half<L>()) {
          return (T)half_value<L>(h);
        } else {
          const uint32_t tw = j < 2 ? t1q.x : j < 4 ? t1q.y : j < 6 ? t1q.z : t1q.w;
          const uint32_t t1 = (j & 1) ? (tw >> 16) : (tw & 0xFFFFu);
          const uint32_t t2 = j == 0 ? t2a.x : j == 1 ? t2a.y : j == 2 ? t2a.z : j == 3 ? t2a.w
                            : j == 4 ? t2b.x : j == 5 ? t2b.y : j == 6 ? t2b.z : t2b.w;
          uint32_t ei = 0u;
          if constexpr (SIDE) ei = ((j < 4 ? sv.x : sv.y) >> (8 * (j & 3))) & 63u;
          if constexpr (FAST) {
            // scale index EI | sign << ei_bits (one funnel shift when EI is in the column)
            const uint32_t idx = SIDE ? (ei | ((h >> 15) << eb))
                                      : __funnelshift_rc(cw[j], h >> 15, p.ei_shift);
            if constexpr (L == 1) {
              const uint32_t D = h & 0x7FFFu;
#if GSE_WIN_HIADD
              if constexpr (sizeof(T) == 8) {  // exact D, exponent + sign by one integer add
                const double dv = __uint2double_rn(D);
                const int e = (int)shadd[idx];
                return __hiloint2double(__double2hiint(dv) + (D ? e : 0), 0);
              }
#endif
              // (2^52 + D) sc - 2^52 sc = D sc exactly (D < 2^31, sc = +-2^k): one FMA
              if constexpr (sizeof(T) == 8)
              {
                const double2 sn = reinterpret_cast<const double2*>(ssc2)[idx];
                return __fma_rn(__hiloint2double(0x43300000, (int)D), sn.x, sn.y);
              } else {
                return (float)(int)D * ssc2[idx];
              }
            } else if constexpr (L == 2) {
              const uint32_t D = ((h & 0x7FFFu) << 16) | t1;
#if GSE_WIN_HIADD
              if constexpr (sizeof(T) == 8) {
                const double dv = __uint2double_rn(D);
                const int e = (int)shadd[idx];
                return __hiloint2double(__double2hiint(dv) + (D ? e : 0), __double2loint(dv));
              }
#endif
              if constexpr (sizeof(T) == 8)
              {
                const double2 sn = reinterpret_cast<const double2*>(ssc2)[idx];
                return __fma_rn(__hiloint2double(0x43300000, (int)D), sn.x, sn.y);
              } else {
                return __uint2float_rz(D) * ssc2[idx];
              }
            } else {
              const uint64_t D = ((uint64_t)(h & 0x7FFFu) << 48) | ((uint64_t)t1 << 32) | t2;
#if GSE_WIN_HIADD3
              if constexpr (sizeof(T) == 8) {  // encoder output: D has <= 53 significant bits
                const double dv = __ull2double_rz(D);
                const int hi = __double2hiint(dv);
                const int e = (int)shadd[idx];
                return __hiloint2double(hi ? hi + e : 0, __double2loint(dv));
              }
#endif
              if constexpr (sizeof(T) == 8)
                return __ull2double_rz(D) * ssc2[2 * idx];
              else
                return __ull2float_rz(D) * ssc2[idx];
            }
          } else {
            if constexpr (!SIDE) ei = __funnelshift_rc(cw[j], 0u, p.ei_shift);
            if constexpr (sizeof(T) == 8)
              return dec64<L, false>(h, t1, t2, sd64, sc64, ei);
            else
              return dec32<L, false>(h, t1, t2, sd32, sc32, ei);
          }
        }
      };
      // ---- this lane's row (the row open at its first element), relative to R0 ---------
      uint32_t rr;
      if constexpr (EMPTY) {
        rr = row_of(p.row_ptr, R0, R1, s, e, p0 - 1u, p0 == 0u) - R0;
      } else {
        const uint32_t cnt = __popc(Mb);
        uint32_t inc = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
          if (lane >= d) inc += o;
        }
        rr = cprev + (inc - cnt) - R0;
      }
      const uint32_t rr_open = rr;
      T hsum = (T)0, acc = (T)0;  // before the lane's first row start / from its last one
      // fast path (warp-uniform): the chunk lies inside the tile and no lane sees two row
      // starts -- every gather is one predicated shared-or-global load, the lane's values
      // go to one of two FMA chains, no stores
      const bool simple = !EMPTY && c * WIN_CH >= s && (c + 1) * WIN_CH <= e &&
                          !__any_sync(0xFFFFFFFFu, (Mb & (Mb - 1u)) != 0u);
      if (simple) {
        T xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t col = cw[j] & p.col_mask;
          const uint32_t o = col - wb;
          x_near_or_far(xv[j], o, wlen, win_s + o * (uint32_t)sizeof(T), p.x + col);
        }
        const uint32_t f = Mb ? (uint32_t)(__ffs(Mb) - 1) : 8u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const bool at = (uint32_t)j == f;  // the lane's row start: close the head piece
          hsum = at ? acc : hsum;
          acc = fma_t(value(j), xv[j], at ? (T)0 : acc);
        }
        if (!Mb) hsum = acc;
        rr += Mb ? 1u : 0u;
      } else {
        uint32_t vm = 0;  // elements of this lane inside the tile
        if (act) {
          const uint32_t lo = s > p0 ? s - p0 : 0u, hi = e - p0 < 8u ? e - p0 : 8u;
          vm = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
        }
        T xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t col = cw[j] & p.col_mask;
          const uint32_t o = col - wb;
          xv[j] = (T)0;
          x_near_or_far_masked(xv[j], o, wlen, win_s + o * (uint32_t)sizeof(T), p.x + col,
                               (vm >> j) & 1u);
        }
        const uint32_t first = Mb & (0u - Mb), rest = Mb ^ first;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t st = (Mb >> j) & 1u;
          if (j > 0) {  // a row that starts and ends inside this lane (never at j = 0)
            const uint32_t wr = ((rest >> j) & 1u) & (rr < nrows ? 1u : 0u);
            if constexpr (EMPTY) {
              if (wr) write_row(R0 + rr, acc);
            } else {
              stg_y(p.y + (R0 + rr), acc, wr);
              if constexpr (DOT) dacc += wr ? xrow(R0 + rr) * (double)acc : 0.0;
            }
          }
          hsum = ((first >> j) & 1u) ? acc : hsum;  // closes the row open before this lane
          if constexpr (EMPTY) {
            if (st) rr = row_of(p.row_ptr, R0, R1, s, e, p0 + j, false) - R0;
          } else {
            rr += st;
          }
          acc = st ? (T)0 : acc;
          T a = value(j);
          if constexpr (L == 0 || is_half<L>()) a = ((vm >> j) & 1u) ? a : (T)0;
          acc = fma_t(a, xv[j], acc);
        }
        if (!Mb) hsum = acc;  // no row starts here: the whole lane continues the open row
      }
      // ---- rows spanning lanes: segmented scan (segments start at lanes with a row start)
      const unsigned fl = __ballot_sync(0xFFFFFFFFu, Mb != 0u);
      const unsigned le = fl & (0xFFFFFFFFu >> (31 - lane));
      const int seg = le ? 31 - __clz(le) : -1;
      T sc = acc;  // the open row's piece at this lane's end (the whole lane if no start)
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const T o = __shfl_up_sync(0xFFFFFFFFu, sc, d);
        if (lane - d >= seg && lane >= d) sc += o;
      }
      T prev = __shfl_up_sync(0xFFFFFFFFu, sc, 1);
      if (lane == 0) prev = (T)0;
      if ((fl & ((1u << lane) - 1u)) == 0u) prev += carry;
      if (fl) {
        const T val = prev + hsum;
        const bool head = need_head && lane == __ffs(fl) - 1;
        if (head) {
          stash.head_row[cur][warp] = R0 + rr_open;
          stash.head_val[cur][warp] = val;
        }
        const uint32_t wr = (Mb != 0u && !head && rr_open < nrows) ? 1u : 0u;
        if constexpr (EMPTY) {
          if (wr) write_row(R0 + rr_open, val);
        } else {
          stg_y(p.y + (R0 + rr_open), val, wr);
          if constexpr (DOT) dacc += wr ? xrow(R0 + rr_open) * (double)val : 0.0;
        }
        need_head = false;
      }
      const T s31 = __shfl_sync(0xFFFFFFFFu, sc, 31);
      carry = fl ? s31 : carry + s31;
      last_row = __shfl_sync(0xFFFFFFFFu, R0 + rr, 31);
    }
    if (lane == 0) {
      stash.tail_row[cur][warp] = last_row;
      stash.tail_val[cur][warp] = carry;
      stash.state[cur][warp] = (w1 > w0 ? 1 : 0) | (need_head ? 0 : 2);
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // rows spanning warps, in warp order (fixed summation order)
      bool pend = false;
      uint32_t pr = 0;
      T pv = (T)0;
      for (int w = 0; w < WIN_WARPS; ++w) {
        const int st = stash.state[cur][w];
        if (!(st & 1)) continue;
        const uint32_t tr = stash.tail_row[cur][w];
        const T tv = stash.tail_val[cur][w];
        if (st & 2) {
          const uint32_t hr = stash.head_row[cur][w];
          T hv = stash.head_val[cur][w];
          if (pend && pr == hr)
            hv = pv + hv;
          else if (pend)
            write_row(pr, pv);
          write_row(hr, hv);
          pend = true;
          pr = tr;
          pv = tv;
        } else if (pend && pr == tr) {
          pv += tv;
        } else {
          if (pend) write_row(pr, pv);
          pend = true;
          pr = tr;
          pv = tv;
        }
      }
      if (pend) write_row(pr, pv);
    }
  }
  if constexpr (DOT) finalize_dot(warp_sum(dacc), p.partials, p.ticket, p.dot_result);
}

// Launch configuration per instantiation: the dynamic shared-memory attribute (two window
// buffers) is set once, the occupancy cached per device.
template <int L, bool SIDE, bool DOT, bool FAST, bool EMPTY, class T>
static void go(const Matrix& M, const SpmvParams<T>& p, cudaStream_t s) {
  static std::mutex mu;
  static int grid[64] = {0};
  auto kern = k_spmv_win<L, SIDE, DOT, FAST, EMPTY, T>;
  const size_t smem = 2 * (size_t)WIN_CAP * sizeof(T);
  const int dev = M.device < 64 ? M.device : 0;
  int cap;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!grid[dev]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int blocks = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, WIN_THREADS, smem);
      grid[dev] = (blocks < 1 ? 1 : blocks) * num_sms(M.device);
    }
    cap = grid[dev];
  }
  const int g = (int)(M.n_tiles < cap ? M.n_tiles : cap);
  launch_k(kern, g < 1 ? 1 : g, WIN_THREADS, smem, s, p);
}

template <int L, bool DOT, bool FAST, class T>
static void go_e(const Matrix& M, const SpmvParams<T>& p, cudaStream_t s) {
  const bool side = M.kind == GSE_KIND_GSE && !M.ei_in_column;
  if (M.n_empty_rows) {
    if (side)
      go<L, true, DOT, FAST, true, T>(M, p, s);
    else
      go<L, false, DOT, FAST, true, T>(M, p, s);
  } else {
    if (side)
      go<L, true, DOT, FAST, false, T>(M, p, s);
    else
      go<L, false, DOT, FAST, false, T>(M, p, s);
  }
}

template <bool DOT, class T>
static void go_dot(const Matrix& M, int level, bool fast, const SpmvParams<T>& p,
                   cudaStream_t s) {
  if (M.kind == GSE_KIND_FP64) {
    if (M.n_empty_rows)
      go<0, false, DOT, false, true, T>(M, p, s);
    else
      go<0, false, DOT, false, false, T>(M, p, s);
  } else if (M.kind == GSE_KIND_FP16 || M.kind == GSE_KIND_BF16) {
    if constexpr (sizeof(T) == 8) {  // FP64 accumulation only
      const bool em = M.n_empty_rows != 0;
      if (M.kind == GSE_KIND_FP16)
        em ? go<L_FP16, false, DOT, false, true, T>(M, p, s)
           : go<L_FP16, false, DOT, false, false, T>(M, p, s);
      else
        em ? go<L_BF16, false, DOT, false, true, T>(M, p, s)
           : go<L_BF16, false, DOT, false, false, T>(M, p, s);
    }
  } else if (level == 1) {
    fast ? go_e<1, DOT, true, T>(M, p, s) : go_e<1, DOT, false, T>(M, p, s);
  } else if (level == 2) {
    fast ? go_e<2, DOT, true, T>(M, p, s) : go_e<2, DOT, false, T>(M, p, s);
  } else {
    fast ? go_e<3, DOT, true, T>(M, p, s) : go_e<3, DOT, false, T>(M, p, s);
  }
}

template <>
void launch_win<double>(const Matrix& M, int level, bool dot, bool fast,
                        const SpmvParams<double>& p, cudaStream_t s) {
  if (dot)
    go_dot<true, double>(M, level, fast, p, s);
  else
    go_dot<false, double>(M, level, fast, p, s);
}

template <>
void launch_win<float>(const Matrix& M, int level, bool dot, bool fast,
                       const SpmvParams<float>& p, cudaStream_t s) {
  (void)dot;
  go_dot<false, float>(M, level, fast, p, s);
}

}  // namespace gse
