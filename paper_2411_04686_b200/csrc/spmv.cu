// spmv.cu -- SpMV entry points: build the kernel parameters for the
// requested level and dispatch to the kernel the encoder chose for this matrix
// (Matrix::spmv_mode: spmv_rw.cu for regular rows, spmv_win.cu otherwise; spmv_sp.cu on
// request for A/B).
// "SpMV kernel" for the design and profiles/ for the measurements behind it.
#include <cstdlib>
#include <cstring>

#include "spmv_common.cuh"

namespace gse {

template <class T>
static SpmvParams<T> make_params(const Matrix& M, int level, const T* x, T* y,
                                 const DotOut* dot) {
  SpmvParams<T> p;
  p.blocks = M.blocks;
  p.row_ptr = M.row_ptr;
  p.col_ei = M.col_ei;
  p.side = M.side_ei;
  p.head = M.head;
  p.tail1 = M.tail1;
  p.tail2 = M.tail2;
  p.val = M.val;
  p.n_blocks = (uint32_t)M.n_blocks;
  p.rows = (uint32_t)M.rows;
  p.n_groups = (uint32_t)M.n_groups;
  p.rw_stage = (uint32_t)((M.rw_span + 15) / 16 * 16 + 16);  // + over-copy (spmv_rw.cu)
  p.rw_stage2 = (uint32_t)((M.rw_span2 + 15) / 16 * 16 + 16);
  p.ei_shift = 32 - M.ei_bits;
  p.col_mask = (M.kind == GSE_KIND_GSE && M.ei_in_column && M.ei_bits)
                   ? ((1u << (32 - M.ei_bits)) - 1u)
                   : 0xFFFFFFFFu;
  p.x = x;
  p.xd = x;
  p.y = y;
  p.partials = dot ? dot->partials : nullptr;
  p.ticket = dot ? dot->ticket : nullptr;
  p.dot_result = dot ? dot->result : nullptr;
  p.stop = nullptr;
  p.tiles = M.tiles;
  p.rowbits = reinterpret_cast<const uint8_t*>(M.rowbits);
  p.chunk_prev = M.chunk_prev;
  p.n_tiles = (uint32_t)M.n_tiles;
  p.nnz_pad = (uint32_t)padded(M.nnz);
  p.cols = (uint32_t)dist_ext_cols(M);
  p.win_on = ((reinterpret_cast<uintptr_t>(x) & 15u) == 0) ? 1 : 0;
  const int L = level >= 1 && level <= 3 ? level : 3;
  for (int i = 0; i < 64; ++i) {
    p.d64[i] = M.htab.d64[L - 1][i];
    p.d32[i] = M.htab.d32[L - 1][i];
    p.sc64[i] = M.htab.sc64[L - 1][i];
    p.sc32[i] = M.htab.sc32[L - 1][i];
  }
  return p;
}

static int mode_of(const Matrix& M) { return M.spmv_mode; }

template <class T>
static void dispatch(const Matrix& M, int level, bool dot, const SpmvParams<T>& p,
                     cudaStream_t s) {
  const int L = level >= 1 && level <= 3 ? level : 3;
  const bool fast = M.kind == GSE_KIND_GSE &&
                    (sizeof(T) == 8 ? M.htab.fast64[L - 1] : M.htab.fast32[L - 1]);
  const int mode = mode_of(M);
  if (mode == SPMV_RW)
    launch_rw<T>(M, level, dot, fast, p, s);
  else if (mode == SPMV_WIN)
    launch_win<T>(M, level, dot, fast, p, s);
  else
    launch_sp<T>(M, level, dot, fast, p, s);
}

static bool empty_matrix(const Matrix& M) {
  return M.kind == GSE_KIND_GSE ? M.rows == 0 : M.rows == 0;
}

gse_status launch_spmv(const Matrix& M, int level, const double* x, double* y,
                       const DotOut* dot, cudaStream_t s, const int* stop) {
  if (empty_matrix(M)) {
    if (dot) GSE_CUDA_TRY(cudaMemsetAsync(dot->result, 0, sizeof(double), s));
    return GSE_OK;
  }
  SpmvParams<double> p = make_params<double>(M, level, x, y, dot);
  p.stop = stop;
  dispatch<double>(M, level, dot != nullptr, p, s);
  GSE_CUDA_TRY(cudaGetLastError());
  return GSE_OK;
}

// y[r0:r1) = (A_L x)[r0:r1): the row-walk kernel over a row view (row_ptr + r0, y + r0;
// the gathers still index the whole x).  r0 must be a multiple of 64 so the view's groups
// are the matrix's own groups (their staged spans are what rw_span bounds).
gse_status launch_spmv_rows(const Matrix& M, int level, const double* x, double* y,
                            const DotOut* dot, cudaStream_t s, const int* stop, int64_t r0,
                            int64_t r1) {
  if (r1 <= r0) return GSE_OK;
  if (M.spmv_mode != SPMV_RW || (r0 & 63) || r1 > M.rows) {
    set_error("internal: row views need a row-walk matrix and 64-aligned starts");
    return GSE_ERR_INVALID_ARG;
  }
  SpmvParams<double> p = make_params<double>(M, level, x, y, dot);
  p.stop = stop;
  p.row_ptr = M.row_ptr + r0;
  p.rows = (uint32_t)(r1 - r0);
  p.y = y + r0;
  p.xd = x + r0;
  launch_rw<double>(M, level, dot != nullptr,
                    M.kind == GSE_KIND_GSE && M.htab.fast64[(level >= 1 && level <= 3 ? level : 3) - 1],
                    p, s);
  GSE_CUDA_TRY(cudaGetLastError());
  return GSE_OK;
}

gse_status launch_spmv_guarded(const Matrix& M, int level, const double* x, double* y,
                               const int* stop, cudaStream_t s) {
  if (empty_matrix(M)) return GSE_OK;
  SpmvParams<double> p = make_params<double>(M, level, x, y, nullptr);
  p.stop = stop;
  dispatch<double>(M, level, false, p, s);
  GSE_CUDA_TRY(cudaGetLastError());
  return GSE_OK;
}

gse_status launch_spmv_f32(const Matrix& M, int level, const float* x, float* y,
                           cudaStream_t s) {
  if (empty_matrix(M)) return GSE_OK;
  dispatch<float>(M, level, false, make_params<float>(M, level, x, y, nullptr), s);
  GSE_CUDA_TRY(cudaGetLastError());
  return GSE_OK;
}

}  // namespace gse
