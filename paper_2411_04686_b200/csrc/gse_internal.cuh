// gse_internal.cuh -- internal types of the B200 GSE-SEM library (not part of the ABI).
// Everything here is the product path; it shares nothing with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only; no-ops unless a profiler injects a handler

#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>

#include "../../include/gse.h"

namespace gse {

// NVTX range around each C-ABI call (encode, SpMV, solves) and marks at level switches, so
// ncu --nvtx / nsys timelines attribute the kernels to the paper's operations
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---------------------------------------------------------------- SpMV partition constants
// A "warp block" (the unit one warp of the SpMV kernel processes) covers a run of
// consecutive rows whose starts fall in one CHUNK of the nnz stream, all of length <= LMAX,
// or a single long row (> LMAX nnz).  A short block holds <= CHUNK - 1 + LMAX <= WTILE
// non-zeros, so one pass of 32 lanes x EPL elements covers it.
constexpr int SPMV_THREADS = 256;            // 8 independent warps per CTA
constexpr int SPMV_WARPS = SPMV_THREADS / 32;
constexpr int EPL = 8;                       // elements per lane per pass
constexpr int WTILE = 32 * EPL;              // 256 non-zeros per warp pass
constexpr uint32_t LMAX = 64;
constexpr uint32_t CHUNK = 192;
static_assert(CHUNK - 1 + LMAX <= WTILE, "short warp block must fit one pass");
// Row-walk mode (regular matrices, e.g. stencils): groups of 32 consecutive rows, the
// group's planes staged into warp-private shared memory with 16-byte loads, lane = row.
constexpr int RW_ROWS = 32;
constexpr int RW_TILE = 1024;  // max staged span (8-aligned non-zeros) of a row-walk group
// Window mode (irregular rows, e.g. the power-law config; spmv_win.cu): row-aligned tiles
// of ~WIN_TNNZ non-zeros and <= WIN_RMAX rows; the CTA stages x[R0 - WIN_HALF, R1 + WIN_HALF)
// in shared memory by one TMA bulk copy, warps walk 256-element chunks with 8 consecutive
// non-zeros per lane, row starts come from a 1-bit-per-non-zero bitmap (encode-time).
constexpr int WIN_EPT = 8;                  // consecutive non-zeros per lane and chunk
constexpr int WIN_CH = 32 * WIN_EPT;        // non-zeros per warp chunk
#ifndef GSE_WIN_HALF
#define GSE_WIN_HALF 384
#endif
#ifndef GSE_WIN_RMAX
#define GSE_WIN_RMAX 1280
#endif
constexpr uint32_t WIN_HALF = GSE_WIN_HALF;  // x window reaches this many columns past the rows
constexpr uint32_t WIN_RMAX = GSE_WIN_RMAX;  // rows per tile (bounds the window)
#ifndef GSE_WIN_TNNZ
#define GSE_WIN_TNNZ 16384
#endif
constexpr uint32_t WIN_TNNZ = GSE_WIN_TNNZ; // target non-zeros per tile
constexpr uint32_t WIN_CAP = WIN_RMAX + 2 * WIN_HALF + 8;  // window buffer (elements)
enum SpmvMode : int { SPMV_SP = 0, SPMV_RW = 1, SPMV_WIN = 2 };
constexpr int NNZ_PAD = 8;  // plane allocations padded to a multiple of 8 elements (+8)

struct BlockDesc {
  uint32_t row0;  // first row of the block
  uint32_t nnz0;  // row_ptr[row0]
};

// decode constants per level: |v| = D_L * 2^(E - 1086 + s_L),
// s_L = 48 / 32 / 0 for L = 1 / 2 / 3, applied by adding delta to the bits of double(D_L).
struct DecodeTable {
  long long d64[3][64];  // (E - 1086 + s_L) << 52
  int d32[3][64];        // (E - 1086 + s_L) << 23 (FP32 accumulation)
  // multiply form used by the SpMV when no decoded value can underflow (E >= 16 / 32 / 64
  // at levels 1 / 2 / 3 for FP64; E - 1086 + s_L >= -126 for FP32): |v| = D_L * scale.
  double sc64[3][64];
  float sc32[3][64];
  int fast64[3], fast32[3];
};

struct SolverWs;  // solvers.cu
struct DistCtx;   // dist.cu
struct Comm;      // dist.cu: NCCL or thread-group collectives of one rank

struct Matrix {
  int kind = GSE_KIND_GSE;
  int device = 0;
  int64_t rows = 0, cols = 0, nnz = 0;
  int k_max = 8, ei_bits = 3, ei_in_column = 1, table_len = 0;
  uint16_t table[64] = {0};
  int64_t n_zero = 0;
  int fp32_ok = 0;
  // device arrays
  uint32_t* row_ptr = nullptr;  // [rows + 1]
  uint32_t* col_ei = nullptr;   // [nnz_pad] column | EI << (32 - ei_bits)  (or plain column)
  uint8_t* side_ei = nullptr;   // [nnz_pad] when !ei_in_column
  uint16_t* head = nullptr;     // [nnz_pad] (FP16 / BF16 kinds: the 16-bit codes)
  uint16_t* tail1 = nullptr;    // [nnz_pad]
  uint32_t* tail2 = nullptr;    // [nnz_pad]
  double* val = nullptr;        // [nnz_pad] FP64 kind
  BlockDesc* blocks = nullptr;  // [n_blocks + 1]
  int64_t n_blocks = 0;
  // window mode (spmv_win.cu)
  BlockDesc* tiles = nullptr;     // [n_tiles + 1] {first row, its row_ptr}
  int64_t n_tiles = 0;
  uint32_t* rowbits = nullptr;    // bit i of the stream: a non-empty row starts at non-zero i
  uint32_t* chunk_prev = nullptr; // [n_chunks] row holding non-zero c * WIN_CH - 1 (~0 for c = 0)
  int64_t n_empty_rows = 0;
  int spmv_mode = SPMV_SP;      // chosen at encode from the row-length statistics
  int64_t n_groups = 0;         // ceil(rows / 32)
  int64_t heavy_groups = 0;     // groups with > RW_TILE non-zeros
  int64_t max_row_len = 0;
  int64_t rw_span = 0;          // max staged span of a group (sizes the RW smem stages)
  int64_t rw_span2 = 0;         // the same for 64-row groups (two rows per lane)
  double rw_efficiency = 0.0;   // sum(len) / sum over groups of 32 * max(len)
  DecodeTable* dtab = nullptr;  // device copy
  DecodeTable htab;             // host copy
  SolverWs* ws = nullptr;
  double eta[2] = {0.0, 0.0};   // R29 ||A_3 - A_L||_inf, L = 1, 2 (valid when eta_ok)
  int eta_ok = 0;
  DistCtx* dist = nullptr;      // non-null for a row-partitioned matrix
  int64_t n_local_cols = 0;     // dist: owned + halo columns
};

// ---------------------------------------------------------------- errors / allocation
void set_error(const std::string& msg);
gse_status cuda_status(cudaError_t e, const char* what);

#define GSE_CUDA_TRY(expr)                                                     \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) return ::gse::cuda_status(_e, #expr);                \
  } while (0)

void* dev_alloc(size_t bytes, cudaStream_t s);
void dev_free(void* p, cudaStream_t s);

template <class T>
T* dev_alloc_n(size_t n, cudaStream_t s) {
  return static_cast<T*>(dev_alloc(n * sizeof(T) + 0, s));
}

// planes are allocated to a multiple of 8 elements + 128 zeroed elements: the SpMV kernels
// over-copy up to 64 elements past a block (spmv_sp.cu / spmv_rw.cu)
inline size_t padded(int64_t nnz) { return (size_t)((nnz + NNZ_PAD - 1) / NNZ_PAD) * NNZ_PAD + 128; }

bool is_device_ptr(const void* p, int* device);

int num_sms(int device);

// ---------------------------------------------------------------- programmatic dependent launch
// The GMRES loop launches its kernels with the programmatic-stream-serialization attribute:
// a kernel may be scheduled while its predecessor drains, runs its prologue on constant
// data (decode tables, barriers, the first matrix tiles), then waits in pdl_wait() until the
// predecessor has completed and its writes are visible.  Every kernel launched through
// launch_pdl calls pdl_wait() before touching data another kernel writes, and pdl_trigger()
// only after its own pdl_wait(), so a kernel never overlaps the one two launches back.
// GSE_NO_PDL=1 launches plainly (the device calls are then no-ops).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();

template <class... KArgs, class... Args>
cudaError_t launch_ex(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// plain stream-ordered launch (measured: PDL slows the CG loop by ~2%, whose kernels are long)
template <class... KArgs, class... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  return launch_ex(false, kern, grid, block, smem, s, std::forward<Args>(args)...);
}
// programmatic dependent launch (GMRES: chains of short MGS kernels, ~6% faster per inner
// iteration on C4 at 64^3)
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  return launch_ex(true, kern, grid, block, smem, s, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- kernels (launchers)
// encode.cu
gse_status build_partition(Matrix& M, cudaStream_t s, const void* extra_d = nullptr,
                           void* extra_h = nullptr, size_t extra_bytes = 0);
// sample_block_rows > 0: table from one sampled row per row block (NEXT-3)
gse_status encode_matrix(Matrix& M, const gse_csr_f64& A, const void* d_row_ptr, int rp64,
                         const int32_t* d_col, const double* d_val, cudaStream_t s,
                         Comm* comm = nullptr, int64_t sample_block_rows = 0,
                         uint64_t sample_seed = 0, int shard_table = 0);
// kind: GSE_KIND_FP64 (values copied) or GSE_KIND_FP16 / GSE_KIND_BF16 (RNE to 16 bits, R26)
gse_status fp64_matrix(Matrix& M, const void* d_row_ptr, int rp64, const int32_t* d_col,
                       const double* d_val, cudaStream_t s, int kind = GSE_KIND_FP64);
void build_decode_table(Matrix& M);
gse_status decode_all(const Matrix& M, int level, double* out, cudaStream_t s);
// R29: M.eta = max_i sum_j |dec_3(a_ij) - dec_L(a_ij)| (row sums in storage order, bit-exact
// with the oracle), computed once per matrix (synchronises s)
gse_status perturbation_bounds(Matrix& M, cudaStream_t s);

// spmv.cu
struct DotOut {
  double* partials = nullptr;   // [n_blocks]
  unsigned* ticket = nullptr;   // last-block counter (reset by the last block)
  double* result = nullptr;     // deterministic sum of partials
};
gse_status launch_spmv(const Matrix& M, int level, const double* x, double* y,
                       const DotOut* dot, cudaStream_t s, const int* stop = nullptr);
gse_status launch_spmv_guarded(const Matrix& M, int level, const double* x, double* y,
                               const int* stop, cudaStream_t s);
gse_status launch_spmv_rows(const Matrix& M, int level, const double* x, double* y,
                            const DotOut* dot, cudaStream_t s, const int* stop, int64_t r0,
                            int64_t r1);
gse_status launch_spmv_f32(const Matrix& M, int level, const float* x, float* y,
                           cudaStream_t s);

// solvers.cu
gse_status solve_cg(Matrix& M, const double* b, double* x, double tol, int64_t max_iters,
                    const gse_step_schedule& sched, gse_solve_report& rep, cudaStream_t s);
gse_status solve_gmres(Matrix& M, const double* b, double* x, double tol, int restart,
                       int64_t max_iters, const gse_step_schedule& sched,
                       gse_solve_report& rep, cudaStream_t s);
void free_solver_ws(Matrix& M);
// y = A_L x and *dot = x . y (device pointers) with the CG's fused SpMV + dot kernel
gse_status spmv_dot_ws(Matrix& M, int level, const double* x, double* y, double* dot,
                       cudaStream_t s);

// dist.cu
gse_status dist_halo_exchange(const Matrix& M, double* x_local_ext, cudaStream_t s);
// SpMV of a distributed matrix on x_ext (owned entries in place): the halo exchange, with the
// interior rows' SpMV overlapped on a side stream when the matrix has an interior row range
gse_status dist_spmv(const Matrix& M, int level, double* x_ext, double* y, const DotOut* dot,
                     cudaStream_t s, const int* stop);
gse_status dist_allreduce_sum(const Matrix& M, double* d_vals, int count, cudaStream_t s);
// the distributed CG iteration batch can be captured in a CUDA graph: NCCL backend (its
// collectives are stream-capturable), not the thread backend (host barriers);
// GSE_DIST_NO_GRAPH=1 keeps the host-driven batches
bool dist_capturable(const Matrix& M);
gse_status comm_allreduce_u64(Comm* c, unsigned long long* d, int count, cudaStream_t s);
gse_status comm_any(Comm* c, int local_flag, int* any);  // host: OR over ranks
double* dist_xext(const Matrix& M);
int64_t dist_ext_cols(const Matrix& M);
int64_t dist_n_local(const Matrix& M);
void free_dist(Matrix& M);
gse_status create_from_csr(const gse_csr_f64* A, int kind, int k_max, int device,
                           gse_matrix* out, cudaStream_t s, Matrix** mout, Comm* comm,
                           const int32_t* local_col, int64_t sample_block_rows = 0,
                           uint64_t sample_seed = 0, int shard_table = 0);

}  // namespace gse

struct gse_matrix_s {
  gse::Matrix m;
};
