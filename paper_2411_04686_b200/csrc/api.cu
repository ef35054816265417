// api.cu -- the extern "C" entry points of include/gse.h: argument validation, host/device
// pointer staging, device selection, error detail, allocator hook.  No arithmetic of the
// method lives here; every step runs in the kernels of encode.cu / spmv.cu / solvers.cu.
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>

#include "gse_internal.cuh"
#include "vec16.cuh"

namespace gse {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

gse_status cuda_status(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  cudaGetLastError();
  return e == cudaErrorMemoryAllocation ? GSE_ERR_OOM : GSE_ERR_CUDA;
}

static void* (*g_alloc)(size_t, void*, void*) = nullptr;
static void (*g_free)(void*, void*, void*) = nullptr;
static void* g_ctx = nullptr;

// The default stream-ordered pool returns freed memory to the OS at every synchronisation
// (release threshold 0), which turns each encode / solver-workspace allocation into fresh
// page mapping (milliseconds).  Keep freed blocks cached in the pool instead.
static void keep_pool_cached() {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done[dev] = true;
}

void* dev_alloc(size_t bytes, cudaStream_t s) {
  if (bytes == 0) bytes = 16;
  bytes = (bytes + 255) & ~(size_t)255;
  if (g_alloc) {
    void* p = g_alloc(bytes, (void*)s, g_ctx);
    if (!p) {
      set_error("the caller allocator returned NULL for " + std::to_string(bytes) + " bytes");
      return nullptr;
    }
    // TMA bulk copies and 16-byte vector loads of the planes need aligned bases
    if (reinterpret_cast<uintptr_t>(p) & 255u) {
      g_free(p, (void*)s, g_ctx);
      set_error("the caller allocator must return 256-byte aligned memory (as cudaMalloc does)");
      return nullptr;
    }
    return p;
  }
  keep_pool_cached();
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) {
    cudaGetLastError();
    set_error("device allocation of " + std::to_string(bytes) + " bytes failed");
    return nullptr;
  }
  return p;
}

void dev_free(void* p, cudaStream_t s) {
  if (!p) return;
  if (g_free)
    g_free(p, (void*)s, g_ctx);
  else
    cudaFreeAsync(p, s);
}

bool is_device_ptr(const void* p, int* device) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
    if (device) *device = a.device;
    return true;
  }
  return false;
}

int num_sms(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) device = 0;
  if (!cache[device]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cache[device] = v > 0 ? v : 148;
  }
  return cache[device];
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("GSE_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// input array: device pointers pass through, host arrays are staged (freed by ~Staging)
struct Staging {
  cudaStream_t s;
  void* bufs[8] = {nullptr};
  int n = 0;
  bool synced_needed = false;
  explicit Staging(cudaStream_t st) : s(st) {}
  template <class T>
  gse_status in(const T* p, size_t count, int dev, const T** out) {
    int d = -1;
    if (count == 0 || p == nullptr || is_device_ptr(p, &d)) {
      if (p && count && d != dev) {
        set_error("device pointer lives on device " + std::to_string(d) + ", matrix on " +
                  std::to_string(dev));
        return GSE_ERR_INVALID_ARG;
      }
      *out = p;
      return GSE_OK;
    }
    T* b = static_cast<T*>(dev_alloc(count * sizeof(T), s));
    if (!b) return GSE_ERR_OOM;
    bufs[n++] = b;
    GSE_CUDA_TRY(cudaMemcpyAsync(b, p, count * sizeof(T), cudaMemcpyHostToDevice, s));
    *out = b;
    return GSE_OK;
  }
  // output (or in/out) array: returns a device pointer; host arrays get a device buffer,
  // filled from the host when copy_in, copied back by out_done()
  template <class T>
  gse_status out(T* p, size_t count, int dev, bool copy_in, T** dptr) {
    int d = -1;
    if (count == 0 || p == nullptr || is_device_ptr(p, &d)) {
      if (p && count && d != dev) {
        set_error("device pointer lives on another device than the matrix");
        return GSE_ERR_INVALID_ARG;
      }
      *dptr = p;
      return GSE_OK;
    }
    T* b = static_cast<T*>(dev_alloc(count * sizeof(T), s));
    if (!b) return GSE_ERR_OOM;
    bufs[n++] = b;
    if (copy_in) GSE_CUDA_TRY(cudaMemcpyAsync(b, p, count * sizeof(T), cudaMemcpyHostToDevice, s));
    *dptr = b;
    return GSE_OK;
  }
  template <class T>
  gse_status out_done(T* host, const T* dptr, size_t count) {
    if (host == dptr || count == 0) return GSE_OK;
    GSE_CUDA_TRY(cudaMemcpyAsync(host, dptr, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    synced_needed = true;
    return GSE_OK;
  }
  gse_status finish() {
    if (synced_needed || n) GSE_CUDA_TRY(cudaStreamSynchronize(s));
    return GSE_OK;
  }
  ~Staging() {
    for (int i = 0; i < n; ++i) dev_free(bufs[i], s);
  }
};

static gse_status check_csr(const gse_csr_f64* A) {
  if (!A) {
    set_error("A is NULL");
    return GSE_ERR_INVALID_ARG;
  }
  if (A->rows < 0 || A->cols < 0 || A->nnz < 0 || (A->nnz > 0 && (!A->col_idx || !A->values)) ||
      !A->row_ptr) {
    set_error("invalid CSR sizes or NULL arrays");
    return GSE_ERR_INVALID_ARG;
  }
  if (A->nnz >= (1LL << 32) || A->rows >= (1LL << 31) || A->cols >= (1LL << 32)) {
    set_error("this build requires nnz < 2^32, rows < 2^31, cols < 2^32");
    return GSE_ERR_INVALID_ARG;
  }
  return GSE_OK;
}

static int pick_device(int requested, const void* probe) {
  if (requested >= 0) return requested;
  int d = 0;
  if (is_device_ptr(probe, &d)) return d;
  return 0;
}

static void destroy_matrix(Matrix& M) {
  DeviceGuard g(M.device);
  cudaStream_t s = nullptr;
  free_solver_ws(M);
  free_dist(M);
  void* ps[] = {M.row_ptr, M.col_ei, M.side_ei, M.head, M.tail1, M.tail2, M.val, M.blocks,
                M.tiles, M.rowbits, M.chunk_prev, M.dtab};
  for (void* p : ps) dev_free(p, s);
  cudaStreamSynchronize(s);
}

gse_status create_from_csr(const gse_csr_f64* A, int kind, int k_max, int device,
                           gse_matrix* out, cudaStream_t s, Matrix** mout, Comm* comm,
                           const int32_t* local_col, int64_t sample_block_rows,
                           uint64_t sample_seed, int shard_table) {
  gse_status rc = check_csr(A);
  if (rc != GSE_OK) return rc;
  if (!out) {
    set_error("out is NULL");
    return GSE_ERR_INVALID_ARG;
  }
  *out = nullptr;
  const int dev = pick_device(device, A->values ? (const void*)A->values : A->row_ptr);
  DeviceGuard g(dev);
  Staging st(s);
  const void* rp = nullptr;
  const int32_t* col = nullptr;
  const double* val = nullptr;
  if (A->row_ptr_64)
    rc = st.in((const long long*)A->row_ptr, (size_t)A->rows + 1, dev, (const long long**)&rp);
  else
    rc = st.in((const int*)A->row_ptr, (size_t)A->rows + 1, dev, (const int**)&rp);
  if (rc == GSE_OK)
    rc = st.in(local_col ? local_col : A->col_idx, (size_t)A->nnz, dev, &col);
  if (rc == GSE_OK) rc = st.in(A->values, (size_t)A->nnz, dev, &val);
  if (rc != GSE_OK) return rc;
  gse_matrix h = new gse_matrix_s();
  Matrix& M = h->m;
  M.device = dev;
  M.rows = A->rows;
  M.cols = A->cols;
  M.nnz = A->nnz;
  M.k_max = k_max;
  if (kind == GSE_KIND_GSE)
    rc = encode_matrix(M, *A, rp, A->row_ptr_64, col, val, s, comm, sample_block_rows,
                       sample_seed, shard_table);
  else
    rc = fp64_matrix(M, rp, A->row_ptr_64, col, val, s, kind);
  if (rc == GSE_OK) rc = st.finish();
  if (rc != GSE_OK) {
    destroy_matrix(M);
    delete h;
    return rc;
  }
  *out = h;
  if (mout) *mout = &h->m;
  return GSE_OK;
}

static gse_status check_sched(const gse_step_schedule* sc) {
  if (sc->start_level < 1 || sc->start_level > 3) {
    set_error("start_level must be 1..3");
    return GSE_ERR_INVALID_ARG;
  }
  if (sc->enabled) {
    if (sc->max_level < sc->start_level || sc->max_level > 3 || sc->t < 1 || sc->m < 1 ||
        sc->l < 0 || sc->t > (1 << 20)) {
      set_error("invalid schedule (need start <= max_level <= 3, t >= 1, m >= 1, l >= 0)");
      return GSE_ERR_INVALID_ARG;
    }
  }
  if (!(sc->perturb_c >= 0.0) || !std::isfinite(sc->perturb_c)) {
    set_error("perturb_c must be finite and >= 0 (0 = off)");
    return GSE_ERR_INVALID_ARG;
  }
  if (sc->cg_keep_direction != 0 && sc->cg_keep_direction != 1) {
    set_error("cg_keep_direction must be 0 or 1");
    return GSE_ERR_INVALID_ARG;
  }
  return GSE_OK;
}

}  // namespace gse

using namespace gse;

extern "C" {

const char* gse_status_string(gse_status s) {
  switch (s) {
    case GSE_OK: return "ok";
    case GSE_NOT_CONVERGED: return "not converged (max iterations)";
    case GSE_NUMERICAL_ABORT: return "numerical abort (breakdown or non-finite residual)";
    case GSE_ERR_INVALID_ARG: return "invalid argument";
    case GSE_ERR_DIM_MISMATCH: return "dimension mismatch";
    case GSE_ERR_NONFINITE: return "non-finite value";
    case GSE_ERR_NO_VALUES: return "no representable values";
    case GSE_ERR_UNREPRESENTABLE: return "unrepresentable exponent";
    case GSE_ERR_INVALID_EXP_INDEX: return "invalid exponent index";
    case GSE_ERR_FP32_RANGE: return "table exceeds the FP32 range";
    case GSE_ERR_WRONG_FORMAT: return "operation not defined for this matrix kind";
    case GSE_ERR_CUDA: return "CUDA error";
    case GSE_ERR_NCCL: return "NCCL error";
    case GSE_ERR_OOM: return "out of device memory";
  }
  return "unknown status";
}

const char* gse_last_error_detail(void) { return g_err.c_str(); }

gse_status gse_set_allocator(void* (*alloc)(size_t, void*, void*), void (*free_)(void*, void*, void*),
                             void* ctx) {
  if ((alloc == nullptr) != (free_ == nullptr)) {
    set_error("alloc and free must both be set or both be NULL");
    return GSE_ERR_INVALID_ARG;
  }
  g_alloc = alloc;
  g_free = free_;
  g_ctx = ctx;
  return GSE_OK;
}

void gse_default_schedule(int solver, gse_step_schedule* o) {
  if (!o) return;
  memset(o, 0, sizeof(*o));
  o->enabled = 1;
  o->start_level = 1;
  o->max_level = 3;
  o->verify_at_full = 1;
  if (solver == 0) {  // CG, P:433 / P:441
    o->l = 3000; o->t = 250; o->m = 500;
    o->rsd_limit = 0.50; o->ndec_limit = 130; o->reldec_limit = 0.45;
  } else {            // GMRES
    o->l = 9000; o->t = 300; o->m = 1500;
    o->rsd_limit = 0.03; o->ndec_limit = 80; o->reldec_limit = 0.08;
  }
}

gse_status gse_encode(const gse_csr_f64* A, const gse_encode_opts* opts, gse_matrix* out,
                      void* stream) {
  gse::NvtxRange nvtx_("gse_encode");
  gse_encode_opts o = {8, -1, 0, 0, 0};
  if (opts) o = *opts;
  if (o.k_max < 1 || o.k_max > 64 || (o.k_max & (o.k_max - 1))) {
    set_error("k_max must be a power of two in [1, 64]");
    return GSE_ERR_INVALID_ARG;
  }
  if (o.sample_block_rows < 0) {
    set_error("sample_block_rows must be >= 0 (0 = full histogram)");
    return GSE_ERR_INVALID_ARG;
  }
  return create_from_csr(A, GSE_KIND_GSE, o.k_max, o.device, out, (cudaStream_t)stream, nullptr,
                         nullptr, nullptr, o.sample_block_rows, o.seed);
}

gse_status gse_fp64_matrix(const gse_csr_f64* A, int device, gse_matrix* out, void* stream) {
  gse::NvtxRange nvtx_("gse_fp64_matrix");
  return create_from_csr(A, GSE_KIND_FP64, 1, device, out, (cudaStream_t)stream, nullptr, nullptr,
                         nullptr);
}

gse_status gse_half_matrix(const gse_csr_f64* A, int kind, int device, gse_matrix* out,
                           void* stream) {
  gse::NvtxRange nvtx_("gse_half_matrix");
  if (kind != GSE_KIND_FP16 && kind != GSE_KIND_BF16) {
    set_error("kind must be GSE_KIND_FP16 or GSE_KIND_BF16");
    return GSE_ERR_INVALID_ARG;
  }
  return create_from_csr(A, kind, 1, device, out, (cudaStream_t)stream, nullptr, nullptr, nullptr);
}

gse_status gse_matrix_get_info(gse_matrix A, gse_matrix_info* info) {
  if (!A || !info) {
    set_error("NULL argument");
    return GSE_ERR_INVALID_ARG;
  }
  const Matrix& M = A->m;
  memset(info, 0, sizeof(*info));
  info->kind = M.kind;
  info->k_max = M.k_max;
  info->ei_bits = M.ei_bits;
  info->ei_in_column = M.ei_in_column;
  info->table_len = M.table_len;
  memcpy(info->table, M.table, sizeof(M.table));
  info->rows = M.rows;
  info->cols = M.cols;
  info->nnz = M.nnz;
  info->n_blocks = M.n_blocks;
  info->n_zero_values = M.n_zero;
  info->device = M.device;
  info->spmv_mode = M.spmv_mode;
  if (M.kind == GSE_KIND_GSE) {
    info->plane_bytes[0] = (size_t)M.nnz * 4;
    info->plane_bytes[1] = (size_t)M.nnz * 2;
    info->plane_bytes[2] = (size_t)M.nnz * 2;
    info->plane_bytes[3] = (size_t)M.nnz * 4;
    info->plane_bytes[4] = M.ei_in_column ? 0 : (size_t)M.nnz;
  } else {
    info->plane_bytes[0] = (size_t)M.nnz * 4;
    info->plane_bytes[1] = (size_t)M.nnz * (M.kind == GSE_KIND_FP64 ? 8 : 2);
  }
  return GSE_OK;
}

gse_status gse_matrix_copy_planes(gse_matrix A, uint32_t* col_ei, uint8_t* side_ei,
                                  uint16_t* head, uint16_t* tail1, uint32_t* tail2,
                                  uint16_t* table, void* stream) {
  if (!A) {
    set_error("NULL matrix");
    return GSE_ERR_INVALID_ARG;
  }
  const Matrix& M = A->m;
  if (M.kind != GSE_KIND_GSE && (side_ei || tail1 || tail2 || table)) {
    set_error("FP64 / FP16 / BF16 matrices have no GSE planes");
    return GSE_ERR_WRONG_FORMAT;
  }
  if (M.kind == GSE_KIND_FP64 && head) {
    set_error("FP64 matrices have no 16-bit plane");
    return GSE_ERR_WRONG_FORMAT;
  }
  DeviceGuard g(M.device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t n = (size_t)M.nnz;
  if (col_ei && n) GSE_CUDA_TRY(cudaMemcpyAsync(col_ei, M.col_ei, n * 4, cudaMemcpyDefault, s));
  if (side_ei && n && M.side_ei)
    GSE_CUDA_TRY(cudaMemcpyAsync(side_ei, M.side_ei, n, cudaMemcpyDefault, s));
  if (head && n) GSE_CUDA_TRY(cudaMemcpyAsync(head, M.head, n * 2, cudaMemcpyDefault, s));
  if (tail1 && n) GSE_CUDA_TRY(cudaMemcpyAsync(tail1, M.tail1, n * 2, cudaMemcpyDefault, s));
  if (tail2 && n) GSE_CUDA_TRY(cudaMemcpyAsync(tail2, M.tail2, n * 4, cudaMemcpyDefault, s));
  if (table) GSE_CUDA_TRY(cudaMemcpyAsync(table, M.table, M.table_len * 2, cudaMemcpyDefault, s));
  GSE_CUDA_TRY(cudaStreamSynchronize(s));
  return GSE_OK;
}

gse_status gse_decode(gse_matrix A, int segments, double* values, void* stream) {
  gse::NvtxRange nvtx_("gse_decode");
  if (!A || segments < 1 || segments > 3) {
    set_error("invalid matrix or segments (must be 1, 2 or 3)");
    return GSE_ERR_INVALID_ARG;
  }
  const Matrix& M = A->m;
  if (M.kind != GSE_KIND_GSE) {
    set_error("decode needs a GSE matrix");
    return GSE_ERR_WRONG_FORMAT;
  }
  DeviceGuard g(M.device);
  cudaStream_t s = (cudaStream_t)stream;
  Staging st(s);
  double* d = nullptr;
  gse_status rc = st.out(values, (size_t)M.nnz, M.device, false, &d);
  if (rc != GSE_OK) return rc;
  rc = decode_all(M, segments, d, s);
  if (rc != GSE_OK) return rc;
  rc = st.out_done(values, d, (size_t)M.nnz);
  if (rc != GSE_OK) return rc;
  return st.finish();
}

gse_status gse_spmv(gse_matrix A, const double* x, double* y, int segments, void* stream) {
  gse::NvtxRange nvtx_("gse_spmv");
  if (!A || segments < 1 || segments > 3) {
    set_error("invalid matrix or segments (must be 1, 2 or 3)");
    return GSE_ERR_INVALID_ARG;
  }
  const Matrix& M = A->m;
  if (M.kind != GSE_KIND_GSE && segments != 3) {
    set_error("an FP64 / FP16 / BF16 CSR matrix is read at full precision only (segments = 3)");
    return GSE_ERR_WRONG_FORMAT;
  }
  const int64_t xlen = M.dist ? dist_n_local(M) : M.cols;  // dist: x is the rank's slice
  if ((xlen > 0 && !x) || (M.rows > 0 && !y)) {
    set_error("x or y is NULL");
    return GSE_ERR_INVALID_ARG;
  }
  DeviceGuard g(M.device);
  cudaStream_t s = (cudaStream_t)stream;
  Staging st(s);
  const double* dx = nullptr;
  double* dy = nullptr;
  gse_status rc = st.in(x, (size_t)xlen, M.device, &dx);
  if (rc == GSE_OK) rc = st.out(y, (size_t)M.rows, M.device, false, &dy);
  if (rc != GSE_OK) return rc;
  if (M.dist) {  // owned entries -> x_ext, halo exchange (interior rows overlapped), SpMV
    double* xe = dist_xext(M);
    if (xlen) GSE_CUDA_TRY(cudaMemcpyAsync(xe, dx, 8 * xlen, cudaMemcpyDeviceToDevice, s));
    rc = dist_spmv(M, segments, xe, dy, nullptr, s, nullptr);
  } else {
    rc = launch_spmv(M, segments, dx, dy, nullptr, s);
  }
  if (rc != GSE_OK) return rc;
  rc = st.out_done(y, dy, (size_t)M.rows);
  if (rc != GSE_OK) return rc;
  return st.finish();
}

gse_status gse_spmv_dot(gse_matrix A, const double* x, double* y, int segments, double* dot,
                        void* stream) {
  gse::NvtxRange nvtx_("gse_spmv_dot");
  if (!A || segments < 1 || segments > 3 || !dot) {
    set_error("invalid matrix, segments (must be 1, 2 or 3) or NULL dot");
    return GSE_ERR_INVALID_ARG;
  }
  Matrix& M = A->m;
  if (M.kind != GSE_KIND_GSE && segments != 3) {
    set_error("an FP64 / FP16 / BF16 CSR matrix is read at full precision only (segments = 3)");
    return GSE_ERR_WRONG_FORMAT;
  }
  if (M.dist) {
    set_error("gse_spmv_dot is single-GPU (a distributed dot needs the allreduce of a solve)");
    return GSE_ERR_WRONG_FORMAT;
  }
  if (M.rows != M.cols) {
    set_error("x . y needs a square matrix");
    return GSE_ERR_DIM_MISMATCH;
  }
  if ((M.cols > 0 && !x) || (M.rows > 0 && !y)) {
    set_error("x or y is NULL");
    return GSE_ERR_INVALID_ARG;
  }
  DeviceGuard g(M.device);
  cudaStream_t s = (cudaStream_t)stream;
  Staging st(s);
  const double* dx = nullptr;
  double* dy = nullptr;
  double* dd = nullptr;
  gse_status rc = st.in(x, (size_t)M.cols, M.device, &dx);
  if (rc == GSE_OK) rc = st.out(y, (size_t)M.rows, M.device, false, &dy);
  if (rc == GSE_OK) rc = st.out(dot, 1, M.device, false, &dd);
  if (rc != GSE_OK) return rc;
  rc = spmv_dot_ws(M, segments, dx, dy, dd, s);
  if (rc != GSE_OK) return rc;
  rc = st.out_done(y, dy, (size_t)M.rows);
  if (rc == GSE_OK) rc = st.out_done(dot, dd, 1);
  if (rc != GSE_OK) return rc;
  return st.finish();
}

gse_status gse_perturbation_bounds(gse_matrix A, double* eta, void* stream) {
  gse::NvtxRange nvtx_("gse_perturbation_bounds");
  if (!A || !eta) {
    set_error("NULL matrix or eta");
    return GSE_ERR_INVALID_ARG;
  }
  Matrix& M = A->m;
  DeviceGuard g(M.device);
  gse_status rc = perturbation_bounds(M, (cudaStream_t)stream);
  if (rc != GSE_OK) return rc;
  eta[0] = M.eta[0];
  eta[1] = M.eta[1];
  return GSE_OK;
}

gse_status gse_spmv_f32acc(gse_matrix A, const float* x, float* y, int segments, void* stream) {
  gse::NvtxRange nvtx_("gse_spmv_f32acc");
  if (!A || segments < 1 || segments > 3) {
    set_error("invalid matrix or segments (must be 1, 2 or 3)");
    return GSE_ERR_INVALID_ARG;
  }
  const Matrix& M = A->m;
  if (M.kind != GSE_KIND_GSE || M.dist) {
    set_error("FP32 accumulation is defined for single-GPU GSE matrices");
    return GSE_ERR_WRONG_FORMAT;
  }
  if (!M.fp32_ok) {
    set_error("the shared-exponent table represents values >= 2^128 (outside FP32)");
    return GSE_ERR_FP32_RANGE;
  }
  if ((M.cols > 0 && !x) || (M.rows > 0 && !y)) {
    set_error("x or y is NULL");
    return GSE_ERR_INVALID_ARG;
  }
  DeviceGuard g(M.device);
  cudaStream_t s = (cudaStream_t)stream;
  Staging st(s);
  const float* dx = nullptr;
  float* dy = nullptr;
  gse_status rc = st.in(x, (size_t)M.cols, M.device, &dx);
  if (rc == GSE_OK) rc = st.out(y, (size_t)M.rows, M.device, false, &dy);
  if (rc != GSE_OK) return rc;
  rc = launch_spmv_f32(M, segments, dx, dy, s);
  if (rc != GSE_OK) return rc;
  rc = st.out_done(y, dy, (size_t)M.rows);
  if (rc != GSE_OK) return rc;
  return st.finish();
}

static gse_status solve_common(gse_matrix A, const double* b, double* x, double tol,
                               int64_t max_iters, const gse_step_schedule* sched, int restart,
                               gse_solve_report* rep, void* stream, bool gmres) {
  if (!A) {
    set_error("NULL matrix");
    return GSE_ERR_INVALID_ARG;
  }
  Matrix& M = A->m;
  if (!M.dist && M.rows != M.cols) {  // (a distributed matrix was checked square at encode)
    set_error("solvers need a square matrix");
    return GSE_ERR_DIM_MISMATCH;
  }
  if (!(tol > 0.0) || max_iters < 0 || (M.rows > 0 && (!b || !x))) {
    set_error("invalid tol (must be > 0), max_iters or NULL b/x");
    return GSE_ERR_INVALID_ARG;
  }
  if (gmres && (restart < 1 || restart > 64)) {
    set_error("restart must be in [1, 64]");
    return GSE_ERR_INVALID_ARG;
  }
  gse_step_schedule sc;
  if (sched) {
    sc = *sched;
  } else {
    gse_default_schedule(gmres ? 1 : 0, &sc);
    sc.enabled = 0;
    sc.start_level = 3;
  }
  gse_status rc = check_sched(&sc);
  if (rc != GSE_OK) return rc;
  if (M.dist && sc.enabled && sc.perturb_c > 0.0) {
    set_error("the R29 perturbation trigger (perturb_c) is single-GPU only");
    return GSE_ERR_WRONG_FORMAT;
  }
  if (M.dist && sc.enabled && sc.cg_keep_direction) {
    set_error("the R30 kept direction (cg_keep_direction) is single-GPU only");
    return GSE_ERR_WRONG_FORMAT;
  }
  gse_solve_report r;
  memset(&r, 0, sizeof(r));
  DeviceGuard g(M.device);
  cudaStream_t s = (cudaStream_t)stream;
  Staging st(s);
  const double* db = nullptr;
  double* dx = nullptr;
  rc = st.in(b, (size_t)M.rows, M.device, &db);
  if (rc == GSE_OK) rc = st.out(x, (size_t)M.rows, M.device, true, &dx);
  if (rc != GSE_OK) return rc;
  gse_status status;
  if (M.rows == 0) {
    r.converged = 1;
    status = GSE_OK;
  } else if (gmres) {
    status = solve_gmres(M, db, dx, tol, restart, max_iters, sc, r, s);
  } else {
    status = solve_cg(M, db, dx, tol, max_iters, sc, r, s);
  }
  if (status >= GSE_ERR_INVALID_ARG) return status;
  rc = st.out_done(x, dx, (size_t)M.rows);
  if (rc == GSE_OK) rc = st.finish();
  if (rc != GSE_OK) return rc;
  if (rep) *rep = r;
  return status;
}

gse_status gse_solve_cg(gse_matrix A, const double* b, double* x, double tol, int64_t max_iters,
                        const gse_step_schedule* sched, gse_solve_report* rep, void* stream) {
  gse::NvtxRange nvtx_("gse_solve_cg");
  return solve_common(A, b, x, tol, max_iters, sched, 0, rep, stream, false);
}

gse_status gse_solve_gmres(gse_matrix A, const double* b, double* x, double tol, int restart,
                           int64_t max_iters, const gse_step_schedule* sched,
                           gse_solve_report* rep, void* stream) {
  gse::NvtxRange nvtx_("gse_solve_gmres");
  return solve_common(A, b, x, tol, max_iters, sched, restart, rep, stream, true);
}

gse_status gse_encode_vector16(const double* v, int64_t n, int k_max, uint16_t* words,
                               uint16_t* table, int* table_len, void* stream) {
  gse::NvtxRange nvtx_("gse_encode_vector16");
  if (n < 0 || (n > 0 && (!v || !words)) || !table || !table_len || k_max < 1 ||
      k_max > V16_KMAX || (k_max & (k_max - 1))) {
    set_error("invalid arguments (k_max a power of two in [1, 16], non-NULL arrays)");
    return GSE_ERR_INVALID_ARG;
  }
  int dev = 0;
  if (!(v && is_device_ptr(v, &dev))) cudaGetDevice(&dev);
  DeviceGuard g(dev);
  cudaStream_t s = (cudaStream_t)stream;
  int eb = 0;
  while ((1 << eb) < k_max) ++eb;
  Staging st(s);
  const double* dv = nullptr;
  uint16_t* dw = nullptr;
  gse_status rc = st.in(v, (size_t)n, dev, &dv);
  if (rc == GSE_OK) rc = st.out(words, (size_t)n, dev, false, &dw);
  if (rc != GSE_OK) return rc;
  unsigned* hist = dev_alloc_n<unsigned>(2048, s);
  uint16_t* dt = dev_alloc_n<uint16_t>(V16_KMAX, s);
  int* dl = dev_alloc_n<int>(1, s);
  if (!hist || !dt || !dl) return GSE_ERR_OOM;
  GSE_CUDA_TRY(cudaMemsetAsync(hist, 0, 2048 * sizeof(unsigned), s));
  const int grid = num_sms(dev) * 4;
  if (n > 0) v16_hist(dv, nullptr, n, hist, nullptr, grid, s);
  v16_select(hist, k_max, dt, dl, nullptr, s);
  if (n > 0) v16_encode(dv, nullptr, n, dt, dl, eb, dw, nullptr, nullptr, grid, s);
  GSE_CUDA_TRY(cudaGetLastError());
  rc = st.out_done(words, dw, (size_t)n);
  if (rc != GSE_OK) return rc;
  uint16_t ht[V16_KMAX];
  int hl = 0;
  GSE_CUDA_TRY(cudaMemcpyAsync(ht, dt, sizeof(ht), cudaMemcpyDeviceToHost, s));
  GSE_CUDA_TRY(cudaMemcpyAsync(&hl, dl, sizeof(int), cudaMemcpyDeviceToHost, s));
  GSE_CUDA_TRY(cudaStreamSynchronize(s));
  dev_free(hist, s);
  dev_free(dt, s);
  dev_free(dl, s);
  for (int i = 0; i < hl; ++i) table[i] = ht[i];
  *table_len = hl;
  return st.finish();
}

gse_status gse_decode_vector16(const uint16_t* words, int64_t n, const uint16_t* table,
                               int table_len, int ei_bits, double* out, void* stream) {
  gse::NvtxRange nvtx_("gse_decode_vector16");
  if (n < 0 || (n > 0 && (!words || !out)) || (table_len > 0 && !table) || ei_bits < 0 ||
      ei_bits > 4 || table_len < 0 || table_len > (1 << ei_bits) || table_len > V16_KMAX) {
    set_error("invalid arguments (ei_bits in [0, 4], table_len <= 2^ei_bits)");
    return GSE_ERR_INVALID_ARG;
  }
  if (n == 0) return GSE_OK;
  int dev = 0;
  if (!is_device_ptr(words, &dev)) cudaGetDevice(&dev);
  DeviceGuard g(dev);
  cudaStream_t s = (cudaStream_t)stream;
  Staging st(s);
  const uint16_t* dw = nullptr;
  double* dout = nullptr;
  gse_status rc = st.in(words, (size_t)n, dev, &dw);
  if (rc == GSE_OK) rc = st.out(out, (size_t)n, dev, false, &dout);
  if (rc != GSE_OK) return rc;
  uint16_t ht[V16_KMAX] = {0};
  for (int i = 0; i < table_len; ++i) ht[i] = table[i];
  uint16_t* dt = dev_alloc_n<uint16_t>(V16_KMAX, s);
  int* dl = dev_alloc_n<int>(1, s);
  if (!dt || !dl) return GSE_ERR_OOM;
  GSE_CUDA_TRY(cudaMemcpyAsync(dt, ht, sizeof(ht), cudaMemcpyHostToDevice, s));
  GSE_CUDA_TRY(cudaMemcpyAsync(dl, &table_len, sizeof(int), cudaMemcpyHostToDevice, s));
  v16_decode(dw, n, dt, dl, ei_bits, dout, num_sms(dev) * 4, s);
  GSE_CUDA_TRY(cudaGetLastError());
  rc = st.out_done(out, dout, (size_t)n);
  if (rc != GSE_OK) return rc;
  GSE_CUDA_TRY(cudaStreamSynchronize(s));  // (host table staged through pageable memory)
  dev_free(dt, s);
  dev_free(dl, s);
  return st.finish();
}

void gse_matrix_free(gse_matrix A) {
  if (!A) return;
  destroy_matrix(A->m);
  delete A;
}

}  // extern "C"
