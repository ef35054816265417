// dist.cu -- row-partitioned multi-GPU execution (the paper is single-GPU).
//
// One process (or thread) per GPU rank.  A rank owns rows [row_begin, row_begin + n_local)
// and keeps GLOBAL column ids only at encode time:
//  * the shared-exponent table is global: the exponent histograms are summed over ranks
//    before the table is selected (R21), so every rank encodes with the identical table;
//  * columns are renumbered locally: owned -> [0, n_local), halo -> n_local + position in the
//    sorted list of referenced non-owned columns (grouped by owner rank because ownership
//    ranges are contiguous); the EI is embedded into the LOCAL index;
//  * every SpMV packs the owned entries peers need and exchanges halos (NCCL grouped
//    send/recv, or device copies in the thread backend) into x_ext[n_local ...];
//  * dot products are local partials + an allreduce; all ranks see identical sums, so the
//    residual monitor takes identical decisions everywhere without extra synchronisation.
//
// Two communication backends with one interface:
//  * NcclComm: NCCL over NVLink / NVSwitch (one process per GPU, unique id bootstrap);
//  * ThreadComm: P host threads in one process sharing one or more GPUs (streams + events +
//    device copies).  It runs the identical distributed code path on a single GPU, which is
//    how the P-rank CG is parity-tested on the one-GPU test box.
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "gse_internal.cuh"
#include "scan.cuh"

namespace gse {

// ---------------------------------------------------------------- communicator interface
struct Comm {
  int rank = 0, nranks = 1, device = 0;
  virtual ~Comm() {}
  virtual gse_status allreduce_sum_f64(double* d, int count, cudaStream_t s) = 0;
  virtual gse_status allreduce_sum_u64(unsigned long long* d, int count, cudaStream_t s) = 0;
  // synchronous host-level helpers (setup only)
  virtual gse_status host_allgather(int64_t v, std::vector<int64_t>& out) = 0;
  virtual gse_status host_alltoallv(const std::vector<std::vector<int64_t>>& send,
                                    std::vector<std::vector<int64_t>>& recv) = 0;
  // halo exchange: send_buf[send_off[p] .. +send_cnt[p]) -> rank p; receive from rank p into
  // recv_base + recv_off[p]
  virtual gse_status exchange(const double* send_buf, const std::vector<int64_t>& send_cnt,
                              const std::vector<int64_t>& send_off, double* recv_base,
                              const std::vector<int64_t>& recv_cnt,
                              const std::vector<int64_t>& recv_off, cudaStream_t s) = 0;
};

// ---------------------------------------------------------------- NCCL backend
static gse_status nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return GSE_OK;
  set_error(std::string(what) + ": " + ncclGetErrorString(r));
  return GSE_ERR_NCCL;
}
#define GSE_NCCL_TRY(expr)                                      \
  do {                                                          \
    gse_status _s = nccl_status((expr), #expr);                 \
    if (_s != GSE_OK) return _s;                                \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  cudaStream_t setup = nullptr;
  ~NcclComm() override {
    if (comm) ncclCommDestroy(comm);
    if (setup) cudaStreamDestroy(setup);
  }
  gse_status allreduce_sum_f64(double* d, int count, cudaStream_t s) override {
    GSE_NCCL_TRY(ncclAllReduce(d, d, count, ncclDouble, ncclSum, comm, s));
    return GSE_OK;
  }
  gse_status allreduce_sum_u64(unsigned long long* d, int count, cudaStream_t s) override {
    GSE_NCCL_TRY(ncclAllReduce(d, d, count, ncclUint64, ncclSum, comm, s));
    return GSE_OK;
  }
  gse_status host_allgather(int64_t v, std::vector<int64_t>& out) override {
    int64_t* buf = dev_alloc_n<int64_t>((size_t)nranks + 1, setup);
    if (!buf) return GSE_ERR_OOM;
    GSE_CUDA_TRY(cudaMemcpyAsync(buf + rank, &v, 8, cudaMemcpyHostToDevice, setup));
    GSE_NCCL_TRY(ncclAllGather(buf + rank, buf, 1, ncclInt64, comm, setup));
    out.assign(nranks, 0);
    GSE_CUDA_TRY(cudaMemcpyAsync(out.data(), buf, 8 * nranks, cudaMemcpyDeviceToHost, setup));
    GSE_CUDA_TRY(cudaStreamSynchronize(setup));
    dev_free(buf, setup);
    return GSE_OK;
  }
  gse_status host_alltoallv(const std::vector<std::vector<int64_t>>& send,
                            std::vector<std::vector<int64_t>>& recv) override {
    // counts first (every rank learns what it receives), then the payloads
    recv.assign(nranks, {});
    std::vector<int64_t> rc(nranks, 0);
    std::vector<int64_t> mine(nranks);
    for (int p = 0; p < nranks; ++p) mine[p] = (int64_t)send[p].size();
    int64_t* dcnt = dev_alloc_n<int64_t>((size_t)nranks * nranks, setup);
    if (!dcnt) return GSE_ERR_OOM;
    GSE_CUDA_TRY(cudaMemcpyAsync(dcnt + (size_t)rank * nranks, mine.data(), 8 * nranks,
                                 cudaMemcpyHostToDevice, setup));
    GSE_NCCL_TRY(ncclAllGather(dcnt + (size_t)rank * nranks, dcnt, nranks, ncclInt64, comm, setup));
    std::vector<int64_t> all((size_t)nranks * nranks);
    GSE_CUDA_TRY(cudaMemcpyAsync(all.data(), dcnt, 8 * all.size(), cudaMemcpyDeviceToHost, setup));
    GSE_CUDA_TRY(cudaStreamSynchronize(setup));
    dev_free(dcnt, setup);
    int64_t tot_s = 0, tot_r = 0;
    for (int p = 0; p < nranks; ++p) {
      rc[p] = all[(size_t)p * nranks + rank];
      tot_s += mine[p];
      tot_r += rc[p];
    }
    int64_t* sbuf = dev_alloc_n<int64_t>((size_t)tot_s + 1, setup);
    int64_t* rbuf = dev_alloc_n<int64_t>((size_t)tot_r + 1, setup);
    if (!sbuf || !rbuf) return GSE_ERR_OOM;
    int64_t off = 0;
    for (int p = 0; p < nranks; ++p) {
      if (mine[p])
        GSE_CUDA_TRY(cudaMemcpyAsync(sbuf + off, send[p].data(), 8 * mine[p],
                                     cudaMemcpyHostToDevice, setup));
      off += mine[p];
    }
    GSE_NCCL_TRY(ncclGroupStart());
    int64_t so = 0, ro = 0;
    for (int p = 0; p < nranks; ++p) {
      if (mine[p]) GSE_NCCL_TRY(ncclSend(sbuf + so, mine[p], ncclInt64, p, comm, setup));
      if (rc[p]) GSE_NCCL_TRY(ncclRecv(rbuf + ro, rc[p], ncclInt64, p, comm, setup));
      so += mine[p];
      ro += rc[p];
    }
    GSE_NCCL_TRY(ncclGroupEnd());
    std::vector<int64_t> flat((size_t)tot_r);
    if (tot_r)
      GSE_CUDA_TRY(cudaMemcpyAsync(flat.data(), rbuf, 8 * tot_r, cudaMemcpyDeviceToHost, setup));
    GSE_CUDA_TRY(cudaStreamSynchronize(setup));
    dev_free(sbuf, setup);
    dev_free(rbuf, setup);
    ro = 0;
    for (int p = 0; p < nranks; ++p) {
      recv[p].assign(flat.begin() + ro, flat.begin() + ro + rc[p]);
      ro += rc[p];
    }
    return GSE_OK;
  }
  gse_status exchange(const double* send_buf, const std::vector<int64_t>& send_cnt,
                      const std::vector<int64_t>& send_off, double* recv_base,
                      const std::vector<int64_t>& recv_cnt, const std::vector<int64_t>& recv_off,
                      cudaStream_t s) override {
    GSE_NCCL_TRY(ncclGroupStart());
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      if (send_cnt[p])
        GSE_NCCL_TRY(ncclSend(send_buf + send_off[p], send_cnt[p], ncclDouble, p, comm, s));
      if (recv_cnt[p])
        GSE_NCCL_TRY(ncclRecv(recv_base + recv_off[p], recv_cnt[p], ncclDouble, p, comm, s));
    }
    GSE_NCCL_TRY(ncclGroupEnd());
    return GSE_OK;
  }
};

// ---------------------------------------------------------------- thread backend
struct ThreadGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<const void*> ptr;   // per-rank published device pointers
  std::vector<cudaEvent_t> ev;    // per-rank "published data ready" events
  std::vector<cudaEvent_t> ev2;   // per-rank "done reading peers" events
  std::vector<const std::vector<int64_t>*> vec;  // per-rank host vectors (setup)
  std::vector<const std::vector<std::vector<int64_t>>*> vv;
  std::vector<int64_t> scalar;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long gen = generation;
    if (++arrived == n) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

struct RankPtrs {
  const double* p[16];
};
__global__ void k_sum_ranks(RankPtrs rp, int nranks, int count, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int r = 0; r < nranks; ++r) s += rp.p[r][i];  // rank order: deterministic
  out[i] = s;
}
struct RankPtrsU {
  const unsigned long long* p[16];
};
__global__ void k_sum_ranks_u64(RankPtrsU rp, int nranks, int count, unsigned long long* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  unsigned long long s = 0;
  for (int r = 0; r < nranks; ++r) s += rp.p[r][i];
  out[i] = s;
}

struct ThreadComm : Comm {
  ThreadGroup* g = nullptr;
  cudaEvent_t my_ev = nullptr, my_ev2 = nullptr;
  double* tmp = nullptr;
  int tmp_cap = 0;
  ~ThreadComm() override {
    if (my_ev) cudaEventDestroy(my_ev);
    if (my_ev2) cudaEventDestroy(my_ev2);
    if (tmp) cudaFree(tmp);
  }
  gse_status ensure_tmp(int count) {
    if (count <= tmp_cap) return GSE_OK;
    if (tmp) cudaFree(tmp);
    tmp_cap = count < 4096 ? 4096 : count;
    GSE_CUDA_TRY(cudaMalloc(&tmp, (size_t)tmp_cap * 8));
    return GSE_OK;
  }
  // publish `p` (device) + an event on s; after all ranks published, s waits for everyone
  void publish_and_wait(const void* p, cudaStream_t s) {
    cudaEventRecord(my_ev, s);
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->ptr[rank] = p;
      g->ev[rank] = my_ev;
    }
    g->barrier();
    for (int r = 0; r < nranks; ++r)
      if (r != rank) cudaStreamWaitEvent(s, g->ev[r], 0);
  }
  // after reading peers' data: nobody may overwrite published buffers until all are done
  void done_reading(cudaStream_t s) {
    cudaEventRecord(my_ev2, s);
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->ev2[rank] = my_ev2;
    }
    g->barrier();
    for (int r = 0; r < nranks; ++r)
      if (r != rank) cudaStreamWaitEvent(s, g->ev2[r], 0);
    g->barrier();  // ev2 slots may be reused only after every rank enqueued its waits
  }
  gse_status allreduce_sum_f64(double* d, int count, cudaStream_t s) override {
    gse_status rc = ensure_tmp(count);
    if (rc != GSE_OK) return rc;
    publish_and_wait(d, s);
    RankPtrs rp{};
    for (int r = 0; r < nranks; ++r) rp.p[r] = static_cast<const double*>(g->ptr[r]);
    k_sum_ranks<<<(count + 255) / 256, 256, 0, s>>>(rp, nranks, count, tmp);
    done_reading(s);
    GSE_CUDA_TRY(cudaMemcpyAsync(d, tmp, (size_t)count * 8, cudaMemcpyDeviceToDevice, s));
    return GSE_OK;
  }
  gse_status allreduce_sum_u64(unsigned long long* d, int count, cudaStream_t s) override {
    gse_status rc = ensure_tmp(count);
    if (rc != GSE_OK) return rc;
    publish_and_wait(d, s);
    RankPtrsU rp{};
    for (int r = 0; r < nranks; ++r) rp.p[r] = static_cast<const unsigned long long*>(g->ptr[r]);
    k_sum_ranks_u64<<<(count + 255) / 256, 256, 0, s>>>(rp, nranks, count,
                                                        reinterpret_cast<unsigned long long*>(tmp));
    done_reading(s);
    GSE_CUDA_TRY(cudaMemcpyAsync(d, tmp, (size_t)count * 8, cudaMemcpyDeviceToDevice, s));
    return GSE_OK;
  }
  gse_status host_allgather(int64_t v, std::vector<int64_t>& out) override {
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->scalar[rank] = v;
    }
    g->barrier();
    out = g->scalar;
    g->barrier();
    return GSE_OK;
  }
  gse_status host_alltoallv(const std::vector<std::vector<int64_t>>& send,
                            std::vector<std::vector<int64_t>>& recv) override {
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->vv[rank] = &send;
    }
    g->barrier();
    recv.assign(nranks, {});
    for (int p = 0; p < nranks; ++p) recv[p] = (*g->vv[p])[rank];
    g->barrier();
    return GSE_OK;
  }
  gse_status exchange(const double* send_buf, const std::vector<int64_t>& send_cnt,
                      const std::vector<int64_t>& send_off, double* recv_base,
                      const std::vector<int64_t>& recv_cnt, const std::vector<int64_t>& recv_off,
                      cudaStream_t s) override {
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->vec[rank] = &send_off;
    }
    publish_and_wait(send_buf, s);
    for (int p = 0; p < nranks; ++p) {
      if (p == rank || !recv_cnt[p]) continue;
      const double* src = static_cast<const double*>(g->ptr[p]) + (*g->vec[p])[rank];
      GSE_CUDA_TRY(cudaMemcpyAsync(recv_base + recv_off[p], src, 8 * recv_cnt[p],
                                   cudaMemcpyDeviceToDevice, s));
    }
    done_reading(s);
    return GSE_OK;
  }
};

// ---------------------------------------------------------------- distributed matrix state
struct DistCtx {
  Comm* comm = nullptr;          // not owned (owned by the gse_dist handle)
  int64_t row_begin = 0, n_local = 0, global_rows = 0, n_halo = 0;
  std::vector<int64_t> rank_rows;   // nranks + 1 row offsets
  std::vector<int64_t> send_cnt, send_off, recv_cnt, recv_off;
  int32_t* d_send_idx = nullptr;    // local indices of owned entries to send (grouped by peer)
  double* d_send_buf = nullptr;
  double* d_xext = nullptr;         // n_local + n_halo, used by gse_spmv on this matrix
  int64_t send_total = 0;
  // halo / interior overlap (row-walk matrices): rows [ov_i0, ov_i1) read owned columns only
  // and run on `side` while the halo is exchanged; the other rows follow on the caller's
  // stream.  Three partial dots (interior, top, bottom) summed in that order.
  bool overlap = false;
  int64_t ov_i0 = 0, ov_i1 = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_x = nullptr, ev_int = nullptr;
  DotOut part[3];
  double* part_buf = nullptr;
  unsigned* part_ticket = nullptr;
};

// first row / end of the longest run of rows whose columns are all owned (< n_local), given
// the ascending list of the rows that read halo columns; aligned inward to 64 rows; empty
// when shorter than max(4096, n_local / 8)
static void interior_from_halo_rows(int64_t n_local, const std::vector<uint32_t>& hrows,
                                    int64_t* i0, int64_t* i1) {
  int64_t best0 = 0, best1 = 0, prev = -1;
  for (size_t k = 0; k <= hrows.size(); ++k) {
    const int64_t r = k < hrows.size() ? (int64_t)hrows[k] : n_local;
    if (r - (prev + 1) > best1 - best0) {
      best0 = prev + 1;
      best1 = r;
    }
    prev = r;
  }
  // the end moves in by 128 rows besides the 64-row alignment: the row walk's stage
  // over-copies (and gathers, then masks) up to 8 stored entries past a group's last row,
  // which must still belong to interior rows so the interior SpMV never reads halo entries
  // of x_ext while the exchange writes them (advisor finding)
  const int64_t e = best1 > 128 ? best1 - 128 : 0;
  int64_t a = (best0 + 63) / 64 * 64, b = e / 64 * 64;
  const int64_t min_len = n_local / 8 > 4096 ? n_local / 8 : 4096;
  if (b - a < min_len) a = b = 0;
  *i0 = a;
  *i1 = b;
}

__global__ void k_add_parts(const double* a, const double* b, const double* c, int use_b,
                            int use_c, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = *a;
    if (use_b) s += *b;
    if (use_c) s += *c;
    *out = s;
  }
}

static int plan_grid(int64_t n, int dev) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms(dev) * 8;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

// ---------------------------------------------------------------- plan (device)
// The local renumbering of gse_encode_dist on the GPU (the host version build_plan_host is
// kept for gse_dist_plan and the CPU tests): a bitmap over the GLOBAL columns marks the
// non-owned columns the rank references; its set bits in ascending order ARE the sorted,
// duplicate-free halo list, and a column's halo position is the number of set bits before
// it (per-word exclusive prefix + popcount).  C5 at P = 2: 469M columns renumbered without
// leaving the device (the host loops took seconds per encode).
constexpr int PLAN_THREADS = 256, PLAN_ITEMS = 16, PLAN_TILE = PLAN_THREADS * PLAN_ITEMS;

__global__ void k_plan_mark(const int32_t* __restrict__ col, int64_t nnz, int64_t rb,
                            int64_t re, int64_t gcols, uint32_t* __restrict__ bm,
                            unsigned long long* __restrict__ bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    const int64_t c = col[i];
    if (c < 0 || c >= gcols) {
      atomicMin(bad, (unsigned long long)i);
    } else if (c < rb || c >= re) {
      const uint32_t b = 1u << (c & 31);
      if (!(bm[c >> 5] & b)) atomicOr(&bm[c >> 5], b);
    }
  }
}

__global__ void __launch_bounds__(PLAN_THREADS) k_plan_bcount(const uint32_t* __restrict__ bm,
                                                              int64_t nw,
                                                              uint32_t* __restrict__ bcnt) {
  const int64_t base = (int64_t)blockIdx.x * PLAN_TILE + (int64_t)threadIdx.x * PLAN_ITEMS;
  uint32_t c = 0;
  for (int i = 0; i < PLAN_ITEMS; ++i) c += base + i < nw ? __popc(bm[base + i]) : 0u;
  uint32_t tot;
  block_excl_scan(c, &tot);
  if (threadIdx.x == 0) bcnt[blockIdx.x] = tot;
}

// per-word exclusive prefix of the set bits, and the halo list (ascending columns)
__global__ void __launch_bounds__(PLAN_THREADS) k_plan_words(const uint32_t* __restrict__ bm,
                                                             int64_t nw,
                                                             const uint32_t* __restrict__ boff,
                                                             uint32_t* __restrict__ wpre,
                                                             int32_t* __restrict__ halo) {
  const int64_t base = (int64_t)blockIdx.x * PLAN_TILE + (int64_t)threadIdx.x * PLAN_ITEMS;
  uint32_t c = 0;
  for (int i = 0; i < PLAN_ITEMS; ++i) c += base + i < nw ? __popc(bm[base + i]) : 0u;
  uint32_t tot;
  uint32_t o = boff[blockIdx.x] + block_excl_scan(c, &tot);
  for (int i = 0; i < PLAN_ITEMS && base + i < nw; ++i) {
    uint32_t w = bm[base + i];
    wpre[base + i] = o;
    while (w) {
      const int b = __ffs(w) - 1;
      halo[o++] = (int32_t)((base + i) * 32 + b);
      w &= w - 1u;
    }
  }
}

__global__ void k_plan_renumber(const int32_t* __restrict__ col, int64_t nnz, int64_t rb,
                                int64_t re, int64_t n_local, const uint32_t* __restrict__ bm,
                                const uint32_t* __restrict__ wpre,
                                int32_t* __restrict__ local_col) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    const int64_t c = col[i];
    if (c >= rb && c < re) {
      local_col[i] = (int32_t)(c - rb);
    } else {
      const uint32_t below = bm[c >> 5] & ((1u << (c & 31)) - 1u);
      local_col[i] = (int32_t)(n_local + wpre[c >> 5] + __popc(below));
    }
  }
}

// 1 for rows that read a halo column (local id >= n_local)
template <class RP>
__global__ void k_plan_rowflag(const RP* __restrict__ rp, int64_t n_local,
                               const int32_t* __restrict__ local_col, uint8_t* __restrict__ f) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_local; r += stride) {
    uint8_t h = 0;
    for (int64_t j = rp[r]; j < rp[r + 1]; ++j)
      if (local_col[j] >= n_local) {
        h = 1;
        break;
      }
    f[r] = h;
  }
}

// a device view of a caller array (host arrays are copied; *owned is then freed by the caller)
template <class T>
static gse_status device_view(const T* p, size_t n, int dev, cudaStream_t s, const T** out,
                              void** owned) {
  *owned = nullptr;
  int d = -1;
  if (n == 0 || p == nullptr || is_device_ptr(p, &d)) {
    if (p && n && d != dev) {
      set_error("device array lives on another device than the rank's");
      return GSE_ERR_INVALID_ARG;
    }
    *out = p;
    return GSE_OK;
  }
  T* b = static_cast<T*>(dev_alloc(n * sizeof(T), s));
  if (!b) return GSE_ERR_OOM;
  GSE_CUDA_TRY(cudaMemcpyAsync(b, p, n * sizeof(T), cudaMemcpyHostToDevice, s));
  *owned = b;
  *out = b;
  return GSE_OK;
}

}  // namespace gse

struct gse_dist_s {
  gse::Comm* comm = nullptr;
};

namespace gse {

__global__ void k_pack(const double* __restrict__ x, const int32_t* __restrict__ idx, int64_t n,
                       double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = x[idx[i]];
}

// x_ext[0 .. n_local) must hold the owned entries; fills x_ext[n_local ..) from the peers
gse_status dist_halo_exchange(const Matrix& M, double* x_ext, cudaStream_t s) {
  DistCtx* D = M.dist;
  if (!D) return GSE_OK;
  if (D->send_total > 0) {
    int g = (int)std::min<int64_t>((D->send_total + 255) / 256, (int64_t)num_sms(M.device) * 4);
    k_pack<<<g, 256, 0, s>>>(x_ext, D->d_send_idx, D->send_total, D->d_send_buf);
    GSE_CUDA_TRY(cudaGetLastError());
  }
  return D->comm->exchange(D->d_send_buf, D->send_cnt, D->send_off, x_ext + D->n_local,
                           D->recv_cnt, D->recv_off, s);
}

gse_status dist_spmv(const Matrix& M, int level, double* xe, double* y, const DotOut* dot,
                     cudaStream_t s, const int* stop) {
  DistCtx* D = M.dist;
  if (!D->overlap || getenv("GSE_NO_OVERLAP")) {
    gse_status rc = dist_halo_exchange(M, xe, s);
    if (rc != GSE_OK) return rc;
    return launch_spmv(M, level, xe, y, dot, s, stop);
  }
  // interior rows on the side stream as soon as the owned entries are ready
  GSE_CUDA_TRY(cudaEventRecord(D->ev_x, s));
  GSE_CUDA_TRY(cudaStreamWaitEvent(D->side, D->ev_x, 0));
  gse_status rc = launch_spmv_rows(M, level, xe, y, dot ? &D->part[0] : nullptr, D->side, stop,
                                   D->ov_i0, D->ov_i1);
  if (rc != GSE_OK) return rc;
  GSE_CUDA_TRY(cudaEventRecord(D->ev_int, D->side));
  rc = dist_halo_exchange(M, xe, s);
  if (rc != GSE_OK) return rc;
  const int64_t n = M.rows;
  const bool top = D->ov_i0 > 0, bot = D->ov_i1 < n;
  if (top) rc = launch_spmv_rows(M, level, xe, y, dot ? &D->part[1] : nullptr, s, stop, 0, D->ov_i0);
  if (rc == GSE_OK && bot)
    rc = launch_spmv_rows(M, level, xe, y, dot ? &D->part[2] : nullptr, s, stop, D->ov_i1, n);
  if (rc != GSE_OK) return rc;
  GSE_CUDA_TRY(cudaStreamWaitEvent(s, D->ev_int, 0));
  if (dot) {  // fixed order: interior, top, bottom
    const double* a = D->part[0].result;
    const double* b = top ? D->part[1].result : D->part[2].result;
    const double* c = D->part[2].result;
    k_add_parts<<<1, 32, 0, s>>>(a, b, c, (top || bot) ? 1 : 0, (top && bot) ? 1 : 0, dot->result);
    GSE_CUDA_TRY(cudaGetLastError());
  }
  return GSE_OK;
}

bool dist_capturable(const Matrix& M) {
  static const bool off = [] {
    const char* e = getenv("GSE_DIST_NO_GRAPH");
    return e && e[0] == '1';
  }();
  return M.dist && !off && dynamic_cast<NcclComm*>(M.dist->comm) != nullptr;
}

gse_status dist_allreduce_sum(const Matrix& M, double* d_vals, int count, cudaStream_t s) {
  if (!M.dist) return GSE_OK;
  return M.dist->comm->allreduce_sum_f64(d_vals, count, s);
}

gse_status dist_allreduce_hist(const Matrix& M, unsigned long long* d, int count, cudaStream_t s) {
  if (!M.dist) return GSE_OK;
  return M.dist->comm->allreduce_sum_u64(d, count, s);
}

void free_dist(Matrix& M) {
  DistCtx* D = M.dist;
  if (!D) return;
  dev_free(D->d_send_idx, nullptr);
  dev_free(D->d_send_buf, nullptr);
  dev_free(D->d_xext, nullptr);
  if (D->side) {
    cudaStreamSynchronize(D->side);
    cudaStreamDestroy(D->side);
  }
  if (D->ev_x) cudaEventDestroy(D->ev_x);
  if (D->ev_int) cudaEventDestroy(D->ev_int);
  if (D->part_buf) dev_free(D->part_buf, nullptr);
  if (D->part_ticket) dev_free(D->part_ticket, nullptr);
  delete D;
  M.dist = nullptr;
}

int64_t dist_ext_cols(const Matrix& M) { return M.dist ? M.dist->n_local + M.dist->n_halo : M.cols; }

// ---------------------------------------------------------------- plan (host, setup time)
// Local renumbering of one rank's column ids (see the file comment).  Returns the sorted
// halo list and the local column array.  Pure host code (also exported for CPU tests).
gse_status build_plan_host(int64_t nnz, const int32_t* col, int64_t row_begin, int64_t n_local,
                           int nranks, const int64_t* rank_rows, int32_t* local_col,
                           std::vector<int64_t>& halo, std::vector<int64_t>& recv_cnt) {
  const int64_t row_end = row_begin + n_local;
  halo.clear();
  for (int64_t i = 0; i < nnz; ++i) {
    const int64_t c = col[i];
    if (c < row_begin || c >= row_end) halo.push_back(c);
  }
  std::sort(halo.begin(), halo.end());
  halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
  if ((int64_t)halo.size() + n_local >= (1LL << 31)) {
    set_error("local column space exceeds 2^31");
    return GSE_ERR_INVALID_ARG;
  }
  for (int64_t i = 0; i < nnz; ++i) {
    const int64_t c = col[i];
    if (c >= row_begin && c < row_end) {
      local_col[i] = (int32_t)(c - row_begin);
    } else {
      const int64_t pos = std::lower_bound(halo.begin(), halo.end(), c) - halo.begin();
      local_col[i] = (int32_t)(n_local + pos);
    }
  }
  recv_cnt.assign(nranks, 0);
  int owner = 0;
  for (int64_t c : halo) {
    while (owner < nranks - 1 && c >= rank_rows[owner + 1]) ++owner;
    recv_cnt[owner]++;
  }
  return GSE_OK;
}

gse_status comm_allreduce_u64(Comm* c, unsigned long long* d, int count, cudaStream_t s) {
  return c ? c->allreduce_sum_u64(d, count, s) : GSE_OK;
}

gse_status comm_any(Comm* c, int local_flag, int* any) {
  *any = local_flag;
  if (!c) return GSE_OK;
  std::vector<int64_t> all;
  gse_status st = c->host_allgather(local_flag, all);
  if (st != GSE_OK) return st;
  for (int64_t v : all) *any |= (v != 0);
  return GSE_OK;
}

double* dist_xext(const Matrix& M) { return M.dist ? M.dist->d_xext : nullptr; }
int64_t dist_n_local(const Matrix& M) { return M.dist ? M.dist->n_local : M.rows; }

}  // namespace gse

using namespace gse;

extern "C" {

gse_status gse_nccl_unique_id(void* id128) {
  if (!id128) {
    set_error("id buffer is NULL");
    return GSE_ERR_INVALID_ARG;
  }
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_status(r, "ncclGetUniqueId");
  memcpy(id128, &id, sizeof(id) < 128 ? sizeof(id) : 128);
  return GSE_OK;
}

gse_status gse_dist_create(const void* nccl_unique_id, int rank, int nranks, int device,
                           gse_dist* out) {
  if (!out || !nccl_unique_id || nranks < 1 || rank < 0 || rank >= nranks || nranks > 16) {
    set_error("invalid dist arguments (nranks in [1, 16])");
    return GSE_ERR_INVALID_ARG;
  }
  *out = nullptr;
  cudaSetDevice(device);
  NcclComm* c = new NcclComm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_status(r, "ncclCommInitRank");
  }
  cudaStreamCreateWithFlags(&c->setup, cudaStreamNonBlocking);
  gse_dist d = new gse_dist_s();
  d->comm = c;
  *out = d;
  return GSE_OK;
}

gse_status gse_dist_thread_group_create(int nranks, void** group) {
  if (!group || nranks < 1 || nranks > 16) {
    set_error("nranks must be in [1, 16]");
    return GSE_ERR_INVALID_ARG;
  }
  ThreadGroup* g = new ThreadGroup();
  g->n = nranks;
  g->ptr.assign(nranks, nullptr);
  g->ev.assign(nranks, nullptr);
  g->ev2.assign(nranks, nullptr);
  g->vec.assign(nranks, nullptr);
  g->vv.assign(nranks, nullptr);
  g->scalar.assign(nranks, 0);
  *group = g;
  return GSE_OK;
}

void gse_dist_thread_group_free(void* group) { delete static_cast<ThreadGroup*>(group); }

gse_status gse_dist_create_thread(void* group, int rank, int device, gse_dist* out) {
  ThreadGroup* g = static_cast<ThreadGroup*>(group);
  if (!out || !g || rank < 0 || rank >= g->n) {
    set_error("invalid thread-group rank");
    return GSE_ERR_INVALID_ARG;
  }
  cudaSetDevice(device);
  ThreadComm* c = new ThreadComm();
  c->g = g;
  c->rank = rank;
  c->nranks = g->n;
  c->device = device;
  if (cudaEventCreateWithFlags(&c->my_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->my_ev2, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return cuda_status(cudaGetLastError(), "cudaEventCreate");
  }
  gse_dist d = new gse_dist_s();
  d->comm = c;
  *out = d;
  return GSE_OK;
}

void gse_dist_free(gse_dist D) {
  if (!D) return;
  delete D->comm;
  delete D;
}

gse_status gse_dist_plan(int64_t nnz, const int32_t* col, int64_t row_begin, int64_t n_local,
                         int nranks, const int64_t* rank_rows, int32_t* local_col,
                         int64_t* n_halo, int64_t* halo_cols, int64_t* recv_count) {
  if (nnz < 0 || (nnz > 0 && (!col || !local_col)) || !rank_rows || !n_halo || nranks < 1) {
    set_error("invalid plan arguments");
    return GSE_ERR_INVALID_ARG;
  }
  std::vector<int64_t> halo, rc;
  gse_status st =
      build_plan_host(nnz, col, row_begin, n_local, nranks, rank_rows, local_col, halo, rc);
  if (st != GSE_OK) return st;
  *n_halo = (int64_t)halo.size();
  if (halo_cols) std::copy(halo.begin(), halo.end(), halo_cols);
  if (recv_count) std::copy(rc.begin(), rc.end(), recv_count);
  return GSE_OK;
}

gse_status gse_encode_dist(gse_dist Dh, const gse_csr_f64* A, int64_t row_begin,
                           int64_t global_rows, const gse_encode_opts* opts, gse_matrix* out,
                           void* stream) {
  if (opts && opts->sample_block_rows != 0) {  // (checked before any collective)
    set_error("sampled tables (sample_block_rows > 0) are single-GPU only");
    return GSE_ERR_INVALID_ARG;
  }
  if (!Dh || !A || !out) {
    set_error("NULL argument");
    return GSE_ERR_INVALID_ARG;
  }
  *out = nullptr;
  Comm* comm = Dh->comm;
  cudaSetDevice(comm->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n_local = A->rows;
  if (row_begin < 0 || row_begin + n_local > global_rows || A->cols != global_rows) {
    set_error("rank rows must lie in [0, global_rows) and cols == global_rows (square)");
    return GSE_ERR_DIM_MISMATCH;
  }
  // row partition of all ranks (contiguous, in rank order)
  std::vector<int64_t> begins, counts;
  gse_status st = comm->host_allgather(row_begin, begins);
  if (st == GSE_OK) st = comm->host_allgather(n_local, counts);
  if (st != GSE_OK) return st;
  std::vector<int64_t> rank_rows(comm->nranks + 1, 0);
  for (int r = 0; r < comm->nranks; ++r) {
    if (begins[r] != rank_rows[r]) {
      set_error("ranks must own contiguous row blocks in rank order");
      return GSE_ERR_INVALID_ARG;
    }
    rank_rows[r + 1] = begins[r] + counts[r];
  }
  if (rank_rows[comm->nranks] != global_rows) {
    set_error("row blocks do not cover [0, global_rows)");
    return GSE_ERR_DIM_MISMATCH;
  }
  // local renumbering + halo plan on the device (k_plan_*); only the halo list comes back
  const int32_t* dcol = nullptr;
  void* col_owned = nullptr;
  st = device_view(A->col_idx, (size_t)A->nnz, comm->device, s, &dcol, &col_owned);
  if (st != GSE_OK) return st;
  const int64_t nw = (global_rows + 31) / 32 + 1;
  const int64_t nbw = (nw + PLAN_TILE - 1) / PLAN_TILE;
  uint32_t* bm = dev_alloc_n<uint32_t>((size_t)nw, s);
  uint32_t* wpre = dev_alloc_n<uint32_t>((size_t)nw, s);
  uint32_t* bcnt = dev_alloc_n<uint32_t>((size_t)nbw + 1, s);
  unsigned long long* dbad = dev_alloc_n<unsigned long long>(1, s);
  int* dnh = dev_alloc_n<int>(1, s);
  int32_t* d_local_col = dev_alloc_n<int32_t>((size_t)A->nnz + 1, s);
  if (!bm || !wpre || !bcnt || !dbad || !dnh || !d_local_col) return GSE_ERR_OOM;
  GSE_CUDA_TRY(cudaMemsetAsync(bm, 0, 4 * (size_t)nw, s));
  GSE_CUDA_TRY(cudaMemsetAsync(dbad, 0xFF, 8, s));
  const int gsz = plan_grid(A->nnz, comm->device);
  if (A->nnz)
    k_plan_mark<<<gsz, 256, 0, s>>>(dcol, A->nnz, row_begin, row_begin + n_local, global_rows, bm,
                                    dbad);
  k_plan_bcount<<<(unsigned)nbw, PLAN_THREADS, 0, s>>>(bm, nw, bcnt);
  k_cmp_scan<<<1, 1024, 0, s>>>(bcnt, nbw, dnh);
  int nh_bad[3] = {0, 0, 0};
  unsigned long long badi = 0;
  GSE_CUDA_TRY(cudaMemcpyAsync(&nh_bad[0], dnh, sizeof(int), cudaMemcpyDeviceToHost, s));
  GSE_CUDA_TRY(cudaMemcpyAsync(&badi, dbad, 8, cudaMemcpyDeviceToHost, s));
  GSE_CUDA_TRY(cudaStreamSynchronize(s));
  if (badi != ~0ull) {
    set_error("column index out of range at non-zero " + std::to_string(badi));
    return GSE_ERR_INVALID_ARG;
  }
  const int64_t n_halo = nh_bad[0];
  if (n_halo + n_local >= (1LL << 31)) {
    set_error("local column space exceeds 2^31");
    return GSE_ERR_INVALID_ARG;
  }
  int32_t* d_halo = dev_alloc_n<int32_t>((size_t)n_halo + 1, s);
  if (!d_halo) return GSE_ERR_OOM;
  k_plan_words<<<(unsigned)nbw, PLAN_THREADS, 0, s>>>(bm, nw, bcnt, wpre, d_halo);
  if (A->nnz)
    k_plan_renumber<<<gsz, 256, 0, s>>>(dcol, A->nnz, row_begin, row_begin + n_local, n_local, bm,
                                        wpre, d_local_col);
  GSE_CUDA_TRY(cudaGetLastError());
  std::vector<int32_t> halo32((size_t)n_halo);
  if (n_halo)
    GSE_CUDA_TRY(cudaMemcpyAsync(halo32.data(), d_halo, 4 * (size_t)n_halo, cudaMemcpyDeviceToHost, s));
  GSE_CUDA_TRY(cudaStreamSynchronize(s));
  for (void* q : {(void*)bm, (void*)wpre, (void*)bcnt, (void*)dbad, (void*)d_halo}) dev_free(q, s);
  std::vector<int64_t> halo(halo32.begin(), halo32.end()), recv_cnt(comm->nranks, 0);
  {
    int owner = 0;
    for (int64_t c : halo) {
      while (owner < comm->nranks - 1 && c >= rank_rows[owner + 1]) ++owner;
      recv_cnt[owner]++;
    }
  }
  // tell every owner which of its entries this rank needs
  std::vector<std::vector<int64_t>> want(comm->nranks), give;
  {
    size_t o = 0;
    for (int p = 0; p < comm->nranks; ++p) {
      want[p].assign(halo.begin() + o, halo.begin() + o + recv_cnt[p]);
      o += recv_cnt[p];
    }
  }
  st = comm->host_alltoallv(want, give);
  if (st != GSE_OK) return st;
  // encode the local rows with local column ids and the GLOBAL table
  gse_csr_f64 L = *A;
  L.cols = n_local + (int64_t)halo.size();
  gse_encode_opts o = {8, comm->device, 0, 0, 0};
  if (opts) o = *opts;
  o.device = comm->device;
  Matrix* M = nullptr;
  st = create_from_csr(&L, GSE_KIND_GSE, o.k_max, o.device, out, s, &M, comm, d_local_col,
                       0, 0, o.per_shard_table ? 1 : 0);
  if (st != GSE_OK) return st;
  DistCtx* D = new DistCtx();
  D->comm = comm;
  D->row_begin = row_begin;
  D->n_local = n_local;
  D->global_rows = global_rows;
  D->n_halo = (int64_t)halo.size();
  D->rank_rows = rank_rows;
  D->recv_cnt = recv_cnt;
  D->recv_off.assign(comm->nranks, 0);
  D->send_cnt.assign(comm->nranks, 0);
  D->send_off.assign(comm->nranks, 0);
  int64_t ro = 0, so = 0;
  std::vector<int32_t> send_idx;
  for (int p = 0; p < comm->nranks; ++p) {
    D->recv_off[p] = ro;
    ro += recv_cnt[p];
    D->send_off[p] = so;
    D->send_cnt[p] = (int64_t)give[p].size();
    so += D->send_cnt[p];
    for (int64_t c : give[p]) send_idx.push_back((int32_t)(c - row_begin));
  }
  D->send_total = so;
  D->d_send_idx = dev_alloc_n<int32_t>((size_t)so + 1, s);
  D->d_send_buf = dev_alloc_n<double>((size_t)so + 1, s);
  D->d_xext = dev_alloc_n<double>((size_t)(n_local + D->n_halo) + 1, s);
  if (!D->d_send_idx || !D->d_send_buf || !D->d_xext) {
    delete D;
    gse_matrix_free(*out);
    *out = nullptr;
    return GSE_ERR_OOM;
  }
  // x_ext starts zeroed: no SpMV ever reads pool garbage
  GSE_CUDA_TRY(cudaMemsetAsync(D->d_xext, 0, sizeof(double) * ((size_t)(n_local + D->n_halo) + 1), s));
  if (so)
    GSE_CUDA_TRY(cudaMemcpyAsync(D->d_send_idx, send_idx.data(), 4 * so, cudaMemcpyHostToDevice, s));
  M->dist = D;
  // halo / interior overlap for row-walk matrices (local decision: every rank issues the
  // same collectives either way)
  if (M->spmv_mode == SPMV_RW && n_local > 0 && !getenv("GSE_NO_OVERLAP")) {
    // rows reading halo columns, compacted on the device; the longest run between them is
    // the interior (host, on the short list)
    const void* drp = nullptr;
    void* rp_owned = nullptr;
    if (A->row_ptr_64)
      st = device_view((const long long*)A->row_ptr, (size_t)n_local + 1, comm->device, s,
                       (const long long**)&drp, &rp_owned);
    else
      st = device_view((const int*)A->row_ptr, (size_t)n_local + 1, comm->device, s,
                       (const int**)&drp, &rp_owned);
    if (st != GSE_OK) return st;
    uint8_t* rf = dev_alloc_n<uint8_t>((size_t)n_local, s);
    uint32_t* hr = dev_alloc_n<uint32_t>((size_t)n_local + 1, s);
    int* dcnt = dev_alloc_n<int>(1, s);
    if (!rf || !hr || !dcnt) return GSE_ERR_OOM;
    const int gr = plan_grid(n_local, comm->device);
    if (A->row_ptr_64)
      k_plan_rowflag<<<gr, 256, 0, s>>>((const long long*)drp, n_local, d_local_col, rf);
    else
      k_plan_rowflag<<<gr, 256, 0, s>>>((const int*)drp, n_local, d_local_col, rf);
    GSE_CUDA_TRY(cudaGetLastError());
    st = compact_flags(rf, n_local, hr, dcnt, s);
    if (st != GSE_OK) return st;
    int nhr = 0;
    GSE_CUDA_TRY(cudaMemcpyAsync(&nhr, dcnt, sizeof(int), cudaMemcpyDeviceToHost, s));
    GSE_CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<uint32_t> hrows((size_t)nhr);
    if (nhr)
      GSE_CUDA_TRY(cudaMemcpyAsync(hrows.data(), hr, 4 * (size_t)nhr, cudaMemcpyDeviceToHost, s));
    GSE_CUDA_TRY(cudaStreamSynchronize(s));
    for (void* q : {(void*)rf, (void*)hr, (void*)dcnt, rp_owned}) dev_free(q, s);
    interior_from_halo_rows(n_local, hrows, &D->ov_i0, &D->ov_i1);
    if (D->ov_i1 > D->ov_i0) {
      const int np = 2048;  // partials per part (>= any persistent SpMV grid)
      D->part_buf = dev_alloc_n<double>((size_t)3 * (np + 1), s);
      D->part_ticket = dev_alloc_n<unsigned>(4, s);
      if (!D->part_buf || !D->part_ticket) return GSE_ERR_OOM;
      GSE_CUDA_TRY(cudaMemsetAsync(D->part_ticket, 0, 16, s));
      GSE_CUDA_TRY(cudaMemsetAsync(D->part_buf, 0, 8 * (size_t)3 * (np + 1), s));
      for (int k = 0; k < 3; ++k) {
        D->part[k].partials = D->part_buf + (size_t)k * (np + 1);
        D->part[k].result = D->part_buf + (size_t)k * (np + 1) + np;
        D->part[k].ticket = D->part_ticket + k;
      }
      GSE_CUDA_TRY(cudaStreamCreateWithFlags(&D->side, cudaStreamNonBlocking));
      GSE_CUDA_TRY(cudaEventCreateWithFlags(&D->ev_x, cudaEventDisableTiming));
      GSE_CUDA_TRY(cudaEventCreateWithFlags(&D->ev_int, cudaEventDisableTiming));
      D->overlap = true;
    }
  }
  GSE_CUDA_TRY(cudaStreamSynchronize(s));
  dev_free(d_local_col, s);
  dev_free(col_owned, s);
  GSE_CUDA_TRY(cudaStreamSynchronize(s));
  return GSE_OK;
}

}  // extern "C"
