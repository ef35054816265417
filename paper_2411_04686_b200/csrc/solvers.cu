// solvers.cu -- stepped mixed-precision CG and GMRES(m) on the GPU.
//
// Paper: Alg. stepped-GMRES: w_j = A_tag v_j, tag raised when the residual
// monitor (Eqs. 3-6, Conditions 1-3) asks for more precision; CG / GMRES(30)
// settings of P:299.  The paper's vector ops were cuBLAS calls -- prior art.
//
// B200 design:
//  * every iteration is a fixed sequence of fused kernels with deterministic last-block
//    reductions -- CG: [spmv + p.q] -> [x += a p, r -= a q, r.r, monitor] -> [p = r + b p];
//    GMRES inner step j: [spmv] -> (j+1) x [w -= h v_{i-1}, w.v_i] -> [w -= h v_j, ||w||,
//    Givens, monitor] -> [v_{j+1} = w / h];
//  * the residual monitor (ring of t+1 residuals, RSD / nDec / relDec, Conditions 1-3)
//    runs on the device in the last CTA of the update kernel: no host round trip per
//    iteration;
//  * CG iterations run inside a CUDA-graph WHILE node: the update kernel clears the
//    condition (cudaGraphSetConditional) when an event occurs (converged recurrence,
//    escalation request, breakdown, max iterations).  GMRES runs one graph per restart
//    cycle (kernels early-exit once the cycle is stopped).  The host only handles events:
//    level switch with residual replacement (R15), verification with A_3 (R16).
#include <cooperative_groups.h>

#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "gse_internal.cuh"
#include "vec16.cuh"

namespace gse {

enum Event : int {
  EV_NONE = 0,
  EV_CONVERGED = 1,   // recurrence / estimate <= tol
  EV_ESCALATE = 2,    // monitor asks for a higher level
  EV_ABORT = 3,       // breakdown / non-finite
  EV_MAXITER = 4,     // iteration budget exhausted
  EV_EXPLICIT_OK = 5  // GMRES restart: explicit residual <= tol
};

constexpr int MAX_RESTART = 64;

struct SolveCtrl {
  double bnorm, tol;
  double rr, rr_new, pq, beta, resid;
  double dot;  // scratch reduction target
  double rr_part;  // distributed CG: this rank's r.r partial (allreduced before k_cg_events)
  double alpha;    // CG: step of the current iteration, applied to x by k_cg_xpay (0: none)
  double perturb_c, eta[2];  // R29 trigger: c and ||A_3 - A_L||_inf (L = 1, 2); c = 0: off
  double xx;       // R29: ||x||^2 of the latest iterate (CG: after the previous iteration's
                   // x update; GMRES: at the start of the cycle)
  int upd_ok;
  long long iter, max_iters;
  int level, event, stop, stepped, max_level;
  long long l, t, m, ndec_limit;
  double rsd_limit, reldec_limit, floor_[2];
  long long ring_count, ring_head;
  // GMRES
  int restart, k;
  double hn;
  double H[(MAX_RESTART + 1) * MAX_RESTART];
  double cs[MAX_RESTART], sn[MAX_RESTART], g[MAX_RESTART + 1], y[MAX_RESTART];
};

struct SolverWs {
  int64_t n = 0;
  int vgrid = 0;
  double *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr, *b = nullptr, *tmp = nullptr;
  double* V = nullptr;  // GMRES basis (restart + 1) x n
  int V_cols = 0;
  // 16-bit Krylov basis (NEXT-4): words, per-vector tables, histogram, decoded current vector
  uint16_t* V16 = nullptr;
  int V16_cols = 0;
  uint16_t* vtab = nullptr;  // [V16_cols][V16_KMAX]
  int* vlen = nullptr;       // [V16_cols]
  unsigned* vhist = nullptr; // [2048]
  unsigned* vhist2 = nullptr; // [2][2048] (cooperative 16-bit Arnoldi)
  double* vcur = nullptr;    // [n]
  int gm_k16 = 0;            // basis format the GMRES graphs were built for
  double* partials = nullptr;
  unsigned* ticket = nullptr;
  SolveCtrl* ctrl = nullptr;
  double* ring = nullptr;
  int64_t ring_cap = 0;
  SolveCtrl* hctrl = nullptr;  // pinned host mirror
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t cg_exec[3] = {nullptr, nullptr, nullptr};
  cudaGraph_t cg_graph[3] = {nullptr, nullptr, nullptr};
  cudaGraphExec_t gm_exec[3] = {nullptr, nullptr, nullptr};
  // distributed CG (NCCL backend): one captured batch of DIST_BATCH iterations per level
  cudaGraphExec_t dcg_exec[3] = {nullptr, nullptr, nullptr};
  cudaGraph_t dcg_graph[3] = {nullptr, nullptr, nullptr};
  // distributed GMRES (NCCL backend): one captured restart cycle per level
  cudaGraphExec_t dgm_exec[3] = {nullptr, nullptr, nullptr};
  cudaGraph_t dgm_graph[3] = {nullptr, nullptr, nullptr};
  int dgm_restart = 0;
  cudaGraph_t gm_graph[3] = {nullptr, nullptr, nullptr};
  int gm_restart = 0;
  int cg_xx = 0;  // the CG graphs compute ||x||^2 in k_cg_xpay (R29 trigger on)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

// The scalar head of SolveCtrl (everything before the GMRES arrays H, cs, sn, g, y).  The single thread
// that runs the CG event logic works on a shared-memory snapshot loaded by warp 0 at
// kernel start (overlapped with the vector pass) and writes it back: done directly on
// global memory the logic is a chain of ~20 dependent L2 round trips (~7 us per iteration).
constexpr int CTRL_HEAD_WORDS = (int)(offsetof(SolveCtrl, H) / 8);
static_assert(offsetof(SolveCtrl, H) % 8 == 0, "SolveCtrl head must be 8-byte words");

__device__ __forceinline__ void ctrl_load_head(const SolveCtrl* c, unsigned long long* sm) {
  if (threadIdx.x < 32) {
    const unsigned long long* g = reinterpret_cast<const unsigned long long*>(c);
    for (int i = threadIdx.x; i < CTRL_HEAD_WORDS; i += 32) sm[i] = __ldcg(g + i);
  }
}
__device__ __forceinline__ void ctrl_store_head(SolveCtrl* c, const unsigned long long* sm) {
  unsigned long long* g = reinterpret_cast<unsigned long long*>(c);
  for (int i = 0; i < CTRL_HEAD_WORDS; ++i) g[i] = sm[i];
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
  return v;
}

__device__ double block_sum_d(double v) {
  __shared__ double red[32];
  v = warp_sum_d(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    red[0] = s;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

// returns true in (all threads of) the last CTA; *total = deterministic grid sum
__device__ bool grid_sum(double part, double* partials, unsigned* ticket, double* total) {
  __shared__ unsigned s_last;
  __shared__ double s_tot;
  const double bs = block_sum_d(part);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bs;
    __threadfence();
    s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  double acc = 0.0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) acc += __ldcg(partials + i);
  const double tot = block_sum_d(acc);
  if (threadIdx.x == 0) {
    s_tot = tot;
    *ticket = 0u;
  }
  __syncthreads();
  *total = s_tot;
  return true;
}

#define GRID_LOOP(i, n) \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------- residual monitor
// Mirrors the oracle's order of operations (ring push, RSD Eq. 3, nDec Eqs. 4-5, relDec
// Eq. 6, Conditions 1-3 with nDec_limit (R13), optional floors (R17)).
__device__ void ring_push(SolveCtrl* c, double* ring, double v) {
  const long long cap = c->t + 1;
  if (!c->stepped || cap <= 0) return;
  if (c->ring_count < cap) {
    ring[(c->ring_head + c->ring_count) % cap] = v;
    c->ring_count++;
  } else {
    ring[c->ring_head] = v;
    c->ring_head = (c->ring_head + 1) % cap;
  }
}

__device__ int monitor_check(const SolveCtrl* c, const double* ring, long long j, double resid) {
  if (!c->stepped || c->level >= c->max_level) return 0;
  if (c->level <= 2 && c->floor_[c->level - 1] > 0.0 && resid < c->floor_[c->level - 1]) return 1;
  // R29: the level's attainable-accuracy floor c eta_L ||x|| / ||b|| (oracle's operation order)
  if (c->level <= 2 && c->perturb_c > 0.0 && c->xx > 0.0) {
    double thr = __dmul_rn(c->perturb_c, c->eta[c->level - 1]);
    thr = __dmul_rn(thr, sqrt(c->xx));
    thr = thr / c->bnorm;
    if (resid <= thr) return 1;
  }
  const long long t = c->t, cap = t + 1;
  if (j < c->l || ((j - c->l) % c->m) != 0 || c->ring_count < cap) return 0;
  auto w = [&](long long i) { return ring[(c->ring_head + i) % cap]; };
  if (!(w(0) > 0.0)) return 0;
  double sum = 0.0;
  for (long long i = 0; i < t; ++i) sum = __dadd_rn(sum, w(i));
  const double avg = sum / (double)t;
  double rsd = 0.0;
  if (!(avg < 1e-300)) {
    double ss = 0.0;
    for (long long i = 0; i < t; ++i) {
      const double dv = __dsub_rn(w(i), avg);
      ss = __dadd_rn(ss, __dmul_rn(dv, dv));
    }
    rsd = sqrt(ss / (double)t) / avg;
  }
  long long nd = 0;
  for (long long i = 0; i < t; ++i) nd += (w(i) > w(i + 1)) ? 1 : 0;
  const double rd = (w(0) - w(t - 1)) / w(0);
  const int c1 = (rsd > c->rsd_limit) && (nd < c->ndec_limit);
  const int c2 = (nd >= c->ndec_limit) && (rd < c->reldec_limit);
  const int c3 = (nd == 0);
  return c1 || c2 || c3;
}

// ---------------------------------------------------------------- generic vector kernels
// tot = a . b  (into *out)
__global__ void __launch_bounds__(256, 4) k_dot(const double* __restrict__ a,
                                             const double* __restrict__ b, int64_t n,
                                             double* partials, unsigned* ticket, double* out) {
  pdl_wait();
  pdl_trigger();
  double acc = 0.0;
  GRID_LOOP(i, n) acc = __dadd_rn(acc, __dmul_rn(a[i], b[i]));
  double tot;
  if (grid_sum(acc, partials, ticket, &tot) && threadIdx.x == 0) *out = tot;
}

// r = b - Ax ; (optionally p = r) ; *out = r.r
__global__ void __launch_bounds__(256, 4) k_residual(const double* __restrict__ b,
                                                  const double* Ax,  // may alias r
                                                  double* r, double* __restrict__ p,
                                                  int64_t n, double* partials, unsigned* ticket,
                                                  double* out) {
  pdl_wait();
  pdl_trigger();
  double acc = 0.0;
  GRID_LOOP(i, n) {
    const double v = __dsub_rn(b[i], Ax[i]);
    r[i] = v;
    if (p) p[i] = v;
    acc = __dadd_rn(acc, __dmul_rn(v, v));
  }
  double tot;
  if (grid_sum(acc, partials, ticket, &tot) && threadIdx.x == 0) *out = tot;
}

// ---------------------------------------------------------------- CG kernels
// residual, monitor and events after CG iteration j (one thread)
__device__ void cg_events(SolveCtrl* c, double* ring, double tot, bool ok,
                          cudaGraphConditionalHandle handle, int in_graph) {
  const double rr = c->rr;
  const long long j = c->iter + 1;
  c->iter = j;
  int ev = EV_NONE;
  if (!ok) {
    ev = EV_ABORT;
  } else {
    const double resid = sqrt(tot) / c->bnorm;
    c->resid = resid;
    c->rr_new = tot;
    if (!isfinite(resid)) {
      ev = EV_ABORT;
    } else {
      ring_push(c, ring, resid);
      if (resid <= c->tol)
        ev = EV_CONVERGED;
      else if (monitor_check(c, ring, j, resid))
        ev = EV_ESCALATE;
      else if (j >= c->max_iters)
        ev = EV_MAXITER;
    }
  }
  c->event = ev;
  if (ev != EV_NONE) {
    if (in_graph) cudaGraphSetConditional(handle, 0u);
  } else {
    c->beta = tot / rr;
    c->rr = tot;
  }
}

// pairs in flight per thread in k_cg_update (A/B knob)
#ifndef GSE_UPD_K
#define GSE_UPD_K 1
#endif
constexpr int UPD_K = GSE_UPD_K;
#ifndef GSE_XPAY_K
#define GSE_XPAY_K 1
#endif
constexpr int XPAY_K = GSE_XPAY_K;

// r -= alpha q ; rr_new = r.r ; monitor ; events.  x += alpha p is deferred to k_cg_xpay,
// which reads p anyway (same arithmetic, one vector pass less per iteration); alpha is
// handed over in c->alpha (0 when this iteration did not update).
__global__ void __launch_bounds__(256, 4) k_cg_update(SolveCtrl* __restrict__ c, double* ring,
                                                   double* __restrict__ r,
                                                   const double* __restrict__ q, int64_t n,
                                                   double* partials, unsigned* ticket,
                                                   cudaGraphConditionalHandle handle,
                                                   int in_graph, int defer) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned long long sctrl[CTRL_HEAD_WORDS];
  if (c->event != EV_NONE) {  // host-driven mode: iterations after an event are no-ops
    if (blockIdx.x == 0 && threadIdx.x == 0) c->alpha = 0.0;
    return;
  }
  ctrl_load_head(c, sctrl);  // consumed only by the last CTA, after grid_sum's barriers
  const double pq = c->pq, rr = c->rr;
  const bool ok = (pq > 0.0) && isfinite(pq);
  const double alpha = rr / pq;
  double acc = 0.0;
  if (ok) {
    // 16-byte accesses (pairs of elements), 4 pairs in flight per thread; the element
    // order of each thread (and so its reduction order) is fixed by the grid
    const int64_t n2 = n >> 1;
    const double2* __restrict__ q2 = reinterpret_cast<const double2*>(q);
    double2* __restrict__ r2 = reinterpret_cast<double2*>(r);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += UPD_K * stride) {
      double2 rv[UPD_K], qv[UPD_K];
#pragma unroll
      for (int k = 0; k < UPD_K; ++k) {
        const int64_t j = i + k * stride;
        if (j < n2) {
          rv[k] = r2[j];
          qv[k] = q2[j];
        }
      }
#pragma unroll
      for (int k = 0; k < UPD_K; ++k) {
        const int64_t j = i + k * stride;
        if (j < n2) {
          double2 ro;
          ro.x = __dsub_rn(rv[k].x, __dmul_rn(alpha, qv[k].x));
          ro.y = __dsub_rn(rv[k].y, __dmul_rn(alpha, qv[k].y));
          r2[j] = ro;
          acc = __dadd_rn(acc, __dmul_rn(ro.x, ro.x));
          acc = __dadd_rn(acc, __dmul_rn(ro.y, ro.y));
        }
      }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd tail element
      const int64_t j = n - 1;
      const double ri = __dsub_rn(r[j], __dmul_rn(alpha, q[j]));
      r[j] = ri;
      acc = __dadd_rn(acc, __dmul_rn(ri, ri));
    }
  }
  double tot;
  if (grid_sum(acc, partials, ticket, &tot) && threadIdx.x == 0) {
    SolveCtrl* sc = reinterpret_cast<SolveCtrl*>(sctrl);
    sc->alpha = ok ? alpha : 0.0;
    if (defer) {  // distributed: r.r is this rank's partial; k_cg_events runs after the allreduce
      sc->rr_part = tot;
      sc->upd_ok = ok ? 1 : 0;
    } else {
      cg_events(sc, ring, tot, ok, handle, in_graph);
    }
    ctrl_store_head(c, sctrl);
  }
}

// distributed CG: the event logic on the allreduced r.r (all ranks decide identically)
__global__ void k_cg_events(SolveCtrl* __restrict__ c, double* ring) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0 || blockIdx.x != 0 || c->event != EV_NONE) return;
  cg_events(c, ring, c->rr_part, c->upd_ok != 0, 0, 0);
}

// x += alpha p (the update deferred by k_cg_update) ; p = r + beta p (skipped when an event
// is pending: the host restarts / stops).  Both read the old p.  XX (R29 trigger on): also
// ||x_new||^2 -> c->xx (deterministic grid sum; x unchanged -> xx kept).
template <bool XX>
__global__ void __launch_bounds__(256, 4) k_cg_xpay(SolveCtrl* __restrict__ c,
                                                 double* __restrict__ x, double* __restrict__ p,
                                                 const double* __restrict__ r, int64_t n,
                                                 double* partials, unsigned* ticket) {
  pdl_wait();
  pdl_trigger();
  const double alpha = c->alpha, beta = c->beta;
  const bool do_x = alpha != 0.0, do_p = c->event == EV_NONE;
  if (!do_x && !do_p) return;
  double acc = 0.0;
  const int64_t n2 = n >> 1;
  double2* __restrict__ x2 = reinterpret_cast<double2*>(x);
  double2* __restrict__ p2 = reinterpret_cast<double2*>(p);
  const double2* __restrict__ r2 = reinterpret_cast<const double2*>(r);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += XPAY_K * stride) {
    double2 pv[XPAY_K], rv[XPAY_K], xv[XPAY_K];
#pragma unroll
    for (int k = 0; k < XPAY_K; ++k) {
      const int64_t j = i + k * stride;
      if (j < n2) {
        pv[k] = p2[j];
        if (do_p) rv[k] = r2[j];
        if (do_x) xv[k] = x2[j];
      }
    }
#pragma unroll
    for (int k = 0; k < XPAY_K; ++k) {
      const int64_t j = i + k * stride;
      if (j < n2) {
        if (do_x) {
          double2 o;
          o.x = __dadd_rn(xv[k].x, __dmul_rn(alpha, pv[k].x));
          o.y = __dadd_rn(xv[k].y, __dmul_rn(alpha, pv[k].y));
          x2[j] = o;
          if constexpr (XX) {
            acc = __dadd_rn(acc, __dmul_rn(o.x, o.x));
            acc = __dadd_rn(acc, __dmul_rn(o.y, o.y));
          }
        }
        if (do_p) {
          double2 o;
          o.x = __dadd_rn(rv[k].x, __dmul_rn(beta, pv[k].x));
          o.y = __dadd_rn(rv[k].y, __dmul_rn(beta, pv[k].y));
          p2[j] = o;
        }
      }
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t j = n - 1;
    const double pv = p[j];
    if (do_x) {
      x[j] = __dadd_rn(x[j], __dmul_rn(alpha, pv));
      if constexpr (XX) acc = __dadd_rn(acc, __dmul_rn(x[j], x[j]));
    }
    if (do_p) p[j] = __dadd_rn(r[j], __dmul_rn(beta, pv));
  }
  if constexpr (XX) {
    double tot;
    if (do_x && grid_sum(acc, partials, ticket, &tot) && threadIdx.x == 0) c->xx = tot;
  }
}

// ---------------------------------------------------------------- GMRES kernels
// prologue: w = b - A x ; beta = ||w|| ; explicit convergence / budget checks
__device__ void gm_restart_logic(SolveCtrl* c, double tot) {
    const double beta = sqrt(tot);
    const double resid = beta / c->bnorm;
    c->resid = resid;
    c->beta = beta;
    c->k = 0;
    c->stop = 0;
    c->event = EV_NONE;
    if (!isfinite(resid)) {
      c->event = EV_ABORT;
      c->stop = 1;
    } else if (resid <= c->tol) {
      c->event = EV_EXPLICIT_OK;
      c->stop = 1;
    } else if (c->iter >= c->max_iters) {
      c->event = EV_MAXITER;
      c->stop = 1;
    } else {
      for (int i = 0; i <= c->restart; ++i) c->g[i] = 0.0;
      c->g[0] = beta;
    }
}

// defer (distributed): only this rank's ||w||^2 partial -> c->dot; the host allreduces it
// and k_gm_restart_fin applies the logic on the global sum (identically on every rank)
__global__ void __launch_bounds__(256, 4) k_gm_restart(SolveCtrl* __restrict__ c,
                                                    const double* __restrict__ b,
                                                    double* __restrict__ w, int64_t n,
                                                    double* partials, unsigned* ticket,
                                                    int defer) {
  pdl_wait();
  pdl_trigger();
  double acc = 0.0;
  GRID_LOOP(i, n) {
    const double v = __dsub_rn(b[i], w[i]);
    w[i] = v;
    acc = __dadd_rn(acc, __dmul_rn(v, v));
  }
  double tot;
  if (grid_sum(acc, partials, ticket, &tot) && threadIdx.x == 0) {
    if (defer)
      c->dot = tot;
    else
      gm_restart_logic(c, tot);
  }
}

__global__ void k_gm_restart_fin(SolveCtrl* __restrict__ c) {
  if (threadIdx.x == 0 && blockIdx.x == 0) gm_restart_logic(c, c->dot);
}

// dst = src / *den   (skipped when stopped)
__global__ void __launch_bounds__(256, 4) k_gm_scale(const SolveCtrl* __restrict__ c,
                                                  const double* __restrict__ src,
                                                  double* __restrict__ dst, int64_t n,
                                                  int use_hn) {
  pdl_wait();
  pdl_trigger();
  if (c->stop) return;
  const double den = use_hn ? c->hn : c->beta;
  GRID_LOOP(i, n) dst[i] = src[i] / den;
}

// MGS step i of inner iteration j: (i > 0) w -= H[i-1][j] v_{i-1}; H[i][j] = w . v_i
__global__ void __launch_bounds__(256, 4) k_gm_mgs(SolveCtrl* __restrict__ c, double* __restrict__ w,
                                                const double* __restrict__ V, int64_t n, int i,
                                                int j, double* partials, unsigned* ticket) {
  pdl_wait();
  pdl_trigger();
  if (c->stop) return;
  const int m = c->restart;
  const double* vi = V + (size_t)i * n;
  double acc = 0.0;
  // 16-byte accesses, 2 pairs in flight per thread (V rows are n doubles apart: pairs are
  // 16-byte aligned only for even n, else the scalar loop)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double h = i > 0 ? c->H[(i - 1) * m + j] : 0.0;
  const double* vp = V + (size_t)(i > 0 ? i - 1 : 0) * n;
  if ((n & 1) == 0) {
    const int64_t n2 = n >> 1;
    double2* w2 = reinterpret_cast<double2*>(w);
    const double2* vi2 = reinterpret_cast<const double2*>(vi);
    const double2* vp2 = reinterpret_cast<const double2*>(vp);
    for (int64_t q = t0; q < n2; q += 2 * stride) {
      double2 wv[2], a[2], bp[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int64_t e = q + k * stride;
        if (e < n2) {
          wv[k] = w2[e];
          a[k] = vi2[e];
          if (i > 0) bp[k] = vp2[e];
        }
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int64_t e = q + k * stride;
        if (e < n2) {
          if (i > 0) {
            wv[k].x = __dsub_rn(wv[k].x, __dmul_rn(h, bp[k].x));
            wv[k].y = __dsub_rn(wv[k].y, __dmul_rn(h, bp[k].y));
            w2[e] = wv[k];
          }
          acc = __dadd_rn(acc, __dmul_rn(wv[k].x, a[k].x));
          acc = __dadd_rn(acc, __dmul_rn(wv[k].y, a[k].y));
        }
      }
    }
  } else if (i > 0) {
    GRID_LOOP(q, n) {
      const double wv = __dsub_rn(w[q], __dmul_rn(h, vp[q]));
      w[q] = wv;
      acc = __dadd_rn(acc, __dmul_rn(wv, vi[q]));
    }
  } else {
    GRID_LOOP(q, n) acc = __dadd_rn(acc, __dmul_rn(w[q], vi[q]));
  }
  double tot;
  if (grid_sum(acc, partials, ticket, &tot) && threadIdx.x == 0) c->H[i * m + j] = tot;
}

// End of inner iteration j (one thread): h_{j+1,j} = hn, previous Givens rotations applied
// to column j, new rotation (R18), residual estimate |g_{j+1}| / ||b||, monitor and events.
// col[i * cstride] = H[i][j] (i <= j + 1); cs, sn, g and the scalars in *c may be the
// control block itself or a shared-memory snapshot of it (written back by the caller).
__device__ void gm_finish(SolveCtrl* c, double* ring, int j, double hn, double* col,
                          int cstride, double* cs, double* sn, double* g) {
  c->hn = hn;
  col[(j + 1) * cstride] = hn;
  for (int i = 0; i < j; ++i) {  // apply previous rotations to column j
    const double h1 = col[i * cstride], h2 = col[(i + 1) * cstride];
    const double a1 = __dmul_rn(cs[i], h1), a2 = __dmul_rn(sn[i], h2);
    const double b1 = __dmul_rn(sn[i], h1), b2 = __dmul_rn(cs[i], h2);
    col[i * cstride] = __dadd_rn(a1, a2);
    col[(i + 1) * cstride] = __dsub_rn(b2, b1);
  }
  const double h1 = col[j * cstride], h2 = col[(j + 1) * cstride];
  double cc, ss;
  if (h2 == 0.0) {
    cc = 1.0;
    ss = 0.0;
  } else if (fabs(h2) > fabs(h1)) {
    const double tau = h1 / h2;
    ss = 1.0 / sqrt(__dadd_rn(1.0, __dmul_rn(tau, tau)));
    cc = __dmul_rn(ss, tau);
  } else {
    const double tau = h2 / h1;
    cc = 1.0 / sqrt(__dadd_rn(1.0, __dmul_rn(tau, tau)));
    ss = __dmul_rn(cc, tau);
  }
  cs[j] = cc;
  sn[j] = ss;
  col[j * cstride] = __dadd_rn(__dmul_rn(cc, h1), __dmul_rn(ss, h2));
  col[(j + 1) * cstride] = 0.0;
  g[j + 1] = -__dmul_rn(ss, g[j]);
  g[j] = __dmul_rn(cc, g[j]);
  const double resid = fabs(g[j + 1]) / c->bnorm;
  c->resid = resid;
  const long long jg = c->iter + 1;
  c->iter = jg;
  c->k = j + 1;
  if (!isfinite(resid)) {
    c->event = EV_ABORT;
    c->stop = 1;
  } else {
    ring_push(c, ring, resid);
    if (resid <= c->tol || hn == 0.0) {
      c->event = EV_CONVERGED;
      c->stop = 1;
    } else if (monitor_check(c, ring, jg, resid)) {
      c->event = EV_ESCALATE;
      c->stop = 1;
    } else if (jg >= c->max_iters) {
      c->stop = 1;  // the next restart reports MAXITER after the explicit check
    }
  }
}

// Whole Arnoldi step j after the SpMV w = A v_j, in ONE cooperative launch (the per-step
// kernels below are the fallback for vectors too long for the shared-memory slice):
//   for i = 0..j: w -= h_{i-1,j} v_{i-1} (i > 0); h_{i,j} = w . v_i     (MGS, oracle order)
//   w -= h_{j,j} v_j ; hn = ||w|| ; v_{j+1} = w / hn ; gm_finish
// Each thread owns elements e0 + k T (T = grid threads, k < E) of w, kept in shared memory
// across the j + 2 grid-wide reductions, so a step reads only v_{i-1} and v_i from memory
// (the per-step kernels also read and write w).  Each reduction: CTA partial -> grid
// barrier -> every CTA sums all partials in the same fixed order (identical totals
// everywhere; partials double-buffered across consecutive reductions).
constexpr int GM_THREADS = 1024;  // one CTA per SM: 148 barrier arrivals and partials

__device__ __forceinline__ double gm_grid_total(double part, double* partials, int buf,
                                                double* red, double* s_tot) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  part = warp_sum_d(part);
  if (lane == 0) red[warp] = part;
  __syncthreads();
  const unsigned G = gridDim.x;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < GM_THREADS / 32; ++w) s += red[w];
    partials[(size_t)buf * G + blockIdx.x] = s;
  }
  cooperative_groups::this_grid().sync();
  if (warp == 0) {
    double s = 0.0;
    for (unsigned q = lane; q < G; q += 32) s += __ldcg(partials + (size_t)buf * G + q);
    s = warp_sum_d(s);
    if (lane == 0) *s_tot = s;
  }
  __syncthreads();
  return *s_tot;
}

// GW = false: w's slice lives in shared memory (vectors up to ~3.8M rows); GW = true (longer
// vectors): w stays in global memory -- the same HBM traffic as the per-step kernels, but
// one kernel per Arnoldi step (grid barriers instead of j + 3 kernel boundaries)
template <bool GW>
__global__ void __launch_bounds__(GM_THREADS, 1) k_gm_arnoldi(SolveCtrl* __restrict__ c,
                                                             double* ring,
                                                             double* __restrict__ w_in,
                                                             double* __restrict__ V, int64_t n,
                                                             int j, int E, double* partials) {
  extern __shared__ double wsm_[];  // !GW: E * GM_THREADS, this thread's slice at [k * GM_THREADS + t]
  __shared__ unsigned long long sctrl[CTRL_HEAD_WORDS];
  __shared__ double s_col[MAX_RESTART + 1], s_cs[MAX_RESTART], s_sn[MAX_RESTART];
  __shared__ double s_g[MAX_RESTART + 1];
  __shared__ double red[GM_THREADS / 32];
  __shared__ double s_tot;
  if (c->stop) return;  // uniform: written only before this launch
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // snapshots for the end-of-step logic (consumed by CTA 0 after the barriers)
  if (blockIdx.x == 0) {
    if (warp == 0) ctrl_load_head(c, sctrl);
    if (warp == 1)
      for (int i = lane; i < j; i += 32) {
        s_cs[i] = c->cs[i];
        s_sn[i] = c->sn[i];
      }
    if (warp == 2)
      for (int i = lane; i <= j + 1; i += 32) s_g[i] = c->g[i];
  }
  const int64_t T = (int64_t)gridDim.x * GM_THREADS;
  const int64_t e0 = (int64_t)blockIdx.x * GM_THREADS + tid;
  // element k of this thread's slice: e0 + k T, stored at W(k)
  auto W = [&](int k) -> double& {
    if constexpr (GW)
      return w_in[e0 + (int64_t)k * T];
    else
      return wsm_[k * GM_THREADS + tid];
  };
  if constexpr (!GW) {
    for (int k = 0; k < E; ++k) {
      const int64_t e = e0 + k * T;
      wsm_[k * GM_THREADS + tid] = e < n ? w_in[e] : 0.0;
    }
  }
  double h_prev = 0.0;
  for (int i = 0; i <= j; ++i) {
    const double* vi = V + (size_t)i * n;
    const double* vp = V + (size_t)(i > 0 ? i - 1 : 0) * n;
    double acc = 0.0;
    // batches of 4 slice elements: all 8 loads issued before the dependent arithmetic
    for (int k0 = 0; k0 < E; k0 += 4) {
      double a[4], bp[4], wq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t e = e0 + (int64_t)(k0 + q) * T;
        const bool in = k0 + q < E && e < n;
        a[q] = in ? __ldg(vi + e) : 0.0;
        bp[q] = (in && i > 0) ? __ldg(vp + e) : 0.0;
        if constexpr (GW) wq[q] = in ? w_in[e] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t e = e0 + (int64_t)(k0 + q) * T;
        if (k0 + q < E && e < n) {
          double wv = GW ? wq[q] : W(k0 + q);
          if (i > 0) {
            wv = __dsub_rn(wv, __dmul_rn(h_prev, bp[q]));
            W(k0 + q) = wv;
          }
          acc = __dadd_rn(acc, __dmul_rn(wv, a[q]));
        }
      }
    }
    h_prev = gm_grid_total(acc, partials, i & 1, red, &s_tot);
    if (blockIdx.x == 0 && tid == 0) s_col[i] = h_prev;
  }
  {  // w -= h_{j,j} v_j ; ||w||
    const double* vj = V + (size_t)j * n;
    double acc = 0.0;
    for (int k0 = 0; k0 < E; k0 += 4) {
      double a[4], wq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t e = e0 + (int64_t)(k0 + q) * T;
        const bool in = k0 + q < E && e < n;
        a[q] = in ? __ldg(vj + e) : 0.0;
        if constexpr (GW) wq[q] = in ? w_in[e] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t e = e0 + (int64_t)(k0 + q) * T;
        if (k0 + q < E && e < n) {
          const double wv = __dsub_rn(GW ? wq[q] : W(k0 + q), __dmul_rn(h_prev, a[q]));
          W(k0 + q) = wv;
          acc = __dadd_rn(acc, __dmul_rn(wv, wv));
        }
      }
    }
    const double hn = sqrt(gm_grid_total(acc, partials, (j + 1) & 1, red, &s_tot));
    double* vn = V + (size_t)(j + 1) * n;  // V holds restart + 1 vectors
    for (int k = 0; k < E; ++k) {
      const int64_t e = e0 + k * T;
      if (e < n) vn[e] = W(k) / hn;
    }
    if (blockIdx.x == 0 && tid == 0) {
      SolveCtrl* sc = reinterpret_cast<SolveCtrl*>(sctrl);
      gm_finish(sc, ring, j, hn, s_col, 1, s_cs, s_sn, s_g);
      const int m = sc->restart;
      for (int i = 0; i <= j + 1; ++i) c->H[i * m + j] = s_col[i];
      c->cs[j] = s_cs[j];
      c->sn[j] = s_sn[j];
      c->g[j] = s_g[j];
      c->g[j + 1] = s_g[j + 1];
      ctrl_store_head(c, sctrl);
    }
  }
}

// last MGS step: w -= H[j][j] v_j ; hn = ||w|| ; Givens (R18) ; estimate ; monitor
__global__ void __launch_bounds__(256, 4) k_gm_last(SolveCtrl* __restrict__ c, double* ring,
                                                 double* __restrict__ w,
                                                 const double* __restrict__ V, int64_t n, int j,
                                                 double* partials, unsigned* ticket,
                                                 int defer) {
  pdl_wait();
  pdl_trigger();
  if (c->stop) return;
  const int m = c->restart;
  const double h = c->H[j * m + j];
  const double* vj = V + (size_t)j * n;
  double acc = 0.0;
  if ((n & 1) == 0) {
    const int64_t n2 = n >> 1, stride = (int64_t)gridDim.x * blockDim.x;
    double2* w2 = reinterpret_cast<double2*>(w);
    const double2* vj2 = reinterpret_cast<const double2*>(vj);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n2; q += 2 * stride) {
      double2 wv[2], a[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int64_t e = q + k * stride;
        if (e < n2) {
          wv[k] = w2[e];
          a[k] = vj2[e];
        }
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int64_t e = q + k * stride;
        if (e < n2) {
          wv[k].x = __dsub_rn(wv[k].x, __dmul_rn(h, a[k].x));
          wv[k].y = __dsub_rn(wv[k].y, __dmul_rn(h, a[k].y));
          w2[e] = wv[k];
          acc = __dadd_rn(acc, __dmul_rn(wv[k].x, wv[k].x));
          acc = __dadd_rn(acc, __dmul_rn(wv[k].y, wv[k].y));
        }
      }
    }
  } else {
    GRID_LOOP(q, n) {
      const double wv = __dsub_rn(w[q], __dmul_rn(h, vj[q]));
      w[q] = wv;
      acc = __dadd_rn(acc, __dmul_rn(wv, wv));
    }
  }
  double tot;
  if (grid_sum(acc, partials, ticket, &tot) && threadIdx.x == 0) {
    if (defer)  // distributed: ||w||^2 partial, finished by k_gm_last_fin after the allreduce
      c->dot = tot;
    else
      gm_finish(c, ring, j, sqrt(tot), c->H + j, m, c->cs, c->sn, c->g);
  }
}

__global__ void k_gm_last_fin(SolveCtrl* __restrict__ c, double* ring, int j) {
  if (threadIdx.x != 0 || blockIdx.x != 0 || c->stop) return;
  gm_finish(c, ring, j, sqrt(c->dot), c->H + j, c->restart, c->cs, c->sn, c->g);
}

// back substitution H[0:k,0:k] y = g[0:k] (one thread; k <= restart)
__global__ void k_gm_backsolve(SolveCtrl* __restrict__ c) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (c->event == EV_ABORT) {
    c->k = 0;
    return;
  }
  const int k = c->k, m = c->restart;
  for (int i = k - 1; i >= 0; --i) {
    double s = c->g[i];
    for (int l = i + 1; l < k; ++l) s = __dsub_rn(s, __dmul_rn(c->H[i * m + l], c->y[l]));
    c->y[i] = s / c->H[i * m + i];
  }
}

// x += sum_i y_i v_i (same per-element operation order as the oracle)
__global__ void __launch_bounds__(256, 4) k_gm_xupdate(const SolveCtrl* __restrict__ c,
                                                    double* __restrict__ x,
                                                    const double* __restrict__ V, int64_t n) {
  pdl_wait();
  pdl_trigger();
  const int k = c->k;
  if (k == 0) return;
  GRID_LOOP(q, n) {
    double xv = x[q];
    for (int i = 0; i < k; ++i) xv = __dadd_rn(xv, __dmul_rn(c->y[i], V[(size_t)i * n + q]));
    x[q] = xv;
  }
}



// ---------------------------------------------------------------- 16-bit Krylov basis
// NEXT-4 (R28): v_j stored as 16-bit GSE-SEM words with a table per vector (vec16.cuh);
// the same MGS / norm / update arithmetic as the FP64 kernels above, on the decoded values.
constexpr int K16_EB = 3;  // k = 8 shared exponents per basis vector: 3 EI bits, 12 significand bits

__global__ void __launch_bounds__(256, 4) k_gm_mgs16(SolveCtrl* __restrict__ c,
                                                  double* __restrict__ w,
                                                  const uint16_t* __restrict__ V16,
                                                  const uint16_t* __restrict__ vtab,
                                                  const int* __restrict__ vlen, int64_t n, int i,
                                                  int j, double* partials, unsigned* ticket) {
  __shared__ double sci[V16_KMAX], scp[V16_KMAX];
  pdl_wait();
  pdl_trigger();
  if (c->stop) return;
  const int ip = i > 0 ? i - 1 : 0;
  load_scales16(vtab + (size_t)i * V16_KMAX, vlen[i], K16_EB, sci);
  load_scales16(vtab + (size_t)ip * V16_KMAX, vlen[ip], K16_EB, scp);
  __syncthreads();
  const int m = c->restart;
  const double h = i > 0 ? c->H[(i - 1) * m + j] : 0.0;
  const uint16_t* vi = V16 + (size_t)i * n;
  const uint16_t* vp = V16 + (size_t)ip * n;
  double acc = 0.0;
  if ((n & 3) == 0) {
    // 4 elements per step: 2 x 16-byte w accesses, one 8-byte access per basis vector
    // (basis rows are n elements apart: 8-byte aligned when n % 4 == 0); the per-element
    // operation order is the scalar loop's
    const int64_t n4 = n >> 2;
    double2* w2 = reinterpret_cast<double2*>(w);
    const uint2* vi4 = reinterpret_cast<const uint2*>(vi);
    const uint2* vp4 = reinterpret_cast<const uint2*>(vp);
    GRID_LOOP(q, n4) {
      double2 wa = w2[2 * q], wb = w2[2 * q + 1];
      const uint2 a = vi4[q];
      double wv[4] = {wa.x, wa.y, wb.x, wb.y};
      const uint32_t ai[4] = {a.x & 0xFFFFu, a.x >> 16, a.y & 0xFFFFu, a.y >> 16};
      if (i > 0) {
        const uint2 bp = vp4[q];
        const uint32_t bi[4] = {bp.x & 0xFFFFu, bp.x >> 16, bp.y & 0xFFFFu, bp.y >> 16};
#pragma unroll
        for (int t = 0; t < 4; ++t) wv[t] = __dsub_rn(wv[t], __dmul_rn(h, dec16(bi[t], scp, K16_EB)));
        w2[2 * q] = make_double2(wv[0], wv[1]);
        w2[2 * q + 1] = make_double2(wv[2], wv[3]);
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) acc = __dadd_rn(acc, __dmul_rn(wv[t], dec16(ai[t], sci, K16_EB)));
    }
  } else {
    GRID_LOOP(q, n) {
      double wv = w[q];
      if (i > 0) {
        wv = __dsub_rn(wv, __dmul_rn(h, dec16(vp[q], scp, K16_EB)));
        w[q] = wv;
      }
      acc = __dadd_rn(acc, __dmul_rn(wv, dec16(vi[q], sci, K16_EB)));
    }
  }
  double tot;
  if (grid_sum(acc, partials, ticket, &tot) && threadIdx.x == 0) c->H[i * m + j] = tot;
}

__global__ void __launch_bounds__(256, 4) k_gm_last16(SolveCtrl* __restrict__ c, double* ring,
                                                   double* __restrict__ w,
                                                   const uint16_t* __restrict__ V16,
                                                   const uint16_t* __restrict__ vtab,
                                                   const int* __restrict__ vlen, int64_t n, int j,
                                                   double* partials, unsigned* ticket) {
  __shared__ double sc[V16_KMAX];
  pdl_wait();
  pdl_trigger();
  if (c->stop) return;
  load_scales16(vtab + (size_t)j * V16_KMAX, vlen[j], K16_EB, sc);
  __syncthreads();
  const int m = c->restart;
  const double h = c->H[j * m + j];
  const uint16_t* vj = V16 + (size_t)j * n;
  double acc = 0.0;
  if ((n & 3) == 0) {
    const int64_t n4 = n >> 2;
    double2* w2 = reinterpret_cast<double2*>(w);
    const uint2* vj4 = reinterpret_cast<const uint2*>(vj);
    GRID_LOOP(q, n4) {
      const double2 wa = w2[2 * q], wb = w2[2 * q + 1];
      const uint2 a = vj4[q];
      double wv[4] = {wa.x, wa.y, wb.x, wb.y};
      const uint32_t ai[4] = {a.x & 0xFFFFu, a.x >> 16, a.y & 0xFFFFu, a.y >> 16};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        wv[t] = __dsub_rn(wv[t], __dmul_rn(h, dec16(ai[t], sc, K16_EB)));
        acc = __dadd_rn(acc, __dmul_rn(wv[t], wv[t]));
      }
      w2[2 * q] = make_double2(wv[0], wv[1]);
      w2[2 * q + 1] = make_double2(wv[2], wv[3]);
    }
  } else {
    GRID_LOOP(q, n) {
      const double wv = __dsub_rn(w[q], __dmul_rn(h, dec16(vj[q], sc, K16_EB)));
      w[q] = wv;
      acc = __dadd_rn(acc, __dmul_rn(wv, wv));
    }
  }
  double tot;
  if (grid_sum(acc, partials, ticket, &tot) && threadIdx.x == 0)
    gm_finish(c, ring, j, sqrt(tot), c->H + j, m, c->cs, c->sn, c->g);
}

// x += sum_i y_i v_i over the decoded 16-bit basis (the oracle's per-element order)
__global__ void __launch_bounds__(256, 4) k_gm_xupdate16(const SolveCtrl* __restrict__ c,
                                                      double* __restrict__ x,
                                                      const uint16_t* __restrict__ V16,
                                                      const uint16_t* __restrict__ vtab,
                                                      const int* __restrict__ vlen, int64_t n) {
  __shared__ double sc[MAX_RESTART][V16_KMAX];
  pdl_wait();
  pdl_trigger();
  const int k = c->k;
  if (k == 0) return;
  for (int t = threadIdx.x; t < k * V16_KMAX; t += blockDim.x) {
    const int i = t / V16_KMAX, e = t % V16_KMAX;
    sc[i][e] = e < vlen[i] ? ldexp(1.0, (int)vtab[(size_t)i * V16_KMAX + e] - 1023 - (15 - K16_EB))
                           : 0.0;
  }
  __syncthreads();
  GRID_LOOP(q, n) {
    double xv = x[q];
    for (int i = 0; i < k; ++i)
      xv = __dadd_rn(xv, __dmul_rn(c->y[i], dec16(V16[(size_t)i * n + q], sc[i], K16_EB)));
    x[q] = xv;
  }
}

// One Arnoldi step on the 16-bit basis (NEXT-4) as ONE cooperative kernel (w in global
// memory): the MGS passes and the norm on the decoded v_i (grid reductions as in
// k_gm_arnoldi), then v_{j+1} = w / h_{j+1,j} encoded in 16-bit form -- exponent histogram
// of the grid (shared-memory bins -> global atomics into hist[j & 1]), grid barrier, the
// table selected redundantly by every CTA (same histogram, same rule -> the same table;
// CTA 0 stores it), the encode of this CTA's slice plus the decoded copy for the next SpMV.
// hist[(j + 1) & 1] is cleared for the next step (both are cleared at every restart).
__device__ void v16_select_block(const unsigned* hist, int k_max, int* sel, int* take_out,
                                 unsigned long long* key, unsigned long long* red) {
  __shared__ int s_nd, s_emax;
  if (threadIdx.x == 0) {
    s_nd = 0;
    s_emax = 0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 2048; e += blockDim.x) {
    const unsigned cnt = (e >= 1 && e <= 2046) ? __ldcg(hist + e) : 0u;
    key[e] = cnt ? (((unsigned long long)cnt << 11) | (unsigned long long)e) : 0ull;
    if (cnt) {
      atomicAdd(&s_nd, 1);
      atomicMax(&s_emax, e);
    }
  }
  __syncthreads();
  const int take = s_nd < k_max ? s_nd : k_max;
  for (int k = 0; k < take; ++k) {
    unsigned long long loc = 0;
    for (int e = threadIdx.x; e < 2048; e += blockDim.x) loc = max(loc, key[e]);
    for (int o = 16; o > 0; o >>= 1) loc = max(loc, __shfl_xor_sync(0xFFFFFFFFu, loc, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = loc;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long b = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b = max(b, red[w]);
      sel[k] = (int)(b & 0x7FFull);
      key[b & 0x7FFull] = 0ull;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bool have = false;
    for (int k = 0; k < take; ++k) have |= (sel[k] == s_emax);
    if (take > 0 && !have) sel[take - 1] = s_emax;  // P:123 (R5)
    *take_out = take;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(GM_THREADS, 1) k_gm_arnoldi16(
    SolveCtrl* __restrict__ c, double* ring, double* __restrict__ w,
    uint16_t* __restrict__ V16, uint16_t* __restrict__ vtab, int* __restrict__ vlen,
    double* __restrict__ vcur, unsigned* __restrict__ hist2, int64_t n, int j, int E,
    double* partials) {
  __shared__ unsigned long long sctrl[CTRL_HEAD_WORDS];
  __shared__ double s_col[MAX_RESTART + 1], s_cs[MAX_RESTART], s_sn[MAX_RESTART];
  __shared__ double s_g[MAX_RESTART + 1];
  __shared__ double red[GM_THREADS / 32];
  __shared__ double s_tot;
  __shared__ double sci[V16_KMAX], scp[V16_KMAX];
  __shared__ unsigned long long key[2048];
  __shared__ unsigned long long redk[GM_THREADS / 32];
  __shared__ unsigned hsm[2048];
  __shared__ int sel[V16_KMAX];
  __shared__ int s_take;
  __shared__ int Etab[V16_KMAX];
  if (c->stop) return;  // uniform: written only before this launch
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (blockIdx.x == 0) {
    if (warp == 0) ctrl_load_head(c, sctrl);
    if (warp == 1)
      for (int i = lane; i < j; i += 32) {
        s_cs[i] = c->cs[i];
        s_sn[i] = c->sn[i];
      }
    if (warp == 2)
      for (int i = lane; i <= j + 1; i += 32) s_g[i] = c->g[i];
  }
  const int64_t T = (int64_t)gridDim.x * GM_THREADS;
  const int64_t e0 = (int64_t)blockIdx.x * GM_THREADS + tid;  // first 4-element chunk
  const int64_t n4 = n >> 2;  // n % 4 == 0 (host check)
  // clear the other step's histogram (unused in this step)
  unsigned* hcur = hist2 + (size_t)(j & 1) * 2048;
  unsigned* hnext = hist2 + (size_t)((j + 1) & 1) * 2048;
  for (int e = (int)(blockIdx.x * GM_THREADS + tid); e < 2048; e += (int)T) hnext[e] = 0u;
  double h_prev = 0.0;
  for (int i = 0; i <= j; ++i) {
    const int ip = i > 0 ? i - 1 : 0;
    load_scales16(vtab + (size_t)i * V16_KMAX, vlen[i], K16_EB, sci);
    load_scales16(vtab + (size_t)ip * V16_KMAX, vlen[ip], K16_EB, scp);
    __syncthreads();
    const uint2* vi4 = reinterpret_cast<const uint2*>(V16 + (size_t)i * n);
    const uint2* vp4 = reinterpret_cast<const uint2*>(V16 + (size_t)ip * n);
    double2* w2 = reinterpret_cast<double2*>(w);
    double acc = 0.0;
    // 4 consecutive elements per chunk: one 8-byte load per basis vector, two 16-byte w
    // accesses; chunks c = c0 + k T, two chunks in flight
    for (int k0 = 0; k0 < E; k0 += 2) {
      double2 wa[2], wb[2];
      uint2 a4[2], b4[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t cc = e0 + (int64_t)(k0 + q) * T;
        const bool in = k0 + q < E && cc < n4;
        a4[q] = in ? vi4[cc] : make_uint2(0u, 0u);
        b4[q] = (in && i > 0) ? vp4[cc] : make_uint2(0u, 0u);
        wa[q] = in ? w2[2 * cc] : make_double2(0.0, 0.0);
        wb[q] = in ? w2[2 * cc + 1] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t cc = e0 + (int64_t)(k0 + q) * T;
        if (k0 + q < E && cc < n4) {
          double wv[4] = {wa[q].x, wa[q].y, wb[q].x, wb[q].y};
          const uint32_t av[4] = {a4[q].x & 0xFFFFu, a4[q].x >> 16, a4[q].y & 0xFFFFu, a4[q].y >> 16};
          if (i > 0) {
            const uint32_t bv[4] = {b4[q].x & 0xFFFFu, b4[q].x >> 16, b4[q].y & 0xFFFFu, b4[q].y >> 16};
#pragma unroll
            for (int t = 0; t < 4; ++t) wv[t] = __dsub_rn(wv[t], __dmul_rn(h_prev, dec16(bv[t], scp, K16_EB)));
            w2[2 * cc] = make_double2(wv[0], wv[1]);
            w2[2 * cc + 1] = make_double2(wv[2], wv[3]);
          }
#pragma unroll
          for (int t = 0; t < 4; ++t) acc = __dadd_rn(acc, __dmul_rn(wv[t], dec16(av[t], sci, K16_EB)));
        }
      }
    }
    h_prev = gm_grid_total(acc, partials, i & 1, red, &s_tot);
    if (blockIdx.x == 0 && tid == 0) s_col[i] = h_prev;
    __syncthreads();  // sci / scp reused by the next pass
  }
  double hn;
  {  // w -= h_{j,j} v_j ; ||w||
    load_scales16(vtab + (size_t)j * V16_KMAX, vlen[j], K16_EB, sci);
    __syncthreads();
    const uint2* vj4 = reinterpret_cast<const uint2*>(V16 + (size_t)j * n);
    double2* w2 = reinterpret_cast<double2*>(w);
    double acc = 0.0;
    for (int k0 = 0; k0 < E; k0 += 2) {
      double2 wa[2], wb[2];
      uint2 a4[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t cc = e0 + (int64_t)(k0 + q) * T;
        const bool in = k0 + q < E && cc < n4;
        a4[q] = in ? vj4[cc] : make_uint2(0u, 0u);
        wa[q] = in ? w2[2 * cc] : make_double2(0.0, 0.0);
        wb[q] = in ? w2[2 * cc + 1] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t cc = e0 + (int64_t)(k0 + q) * T;
        if (k0 + q < E && cc < n4) {
          double wv[4] = {wa[q].x, wa[q].y, wb[q].x, wb[q].y};
          const uint32_t av[4] = {a4[q].x & 0xFFFFu, a4[q].x >> 16, a4[q].y & 0xFFFFu, a4[q].y >> 16};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            wv[t] = __dsub_rn(wv[t], __dmul_rn(h_prev, dec16(av[t], sci, K16_EB)));
            acc = __dadd_rn(acc, __dmul_rn(wv[t], wv[t]));
          }
          w2[2 * cc] = make_double2(wv[0], wv[1]);
          w2[2 * cc + 1] = make_double2(wv[2], wv[3]);
        }
      }
    }
    hn = sqrt(gm_grid_total(acc, partials, (j + 1) & 1, red, &s_tot));
  }
  if (blockIdx.x == 0 && tid == 0) {
    SolveCtrl* sc = reinterpret_cast<SolveCtrl*>(sctrl);
    gm_finish(sc, ring, j, hn, s_col, 1, s_cs, s_sn, s_g);
    const int m = sc->restart;
    for (int i = 0; i <= j + 1; ++i) c->H[i * m + j] = s_col[i];
    c->cs[j] = s_cs[j];
    c->sn[j] = s_sn[j];
    c->g[j] = s_g[j];
    c->g[j + 1] = s_g[j + 1];
    ctrl_store_head(c, sctrl);
  }
  if (j + 1 >= c->restart) return;  // (uniform) no v_{j+1} in this cycle
  // v_{j+1} = w / hn in 16-bit form: histogram of the grid ...
  for (int e = tid; e < 2048; e += GM_THREADS) hsm[e] = 0u;
  __syncthreads();
  for (int k = 0; k < E; ++k) {
    const int64_t cc = e0 + (int64_t)k * T;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      unsigned ex = 0xFFFFFFFFu;
      if (cc < n4) {
        const double v = w[4 * cc + t] / hn;
        ex = (unsigned)((unsigned long long)__double_as_longlong(v) >> 52) & 0x7FFu;
        if (ex == 0u || ex == 0x7FFu) ex = 0xFFFFFFFFu;
      }
      const unsigned peers = __match_any_sync(0xFFFFFFFFu, ex);
      if (ex != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hsm[ex], (unsigned)__popc(peers));
    }
  }
  __syncthreads();
  for (int e = tid; e < 2048; e += GM_THREADS)
    if (hsm[e]) atomicAdd(&hcur[e], hsm[e]);
  __threadfence();
  cooperative_groups::this_grid().sync();
  // ... the table (every CTA, same result) ...
  v16_select_block(hcur, 8, sel, &s_take, key, redk);
  const int take = s_take;
  if (tid < V16_KMAX) Etab[tid] = tid < take ? sel[tid] + 1 : 0;
  __syncthreads();
  uint16_t* tabn = vtab + (size_t)(j + 1) * V16_KMAX;
  if (blockIdx.x == 0 && tid < V16_KMAX) tabn[tid] = (uint16_t)Etab[tid];
  if (blockIdx.x == 0 && tid == 0) vlen[j + 1] = take;
  if (tid < V16_KMAX) sci[tid] = tid < take ? ldexp(1.0, Etab[tid] - 1023 - (15 - K16_EB)) : 0.0;
  __syncthreads();
  // ... and the encode of this CTA's slice (+ the decoded copy for the next SpMV)
  uint2* vn4 = reinterpret_cast<uint2*>(V16 + (size_t)(j + 1) * n);
  const double2* w2c = reinterpret_cast<const double2*>(w);
  double2* vc2 = reinterpret_cast<double2*>(vcur);
  for (int k = 0; k < E; ++k) {
    const int64_t cc = e0 + (int64_t)k * T;
    if (cc < n4) {
      const double2 wa = w2c[2 * cc], wb = w2c[2 * cc + 1];
      const double wv[4] = {wa.x, wa.y, wb.x, wb.y};
      uint32_t wd[4];
      double dv[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        wd[t] = enc16(wv[t] / hn, Etab, take, K16_EB);
        dv[t] = dec16(wd[t], sci, K16_EB);
      }
      vn4[cc] = make_uint2(wd[0] | (wd[1] << 16), wd[2] | (wd[3] << 16));
      vc2[2 * cc] = make_double2(dv[0], dv[1]);
      vc2[2 * cc + 1] = make_double2(dv[2], dv[3]);
    }
  }
}

// ---------------------------------------------------------------- workspace
// Pinned host mirrors of the control block and the capture streams are process-wide
// caches: cudaMallocHost / cudaStreamCreate cost milliseconds, and a matrix (with its
// solver workspace) may be created per solve.
static std::mutex g_cache_mu;
static std::vector<SolveCtrl*> g_pinned_free;
static cudaStream_t g_cap_stream[64] = {nullptr};

static SolveCtrl* pinned_ctrl_get() {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (!g_pinned_free.empty()) {
    SolveCtrl* p = g_pinned_free.back();
    g_pinned_free.pop_back();
    return p;
  }
  SolveCtrl* p = nullptr;
  if (cudaMallocHost(&p, sizeof(SolveCtrl)) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

static void pinned_ctrl_put(SolveCtrl* p) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_pinned_free.push_back(p);
}

static cudaStream_t capture_stream(int dev) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!g_cap_stream[dev]) cudaStreamCreateWithFlags(&g_cap_stream[dev], cudaStreamNonBlocking);
  return g_cap_stream[dev];
}

static gse_status ensure_ws(Matrix& M, int64_t ring_t, int gm_restart, cudaStream_t s,
                            int k16 = 0) {
  SolverWs*& ws = M.ws;
  const int64_t n = M.rows;
  if (!ws) {
    ws = new SolverWs();
    ws->n = n;
    ws->vgrid = num_sms(M.device) * 4;  // one wave: every vector kernel fits 4 CTAs of 256 per SM
    const size_t nn = (size_t)(n > 0 ? n : 1);
    ws->x = dev_alloc_n<double>(nn, s);
    ws->r = dev_alloc_n<double>(nn, s);
    // p is gathered by the SpMV: distributed -> owned + halo entries
    ws->p = dev_alloc_n<double>((size_t)dist_ext_cols(M) + 1, s);
    ws->q = dev_alloc_n<double>(nn, s);
    ws->b = dev_alloc_n<double>(nn, s);
    ws->tmp = dev_alloc_n<double>(nn, s);
    const int64_t np = (M.n_blocks > 2 * ws->vgrid ? M.n_blocks : 2 * ws->vgrid) + 1;
    ws->partials = dev_alloc_n<double>((size_t)np, s);
    ws->ticket = dev_alloc_n<unsigned>(4, s);
    ws->ctrl = dev_alloc_n<SolveCtrl>(1, s);
    if (!ws->x || !ws->r || !ws->p || !ws->q || !ws->b || !ws->tmp || !ws->partials ||
        !ws->ticket || !ws->ctrl)
      return GSE_ERR_OOM;
    GSE_CUDA_TRY(cudaMemsetAsync(ws->ticket, 0, 16, s));
    ws->hctrl = pinned_ctrl_get();
    ws->cap_stream = capture_stream(M.device);
    if (!ws->hctrl || !ws->cap_stream) return GSE_ERR_CUDA;
    GSE_CUDA_TRY(cudaEventCreate(&ws->ev0));
    GSE_CUDA_TRY(cudaEventCreate(&ws->ev1));
  }
  if (ring_t + 1 > ws->ring_cap) {
    if (ws->ring) dev_free(ws->ring, s);
    ws->ring_cap = ring_t + 1;
    ws->ring = dev_alloc_n<double>((size_t)ws->ring_cap, s);
    if (!ws->ring) return GSE_ERR_OOM;
  }
  if (gm_restart > 0 && !k16 && gm_restart + 1 > ws->V_cols) {
    if (ws->V) dev_free(ws->V, s);
    ws->V_cols = gm_restart + 1;
    ws->V = dev_alloc_n<double>((size_t)ws->V_cols * (size_t)(n > 0 ? n : 1), s);
    if (!ws->V) return GSE_ERR_OOM;
  }
  if (gm_restart > 0 && k16 && gm_restart + 1 > ws->V16_cols) {
    for (void* p : {(void*)ws->V16, (void*)ws->vtab, (void*)ws->vlen})
      if (p) dev_free(p, s);
    ws->V16_cols = gm_restart + 1;
    const size_t nn = (size_t)(n > 0 ? n : 1);
    ws->V16 = dev_alloc_n<uint16_t>((size_t)ws->V16_cols * nn, s);
    ws->vtab = dev_alloc_n<uint16_t>((size_t)ws->V16_cols * V16_KMAX, s);
    ws->vlen = dev_alloc_n<int>((size_t)ws->V16_cols, s);
    if (!ws->vhist) ws->vhist = dev_alloc_n<unsigned>(2048, s);
    if (!ws->vhist2) ws->vhist2 = dev_alloc_n<unsigned>(2 * 2048, s);
    if (!ws->vcur) ws->vcur = dev_alloc_n<double>(nn, s);
    if (!ws->V16 || !ws->vtab || !ws->vlen || !ws->vhist || !ws->vhist2 || !ws->vcur)
      return GSE_ERR_OOM;
    GSE_CUDA_TRY(cudaMemsetAsync(ws->vhist, 0, 2048 * sizeof(unsigned), s));
    GSE_CUDA_TRY(cudaMemsetAsync(ws->vlen, 0, (size_t)ws->V16_cols * sizeof(int), s));
  }
  return GSE_OK;
}

void free_solver_ws(Matrix& M) {
  SolverWs* ws = M.ws;
  if (!ws) return;
  cudaStream_t s = nullptr;
  for (int L = 0; L < 3; ++L) {
    if (ws->cg_exec[L]) cudaGraphExecDestroy(ws->cg_exec[L]);
    if (ws->cg_graph[L]) cudaGraphDestroy(ws->cg_graph[L]);
    if (ws->gm_exec[L]) cudaGraphExecDestroy(ws->gm_exec[L]);
    if (ws->gm_graph[L]) cudaGraphDestroy(ws->gm_graph[L]);
    if (ws->dcg_exec[L]) cudaGraphExecDestroy(ws->dcg_exec[L]);
    if (ws->dcg_graph[L]) cudaGraphDestroy(ws->dcg_graph[L]);
    if (ws->dgm_exec[L]) cudaGraphExecDestroy(ws->dgm_exec[L]);
    if (ws->dgm_graph[L]) cudaGraphDestroy(ws->dgm_graph[L]);
  }
  for (double* p : {ws->x, ws->r, ws->p, ws->q, ws->b, ws->tmp, ws->V, ws->partials,
                    ws->ring, ws->vcur})
    if (p) dev_free(p, s);
  for (void* p : {(void*)ws->V16, (void*)ws->vtab, (void*)ws->vlen, (void*)ws->vhist,
                  (void*)ws->vhist2})
    if (p) dev_free(p, s);
  if (ws->ticket) dev_free(ws->ticket, s);
  if (ws->ctrl) dev_free(ws->ctrl, s);
  if (ws->hctrl) pinned_ctrl_put(ws->hctrl);
  if (ws->ev0) cudaEventDestroy(ws->ev0);
  if (ws->ev1) cudaEventDestroy(ws->ev1);
  delete ws;
  M.ws = nullptr;
}

static gse_status read_ctrl(SolverWs* ws, cudaStream_t s) {
  GSE_CUDA_TRY(cudaMemcpyAsync(ws->hctrl, ws->ctrl, sizeof(SolveCtrl), cudaMemcpyDeviceToHost, s));
  GSE_CUDA_TRY(cudaStreamSynchronize(s));
  return GSE_OK;
}

template <class T>
static gse_status set_field(SolverWs* ws, T SolveCtrl::*field, T v, cudaStream_t s) {
  // stream-ordered host->device write of one control field (pinned staging)
  size_t off = (size_t)(&(((SolveCtrl*)nullptr)->*field));
  T* staging = (T*)((char*)ws->hctrl + off);
  *staging = v;
  GSE_CUDA_TRY(cudaMemcpyAsync((char*)ws->ctrl + off, staging, sizeof(T), cudaMemcpyHostToDevice, s));
  return GSE_OK;
}

static DotOut dot_to(SolverWs* ws, double* target) {
  DotOut d;
  d.partials = ws->partials;
  d.ticket = ws->ticket;
  d.result = target;
  return d;
}

gse_status spmv_dot_ws(Matrix& M, int level, const double* x, double* y, double* dot,
                       cudaStream_t s) {
  gse_status rc = ensure_ws(M, 0, 0, s);
  if (rc != GSE_OK) return rc;
  DotOut d = dot_to(M.ws, dot);
  return launch_spmv(M, level, x, y, &d, s, nullptr);
}

// GSE_NO_GRAPH=1: drive solver iterations from the host instead of CUDA graphs (ncu cannot
// profile kernel nodes of graphs with conditional nodes; also a fallback)
static bool no_graph() {
  static const bool v = [] {
    const char* e = getenv("GSE_NO_GRAPH");
    return e && e[0] == '1';
  }();
  return v;
}

// x += alpha p ; p = r + beta p (+ ||x||^2 when the R29 trigger is on: ws->cg_xx)
static void launch_xpay(SolverWs* ws, cudaStream_t s, int64_t n) {
  if (ws->cg_xx)
    launch_k(k_cg_xpay<true>, ws->vgrid, 256, 0, s, ws->ctrl, ws->x, ws->p, (const double*)ws->r,
             n, ws->partials, ws->ticket);
  else
    launch_k(k_cg_xpay<false>, ws->vgrid, 256, 0, s, ws->ctrl, ws->x, ws->p, (const double*)ws->r,
             n, ws->partials, ws->ticket);
}

static void drop_cg_graphs(SolverWs* ws) {
  for (int L = 0; L < 3; ++L) {
    if (ws->cg_exec[L]) cudaGraphExecDestroy(ws->cg_exec[L]);
    if (ws->cg_graph[L]) cudaGraphDestroy(ws->cg_graph[L]);
    ws->cg_exec[L] = nullptr;
    ws->cg_graph[L] = nullptr;
  }
}

// ---------------------------------------------------------------- distributed CG batch
// One distributed CG iteration (every rank issues the same collectives): halo of p + SpMV
// (interior rows overlapped with the exchange) + local p.q, allreduce, update + local r.r,
// allreduce, the event logic on the global sums, x / p update.  After an event every kernel
// returns at once and the collectives sum values nobody reads (all ranks stop together).
constexpr int DIST_BATCH = 16;
static gse_status dist_cg_iteration(Matrix& M, int level, cudaStream_t s) {
  SolverWs* ws = M.ws;
  const int64_t n = M.rows;
  DotOut d = dot_to(ws, &ws->ctrl->pq);
  gse_status rc = dist_spmv(M, level, ws->p, ws->q, &d, s, &ws->ctrl->event);
  if (rc != GSE_OK) return rc;
  rc = dist_allreduce_sum(M, &ws->ctrl->pq, 1, s);
  if (rc != GSE_OK) return rc;
  launch_k(k_cg_update, ws->vgrid, 256, 0, s, ws->ctrl, ws->ring, ws->r, ws->q, n, ws->partials,
           ws->ticket, 0, 0, 1);
  rc = dist_allreduce_sum(M, &ws->ctrl->rr_part, 1, s);
  if (rc != GSE_OK) return rc;
  launch_k(k_cg_events, 1, 32, 0, s, ws->ctrl, ws->ring);
  launch_xpay(ws, s, n);
  GSE_CUDA_TRY(cudaGetLastError());
  return GSE_OK;
}

// NCCL backend: the batch captured once per level as a CUDA graph (NCCL grouped send/recv,
// the two 8-byte allreduces, the side-stream interior SpMV and the kernels), replayed with
// one launch per DIST_BATCH iterations instead of ~8 launches + 2 collectives per iteration
static gse_status build_dist_cg_graph(Matrix& M, int level) {
  SolverWs* ws = M.ws;
  if (ws->dcg_exec[level - 1]) return GSE_OK;
  cudaStream_t cs = ws->cap_stream;
  GSE_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
  gse_status rc = GSE_OK;
  for (int it = 0; it < DIST_BATCH && rc == GSE_OK; ++it) rc = dist_cg_iteration(M, level, cs);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(cs, &g);
  if (rc != GSE_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  GSE_CUDA_TRY(e);
  GSE_CUDA_TRY(cudaGraphInstantiate(&ws->dcg_exec[level - 1], g, 0));
  ws->dcg_graph[level - 1] = g;
  return GSE_OK;
}

// ---------------------------------------------------------------- CG graph per level
static gse_status build_cg_graph(Matrix& M, int level) {
  SolverWs* ws = M.ws;
  if (ws->cg_exec[level - 1]) return GSE_OK;
  cudaGraph_t g;
  GSE_CUDA_TRY(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  GSE_CUDA_TRY(cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  GSE_CUDA_TRY(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaStream_t cs = ws->cap_stream;
  GSE_CUDA_TRY(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                             cudaStreamCaptureModeRelaxed));
  const int64_t n = M.rows;
  DotOut d = dot_to(ws, &ws->ctrl->pq);
  // iterations per pass of the while body (the kernels of an iteration after an event are
  // no-ops, so the body may hold several): each evaluation of the conditional node costs
  // ~1.7 us; 8 per body: 49.0 -> 45.5 us per C2 iteration (GSE_CG_UNROLL overrides)
  const int unroll = [] {  // read when a graph is built (once per matrix and level)
    const char* e = getenv("GSE_CG_UNROLL");
    const int u = e ? atoi(e) : 8;
    return u < 1 ? 1 : (u > 32 ? 32 : u);
  }();
  gse_status rc = GSE_OK;
  for (int u = 0; u < unroll && rc == GSE_OK; ++u) {
    rc = launch_spmv(M, level, ws->p, ws->q, &d, cs, &ws->ctrl->event);
    launch_k(k_cg_update, ws->vgrid, 256, 0, cs, ws->ctrl, ws->ring, ws->r, ws->q, n,
             ws->partials, ws->ticket, h, 1, 0);
    launch_xpay(ws, cs, n);
  }
  cudaGraph_t captured;
  cudaError_t e = cudaStreamEndCapture(cs, &captured);
  if (rc != GSE_OK) return rc;
  GSE_CUDA_TRY(e);
  GSE_CUDA_TRY(cudaGraphInstantiate(&ws->cg_exec[level - 1], g, 0));
  ws->cg_graph[level - 1] = g;
  return GSE_OK;
}

static void fill_sched(SolveCtrl* h, const gse_step_schedule& sc, int stepped, const Matrix& M) {
  h->stepped = stepped;
  h->perturb_c = (stepped && M.eta_ok) ? sc.perturb_c : 0.0;
  h->eta[0] = M.eta[0];
  h->eta[1] = M.eta[1];
  h->xx = 0.0;
  h->max_level = sc.max_level;
  h->l = sc.l;
  h->t = sc.t;
  h->m = sc.m;
  h->ndec_limit = sc.ndec_limit;
  h->rsd_limit = sc.rsd_limit;
  h->reldec_limit = sc.reldec_limit;
  h->floor_[0] = sc.level_floor[0];
  h->floor_[1] = sc.level_floor[1];
  h->ring_count = 0;
  h->ring_head = 0;
}

static void log_switch(gse_solve_report& rep, int64_t j, int lvl) {
  char mark[64];  // NVTX mark on the profiler timeline
  snprintf(mark, sizeof(mark), "gse level switch -> %d at iteration %lld", lvl, (long long)j);
  nvtxMarkA(mark);
  if (rep.n_switches < 2) {
    rep.switch_iter[rep.n_switches] = j;
    rep.switch_to_level[rep.n_switches] = lvl;
  }
  rep.n_switches++;
}

// true relative residual ||b - A_3 x|| / ||b|| (x = ws->x); uses ws->tmp / ws->q
// SpMV of a vector held in the rank-local layout: single GPU -> as is; distributed -> the
// owned entries are copied to x_ext and the halo is exchanged first
static gse_status spmv_local(Matrix& M, int level, const double* v, double* out,
                             const DotOut* dot, cudaStream_t s, const int* stop = nullptr) {
  if (M.dist) {
    double* xe = dist_xext(M);
    if (v != xe)
      GSE_CUDA_TRY(cudaMemcpyAsync(xe, v, 8 * M.rows, cudaMemcpyDeviceToDevice, s));
    return dist_spmv(M, level, xe, out, dot, s, stop);
  }
  return launch_spmv(M, level, v, out, dot, s, stop);
}

// r = b - A_level x (p = r when p != null); *out = ||r||^2 (allreduced over ranks)
static gse_status residual(Matrix& M, int level, const double* x, double* r, double* p,
                           double* out, gse_solve_report& rep, cudaStream_t s) {
  SolverWs* ws = M.ws;
  gse_status rc = spmv_local(M, level, x, ws->q, nullptr, s);
  if (rc != GSE_OK) return rc;
  rep.spmv_count[level - 1]++;
  launch_k(k_residual, ws->vgrid, 256, 0, s, ws->b, ws->q, r, p, M.rows, ws->partials, ws->ticket,
                                       out);
  GSE_CUDA_TRY(cudaGetLastError());
  return dist_allreduce_sum(M, out, 1, s);
}

// true relative residual ||b - A_3 x|| / ||b||
static gse_status true_resid(Matrix& M, const double* x, double bnorm, gse_solve_report& rep,
                             double* out, cudaStream_t s) {
  SolverWs* ws = M.ws;
  gse_status rc = residual(M, 3, x, ws->tmp, nullptr, &ws->ctrl->dot, rep, s);
  if (rc != GSE_OK) return rc;
  rc = read_ctrl(ws, s);
  if (rc != GSE_OK) return rc;
  *out = sqrt(ws->hctrl->dot) / bnorm;
  return GSE_OK;
}

gse_status solve_cg(Matrix& M, const double* b, double* x, double tol, int64_t max_iters,
                    const gse_step_schedule& sched, gse_solve_report& rep, cudaStream_t s) {
  const int64_t n = M.rows;  // local rows (distributed: this rank's slice)
  const int stepped = sched.enabled && M.kind == GSE_KIND_GSE;
  int level = (M.kind != GSE_KIND_GSE) ? 3 : sched.start_level;  // FP64/FP16/BF16: one precision
  const bool dist = M.dist != nullptr;
  gse_status rc = ensure_ws(M, stepped ? sched.t : 0, 0, s);
  if (rc != GSE_OK) return rc;
  SolverWs* ws = M.ws;
  const bool xx_on = stepped && sched.perturb_c > 0.0;
  if (xx_on) {
    rc = perturbation_bounds(M, s);  // once per matrix (R29)
    if (rc != GSE_OK) return rc;
  }
  if ((int)xx_on != ws->cg_xx) {  // the graphs' xpay variant follows the trigger
    drop_cg_graphs(ws);
    ws->cg_xx = xx_on ? 1 : 0;
  }
  GSE_CUDA_TRY(cudaEventRecord(ws->ev0, s));
  GSE_CUDA_TRY(cudaMemcpyAsync(ws->b, b, n * 8, cudaMemcpyDeviceToDevice, s));
  GSE_CUDA_TRY(cudaMemcpyAsync(ws->x, x, n * 8, cudaMemcpyDeviceToDevice, s));
  // ||b||, r0 = b - A_L x0, p0 = r0, rr
  launch_k(k_dot, ws->vgrid, 256, 0, s, ws->b, ws->b, n, ws->partials, ws->ticket, &ws->ctrl->dot);
  GSE_CUDA_TRY(cudaGetLastError());
  rc = dist_allreduce_sum(M, &ws->ctrl->dot, 1, s);
  if (rc != GSE_OK) return rc;
  rc = residual(M, level, ws->x, ws->r, ws->p, &ws->ctrl->rr, rep, s);
  if (rc != GSE_OK) return rc;
  rc = read_ctrl(ws, s);
  if (rc != GSE_OK) return rc;
  SolveCtrl* hc = ws->hctrl;
  const double bnorm = sqrt(hc->dot);
  gse_status status = GSE_NOT_CONVERGED;
  int64_t iter = 0;
  if (bnorm == 0.0) {
    GSE_CUDA_TRY(cudaMemsetAsync(x, 0, n * 8, s));
    rep.converged = 1;
    rep.rel_residual_true = 0.0;
    GSE_CUDA_TRY(cudaStreamSynchronize(s));
    return GSE_OK;
  }
  double resid = sqrt(hc->rr) / bnorm;
  rep.rel_residual_recurrence = resid;
  bool done = false;
  if (resid <= tol) {
    double rt = 0;
    if (!(stepped && level < 3 && sched.verify_at_full)) {
      status = GSE_OK;
      done = true;
    } else {
      rc = true_resid(M, ws->x, bnorm, rep, &rt, s);
      if (rc != GSE_OK) return rc;
      if (rt <= tol) {
        status = GSE_OK;
        done = true;
      } else if (level >= sched.max_level) {  // R16 capped by max_level: not converged
        status = GSE_NOT_CONVERGED;
        done = true;
      } else {
        level = sched.max_level;  // x0 converged at A_L only: the highest allowed level
        log_switch(rep, 0, level);
        rc = residual(M, level, ws->x, ws->r, ws->p, &ws->ctrl->rr, rep, s);
        if (rc != GSE_OK) return rc;
      }
    }
  }
  // control block (scalars live on the device from here on)
  hc = ws->hctrl;
  if (!done) {
    rc = read_ctrl(ws, s);  // refresh rr
    if (rc != GSE_OK) return rc;
    hc->bnorm = bnorm;
    hc->tol = tol;
    hc->iter = 0;
    hc->max_iters = max_iters;
    hc->level = level;
    hc->event = EV_NONE;
    hc->alpha = hc->beta = 0.0;
    fill_sched(hc, sched, stepped, M);
    GSE_CUDA_TRY(cudaMemcpyAsync(ws->ctrl, hc, sizeof(SolveCtrl), cudaMemcpyHostToDevice, s));
    if (xx_on)  // R29: ||x0||^2 for the first iteration's check
      launch_k(k_dot, ws->vgrid, 256, 0, s, (const double*)ws->x, (const double*)ws->x, n,
               ws->partials, ws->ticket, &ws->ctrl->xx);
  }
  int64_t last_iter = 0;
  while (!done) {
    if (iter >= max_iters) {
      status = GSE_NOT_CONVERGED;
      break;
    }
    if (dist) {
      // distributed: batches of DIST_BATCH iterations, captured (NCCL) or host-driven
      const bool graph = dist_capturable(M) && !no_graph();
      if (graph) {
        rc = build_dist_cg_graph(M, level);
        if (rc != GSE_OK) return rc;
      }
      do {
        if (graph) {
          GSE_CUDA_TRY(cudaGraphLaunch(ws->dcg_exec[level - 1], s));
        } else {
          for (int bt = 0; bt < DIST_BATCH; ++bt) {
            rc = dist_cg_iteration(M, level, s);
            if (rc != GSE_OK) return rc;
          }
        }
        rc = read_ctrl(ws, s);
        if (rc != GSE_OK) return rc;
      } while (hc->event == EV_NONE);
    } else if (no_graph()) {
      // host-driven iterations (profiling / fallback): batches of 16, then poll the event
      do {
        DotOut d = dot_to(ws, &ws->ctrl->pq);
        for (int bt = 0; bt < 16; ++bt) {
          rc = launch_spmv(M, level, ws->p, ws->q, &d, s, &ws->ctrl->event);
          if (rc != GSE_OK) return rc;
          launch_k(k_cg_update, ws->vgrid, 256, 0, s, ws->ctrl, ws->ring, ws->r, ws->q, n,
                   ws->partials, ws->ticket, 0, 0, 0);
          launch_xpay(ws, s, n);
        }
        GSE_CUDA_TRY(cudaGetLastError());
        rc = read_ctrl(ws, s);
        if (rc != GSE_OK) return rc;
      } while (hc->event == EV_NONE);
    } else {
      rc = build_cg_graph(M, level);
      if (rc != GSE_OK) return rc;
      GSE_CUDA_TRY(cudaGraphLaunch(ws->cg_exec[level - 1], s));
    }
    rc = read_ctrl(ws, s);
    if (rc != GSE_OK) return rc;
    iter = hc->iter;
    rep.iters_per_level[level - 1] += iter - last_iter;
    rep.spmv_count[level - 1] += iter - last_iter;
    last_iter = iter;
    rep.rel_residual_recurrence = hc->resid;
    const int ev = hc->event;
    bool escalate = false;
    if (ev == EV_ABORT) {
      status = GSE_NUMERICAL_ABORT;
      break;
    } else if (ev == EV_CONVERGED) {
      if (!(stepped && level < 3 && sched.verify_at_full)) {
        status = GSE_OK;
        break;
      }
      double rt = 0;
      rc = true_resid(M, ws->x, bnorm, rep, &rt, s);
      if (rc != GSE_OK) return rc;
      if (rt <= tol) {
        status = GSE_OK;
        break;
      }
      if (level >= sched.max_level) {  // R16 capped by max_level: not converged
        status = GSE_NOT_CONVERGED;
        break;
      }
      escalate = true;
    } else if (ev == EV_ESCALATE) {
      escalate = true;
    } else if (ev == EV_MAXITER) {
      status = GSE_NOT_CONVERGED;
      break;
    } else {
      set_error("internal: CG loop returned without an event");
      return GSE_ERR_CUDA;
    }
    if (escalate) {
      level++;
      log_switch(rep, iter, level);
      if (sched.cg_keep_direction) {
        // R30: residual replacement at the new level, the search direction kept:
        // r = b - A_new x ; beta = r.r / rr_old ; p = r + beta p ; rr = r.r
        rc = residual(M, level, ws->x, ws->r, nullptr, &ws->ctrl->rr_new, rep, s);
        if (rc != GSE_OK) return rc;
        rc = read_ctrl(ws, s);
        if (rc != GSE_OK) return rc;
        const double rr_new = hc->rr_new, beta = rr_new / hc->rr;
        rc = set_field(ws, &SolveCtrl::alpha, 0.0, s);
        if (rc != GSE_OK) return rc;
        rc = set_field(ws, &SolveCtrl::beta, beta, s);
        if (rc != GSE_OK) return rc;
        rc = set_field(ws, &SolveCtrl::event, (int)EV_NONE, s);
        if (rc != GSE_OK) return rc;
        launch_k(k_cg_xpay<false>, ws->vgrid, 256, 0, s, ws->ctrl, ws->x, ws->p,
                 (const double*)ws->r, n, ws->partials, ws->ticket);  // alpha = 0: p only
        GSE_CUDA_TRY(cudaGetLastError());
        rc = set_field(ws, &SolveCtrl::rr, rr_new, s);
        if (rc != GSE_OK) return rc;
      } else {
        // R15: restart from the current x at the new level: r = b - A_new x, p = r
        rc = residual(M, level, ws->x, ws->r, ws->p, &ws->ctrl->rr, rep, s);
        if (rc != GSE_OK) return rc;
      }
      rc = set_field(ws, &SolveCtrl::level, level, s);
      if (rc != GSE_OK) return rc;
      rc = set_field(ws, &SolveCtrl::event, (int)EV_NONE, s);
      if (rc != GSE_OK) return rc;
      // (R30 already set them; a second set_field of beta would race its pinned staging
      // with the p-update kernel's read)
      if (!sched.cg_keep_direction) {
        for (double SolveCtrl::*f : {&SolveCtrl::alpha, &SolveCtrl::beta}) {
          rc = set_field(ws, f, 0.0, s);
          if (rc != GSE_OK) return rc;
        }
      }
      if (iter >= max_iters) {
        status = GSE_NOT_CONVERGED;
        break;
      }
    }
  }
  rep.iterations = iter;
  rep.converged = (status == GSE_OK);
  double rt = 0;
  rc = true_resid(M, ws->x, bnorm, rep, &rt, s);
  if (rc != GSE_OK) return rc;
  rep.rel_residual_true = rt;
  GSE_CUDA_TRY(cudaMemcpyAsync(x, ws->x, n * 8, cudaMemcpyDeviceToDevice, s));
  GSE_CUDA_TRY(cudaEventRecord(ws->ev1, s));
  GSE_CUDA_TRY(cudaEventSynchronize(ws->ev1));
  float ms = 0;
  cudaEventElapsedTime(&ms, ws->ev0, ws->ev1);
  rep.seconds = ms * 1e-3;
  return status;
}

// ---------------------------------------------------------------- GMRES
// Launch shape of k_gm_arnoldi: one CTA of GM_THREADS per SM, E elements of w per thread
// in shared memory.  False (per-step kernels) when the slice does not fit or GSE_GM_COOP=0.
static bool gm_coop_config(const Matrix& M, int64_t n, int* grid, int* E, size_t* smem,
                           bool* gw) {
  const char* env = getenv("GSE_GM_COOP");
  if ((env && env[0] == '0') || n <= 0) return false;
  *gw = false;
  // the dynamic shared-memory attribute is per function and process-wide, and graphs built
  // for other vector lengths (or other threads' solves) launch with other sizes: set it
  // once to the largest size this configuration uses (200 KB), never lower
  static std::once_flag attr_once;
  static bool attr_ok = false;
  std::call_once(attr_once, [] {
    attr_ok = cudaFuncSetAttribute(k_gm_arnoldi<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   200 * 1024) == cudaSuccess;
    cudaGetLastError();
  });
  if (!attr_ok) return false;
  const int sms = num_sms(M.device);
  // GSE_GM_COOP=g: the global-w variant at any size (tests)
  for (int per = (env && env[0] == 'g') ? 0 : 1; per >= 1; --per) {
    int64_t G = (int64_t)sms * per;
    const int64_t need = (n + GM_THREADS - 1) / GM_THREADS;
    if (G > need) G = need;
    const int64_t e = (n + G * GM_THREADS - 1) / (G * GM_THREADS);
    const size_t sm = (size_t)e * GM_THREADS * sizeof(double);
    if (sm > 200 * 1024) continue;
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_gm_arnoldi<false>, GM_THREADS, sm) !=
        cudaSuccess)
      continue;
    if ((int64_t)blocks * sms >= G) {
      *grid = (int)G;
      *E = (int)e;
      *smem = sm;
      return true;
    }
  }
  // longer vectors: w stays in global memory, one CTA of GM_THREADS per SM
  // (GSE_GM_COOP=s keeps the per-step kernels for them)
  if (env && env[0] == 's') return false;
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_gm_arnoldi<true>, GM_THREADS, 0) ==
          cudaSuccess &&
      blocks >= 1) {
    const int64_t G = sms;
    *grid = (int)G;
    *E = (int)((n + G * GM_THREADS - 1) / (G * GM_THREADS));
    *smem = 0;
    *gw = true;
    return true;
  }
  cudaGetLastError();
  return false;
}

static gse_status build_gm_graph(Matrix& M, int level, int restart, int k16) {
  SolverWs* ws = M.ws;
  if (ws->gm_restart != restart || ws->gm_k16 != k16) {
    for (int L = 0; L < 3; ++L) {
      if (ws->gm_exec[L]) cudaGraphExecDestroy(ws->gm_exec[L]);
      if (ws->gm_graph[L]) cudaGraphDestroy(ws->gm_graph[L]);
      ws->gm_exec[L] = nullptr;
      ws->gm_graph[L] = nullptr;
    }
    ws->gm_restart = restart;
    ws->gm_k16 = k16;
  }
  if (ws->gm_exec[level - 1]) return GSE_OK;
  cudaStream_t cs = ws->cap_stream;
  const int64_t n = M.rows;
  SolveCtrl* c = ws->ctrl;
  double* w = ws->tmp;
  GSE_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
  // R29: ||x||^2 at the start of the cycle (one vector read per cycle; read only when the
  // perturbation trigger is on)
  launch_k(k_dot, ws->vgrid, 256, 0, cs, (const double*)ws->x, (const double*)ws->x, n,
           ws->partials, ws->ticket, &c->xx);
  gse_status rc = launch_spmv(M, level, ws->x, w, nullptr, cs);
  launch_pdl(k_gm_restart, ws->vgrid, 256, 0, cs, c, ws->b, w, n, ws->partials, ws->ticket, 0);
  if (k16) {
    // NEXT-4: v_j = w / den in 16-bit GSE form (histogram -> table -> encode); the decoded
    // v_j also goes to vcur, the SpMV input of the next step.  Every kernel skips on stop.
    auto encode16 = [&](int col, const double* den) {
      v16_hist(w, den, n, ws->vhist, &c->stop, ws->vgrid, cs);
      v16_select(ws->vhist, 8, ws->vtab + (size_t)col * V16_KMAX, ws->vlen + col, &c->stop, cs);
      v16_encode(w, den, n, ws->vtab + (size_t)col * V16_KMAX, ws->vlen + col, K16_EB,
                 ws->V16 + (size_t)col * n, ws->vcur, &c->stop, ws->vgrid, cs);
    };
    encode16(0, &c->beta);
    // one cooperative kernel per inner step when the grid fits (w in global memory)
    const char* env = getenv("GSE_GM_COOP");
    const bool coop16 = !(env && (env[0] == '0' || env[0] == 's'));
    int occ = 0;
    if (coop16)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gm_arnoldi16, GM_THREADS, 0);
    cudaGetLastError();
    if (coop16 && occ >= 1 && n > 0 && (n & 3) == 0) {
      GSE_CUDA_TRY(cudaMemsetAsync(ws->vhist2, 0, 2 * 2048 * sizeof(unsigned), cs));
      const int G = num_sms(M.device);
      const int64_t n4 = n >> 2;
      const int E = (int)((n4 + (int64_t)G * GM_THREADS - 1) / ((int64_t)G * GM_THREADS));
      for (int j = 0; j < restart && rc == GSE_OK; ++j) {
        rc = launch_spmv_guarded(M, level, ws->vcur, w, &c->stop, cs);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(GM_THREADS);
        cfg.stream = cs;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const cudaError_t le = cudaLaunchKernelEx(&cfg, k_gm_arnoldi16, c, ws->ring, w, ws->V16,
                                                  ws->vtab, ws->vlen, ws->vcur, ws->vhist2, n,
                                                  j, E, ws->partials);
        if (le != cudaSuccess) {
          cudaStreamEndCapture(cs, nullptr);
          return cuda_status(le, "cooperative k_gm_arnoldi16");
        }
      }
    } else
    for (int j = 0; j < restart && rc == GSE_OK; ++j) {
      rc = launch_spmv_guarded(M, level, ws->vcur, w, &c->stop, cs);
      for (int i = 0; i <= j; ++i)
        launch_k(k_gm_mgs16, ws->vgrid, 256, 0, cs, c, w, (const uint16_t*)ws->V16,
                 (const uint16_t*)ws->vtab, (const int*)ws->vlen, n, i, j, ws->partials,
                 ws->ticket);
      launch_k(k_gm_last16, ws->vgrid, 256, 0, cs, c, ws->ring, w, (const uint16_t*)ws->V16,
               (const uint16_t*)ws->vtab, (const int*)ws->vlen, n, j, ws->partials, ws->ticket);
      if (j + 1 < restart) encode16(j + 1, &c->hn);
    }
    launch_k(k_gm_backsolve, 1, 32, 0, cs, c);
    launch_k(k_gm_xupdate16, ws->vgrid, 256, 0, cs, c, ws->x, (const uint16_t*)ws->V16,
             (const uint16_t*)ws->vtab, (const int*)ws->vlen, n);
    cudaGraph_t g;
    cudaError_t e = cudaStreamEndCapture(cs, &g);
    if (rc != GSE_OK) return rc;
    GSE_CUDA_TRY(e);
    GSE_CUDA_TRY(cudaGraphInstantiate(&ws->gm_exec[level - 1], g, 0));
    ws->gm_graph[level - 1] = g;
    return GSE_OK;
  }
  launch_pdl(k_gm_scale, ws->vgrid, 256, 0, cs, c, w, ws->V, n, 0);
  int cg_grid = 0, cg_e = 0;
  size_t cg_smem = 0;
  bool cg_gw = false;
  const bool coop = gm_coop_config(M, n, &cg_grid, &cg_e, &cg_smem, &cg_gw);
  for (int j = 0; j < restart && rc == GSE_OK; ++j) {
    rc = launch_spmv_guarded(M, level, ws->V + (size_t)j * n, w, &c->stop, cs);
    if (coop) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cg_grid);
      cfg.blockDim = dim3(GM_THREADS);
      cfg.dynamicSmemBytes = cg_smem;
      cfg.stream = cs;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const cudaError_t le =
          cg_gw ? cudaLaunchKernelEx(&cfg, k_gm_arnoldi<true>, c, ws->ring, w, ws->V, n, j, cg_e,
                                     ws->partials)
                : cudaLaunchKernelEx(&cfg, k_gm_arnoldi<false>, c, ws->ring, w, ws->V, n, j, cg_e,
                                     ws->partials);
      if (le != cudaSuccess) {
        cudaStreamEndCapture(cs, nullptr);
        return cuda_status(le, "cooperative k_gm_arnoldi");
      }
      continue;
    }
    for (int i = 0; i <= j; ++i)
      launch_pdl(k_gm_mgs, ws->vgrid, 256, 0, cs, c, w, ws->V, n, i, j, ws->partials, ws->ticket);
    launch_pdl(k_gm_last, ws->vgrid, 256, 0, cs, c, ws->ring, w, ws->V, n, j, ws->partials, ws->ticket, 0);
    if (j + 1 < restart)
      launch_pdl(k_gm_scale, ws->vgrid, 256, 0, cs, c, w, ws->V + (size_t)(j + 1) * n, n, 1);
  }
  launch_pdl(k_gm_backsolve, 1, 32, 0, cs, c);
  launch_pdl(k_gm_xupdate, ws->vgrid, 256, 0, cs, c, ws->x, ws->V, n);
  cudaGraph_t g;
  cudaError_t e = cudaStreamEndCapture(cs, &g);
  if (rc != GSE_OK) return rc;
  GSE_CUDA_TRY(e);
  GSE_CUDA_TRY(cudaGraphInstantiate(&ws->gm_exec[level - 1], g, 0));
  ws->gm_graph[level - 1] = g;
  return GSE_OK;
}

// One restart cycle enqueued directly (no graph) for a row-partitioned matrix: every rank
// enqueues the same kernels and collectives (halo exchange before each SpMV, one 8-byte
// allreduce per MGS dot, per ||w||^2 and per restart norm -- j + 2 per inner step, MGS
// order kept); kernels after a stop return early, so the collectives of the
// skipped steps sum values nobody reads.  All ranks see bit-identical scalars (allreduce),
// hence identical H, Givens rotations, monitor decisions and events.
static gse_status gm_cycle_dist(Matrix& M, int level, int restart, cudaStream_t s) {
  SolverWs* ws = M.ws;
  const int64_t n = M.rows;
  SolveCtrl* c = ws->ctrl;
  double* w = ws->tmp;
  gse_status rc = spmv_local(M, level, ws->x, w, nullptr, s);
  if (rc != GSE_OK) return rc;
  launch_k(k_gm_restart, ws->vgrid, 256, 0, s, c, ws->b, w, n, ws->partials, ws->ticket, 1);
  if ((rc = dist_allreduce_sum(M, &c->dot, 1, s)) != GSE_OK) return rc;
  launch_k(k_gm_restart_fin, 1, 32, 0, s, c);
  launch_k(k_gm_scale, ws->vgrid, 256, 0, s, c, w, ws->V, n, 0);
  for (int j = 0; j < restart; ++j) {
    rc = spmv_local(M, level, ws->V + (size_t)j * n, w, nullptr, s, &c->stop);
    if (rc != GSE_OK) return rc;
    for (int i = 0; i <= j; ++i) {
      launch_k(k_gm_mgs, ws->vgrid, 256, 0, s, c, w, ws->V, n, i, j, ws->partials, ws->ticket);
      if ((rc = dist_allreduce_sum(M, &c->H[i * restart + j], 1, s)) != GSE_OK) return rc;
    }
    launch_k(k_gm_last, ws->vgrid, 256, 0, s, c, ws->ring, w, ws->V, n, j, ws->partials,
             ws->ticket, 1);
    if ((rc = dist_allreduce_sum(M, &c->dot, 1, s)) != GSE_OK) return rc;
    launch_k(k_gm_last_fin, 1, 32, 0, s, c, ws->ring, j);
    if (j + 1 < restart)
      launch_k(k_gm_scale, ws->vgrid, 256, 0, s, c, w, ws->V + (size_t)(j + 1) * n, n, 1);
  }
  launch_k(k_gm_backsolve, 1, 32, 0, s, c);
  launch_k(k_gm_xupdate, ws->vgrid, 256, 0, s, c, ws->x, ws->V, n);
  GSE_CUDA_TRY(cudaGetLastError());
  return GSE_OK;
}

// NCCL backend: the whole restart cycle (halo + SpMV per inner step, the j + 2 scalar
// allreduces of MGS, Givens / monitor, the x update) captured once per level and restart
// length, replayed with one launch per cycle
static gse_status build_dist_gm_graph(Matrix& M, int level, int restart) {
  SolverWs* ws = M.ws;
  if (ws->dgm_restart != restart) {
    for (int L = 0; L < 3; ++L) {
      if (ws->dgm_exec[L]) cudaGraphExecDestroy(ws->dgm_exec[L]);
      if (ws->dgm_graph[L]) cudaGraphDestroy(ws->dgm_graph[L]);
      ws->dgm_exec[L] = nullptr;
      ws->dgm_graph[L] = nullptr;
    }
    ws->dgm_restart = restart;
  }
  if (ws->dgm_exec[level - 1]) return GSE_OK;
  cudaStream_t cs = ws->cap_stream;
  GSE_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
  gse_status rc = gm_cycle_dist(M, level, restart, cs);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(cs, &g);
  if (rc != GSE_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  GSE_CUDA_TRY(e);
  GSE_CUDA_TRY(cudaGraphInstantiate(&ws->dgm_exec[level - 1], g, 0));
  ws->dgm_graph[level - 1] = g;
  return GSE_OK;
}

gse_status solve_gmres(Matrix& M, const double* b, double* x, double tol, int restart,
                       int64_t max_iters, const gse_step_schedule& sched, gse_solve_report& rep,
                       cudaStream_t s) {
  const int64_t n = M.rows;
  const int stepped = sched.enabled && M.kind == GSE_KIND_GSE;
  int level = (M.kind != GSE_KIND_GSE) ? 3 : sched.start_level;  // FP64/FP16/BF16: one precision
  const int k16 = sched.krylov_gse16 ? 1 : 0;
  if (k16 && M.dist) {
    set_error("the 16-bit Krylov basis (krylov_gse16) is single-GPU only");
    return GSE_ERR_WRONG_FORMAT;
  }
  gse_status rc = ensure_ws(M, stepped ? sched.t : 0, restart, s, k16);
  if (rc != GSE_OK) return rc;
  SolverWs* ws = M.ws;
  if (stepped && sched.perturb_c > 0.0) {
    rc = perturbation_bounds(M, s);  // once per matrix (R29)
    if (rc != GSE_OK) return rc;
  }
  GSE_CUDA_TRY(cudaEventRecord(ws->ev0, s));
  GSE_CUDA_TRY(cudaMemcpyAsync(ws->b, b, n * 8, cudaMemcpyDeviceToDevice, s));
  GSE_CUDA_TRY(cudaMemcpyAsync(ws->x, x, n * 8, cudaMemcpyDeviceToDevice, s));
  launch_k(k_dot, ws->vgrid, 256, 0, s, ws->b, ws->b, n, ws->partials, ws->ticket, &ws->ctrl->dot);
  GSE_CUDA_TRY(cudaGetLastError());
  rc = dist_allreduce_sum(M, &ws->ctrl->dot, 1, s);
  if (rc != GSE_OK) return rc;
  rc = read_ctrl(ws, s);
  if (rc != GSE_OK) return rc;
  SolveCtrl* hc = ws->hctrl;
  const double bnorm = sqrt(hc->dot);
  if (bnorm == 0.0) {
    GSE_CUDA_TRY(cudaMemsetAsync(x, 0, n * 8, s));
    rep.converged = 1;
    GSE_CUDA_TRY(cudaStreamSynchronize(s));
    return GSE_OK;
  }
  hc->bnorm = bnorm;
  hc->tol = tol;
  hc->iter = 0;
  hc->max_iters = max_iters;
  hc->level = level;
  hc->event = EV_NONE;
  hc->stop = 0;
  hc->restart = restart;
  hc->k = 0;
  fill_sched(hc, sched, stepped, M);
  GSE_CUDA_TRY(cudaMemcpyAsync(ws->ctrl, hc, sizeof(SolveCtrl), cudaMemcpyHostToDevice, s));
  gse_status status = GSE_NOT_CONVERGED;
  int64_t last_iter = 0, iter = 0;
  for (;;) {
    if (M.dist) {
      if (dist_capturable(M) && !no_graph()) {
        rc = build_dist_gm_graph(M, level, restart);
        if (rc != GSE_OK) return rc;
        GSE_CUDA_TRY(cudaGraphLaunch(ws->dgm_exec[level - 1], s));
      } else {
        rc = gm_cycle_dist(M, level, restart, s);
        if (rc != GSE_OK) return rc;
      }
    } else {
      rc = build_gm_graph(M, level, restart, k16);
      if (rc != GSE_OK) return rc;
      GSE_CUDA_TRY(cudaGraphLaunch(ws->gm_exec[level - 1], s));
    }
    rc = read_ctrl(ws, s);
    if (rc != GSE_OK) return rc;
    iter = hc->iter;
    rep.iters_per_level[level - 1] += iter - last_iter;
    rep.spmv_count[level - 1] += iter - last_iter + 1;  // inner SpMVs + restart residual
    last_iter = iter;
    rep.rel_residual_recurrence = hc->resid;
    const int ev = hc->event;
    if (ev == EV_ABORT) {
      status = GSE_NUMERICAL_ABORT;
      break;
    }
    if (ev == EV_EXPLICIT_OK) {
      if (!(stepped && level < 3 && sched.verify_at_full)) {
        status = GSE_OK;
        break;
      }
      double rt = 0;
      rc = true_resid(M, ws->x, bnorm, rep, &rt, s);
      if (rc != GSE_OK) return rc;
      if (rt <= tol) {
        status = GSE_OK;
        break;
      }
      if (level >= sched.max_level) {  // R16 capped by max_level: not converged
        status = GSE_NOT_CONVERGED;
        break;
      }
      level++;
      log_switch(rep, iter, level);
    } else if (ev == EV_MAXITER) {
      status = GSE_NOT_CONVERGED;
      break;
    } else if (ev == EV_ESCALATE) {
      level++;
      log_switch(rep, iter, level);
    }
    rc = set_field(ws, &SolveCtrl::level, level, s);
    if (rc != GSE_OK) return rc;
  }
  rep.iterations = iter;
  rep.converged = (status == GSE_OK);
  double rt = 0;
  rc = true_resid(M, ws->x, bnorm, rep, &rt, s);
  if (rc != GSE_OK) return rc;
  rep.rel_residual_true = rt;
  GSE_CUDA_TRY(cudaMemcpyAsync(x, ws->x, n * 8, cudaMemcpyDeviceToDevice, s));
  GSE_CUDA_TRY(cudaEventRecord(ws->ev1, s));
  GSE_CUDA_TRY(cudaEventSynchronize(ws->ev1));
  float ms = 0;
  cudaEventElapsedTime(&ms, ws->ev0, ws->ev1);
  rep.seconds = ms * 1e-3;
  return status;
}

}  // namespace gse
