/*
 * gse.h -- C-ABI of the B200-native GSE-SEM library (arXiv 2411.04686, "Precision-Aware
 * Iterative Algorithms Based on Group-Shared Exponents of Floating-Point Numbers").
 *
 * Citations: P:n = PAPER.md line n (section / equation / algorithm in brackets), S:n =
 * SPEC.md line n, R<k> = reading k of the DESIGN.md ledger (where the paper is silent).
 *
 * Problem statement (P:29 [section 1]): solve A x = b with CG / GMRES for a sparse A.  The
 * library stores A once in GSE-SEM form -- a table of k shared exponents (P:113-123
 * [section 3.2]), a per-value sign + exponent index (EI) + denormalised significand split
 * into head/tail1/tail2 planes (P:163 [section 3.2.3]), the EI riding in the spare high
 * bits of the CSR column index (P:168 [section 3.3.1]) -- and reads it at 1, 2 or 3
 * segments (P:180-212 [section 3.3.2, Alg. spmv]) inside the stepped mixed-precision
 * solvers (P:217-294 [section 3.4, Alg. stepped-GMRES, Eqs. 3-6]).
 *
 * CONVENTIONS (apply to every entry point)
 *  - Pointers: every array argument may be HOST (pageable or pinned) or DEVICE memory;
 *    the library inspects it (cudaPointerGetAttributes) and stages host arrays through
 *    device buffers on `stream`.  Device arrays must live on the device the matrix lives
 *    on.  Host outputs are complete when the call returns (the call synchronises
 *    `stream`); device outputs are stream-ordered on `stream`.
 *  - stream: a cudaStream_t passed as void* (NULL = the legacy default stream).
 *  - Ownership: the caller owns every array it passes and keeps it alive until the stream
 *    work completes; the library never frees caller memory.  A gse_matrix owns all its
 *    device memory (planes, table, LUT, partition, solver workspaces) until
 *    gse_matrix_free.  A gse_matrix is immutable after creation: concurrent gse_spmv on
 *    different streams is safe; solver calls on one matrix must be
 *    serialised by the caller (they share the matrix's solver workspace).
 *  - Errors: every entry point returns gse_status and never aborts; details of the last
 *    error of the calling thread are in gse_last_error_detail().  Asynchronous kernel
 *    faults surface at the next synchronising call (encode, solvers, host-pointer calls).
 */
#ifndef GSE_H
#define GSE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSE_VERSION_MAJOR 0
#define GSE_VERSION_MINOR 1

typedef enum {
  GSE_OK = 0,
  GSE_NOT_CONVERGED = 2,          /* max iterations reached; report valid (S:413 exit 2)   */
  GSE_NUMERICAL_ABORT = 3,        /* CG breakdown p.Ap <= 0 or non-finite residual */
  GSE_ERR_INVALID_ARG = 10,       /* bad segments/k_max/tol<=0/schedule/CSR structure      */
  GSE_ERR_DIM_MISMATCH = 11,      /* non-square matrix for a solver, wrong slice sizes     */
  GSE_ERR_NONFINITE = 12,         /* NaN/Inf value in the input matrix       */
  GSE_ERR_NO_VALUES = 13,         /* no normal non-zero value: empty histogram      */
  GSE_ERR_UNREPRESENTABLE = 14,   /* reserved: caller table without an entry > e    */
  GSE_ERR_INVALID_EXP_INDEX = 15, /* reserved: EI >= table length                   */
  GSE_ERR_FP32_RANGE = 16,        /* FP32 accumulation asked but table exceeds FP32 (R20)  */
  GSE_ERR_WRONG_FORMAT = 17,      /* operation not defined for this matrix kind            */
  GSE_ERR_CUDA = 20,
  GSE_ERR_NCCL = 21,
  GSE_ERR_OOM = 22
} gse_status;

typedef struct gse_matrix_s* gse_matrix; /* opaque; owns its device memory   */
typedef struct gse_dist_s* gse_dist;     /* opaque; owns its NCCL communicator */

/* Plain FP64 CSR input: 0-based, rows sorted by column, no duplicates,
 * row_ptr[0] = 0, row_ptr[rows] = nnz.  row_ptr is int32 (row_ptr_64 = 0) or int64. */
typedef struct {
  int64_t rows, cols, nnz;
  const void* row_ptr;
  int row_ptr_64;
  const int32_t* col_idx;
  const double* values;
} gse_csr_f64;

typedef struct {
  int k_max;      /* number of shared exponents k: power of two in [1, 64]; default 8 */
  int device;     /* CUDA device ordinal for the matrix; -1 = infer from device pointers, else 0 */
  int64_t sample_block_rows; /* 0: table from the full exponent histogram; B >= 1: from one
                              * random row per block of B rows ("calculated using
                              * sampling techniques"; NEXT-3), the max-exponent rule
                              * still on the true maximum of all values (so every value stays
                              * representable).  Single-GPU gse_encode only.                */
  uint64_t seed;             /* sampling: row of block b = b*B + splitmix64(seed, b+1) mod
                              * len_b (R27: SplitMix64 output for counter b+1)              */
  int per_shard_table;       /* gse_encode_dist only: 0 = one GLOBAL table from the
                              * allreduced histogram (R21, default); 1 = each rank selects
                              * its own table from its rows' histogram (the paper's "group"
                              * read as the row block): no histogram
                              * allreduce, rank-local decode constants.  Ignored by
                              * gse_encode.                                                */
} gse_encode_opts;

typedef enum {
  GSE_KIND_GSE = 0,  /* GSE-SEM planes (gse_encode)                                      */
  GSE_KIND_FP64 = 1, /* plain FP64 CSR (gse_fp64_matrix)                                 */
  GSE_KIND_FP16 = 2, /* FP16 storage baseline (gse_half_matrix)                   */
  GSE_KIND_BF16 = 3  /* BF16 storage baseline (gse_half_matrix)                   */
} gse_matrix_kind;

typedef struct {
  int kind;          /* gse_matrix_kind                                                     */
  int k_max, ei_bits, ei_in_column, table_len;
  uint16_t table[64]; /* stored exponents E = e + 1, EI order (R4-R5)                 */
  int64_t rows, cols, nnz;
  int64_t n_blocks;   /* SpMV row blocks                           */
  int64_t n_zero_values; /* zero / subnormal inputs encoded as signed zero (R2)              */
  int device;
  size_t plane_bytes[5]; /* col_ei, head, tail1, tail2, side_ei (kind GSE); col, val (FP64);
                          col, 16-bit codes (FP16 / BF16)                                 */
  int spmv_mode;      /* SpMV kernel chosen at encode: 1 = row walk, 2 = x window (0 = warp blocks, A/B only) */
} gse_matrix_info;

/* ---------------------------------------------------------------------------------------
 * gse_encode -- build the GSE-SEM form of A (steps a1-a3 of SURVEY 8(a)).
 *   a1 histogram of biased exponents over all values (P:116 [3.2.1]; zero/subnormal counted
 *      apart; first NaN/Inf reported as GSE_ERR_NONFINITE with "(row, col)" in the detail);
 *   a2 table: the k_max most frequent exponents, ties to the larger exponent, e_max forced
 *      into the last slot, entries e+1 (P:116, P:123 [3.2.1-3.2.2]; R4, R5);
 *   a3 per value: nearest entry E > e, d = E - e, D = 1<<(63-d) | f shifted by 11-d
 *      (truncation), split into head 16 b / tail1 16 b / tail2 32 b; EI embedded in the top
 *      log2(k_max) bits of the column index iff cols < 2^(32-ei_bits), else a uint8 side
 *      array (Alg. formatConvert P:128-160 generalised to 64 bits; R1-R3, R6).
 * Output planes are bit-identical to the oracle (tests/test_gpu_parity.py).
 * Errors: INVALID_ARG (structure: row_ptr not monotone, col out of range, k_max),
 * NONFINITE, NO_VALUES, OOM, CUDA.  Synchronises `stream` (reads back the table).
 * ------------------------------------------------------------------------------------- */
gse_status gse_encode(const gse_csr_f64* A, const gse_encode_opts* opts, gse_matrix* out,
                      void* stream);

/* The FP64-CSR comparator matrix (the paper's FP64-SpMV baseline): copies
 * row_ptr/col/values to the device; usable with gse_spmv (segments must be 3) and the
 * solvers with a disabled schedule (fixed FP64). */
gse_status gse_fp64_matrix(const gse_csr_f64* A, int device, gse_matrix* out, void* stream);

/* The FP16 / BF16 storage baselines of the paper's evaluation (P:406 [4.3]: "FP16-SpMV" /
 * "BF16-SpMV" -- values stored in 16 bits, products and sums in FP64; Tables IV-V,
 * P:449-505, for the solvers).  kind = GSE_KIND_FP16 (IEEE binary16) or GSE_KIND_BF16
 * (bfloat16).  Each FP64 value is rounded to nearest, ties to even, directly from the double
 * (R26: the paper does not state the conversion); beyond the largest finite value -> +-Inf
 * (FP16 overflows above 65504: the "/" entries of Tables IV-V), below the smallest
 * subnormal -> signed zero.  The 16-bit codes are stored in the `head` plane (readable with
 * gse_matrix_copy_planes; bit-identical to the oracle), columns in `col_ei` (no EI).  The
 * matrix is read at full precision only (gse_spmv with segments = 3: each code is converted
 * exactly to FP64, multiplied and summed in FP64) and the solvers run it at that one
 * precision (a schedule is accepted but never steps).  Errors as gse_fp64_matrix;
 * NaN inputs are kept as NaN codes (no error: the baseline reproduces the paper's overflow
 * behaviour instead of rejecting it). */
gse_status gse_half_matrix(const gse_csr_f64* A, int kind, int device, gse_matrix* out,
                           void* stream);

gse_status gse_matrix_get_info(gse_matrix A, gse_matrix_info* info);

/* Copy the encoded planes out (any pointer may be NULL to skip): col_ei[nnz] uint32,
 * side_ei[nnz] uint8 (only when !ei_in_column), head[nnz] / tail1[nnz] uint16,
 * tail2[nnz] uint32, table[table_len] uint16.  Host or device destinations.  FP16 / BF16
 * matrices: col_ei (plain columns) and head (the 16-bit codes) only; FP64: col_ei only. */
gse_status gse_matrix_copy_planes(gse_matrix A, uint32_t* col_ei, uint8_t* side_ei,
                                  uint16_t* head, uint16_t* tail1, uint32_t* tail2,
                                  uint16_t* table, void* stream);

/* a4: decode every stored value at `segments` (1, 2, 3) to FP64 (Alg. spmv l.6-17,
 * P:191-201 and P:212; signed zero for a zero significand, R10; flush when the true
 * exponent <= 0, R11).  values[nnz].  Bit-exact with the oracle. */
gse_status gse_decode(gse_matrix A, int segments, double* values, void* stream);

/* ---------------------------------------------------------------------------------------
 * gse_spmv -- a5: y = A_L x with L = segments in {1, 2, 3}: only the requested planes are
 * read, each value decoded on the fly to FP64 and multiplied/accumulated in FP64 ("we load
 * low-precision sparse matrices only during memory access and still perform multiplication
 * and accumulation operations based on double-precision"; Alg. spmv).
 * x[cols], y[rows] FP64.  For a GSE_KIND_FP64 matrix (segments = 3) this is plain CSR
 * SpMV (a6).  Within-row products are summed in storage order for rows up to the short-row
 * limit; the result is within 1e-12 * sum_j |a_ij x_j| of the oracle.
 * ------------------------------------------------------------------------------------- */
gse_status gse_spmv(gse_matrix A, const double* x, double* y, int segments, void* stream);

/* FP32-accumulation variant (BASELINE north_star; R20): x, y float; each decoded value is
 * rounded toward zero to FP32 (FP32-underflow -> 0), multiplied and accumulated in FP32.
 * GSE_ERR_FP32_RANGE if the table can represent values >= 2^128. */
gse_status gse_spmv_f32acc(gse_matrix A, const float* x, float* y, int segments, void* stream);

/* y = A_L x and dot = x . y in ONE launch: the fused SpMV + dot kernel the CG iteration runs
 * (q = A p, p . q).  Single-GPU matrices only (a distributed CG sums
 * its dots with an allreduce).  x[cols], y[rows] FP64 host or device; dot: ONE double, host
 * or device.  The dot is the deterministic fixed-order reduction of per-CTA partials, so
 * repeated calls give bit-identical results.  Uses the matrix's solver workspace: do not
 * run concurrently with a solve or another gse_spmv_dot on the same matrix.
 * GSE_ERR_WRONG_FORMAT for a distributed matrix. */
gse_status gse_spmv_dot(gse_matrix A, const double* x, double* y, int segments, double* dot,
                        void* stream);

/* ---------------------------------------------------------------------------------------
 * Stepped mixed-precision solvers (P:217-294 [3.4]).
 * ------------------------------------------------------------------------------------- */
typedef struct {
  int enabled;                 /* 1: stepped (Alg. stepped-GMRES); 0: fixed start_level     */
  int start_level, max_level;  /* 1..3 (A_1 head, A_2 head+tail1, A_3 full)          */
  int64_t l, t, m;             /* first check at l, window t, period m (t < l in the
                                * paper's settings; t >= l is accepted -- a check also needs a
                                * full window of t + 1 residuals, so the first one waits)     */
  double rsd_limit;            /* Condition 1, Eq. 3                                  */
  int64_t ndec_limit;          /* replaces t/2 in Conditions 1-2 (R13)                */
  double reldec_limit;         /* Condition 2, Eq. 6                                  */
  int verify_at_full;          /* R16: a converged recurrence at L < 3 is checked with A_3   */
  double level_floor[2];       /* R17: escalate when resid < floor[L-1] at L = 1, 2; 0 = off */
  int krylov_gse16;            /* GMRES only, single GPU: 1 = keep the Krylov basis as 16-bit
                                * GSE-SEM vectors (Alg. 1 layout, k = 8: 3 EI bits, 12
                                * significand bits; a table per basis vector; NEXT-4, R28):
                                * the Arnoldi steps and the solution update read the decoded
                                * 16-bit values; 0 = FP64 basis (default)                    */
  double perturb_c;            /* R29 (build reading, single GPU): escalate at L < 3 when the
                                * monitored residual <= perturb_c * eta_L * ||x|| / ||b||,
                                * eta_L = ||A_3 - A_L||_inf (gse_perturbation_bounds): the
                                * residual level below which level-L iterations cannot lower
                                * the true residual.  x = the iterate before the current CG
                                * iteration's update / at the start of the GMRES cycle.
                                * 0 = off (default, the paper's monitor only); must be >= 0 */
  int cg_keep_direction;       /* R30 (build reading, CG, single GPU): at a level switch replace
                                * the residual, r = b - A_new x, but keep the search direction:
                                * beta = r.r / rr_{j-1}, p = r + beta p (a residual-replacement
                                * step instead of the R15 restart p = r); 0 = R15 restart
                                * (default), 1 = keep; GMRES ignores it                       */
} gse_step_schedule;

typedef struct {
  int64_t iterations;          /* CG iterations / GMRES inner iterations (global counter)    */
  int64_t iters_per_level[3];
  int converged, n_switches;
  int64_t switch_iter[2];
  int switch_to_level[2];
  double rel_residual_recurrence; /* last monitored residual (CG recurrence / Givens est.)  */
  double rel_residual_true;       /* ||b - A_3 x|| / ||b|| computed at exit                 */
  double seconds;                 /* device time of the solve (CUDA events)                 */
  int64_t spmv_count[3];          /* SpMVs issued per level (incl. replacement / verify)    */
} gse_solve_report;

/* R29: eta[L-1] = ||A_3 - A_L||_inf = max_i sum_j |dec_3(a_ij) - dec_L(a_ij)|, L = 1, 2
 * (row sums in storage order: bit-identical to the oracle), computed once per matrix and
 * cached.  eta: two doubles, host memory.  Synchronises the stream.  GSE matrices only
 * (GSE_ERR_WRONG_FORMAT otherwise). */
gse_status gse_perturbation_bounds(gse_matrix A, double* eta, void* stream);

/* Paper defaults (P:433, P:441 [4.4.1]): CG l=3000 t=250 m=500 0.50/130/0.45; GMRES
 * l=9000 t=300 m=1500 0.03/80/0.08; enabled, start 1, max 3, verify_at_full 1, floors 0. */
void gse_default_schedule(int solver /* 0 = CG, 1 = GMRES */, gse_step_schedule* out);

/* Unpreconditioned CG with the stepped driver: w = A_tag p each iteration; the
 * monitor (Eqs. 3-6, Conditions 1-3) sees ||r_j||/||b|| after iteration j, checks at
 * j >= l, (j - l) % m == 0, window of t+1 full; one level per trigger (R12); at a switch
 * CG restarts from the current x with r = b - A_new x, p = r (R15), or keeps its direction,
 * p = r + (r.r / rr) p (R30, sched->cg_keep_direction = 1).  b[n], x[n] (in: x0,
 * out: solution); n = rows = cols.  Returns OK (converged), NOT_CONVERGED, NUMERICAL_ABORT
 * or an error; rep may be NULL.  sched NULL = fixed level 3. */
gse_status gse_solve_cg(gse_matrix A, const double* b, double* x, double tol, int64_t max_iters,
                        const gse_step_schedule* sched, gse_solve_report* rep, void* stream);

/* Restarted GMRES(restart) (restart 30, 500 outer): MGS Arnoldi, Givens rotations
 * (R18), estimate |g_{j+1}|/||b|| monitored per inner iteration with a global counter,
 * explicit residual at restarts; a switch ends the cycle (x += V y) and restarts at the
 * new level (R15). */
gse_status gse_solve_gmres(gse_matrix A, const double* b, double* x, double tol, int restart,
                           int64_t max_iters, const gse_step_schedule* sched,
                           gse_solve_report* rep, void* stream);

/* ---------------------------------------------------------------------------------------
 * 16-bit GSE-SEM vectors (Alg. 1: "converting double-precision vector to GSE-SEM
 * vector", in its own 16-bit layout; R28).
 * gse_encode_vector16: table = the k_max most frequent exponents of v (ties to the larger,
 *   e_max forced into the last slot, entries e + 1), then per element
 *   word = sign << 15 | EI << (15 - ei_bits) | significand with its explicit one, truncated
 *   (ei_bits = log2 k_max; zero / subnormal -> signed zero; d > 15 - ei_bits -> signed zero).
 *   v[n] FP64, words[n] uint16 (host or device), table[16] / table_len host outputs.
 *   k_max: power of two in [1, 16].  Bit-identical to the oracle.
 * gse_decode_vector16: |v| = significand * 2^(E_EI - 1023 - (15 - ei_bits)), flush below the
 *   normal range (R11).  out[n] FP64.  INVALID_ARG for bad sizes / ei_bits > 4.
 * ------------------------------------------------------------------------------------- */
gse_status gse_encode_vector16(const double* v, int64_t n, int k_max, uint16_t* words,
                               uint16_t* table, int* table_len, void* stream);
gse_status gse_decode_vector16(const uint16_t* words, int64_t n, const uint16_t* table,
                               int table_len, int ei_bits, double* out, void* stream);

void gse_matrix_free(gse_matrix A);

const char* gse_status_string(gse_status s);
const char* gse_last_error_detail(void);

/* Route library device allocations (planes, workspaces) through a caller allocator, e.g.
 * torch's caching allocator.  NULL alloc restores cudaMallocAsync / cudaFreeAsync.  The
 * allocator must return 256-byte aligned device memory (cudaMalloc's guarantee: the SpMV
 * kernels stage planes with TMA bulk copies); a misaligned block is handed back to free_
 * and the calling entry point fails with GSE_ERR_OOM and a detail message.  A size may be
 * rounded up to a multiple of 256 bytes. */
gse_status gse_set_allocator(void* (*alloc)(size_t bytes, void* stream, void* ctx),
                             void (*free_)(void* ptr, void* stream, void* ctx), void* ctx);

/* ---------------------------------------------------------------------------------------
 * Multi-GPU, one process per GPU: contiguous row blocks; a rank holds rows
 * [row_begin, row_begin + local_rows) with GLOBAL column ids; the table is global
 * (histogram allreduce, R21); columns are renumbered locally (owned first, halo after).
 * b, x, y are the rank's row slices.  gse_spmv / gse_solve_* on a distributed matrix
 * exchange the halo and allreduce dot products over NCCL.
 * ------------------------------------------------------------------------------------- */
gse_status gse_nccl_unique_id(void* id128 /* host, 128 bytes */);
/* NCCL backend: one process per GPU; rank 0 creates the unique id, the caller broadcasts
 * it (e.g. torch.distributed), every rank calls this collectively.  nranks <= 16. */
gse_status gse_dist_create(const void* nccl_unique_id /* host, 128 B */, int rank, int nranks,
                           int device, gse_dist* out);
/* Thread backend: nranks host threads of ONE process (one GPU or several), collectives by
 * device copies + events + host barriers.  Runs the same distributed code path as NCCL and
 * is how the multi-rank path is tested on a single GPU.  Create the group once, then each
 * thread calls gse_dist_create_thread with its rank; all collective calls must be made by
 * all threads in the same order. */
gse_status gse_dist_thread_group_create(int nranks, void** group);
void gse_dist_thread_group_free(void* group);
gse_status gse_dist_create_thread(void* group, int rank, int device, gse_dist* out);
/* Collective over the ranks of D: encode this rank's row block.  local_rows holds rows
 * [row_begin, row_begin + local_rows->rows) of a square global_rows x global_rows matrix
 * with GLOBAL column ids (host or device arrays); ranks own contiguous blocks in rank order.
 * The exponent histogram is summed over ranks before the table is chosen, so all ranks
 * share one table (R21); columns are renumbered locally (owned first, then the halo in
 * global order).  gse_spmv on the result takes / returns the rank's slices (x: local_rows
 * entries); gse_solve_cg runs the distributed CG (halo exchange + two allreduces per
 * iteration); gse_solve_gmres the distributed GMRES(m) (halo exchange per SpMV, one
 * allreduce per MGS dot and per norm: j + 2 per inner step, MGS order kept).  FP32
 * accumulation is single-GPU only (GSE_ERR_WRONG_FORMAT). */
gse_status gse_encode_dist(gse_dist D, const gse_csr_f64* local_rows, int64_t row_begin,
                           int64_t global_rows, const gse_encode_opts* opts, gse_matrix* out,
                           void* stream);
void gse_dist_free(gse_dist D);
/* Host-only planning helper (no GPU, no communicator): the local renumbering used by
 * gse_encode_dist.  col[nnz] global ids of a rank owning rows [row_begin, row_begin+n_local);
 * rank_rows[nranks+1] = row offsets of all ranks.  Outputs: local_col[nnz] (owned -> col -
 * row_begin, halo -> n_local + position in halo_cols), *n_halo, halo_cols[<= nnz] (sorted
 * unique non-owned ids; may be NULL), recv_count[nranks] (halo entries owned by each rank;
 * may be NULL). */
gse_status gse_dist_plan(int64_t nnz, const int32_t* col, int64_t row_begin, int64_t n_local,
                         int nranks, const int64_t* rank_rows, int32_t* local_col,
                         int64_t* n_halo, int64_t* halo_cols, int64_t* recv_count);

#ifdef __cplusplus
}
#endif
#endif /* GSE_H */
