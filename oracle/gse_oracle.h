/*
 * gse_oracle.h -- ORACLE: plain, slow, CPU-only reference of the GSE-SEM method
 * (arXiv 2411.04686).  TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this code.  It shares
 * no code, header, table or constant generator with the CUDA library under
 * paper_2411_04686_b200/ (which has its own header include/gse.h).
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
 */
#ifndef GSE_ORACLE_H
#define GSE_ORACLE_H
#include <stdint.h>

#define ORC_OK 0
#define ORC_NOT_CONVERGED 2
#define ORC_NUMERICAL_ABORT 3
#define ORC_ERR_INVALID_ARG 10
#define ORC_ERR_DIM 11
#define ORC_ERR_NONFINITE 12
#define ORC_ERR_NO_VALUES 13
#define ORC_ERR_UNREPRESENTABLE 14
#define ORC_ERR_INVALID_EXP_INDEX 15

/* ---- codec (Alg. 1) ---- */
int orc_exponent_histogram(int64_t nnz, const double* val, uint64_t* hist2048,
                           int64_t* n_zero, int64_t* first_nonfinite);
int orc_build_table(const uint64_t* hist2048, int k_max, uint16_t* table, int* table_len);
int orc_build_table_emax(const uint64_t* hist2048, int k_max, int e_max_true, uint16_t* table,
                         int* table_len);
uint64_t orc_sample_z(uint64_t seed, int64_t b);
int64_t orc_sample_row(int64_t rows, int64_t block_rows, uint64_t seed, int64_t b);
int orc_sampled_histogram(int64_t rows, const int64_t* row_ptr, const double* val,
                          int64_t block_rows, uint64_t seed, uint64_t* hist2048);
int orc_encode_value(double x, const uint16_t* table, int table_len, uint64_t* word, int* ei);
void orc_segment(uint64_t word, uint16_t* head, uint16_t* tail1, uint32_t* tail2);
uint64_t orc_assemble(uint16_t head, uint16_t tail1, uint32_t tail2, int level);
int orc_decode(uint64_t word, int ei, const uint16_t* table, int table_len, double* out);
int orc_encode_head16_with_ei(double x, const uint16_t* table, int table_len, int ei_bits,
                              uint16_t* out);
int orc_decode_head16_with_ei(uint16_t w, const uint16_t* table, int table_len, int ei_bits,
                              double* out);
int orc_encode_vector16(int64_t n, const double* v, int k_max, uint16_t* words, uint16_t* table,
                        int* table_len);
int orc_decode_vector16(int64_t n, const uint16_t* words, const uint16_t* table, int table_len,
                        int ei_bits, double* out);

/* ---- CSR conversion ---- */
int orc_encode_csr(int64_t rows, int64_t cols, int64_t nnz, const int64_t* row_ptr,
                   const int32_t* col, const double* val, int k_max,
                   uint16_t* table /* k_max */, int* table_len, int* ei_bits, int* ei_in_column,
                   uint32_t* col_ei, uint8_t* side_ei, uint16_t* head, uint16_t* tail1,
                   uint32_t* tail2, int64_t* bad_index);
int orc_encode_csr_sampled(int64_t rows, int64_t cols, int64_t nnz, const int64_t* row_ptr,
                           const int32_t* col, const double* val, int k_max,
                           int64_t sample_block_rows, uint64_t seed, uint16_t* table,
                           int* table_len, int* ei_bits_out, int* ei_in_column,
                           uint32_t* col_ei, uint8_t* side_ei, uint16_t* head,
                           uint16_t* tail1, uint32_t* tail2, int64_t* bad_index);

/* matrix as seen by the oracle solvers: either plain FP64 CSR (val != NULL) or GSE */
typedef struct {
  int64_t rows, cols;
  const int64_t* row_ptr;
  const int32_t* col;   /* FP64 mode */
  const double* val;    /* FP64 mode; NULL => GSE mode */
  const uint32_t* col_ei;
  const uint8_t* side_ei;
  int ei_bits, ei_in_column;
  const uint16_t* head;
  const uint16_t* tail1;
  const uint32_t* tail2;
  const uint16_t* table;
  int table_len;
  int half_kind;        /* 0: not a 16-bit baseline; ORC_FP16 / ORC_BF16: values in half[] */
  const uint16_t* half; /* with col[]: the FP16 / BF16 storage baseline       */
} orc_matrix;

/* ---- SpMV (Alg. 2) ---- */
int orc_spmv_fp64(int64_t rows, const int64_t* row_ptr, const int32_t* col, const double* val,
                  const double* x, double* y);
int orc_spmv_gse(const orc_matrix* A, int level, const double* x, double* y);
int orc_apply(const orc_matrix* A, int level, const double* x, double* y);

/* ---- FP16 / BF16 storage baselines (P:406 [4.3]; R26) ----
 * values rounded FP64 -> 16 bit with round-to-nearest-even (overflow -> +-Inf), stored,
 * converted back to FP64 exactly and multiplied by the FP64 vector, FP64 accumulation. */
#define ORC_FP16 1
#define ORC_BF16 2
uint16_t orc_round_half(double v, int kind);
double orc_half_value(uint16_t h, int kind);
int orc_spmv_half(const orc_matrix* A, const double* x, double* y);
void orc_round_half_array(int64_t n, const double* v, uint16_t* out, int kind);
void orc_half_value_array(int64_t n, const uint16_t* h, double* out, int kind);

/* ---- residual monitor (Eqs. 3-6) ---- */
double orc_rsd(const double* w, int64_t t);
int64_t orc_ndec(const double* w, int64_t t);
double orc_reldec(const double* w, int64_t t);
int orc_should_escalate(const double* w, int64_t t, double rsd_limit, int64_t ndec_limit,
                        double reldec_limit);

typedef struct {
  int enabled, start_level, max_level;
  int64_t l, t, m;
  double rsd_limit;
  int64_t ndec_limit;
  double reldec_limit;
  int verify_at_full;
  double level_floor[2];
  int krylov_gse16; /* GMRES: Krylov basis stored as 16-bit GSE-SEM vectors (NEXT-4, R28) */
  double perturb_c; /* R29: escalate at L < 3 when resid <= c * eta_L * ||x|| / ||b||; 0 = off */
  int cg_keep_direction; /* R30: CG switch keeps p (r = b - A_new x, p = r + beta p); 0 = R15 */
} orc_schedule;

typedef struct {
  int64_t iterations, iters_per_level[3];
  int converged, n_switches;
  int64_t switch_iter[2];
  int switch_to_level[2];
  double rel_residual_recurrence, rel_residual_true;
  int64_t spmv_count[3];
} orc_report;

void orc_default_schedule(int solver, orc_schedule* s);

/* R29: eta[L-1] = max_i sum_j |dec_3(a_ij) - dec_L(a_ij)| (= ||A_3 - A_L||_inf) for
 * L = 1, 2; row sums in storage order.  GSE matrices only. */
int orc_perturbation_bounds(const orc_matrix* A, double eta[2]);

/* ---- solvers ---- */
int orc_cg(const orc_matrix* A, const double* b, double* x, double tol, int64_t max_iters,
           const orc_schedule* sched, orc_report* rep);
int orc_gmres(const orc_matrix* A, const double* b, double* x, double tol, int restart,
              int64_t max_iters, const orc_schedule* sched, orc_report* rep);
/* c.1 step 10 partitioned mode: P simulated ranks own rows [bounds[r], bounds[r+1])
 * (bounds[0] = 0, bounds[P] = rows, non-decreasing); dots summed per rank, then in rank
 * order.  ORC_ERR_INVALID_ARG for bad bounds. */
int orc_cg_part(const orc_matrix* A, const double* b, double* x, double tol, int64_t max_iters,
                const orc_schedule* sched, int P, const int64_t* bounds, orc_report* rep);
int orc_gmres_part(const orc_matrix* A, const double* b, double* x, double tol, int restart,
                   int64_t max_iters, const orc_schedule* sched, int P, const int64_t* bounds,
                   orc_report* rep);

/* cost of the oracle's plain threads knob (GSE_THREADS); returns threads used */
int orc_set_threads(int n);
#endif
