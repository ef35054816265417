/*
 * gse_oracle.c -- ORACLE for the GSE-SEM hot path of arXiv 2411.04686.
 *
 *   TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 *   cpu_baseline / `--impl reference` legs may load or execute this file.  The product
 *   (paper_2411_04686_b200/, include/gse.h) never links it, and this file shares no
 *   code, header, table or constant generator with it.
 *
 * Plain, slow, obviously correct C99.  All floating point is IEEE binary64 with
 * separate multiply and add (compiled with -ffp-contract=off, no fast-math), vectors
 * reduced sequentially in index order.  Each function cites the passage it follows:
 * P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n, and "R<k>" = reading k
 * of the DESIGN.md ledger where the paper is silent/ambiguous.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): worked examples of S:60-105, S:162-173,
 * S:268-278; closed forms (|v| = D_L * 2^(E-1086), bit-exact round trip for
 * d <= 11, Poisson head-exactness); brute-force dense matvec; dense direct solves;
 * literal transcriptions of Alg. 1 / Alg. 2 in the tests; scipy CG / GMRES(30) iteration
 * gauges; the R29 bound eta_L against a closed form; the R30 kept-direction switch against
 * an independent numpy CG and, on a head-exact matrix with forced switches, against the
 * fixed-level CG's iteration count (a pure residual replacement leaves CG unchanged); the
 * partitioned mode (c.1 step 10, orc_cg_part / orc_gmres_part) against an independent numpy
 * CG with per-rank sequential dots summed in rank order (identical iterations and switches).
 *
 * Parity unpinned by the paper (pinned only by agreement with this file under the DESIGN.md
 * readings): FP32 accumulation (R20), the level floors (R17), verify-at-full (R16, R16b),
 * the CG restart at a switch (R15), the R29 trigger's constant c.
 */
#include "gse_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static uint64_t bits_of(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static double double_of(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }

int orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

/* ------------------------------------------------------------------------------------
 * c.1 step 1 -- exponent histogram.  P:116 "we first count the occurrences N_i for each
 * distinct exponent e_i".  Biased exponent e in [1,2046] counted; e = 0
 * (zero / subnormal) counted separately; e = 2047 (NaN/Inf) is an error.
 * ------------------------------------------------------------------------------------ */
int orc_exponent_histogram(int64_t nnz, const double* val, uint64_t* hist, int64_t* n_zero,
                           int64_t* first_nonfinite) {
  memset(hist, 0, 2048 * sizeof(uint64_t));
  *n_zero = 0;
  *first_nonfinite = -1;
  for (int64_t i = 0; i < nnz; ++i) {
    unsigned e = (unsigned)((bits_of(val[i]) >> 52) & 0x7FF);
    if (e == 0x7FF) {
      if (*first_nonfinite < 0) *first_nonfinite = i;
    } else if (e == 0) {
      *n_zero += 1;
    } else {
      hist[e] += 1;
    }
  }
  return *first_nonfinite >= 0 ? ORC_ERR_NONFINITE : ORC_OK;
}

/* ------------------------------------------------------------------------------------
 * c.1 step 2 -- shared-exponent table.  P:116 "the exponents are sorted in descending
 * order based on their occurrence counts to identify the k most frequent exponents";
 * P:123 "we increment all the shared exponents by 1 ... one of the shared exponents must
 * be the maximum exponent of all non-zeros plus one".  Ties: larger exponent first (R4,
 * S:57); e_max forced into the LAST (least frequent) slot if not selected (R5).
 * ------------------------------------------------------------------------------------ */
static const uint64_t* g_sort_hist;
static int cmp_count_desc_e_desc(const void* a, const void* b) {
  int ea = *(const int*)a, eb = *(const int*)b;
  uint64_t ca = g_sort_hist[ea], cb = g_sort_hist[eb];
  if (ca != cb) return ca > cb ? -1 : 1;
  return ea > eb ? -1 : (ea < eb ? 1 : 0);
}

/* e_max_true >= 1: the exponent the max-exponent rule must cover (the TRUE maximum of all
 * values when hist is a sample); 0: the largest exponent in hist. */
int orc_build_table_emax(const uint64_t* hist, int k_max, int e_max_true, uint16_t* table,
                         int* table_len) {
  int es[2048];
  int n = 0, e_max = 0;
  if (k_max < 1 || k_max > 64 || (k_max & (k_max - 1)) != 0) return ORC_ERR_INVALID_ARG;
  for (int e = 1; e <= 2046; ++e) {
    if (hist[e] > 0) {
      es[n++] = e;
      e_max = e;
    }
  }
  if (e_max_true > 0) e_max = e_max_true;
  if (n == 0 && e_max == 0) return ORC_ERR_NO_VALUES; /* S:58 "no representable values" */
  if (n == 0) { /* a sample without normal values: the forced entry alone */
    table[0] = (uint16_t)(e_max + 1);
    *table_len = 1;
    return ORC_OK;
  }
  g_sort_hist = hist;
  qsort(es, (size_t)n, sizeof(int), cmp_count_desc_e_desc);
  int take = n < k_max ? n : k_max;
  int have_max = 0;
  for (int i = 0; i < take; ++i) have_max |= (es[i] == e_max);
  /* R27b: a free slot (fewer than k_max sampled exponents) takes e_max; otherwise it
   * replaces the least frequent selected entry (R5) */
  if (!have_max) {
    if (take < k_max)
      es[take++] = e_max;
    else
      es[take - 1] = e_max;
  }
  for (int i = 0; i < take; ++i) table[i] = (uint16_t)(es[i] + 1);
  *table_len = take;
  return ORC_OK;
}

int orc_build_table(const uint64_t* hist, int k_max, uint16_t* table, int* table_len) {
  return orc_build_table_emax(hist, k_max, 0, table, table_len);
}

/* ------------------------------------------------------------------------------------
 * NEXT-3 -- sampled table extraction.  P:116 "the shared exponents can be calculated using
 * sampling techniques. For instance, a sparse matrix is divided into several row blocks,
 * and the exponents' distribution in a random row is calculated for each row block,
 * serving as the exponents' distribution in that block"; one uniformly chosen
 * row per contiguous block of block_rows rows, histogram fed to the table selection, the
 * max-exponent rule on the TRUE global maximum (full scan), so every value stays
 * representable.  The random row (R27; the paper names no generator): block b covers rows
 * [b*B, min((b+1)*B, rows)) of length len_b, and its row is b*B + (z mod len_b) with z the
 * SplitMix64 output for counter (b + 1) from the seed:
 *   z = seed + (b + 1) * 0x9E3779B97F4A7C15;
 *   z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9;  z = (z ^ (z >> 27)) * 0x94D049BB133111EB;
 *   z = z ^ (z >> 31)   (all mod 2^64).
 * ------------------------------------------------------------------------------------ */
uint64_t orc_sample_z(uint64_t seed, int64_t b) {
  uint64_t z = seed + (uint64_t)(b + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int64_t orc_sample_row(int64_t rows, int64_t block_rows, uint64_t seed, int64_t b) {
  int64_t r0 = b * block_rows;
  int64_t len = rows - r0 < block_rows ? rows - r0 : block_rows;
  return r0 + (int64_t)(orc_sample_z(seed, b) % (uint64_t)len);
}

/* histogram of the sampled rows' values (zero / subnormal / non-finite not counted) */
int orc_sampled_histogram(int64_t rows, const int64_t* row_ptr, const double* val,
                          int64_t block_rows, uint64_t seed, uint64_t* hist) {
  if (block_rows < 1) return ORC_ERR_INVALID_ARG;
  memset(hist, 0, 2048 * sizeof(uint64_t));
  int64_t nblocks = (rows + block_rows - 1) / block_rows;
  for (int64_t b = 0; b < nblocks; ++b) {
    int64_t r = orc_sample_row(rows, block_rows, seed, b);
    for (int64_t j = row_ptr[r]; j < row_ptr[r + 1]; ++j) {
      unsigned e = (unsigned)((bits_of(val[j]) >> 52) & 0x7FF);
      if (e >= 1 && e <= 2046) hist[e] += 1;
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------
 * c.1 step 3 -- encode one value to the 64-bit SEM word.  Alg. 1 generalised
 * to a 64-bit SEM with the EI kept outside the word:
 *   l.3-4 sign and exponent; l.6-21 nearest shared exponent E > e, d = minDiff = E - e;
 *   l.23-25 denormalise: explicit one at bit 63-d, fraction shifted by (11-d)
 *   (truncation, R1); zero/subnormal -> signed zero, EI 0 (R2); d > 63 -> signed zero
 *   (R3).
 * ------------------------------------------------------------------------------------ */
int orc_encode_value(double x, const uint16_t* table, int table_len, uint64_t* word, int* ei) {
  uint64_t u = bits_of(x);
  uint64_t s = u >> 63;
  int e = (int)((u >> 52) & 0x7FF);
  uint64_t f = u & ((1ULL << 52) - 1);
  if (e == 0x7FF) return ORC_ERR_NONFINITE;
  if (e == 0) {
    *word = s << 63;
    *ei = 0;
    return ORC_OK;
  }
  int best = -1, dbest = 1 << 30;
  for (int i = 0; i < table_len; ++i) {
    int d = (int)table[i] - e;
    if (d >= 1 && d < dbest) {
      dbest = d;
      best = i;
    }
  }
  if (best < 0) return ORC_ERR_UNREPRESENTABLE;
  *ei = best;
  if (dbest > 63) {
    *word = s << 63;
    return ORC_OK;
  }
  uint64_t D = 1ULL << (63 - dbest);
  if (dbest <= 11)
    D |= f << (11 - dbest);
  else
    D |= f >> (dbest - 11);
  *word = (s << 63) | D;
  return ORC_OK;
}

/* c.1 step 4 -- segmentation.  P:163 "the first segment contains the most significant 16
 * bits ... the top 16 bits form the second segment called tail1, and the remaining least
 * significant bits form the third segment called tail2". */
void orc_segment(uint64_t w, uint16_t* head, uint16_t* tail1, uint32_t* tail2) {
  *head = (uint16_t)(w >> 48);
  *tail1 = (uint16_t)((w >> 32) & 0xFFFF);
  *tail2 = (uint32_t)(w & 0xFFFFFFFFULL);
}

/* P:212 "the head can be concatenated with tail1 or with tail1 and tail2"; absent low
 * segments are zero. */
uint64_t orc_assemble(uint16_t head, uint16_t tail1, uint32_t tail2, int level) {
  uint64_t w = (uint64_t)head << 48;
  if (level >= 2) w |= (uint64_t)tail1 << 32;
  if (level >= 3) w |= (uint64_t)tail2;
  return w;
}

/* ------------------------------------------------------------------------------------
 * c.1 step 5 -- decode.  Alg. 2 l.6-17: sign to bit 63; find the first one
 * below the sign ("__fns(val, 14, -1)", R7); exponent = expArr[EI] - (distance of that
 * one from bit 63) (R8); fraction = bits below the one, realigned to 52 bits (truncating);
 * no one found -> zero (sign kept, R10); exponent <= 0 -> signed zero (R11).
 * ------------------------------------------------------------------------------------ */
int orc_decode(uint64_t w, int ei, const uint16_t* table, int table_len, double* out) {
  if (ei < 0 || ei >= table_len) return ORC_ERR_INVALID_EXP_INDEX;
  uint64_t s = w >> 63;
  uint64_t D = w & 0x7FFFFFFFFFFFFFFFULL;
  if (D == 0) {
    *out = double_of(s << 63);
    return ORC_OK;
  }
  int pos = 62;
  while (((D >> pos) & 1ULL) == 0) --pos;
  int d = 63 - pos;
  int eb = (int)table[ei] - d;
  if (eb <= 0) {
    *out = double_of(s << 63);
    return ORC_OK;
  }
  uint64_t F = D & ((1ULL << pos) - 1);
  if (pos >= 52)
    F >>= (pos - 52);
  else
    F <<= (52 - pos);
  *out = double_of((s << 63) | ((uint64_t)eb << 52) | F);
  return ORC_OK;
}

/* Alg. 1's literal 16-bit output layout: bit 15 sign, bits 14..15-ei_bits the
 * EI, then the denormalised significand with its explicit one at bit 15-ei_bits-d
 * (P:152-156); d > 15-ei_bits flushes to signed zero (R3). */
int orc_encode_head16_with_ei(double x, const uint16_t* table, int table_len, int ei_bits,
                              uint16_t* out) {
  uint64_t word;
  int ei;
  int st = orc_encode_value(x, table, table_len, &word, &ei);
  if (st != ORC_OK) return st;
  uint16_t sign = (uint16_t)((word >> 63) << 15);
  uint64_t D = word & 0x7FFFFFFFFFFFFFFFULL;
  if (D == 0) {
    *out = sign;
    return ORC_OK;
  }
  int pos = 62;
  while (((D >> pos) & 1ULL) == 0) --pos;
  int d = 63 - pos;
  int mbits = 15 - ei_bits; /* bits below the EI field */
  if (d > mbits) {
    *out = sign;
    return ORC_OK;
  }
  /* keep the top (mbits - d + 1) significand bits: explicit one lands at bit mbits-d */
  uint16_t mant = (uint16_t)(D >> (63 - mbits));
  *out = (uint16_t)(sign | (uint16_t)(ei << mbits) | mant);
  return ORC_OK;
}

/* Inverse of the 16-bit SEM word of Alg. 1 (EI inside the word): sign = bit 15, EI = the
 * ei_bits below it, significand = the remaining mbits = 15 - ei_bits bits with its explicit
 * one (Alg. 2's reading, applied to the Alg. 1 layout).  Closed form of the
 * value (R28): |v| = mant * 2^(E_EI - 1023 - mbits), E_EI the stored (e+1) entry; mant = 0
 * -> signed zero (R10); a result below the normal range -> signed zero (R11). */
int orc_decode_head16_with_ei(uint16_t w, const uint16_t* table, int table_len, int ei_bits,
                              double* out) {
  const int mbits = 15 - ei_bits;
  const int sign = (w >> 15) & 1;
  const int ei = (w >> mbits) & ((1 << ei_bits) - 1);
  const unsigned mant = w & ((1u << mbits) - 1u);
  if (ei >= table_len && mant) return ORC_ERR_INVALID_EXP_INDEX;
  double v = 0.0;
  if (mant) {
    v = ldexp((double)mant, (int)table[ei] - 1023 - mbits);
    if (v < 2.2250738585072014e-308) v = 0.0; /* below the normal range: flush (R11) */
  }
  *out = sign ? -v : v;
  return ORC_OK;
}

/* NEXT-4 -- a vector in 16-bit GSE-SEM form (Alg. 1, verbatim layout): the
 * table from the vector's own exponent histogram (top k_max, e_max forced),
 * each element encoded by Alg. 1 into sign | EI | denormalised significand.  Returns the
 * table (<= 64 entries) and the words; an all-zero vector gives table_len 0, words = signs. */
int orc_encode_vector16(int64_t n, const double* v, int k_max, uint16_t* words, uint16_t* table,
                        int* table_len) {
  uint64_t* hist = (uint64_t*)malloc(2048 * sizeof(uint64_t));
  int64_t nz, bad;
  int st = orc_exponent_histogram(n, v, hist, &nz, &bad);
  if (st != ORC_OK) { free(hist); return st; }
  int eb = 0;
  while ((1 << eb) < k_max) ++eb;
  st = orc_build_table(hist, k_max, table, table_len);
  free(hist);
  if (st == ORC_ERR_NO_VALUES) { /* all zero / subnormal */
    *table_len = 0;
    for (int64_t i = 0; i < n; ++i) words[i] = (uint16_t)((bits_of(v[i]) >> 63) << 15);
    return ORC_OK;
  }
  if (st != ORC_OK) return st;
  for (int64_t i = 0; i < n; ++i) {
    st = orc_encode_head16_with_ei(v[i], table, *table_len, eb, &words[i]);
    if (st != ORC_OK) return st;
  }
  return ORC_OK;
}

int orc_decode_vector16(int64_t n, const uint16_t* words, const uint16_t* table, int table_len,
                        int ei_bits, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    int st = orc_decode_head16_with_ei(words[i], table, table_len, ei_bits, &out[i]);
    if (st != ORC_OK) return st;
  }
  return ORC_OK;
}

/* v <- dec16(enc16(v)): the value a Krylov vector takes when stored in 16-bit GSE form
 * (k = 8: 3 EI bits, 12 significand bits) -- every later use reads these values */
static void compress16(int64_t n, double* v) {
  uint16_t* w = (uint16_t*)malloc((size_t)(n ? n : 1) * sizeof(uint16_t));
  uint16_t table[64];
  int tl = 0;
  if (orc_encode_vector16(n, v, 8, w, table, &tl) == ORC_OK)
    orc_decode_vector16(n, w, table, tl, 3, v);
  free(w);
}

/* ------------------------------------------------------------------------------------
 * CSR conversion.  P:168 "the indices of shared exponents can be encoded into the column
 * indices of non-zeros ... When the column size of a sparse matrix is so large that there
 * are not enough binary bits ... we can encode them into the value array"; Alg. 2 l.3-5
 * (expIdx = col >> 29 for 3 EI bits).  ei_bits = log2(k_max) (R6); EI embedded iff
 * cols < 2^(32-ei_bits), else a side array.
 * ------------------------------------------------------------------------------------ */
int orc_encode_csr(int64_t rows, int64_t cols, int64_t nnz, const int64_t* row_ptr,
                   const int32_t* col, const double* val, int k_max, uint16_t* table,
                   int* table_len, int* ei_bits_out, int* ei_in_column, uint32_t* col_ei,
                   uint8_t* side_ei, uint16_t* head, uint16_t* tail1, uint32_t* tail2,
                   int64_t* bad_index) {
  return orc_encode_csr_sampled(rows, cols, nnz, row_ptr, col, val, k_max, 0, 0, table,
                                table_len, ei_bits_out, ei_in_column, col_ei, side_ei, head,
                                tail1, tail2, bad_index);
}

/* sample_block_rows = 0: full histogram; >= 1: the sampled table of NEXT-3 (above) */
int orc_encode_csr_sampled(int64_t rows, int64_t cols, int64_t nnz, const int64_t* row_ptr,
                           const int32_t* col, const double* val, int k_max,
                           int64_t sample_block_rows, uint64_t seed, uint16_t* table,
                           int* table_len, int* ei_bits_out, int* ei_in_column,
                           uint32_t* col_ei, uint8_t* side_ei, uint16_t* head,
                           uint16_t* tail1, uint32_t* tail2, int64_t* bad_index) {
  *bad_index = -1;
  if (rows < 0 || cols < 0 || nnz < 0) return ORC_ERR_INVALID_ARG;
  if (row_ptr[0] != 0 || row_ptr[rows] != nnz) return ORC_ERR_INVALID_ARG;
  for (int64_t r = 0; r < rows; ++r)
    if (row_ptr[r + 1] < row_ptr[r]) return ORC_ERR_INVALID_ARG;
  for (int64_t i = 0; i < nnz; ++i)
    if (col[i] < 0 || (int64_t)col[i] >= cols) {
      *bad_index = i;
      return ORC_ERR_INVALID_ARG;
    }
  uint64_t* hist = (uint64_t*)malloc(2048 * sizeof(uint64_t));
  int64_t nz, bad;
  int st = orc_exponent_histogram(nnz, val, hist, &nz, &bad);
  if (st != ORC_OK) {
    *bad_index = bad;
    free(hist);
    return st;
  }
  if (sample_block_rows > 0 && rows > 0) {
    int e_max_true = 0; /* true maximum from the full histogram */
    for (int e = 1; e <= 2046; ++e)
      if (hist[e] > 0) e_max_true = e;
    if (e_max_true == 0) {
      free(hist);
      return ORC_ERR_NO_VALUES;
    }
    orc_sampled_histogram(rows, row_ptr, val, sample_block_rows, seed, hist);
    st = orc_build_table_emax(hist, k_max, e_max_true, table, table_len);
  } else {
    st = orc_build_table(hist, k_max, table, table_len);
  }
  free(hist);
  if (st != ORC_OK) return st;
  int eb = 0;
  while ((1 << eb) < k_max) ++eb;
  *ei_bits_out = eb;
  int in_col = (cols < (1LL << (32 - eb)));
  *ei_in_column = in_col;
  int fail = 0;
#pragma omp parallel for schedule(static) reduction(| : fail)
  for (int64_t i = 0; i < nnz; ++i) {
    uint64_t w;
    int ei;
    if (orc_encode_value(val[i], table, *table_len, &w, &ei) != ORC_OK) {
      fail = 1;
      continue;
    }
    orc_segment(w, &head[i], &tail1[i], &tail2[i]);
    if (in_col) {
      col_ei[i] = (uint32_t)col[i] | (eb ? ((uint32_t)ei << (32 - eb)) : 0u);
    } else {
      col_ei[i] = (uint32_t)col[i];
      side_ei[i] = (uint8_t)ei;
    }
  }
  return fail ? ORC_ERR_UNREPRESENTABLE : ORC_OK;
}

/* ------------------------------------------------------------------------------------
 * c.1 step 6 -- SpMV.  S:265 "y[i] = sum_j values[j]*x[col[j]] accumulated left-to-right
 * in column order within each row"; "we load low-precision sparse matrices only
 * during memory access and still perform multiplication and accumulation operations based
 * on double-precision"; Alg. 2, sum reset per row (R9).  Row-parallel only
 * (S:304), in-row order sequential.
 * ------------------------------------------------------------------------------------ */
int orc_spmv_fp64(int64_t rows, const int64_t* row_ptr, const int32_t* col, const double* val,
                  const double* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows; ++i) {
    double sum = 0.0;
    for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; ++j) {
      double prod = val[j] * x[col[j]];
      sum = sum + prod;
    }
    y[i] = sum;
  }
  return ORC_OK;
}

int orc_spmv_gse(const orc_matrix* A, int level, const double* x, double* y) {
  if (level < 1 || level > 3) return ORC_ERR_INVALID_ARG;
  const int eb = A->ei_bits;
  const uint32_t mask = (eb && A->ei_in_column) ? ((1u << (32 - eb)) - 1u) : 0xFFFFFFFFu;
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t i = 0; i < A->rows; ++i) {
    double sum = 0.0;
    for (int64_t j = A->row_ptr[i]; j < A->row_ptr[i + 1]; ++j) {
      uint32_t c = A->col_ei[j];
      int ei = A->ei_in_column ? (eb ? (int)(c >> (32 - eb)) : 0) : (int)A->side_ei[j];
      uint32_t colj = c & mask;
      uint64_t w = orc_assemble(A->head[j], A->tail1[j], A->tail2[j], level);
      double v;
      if (orc_decode(w, ei, A->table, A->table_len, &v) != ORC_OK) {
        bad = 1;
        v = 0.0;
      }
      double prod = v * x[colj];
      sum = sum + prod;
    }
    y[i] = sum;
  }
  return bad ? ORC_ERR_INVALID_EXP_INDEX : ORC_OK;
}

/* ------------------------------------------------------------------------------------
 * FP16 / BF16 storage baselines.  P:406 [4.3]: "all non-zero elements are stored and
 * loaded in FP16 or BF16 format, then converted to FP64 and multiplied by the
 * double-precision vector. All intermediate results are accumulated in double-precision".
 * The FP64 -> 16-bit conversion is round-to-nearest-even, directly from the double (R26;
 * the paper does not state it).  Formats (IEEE 754 binary16 / bfloat16):
 *   FP16: 1 sign, 5 exponent bits (bias 15), 10 fraction bits; min normal 2^-14,
 *         subnormal spacing 2^-24, max finite 65504;
 *   BF16: 1 sign, 8 exponent bits (bias 127), 7 fraction bits; min normal 2^-126,
 *         subnormal spacing 2^-133, max finite (2 - 2^-7) 2^127.
 * Rounding, written out: with a = |v| = 1.f * 2^E, the representable numbers near a are
 * the integer multiples of the quantum 2^q, q = E - fraction_bits (or the subnormal
 * spacing below the normal range); n = a / 2^q is exact (power-of-two scaling) and
 * nearbyint() rounds it to the nearest integer, ties to even (the default rounding
 * mode).  A result above the largest finite value is an overflow (+-Inf).
 * ------------------------------------------------------------------------------------ */
uint16_t orc_round_half(double v, int kind) {
  const int fb = (kind == ORC_FP16) ? 10 : 7;          /* fraction bits */
  const int bias = (kind == ORC_FP16) ? 15 : 127;
  const int emin = 1 - bias;                           /* exponent of the min normal */
  const uint16_t inf_bits = (kind == ORC_FP16) ? 0x7C00 : 0x7F80;
  const uint16_t nan_bits = (kind == ORC_FP16) ? 0x7E00 : 0x7FC0;
  const double max_finite = ldexp(2.0 - ldexp(1.0, -fb), bias);
  const uint16_t sign = (bits_of(v) >> 63) ? 0x8000 : 0;
  if (isnan(v)) return (uint16_t)(sign | nan_bits);
  const double a = fabs(v);
  if (isinf(a)) return (uint16_t)(sign | inf_bits);
  if (a == 0.0) return sign;
  int e2;
  frexp(a, &e2);       /* a = f 2^e2, f in [0.5, 1) */
  const int E = e2 - 1; /* a = 1.f 2^E */
  const int q = (E < emin) ? emin - fb : E - fb;       /* quantum exponent */
  const double n = nearbyint(ldexp(a, -q));            /* RNE to an integer multiple */
  const double r = ldexp(n, q);
  if (r > max_finite) return (uint16_t)(sign | inf_bits);
  if (r < ldexp(1.0, emin)) return (uint16_t)(sign | (uint16_t)n); /* subnormal (or 0) */
  int er;
  frexp(r, &er);
  const int Er = er - 1;
  const double frac = ldexp(r, -Er) - 1.0;             /* in [0, 1), exact */
  const uint16_t m = (uint16_t)ldexp(frac, fb);
  return (uint16_t)(sign | (uint16_t)((Er + bias) << fb) | m);
}

double orc_half_value(uint16_t h, int kind) {
  const int fb = (kind == ORC_FP16) ? 10 : 7;
  const int eb = (kind == ORC_FP16) ? 5 : 8;
  const int bias = (kind == ORC_FP16) ? 15 : 127;
  const int emax_field = (1 << eb) - 1;
  const int s = (h >> 15) & 1;
  const int e = (h >> fb) & emax_field;
  const int m = h & ((1 << fb) - 1);
  double a;
  if (e == 0)
    a = ldexp((double)m, 1 - bias - fb);               /* subnormal: m 2^(emin - fb) */
  else if (e == emax_field)
    a = m ? NAN : INFINITY;
  else
    a = ldexp((double)((1 << fb) + m), e - bias - fb); /* (1.m) 2^(e - bias) */
  return s ? -a : a;
}

void orc_round_half_array(int64_t n, const double* v, uint16_t* out, int kind) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = orc_round_half(v[i], kind);
}

void orc_half_value_array(int64_t n, const uint16_t* h, double* out, int kind) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = orc_half_value(h[i], kind);
}

int orc_spmv_half(const orc_matrix* A, const double* x, double* y) {
  if (A->half_kind != ORC_FP16 && A->half_kind != ORC_BF16) return ORC_ERR_INVALID_ARG;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < A->rows; ++i) {
    double sum = 0.0;
    for (int64_t j = A->row_ptr[i]; j < A->row_ptr[i + 1]; ++j) {
      double v = orc_half_value(A->half[j], A->half_kind);
      double prod = v * x[A->col[j]];
      sum = sum + prod;
    }
    y[i] = sum;
  }
  return ORC_OK;
}

int orc_apply(const orc_matrix* A, int level, const double* x, double* y) {
  if (A->half_kind) return orc_spmv_half(A, x, y);
  if (A->val) return orc_spmv_fp64(A->rows, A->row_ptr, A->col, A->val, x, y);
  return orc_spmv_gse(A, level, x, y);
}

/* ------------------------------------------------------------------------------------
 * R29 (build reading; the paper's switching rule is the monitor of P:258-294, whose
 * defaults never fire before convergence on the BASELINE configs, R17): the level-L
 * matrix A_L = A_3 - E_L differs from the full-precision one by the truncated tail bits,
 * so the true residual of ANY iterate satisfies
 *   ||b - A_3 x|| <= ||b - A_L x|| + ||E_L|| ||x||,
 * and once the level-L residual falls below ~||E_L|| ||x|| / ||b|| further level-L
 * iterations cannot lower the true residual (the attainable-accuracy floor of level L).
 * eta_L = ||E_L||_inf = max_i sum_j |dec_3(a_ij) - dec_L(a_ij)| (a bound on ||E_L||_2 for
 * symmetric E_L; a heuristic scale otherwise), row sums in storage order.
 * ------------------------------------------------------------------------------------ */
int orc_perturbation_bounds(const orc_matrix* A, double eta[2]) {
  eta[0] = eta[1] = 0.0;
  if (A->val || A->half_kind) return ORC_ERR_INVALID_ARG;
  const int eb = A->ei_bits;
  int bad = 0;
  for (int64_t i = 0; i < A->rows; ++i) {
    double s1 = 0.0, s2 = 0.0;
    for (int64_t j = A->row_ptr[i]; j < A->row_ptr[i + 1]; ++j) {
      uint32_t c = A->col_ei[j];
      int ei = A->ei_in_column ? (eb ? (int)(c >> (32 - eb)) : 0) : (int)A->side_ei[j];
      double v3, v1, v2;
      bad |= orc_decode(orc_assemble(A->head[j], A->tail1[j], A->tail2[j], 3), ei, A->table,
                        A->table_len, &v3) != ORC_OK;
      bad |= orc_decode(orc_assemble(A->head[j], A->tail1[j], A->tail2[j], 1), ei, A->table,
                        A->table_len, &v1) != ORC_OK;
      bad |= orc_decode(orc_assemble(A->head[j], A->tail1[j], A->tail2[j], 2), ei, A->table,
                        A->table_len, &v2) != ORC_OK;
      double e1 = fabs(v3 - v1), e2 = fabs(v3 - v2);
      s1 = s1 + e1;
      s2 = s2 + e2;
    }
    if (s1 > eta[0]) eta[0] = s1;
    if (s2 > eta[1]) eta[1] = s2;
  }
  return bad ? ORC_ERR_INVALID_EXP_INDEX : ORC_OK;
}

/* ------------------------------------------------------------------------------------
 * c.1 step 9 -- residual monitor, window w[0..t] = resid[j-t .. j] (oldest first).
 * Eq. 3: RSD = sqrt((1/t) sum_{i=j-t}^{j-1} (resid[i]-avg)^2) / avg, avg over
 *   the same t values; 0 if avg < 1e-300.
 * Eqs. 4-5: nDec = #{i in [j-t, j-1] : resid[i] > resid[i+1]}.
 * Eq. 6: relDec = (resid[j-t] - resid[j-1]) / resid[j-t].
 * Conditions 1-3 with t/2 replaced by nDec_limit (R13).
 * ------------------------------------------------------------------------------------ */
double orc_rsd(const double* w, int64_t t) {
  double sum = 0.0;
  for (int64_t i = 0; i < t; ++i) sum = sum + w[i];
  double avg = sum / (double)t;
  if (avg < 1e-300) return 0.0;
  double ss = 0.0;
  for (int64_t i = 0; i < t; ++i) {
    double dv = w[i] - avg;
    double sq = dv * dv;
    ss = ss + sq;
  }
  return sqrt(ss / (double)t) / avg;
}

int64_t orc_ndec(const double* w, int64_t t) {
  int64_t n = 0;
  for (int64_t i = 0; i < t; ++i) n += (w[i] > w[i + 1]) ? 1 : 0;
  return n;
}

double orc_reldec(const double* w, int64_t t) { return (w[0] - w[t - 1]) / w[0]; }

int orc_should_escalate(const double* w, int64_t t, double rsd_limit, int64_t ndec_limit,
                        double reldec_limit) {
  if (!(w[0] > 0.0)) return 0; /* S:355 zero leading residual: treated as converged */
  double rsd = orc_rsd(w, t);
  int64_t nd = orc_ndec(w, t);
  double rd = orc_reldec(w, t);
  int c1 = (rsd > rsd_limit) && (nd < ndec_limit);
  int c2 = (nd >= ndec_limit) && (rd < reldec_limit);
  int c3 = (nd == 0);
  return c1 || c2 || c3;
}

/* P:433 and P:441 (section 4.4.1): GMRES l=9000 t=300 m=1500, 0.03/80/0.08;
 * CG l=3000 t=250 m=500, 0.50/130/0.45.  verify_at_full (R16) default on, floors off. */
void orc_default_schedule(int solver, orc_schedule* s) {
  memset(s, 0, sizeof(*s));
  s->enabled = 1;
  s->start_level = 1;
  s->max_level = 3;
  s->verify_at_full = 1;
  if (solver == 0) {
    s->l = 3000; s->t = 250; s->m = 500;
    s->rsd_limit = 0.50; s->ndec_limit = 130; s->reldec_limit = 0.45;
  } else {
    s->l = 9000; s->t = 300; s->m = 1500;
    s->rsd_limit = 0.03; s->ndec_limit = 80; s->reldec_limit = 0.08;
  }
}

/* ---- plain FP64 vector helpers (sequential, index order) ---- */
static double vdot_seq(int64_t n, const double* a, const double* b) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double p = a[i] * b[i];
    s = s + p;
  }
  return s;
}

/* c.1 step 10 (partitioned mode): the solvers' vectors are split into P
 * row blocks [bounds[r], bounds[r+1]) as the row-partitioned GPU path splits them; every
 * dot product is summed per simulated rank (sequentially, as vdot_seq) and the P partial
 * sums are added in rank order (the allreduce).  SpMV rows are independent, so a rank's
 * rows -- computed with the halo entries of x gathered -- are the same numbers as in the
 * single-rank product.  Set only for the duration of orc_cg_part / orc_gmres_part. */
static __thread int t_parts = 0;
static __thread const int64_t* t_bounds = NULL;

static double vdot(int64_t n, const double* a, const double* b) {
  if (t_parts > 1 && t_bounds[t_parts] == n) {
    double s = 0.0;
    for (int r = 0; r < t_parts; ++r) {
      const int64_t lo = t_bounds[r], hi = t_bounds[r + 1];
      s = s + vdot_seq(hi - lo, a + lo, b + lo);
    }
    return s;
  }
  return vdot_seq(n, a, b);
}

static int valid_parts(const orc_matrix* A, int P, const int64_t* bounds) {
  if (P < 1 || !bounds || bounds[0] != 0 || bounds[P] != A->rows) return 0;
  for (int r = 0; r < P; ++r)
    if (bounds[r + 1] < bounds[r]) return 0;
  return 1;
}

/* ring of the last t+1 residuals */
typedef struct {
  double* buf;
  int64_t cap, count, head; /* head = index of the oldest entry */
} ring_t;

static void ring_push(ring_t* r, double v) {
  if (r->cap <= 0) return;
  if (r->count < r->cap) {
    r->buf[(r->head + r->count) % r->cap] = v;
    r->count++;
  } else {
    r->buf[r->head] = v;
    r->head = (r->head + 1) % r->cap;
  }
}

static void ring_window(const ring_t* r, double* w) {
  for (int64_t i = 0; i < r->count; ++i) w[i] = r->buf[(r->head + i) % r->cap];
}

/* check point rule: j >= l, (j - l) mod m == 0, window full; returns 1 to
 * escalate.  Level floors (R17) are an optional build heuristic, default off. */
static int monitor_check(const orc_schedule* s, const ring_t* ring, double* wbuf, int64_t j,
                         int level, double resid, const double* eta, double xx, double bnorm) {
  if (!s->enabled || level >= s->max_level) return 0;
  if (level <= 2 && s->level_floor[level - 1] > 0.0 && resid < s->level_floor[level - 1])
    return 1;
  /* R29: the level's attainable-accuracy floor, with x the iterate before this iteration's
   * update (CG) or at the start of the cycle (GMRES) */
  if (level <= 2 && s->perturb_c > 0.0 && xx > 0.0) {
    double thr = s->perturb_c * eta[level - 1];
    thr = thr * sqrt(xx);
    thr = thr / bnorm;
    if (resid <= thr) return 1;
  }
  if (j < s->l || ((j - s->l) % s->m) != 0 || ring->count < s->t + 1) return 0;
  ring_window(ring, wbuf);
  return orc_should_escalate(wbuf, s->t, s->rsd_limit, s->ndec_limit, s->reldec_limit);
}

static int validate_sched(const orc_schedule* s) {
  if (s->start_level < 1 || s->start_level > 3) return 0;
  if (!(s->perturb_c >= 0.0)) return 0;
  if (s->cg_keep_direction != 0 && s->cg_keep_direction != 1) return 0;
  if (s->enabled) {
    if (s->max_level < s->start_level || s->max_level > 3) return 0;
    if (s->t < 1 || s->m < 1) return 0;
  }
  return 1;
}

static void log_switch(orc_report* rep, int64_t j, int new_level) {
  if (rep->n_switches < 2) {
    rep->switch_iter[rep->n_switches] = j;
    rep->switch_to_level[rep->n_switches] = new_level;
  }
  rep->n_switches++;
}

/* true relative residual ||b - A_level x|| / ||b|| */
static double true_resid(const orc_matrix* A, int level, const double* b, const double* x,
                         double* tmp, double bnorm, orc_report* rep) {
  orc_apply(A, level, x, tmp);
  rep->spmv_count[level - 1]++;
  for (int64_t i = 0; i < A->rows; ++i) tmp[i] = b[i] - tmp[i];
  return sqrt(vdot(A->rows, tmp, tmp)) / bnorm;
}

/* ------------------------------------------------------------------------------------
 * c.1 step 7 -- CG (unpreconditioned) inside the stepped driver of
 * Alg. stepped-GMRES: w_j = A_tag v_j; one level per trigger (R12); the
 * monitor sees the recurrence residual ||r_j||/||b|| (R14); at a switch r <- b - A_new x
 * (residual replacement, R15); at L < 3 a converged recurrence is verified with A_3
 * (R16).  With sched->enabled == 0 the solve runs at fixed start_level (FP64 matrix:
 * level ignored) and stops on the recurrence residual.
 * ------------------------------------------------------------------------------------ */
int orc_cg(const orc_matrix* A, const double* b, double* x, double tol, int64_t max_iters,
           const orc_schedule* sched, orc_report* rep) {
  memset(rep, 0, sizeof(*rep));
  if (!(tol > 0.0) || max_iters < 0 || !validate_sched(sched) || A->rows != A->cols)
    return ORC_ERR_INVALID_ARG;
  const int64_t n = A->rows;
  const int stepped = sched->enabled && !A->val;
  int level = A->val ? 3 : sched->start_level;
  double* r = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  double* p = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  double* q = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  ring_t ring = {0};
  ring.cap = stepped ? sched->t + 1 : 0;
  ring.buf = (double*)malloc((size_t)(ring.cap ? ring.cap : 1) * sizeof(double));
  double* wbuf = (double*)malloc((size_t)(ring.cap ? ring.cap : 1) * sizeof(double));
  int status = ORC_NOT_CONVERGED;
  double eta[2] = {0.0, 0.0};
  if (stepped && sched->perturb_c > 0.0) orc_perturbation_bounds(A, eta);

  double bnorm = sqrt(vdot(n, b, b));
  if (bnorm == 0.0) { /* b = 0 -> x = 0 is exact */
    for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
    rep->converged = 1;
    status = ORC_OK;
    goto done;
  }
  /* r0 = b - A_L x0 ; p0 = r0 */
  orc_apply(A, level, x, q);
  rep->spmv_count[level - 1]++;
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - q[i];
  for (int64_t i = 0; i < n; ++i) p[i] = r[i];
  double rr = vdot(n, r, r);
  double resid = sqrt(rr) / bnorm;
  rep->rel_residual_recurrence = resid;
  int64_t j = 0;
  if (resid <= tol) {
    if (!(stepped && level < 3 && sched->verify_at_full)) { status = ORC_OK; goto out; }
    if (true_resid(A, 3, b, x, q, bnorm, rep) <= tol) { status = ORC_OK; goto out; }
    /* x0 already converged at A_L but not at A: finish at the highest allowed level (R16;
     * capped by max_level: no higher level allowed -> not converged) */
    if (level >= sched->max_level) { status = ORC_NOT_CONVERGED; goto out; }
    level = sched->max_level;
    log_switch(rep, 0, level);
    orc_apply(A, level, x, q);
    rep->spmv_count[level - 1]++;
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - q[i];
    for (int64_t i = 0; i < n; ++i) p[i] = r[i];
    rr = vdot(n, r, r);
  }
  while (j < max_iters) {
    j++;
    /* q = A_tag p  (Alg. stepped-GMRES l.3-8: w_j = A_tag v_j) */
    orc_apply(A, level, p, q);
    rep->spmv_count[level - 1]++;
    rep->iters_per_level[level - 1]++;
    double pq = vdot(n, p, q);
    if (!(pq > 0.0) || !isfinite(pq)) { status = ORC_NUMERICAL_ABORT; break; }
    double xx = (stepped && sched->perturb_c > 0.0) ? vdot(n, x, x) : 0.0; /* R29: x_{j-1} */
    double alpha = rr / pq;
    for (int64_t i = 0; i < n; ++i) { double t2 = alpha * p[i]; x[i] = x[i] + t2; }
    for (int64_t i = 0; i < n; ++i) { double t2 = alpha * q[i]; r[i] = r[i] - t2; }
    double rr_new = vdot(n, r, r);
    resid = sqrt(rr_new) / bnorm;
    rep->rel_residual_recurrence = resid;
    if (!isfinite(resid)) { status = ORC_NUMERICAL_ABORT; break; }
    if (stepped) ring_push(&ring, resid);
    int escalate = 0;
    if (resid <= tol) {
      if (!(stepped && level < 3 && sched->verify_at_full)) { status = ORC_OK; break; }
      if (true_resid(A, 3, b, x, q, bnorm, rep) <= tol) { status = ORC_OK; break; }
      /* R16: converged at A_L but not at A -> one level up, within max_level */
      if (level >= sched->max_level) { status = ORC_NOT_CONVERGED; break; }
      escalate = 1;
    } else if (stepped && monitor_check(sched, &ring, wbuf, j, level, resid, eta, xx, bnorm)) {
      escalate = 1;
    }
    if (escalate) {
      level++;
      log_switch(rep, j, level);
      orc_apply(A, level, x, q);
      rep->spmv_count[level - 1]++;
      for (int64_t i = 0; i < n; ++i) r[i] = b[i] - q[i];
      if (sched->cg_keep_direction) {
        /* R30: residual replacement r <- b - A_new x with the search direction kept:
         * beta = r.r / rr_{j-1}, p <- r + beta p, rr <- r.r (the CG step with the
         * replaced residual in place of the recurrence one) */
        double rr_rep = vdot(n, r, r);
        double beta = rr_rep / rr;
        for (int64_t i = 0; i < n; ++i) { double t2 = beta * p[i]; p[i] = r[i] + t2; }
        rr = rr_rep;
      } else {
        /* R15: the operator changed, so CG restarts from the current x at the new level:
         * r <- b - A_new x (residual replacement), p <- r, rr <- r.r */
        for (int64_t i = 0; i < n; ++i) p[i] = r[i];
        rr = vdot(n, r, r);
      }
      resid = sqrt(rr) / bnorm;
      rep->rel_residual_recurrence = resid;
      continue;
    }
    double beta = rr_new / rr;
    for (int64_t i = 0; i < n; ++i) { double t2 = beta * p[i]; p[i] = r[i] + t2; }
    rr = rr_new;
  }
out:
  rep->iterations = j;
done:
  rep->converged = (status == ORC_OK);
  if (n > 0 && bnorm > 0.0) rep->rel_residual_true = true_resid(A, 3, b, x, q, bnorm, rep);
  free(r); free(p); free(q); free(ring.buf); free(wbuf);
  return status;
}

/* Givens rotation of R18 (Golub-Van Loan form): returns (c, s) with c*h1 + s*h2 = rho,
 * -s*h1 + c*h2 = 0. */
static void givens(double h1, double h2, double* c, double* s) {
  if (h2 == 0.0) {
    *c = 1.0; *s = 0.0;
  } else if (fabs(h2) > fabs(h1)) {
    double tau = h1 / h2;
    double t2 = tau * tau;
    *s = 1.0 / sqrt(1.0 + t2);
    *c = *s * tau;
  } else {
    double tau = h2 / h1;
    double t2 = tau * tau;
    *c = 1.0 / sqrt(1.0 + t2);
    *s = *c * tau;
  }
}

/* ------------------------------------------------------------------------------------
 * c.1 step 8 -- restarted GMRES(m) ("restart is set to 30 ... maximum outer
 * iterations are set to 500"): Arnoldi by modified Gram-Schmidt, least squares
 * by Givens rotations (R18), the rotation residual estimate |g_{j+1}|/||b|| fed to the
 * monitor every inner iteration with a global inner counter.  Explicit residual
 * r = b - A_L x at every restart and at termination.  A switch ends the current cycle
 * (x += V y) and restarts at the new level (R15); at L < 3 convergence is verified with
 * A_3 (R16).
 * ------------------------------------------------------------------------------------ */
int orc_gmres(const orc_matrix* A, const double* b, double* x, double tol, int restart,
              int64_t max_iters, const orc_schedule* sched, orc_report* rep) {
  memset(rep, 0, sizeof(*rep));
  if (!(tol > 0.0) || restart < 1 || max_iters < 0 || !validate_sched(sched) ||
      A->rows != A->cols)
    return ORC_ERR_INVALID_ARG;
  const int64_t n = A->rows;
  const int m = restart;
  const int stepped = sched->enabled && !A->val;
  int level = A->val ? 3 : sched->start_level;
  double* V = (double*)malloc((size_t)(m + 1) * (size_t)(n ? n : 1) * sizeof(double));
  double* w = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  double* H = (double*)calloc((size_t)(m + 1) * (size_t)m, sizeof(double)); /* H[i*m + j] */
  double* cs = (double*)malloc((size_t)m * sizeof(double));
  double* sn = (double*)malloc((size_t)m * sizeof(double));
  double* g = (double*)malloc((size_t)(m + 1) * sizeof(double));
  double* yv = (double*)malloc((size_t)m * sizeof(double));
  ring_t ring = {0};
  ring.cap = stepped ? sched->t + 1 : 0;
  ring.buf = (double*)malloc((size_t)(ring.cap ? ring.cap : 1) * sizeof(double));
  double* wbuf = (double*)malloc((size_t)(ring.cap ? ring.cap : 1) * sizeof(double));
  int status = ORC_NOT_CONVERGED;
  int64_t jg = 0;
  double eta[2] = {0.0, 0.0};
  if (stepped && sched->perturb_c > 0.0) orc_perturbation_bounds(A, eta);

  double bnorm = sqrt(vdot(n, b, b));
  if (bnorm == 0.0) {
    for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
    status = ORC_OK;
    goto done;
  }
  for (;;) {
    /* explicit residual at (re)start with the current level */
    orc_apply(A, level, x, w);
    rep->spmv_count[level - 1]++;
    for (int64_t i = 0; i < n; ++i) w[i] = b[i] - w[i];
    double beta = sqrt(vdot(n, w, w));
    double resid = beta / bnorm;
    rep->rel_residual_recurrence = resid;
    if (!isfinite(resid)) { status = ORC_NUMERICAL_ABORT; break; }
    if (resid <= tol) {
      if (stepped && level < 3 && sched->verify_at_full) {
        double rt = true_resid(A, 3, b, x, w, bnorm, rep);
        if (rt <= tol) { status = ORC_OK; break; }
        if (level >= sched->max_level) { status = ORC_NOT_CONVERGED; break; } /* capped */
        level++;
        log_switch(rep, jg, level);
        continue; /* restart with an explicit residual at the new level */
      }
      status = ORC_OK;
      break;
    }
    if (jg >= max_iters) { status = ORC_NOT_CONVERGED; break; }
    double xx = (stepped && sched->perturb_c > 0.0) ? vdot(n, x, x) : 0.0; /* R29: cycle start */
    for (int64_t i = 0; i < n; ++i) V[i] = w[i] / beta;
    if (sched->krylov_gse16) compress16(n, V); /* NEXT-4 (R28) */
    for (int i = 0; i <= m; ++i) g[i] = 0.0;
    g[0] = beta;
    int k = 0;          /* basis vectors used in this cycle */
    int escalate = 0;
    for (int jj = 0; jj < m; ++jj) {
      jg++;
      rep->iters_per_level[level - 1]++;
      double* vj = V + (size_t)jj * (size_t)n;
      orc_apply(A, level, vj, w);
      rep->spmv_count[level - 1]++;
      for (int i = 0; i <= jj; ++i) { /* modified Gram-Schmidt */
        double* vi = V + (size_t)i * (size_t)n;
        double h = vdot(n, w, vi);
        H[i * m + jj] = h;
        for (int64_t q = 0; q < n; ++q) { double t2 = h * vi[q]; w[q] = w[q] - t2; }
      }
      double hn = sqrt(vdot(n, w, w));
      H[(jj + 1) * m + jj] = hn;
      for (int i = 0; i < jj; ++i) { /* apply previous rotations to column jj */
        double h1 = H[i * m + jj], h2 = H[(i + 1) * m + jj];
        double a1 = cs[i] * h1, a2 = sn[i] * h2;
        double b1 = sn[i] * h1, b2 = cs[i] * h2;
        H[i * m + jj] = a1 + a2;
        H[(i + 1) * m + jj] = b2 - b1;
      }
      double c, s;
      givens(H[jj * m + jj], H[(jj + 1) * m + jj], &c, &s);
      cs[jj] = c; sn[jj] = s;
      {
        double h1 = H[jj * m + jj], h2 = H[(jj + 1) * m + jj];
        double a1 = c * h1, a2 = s * h2;
        H[jj * m + jj] = a1 + a2;
        H[(jj + 1) * m + jj] = 0.0;
      }
      g[jj + 1] = -(s * g[jj]);
      g[jj] = c * g[jj];
      resid = fabs(g[jj + 1]) / bnorm;
      rep->rel_residual_recurrence = resid;
      k = jj + 1;
      if (!isfinite(resid)) { status = ORC_NUMERICAL_ABORT; break; }
      if (stepped) ring_push(&ring, resid);
      if (resid <= tol || hn == 0.0) break; /* converged estimate / happy breakdown */
      if (stepped && monitor_check(sched, &ring, wbuf, jg, level, resid, eta, xx, bnorm)) {
        escalate = 1;
        break;
      }
      if (jg >= max_iters) break;
      double* vn = V + (size_t)(jj + 1) * (size_t)n;
      for (int64_t q = 0; q < n; ++q) vn[q] = w[q] / hn;
      if (sched->krylov_gse16) compress16(n, vn);
    }
    if (status == ORC_NUMERICAL_ABORT) break;
    /* back substitution H[0:k,0:k] y = g[0:k]; x += V y */
    for (int i = k - 1; i >= 0; --i) {
      double sacc = g[i];
      for (int l2 = i + 1; l2 < k; ++l2) { double t2 = H[i * m + l2] * yv[l2]; sacc = sacc - t2; }
      yv[i] = sacc / H[i * m + i];
    }
    for (int i = 0; i < k; ++i) {
      const double* vi = V + (size_t)i * (size_t)n;
      for (int64_t q = 0; q < n; ++q) { double t2 = yv[i] * vi[q]; x[q] = x[q] + t2; }
    }
    if (escalate) {
      level++;
      log_switch(rep, jg, level);
    }
  }
done:
  rep->iterations = jg;
  rep->converged = (status == ORC_OK);
  if (n > 0 && bnorm > 0.0) rep->rel_residual_true = true_resid(A, 3, b, x, w, bnorm, rep);
  free(V); free(w); free(H); free(cs); free(sn); free(g); free(yv); free(ring.buf); free(wbuf);
  return status;
}

/* c.1 step 10: CG / GMRES(m) in partitioned mode (P simulated ranks, row blocks
 * [bounds[r], bounds[r+1]), dots summed per rank then in rank order).  P = 1 is orc_cg /
 * orc_gmres exactly. */
int orc_cg_part(const orc_matrix* A, const double* b, double* x, double tol, int64_t max_iters,
                const orc_schedule* sched, int P, const int64_t* bounds, orc_report* rep) {
  if (!valid_parts(A, P, bounds)) return ORC_ERR_INVALID_ARG;
  t_parts = P;
  t_bounds = bounds;
  int st = orc_cg(A, b, x, tol, max_iters, sched, rep);
  t_parts = 0;
  t_bounds = NULL;
  return st;
}

int orc_gmres_part(const orc_matrix* A, const double* b, double* x, double tol, int restart,
                   int64_t max_iters, const orc_schedule* sched, int P, const int64_t* bounds,
                   orc_report* rep) {
  if (!valid_parts(A, P, bounds)) return ORC_ERR_INVALID_ARG;
  t_parts = P;
  t_bounds = bounds;
  int st = orc_gmres(A, b, x, tol, restart, max_iters, sched, rep);
  t_parts = 0;
  t_bounds = NULL;
  return st;
}
