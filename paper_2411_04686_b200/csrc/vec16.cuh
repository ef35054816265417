// vec16.cuh -- 16-bit GSE-SEM vectors: Alg. 1 of the paper
// ("converting double-precision vector to GSE-SEM vector") in its own 16-bit
// layout -- sign (bit 15) | exponent index (ei_bits) | denormalised significand with the
// explicit one (mbits = 15 - ei_bits) -- and its inverse (Alg. 2's decode, with
// the EI read from the word; R28).  Used for the 16-bit Krylov basis of GMRES and by
// gse_encode_vector16 / gse_decode_vector16.
#pragma once
#include <cstdint>

#include "gse_internal.cuh"

namespace gse {

constexpr int V16_KMAX = 16;  // tables of up to 16 entries (ei_bits <= 4, >= 11 significand bits)

// Alg. 1 for one value with the table E[0..len) (stored entries e + 1): nearest E > e,
// d = E - e (l.6-21); the explicit one at bit mbits - d and the top fraction bits below it
// (l.23-25, truncation, R1); zero / subnormal -> signed zero with EI 0 (R2); d > mbits ->
// signed zero (R3).  Non-finite values never reach here (the solve aborts on them first);
// they encode as signed zero.
__device__ __forceinline__ uint16_t enc16(double v, const int* E, int len, int eb) {
  const uint64_t u = (uint64_t)__double_as_longlong(v);
  const uint32_t sign = (uint32_t)(u >> 63) << 15;
  const int e = (int)((u >> 52) & 0x7FF);
  if (e == 0 || e == 0x7FF) return (uint16_t)sign;
  int best = -1, dbest = 1 << 30;
  for (int k = 0; k < len; ++k) {
    const int d = E[k] - e;
    if (d >= 1 && d < dbest) {
      dbest = d;
      best = k;
    }
  }
  const int mbits = 15 - eb;
  if (best < 0 || dbest > mbits) return (uint16_t)sign;
  const uint64_t f = u & ((1ull << 52) - 1);
  const uint32_t mant = (1u << (mbits - dbest)) | (uint32_t)(f >> (52 - mbits + dbest));
  return (uint16_t)(sign | ((uint32_t)best << mbits) | mant);
}

// inverse: |v| = mant * 2^(E_EI - 1023 - mbits) (R28); scale[ei] = 2^(E_ei - 1023 - mbits)
// (an exact power of two, so the product is the correctly rounded value); results below
// the normal range flush to signed zero (R11)
__device__ __forceinline__ double dec16(uint32_t w, const double* scale, int eb) {
  const int mbits = 15 - eb;
  const uint32_t mant = w & ((1u << mbits) - 1u);
  const uint32_t ei = (w >> mbits) & ((1u << eb) - 1u);
  double v = (double)mant * scale[ei];
  if (v < 2.2250738585072014e-308) v = 0.0;
  return (w & 0x8000u) ? -v : v;
}

// scale table of a vector's entries (threads < V16_KMAX fill it)
__device__ __forceinline__ void load_scales16(const uint16_t* tab, int len, int eb, double* sc) {
  const int t = threadIdx.x;
  if (t < V16_KMAX) sc[t] = t < len ? ldexp(1.0, (int)tab[t] - 1023 - (15 - eb)) : 0.0;
}

// launchers (vec16.cu).  den: optional device scalar the source is divided by (v = src/den,
// the GMRES basis normalisation); stop: optional device flag, the kernels return when set.
// hist (2048 uint32, zero on entry) is zeroed again by the selection.
void v16_hist(const double* src, const double* den, int64_t n, unsigned* hist, const int* stop,
              int grid, cudaStream_t s);
void v16_select(unsigned* hist, int k_max, uint16_t* table, int* table_len, const int* stop,
                cudaStream_t s);
void v16_encode(const double* src, const double* den, int64_t n, const uint16_t* table,
                const int* table_len, int eb, uint16_t* words, double* decoded, const int* stop,
                int grid, cudaStream_t s);
void v16_decode(const uint16_t* words, int64_t n, const uint16_t* table, const int* table_len,
                int eb, double* out, int grid, cudaStream_t s);

}  // namespace gse
