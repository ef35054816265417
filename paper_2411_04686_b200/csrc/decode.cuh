// decode.cuh -- on-the-fly GSE-SEM decode used by the SpMV kernels and gse_decode.
//
// Alg. spmv l.6-17 finds the first one of the head with __fns and rebuilds the
// FP64 exponent as expArr[EI] - (15 - pos).  On sm_100a the branch-free equivalent is:
//     D_L   = the 15 / 31 / 63 significand bits visible at level L (sign stripped)
//     |v|   = D_L * 2^(E - 1086 + s_L)            (s_L = 48, 32, 0)
// evaluated as  bits(double(D_L)) + ((E - 1086 + s_L) << 52): the int->double conversion
// normalises D_L exactly (D_L has <= 53 significant bits for encoder output, and the
// conversion truncates nothing below 2^53), and the integer add rescales the exponent.
// The result's exponent field is E - d'; a field <= 0 (true exponent <= 0, R11) or
// D_L = 0 (R10) gives signed zero.  Bit-identical to the oracle's shift/mask decode
// (tests/test_gpu_parity.py::test_decode_bit_exact).
#pragma once
#include <cstdint>

namespace gse {

__device__ __forceinline__ double decode_bits_to_double(uint64_t D, long long delta,
                                                        uint32_t head) {
  // D: level-visible significand bits (no sign)
  long long b = __double_as_longlong(__ull2double_rz(D));
  long long r = b + delta;
  r = (D == 0 || r < (1LL << 52)) ? 0LL : r;
  r |= (long long)(head & 0x8000u) << 48;
  return __longlong_as_double(r);
}

__device__ __forceinline__ double decode_l1(uint32_t head, long long delta) {
  uint32_t D = head & 0x7FFFu;
  long long b = __double_as_longlong(__uint2double_rn(D));  // exact (<= 15 bits)
  long long r = b + delta;
  r = (D == 0u || r < (1LL << 52)) ? 0LL : r;
  r |= (long long)(head & 0x8000u) << 48;
  return __longlong_as_double(r);
}

__device__ __forceinline__ double decode_l2(uint32_t head, uint32_t tail1, long long delta) {
  uint32_t D = ((head & 0x7FFFu) << 16) | tail1;
  long long b = __double_as_longlong(__uint2double_rn(D));  // exact (<= 31 bits)
  long long r = b + delta;
  r = (D == 0u || r < (1LL << 52)) ? 0LL : r;
  r |= (long long)(head & 0x8000u) << 48;
  return __longlong_as_double(r);
}

__device__ __forceinline__ double decode_l3(uint32_t head, uint32_t tail1, uint32_t tail2,
                                            long long delta) {
  uint64_t D = ((uint64_t)(head & 0x7FFFu) << 48) | ((uint64_t)tail1 << 32) | tail2;
  // D may carry up to 63 significant bits for arbitrary words; the oracle truncates
  // (keeps the top 53 bits), so convert with round-toward-zero.
  return decode_bits_to_double(D, delta, head);
}

// FP32 decode (R20): the level-L value rounded toward zero to FP32; values whose FP32
// exponent field would be <= 0 flush to signed zero.  Overflow is excluded at call time
// (GSE_ERR_FP32_RANGE).
__device__ __forceinline__ float decode_f32(uint64_t D, int delta32, uint32_t head) {
  int b = __float_as_int(__ull2float_rz(D));
  int r = b + delta32;
  r = (D == 0 || r < (1 << 23)) ? 0 : r;
  r |= (int)((head & 0x8000u) << 16);
  return __int_as_float(r);
}

__device__ __forceinline__ float decode_f32_u32(uint32_t D, int delta32, uint32_t head) {
  int b = __float_as_int(__uint2float_rz(D));
  int r = b + delta32;
  r = (D == 0u || r < (1 << 23)) ? 0 : r;
  r |= (int)((head & 0x8000u) << 16);
  return __int_as_float(r);
}

}  // namespace gse
