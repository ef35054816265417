// vec16.cu -- 16-bit GSE-SEM vectors (NEXT-4; Alg. 1 P:128-160 in its 16-bit layout, R28):
// exponent histogram of a vector (a1 for a vector), table selection (a2: top k by count,
// ties to the larger exponent, e_max forced into the last slot, P:116 / P:123), encode
// (Alg. 1) and decode.  Every kernel is stream-ordered and can be captured in a graph.
#include "vec16.cuh"

namespace gse {

__global__ void __launch_bounds__(256) k_v16_hist(const double* __restrict__ src,
                                                  const double* den, int64_t n,
                                                  unsigned* __restrict__ hist, const int* stop) {
  __shared__ unsigned h[2048];
  if (stop && *stop) return;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const double dv = den ? *den : 1.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = den ? src[i] / dv : src[i];
    unsigned e = (unsigned)((unsigned long long)__double_as_longlong(v) >> 52) & 0x7FFu;
    if (e == 0u || e == 0x7FFu) e = 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(__activemask(), e);
    if (e != 0xFFFFFFFFu && (int)(threadIdx.x & 31) == __ffs(peers) - 1)
      atomicAdd(&h[e], (unsigned)__popc(peers));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// one CTA of 1024: k rounds of block arg-max over (count << 11 | e); e_max forced into the
// last selected slot; entries e + 1; the histogram is cleared for the next vector
__global__ void __launch_bounds__(1024) k_v16_select(unsigned* __restrict__ hist, int k_max,
                                                     uint16_t* __restrict__ table,
                                                     int* __restrict__ table_len,
                                                     const int* stop) {
  __shared__ unsigned long long key[2048];
  __shared__ unsigned long long red[32];
  __shared__ int sel[V16_KMAX];
  __shared__ int s_nd, s_emax;
  if (stop && *stop) return;
  if (threadIdx.x == 0) {
    s_nd = 0;
    s_emax = 0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 2048; e += blockDim.x) {
    const unsigned c = (e >= 1 && e <= 2046) ? hist[e] : 0u;
    key[e] = c ? (((unsigned long long)c << 11) | (unsigned long long)e) : 0ull;
    if (c) {
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
    for (int k = 0; k < V16_KMAX; ++k) table[k] = (uint16_t)(k < take ? sel[k] + 1 : 0);
    *table_len = take;
  }
  for (int e = threadIdx.x; e < 2048; e += blockDim.x) hist[e] = 0u;
}

__global__ void __launch_bounds__(256) k_v16_encode(const double* __restrict__ src,
                                                    const double* den, int64_t n,
                                                    const uint16_t* __restrict__ table,
                                                    const int* __restrict__ table_len, int eb,
                                                    uint16_t* __restrict__ words,
                                                    double* __restrict__ decoded,
                                                    const int* stop) {
  __shared__ int E[V16_KMAX];
  __shared__ double sc[V16_KMAX];
  if (stop && *stop) return;
  const int len = *table_len;
  if (threadIdx.x < V16_KMAX) E[threadIdx.x] = threadIdx.x < len ? (int)table[threadIdx.x] : 0;
  load_scales16(table, len, eb, sc);
  __syncthreads();
  const double dv = den ? *den : 1.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = den ? src[i] / dv : src[i];
    const uint16_t w = enc16(v, E, len, eb);
    words[i] = w;
    if (decoded) decoded[i] = dec16(w, sc, eb);
  }
}

__global__ void __launch_bounds__(256) k_v16_decode(const uint16_t* __restrict__ words, int64_t n,
                                                    const uint16_t* __restrict__ table,
                                                    const int* __restrict__ table_len, int eb,
                                                    double* __restrict__ out) {
  __shared__ double sc[V16_KMAX];
  load_scales16(table, *table_len, eb, sc);
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = dec16(words[i], sc, eb);
}

void v16_hist(const double* src, const double* den, int64_t n, unsigned* hist, const int* stop,
              int grid, cudaStream_t s) {
  launch_k(k_v16_hist, grid, 256, 0, s, src, den, n, hist, stop);
}
void v16_select(unsigned* hist, int k_max, uint16_t* table, int* table_len, const int* stop,
                cudaStream_t s) {
  launch_k(k_v16_select, 1, 1024, 0, s, hist, k_max, table, table_len, stop);
}
void v16_encode(const double* src, const double* den, int64_t n, const uint16_t* table,
                const int* table_len, int eb, uint16_t* words, double* decoded, const int* stop,
                int grid, cudaStream_t s) {
  launch_k(k_v16_encode, grid, 256, 0, s, src, den, n, table, table_len, eb, words, decoded, stop);
}
void v16_decode(const uint16_t* words, int64_t n, const uint16_t* table, const int* table_len,
                int eb, double* out, int grid, cudaStream_t s) {
  launch_k(k_v16_decode, grid, 256, 0, s, words, n, table, table_len, eb, out);
}

}  // namespace gse
