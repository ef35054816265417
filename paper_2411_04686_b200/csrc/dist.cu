// dist.cu -- row-partitioned multi-GPU support.  Placeholder: the NCCL path
// lands in a later commit; the entry points exist so the ABI is stable.
#include "gse_internal.cuh"

namespace gse {
struct DistCtx {};
gse_status dist_halo_exchange(const Matrix&, double*, cudaStream_t) { return GSE_ERR_NCCL; }
gse_status dist_allreduce_sum(const Matrix&, double*, int, cudaStream_t) { return GSE_ERR_NCCL; }
void free_dist(Matrix& M) { M.dist = nullptr; }
}  // namespace gse

using namespace gse;
extern "C" {
gse_status gse_nccl_unique_id(void*) {
  set_error("multi-GPU path not built yet");
  return GSE_ERR_NCCL;
}
gse_status gse_dist_create(const void*, int, int, int, gse_dist* out) {
  if (out) *out = nullptr;
  set_error("multi-GPU path not built yet");
  return GSE_ERR_NCCL;
}
gse_status gse_encode_dist(gse_dist, const gse_csr_f64*, int64_t, int64_t, const gse_encode_opts*,
                           gse_matrix* out, void*) {
  if (out) *out = nullptr;
  set_error("multi-GPU path not built yet");
  return GSE_ERR_NCCL;
}
void gse_dist_free(gse_dist) {}
}
