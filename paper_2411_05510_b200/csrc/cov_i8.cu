// SSI_COV_INT8X3 placeholder: reports SSI_ERR_DTYPE until the tcgen05 kernel lands.
#include "cov_i8.cuh"

namespace ssi {

bool cov_i8_supported(int, int, int64_t, int) { return false; }
void cov_i8_carve(Carver&, int64_t, int, int, int) {}
ssi_status cov_i8(const void*, int, int64_t, int, int64_t, int, int, int64_t, int64_t, int, double*,
                  void*, int32_t*, cudaStream_t) {
  set_last_error("SSI_COV_INT8X3 not built");
  return SSI_ERR_DTYPE;
}

}  // namespace ssi
