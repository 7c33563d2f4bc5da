// gemm.cu — placeholder until the tcgen05 GEMM lands: no block size is implemented, so the
// sweep records every GEMM point as LSCAT_ROW_INVALID_CONFIG.
#include "common.h"

namespace lscat {
cudaError_t gemm_prepare(SuiteEntry&) { return cudaSuccess; }
const KernelTable& table_gemm() {
  static KernelTable t{};
  return t;
}
}  // namespace lscat
