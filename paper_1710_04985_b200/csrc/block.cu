// block.cu -- SPTRSV_ALGO_BLOCK: placeholder until the
// blocked self-scheduled kernel lands.
#include "internal.h"

namespace sptrsv {
sptrsv_status_t block_build(sptrsv_handle_t, cudaStream_t) { return SPTRSV_ERR_NOT_SUPPORTED; }
sptrsv_status_t block_solve(sptrsv_handle_t, const void *, void *, cudaStream_t) { return SPTRSV_ERR_NOT_SUPPORTED; }
}  // namespace sptrsv
