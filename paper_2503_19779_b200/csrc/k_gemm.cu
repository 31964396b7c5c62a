// tcgen05 bf16 GEMM for the decoder nodes — placeholder until the kernel lands.
#include <cuda_runtime.h>
#include <stdint.h>

#include "cgx_decoder.h"

namespace cgx {
bool decoder_gemm_supported(uint32_t, uint32_t, uint32_t) { return false; }
int decoder_gemm_build(uint32_t, uint32_t, uint32_t, uint32_t, const void*, const void*, const void*, const void*,
                       void*, void*, size_t*, dim3*, dim3*, size_t*, const void**) {
  return 7;  // CGX_E_UNSUPPORTED
}
}  // namespace cgx
