// pb_gemm_mma.cu -- tensor-pipe engine for steps a3-a5 (placeholder until the
// engine microbenchmarks pick the instruction).
#include <cuda_runtime.h>

#include "pb_internal.h"

namespace pb {

bool mma_supported(const GemmArgs&) { return false; }

cudaError_t launch_gemm_mma(const GemmArgs&, cudaStream_t) { return cudaErrorNotSupported; }

}  // namespace pb
