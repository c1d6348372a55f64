// conv_tc.cu -- tcgen05 kind::i8 implicit-GEMM ternary conv3d (sm_100a).
// Placeholder until the tensor-core kernel lands: reports "not supported" so
// run_conv() uses the CUDA-core popc kernel.
#include "tn_internal.cuh"

namespace tn {

bool conv_tc_supported(const ConvDesc&) { return false; }

cudaError_t launch_conv_tc(const ConvDesc&, cudaStream_t) { return cudaErrorNotSupported; }

}  // namespace tn
