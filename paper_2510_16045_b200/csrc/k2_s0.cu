// k2_s0.cu -- K2 instances of scheme 0 (one translation unit per scheme: parallel builds).
#include "k2.cuh"

namespace amsqb {
template cudaError_t launch_linear_scheme<0>(const LinearParams& p, cudaStream_t s);
}  // namespace amsqb
