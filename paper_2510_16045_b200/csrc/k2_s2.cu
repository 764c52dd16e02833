// k2_s2.cu -- K2 instances of scheme 2 (one translation unit per scheme: parallel builds).
#include "k2.cuh"

namespace amsqb {
template cudaError_t launch_linear_scheme<2>(const LinearParams& p, cudaStream_t s);
}  // namespace amsqb
