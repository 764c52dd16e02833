// k2_s7.cu -- K2 instances of scheme 7 (one translation unit per scheme: parallel builds).
#include "k2.cuh"

namespace amsqb {
template cudaError_t launch_linear_scheme<7>(const LinearParams& p, cudaStream_t s);
}  // namespace amsqb
