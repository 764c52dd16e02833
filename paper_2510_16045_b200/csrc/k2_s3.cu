// k2_s3.cu -- K2 instances of scheme 3 (one translation unit per scheme: parallel builds).
#include "k2.cuh"

namespace amsqb {
template cudaError_t launch_linear_scheme<3>(const LinearParams& p, cudaStream_t s);
}  // namespace amsqb
