// k2_s5.cu -- K2 instances of scheme 5 (one translation unit per scheme: parallel builds).
#include "k2.cuh"

namespace amsqb {
template cudaError_t launch_linear_scheme<5>(const LinearParams& p, cudaStream_t s);
}  // namespace amsqb
