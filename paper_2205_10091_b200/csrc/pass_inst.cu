// pass_inst.cu -- explicit instantiation of pass_kernel for one (precision, mode);
// compiled six times (TCX_REAL x TCX_KM) so the variants build in parallel.
#include "kernels.cuh"

#ifndef TCX_REAL
#error "define TCX_REAL"
#endif
#define TCX_CAT2(a, b, c) a##b##_##c
#define TCX_CAT(a, b, c) TCX_CAT2(a, b, c)

namespace tcx {
namespace dev {
cudaError_t TCX_CAT(launch_, TCX_TAG, TCX_KM)(int rb, const PassArgs& a, int64_t S, int64_t rows,
                                              size_t smem, cudaStream_t st) {
  switch (rb) {
    case 1: return launch_pass<TCX_REAL, 1, TCX_KM>(a, S, rows, smem, st);
    case 2: return launch_pass<TCX_REAL, 2, TCX_KM>(a, S, rows, smem, st);
    case 3: return launch_pass<TCX_REAL, 3, TCX_KM>(a, S, rows, smem, st);
    case 4: return launch_pass<TCX_REAL, 4, TCX_KM>(a, S, rows, smem, st);
  }
  return cudaErrorInvalidValue;
}
}  // namespace dev
}  // namespace tcx
