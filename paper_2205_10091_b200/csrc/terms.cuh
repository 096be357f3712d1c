// terms.cuh -- per-term expectation values <psi_b|P_j|psi_b> (PAPER.md
// :1046-1084 "batched cost function evaluation": vvag over Pauli structures returns every
// term's value f(w, v_j) next to the summed gradient), included by tcx.cu.
//
// For term j with X/Y flip mask x_j, Y|Z mask zy_j and n_Y Y factors (physical bits of
// the final layout): P_j|r> = i^{n_Y} (-1)^{popc(r & zy_j)} |r ^ x_j>, so
//   <psi|P_j|psi> = sum_r conj(psi[r ^ x_j]) i^{n_Y} (-1)^{popc(r & zy_j)} psi[r]
// (SURVEY §8 conventions).  Grid (S, rows): CTA s of row b owns a contiguous chunk of
// 2^n / S amplitudes, walks it once per term (the chunk stays in L1; partners come from
// L1 / L2), reduces per term over the block in fixed order and writes part[b][s][j];
// terms_sum_kernel adds the S partials in fixed order.  Accumulation in fp64.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "device_common.cuh"

namespace tcx {
namespace dev {

struct TTerm {      // one Pauli string in physical bits
  uint64_t x, zy;
  int32_t ny, pad;
};

template <typename Real>
__global__ void __launch_bounds__(256) terms_kernel(const Cx<Real>* psi, int n, const TTerm* terms,
                                                     int T, double* part, int64_t b0) {
  const int64_t b = b0 + blockIdx.y;
  const int64_t N = 1ll << n;
  const int64_t chunk = N / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * chunk;
  const Cx<Real>* p = psi + b * N;
  __shared__ double red[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = 0; j < T; ++j) {
    const TTerm t = terms[j];
    double sx = 0.0, sy = 0.0;
    for (int64_t r = r0 + tid; r < r0 + chunk; r += blockDim.x) {
      const Cx<Real> a = p[r], c = p[r ^ (int64_t)t.x];
      // conj(c) * a
      double re = (double)c.x * a.x + (double)c.y * a.y;
      double im = (double)c.x * a.y - (double)c.y * a.x;
      if (__popcll((uint64_t)r & t.zy) & 1) { re = -re; im = -im; }
      sx += re;
      sy += im;
    }
    // times i^{n_Y}: only the real part is kept (P_j Hermitian: the total is real)
    double v;
    switch (t.ny & 3) {
      case 0: v = sx; break;
      case 1: v = -sy; break;
      case 2: v = -sx; break;
      default: v = sy; break;
    }
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
      part[((size_t)b * gridDim.x + blockIdx.x) * T + j] = s;
    }
    __syncthreads();
  }
}

__global__ void terms_sum_kernel(const double* part, double* out, int S, int T, int64_t b0) {
  const int64_t b = b0 + blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= T) return;
  double s = 0.0;
  for (int sl = 0; sl < S; ++sl) s += part[((size_t)b * S + sl) * T + j];
  out[(size_t)b * T + j] = s;
}

}  // namespace dev
}  // namespace tcx
