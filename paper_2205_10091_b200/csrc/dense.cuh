// dense.cuh -- dense k-qubit block kernels (north_star step 2), included by
// tcx.cu.
//
// A block is a run of gates fused into one 2^k x 2^k unitary U = G_m ... G_1 on k physical
// bits (plan.cpp build_dense).  Viewing the state as Psi = [2^k x 2^(n-k)] (row j = the
// block bits of the index, column c = the other bits), the forward is Psi' = U Psi: every
// column is a 2^k-vector gathered from 2^k strided amplitudes, multiplied by U and
// scattered back in place.  The column -> index map inserts zero bits at the block
// positions, so consecutive threads take consecutive columns and every gather/scatter
// instruction of a warp is coalesced over the non-block bits.  U sits in shared memory
// and is read with warp-uniform (broadcast) loads; each thread takes COLS columns so one U
// read feeds COLS complex MACs.  Intensity: 8 * 2^k flop per amplitude against 2 * s bytes
// (s = 8 / 16): c128 2^(k-2) flop/B, c64 2^(k-1) flop/B -> HBM-bound up to k = 4 on B200,
// FP32/FP64-ALU bound at k = 5.
//
// Backward (adjoint, k <= 4): per column, psi_in = U^dagger psi_out, lam_in = U^dagger
// lam_out, and the block's gradient needs only R' = sum_c psi_out lam_out^dagger (the
// 2^k x 2^k reduction over all 2^(n-k) columns, SURVEY §8a-5 "R = Psi_in Lambda_out^dagger"
// with R = U^dagger R'): grad_g = coeff_g Im Tr(B_g R'), B_g = S_g P_g S_g^dagger,
// S_g = G_m ... G_{g+1}.  Columns are staged per warp in shared memory and the outer
// products are accumulated GEMM-style into lane-owned R' entries.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "device_common.cuh"
#include "plan.h"

namespace tcx {
namespace dev {

struct DenseMatArgs {
  const DBlock* blocks;
  int nblocks;
  const DGate* gates;
  const double* fixed;
  const double* theta;
  int P;
  void* mats;      // shared table (shared == 1) or [B][dmat_row]
  int64_t row_stride;  // complex entries per theta row (0 for the shared table)
  int shared;      // which blocks this launch materialises
  int64_t b0;
};

struct DenseArgs {
  void* psi;        // [B][2^n]
  void* lam;        // [B][2^n] (backward)
  const void* U;    // block matrix of row 0 (Cx<Real>, row-major 2^k x 2^k)
  int64_t u_stride; // complex entries between rows (0: shared)
  double* part;     // backward: [B][S][dacc_total] fp64 R' partials (re, im interleaved)
  int acc_off, acc_total;
  int bits[kMaxDenseK];
  int n;
  int init;         // forward: input is |0...0> (nothing is read)
  int store;        // backward: write psi_in / lam_in (0 for the first block)
  int64_t b0;
};

// ---- matrices: one thread per column of U, fp64 arithmetic ----------------------------
struct cz {
  double x, y;
};
__device__ __forceinline__ cz zmul(cz a, cz b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ cz zadd(cz a, cz b) { return {a.x + b.x, a.y + b.y}; }

// 2x2 (row-major, m[0..3]) or 4x4 (index 2 b_q0 + b_q1, m[0..15]) matrix of a gate, in the
// conventions of tcx.h / SURVEY §8 (R_P(a) = exp(-i a P / 2), a = coeff * theta[param]).
__device__ void dense_gate_matrix(const DGate& g, const double* th, const double* fixed, cz* m) {
  const double r2 = 0.70710678118654752440;
  const double a = g.param >= 0 ? g.coeff * th[g.param] : g.coeff;
  double cs, sn;
  sincos(0.5 * a, &sn, &cs);
  const int d = g.b >= 0 ? 4 : 2;
  for (int i = 0; i < d * d; ++i) m[i] = {0, 0};
  for (int i = 0; i < d; ++i) m[i * d + i] = {1, 0};
  int kind = g.kind;
  if (kind == TCX_RROT) {  // axis of this row: status column index in the payload
    const double x = th[(int)fixed[2 * g.payload]];
    kind = x < 1.0 / 3.0 ? TCX_RX : (x < 2.0 / 3.0 ? TCX_RY : TCX_RZ);
  }
  switch (kind) {
    case TCX_X: m[0] = {0, 0}; m[1] = {1, 0}; m[2] = {1, 0}; m[3] = {0, 0}; break;
    case TCX_Y: m[0] = {0, 0}; m[1] = {0, -1}; m[2] = {0, 1}; m[3] = {0, 0}; break;
    case TCX_Z: m[3] = {-1, 0}; break;
    case TCX_H: m[0] = {r2, 0}; m[1] = {r2, 0}; m[2] = {r2, 0}; m[3] = {-r2, 0}; break;
    case TCX_S: m[3] = {0, 1}; break;
    case TCX_SDG: m[3] = {0, -1}; break;
    case TCX_T: m[3] = {r2, r2}; break;
    case TCX_TDG: m[3] = {r2, -r2}; break;
    case TCX_RX: m[0] = {cs, 0}; m[1] = {0, -sn}; m[2] = {0, -sn}; m[3] = {cs, 0}; break;
    case TCX_RY: m[0] = {cs, 0}; m[1] = {-sn, 0}; m[2] = {sn, 0}; m[3] = {cs, 0}; break;
    case TCX_RZ: m[0] = {cs, -sn}; m[3] = {cs, sn}; break;
    case TCX_U1:
      for (int i = 0; i < 4; ++i) m[i] = {fixed[2 * (g.payload + i)], fixed[2 * (g.payload + i) + 1]};
      break;
    case TCX_CNOT:  // control q0: |10> <-> |11>
      m[10] = {0, 0}; m[11] = {1, 0}; m[14] = {1, 0}; m[15] = {0, 0}; break;
    case TCX_CZ: m[15] = {-1, 0}; break;
    case TCX_RZZ:
      m[0] = {cs, -sn}; m[5] = {cs, sn}; m[10] = {cs, sn}; m[15] = {cs, -sn}; break;
    case TCX_RXX:  // cos I - i sin X(x)X
      for (int i = 0; i < 4; ++i) { m[i * 4 + i] = {cs, 0}; m[i * 4 + (3 - i)] = {0, -sn}; }
      break;
    case TCX_RYY: {  // cos I - i sin Y(x)Y, Y(x)Y = antidiag(-1, 1, 1, -1)
      const double s4[4] = {-1, 1, 1, -1};
      for (int i = 0; i < 4; ++i) { m[i * 4 + i] = {cs, 0}; m[i * 4 + (3 - i)] = {0, -sn * s4[i]}; }
      break;
    }
    case TCX_U2:
      for (int i = 0; i < 16; ++i) m[i] = {fixed[2 * (g.payload + i)], fixed[2 * (g.payload + i) + 1]};
      break;
    case TCX_DEPOL: {  // Monte Carlo depolarizing: status interval -> I, X, Y, Z
      const double x = th[g.param], px = fixed[2 * g.payload], py = fixed[2 * g.payload + 1],
                   pz = fixed[2 * g.payload + 2];
      if (x < 1.0 - px - py - pz) break;
      if (x < 1.0 - py - pz) { m[0] = {0, 0}; m[1] = {1, 0}; m[2] = {1, 0}; m[3] = {0, 0}; break; }
      if (x < 1.0 - pz) { m[0] = {0, 0}; m[1] = {0, -1}; m[2] = {0, 1}; m[3] = {0, 0}; break; }
      m[3] = {-1, 0};
      break;
    }
    default: break;
  }
}

// apply gate g to the 2^k-vector u (local-bit indexing)
__device__ void dense_apply_gate(const DGate& g, const cz* m, cz* u, int D) {
  if (g.b < 0) {
    const int s = 1 << g.a;
    for (int i = 0; i < D; ++i) {
      if (i & s) continue;
      const cz x0 = u[i], x1 = u[i | s];
      u[i] = zadd(zmul(m[0], x0), zmul(m[1], x1));
      u[i | s] = zadd(zmul(m[2], x0), zmul(m[3], x1));
    }
    return;
  }
  const int sa = 1 << g.a, sb = 1 << g.b;  // 4x4 index 2 b_a + b_b
  for (int i = 0; i < D; ++i) {
    if (i & (sa | sb)) continue;
    const int idx[4] = {i, i | sb, i | sa, i | sa | sb};
    cz x[4], y[4];
    for (int r = 0; r < 4; ++r) x[r] = u[idx[r]];
    for (int r = 0; r < 4; ++r) {
      y[r] = {0, 0};
      for (int c = 0; c < 4; ++c) y[r] = zadd(y[r], zmul(m[r * 4 + c], x[c]));
    }
    for (int r = 0; r < 4; ++r) u[idx[r]] = y[r];
  }
}

// grid (nblocks, rows), 32 threads: thread c builds column c of U = G_m ... G_1.
template <typename Real>
__global__ void dense_mat_kernel(const DenseMatArgs a) {
  const DBlock blk = a.blocks[blockIdx.x];
  if (blk.shared != a.shared) return;
  const int D = 1 << blk.k, c = threadIdx.x;
  if (c >= D) return;
  const int64_t b = a.b0 + blockIdx.y;
  const double* th = a.theta ? a.theta + b * a.P : nullptr;
  cz u[1 << kMaxDenseK], m[16];
  for (int i = 0; i < D; ++i) u[i] = {i == c ? 1.0 : 0.0, 0.0};
  for (int gi = 0; gi < blk.gate_count; ++gi) {
    const DGate g = a.gates[blk.gate_begin + gi];
    dense_gate_matrix(g, th, a.fixed, m);
    dense_apply_gate(g, m, u, D);
  }
  Cx<Real>* out = reinterpret_cast<Cx<Real>*>(a.mats) + b * a.row_stride + blk.mat_off;
  for (int i = 0; i < D; ++i) out[i * D + c] = {(Real)u[i].x, (Real)u[i].y};
}

// ---- forward: Psi' = U Psi ------------------------------------------------------------
template <int K>
__device__ __forceinline__ uint64_t dense_insert(uint64_t c, const int* bits) {
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int p = bits[i];
    c = ((c >> p) << (p + 1)) | (c & ((1ull << p) - 1));
  }
  return c;
}

template <int K>
__device__ __forceinline__ uint64_t dense_off(int j, const int* bits) {
  uint64_t o = 0;
#pragma unroll
  for (int i = 0; i < K; ++i)
    if ((j >> i) & 1) o |= 1ull << bits[i];
  return o;
}

// complex multiply-accumulate, complex128: 4 DFMA
__device__ __forceinline__ void cmac(Cx<double>& acc, Cx<double> u, Cx<double> v) {
  acc.x = fma(u.x, v.x, acc.x);
  acc.x = fma(-u.y, v.y, acc.x);
  acc.y = fma(u.x, v.y, acc.y);
  acc.y = fma(u.y, v.x, acc.y);
}

template <typename Real, int K, int COLS>
__global__ void __launch_bounds__(256) dense_fwd_kernel(const DenseArgs a) {
  using C = Cx<Real>;
  constexpr int D = 1 << K;
  // complex64: U kept as packed FFMA2 operand pairs {(ur, ur), (-ui, ui)} so a complex
  // MAC is 2 FFMA2 (acc += (ur,ur)*(vr,vi) + (-ui,ui)*(vi,vr)); complex128: (ur, ui).
  constexpr bool kF = sizeof(Real) == 4;
  __shared__ __align__(16) double sU[kF ? 2 * D * D : 2 * D * D];
  const int tid = threadIdx.x;
  const int64_t b = a.b0 + blockIdx.y;
  {
    const C* src = reinterpret_cast<const C*>(a.U) + b * a.u_stride;
    for (int i = tid; i < D * D; i += blockDim.x) {
      const C u = src[i];
      if (kF) {
        reinterpret_cast<q64*>(sU)[2 * i] = qpk((float)u.x, (float)u.x);
        reinterpret_cast<q64*>(sU)[2 * i + 1] = qpk(-(float)u.y, (float)u.y);
      } else {
        sU[2 * i] = (double)u.x;
        sU[2 * i + 1] = (double)u.y;
      }
    }
  }
  __syncthreads();
  int bits[K];
#pragma unroll
  for (int i = 0; i < K; ++i) bits[i] = a.bits[i];
  const int64_t N = 1ll << a.n;
  const int64_t ncols = N >> K;
  C* psi = reinterpret_cast<C*>(a.psi) + b * N;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c0 = (int64_t)blockIdx.x * blockDim.x + tid; c0 < ncols; c0 += stride * COLS) {
    uint64_t base[COLS];
    bool ok[COLS];
    C v[COLS][D];
#pragma unroll
    for (int u = 0; u < COLS; ++u) {
      const int64_t c = c0 + u * stride;
      ok[u] = c < ncols;
      base[u] = dense_insert<K>(ok[u] ? (uint64_t)c : 0ull, bits);
      if (a.init) {
#pragma unroll
        for (int j = 0; j < D; ++j) v[u][j] = C{Real((ok[u] && c == 0 && j == 0) ? 1 : 0), Real(0)};
      } else {
#pragma unroll
        for (int j = 0; j < D; ++j)
          if (ok[u]) v[u][j] = psi[base[u] | dense_off<K>(j, bits)];
      }
    }
    // IR output rows at a time: 2 * IR * COLS independent accumulation chains per thread
    constexpr int IR = D < 4 ? D : 4;
#pragma unroll
    for (int i0 = 0; i0 < D; i0 += IR) {
      C acc[IR][COLS];
#pragma unroll
      for (int r = 0; r < IR; ++r)
#pragma unroll
        for (int u = 0; u < COLS; ++u) acc[r][u] = C{Real(0), Real(0)};
#pragma unroll
      for (int j = 0; j < D; ++j) {
#pragma unroll
        for (int r = 0; r < IR; ++r) {
          const int i = i0 + r;
          if (kF) {
            const q64 ur = reinterpret_cast<const q64*>(sU)[2 * (i * D + j)];
            const q64 ui = reinterpret_cast<const q64*>(sU)[2 * (i * D + j) + 1];
#pragma unroll
            for (int u = 0; u < COLS; ++u) {
              const q64 vv = f2u_(*reinterpret_cast<const Cx<float>*>(&v[u][j]));
              q64 ac = f2u_(*reinterpret_cast<const Cx<float>*>(&acc[r][u]));
              ac = qfma(ur, vv, ac);
              ac = qfma(ui, qsw(vv), ac);
              *reinterpret_cast<Cx<float>*>(&acc[r][u]) = u2f_(ac);
            }
          } else {
            const Cx<double> uu{sU[2 * (i * D + j)], sU[2 * (i * D + j) + 1]};
#pragma unroll
            for (int u = 0; u < COLS; ++u)
              cmac(*reinterpret_cast<Cx<double>*>(&acc[r][u]), uu,
                   *reinterpret_cast<const Cx<double>*>(&v[u][j]));
          }
        }
      }
#pragma unroll
      for (int r = 0; r < IR; ++r)
#pragma unroll
        for (int u = 0; u < COLS; ++u)
          if (ok[u]) psi[base[u] | dense_off<K>(i0 + r, bits)] = acc[r][u];
    }
  }
}

// ---- backward: psi_in = U^dagger psi_out, lam_in = U^dagger lam_out, R' partials ------
// 256 threads = 8 warps; a warp takes 32 columns at a time (lane = column).  When the
// block has parameters, the loaded columns are staged in the warp's shared-memory slice
// as [lane][j] and every lane accumulates its E = max(1, D^2 / 32) owned entries
// R'_ij = sum_c psi_c[i] conj(lam_c[j]) (one fp32/fp64 batch sum per 32 columns, added
// into fp64 registers).  At the end the 8 warps' entries are summed in a fixed order and
// the CTA's partial is written to part[b][blockIdx.x][2 D^2] (fp64 re, im).
template <int D>
struct DenseBwdSmem {
  static constexpr int E = D * D >= 32 ? D * D / 32 : 1;
};

template <typename Real, int K>
__global__ void __launch_bounds__(256) dense_bwd_kernel(const DenseArgs a) {
  using C = Cx<Real>;
  constexpr int D = 1 << K;
  constexpr int E = DenseBwdSmem<D>::E;
  constexpr int NW = 8;
  __shared__ __align__(16) C sU[D * D];
  extern __shared__ __align__(16) unsigned char dsm[];
  C* stage = reinterpret_cast<C*>(dsm);  // [NW][2][32][D]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t b = a.b0 + blockIdx.y;
  {
    const C* src = reinterpret_cast<const C*>(a.U) + b * a.u_stride;
    for (int i = tid; i < D * D; i += blockDim.x) sU[i] = src[i];
  }
  __syncthreads();
  int bits[K];
#pragma unroll
  for (int i = 0; i < K; ++i) bits[i] = a.bits[i];
  const bool grad = a.part != nullptr;
  const int64_t N = 1ll << a.n;
  const int64_t ncols = N >> K;
  C* psi = reinterpret_cast<C*>(a.psi) + b * N;
  C* lam = reinterpret_cast<C*>(a.lam) + b * N;
  C* Vs = stage + (size_t)warp * 2 * 32 * D;
  C* Ls = Vs + 32 * D;
  // lane-owned R' entries e = lane * E + q (valid when < D^2): i = e / D, j = e % D
  double accx[E], accy[E];
#pragma unroll
  for (int q = 0; q < E; ++q) accx[q] = accy[q] = 0.0;
  const int e0 = lane * E;
  const int oi = e0 / D, oj = e0 % D;  // E entries share row oi (E <= D)
  const bool own = e0 < D * D;
  const int64_t stride = (int64_t)gridDim.x * NW * 32;
  for (int64_t cb = ((int64_t)blockIdx.x * NW + warp) * 32; cb < ncols; cb += stride) {
    const int64_t c = cb + lane;
    const bool ok = c < ncols;
    const uint64_t base = dense_insert<K>(ok ? (uint64_t)c : 0ull, bits);
    C v[D], l[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (ok) {
        v[j] = psi[base | dense_off<K>(j, bits)];
        l[j] = lam[base | dense_off<K>(j, bits)];
      } else {
        v[j] = C{Real(0), Real(0)};
        l[j] = C{Real(0), Real(0)};
      }
    }
    if (grad) {
      __syncwarp();
#pragma unroll
      for (int j = 0; j < D; ++j) {
        Vs[lane * D + j] = v[j];
        Ls[lane * D + j] = l[j];
      }
      __syncwarp();
      if (own) {
        Real sx[E], sy[E];
#pragma unroll
        for (int q = 0; q < E; ++q) sx[q] = sy[q] = Real(0);
#pragma unroll 4
        for (int m = 0; m < 32; ++m) {
          const C pv = Vs[m * D + oi];
#pragma unroll
          for (int q = 0; q < E; ++q) {
            const C pl = Ls[m * D + oj + q];
            // psi_i * conj(lam_j)
            sx[q] = fma(pv.x, pl.x, fma(pv.y, pl.y, sx[q]));
            sy[q] = fma(pv.y, pl.x, fma(-pv.x, pl.y, sy[q]));
          }
        }
#pragma unroll
        for (int q = 0; q < E; ++q) {
          accx[q] += (double)sx[q];
          accy[q] += (double)sy[q];
        }
      }
    }
    if (a.store && ok) {
      constexpr int IR = D < 4 ? D : 4;  // independent accumulation chains
#pragma unroll
      for (int i0 = 0; i0 < D; i0 += IR) {
        C pv[IR], pl[IR];
#pragma unroll
        for (int r = 0; r < IR; ++r) pv[r] = pl[r] = C{Real(0), Real(0)};
#pragma unroll
        for (int j = 0; j < D; ++j) {
#pragma unroll
          for (int r = 0; r < IR; ++r) {
            const C u = sU[j * D + i0 + r];  // conj(U_ji)
            pv[r].x = fma(u.x, v[j].x, fma(u.y, v[j].y, pv[r].x));
            pv[r].y = fma(u.x, v[j].y, fma(-u.y, v[j].x, pv[r].y));
            pl[r].x = fma(u.x, l[j].x, fma(u.y, l[j].y, pl[r].x));
            pl[r].y = fma(u.x, l[j].y, fma(-u.y, l[j].x, pl[r].y));
          }
        }
#pragma unroll
        for (int r = 0; r < IR; ++r) {
          psi[base | dense_off<K>(i0 + r, bits)] = pv[r];
          lam[base | dense_off<K>(i0 + r, bits)] = pl[r];
        }
      }
    }
  }
  if (!grad) return;
  // fixed-order cross-warp sum of the lane-owned entries
  __syncthreads();
  double* red = reinterpret_cast<double*>(dsm);  // [NW][D*D][2]
  if (own) {
#pragma unroll
    for (int q = 0; q < E; ++q) {
      red[((size_t)warp * D * D + e0 + q) * 2] = accx[q];
      red[((size_t)warp * D * D + e0 + q) * 2 + 1] = accy[q];
    }
  }
  __syncthreads();
  double* out = a.part + ((size_t)b * gridDim.x + blockIdx.x) * (2 * D * D);
  for (int e = tid; e < 2 * D * D; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += red[(size_t)w * 2 * D * D + e];
    out[e] = s;
  }
}

// qim[b][p] = sum of the q contributions of parameter p (fixed CSR order)
__global__ void dense_qim_kernel(const double* qcontrib, int ncontrib, const int32_t* pptr,
                                 const int32_t* plist, int P, double* qim, int64_t b0) {
  const int64_t b = b0 + blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double s = 0.0;
  for (int i = pptr[p]; i < pptr[p + 1]; ++i) s += qcontrib[(size_t)b * ncontrib + plist[i]];
  qim[(size_t)b * P + p] = s;
}

// R'[b][acc_off + e] = sum_s part[b][s][e], fixed order (C10)
__global__ void dense_rsum_kernel(const double* part, double* rs, int S, int ne, int acc_off,
                                  int acc_total, int64_t b0) {
  const int64_t b = b0 + blockIdx.y;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  double s = 0.0;
  for (int sl = 0; sl < S; ++sl) s += part[((size_t)b * S + sl) * ne + e];
  rs[(size_t)b * acc_total + acc_off + e] = s;
}

// Gradient contributions of the parameterised gates of a block (one CTA per (block, row),
// D^2 threads, thread = entry (i, j)): walking the block's gates backwards with
// S = G_m ... G_{g+1}, B_g = S P_g S^dagger and contrib_g = coeff_g Im Tr(B_g R').
struct DenseGradArgs {
  const DBlock* blocks;
  const int32_t* pblocks;  // indices of blocks with parameters
  const DGate* gates;
  const double* fixed;
  const double* theta;
  int P;
  const double* rs;        // [B][acc_total] R' (re, im)
  int acc_total;
  double* contrib;         // [B][ncontrib]
  double* qcontrib;        // optional [B][ncontrib]: -coeff_g Re Tr(B_g R') / 2, the
                           //   contributions to Im <psi|H|d psi/d theta>
  int ncontrib;
  int64_t b0;
};

__global__ void dense_grad_kernel(const DenseGradArgs a) {
  const DBlock blk = a.blocks[a.pblocks[blockIdx.x]];
  const int64_t b = a.b0 + blockIdx.y;
  const int D = 1 << blk.k, DD = D * D, tid = threadIdx.x;
  __shared__ cz S[256], T[256];
  __shared__ double red[256], red2[256];
  const double* th = a.theta + b * a.P;
  const double* Rp = a.rs + (size_t)b * a.acc_total + blk.acc_off;
  const int i = tid / D, j = tid % D;
  if (tid < DD) S[tid] = {i == j ? 1.0 : 0.0, 0.0};
  __syncthreads();
  for (int gi = blk.gate_count - 1; gi >= 0; --gi) {
    const DGate g = a.gates[blk.gate_begin + gi];
    if (g.contrib >= 0) {
      // P_g on local bits (X / Y / Z masks of the rotation generator)
      int xm = 0, ym = 0, zm = 0;
      const int sa = 1 << g.a, sb = g.b >= 0 ? 1 << g.b : 0;
      int gk = g.kind;
      if (gk == TCX_RROT) {
        const double x = th[(int)a.fixed[2 * g.payload]];
        gk = x < 1.0 / 3.0 ? TCX_RX : (x < 2.0 / 3.0 ? TCX_RY : TCX_RZ);
      }
      if (gk == TCX_RX || gk == TCX_RXX) xm = sa | sb;
      if (gk == TCX_RY || gk == TCX_RYY) ym = sa | sb;
      if (gk == TCX_RZ || gk == TCX_RZZ) zm = sa | sb;
      xm |= ym;
      double v = 0.0, vr = 0.0;
      if (tid < DD) {
        // (S P)_im = S_{i, m ^ xm} ph(m), P|m> = ph(m) |m ^ xm>,
        // ph(m) = i^{nY} (-1)^{popc(m & (ym | zm))} (Y|0> = i|1>, Y|1> = -i|0>)
        cz iy = {1, 0};
        for (int t = 0; t < (__popc(ym) & 3); ++t) iy = zmul(iy, cz{0, 1});
        // B_ij = sum_m (S P)_im conj(S_jm)
        cz Bij = {0, 0};
        for (int m = 0; m < D; ++m) {
          const cz p2 = (__popc(m & (ym | zm)) & 1) ? cz{-iy.x, -iy.y} : iy;
          const cz X = zmul(S[i * D + (m ^ xm)], p2);
          const cz Sj = S[j * D + m];
          Bij = zadd(Bij, zmul(X, cz{Sj.x, -Sj.y}));
        }
        // Im(B_ij R'_ji)
        const cz R = {Rp[2 * (j * D + i)], Rp[2 * (j * D + i) + 1]};
        v = Bij.x * R.y + Bij.y * R.x;
        vr = Bij.x * R.x - Bij.y * R.y;
      }
      red[tid] = v;
      red2[tid] = vr;
      __syncthreads();
      if (tid == 0) {
        double s = 0.0, sr = 0.0;
        for (int e = 0; e < DD; ++e) {
          s += red[e];
          sr += red2[e];
        }
        a.contrib[(size_t)b * a.ncontrib + g.contrib] = g.coeff * s;  // 2 Re q = Im Tr(B R')
        if (a.qcontrib) a.qcontrib[(size_t)b * a.ncontrib + g.contrib] = -0.5 * g.coeff * sr;
      }
      __syncthreads();
    }
    // S <- S G_g (row i of S times the gate on the local bits): T_ij = sum_k S_ik G_kj
    cz m[16];
    dense_gate_matrix(g, th, a.fixed, m);
    if (tid < DD) {
      cz acc = {0, 0};
      if (g.b < 0) {
        const int s = 1 << g.a;
        const int j0 = j & ~s, bj = (j >> g.a) & 1;
        acc = zadd(zmul(S[i * D + j0], m[0 * 2 + bj]), zmul(S[i * D + (j0 | s)], m[1 * 2 + bj]));
      } else {
        const int sa = 1 << g.a, sb = 1 << g.b;
        const int j0 = j & ~(sa | sb);
        const int cj = 2 * ((j >> g.a) & 1) + ((j >> g.b) & 1);
        const int kk[4] = {j0, j0 | sb, j0 | sa, j0 | sa | sb};
        for (int r = 0; r < 4; ++r) acc = zadd(acc, zmul(S[i * D + kk[r]], m[r * 4 + cj]));
      }
      T[tid] = acc;
    }
    __syncthreads();
    if (tid < DD) S[tid] = T[tid];
    __syncthreads();
  }
}

}  // namespace dev
}  // namespace tcx
