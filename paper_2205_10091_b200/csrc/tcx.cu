// tcx.cu -- sm_100a kernels and the C ABI of libtcx.so.
//
// Hot path:
//   materialize_kernel  per-theta fused gate matrices / diagonal phases (a2)
//   pass_kernel<Real,RB> window pass over 2^t-amplitude tiles: forward gate stages
//                       (a4), lambda = H psi + E partials fused into the last pass (a6),
//                       adjoint backward stages with <lambda|dG|psi> partials (a7)
//   finalize_kernel     deterministic fp64 reductions -> E[B], grad[B][P] (a8)
// Every step of the path runs in these kernels; there is no host fallback.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <type_traits>
#include <atomic>
#include <thread>

#include "jit.h"
#include "kernels.cuh"
#include "dense.cuh"
#include "dense_tc.cuh"
#include "terms.cuh"
#include "plan.h"

using namespace tcx;

namespace {

thread_local std::string g_err;
tcx_status fail(tcx_status s, const std::string& m) {
  g_err = m;
  return s;
}
struct ProfEntry {
  int phase, index;
  cudaEvent_t a, b;
  double flops, bytes;
};
struct ProfLog {
  bool on = false;
  std::vector<ProfEntry> log;
};
thread_local ProfLog g_prof;

#define CUDA_TRY(x)                                                                    \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      return fail(TCX_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));       \
  } while (0)

// ================================================================== device
using namespace tcx::dev;

// ---- per-theta gate matrices (fp64 math, stored in the state precision)
struct cdd {
  double x, y;
};
__device__ __forceinline__ cdd cmul(cdd a, cdd b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ cdd cadd(cdd a, cdd b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ cdd cconj(cdd a) { return {a.x, -a.y}; }

// TCX_RROT: the rotation axis of this theta row (status column index in the payload)
__device__ __forceinline__ int rrot_kind(const double* theta, const double* fixed, int64_t payload) {
  const double x = theta[(int)fixed[2 * payload]];
  return x < 1.0 / 3.0 ? TCX_RX : (x < 2.0 / 3.0 ? TCX_RY : TCX_RZ);
}

// 1-qubit gate matrix g[0..3] (row-major) -- same conventions as tcx.h
__device__ void gate1(const DCons& c, const double* theta, const double* fixed, cdd* g) {
  const double r2 = 0.70710678118654752440;
  const double a = c.param >= 0 ? c.coeff * theta[c.param] : c.coeff;
  double cs, sn;
  sincos(0.5 * a, &sn, &cs);
  g[0] = {1, 0}; g[1] = {0, 0}; g[2] = {0, 0}; g[3] = {1, 0};
  const int kind = c.kind == TCX_RROT ? rrot_kind(theta, fixed, c.payload) : c.kind;
  switch (kind) {
    case TCX_X: g[0] = {0, 0}; g[1] = {1, 0}; g[2] = {1, 0}; g[3] = {0, 0}; break;
    case TCX_Y: g[0] = {0, 0}; g[1] = {0, -1}; g[2] = {0, 1}; g[3] = {0, 0}; break;
    case TCX_Z: g[3] = {-1, 0}; break;
    case TCX_H: g[0] = {r2, 0}; g[1] = {r2, 0}; g[2] = {r2, 0}; g[3] = {-r2, 0}; break;
    case TCX_S: g[3] = {0, 1}; break;
    case TCX_SDG: g[3] = {0, -1}; break;
    case TCX_T: g[3] = {r2, r2}; break;
    case TCX_TDG: g[3] = {r2, -r2}; break;
    case TCX_RX: g[0] = {cs, 0}; g[1] = {0, -sn}; g[2] = {0, -sn}; g[3] = {cs, 0}; break;
    case TCX_RY: g[0] = {cs, 0}; g[1] = {-sn, 0}; g[2] = {sn, 0}; g[3] = {cs, 0}; break;
    case TCX_RZ: g[0] = {cs, -sn}; g[1] = {0, 0}; g[2] = {0, 0}; g[3] = {cs, sn}; break;
    case TCX_U1:
      for (int i = 0; i < 4; ++i) g[i] = {fixed[2 * (c.payload + i)], fixed[2 * (c.payload + i) + 1]};
      break;
    case TCX_DEPOL: {  // status x = theta[param]: I, X, Y, Z on [0,1) in the paper's order
      const double x = theta[c.param], px = fixed[2 * c.payload], py = fixed[2 * c.payload + 1],
                   pz = fixed[2 * c.payload + 2];
      if (x < 1.0 - px - py - pz) break;
      if (x < 1.0 - py - pz) { g[0] = {0, 0}; g[1] = {1, 0}; g[2] = {1, 0}; g[3] = {0, 0}; break; }
      if (x < 1.0 - pz) { g[0] = {0, 0}; g[1] = {0, -1}; g[2] = {0, 1}; g[3] = {0, 0}; break; }
      g[3] = {-1, 0};
      break;
    }
    default: break;
  }
}
__device__ void mat2mul(const cdd* A, const cdd* B, cdd* O) {  // O = A B
  cdd t[4];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) t[i * 2 + j] = cadd(cmul(A[i * 2], B[j]), cmul(A[i * 2 + 1], B[2 + j]));
  for (int i = 0; i < 4; ++i) O[i] = t[i];
}

struct MatArgs {
  const MItem* items;
  int nitems;
  const DCons* cons;
  const double* fixed;
  const double* theta;
  int P;
  void* mats;
  int mat_total;
  double* tanc;  // [B][ntan] u00 of deferred-factor rotations (fp64), or null
  int ntan;
};

template <typename Real>
__global__ void materialize_kernel(const MatArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.nitems) return;
  const int64_t b = blockIdx.y;
  const double* th = a.theta + b * a.P;
  Real* out = reinterpret_cast<Real*>(a.mats) + b * a.mat_total;
  const MItem it = a.items[i];
  if (it.type == OP_U1) {
    cdd M[4] = {{1, 0}, {0, 0}, {0, 0}, {1, 0}}, G[4];
    for (int c = 0; c < it.cons_count; ++c) {
      gate1(a.cons[it.cons_begin + c], th, a.fixed, G);
      mat2mul(G, M, M);
    }
    double al3 = 0.0;
    if (it.tan == 3) {
      // kind 3: U = |u00| Phi (I + K), Phi = diag(u00, u11) / |u00| (applied by the derived
      // diagonal op); the standard slots carry V = Phi^dagger U = |u00| (I + K), which the
      // plain variant applies
      al3 = sqrt(M[0].x * M[0].x + M[0].y * M[0].y);
      const double r1 = sqrt(M[3].x * M[3].x + M[3].y * M[3].y);
      const cdd e0 = al3 > 0.0 ? cdd{M[0].x / al3, -M[0].y / al3} : cdd{1, 0};  // e^{-i alpha}
      const cdd e1 = r1 > 0.0 ? cdd{M[3].x / r1, -M[3].y / r1} : cdd{1, 0};     // e^{-i beta}
      M[0] = cmul(e0, M[0]);
      M[1] = cmul(e0, M[1]);
      M[2] = cmul(e1, M[2]);
      M[3] = cmul(e1, M[3]);
    }
    if (sizeof(Real) == 8) {
      for (int k = 0; k < 4; ++k) {
        out[it.mat_off + 2 * k] = (Real)M[k].x;
        out[it.mat_off + 2 * k + 1] = (Real)M[k].y;
      }
    } else {
      // packed complex64 layout: m_i = (re, im) of u00, u01, u10, u11 flattened to m0..m7;
      // forward pairs (m_i, m_i) / (-m_i, m_i) for even / odd i, then the adjoint pairs
      // (m0,m0) (m1,-m1) (m4,m4) (m5,-m5) (m2,m2) (m3,-m3) (m6,m6) (m7,-m7).
      const double m[8] = {M[0].x, M[0].y, M[1].x, M[1].y, M[2].x, M[2].y, M[3].x, M[3].y};
      static const int dsrc[8] = {0, 1, 4, 5, 2, 3, 6, 7};
      for (int i = 0; i < 8; ++i) {
        out[it.mat_off + 2 * i] = (Real)((i & 1) ? -m[i] : m[i]);
        out[it.mat_off + 2 * i + 1] = (Real)m[i];
        const double d = m[dsrc[i]];
        out[it.mat_off + 16 + 2 * i] = (Real)d;
        out[it.mat_off + 16 + 2 * i + 1] = (Real)((i & 1) ? -d : d);
      }
    }
    if (it.tan == 3) {
      // K01 = kappa = V01 / |u00|, K10 = kappa' = V10 / |u00|; forward pairs (zr, zr), (-zi, zi)
      // for z = kappa, kappa' (reals 32..39), adjoint I + K^dagger: conj(kappa'), conj(kappa)
      a.tanc[b * a.ntan + it.tan_idx] = al3;
      const double ia = al3 > 0.0 ? 1.0 / al3 : 0.0;
      const double kr = M[1].x * ia, ki = M[1].y * ia, qr = M[2].x * ia, qi = M[2].y * ia;
      Real* o = out + it.mat_off;
      if (sizeof(Real) == 8) {
        o[8] = (Real)kr; o[9] = (Real)ki; o[10] = (Real)qr; o[11] = (Real)qi;
        o[12] = (Real)0; o[13] = (Real)0;
      } else {
        const double z[8][2] = {{kr, kr}, {-ki, ki}, {qr, qr}, {-qi, qi},
                                {qr, qr}, {qi, -qi}, {kr, kr}, {ki, -ki}};
        for (int i = 0; i < 8; ++i) {
          o[32 + 2 * i] = (Real)z[i][0];
          o[33 + 2 * i] = (Real)z[i][1];
        }
        o[48] = (Real)0; o[49] = (Real)0;
      }
    } else if (it.tan) {
      // deferred-factor rotation U = al (I + K): al = u00 = u11 (real for RX / RY runs),
      // K = off-diagonal / al.  XT (RX): K01 = K10 = i tau; RE (RY): K01 = rho, K10 = rho'.
      // The plain coefficients above stay for rows whose pass runs the plain variant.
      const double al = 0.5 * (M[0].x + M[3].x);
      a.tanc[b * a.ntan + it.tan_idx] = al;
      const double ia = al != 0.0 ? 1.0 / al : 0.0;
      double k0, k1;  // XT: tau = Im u01 / al (= Im u10 / al); RE: rho = u01 / al, rho' = u10 / al
      if (it.tan == 1) {
        k0 = k1 = 0.5 * (M[1].y + M[2].y) * ia;
      } else {
        k0 = M[1].x * ia;
        k1 = M[2].x * ia;
      }
      Real* o = out + it.mat_off;
      if (sizeof(Real) == 8) {
        o[8] = (Real)k0;
        o[9] = (Real)k1;
      } else if (it.tan == 1) {
        // packed pairs the XT class never reads (adjoint half, so the generic kernel's reads
        // of pairs 0..7 are untouched): fwd (-tau, tau) pair 10, adjoint (tau, -tau) pair 12
        o[20] = (Real)-k0; o[21] = (Real)k0;
        o[24] = (Real)k0; o[25] = (Real)-k0;
      } else {  // RE: (rho, rho) pair 9, (rho', rho') pair 11
        o[18] = o[19] = (Real)k0;
        o[22] = o[23] = (Real)k1;
      }
    }
  } else if (it.type == OP_U2F) {
    for (int k = 0; k < 32; ++k) out[it.mat_off + k] = (Real)a.fixed[2 * it.payload + k];
  } else if (it.tan == 4) {
    // derived phase of a kind-3 U1 op: Phi = diag(e^{i alpha}, e^{i beta}) = e^{i gamma} e^{i w Z},
    // gamma = (alpha + beta) / 2 (term on mask 0), w = (alpha - beta) / 2 (Z term)
    cdd M[4] = {{1, 0}, {0, 0}, {0, 0}, {1, 0}}, G[4];
    for (int c = 0; c < it.cons_count; ++c) {
      gate1(a.cons[it.cons_begin + c], th, a.fixed, G);
      mat2mul(G, M, M);
    }
    const bool z0 = M[0].x == 0.0 && M[0].y == 0.0, z1 = M[3].x == 0.0 && M[3].y == 0.0;
    const double al = z0 ? 0.0 : atan2(M[0].y, M[0].x), be = z1 ? 0.0 : atan2(M[3].y, M[3].x);
    const double w = it.tan_idx ? 0.5 * (al - be) : 0.5 * (al + be);
    double s, c;
    sincos(w, &s, &c);
    out[it.mat_off] = (Real)c;
    out[it.mat_off + 1] = (Real)s;
  } else {
    const double w = it.param >= 0 ? it.w * th[it.param] : it.w;
    double s, c;
    sincos(w, &s, &c);
    out[it.mat_off] = (Real)c;
    out[it.mat_off + 1] = (Real)s;
  }
}

// Deferred rotation factors (plan.cpp tan_kind_of): per theta row and
// pass, decide whether the pass runs its I + K form or its plain form (both tile loops are in
// the pass's JIT kernel, one uniform branch per CTA), and write the pass header [S_fwd, S_bwd, plain]
// (the factors the forward / backward ops leave to the pass end) and, walking the backward
// in reverse execution order, the correction S^2 of every gradient slot (its psi and lambda
// both carry the factors of the U^dagger applied before it in the pass).
struct ScanArgs {
  const SPass* sp;
  int npass;
  const SFwd* fw;
  const SBwd* bw;
  const double* tanc;
  int ntan;
  void* mats;
  int mat_total;
  double* corr;  // [B][acc_total] or null
  int acc_total;
  int64_t b0;
};
template <typename Real>
__global__ void tan_scan_kernel(const ScanArgs a) {
  const int64_t b = a.b0 + blockIdx.x;
  Real* m = reinterpret_cast<Real*>(a.mats) + b * a.mat_total;
  const double* tc = a.tanc + b * a.ntan;
  double* corr = a.corr ? a.corr + b * a.acc_total : nullptr;
  if (corr)
    for (int k = threadIdx.x; k < a.acc_total; k += blockDim.x) corr[k] = 1.0;
  __syncthreads();
  for (int p = threadIdx.x; p < a.npass; p += blockDim.x) {
    const SPass sp = a.sp[p];
    // kernel values = true state / (product of the |u00| applied so far in the pass): the
    // I + K form is used for the whole pass while that product stays >= 2^-40, so the values,
    // the FP32 products of two of them and their tile sums stay finite
    double prod = 1.0, S = 1.0;
    for (int i = 0; i < sp.fcnt; ++i) {
      const double al = tc[a.fw[sp.fbeg + i].idx];
      prod *= fabs(al);
      S *= al;
    }
    const bool fast = prod >= 0x1p-40;
    double Sb = 1.0;
    for (int i = 0; i < sp.bcnt; ++i) {
      const SBwd w = a.bw[sp.bbeg + i];
      if (w.kind == 0) {
        if (corr && fast)
          for (int k = 0; k < w.b; ++k) corr[w.a + k] = Sb * Sb;
      } else {
        Sb *= tc[w.a];
      }
    }
    m[sp.hdr] = (Real)(fast ? S : 1.0);
    m[sp.hdr + 1] = (Real)(fast ? Sb : 1.0);
    m[sp.hdr + 2] = (Real)(fast ? 0 : 1);
    m[sp.hdr + 3] = (Real)0;
  }
}

struct FinArgs {
  const double* part;   // [B][S][K]
  const double* epart;  // [B][S][EU]
  int S, K, EU;
  const GItem* gitems;
  int ngitems;
  const DCons* cons;
  const double* fixed;
  const double* theta;
  int P;
  const int32_t* pptr;
  const int32_t* plist;
  int ncontrib;
  double* tot;          // [B][K]
  double* contrib;      // [B][ncontrib]
  double* qcontrib;     // optional [B][ncontrib]: Im <psi|H|d psi> contributions (q_grad)
  double* E;
  double* grad;         // may be null
  int64_t b0;
  const double* corr;   // [B][K] deferred-factor corrections of the slot sums, or null
};

// Deterministic fixed-order fp64 reductions (C10) and the gradient
// contraction grad_g = coeff_g Im Tr(B_g R') with B_g = S_g P_g S_g^dagger,
// S_g = G_m ... G_{g+1} (SURVEY §8a-5 block adjoint, restricted to 1-qubit blocks).
__global__ void finalize_kernel(const FinArgs a) {
  const int64_t b = a.b0 + blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double red[256];
  // E
  {
    double s = 0.0;
    const int tot = a.S * a.EU;
    const int per = (tot + nt - 1) / nt;
    const double* src = a.epart + b * (int64_t)tot;
    for (int i = tid * per; i < min(tot, (tid + 1) * per); ++i) s += src[i];
    red[tid] = s;
    __syncthreads();
    if (tid == 0) {
      double e = 0.0;
      for (int i = 0; i < nt; ++i) e += red[i];
      a.E[b] = e;
    }
  }
  if (!a.grad) return;
  const double* th = a.theta + b * a.P;
  double* tot = a.tot + b * a.K;
  for (int k = tid; k < a.K; k += nt) {
    double s = 0.0;
    const double* src = a.part + b * (int64_t)a.S * a.K + k;
    for (int sl = 0; sl < a.S; ++sl) s += src[(int64_t)sl * a.K];
    tot[k] = a.corr ? s * a.corr[b * a.K + k] : s;
  }
  __syncthreads();
  double* ctb = a.contrib + b * a.ncontrib;
  for (int gi = tid; gi < a.ngitems; gi += nt) {
    const GItem g = a.gitems[gi];
    if (g.type == OP_DIAG) {
      ctb[g.contrib] = g.factor * tot[g.acc];  // 2 Re q
      if (a.qcontrib && g.re_acc >= 0)           // Im q = w sum s Re(lambda* psi)
        a.qcontrib[b * a.ncontrib + g.contrib] = -0.5 * g.factor * tot[g.re_acc];
      continue;
    }
    // Pauli components of R' (device_common.cuh accum_c3): Im Tr(B R') = bx c0 + by c1 + bz c2
    // structured classes carry only the component their generators read (plan.cpp op_accs)
    double c3[3] = {0.0, 0.0, 0.0}, r3[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < 3; ++k) {
      if (g.cls && k != g.cls - 1) continue;
      c3[k] = tot[g.acc + (g.cls ? 0 : k)];
      if (g.re_acc >= 0) r3[k] = tot[g.re_acc + (g.cls ? 0 : k)];
    }
    // kind-3 ops (plan.cpp tan_kind_of): R' was accumulated before the diagonal phase Phi =
    // diag(e^{i alpha}, e^{i beta}), so B' = Phi^dagger B Phi: B'01 = B01 e^{i (beta - alpha)}
    cdd ph01 = {1, 0};
    if (g.phase) {
      cdd U[4] = {{1, 0}, {0, 0}, {0, 0}, {1, 0}}, G0[4];
      for (int c = 0; c < g.cons_count; ++c) {
        gate1(a.cons[g.cons_begin + c], th, a.fixed, G0);
        mat2mul(G0, U, U);
      }
      const double r0 = sqrt(U[0].x * U[0].x + U[0].y * U[0].y), r1 = sqrt(U[3].x * U[3].x + U[3].y * U[3].y);
      const cdd e0 = r0 > 0.0 ? cdd{U[0].x / r0, -U[0].y / r0} : cdd{1, 0};  // e^{-i alpha}
      const cdd e1 = r1 > 0.0 ? cdd{U[3].x / r1, U[3].y / r1} : cdd{1, 0};   // e^{+i beta}
      ph01 = cmul(e0, e1);
    }
    cdd Sfx[4] = {{1, 0}, {0, 0}, {0, 0}, {1, 0}};
    for (int c = g.cons_count - 1; c >= 0; --c) {
      const DCons cn = a.cons[g.cons_begin + c];
      if (cn.contrib >= 0) {  // differentiable rotations only (not depolarizing statuses)
        cdd Pm[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
        const int ck = cn.kind == TCX_RROT ? rrot_kind(th, a.fixed, cn.payload) : cn.kind;
        if (ck == TCX_RX) { Pm[1] = {1, 0}; Pm[2] = {1, 0}; }
        if (ck == TCX_RY) { Pm[1] = {0, -1}; Pm[2] = {0, 1}; }
        if (ck == TCX_RZ) { Pm[0] = {1, 0}; Pm[3] = {-1, 0}; }
        cdd T1[4], Bm[4], Sd[4] = {cconj(Sfx[0]), cconj(Sfx[2]), cconj(Sfx[1]), cconj(Sfx[3])};
        mat2mul(Sfx, Pm, T1);
        mat2mul(T1, Sd, Bm);
        // B Hermitian traceless: B = bx X + by Y + bz Z, B01 = bx - i by, B00 = bz
        const cdd b01 = cmul(Bm[1], ph01);
        const double bx = b01.x, by = -b01.y, bz = Bm[0].x;
        ctb[cn.contrib] = cn.coeff * (bx * c3[0] + by * c3[1] + bz * c3[2]);
        if (a.qcontrib && g.re_acc >= 0)  // Im q = -coeff Re Tr(B R') / 2
          a.qcontrib[b * a.ncontrib + cn.contrib] =
              -0.5 * cn.coeff * (bx * r3[0] + by * r3[1] + bz * r3[2]);
      }
      cdd G[4];
      gate1(cn, th, a.fixed, G);
      mat2mul(Sfx, G, Sfx);
    }
  }
  __syncthreads();
  for (int p = tid; p < a.P; p += nt) {
    double s = 0.0;
    for (int i = a.pptr[p]; i < a.pptr[p + 1]; ++i) s += ctb[a.plist[i]];
    a.grad[b * a.P + p] = s;
  }
}

// H on one index bit of every row (input states of a plan whose leading H gates were
// folded into the |+> initial state: the _in entries apply them explicitly)
template <typename Real>
__global__ void hadamard_bit_kernel(Cx<Real>* psi, int n, int bit, int64_t pairs_total) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= pairs_total) return;
  const int64_t half = (int64_t)1 << (n - 1);
  const int64_t b = i / half, p = i % half;
  const int64_t lo = p & (((int64_t)1 << bit) - 1);
  const int64_t r0 = ((p >> bit) << (bit + 1)) | lo, r1 = r0 | ((int64_t)1 << bit);
  Cx<Real>* s = psi + (b << n);
  const Real k = Real(0.70710678118654752440);
  const Cx<Real> x0 = s[r0], x1 = s[r1];
  s[r0] = Cx<Real>{k * (x0.x + x1.x), k * (x0.y + x1.y)};
  s[r1] = Cx<Real>{k * (x0.x - x1.x), k * (x0.y - x1.y)};
}

// cut table of a LUT op's (mask, sign) set: c(r) = #{k : parity(r & m_k) xor s_k odd}
__global__ void cut_table_kernel(uint8_t* out, int64_t N, const uint64_t* masks, const int* signs,
                                 int T) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N;
       r += (int64_t)gridDim.x * blockDim.x) {
    int c = 0;
    for (int k = 0; k < T; ++k) c += (__popcll((uint64_t)r & masks[k]) & 1) ^ signs[k];
    out[r] = (uint8_t)c;
  }
}

// gather physical -> paper index order (only when SWAP relabels moved qubits)
template <typename Real>
__global__ void export_kernel(const Cx<Real>* src, Cx<Real>* dst, int n, int64_t total,
                              const int* layout) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int64_t N = 1ll << n;
  const int64_t b = i >> n, r = i & (N - 1);
  int64_t phys = 0;
  for (int q = 0; q < n; ++q)
    if ((r >> (n - 1 - q)) & 1) phys |= 1ll << layout[q];
  dst[b * N + r] = src[b * N + phys];
}

// ================================================================== host
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

}  // namespace

namespace tcx {
struct DeviceTables {
  DevBuf kops, kterms, kstages, mitems, dcons, gitems, pptr, plist, fixed, layout, swb;
  DevBuf dblocks, dgates, dpblocks;  // dense k-qubit blocks (dense.cuh)
  DevBuf spass, sfwd, sbwd;          // deferred-factor scan program (tan_scan_kernel)
  DevBuf cut[15];                    // LUT cut tables (Plan::cut_sets), 2^nloc bytes each
  std::map<std::string, CUfunction> jit;   // key (jit.h)
  std::map<std::string, size_t> jit_smem;  // dynamic smem opted in per function
  std::map<std::string, CUmodule> jit_mod;  // key -> its module (unloaded on eviction)
  std::vector<CUmodule> modules;           // loaded JIT modules (unloaded with the plan)
  ~DeviceTables();
};
}  // namespace tcx

struct tcx_circuit {
  Plan plan;
};
struct tcx_pauli {
  Pauli p;
};

namespace {

template <typename T>
tcx_status upload(DevBuf& d, const std::vector<T>& v) {
  size_t bytes = std::max<size_t>(sizeof(T) * v.size(), 16);
  CUDA_TRY(cudaMalloc(&d.p, bytes));
  if (!v.empty()) CUDA_TRY(cudaMemcpy(d.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return TCX_OK;
}

// Driver API through the runtime's entry-point query (no link-time libcuda dependency).
struct Drv {
  bool ok = false;
  CUresult (*moduleLoadData)(CUmodule*, const void*);
  CUresult (*moduleUnload)(CUmodule);
  CUresult (*moduleGetFunction)(CUfunction*, CUmodule, const char*);
  CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                           unsigned, CUstream, void**, void**);
  CUresult (*funcSetAttribute)(CUfunction, CUfunction_attribute, int);
  CUresult (*launchKernelEx)(const CUlaunchConfig*, CUfunction, void**, void**);
  CUresult (*tensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
};
Drv& drv() {
  static Drv D;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, void** fp) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fp, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess;
    };
    D.ok = get("cuModuleLoadData", (void**)&D.moduleLoadData) &&
           get("cuModuleUnload", (void**)&D.moduleUnload) &&
           get("cuModuleGetFunction", (void**)&D.moduleGetFunction) &&
           get("cuLaunchKernel", (void**)&D.launchKernel) &&
           get("cuFuncSetAttribute", (void**)&D.funcSetAttribute) &&
           get("cuLaunchKernelEx", (void**)&D.launchKernelEx) &&
           get("cuTensorMapEncodeTiled", (void**)&D.tensorMapEncodeTiled);
  });
  return D;
}

}  // namespace

tcx::DeviceTables::~DeviceTables() {
  Drv& D = drv();
  if (D.ok)
    for (CUmodule m : modules) D.moduleUnload(m);
}
tcx::Binding::~Binding() {
  for (auto& kv : dev) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(kv.first);
    cudaFree(kv.second.first);
    cudaFree(kv.second.second);
    cudaSetDevice(cur);
  }
}

namespace {

// Tensor map of a [B][2^n] state buffer viewed through a pass window (plan.cpp tma_dims):
// 8-byte elements, box = one tile, no swizzle (the kernels read the dense tile in the
// load/store thread mapping, which is bank-conflict free).
bool encode_tmap(void* out, void* base, const TmaDims& td, int n, int64_t B) {
  Drv& D = drv();
  if (!D.ok || td.rank == 0 || !base) return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], estr[5];
  const uint64_t total = (uint64_t)B << n;  // amplitudes
  for (int d = 0; d < td.rank; ++d) {
    const uint64_t elems = total * (uint64_t)td.epa;
    dims[d] = td.bits[d] >= 0 ? (1ull << td.bits[d]) : (elems >> td.start[d]);
    box[d] = td.inwin[d] ? (cuuint32_t)(1u << td.bits[d]) : 1u;
    estr[d] = 1;
    if (d > 0) strides[d - 1] = (1ull << td.start[d]) * 8ull;
    if (dims[d] == 0 || dims[d] > (1ull << 32)) return false;
  }
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(out);
  return D.tensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, (cuuint32_t)td.rank, base, dims,
                                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

tcx_status device_tables(Plan& P, DeviceTables*& out) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(P.mu);
  auto it = P.dev.find(dev);
  if (it != P.dev.end()) {
    out = it->second.get();
    return TCX_OK;
  }
  auto T = std::make_shared<DeviceTables>();
  tcx_status s;
  std::vector<uint32_t> swb(16);
  for (int p = 0; p < 16; ++p) swb[p] = swizzle_bit(p, P.dtype == TCX_C128);
  if ((s = upload(T->swb, swb))) return s;
  if ((s = upload(T->kops, P.kops)) || (s = upload(T->kterms, P.kterms)) ||
      (s = upload(T->kstages, P.kstages)) || (s = upload(T->mitems, P.mitems)) ||
      (s = upload(T->dcons, P.dcons)) || (s = upload(T->gitems, P.gitems)) ||
      (s = upload(T->pptr, P.param_ptr)) || (s = upload(T->plist, P.param_list)) ||
      (s = upload(T->fixed, P.fixed)) || (s = upload(T->spass, P.spass)) ||
      (s = upload(T->sfwd, P.sfwd)) || (s = upload(T->sbwd, P.sbwd)))
    return s;
  std::vector<int> lay(P.layout, P.layout + P.n);
  if ((s = upload(T->layout, lay))) return s;
  std::vector<int32_t> pbl;
  for (size_t i = 0; i < P.dblocks.size(); ++i)
    if (P.dblocks[i].has_param) pbl.push_back((int32_t)i);
  if ((s = upload(T->dblocks, P.dblocks)) || (s = upload(T->dgates, P.dgates)) ||
      (s = upload(T->dpblocks, pbl)))
    return s;
  for (size_t c = 0; c < P.cut_sets.size() && c < 15; ++c) {  // built once per plan and device
    std::vector<uint64_t> m;
    std::vector<int> sg;
    for (auto& kv : P.cut_sets[c]) {
      m.push_back(kv.first);
      sg.push_back(kv.second);
    }
    DevBuf dm, ds;
    if ((s = upload(dm, m)) || (s = upload(ds, sg))) return s;
    const int64_t N = (int64_t)1 << P.nloc;
    CUDA_TRY(cudaMalloc(&T->cut[c].p, (size_t)N));
    cut_table_kernel<<<(unsigned)std::min<int64_t>(4096, (N + 255) / 256), 256>>>(
        (uint8_t*)T->cut[c].p, N, (const uint64_t*)dm.p, (const int*)ds.p, (int)m.size());
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());  // dm / ds are freed on return
  }
  out = T.get();
  P.dev[dev] = T;
  return TCX_OK;
}

// Specialised kernel for (pass, km): compiled (NVRTC / disk cache) and loaded into this
// device's context on first use.  Returns nullptr when the plan runs generic kernels.
tcx_status jit_function(Plan& P, DeviceTables* DT, const std::string& key, CUfunction* f) {
  *f = nullptr;
  if (!P.jit_on) return TCX_OK;
  {
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = DT->jit.find(key);
    if (it != DT->jit.end()) {
      *f = it->second;
      return TCX_OK;
    }
  }
  std::string err;
  if (!jit_build(P, {key}, err)) return fail(TCX_E_CUDA, err);
  Drv& D = drv();
  if (!D.ok) return fail(TCX_E_CUDA, "driver entry points unavailable for JIT kernels");
  CUDA_TRY(cudaFree(0));  // primary context current on this thread
  CUmodule m;
  CUfunction fn;
  if (D.moduleLoadData(&m, P.jit.at(key).cubin.data()) != CUDA_SUCCESS) {
    // a stale or damaged cache entry: drop it, compile afresh, and try once more
    jit_evict(P, key);
    if (!jit_build(P, {key}, err)) return fail(TCX_E_CUDA, err);
    if (D.moduleLoadData(&m, P.jit.at(key).cubin.data()) != CUDA_SUCCESS)
      return fail(TCX_E_CUDA, "cuModuleLoadData failed for " + P.jit.at(key).name);
  }
  const JitKernel& k = P.jit.at(key);
  if (D.moduleGetFunction(&fn, m, k.name.c_str()) != CUDA_SUCCESS)
    return fail(TCX_E_CUDA, "cuModuleGetFunction failed for " + k.name);
  std::lock_guard<std::mutex> lk(P.mu);
  DT->modules.push_back(m);
  DT->jit_mod[key] = m;
  DT->jit[key] = fn;
  DT->jit_smem[key] = 0;
  *f = fn;
  return TCX_OK;
}

// Compile every specialised kernel a call of this kind needs, in parallel, before launching.
// grad with one lambda unit: the last forward pass, lambda = H psi and that pass's backward
// run as one kernel per tile (no store / reload of psi and lambda in between)
int jit_key_pass_index(const std::string& key) {  // "p<pass>k<km>"
  return atoi(key.c_str() + 1);
}

bool fuse_last_of(const Plan& P, int kind, bool mega, const Binding* Bd) {
  static const bool no_fuse = getenv("TCX_NO_FUSE_LAST") != nullptr;
  return !no_fuse && kind == 1 && !mega && P.gbits == 0 && P.dblocks.empty() &&
         P.passes.size() > 1 && Bd && Bd->units.size() == 1;
}

tcx_status jit_prepare(Plan& P, int kind, bool mega, const Binding* Bd, bool fuse_last) {
  if (!P.jit_on) return TCX_OK;
  std::vector<std::string> keys;
  if (P.cluster) {  // one megakernel (state kernels are not available for these plans)
    if (!Bd || kind == 2) return TCX_OK;
    std::string err;
    if (!jit_build(P, {jit_key_cluster(Bd->hash, kind == 1 ? 1 : 0)}, err)) return fail(TCX_E_CUDA, err);
    return TCX_OK;
  }
  const int nP = (int)P.passes.size();
  // kernels that compute lambda = H psi of unit 0 carry the binding (specialised terms)
  auto lam_key = [&](int p, int km) {
    return (Bd && kind != 2) ? jit_key_pass_lam(p, km, Bd->hash) : jit_key_pass(p, km);
  };
  if (mega) {
    keys.push_back(lam_key(0, kind == 1 ? 2 : 0));
  } else {
    for (int p = 0; p < nP; ++p) {
      if (fuse_last && p == nP - 1) {  // last pass: forward + lambda + backward in one kernel
        keys.push_back(lam_key(p, 2));
        continue;
      }
      const bool lam_here = p == nP - 1 && P.gbits == 0;
      keys.push_back(lam_here ? lam_key(p, 0) : jit_key_pass(p, 0));
      if (kind == 1) keys.push_back(jit_key_pass(p, 1));
    }
    if (Bd)
      for (int u = P.gbits > 0 ? 0 : 1; u < (int)Bd->units.size(); ++u)
        keys.push_back(jit_key_lambda(Bd->hash, u));
  }
  std::string err;
  if (!jit_build(P, keys, err)) return fail(TCX_E_CUDA, err);
  return TCX_OK;
}

struct BindDev {
  KGroup* groups;
  KPTerm* pterms;
};

// Bindings (lambda schedule, device term tables, per-unit JIT kernels) of at most this many
// Hamiltonians stay cached per plan; beyond it the least recently used one is dropped.
constexpr size_t kMaxBindings = 64;

void evict_binding_locked(Plan& P, uint64_t hash) {  // P.mu held
  P.bindings.erase(hash);
  P.binding_use.erase(hash);
  // its kernels: lambda units "L<hex>u*", specialised pass kernels "p*k*h<hex>", cluster "C<hex>g*"
  const std::string hex = jit_key_lambda(hash, 0).substr(1, 16);
  auto mine = [&](const std::string& k) {
    return (k[0] == 'L' || k[0] == 'C') ? k.compare(1, 16, hex) == 0
                                        : (k.size() > 16 && k.compare(k.size() - 16, 16, hex) == 0 &&
                                           k[k.size() - 17] == 'h');
  };
  {
    std::lock_guard<std::mutex> jl(P.jit_mu);
    for (auto it = P.jit.begin(); it != P.jit.end();)
      it = mine(it->first) ? P.jit.erase(it) : std::next(it);
  }
  bool synced = false;
  Drv& D = drv();
  for (auto& kv : P.dev) {
    DeviceTables* DT = kv.second.get();
    for (auto it = DT->jit.begin(); it != DT->jit.end();) {
      if (!mine(it->first)) {
        ++it;
        continue;
      }
      auto mi = DT->jit_mod.find(it->first);
      if (mi != DT->jit_mod.end()) {
        if (!synced) {  // its kernels may still be queued: unload only once the devices idle
          int cur = 0;
          cudaGetDevice(&cur);
          for (auto& d2 : P.dev) {
            cudaSetDevice(d2.first);
            cudaDeviceSynchronize();
          }
          cudaSetDevice(cur);
          synced = true;
        }
        if (D.ok) D.moduleUnload(mi->second);
        DT->modules.erase(std::remove(DT->modules.begin(), DT->modules.end(), mi->second),
                          DT->modules.end());
        DT->jit_mod.erase(mi);
      }
      DT->jit_smem.erase(it->first);
      it = DT->jit.erase(it);
    }
  }
}

tcx_status binding_for(Plan& P, const tcx_pauli* H, std::shared_ptr<Binding>& out, BindDev* dv) {
  {
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = P.bindings.find(H->p.hash);
    if (it != P.bindings.end()) out = it->second;
  }
  if (!out) {
    auto b = bind(P, H->p);
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = P.bindings.find(H->p.hash);
    if (it != P.bindings.end())
      out = it->second;
    else
      P.bindings[H->p.hash] = out = b;
  }
  {
    std::lock_guard<std::mutex> lk(P.mu);
    P.binding_use[H->p.hash] = ++P.use_clock;
    while (P.bindings.size() > kMaxBindings) {
      uint64_t victim = 0, oldest = UINT64_MAX;
      for (auto& u : P.binding_use)
        if (u.first != H->p.hash && u.second < oldest) {
          oldest = u.second;
          victim = u.first;
        }
      if (oldest == UINT64_MAX) break;
      evict_binding_locked(P, victim);
    }
  }
  if (!out->xmask_ok) return fail(TCX_E_UNSUPPORTED, out->err);
  if (dv) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = out->dev.find(dev);
    if (it == out->dev.end()) {
      void *g = nullptr, *t = nullptr;
      size_t gb = std::max<size_t>(16, sizeof(KGroup) * out->groups.size());
      size_t tb = std::max<size_t>(16, sizeof(KPTerm) * out->pterms.size());
      CUDA_TRY(cudaMalloc(&g, gb));
      CUDA_TRY(cudaMalloc(&t, tb));
      if (!out->groups.empty())
        CUDA_TRY(cudaMemcpy(g, out->groups.data(), sizeof(KGroup) * out->groups.size(), cudaMemcpyHostToDevice));
      if (!out->pterms.empty())
        CUDA_TRY(cudaMemcpy(t, out->pterms.data(), sizeof(KPTerm) * out->pterms.size(), cudaMemcpyHostToDevice));
      it = out->dev.emplace(dev, std::make_pair(g, t)).first;
    }
    dv->groups = (KGroup*)it->second.first;
    dv->pterms = (KPTerm*)it->second.second;
  }
  return TCX_OK;
}

int tiles_per_cta(const Plan& P) { return P.tpc; }

enum { K_EXPECT = 0, K_GRAD = 1, K_STATE = 2 };

struct WsLayout {
  size_t psi, lam, mats, part, epart, tot, contrib, theta, E, grad, total;
  size_t tanc, corr;  // deferred-factor rotations: u00 per row, slot corrections (0: none)
  size_t dmats, dshared, dpart, drs, dq;  // dense blocks: U tables, R' partials / sums, q
  bool mega;
};

// Dense backward CTAs per theta row (fixed by n alone, so a row's reduction order never
// depends on B): 2^(n-13) clamped to [1, 32].
int dense_bwd_ctas(const Plan& P) { return (int)std::min<int64_t>(32, std::max<int64_t>(1, (int64_t)1 << std::max(0, P.n - 13))); }
int dense_max_k(const Plan& P) {
  int k = 0;
  for (auto& d : P.dblocks) k = std::max(k, (int)d.k);
  return k;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// JIT pass kernels: interleaved tile order (PassArgs.tile_ilv = 1) when a launch has at most two
// CTAs per SM per row, else blocked (0) or grouped (g); TCX_TILE_ORDER=0/1/g forces one for A/B
int tile_order_ilv(int64_t ctas_per_row, int run_bytes) {
  static const int forced = [] {
    const char* e = getenv("TCX_TILE_ORDER");
    return e ? atoi(e) : -1;
  }();
  if (forced >= 0) return forced;  // 0 blocked, 1 interleaved, g >= 2 groups of g CTAs
  static int nsm[64] = {0};
  int dev = 0, sms = 148;  // B200; used when no device is visible (plan-time on a CPU host)
  if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64) {
    if (!nsm[dev] && cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      nsm[dev] = 148;
    sms = nsm[dev];
  } else {
    cudaGetLastError();
  }
  if (ctas_per_row <= 2 * (int64_t)sms) return 1;
  // one huge row: blocked order, but 32-byte runs go in groups of 4 neighbouring CTAs so the
  // four sectors of a line are read together (cfg5 backward: 367 -> 142 GB of DRAM reads per
  // pass for 137 GB of psi and lambda, 0.685 -> 0.692 circuits/s; session 3, t16)
  return run_bytes <= 32 ? 4 : 0;
}

WsLayout ws_layout(const Plan& P, const Binding* Bd, int64_t B, int kind, bool host_io,
                   bool inputs = false) {
  WsLayout w{};
  const size_t rs = P.dtype == TCX_C128 ? 8 : 4;
  const size_t N = size_t(1) << P.nloc;  // this rank's amplitudes (= 2^n unless sharded)
  // partial slots per theta row: tiles / CTA, or the CTAs of a cluster-resident row
  const int64_t S = P.cluster ? ((int64_t)1 << P.gbits) : P.tiles / tiles_per_cta(P);
  const int EU = Bd ? (int)Bd->units.size() : 1;
  w.mega = kind != K_STATE && ((P.passes.size() == 1 && EU == 1 && P.gbits == 0 &&
                                P.dblocks.empty() && !inputs) || P.cluster);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + std::max<size_t>(bytes, 16));
    return o;
  };
  const bool need_psi = !w.mega;
  const bool need_lam = kind == K_GRAD && !w.mega;
  w.psi = need_psi ? take(B * N * 2 * rs) : 0;
  // psi and lambda tiles are read and written together at the same relative offset; with a
  // power-of-two state array they would sit exactly 2^k bytes apart (same DRAM channel / L2
  // set hash for every pair), so lambda starts a small odd number of 256-byte units later
  static const size_t lam_pad = [] {
    const char* e = getenv("TCX_LAM_PAD");
    return e ? (size_t)atoll(e) : (size_t)0;
  }();
  if (need_lam && lam_pad) off = align256(off + lam_pad);
  w.lam = need_lam ? take(B * N * 2 * rs) : 0;
  w.mats = take(B * std::max(P.mat_total, 1) * rs);
  w.part = kind == K_GRAD ? take(B * S * std::max(P.acc_total, 1) * 8) : 0;
  w.epart = kind != K_STATE ? take(B * S * EU * 8) : 0;
  w.tot = kind == K_GRAD ? take(B * std::max(P.acc_total, 1) * 8) : 0;
  w.contrib = kind == K_GRAD ? take(B * std::max(P.n_contrib, 1) * 8) : 0;
  w.tanc = P.ntan > 0 ? take(B * P.ntan * 8) : 0;
  w.corr = P.ntan > 0 && kind == K_GRAD ? take(B * std::max(P.acc_total, 1) * 8) : 0;
  if (!P.dblocks.empty()) {
    w.dmats = take(B * std::max(P.dmat_row, 1) * 2 * rs);
    w.dshared = take(std::max(P.dmat_shared, 1) * 2 * rs);
    if (kind == K_GRAD && P.dacc_total > 0) {
      const int k = dense_max_k(P);
      w.dpart = take((size_t)B * dense_bwd_ctas(P) * 2 * (1 << (2 * k)) * 8);
      w.drs = take((size_t)B * P.dacc_total * 8);
      w.dq = take((size_t)B * std::max(P.n_contrib, 1) * 8);
    }
  }
  if (P.dblocks.empty() && P.q_grad && kind == K_GRAD)
    w.dq = take((size_t)B * std::max(P.n_contrib, 1) * 8);
  if (host_io) {
    w.theta = take(B * std::max(P.P, 1) * 8);
    w.E = take(B * 8);
    w.grad = kind == K_GRAD ? take(B * std::max(P.P, 1) * 8) : 0;
  }
  w.total = off;
  return w;
}

// per-term values: CTAs per row (fixed by n alone) and the workspace behind the state layout
int terms_ctas(const Plan& P) {
  return (int)std::min<int64_t>(128, std::max<int64_t>(1, (int64_t)1 << std::max(0, P.n - 11)));
}
size_t terms_extra(const Plan& P, int64_t B, int T) {
  return align256((size_t)B * terms_ctas(P) * std::max(T, 1) * 8) +
         align256(sizeof(TTerm) * std::max(T, 1));
}

// ---- algorithmic cost model: real flops per amplitude, complex
// multiply = 6, complex add = 2, real x complex = 2.
double op_flops(const Op& o, bool bwd) {
  const double nt = (double)o.terms.size();
  double npar = 0;
  for (auto& t : o.terms) npar += t.param >= 0;
  switch (o.type) {
    case OP_U1:
      if (!bwd && o.fold_init) return 0.0;  // written by the first pass's product init
      // gradient: 3 Pauli components of R' = 12 FMA per pair (one component: 4); ops no
      // earlier op touches skip U^dagger in the backward (plan.cpp skip_udag)
      if (u1_class(o.cons))  // structured: real scalar x complex terms
        return bwd ? (o.skip_udag ? 0.0 : 12.0) + (o.has_param ? 4.0 : 0.0) : 6.0;
      return bwd ? (o.skip_udag ? 0.0 : 28.0) + (o.has_param ? 12.0 : 0.0) : 14.0;
    case OP_U2F: return bwd ? 60.0 : 30.0;
    case OP_CX: return 0.0;
    default:
      // one complex multiply per amplitude per phase group (LUT: one table entry); the
      // backward conjugate-multiplies psi and lambda and accumulates Im(lambda* psi) terms
      if (o.lut) return bwd ? (o.skip_udag ? 0.0 : 12.0) + (o.has_param ? 4.0 : 0.0) : 6.0;
      (void)nt;
      return bwd ? (o.skip_udag ? 0.0 : 12.0 * std::max(o.ngroups, 1)) + 2.0 * npar
                 : 6.0 * std::max(o.ngroups, 1);
  }
}
double pass_flops(const Plan& P, const PassInfo& p, bool bwd) {
  double f = 0;
  for (int i : p.ops) f += op_flops(P.ops[i], bwd);
  return f;
}
double lambda_flops(const Binding& B, const LamUnit& u) {
  double f = 4.0;
  for (int g = u.group_begin; g < u.group_begin + u.group_count; ++g)
    f += 8.0 + 2.0 * B.groups[g].term_count;
  return f;
}

// ---- dense block launches (dense.cuh) -------------------------------------------------
template <typename Real, int K>
void dense_fwd_launch(DenseArgs& a, int64_t rows, cudaStream_t st) {
  // columns per thread: enough bytes in flight per thread for the HBM-bound small blocks
  constexpr int COLS = sizeof(Real) == 4 ? (K == 1 ? 4 : (K == 2 ? 2 : 1)) : (K == 1 ? 2 : 1);
  const int64_t ncols = ((int64_t)1 << a.n) >> K;
  const int64_t need = (ncols + 256 * COLS - 1) / (256 * COLS);
  const int64_t gx = std::max<int64_t>(1, std::min<int64_t>(need, std::max<int64_t>(1, 148 * 8 / rows)));
  dense_fwd_kernel<Real, K, COLS><<<dim3((unsigned)gx, (unsigned)rows), 256, 0, st>>>(a);
}
// complex64 k >= 4 blocks on tcgen05 (dense_tc.cuh); TCX_DENSE_TC=0 keeps them on FP32 FMA
bool dense_tc_on(int K) {
  static const int mode = [] {
    const char* e = getenv("TCX_DENSE_TC");
    return e ? atoi(e) : 1;
  }();
  return mode != 0 && K == 5;
}
template <int K>
cudaError_t dense_fwd_tc_launch(DenseArgs& a, int64_t rows, cudaStream_t st) {
  const int sm = dense_tc_smem(K);
  cudaError_t e = cudaFuncSetAttribute(dense_fwd_tc_kernel<K>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e != cudaSuccess) return e;
  const int64_t ncols = ((int64_t)1 << a.n) >> K;
  const int64_t tiles = (ncols + 127) / 128;
  const int64_t gx = std::max<int64_t>(1, std::min<int64_t>(tiles, std::max<int64_t>(1, 148 * 2 / rows)));
  dense_fwd_tc_kernel<K><<<dim3((unsigned)gx, (unsigned)rows), 128, sm, st>>>(a);
  return cudaGetLastError();
}
template <typename Real>
cudaError_t dense_fwd(int K, DenseArgs& a, int64_t rows, cudaStream_t st) {
  if (sizeof(Real) == 4 && dense_tc_on(K))
    return dense_fwd_tc_launch<5>(a, rows, st);
  switch (K) {
    case 1: dense_fwd_launch<Real, 1>(a, rows, st); break;
    case 2: dense_fwd_launch<Real, 2>(a, rows, st); break;
    case 3: dense_fwd_launch<Real, 3>(a, rows, st); break;
    case 4: dense_fwd_launch<Real, 4>(a, rows, st); break;
    case 5: dense_fwd_launch<Real, 5>(a, rows, st); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
template <typename Real, int K>
cudaError_t dense_bwd_launch(DenseArgs& a, int S, int64_t rows, cudaStream_t st) {
  constexpr int D = 1 << K;
  const size_t stage = (size_t)8 * 2 * 32 * D * sizeof(Cx<Real>);
  const size_t red = (size_t)8 * D * D * 2 * sizeof(double);
  const size_t sm = std::max(stage, red);
  cudaError_t e = cudaFuncSetAttribute(dense_bwd_kernel<Real, K>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  dense_bwd_kernel<Real, K><<<dim3((unsigned)S, (unsigned)rows), 256, sm, st>>>(a);
  return cudaGetLastError();
}
template <typename Real>
cudaError_t dense_bwd(int K, DenseArgs& a, int S, int64_t rows, cudaStream_t st) {
  switch (K) {
    case 1: return dense_bwd_launch<Real, 1>(a, S, rows, st);
    case 2: return dense_bwd_launch<Real, 2>(a, S, rows, st);
    case 3: return dense_bwd_launch<Real, 3>(a, S, rows, st);
    case 4: return dense_bwd_launch<Real, 4>(a, S, rows, st);
    default: return cudaErrorInvalidValue;
  }
}

// one step of a sharded program (tcx_shard_exec); nullptr = the whole single-GPU program
struct OneStep {
  int kind, arg, rank;
  bool first_lambda;
  int chunk = -1;  // >= 0: only the tiles of exchange chunk `chunk` (overlapped exchange)
};

// Exchange chunks (sharded plans): the top P.xchunk_bits local bits below the g exchanged ones
// split every block into 2^xchunk_bits column ranges.  A pass whose window leaves those bits
// out can start on chunk c as soon as chunk c of the exchange has landed.
uint64_t xchunk_mask(const Plan& P) {
  if (P.gbits == 0 || P.cluster || P.xchunk_bits == 0) return 0;
  const int hi = P.nloc - P.gbits;
  return (((1ull << P.xchunk_bits) - 1) << (hi - P.xchunk_bits));
}
bool pass_chunkable(const Plan& P, const PassInfo& p) {
  const uint64_t m = xchunk_mask(P);
  if (!m || (p.wmask & m)) return false;
  const int64_t S = P.tiles / P.tpc;
  return S % (1ll << P.xchunk_bits) == 0;
}
// position of the lowest chunk bit in the tile index (non-window local bits, increasing)
int chunk_tile_pos(const Plan& P, uint64_t wmask) {
  const int lo = P.nloc - P.gbits - P.xchunk_bits;
  int k = 0;
  for (int b = 0; b < lo; ++b) k += (wmask >> b & 1) ? 0 : 1;
  return k;
}

// deferred-factor scan after materialize (JIT plans only: the generic interpreter applies the
// plain coefficients and never reads the flags or pass headers)
tcx_status tan_scan(const Plan& P, DeviceTables* DT, char* W, const WsLayout& wl, int64_t b0,
                    int64_t rows, bool c128, cudaStream_t st) {
  if (P.ntan == 0 || !P.jit_on || P.spass.empty()) return TCX_OK;
  ScanArgs sa;
  sa.sp = (const SPass*)DT->spass.p;
  sa.npass = (int)P.spass.size();
  sa.fw = (const SFwd*)DT->sfwd.p;
  sa.bw = (const SBwd*)DT->sbwd.p;
  sa.tanc = (const double*)(W + wl.tanc);
  sa.ntan = P.ntan;
  sa.mats = W + wl.mats;
  sa.mat_total = P.mat_total;
  sa.corr = wl.corr ? (double*)(W + wl.corr) : nullptr;
  sa.acc_total = std::max(P.acc_total, 1);
  sa.b0 = b0;
  if (c128)
    tan_scan_kernel<double><<<(unsigned)rows, 64, 0, st>>>(sa);
  else
    tan_scan_kernel<float><<<(unsigned)rows, 64, 0, st>>>(sa);
  CUDA_TRY(cudaGetLastError());
  return TCX_OK;
}

// Cluster-resident plans (tcx_build_opts.cluster_bits): materialise the per-
// theta matrices, one megakernel launch with a cluster of G = 2^g CTAs per theta row
// (jit.cpp cluster_kernel: psi and lambda stay in registers, exchanges through distributed
// shared memory), then the fixed-order finalize over the G per-CTA partials.
tcx_status run_cluster(Plan& P, const tcx_pauli* H, const double* theta, int64_t B, double* E,
                       double* grad, void* ws, size_t ws_bytes, cudaStream_t st, int kind,
                       const WsLayout* wl_in, const void* psi0, double* qim) {
  if (kind == K_STATE || psi0 || qim)
    return fail(TCX_E_UNSUPPORTED, "cluster-resident plans run tcx_expect_batch / tcx_grad_batch "
                                   "only (the state never leaves the cluster's registers)");
  if (B <= 0) return fail(TCX_E_INVALID, "B must be > 0");
  if (!ws) return fail(TCX_E_INVALID, "null workspace");
  if (P.P > 0 && !theta) return fail(TCX_E_INVALID, "null theta");
  if (!E || (kind == K_GRAD && P.P > 0 && !grad)) return fail(TCX_E_INVALID, "null output");
  if (kind == K_GRAD && !P.unitary)
    return fail(TCX_E_UNSUPPORTED, "grad needs unitary payloads (adjoint applies U^dagger)");
  if (!P.jit_on) return fail(TCX_E_UNSUPPORTED, "cluster-resident plans need per-circuit kernels (" + P.jit_note + ")");
  if (!H) return fail(TCX_E_INVALID, "null pauli");
  if (H->p.n != P.n) return fail(TCX_E_INVALID, "pauli n_qubits != circuit n_qubits");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(TCX_E_CUDA, "no CUDA device (tcx has no CPU fallback)");
  DeviceTables* DT = nullptr;
  tcx_status s = device_tables(P, DT);
  if (s) return s;
  std::shared_ptr<Binding> Bd;
  BindDev bdv{nullptr, nullptr};
  if ((s = binding_for(P, H, Bd, &bdv))) return s;
  const WsLayout wl = wl_in ? *wl_in : ws_layout(P, Bd.get(), B, kind, false);
  if (ws_bytes < wl.total)
    return fail(TCX_E_INVALID, "workspace too small: need " + std::to_string(wl.total) +
                                   " bytes, got " + std::to_string(ws_bytes));
  const int G = 1 << P.gbits;
  const int smem = jit_cluster_smem(P);
  if (smem > 227 * 1024)
    return fail(TCX_E_UNSUPPORTED, "cluster-resident plan needs " + std::to_string(smem) +
                                       " B of shared memory per CTA (> 227 KB)");
  const std::string key = jit_key_cluster(Bd->hash, kind == K_GRAD ? 1 : 0);
  CUfunction jf = nullptr;
  if ((s = jit_function(P, DT, key, &jf))) return s;
  Drv& D = drv();
  if (!D.launchKernelEx) return fail(TCX_E_CUDA, "cuLaunchKernelEx unavailable");
  if ((size_t)smem > DT->jit_smem[key]) {
    if (D.funcSetAttribute(jf, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem) != CUDA_SUCCESS ||
        (G > 8 && D.funcSetAttribute(jf, CU_FUNC_ATTRIBUTE_NON_PORTABLE_CLUSTER_SIZE_ALLOWED, 1) != CUDA_SUCCESS))
      return fail(TCX_E_CUDA, "cuFuncSetAttribute failed for " + jit_kernel_name(key));
    DT->jit_smem[key] = smem;
  }
  char* W = (char*)ws;
  const bool c128 = P.dtype == TCX_C128;
  const int rs = c128 ? 8 : 4;
  const int EU = (int)Bd->units.size();
  const int64_t kMaxRows = 65535;
  auto prof_begin = [&](ProfEntry& pe) -> tcx_status {
    if (g_prof.on) {
      CUDA_TRY(cudaEventCreate(&pe.a));
      CUDA_TRY(cudaEventCreate(&pe.b));
      CUDA_TRY(cudaEventRecord(pe.a, st));
    }
    return TCX_OK;
  };
  // ---- materialize per-theta matrices (as run())
  for (int64_t b0 = 0; b0 < B && !P.mitems.empty(); b0 += kMaxRows) {
    const int64_t rows = std::min(kMaxRows, B - b0);
    MatArgs ma;
    ma.items = (const MItem*)DT->mitems.p;
    ma.nitems = (int)P.mitems.size();
    ma.cons = (const DCons*)DT->dcons.p;
    ma.fixed = (const double*)DT->fixed.p;
    ma.theta = theta + b0 * P.P;
    ma.P = P.P;
    ma.mats = W + wl.mats + b0 * P.mat_total * rs;
    ma.mat_total = P.mat_total;
    ma.tanc = P.ntan > 0 ? (double*)(W + wl.tanc) + b0 * P.ntan : nullptr;
    ma.ntan = P.ntan;
    dim3 g((ma.nitems + 127) / 128, (unsigned)rows);
    if (c128)
      materialize_kernel<double><<<g, 128, 0, st>>>(ma);
    else
      materialize_kernel<float><<<g, 128, 0, st>>>(ma);
    CUDA_TRY(cudaGetLastError());
    if ((s = tan_scan(P, DT, W, wl, b0, rows, c128, st))) return s;
  }
  // ---- the megakernel: rows in chunks (grid.x = rows * G < 2^31)
  PassArgs a;
  std::memset(&a, 0, sizeof(a));
  a.mats = W + wl.mats;
  a.part = (double*)(W + wl.part);
  a.epart = (double*)(W + wl.epart);
  a.groups = bdv.groups;
  a.pterms = bdv.pterms;
  a.swb = (const uint32_t*)DT->swb.p;
  for (int l = 0; l < P.t; ++l) a.W[l] = l;
  a.n = P.nloc;
  a.t = P.t;
  a.h = P.h;
  a.mat_total = P.mat_total;
  a.acc_total = std::max(P.acc_total, 1);
  a.e_units = EU;
  a.mode = 0;
  a.init_hmask = P.init_hmask;
  a.init_amp = P.init_amp;
  a.fold_active = 1;
  ProfEntry pe{};
  if ((s = prof_begin(pe))) return s;
  const int64_t kMaxClusterRows = (int64_t)1 << 24;
  for (int64_t b0 = 0; b0 < B; b0 += kMaxClusterRows) {
    const int64_t rows = std::min(kMaxClusterRows, B - b0);
    a.b0 = b0;
    CUlaunchAttribute attr[1];
    attr[0].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
    attr[0].value.clusterDim.x = (unsigned)G;
    attr[0].value.clusterDim.y = 1;
    attr[0].value.clusterDim.z = 1;
    CUlaunchConfig cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.gridDimX = (unsigned)(rows * G);
    cfg.gridDimY = 1;
    cfg.gridDimZ = 1;
    cfg.blockDimX = 1u << P.h;
    cfg.blockDimY = 1;
    cfg.blockDimZ = 1;
    cfg.sharedMemBytes = (unsigned)smem;
    cfg.hStream = (CUstream)st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* params[] = {&a};
    const CUresult cr = D.launchKernelEx(&cfg, jf, params, nullptr);
    if (cr != CUDA_SUCCESS)
      return fail(TCX_E_CUDA, "cuLaunchKernelEx failed for " + jit_kernel_name(key) + " (CUresult " +
                                  std::to_string((int)cr) + ")");
  }
  if (g_prof.on) {
    CUDA_TRY(cudaEventRecord(pe.b, st));
    double fl = 0;
    for (auto& p : P.passes) fl += pass_flops(P, p, false) + (kind == K_GRAD ? pass_flops(P, p, true) : 0.0);
    for (auto& u : Bd->units) fl += lambda_flops(*Bd, u);
    pe.phase = 10;
    pe.index = 0;
    pe.flops = (double)B * (double)((int64_t)1 << P.n) * fl;
    pe.bytes = (double)B * (P.mat_total * (double)rs + (double)G * 8.0 * (EU + (kind == K_GRAD ? P.acc_total : 0)));
    g_prof.log.push_back(pe);
  }
  // ---- finalize over the G CTA partials of each row
  for (int64_t b0 = 0; b0 < B; b0 += kMaxRows) {
    const int64_t rows = std::min(kMaxRows, B - b0);
    FinArgs f;
    f.part = (const double*)(W + wl.part);
    f.epart = (const double*)(W + wl.epart);
    f.S = G;
    f.K = std::max(P.acc_total, 1);
    f.EU = EU;
    f.gitems = (const GItem*)DT->gitems.p;
    f.ngitems = (int)P.gitems.size();
    f.cons = (const DCons*)DT->dcons.p;
    f.fixed = (const double*)DT->fixed.p;
    f.theta = theta;
    f.P = P.P;
    f.pptr = (const int32_t*)DT->pptr.p;
    f.plist = (const int32_t*)DT->plist.p;
    f.ncontrib = std::max(P.n_contrib, 1);
    f.tot = (double*)(W + wl.tot);
    f.contrib = (double*)(W + wl.contrib);
    f.qcontrib = nullptr;
    f.E = E;
    f.grad = kind == K_GRAD && P.P > 0 ? grad : nullptr;
    f.b0 = b0;
    f.corr = wl.corr && P.jit_on ? (const double*)(W + wl.corr) : nullptr;
    finalize_kernel<<<(unsigned)rows, 256, 0, st>>>(f);
    CUDA_TRY(cudaGetLastError());
  }
  return TCX_OK;
}

tcx_status run(Plan& P, const tcx_pauli* H, const double* theta, int64_t B, double* E,
               double* grad, void* state, void* ws, size_t ws_bytes, cudaStream_t st, int kind,
               const WsLayout* wl_in, const OneStep* one = nullptr, const void* psi0 = nullptr,
               bool keep_state = false, double* qim = nullptr) {
  if (P.cluster)
    return one ? fail(TCX_E_INVALID, "cluster-resident plans have no shard steps")
               : run_cluster(P, H, theta, B, E, grad, ws, ws_bytes, st, kind, wl_in, psi0, qim);
  if (P.gbits > 0 && !one)
    return fail(TCX_E_INVALID, "sharded circuit (global_bits > 0): use tcx_shard_program/exec");
  auto want = [&](int k, int a) { return !one || (one->kind == k && one->arg == a); };
  const uint64_t gbase = one ? ((uint64_t)one->rank << P.nloc) : 0ull;
  if (B <= 0) return fail(TCX_E_INVALID, "B must be > 0");
  if (!ws) return fail(TCX_E_INVALID, "null workspace");
  if (P.P > 0 && !theta) return fail(TCX_E_INVALID, "null theta");
  if (kind != K_STATE && !E) return fail(TCX_E_INVALID, "null E");
  if (kind == K_GRAD && P.P > 0 && !grad) return fail(TCX_E_INVALID, "null grad");
  if (kind == K_STATE && !state && !keep_state) return fail(TCX_E_INVALID, "null state");
  if (kind == K_GRAD && !P.unitary)
    return fail(TCX_E_UNSUPPORTED, "grad needs unitary payloads (adjoint applies U^dagger)");
  if (kind == K_GRAD && dense_max_k(P) > 4)
    return fail(TCX_E_UNSUPPORTED, "grad with dense blocks needs dense_k <= 4");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(TCX_E_CUDA, "no CUDA device (tcx has no CPU fallback)");
  DeviceTables* DT = nullptr;
  tcx_status s = device_tables(P, DT);
  if (s) return s;
  std::shared_ptr<Binding> Bd;
  BindDev bdv{nullptr, nullptr};
  if (kind != K_STATE) {
    if (!H) return fail(TCX_E_INVALID, "null pauli");
    if (H->p.n != P.n) return fail(TCX_E_INVALID, "pauli n_qubits != circuit n_qubits");
    if ((s = binding_for(P, H, Bd, &bdv))) return s;
  }
  if (psi0 && P.gbits > 0) return fail(TCX_E_UNSUPPORTED, "input states with a sharded state");
  WsLayout wl = wl_in ? *wl_in : ws_layout(P, Bd.get(), B, kind, false, psi0 != nullptr);
  if (ws_bytes < wl.total)
    return fail(TCX_E_INVALID, "workspace too small: need " + std::to_string(wl.total) +
                                   " bytes, got " + std::to_string(ws_bytes));
  const bool fuse_last = !one && fuse_last_of(P, kind, wl.mega, Bd.get());
  if ((s = jit_prepare(P, kind, wl.mega, Bd.get(), fuse_last))) return s;
  char* W = (char*)ws;
  const bool c128 = P.dtype == TCX_C128;
  const int rs = c128 ? 8 : 4;
  const int64_t S = P.tiles / tiles_per_cta(P);
  const int EU = Bd ? (int)Bd->units.size() : 1;
  const int64_t kMaxRows = 65535;
  int64_t rlo = 0, rhi = B;  // rows of the current L2 row group (all rows unless grouped)
  // ---- materialize per-theta matrices
  for (int64_t b0 = 0; b0 < B && want(0, 0); b0 += kMaxRows) {
    const int64_t rows = std::min(kMaxRows, B - b0);
    if (P.mitems.empty()) break;
    MatArgs ma;
    ma.items = (const MItem*)DT->mitems.p;
    ma.nitems = (int)P.mitems.size();
    ma.cons = (const DCons*)DT->dcons.p;
    ma.fixed = (const double*)DT->fixed.p;
    ma.theta = theta + b0 * P.P;
    ma.P = P.P;
    ma.mats = W + wl.mats + b0 * P.mat_total * rs;
    ma.mat_total = P.mat_total;
    ma.tanc = P.ntan > 0 ? (double*)(W + wl.tanc) + b0 * P.ntan : nullptr;
    ma.ntan = P.ntan;
    dim3 g((ma.nitems + 127) / 128, (unsigned)rows);
    if (c128)
      materialize_kernel<double><<<g, 128, 0, st>>>(ma);
    else
      materialize_kernel<float><<<g, 128, 0, st>>>(ma);
    CUDA_TRY(cudaGetLastError());
    if ((s = tan_scan(P, DT, W, wl, b0, rows, c128, st))) return s;
  }
  // ---- input states (PAPER.md:1005-1044 inputs): the first pass / block reads them
  if (psi0) {
    if (wl.mega) return fail(TCX_E_INVALID, "workspace sized without TCX_WS_INPUTS");
    CUDA_TRY(cudaMemcpyAsync(W + wl.psi, psi0, (size_t)B * ((size_t)1 << P.n) * 2 * rs,
                             cudaMemcpyDeviceToDevice, st));
    const int64_t pairs = B << (P.n - 1);
    for (int bit = 0; bit < P.n; ++bit) {  // leading H gates folded into the plan's init
      if (!(P.init_hmask >> bit & 1)) continue;
      const unsigned blocks = (unsigned)((pairs + 255) / 256);
      if (c128)
        hadamard_bit_kernel<double><<<blocks, 256, 0, st>>>((Cx<double>*)(W + wl.psi), P.n, bit, pairs);
      else
        hadamard_bit_kernel<float><<<blocks, 256, 0, st>>>((Cx<float>*)(W + wl.psi), P.n, bit, pairs);
      CUDA_TRY(cudaGetLastError());
    }
  }
  // ---- dense block matrices: row-independent blocks once, parameterised ones per row
  const bool dense = !P.dblocks.empty();
  if (dense && want(0, 0)) {
    DenseMatArgs dm;
    dm.blocks = (const DBlock*)DT->dblocks.p;
    dm.nblocks = (int)P.dblocks.size();
    dm.gates = (const DGate*)DT->dgates.p;
    dm.fixed = (const double*)DT->fixed.p;
    dm.theta = P.P > 0 ? theta : nullptr;
    dm.P = P.P;
    if (P.dmat_shared > 0) {
      dm.mats = W + wl.dshared;
      dm.row_stride = 0;
      dm.shared = 1;
      dm.b0 = 0;
      if (c128)
        dense_mat_kernel<double><<<dim3(dm.nblocks, 1), 32, 0, st>>>(dm);
      else
        dense_mat_kernel<float><<<dim3(dm.nblocks, 1), 32, 0, st>>>(dm);
      CUDA_TRY(cudaGetLastError());
    }
    for (int64_t b0 = 0; b0 < B && P.dmat_row > 0; b0 += kMaxRows) {
      const int64_t rows = std::min(kMaxRows, B - b0);
      dm.mats = W + wl.dmats;
      dm.row_stride = P.dmat_row;
      dm.shared = 0;
      dm.b0 = b0;
      if (c128)
        dense_mat_kernel<double><<<dim3(dm.nblocks, (unsigned)rows), 32, 0, st>>>(dm);
      else
        dense_mat_kernel<float><<<dim3(dm.nblocks, (unsigned)rows), 32, 0, st>>>(dm);
      CUDA_TRY(cudaGetLastError());
    }
  }
  auto dense_args = [&](DenseArgs& d, const DBlock& blk) {
    std::memset(&d, 0, sizeof(d));
    d.psi = W + wl.psi;
    d.lam = W + wl.lam;
    const size_t csz2 = 2 * (size_t)rs;
    d.U = blk.shared ? (const void*)(W + wl.dshared + blk.mat_off * csz2)
                     : (const void*)(W + wl.dmats + blk.mat_off * csz2);
    d.u_stride = blk.shared ? 0 : P.dmat_row;
    for (int i = 0; i < blk.k; ++i) d.bits[i] = blk.bits[i];
    d.n = P.n;
  };
  // ---- pass launches
  auto base_args = [&](PassArgs& a, uint64_t wmask, const int* Wl, int mode) {
    std::memset(&a, 0, sizeof(a));
    a.psi = W + wl.psi;
    a.lam = W + wl.lam;
    a.mats = W + wl.mats;
    a.part = (double*)(W + wl.part);
    a.epart = (double*)(W + wl.epart);
    a.stages = (const KStage*)DT->kstages.p;
    a.ops = (const KOp*)DT->kops.p;
    a.terms = (const KTerm*)DT->kterms.p;
    a.groups = bdv.groups;
    a.pterms = bdv.pterms;
    a.swb = (const uint32_t*)DT->swb.p;
    a.wmask = wmask;
    for (int l = 0; l < P.t; ++l) a.W[l] = Wl[l];
    a.n = P.nloc;
    a.t = P.t;
    a.h = P.h;
    a.mat_total = P.mat_total;
    a.acc_total = std::max(P.acc_total, 1);
    a.e_units = EU;
    a.mode = mode;
    a.tiles_per_cta = tiles_per_cta(P);
    a.last_is_top = 1;
    a.init_hmask = P.init_hmask;
    a.init_amp = P.init_amp;
    a.fold_active = psi0 ? 0 : 1;
    for (int c = 0; c < 15; ++c) a.cut[c] = (const uint8_t*)DT->cut[c].p;
    a.cta_stride = S;
    a.cta_base = 0;
    a.chunk_bits = 0;
    a.tile_ilv = 0;
  };
  auto set_pass = [&](PassArgs& a, const PassInfo& p, bool with_ops) {
    a.stages = (const KStage*)DT->kstages.p + p.stage_begin;
    a.ops = (const KOp*)DT->kops.p + p.kop_begin;
    a.terms = (const KTerm*)DT->kterms.p + p.kterm_begin;
    a.nstages = with_ops ? p.stage_count : 0;
    a.mat_begin = p.mat_begin;
    a.mat_count = with_ops ? p.mat_count : 0;
    a.acc_begin = p.acc_begin;
    a.acc_count = p.acc_count;
    a.max_stage_acc = p.max_stage_acc;
    a.last_is_top = p.last_is_top;
  };
  auto launch_raw = [&](PassArgs& a, const std::string& jkey) -> tcx_status {
    const bool fwd = (a.mode & (M_FWD | M_LAMBDA)) != 0;
    const bool two = (a.mode & M_BWD) != 0;
    const int km = (fwd && two) ? KM_MEGA : (two ? KM_BWD : KM_FWD);
    SmemLayout L = smem_layout(a.t, a.h, rs, a.mat_count, a.max_stage_acc,
                               (a.mode & M_BWD) ? a.acc_count : 0, a.nstages, two);
    if (!(a.mode & M_BWD)) {
      a.acc_count = 0;
      a.max_stage_acc = 0;
      L = smem_layout(a.t, a.h, rs, a.mat_count, 0, 0, a.nstages, two);
    }
    if (L.total > 227 * 1024 - 256)
      return fail(TCX_E_UNSUPPORTED, "pass needs " + std::to_string(L.total) +
                                         " B of shared memory (> 227 KB); lower tile_bits");
    CUfunction jf = nullptr;  // specialised kernel for this pass / lambda unit and mode
    if (!jkey.empty()) {
      tcx_status js = jit_function(P, DT, jkey, &jf);
      if (js) return js;
    }
    int64_t Sg = S;  // CTAs per row of this launch
    if (one && one->chunk >= 0 && (a.mode & (M_FWD | M_BWD))) {  // one exchange chunk's tiles
      const int nc = 1 << P.xchunk_bits;
      Sg = S / nc;
      a.chunk_bits = P.xchunk_bits;
      a.chunk_pos = chunk_tile_pos(P, a.wmask);
      a.chunk_val = one->chunk;
      a.cta_base = (int)(one->chunk * Sg);
    }
    // interleaved tile order when the CTAs of a row are co-resident (a few rows' worth fit the
    // GPU at once: cfg2 / cfg3), blocked otherwise (one huge row: cfg5 measured slower with it)
    a.tile_ilv = tile_order_ilv(Sg, (rs * 2) << P.c);
    if (a.tile_ilv >= 2 && (Sg % a.tile_ilv)) a.tile_ilv = 0;  // groups must tile the grid
    for (int64_t b0 = rlo; b0 < rhi; b0 += kMaxRows) {
      const int64_t rows = std::min(kMaxRows, rhi - b0);
      a.b0 = b0;
      if (jf) {
        Drv& D = drv();
        const int ns = jkey[0] == 'p' ? P.jit_nsub : 1;  // lambda kernels: one tile per CTA
        if (b0 == rlo) {
          const TmaDims td = tma_dims(P.nloc, a.wmask, c128);
          a.use_tma = 0;
          if (td.rank > 0 && ns == 1 && encode_tmap(a.tmap[0], a.psi, td, P.nloc, B))
            a.use_tma = (wl.lam == 0 || encode_tmap(a.tmap[1], a.lam, td, P.nloc, B)) ? 1 : 0;
          if (!(a.mode & (M_LOAD_PSI | M_LOAD_LAM | M_STORE_PSI | M_STORE_LAM))) a.use_tma = 0;
        }
        const int pipe = jkey[0] != 'p' ? 0 : jit_pipe_on(P, P.passes[jit_key_pass_index(jkey)], two);
        const SmemLayout LJ = smem_layout(a.t, a.h, rs, a.mat_count, a.max_stage_acc,
                                          (a.mode & M_BWD) ? a.acc_count : 0, a.nstages, two, ns, pipe);
        if (LJ.total > 227 * 1024 - 1280)
          return fail(TCX_E_UNSUPPORTED, "JIT pass needs too much shared memory");
        if (LJ.total > 48 * 1024 && (size_t)LJ.total > DT->jit_smem[jkey]) {
          if (D.funcSetAttribute(jf, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, LJ.total) !=
              CUDA_SUCCESS)
            return fail(TCX_E_CUDA, "cuFuncSetAttribute failed for " + jit_kernel_name(jkey));
          DT->jit_smem[jkey] = LJ.total;
        }
        void* params[] = {&a};
        if (D.launchKernel(jf, (unsigned)Sg, (unsigned)rows, 1, (unsigned)(ns << a.h), 1, 1,
                           (unsigned)LJ.total, (CUstream)st, params, nullptr) != CUDA_SUCCESS)
          return fail(TCX_E_CUDA, "cuLaunchKernel failed for " + jit_kernel_name(jkey));
        continue;
      }
      cudaError_t e;
      if (c128)
        e = km == 0 ? launch_f64_0(P.r, a, Sg, rows, L.total, st)
                    : (km == 1 ? launch_f64_1(P.r, a, Sg, rows, L.total, st)
                               : launch_f64_2(P.r, a, Sg, rows, L.total, st));
      else
        e = km == 0 ? launch_f32_0(P.r, a, Sg, rows, L.total, st)
                    : (km == 1 ? launch_f32_1(P.r, a, Sg, rows, L.total, st)
                               : launch_f32_2(P.r, a, Sg, rows, L.total, st));
      if (e != cudaSuccess) return fail(TCX_E_CUDA, std::string("pass launch: ") + cudaGetErrorString(e));
    }
    return TCX_OK;
  };
  const double Nf = (double)((int64_t)1 << P.nloc), csz = 2.0 * rs;
  double Bf = (double)B;  // rows of the current group (profiling cost model)
  auto launch = [&](PassArgs& a, int phase, int index, double flops_amp) -> tcx_status {
    std::string jkey;
    if (P.jit_on) {
      const bool fwdk = (a.mode & (M_FWD | M_LAMBDA)) != 0, bwdk = (a.mode & M_BWD) != 0;
      if (phase == 1 || phase == 3 || phase == 5 || phase == 9) {
        const int km = (fwdk && bwdk) ? 2 : (bwdk ? 1 : 0);
        jkey = ((a.mode & M_LAMBDA) && Bd) ? jit_key_pass_lam(index, km, Bd->hash) : jit_key_pass(index, km);
      }
      else if (phase == 2 && Bd)
        jkey = jit_key_lambda(Bd->hash, index);
    }
    ProfEntry pe{};
    if (g_prof.on) {
      CUDA_TRY(cudaEventCreate(&pe.a));
      CUDA_TRY(cudaEventCreate(&pe.b));
      CUDA_TRY(cudaEventRecord(pe.a, st));
    }
    tcx_status r0 = launch_raw(a, jkey);
    if (r0) return r0;

    if (g_prof.on) {
      CUDA_TRY(cudaEventRecord(pe.b, st));
      const int m = a.mode;
      const double touches = ((m & M_LOAD_PSI) ? 1 : 0) + ((m & M_STORE_PSI) ? 1 : 0) +
                             ((m & M_LOAD_LAM) ? 1 : 0) + ((m & M_STORE_LAM) ? 1 : 0);
      const double part = (one && one->chunk >= 0) ? 1.0 / (double)(1 << P.xchunk_bits) : 1.0;
      pe.phase = phase;
      pe.index = index;
      pe.flops = Bf * Nf * flops_amp * part;
      pe.bytes = Bf * Nf * csz * touches * part;
      g_prof.log.push_back(pe);
    }
    return TCX_OK;
  };
  const int nP = (int)P.passes.size();
  if (wl.mega) {
    const PassInfo& p = P.passes[0];
    PassArgs a;
    int mode = M_INIT | M_FWD | M_LAMBDA | (kind == K_GRAD ? M_BWD : 0);
    base_args(a, p.wmask, p.W, mode);
    set_pass(a, p, true);
    a.group_count = Bd->units[0].group_count;
    a.groups = bdv.groups + Bd->units[0].group_begin;
    a.e_index = 0;
    const double fl = pass_flops(P, p, false) + lambda_flops(*Bd, Bd->units[0]) +
                      (kind == K_GRAD ? pass_flops(P, p, true) : 0.0);
    if ((s = launch(a, 5, 0, fl))) return s;
  } else {
   // L2-resident row groups: all passes of a group of theta rows run before
   // the next group, so a group's psi and lambda stay in the 126 MB L2 between passes
   const int64_t G = (P.l2_rows > 0 && P.gbits == 0 && !one) ? std::min<int64_t>(P.l2_rows, B) : B;
   for (int64_t g0 = 0; g0 < B; g0 += G) {
    rlo = g0;
    rhi = std::min(B, g0 + G);
    Bf = (double)(rhi - rlo);
    const bool sharded = P.gbits > 0;
    for (size_t di = 0; di < P.dblocks.size(); ++di) {
      const DBlock& blk = P.dblocks[di];
      ProfEntry pe{};
      if (g_prof.on) {
        CUDA_TRY(cudaEventCreate(&pe.a));
        CUDA_TRY(cudaEventCreate(&pe.b));
        CUDA_TRY(cudaEventRecord(pe.a, st));
      }
      for (int64_t b0 = rlo; b0 < rhi; b0 += kMaxRows) {
        const int64_t rows = std::min(kMaxRows, rhi - b0);
        DenseArgs d;
        dense_args(d, blk);
        d.init = (di == 0 && !psi0) ? 1 : 0;
        d.b0 = b0;
        cudaError_t e = c128 ? dense_fwd<double>(blk.k, d, rows, st) : dense_fwd<float>(blk.k, d, rows, st);
        if (e != cudaSuccess) return fail(TCX_E_CUDA, std::string("dense block launch: ") + cudaGetErrorString(e));
      }
      if (g_prof.on) {
        CUDA_TRY(cudaEventRecord(pe.b, st));
        pe.phase = 6;
        pe.index = (int)di;
        pe.flops = Bf * Nf * 8.0 * (double)(1 << blk.k);  // one complex MAC per U entry
        pe.bytes = Bf * Nf * csz * (di == 0 ? 1.0 : 2.0);
        g_prof.log.push_back(pe);
      }
    }
    for (int pi = 0; pi < nP; ++pi) {
      if (!want(1, pi)) continue;
      const PassInfo& p = P.passes[pi];
      const bool last = pi == nP - 1 && !sharded;  // sharded: every lambda unit is its own step
      if (dense && kind == K_STATE && p.ops.empty()) continue;  // trailing pass: nothing to do
      int mode = M_FWD | M_STORE_PSI | ((pi == 0 && !dense && !psi0) ? M_INIT : M_LOAD_PSI);
      PassArgs a;
      base_args(a, p.wmask, p.W, mode);
      set_pass(a, p, true);
      a.gbase = gbase;
      if (last && kind != K_STATE) {
        a.mode |= M_LAMBDA | (kind == K_GRAD ? M_STORE_LAM : 0);
        if (kind != K_GRAD && EU == 1) a.mode &= ~M_STORE_PSI;
        if (fuse_last) a.mode |= M_BWD;  // stores psi_in / lambda_in for pass nP - 2
        a.group_count = Bd->units[0].group_count;
        a.groups = bdv.groups + Bd->units[0].group_begin;
        a.e_index = 0;
      }
      double fl = pass_flops(P, p, false);
      if (last && kind != K_STATE) fl += lambda_flops(*Bd, Bd->units[0]);
      if (last && fuse_last) fl += pass_flops(P, p, true);
      // the fused last pass (forward + lambda + backward) is its own profiling class
      if ((s = launch(a, (last && fuse_last) ? 9 : 1, pi, fl))) return s;
    }
    if (kind != K_STATE) {
      for (int u = sharded ? 0 : 1; u < EU; ++u) {
        if (!want(2, u)) continue;
        const LamUnit& U = Bd->units[u];
        PassArgs a;
        const bool load_lam = sharded ? !one->first_lambda : true;
        int mode = M_LOAD_PSI | M_LAMBDA |
                   (kind == K_GRAD ? ((load_lam ? M_LOAD_LAM : 0) | M_STORE_LAM) : 0);
        base_args(a, U.wmask, U.W, mode);
        a.gbase = gbase;
        a.nstages = 0;
        a.mat_count = 0;
        a.acc_count = 0;
        a.group_count = U.group_count;
        a.groups = bdv.groups + U.group_begin;
        a.e_index = u;
        if ((s = launch(a, 2, u, lambda_flops(*Bd, U)))) return s;
      }
    }
    if (kind == K_GRAD) {
      for (int pi = nP - 1; pi >= 0; --pi) {
        if (!want(3, pi)) continue;
        if (fuse_last && pi == nP - 1) continue;  // ran fused with the last forward pass
        const PassInfo& p = P.passes[pi];
        if (dense && p.ops.empty()) continue;  // the trailing E / lambda pass has no gates
        int mode = M_LOAD_PSI | M_LOAD_LAM | M_BWD | (pi > 0 ? (M_STORE_PSI | M_STORE_LAM) : 0);
        PassArgs a;
        base_args(a, p.wmask, p.W, mode);
        set_pass(a, p, true);
        a.gbase = gbase;
        if ((s = launch(a, 3, pi, pass_flops(P, p, true)))) return s;
      }
      const int Sd = dense_bwd_ctas(P);
      for (int di = (int)P.dblocks.size() - 1; di >= 0; --di) {
        const DBlock& blk = P.dblocks[di];
        if ((di == 0 || blk.first) && !blk.has_param) continue;  // nothing left to compute
        ProfEntry pe{};
        if (g_prof.on) {
          CUDA_TRY(cudaEventCreate(&pe.a));
          CUDA_TRY(cudaEventCreate(&pe.b));
          CUDA_TRY(cudaEventRecord(pe.a, st));
        }
        for (int64_t b0 = rlo; b0 < rhi; b0 += kMaxRows) {
          const int64_t rows = std::min(kMaxRows, rhi - b0);
          DenseArgs d;
          dense_args(d, blk);
          d.store = (di > 0 && !blk.first) ? 1 : 0;
          d.part = blk.has_param ? (double*)(W + wl.dpart) : nullptr;
          d.b0 = b0;
          cudaError_t e = c128 ? dense_bwd<double>(blk.k, d, Sd, rows, st)
                               : dense_bwd<float>(blk.k, d, Sd, rows, st);
          if (e != cudaSuccess) return fail(TCX_E_CUDA, std::string("dense backward launch: ") + cudaGetErrorString(e));
          if (blk.has_param) {
            const int ne = 2 << (2 * blk.k);
            dense_rsum_kernel<<<dim3((ne + 127) / 128, (unsigned)rows), 128, 0, st>>>(
                (const double*)(W + wl.dpart), (double*)(W + wl.drs), Sd, ne, blk.acc_off,
                P.dacc_total, b0);
            CUDA_TRY(cudaGetLastError());
          }
        }
        if (g_prof.on) {
          CUDA_TRY(cudaEventRecord(pe.b, st));
          pe.phase = 7;
          pe.index = di;
          const bool st_ = di > 0 && !blk.first;  // U^dagger applied and stored
          pe.flops = Bf * Nf * 8.0 * (double)(1 << blk.k) * ((blk.has_param ? 1.0 : 0.0) + (st_ ? 2.0 : 0.0));
          pe.bytes = Bf * Nf * csz * (st_ ? 4.0 : 2.0);
          g_prof.log.push_back(pe);
        }
      }
    }
   }  // row groups
   rlo = 0;
   rhi = B;
   Bf = (double)B;
  }
  // ---- dense block gradient contributions (before finalize sums them per parameter)
  if (kind == K_GRAD && dense && P.dacc_total > 0 && want(4, 0)) {
    int npb = 0;
    for (auto& d : P.dblocks) npb += d.has_param;
    for (int64_t b0 = 0; b0 < B; b0 += kMaxRows) {
      const int64_t rows = std::min(kMaxRows, B - b0);
      DenseGradArgs g;
      g.blocks = (const DBlock*)DT->dblocks.p;
      g.pblocks = (const int32_t*)DT->dpblocks.p;
      g.gates = (const DGate*)DT->dgates.p;
      g.fixed = (const double*)DT->fixed.p;
      g.theta = theta;
      g.P = P.P;
      g.rs = (const double*)(W + wl.drs);
      g.acc_total = P.dacc_total;
      g.contrib = (double*)(W + wl.contrib);
      g.qcontrib = qim ? (double*)(W + wl.dq) : nullptr;
      g.ncontrib = std::max(P.n_contrib, 1);
      g.b0 = b0;
      dense_grad_kernel<<<dim3(npb, (unsigned)rows), 256, 0, st>>>(g);
      CUDA_TRY(cudaGetLastError());
      if (qim && P.P > 0) {
        dense_qim_kernel<<<dim3((P.P + 127) / 128, (unsigned)rows), 128, 0, st>>>(
            g.qcontrib, g.ncontrib, (const int32_t*)DT->pptr.p, (const int32_t*)DT->plist.p, P.P,
            qim, b0);
        CUDA_TRY(cudaGetLastError());
      }
    }
  } else if (qim && P.P > 0) {
    CUDA_TRY(cudaMemsetAsync(qim, 0, sizeof(double) * (size_t)B * P.P, st));  // no parameters
  }
  // ---- finalize / export
  if (kind != K_STATE) {
    for (int64_t b0 = 0; b0 < B && want(4, 0); b0 += kMaxRows) {
      const int64_t rows = std::min(kMaxRows, B - b0);
      FinArgs f;
      f.part = (const double*)(W + wl.part);
      f.epart = (const double*)(W + wl.epart);
      f.S = (int)S;
      f.K = std::max(P.acc_total, 1);
      f.EU = EU;
      f.gitems = (const GItem*)DT->gitems.p;
      f.ngitems = (int)P.gitems.size();
      f.cons = (const DCons*)DT->dcons.p;
      f.fixed = (const double*)DT->fixed.p;
      f.theta = theta;
      f.P = P.P;
      f.pptr = (const int32_t*)DT->pptr.p;
      f.plist = (const int32_t*)DT->plist.p;
      f.ncontrib = std::max(P.n_contrib, 1);
      f.tot = (double*)(W + wl.tot);
      f.contrib = (double*)(W + wl.contrib);
      f.qcontrib = (qim && !dense) ? (double*)(W + wl.dq) : nullptr;
      f.E = E;
      f.grad = kind == K_GRAD && P.P > 0 ? grad : nullptr;
      f.b0 = b0;
      f.corr = wl.corr && P.jit_on ? (const double*)(W + wl.corr) : nullptr;
      finalize_kernel<<<(unsigned)rows, 256, 0, st>>>(f);
      CUDA_TRY(cudaGetLastError());
      if (f.qcontrib && P.P > 0) {  // window q_grad plans: per-parameter CSR sums
        dense_qim_kernel<<<dim3((P.P + 127) / 128, (unsigned)rows), 128, 0, st>>>(
            f.qcontrib, f.ncontrib, (const int32_t*)DT->pptr.p, (const int32_t*)DT->plist.p, P.P,
            qim, b0);
        CUDA_TRY(cudaGetLastError());
      }
    }
  } else if (!one && !keep_state) {
    const size_t bytes = (size_t)B * ((size_t)1 << P.n) * 2 * rs;
    if (!P.relabeled) {
      CUDA_TRY(cudaMemcpyAsync(state, W + wl.psi, bytes, cudaMemcpyDeviceToDevice, st));
    } else {
      const int64_t total = B << P.n;
      const unsigned blocks = (unsigned)((total + 255) / 256);
      if (c128)
        export_kernel<double><<<blocks, 256, 0, st>>>((const Cx<double>*)(W + wl.psi), (Cx<double>*)state, P.n, total, (const int*)DT->layout.p);
      else
        export_kernel<float><<<blocks, 256, 0, st>>>((const Cx<float>*)(W + wl.psi), (Cx<float>*)state, P.n, total, (const int*)DT->layout.p);
      CUDA_TRY(cudaGetLastError());
    }
  }
  return TCX_OK;
}


}  // namespace

// ================================================================== C ABI
extern "C" {

const char* tcx_last_error(void) { return g_err.c_str(); }
const char* tcx_version(void) { return "tcx 0.2 (sm_100a)"; }

tcx_status tcx_circuit_build(int32_t n_qubits, int32_t n_params, const tcx_gate* gates,
                             int64_t n_gates, const double* matrices, int64_t n_matrix_elems,
                             tcx_dtype dtype, const tcx_build_opts* opts, tcx_circuit** out) {
  g_err.clear();
  if (!out) return fail(TCX_E_INVALID, "null out");
  *out = nullptr;
  tcx_circuit* c = new (std::nothrow) tcx_circuit();
  if (!c) return fail(TCX_E_OOM, "out of host memory");
  std::string err;
  tcx_status s;
  try {
    s = build_plan(n_qubits, n_params, gates, n_gates, matrices, n_matrix_elems, dtype, opts,
                   c->plan, err);
  } catch (const std::bad_alloc&) {
    s = TCX_E_OOM;
    err = "out of host memory";
  }
  if (s) {
    delete c;
    return fail(s, err);
  }
  // Contiguous-run width (coalesce_bits) when the caller leaves it to the library: every
  // window holds the lowest c index bits, so c trades the length of the contiguous runs a tile
  // is made of against the freedom of the light-cone windows (fewer passes).  The neighbours
  // c - 1 and c + 1 of the default are planned too and the plan with the lowest
  // passes x w(run bytes) wins, w = 1.0 (128-byte runs), 1.1 (64), 1.25 (32, interleaved tile
  // order: the rest of each line is read by concurrent CTAs) or 1.5 (32, blocked order); runs
  // under 32 bytes (a partial sector) are not considered.  The weights are the session-3
  // measurements (profiles/bench_r2_s3_*.jsonl): cfg3 8 passes of 128-byte runs beat 7 of
  // 32-byte runs (623 vs 598 circuits/s), cfg5 4 passes of 32-byte runs beat 7 of 64 (0.638 vs
  // 0.618), cfg4 86 passes of 64-byte runs beat 74 of 32 (0.404 vs 0.355), cfg2 6 of 128
  // beat 7 of 64 (3671 vs 3635).  TCX_AUTO_COALESCE=0 keeps the default width.
  {
    static const bool auto_c = !(getenv("TCX_AUTO_COALESCE") && atoi(getenv("TCX_AUTO_COALESCE")) == 0);
    const Plan& P0 = c->plan;
    const int c0 = P0.c, t0 = P0.t;  // P0 goes away if a neighbour wins
    const int asz = dtype == TCX_C128 ? 16 : 8;
    auto cost = [&](const Plan& A) {
      const int run = asz << A.c;
      const int64_t ctas_per_row = A.tiles / std::max(A.tpc, 1);
      double w = run >= 128 ? 1.0 : (run >= 64 ? 1.1 : (tile_order_ilv(ctas_per_row, run) == 1 ? 1.25 : 1.5));
      return (double)A.passes.size() * w;
    };
    if (auto_c && (!opts || opts->coalesce_bits <= 0) && P0.gbits == 0 && !P0.cluster &&
        P0.dblocks.empty() && (int64_t)P0.tiles > 1 && (!opts || opts->dense_k <= 0)) {
      tcx_build_opts o2{};
      if (opts) o2 = *opts;
      for (int dc : {-1, 1}) {
        o2.coalesce_bits = c0 + dc;
        if (o2.coalesce_bits < 1 || t0 - o2.coalesce_bits < 2 || (asz << o2.coalesce_bits) < 32) continue;
        tcx_circuit* alt = new (std::nothrow) tcx_circuit();
        if (!alt) break;
        std::string e2;
        tcx_status s2;
        try {
          s2 = build_plan(n_qubits, n_params, gates, n_gates, matrices, n_matrix_elems, dtype, &o2,
                          alt->plan, e2);
        } catch (const std::bad_alloc&) {
          s2 = TCX_E_OOM;
        }
        if (s2 == TCX_OK && cost(alt->plan) < cost(c->plan)) std::swap(c, alt);
        delete alt;
      }
    }
  }
  if (c->plan.gbits > 0 && !getenv("TCX_SHARD_NO_LAYOUT_SEARCH")) {
    // Sharded layout search.  The exchange always swaps the g global bits (qubits 0..g-1,
    // the state's top bits) with the g top LOCAL bits, so which qubits sit in those bits
    // decides how often the two sets must trade places.  Try every contiguous run of g
    // qubits there (the rest keep paper order below them) and keep the plan with the fewest
    // segments (exchanges), then the fewest passes.  HEA: the run at the far end of the
    // CNOT ladder lets the light cone sweep a whole band of layers per segment.
    // Each layout is planned twice: with and without keeping the exchange chunk bits out of
    // the first window after an exchange (which lets that pass start on chunk c while the
    // other chunks are still moving, comm.cuh); the winner has the fewest segments, then the
    // fewest passes, then the most exchanges that overlap the next pass.
    const int n = n_qubits, g = c->plan.gbits, nl = n - g;
    std::vector<int> cands;
    for (int b = g; b + g <= n; ++b) {
      cands.push_back(b);
      if (!c->plan.cluster) cands.push_back(-b);  // negative: with the chunk-bit constraint
    }
    std::vector<tcx_circuit*> built(cands.size(), nullptr);
    std::atomic<int> next{0};
    auto work = [&] {
      for (int i = next++; i < (int)cands.size(); i = next++) {
        tcx_circuit* t = new (std::nothrow) tcx_circuit();
        if (!t) continue;
        const int b0 = std::abs(cands[i]);
        std::vector<int> pos(n);
        for (int q = 0; q < g; ++q) pos[q] = n - 1 - q;                  // global: top bits
        for (int j = 0; j < g; ++j) pos[b0 + j] = nl - 1 - j;            // top local bits
        int bit = nl - g - 1;
        for (int q = g; q < n; ++q)
          if (q < b0 || q >= b0 + g) pos[q] = bit--;
        t->plan.init_pos = pos;
        t->plan.xchunk_forbid = cands[i] < 0;
        std::string e2;
        tcx_status s2;
        try {
          s2 = build_plan(n_qubits, n_params, gates, n_gates, matrices, n_matrix_elems, dtype,
                          opts, t->plan, e2);
        } catch (...) {
          s2 = TCX_E_OOM;
        }
        if (s2) {
          delete t;
          t = nullptr;
        }
        built[i] = t;
      }
    };
    const int nth = std::max(1, std::min<int>((int)cands.size(),
                                              (int)std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (int i = 0; i < nth; ++i) th.emplace_back(work);
    for (auto& x : th) x.join();
    auto overlapped = [](const Plan& Q) {  // exchanges whose next pass can run by chunks
      int k = 0;
      for (size_t p = 1; p < Q.passes.size(); ++p)
        if (Q.passes[p].seg != Q.passes[p - 1].seg)
          k += pass_chunkable(Q, Q.passes[p]) + pass_chunkable(Q, Q.passes[p - 1]);
      return k;
    };
    for (auto*& t : built) {
      if (!t) continue;
      const Plan &A = t->plan, &Bp = c->plan;
      if (A.nseg < Bp.nseg ||
          (A.nseg == Bp.nseg && (A.passes.size() < Bp.passes.size() ||
                                 (A.passes.size() == Bp.passes.size() && overlapped(A) > overlapped(Bp)))))
        std::swap(c, t);
      delete t;
      t = nullptr;
    }
  }
  if (!opts || opts->jit >= 0) {
    std::string why;
    const Plan& P = c->plan;
    if (!jit_available(&why)) {
      c->plan.jit_note = why;
    } else if (P.passes.size() > 512 || P.ops.size() > 32768) {
      c->plan.jit_note = "circuit too large for per-pass specialisation";
    } else {
      c->plan.jit_on = true;  // kernels are generated and compiled on first use
    }
  } else {
    c->plan.jit_note = "disabled by tcx_build_opts.jit";
  }
  *out = c;
  return TCX_OK;
}

tcx_status tcx_pauli_build(int32_t n_qubits, int32_t n_terms, const uint8_t* codes,
                           const double* weights, tcx_pauli** out) {
  g_err.clear();
  if (!out) return fail(TCX_E_INVALID, "null out");
  *out = nullptr;
  tcx_pauli* p = new (std::nothrow) tcx_pauli();
  if (!p) return fail(TCX_E_OOM, "out of host memory");
  std::string err;
  tcx_status s = build_pauli(n_qubits, n_terms, codes, weights, p->p, err);
  if (s) {
    delete p;
    return fail(s, err);
  }
  *out = p;
  return TCX_OK;
}

void tcx_circuit_free(tcx_circuit* c) { delete c; }
void tcx_pauli_free(tcx_pauli* p) {
  delete p;
}

tcx_status tcx_workspace_bytes(const tcx_circuit* circ, const tcx_pauli* pauli, int64_t B,
                               int32_t mode, size_t* bytes) {
  g_err.clear();
  if (!circ || !bytes) return fail(TCX_E_INVALID, "null argument");
  if (B <= 0) return fail(TCX_E_INVALID, "B must be > 0");
  Plan& P = const_cast<tcx_circuit*>(circ)->plan;
  int kind = (mode & TCX_WS_STATE) ? K_STATE : ((mode & TCX_WS_GRAD) ? K_GRAD : K_EXPECT);
  std::shared_ptr<Binding> Bd;
  if (kind != K_STATE) {
    if (!pauli) return fail(TCX_E_INVALID, "null pauli");
    if (pauli->p.n != P.n) return fail(TCX_E_INVALID, "pauli n_qubits != circuit n_qubits");
    tcx_status s = binding_for(P, pauli, Bd, nullptr);
    if (s) return s;
  }
  if (mode & TCX_WS_TERMS) {
    if (!pauli) return fail(TCX_E_INVALID, "null pauli");
    *bytes = ws_layout(P, nullptr, B, K_STATE, false, (mode & TCX_WS_INPUTS) != 0).total +
             terms_extra(P, B, (int)pauli->p.weights.size());
    return TCX_OK;
  }
  *bytes = ws_layout(P, Bd.get(), B, kind, (mode & TCX_WS_HOST_IO) != 0,
                     (mode & TCX_WS_INPUTS) != 0).total;
  return TCX_OK;
}

tcx_status tcx_expect_batch(const tcx_circuit* circ, const tcx_pauli* pauli, const double* theta,
                            int64_t B, double* E, void* ws, size_t ws_bytes, void* stream) {
  g_err.clear();
  if (!circ) return fail(TCX_E_INVALID, "null circuit");
  return run(const_cast<tcx_circuit*>(circ)->plan, pauli, theta, B, E, nullptr, nullptr, ws,
             ws_bytes, (cudaStream_t)stream, K_EXPECT, nullptr);
}

tcx_status tcx_grad_batch(const tcx_circuit* circ, const tcx_pauli* pauli, const double* theta,
                          int64_t B, double* E, double* grad, void* ws, size_t ws_bytes,
                          void* stream) {
  g_err.clear();
  if (!circ) return fail(TCX_E_INVALID, "null circuit");
  return run(const_cast<tcx_circuit*>(circ)->plan, pauli, theta, B, E, grad, nullptr, ws,
             ws_bytes, (cudaStream_t)stream, K_GRAD, nullptr);
}

tcx_status tcx_state_batch(const tcx_circuit* circ, const double* theta, int64_t B, void* state,
                           void* ws, size_t ws_bytes, void* stream) {
  g_err.clear();
  if (!circ) return fail(TCX_E_INVALID, "null circuit");
  return run(const_cast<tcx_circuit*>(circ)->plan, nullptr, theta, B, nullptr, nullptr, state,
             ws, ws_bytes, (cudaStream_t)stream, K_STATE, nullptr);
}

tcx_status tcx_grad_batch_q(const tcx_circuit* circ, const tcx_pauli* pauli, const double* theta,
                            int64_t B, double* E, double* grad, double* q_im, void* ws,
                            size_t ws_bytes, void* stream) {
  g_err.clear();
  if (!circ || !q_im) return fail(TCX_E_INVALID, "null circuit or q_im");
  Plan& P = const_cast<tcx_circuit*>(circ)->plan;
  if (P.dblocks.empty() && !(P.q_grad && P.jit_on))
    return fail(TCX_E_UNSUPPORTED,
                "Im <psi|H|d psi> needs a dense plan (dense_k in 1..4) or a window plan built "
                "with q_grad = 1 (per-circuit kernels)");
  return run(P, pauli, theta, B, E, grad, nullptr, ws, ws_bytes, (cudaStream_t)stream, K_GRAD,
             nullptr, nullptr, nullptr, false, q_im);
}

tcx_status tcx_expect_batch_in(const tcx_circuit* circ, const tcx_pauli* pauli,
                               const double* theta, int64_t B, const void* psi0, double* E,
                               void* ws, size_t ws_bytes, void* stream) {
  g_err.clear();
  if (!circ || !psi0) return fail(TCX_E_INVALID, "null circuit or input states");
  return run(const_cast<tcx_circuit*>(circ)->plan, pauli, theta, B, E, nullptr, nullptr, ws,
             ws_bytes, (cudaStream_t)stream, K_EXPECT, nullptr, nullptr, psi0);
}

tcx_status tcx_grad_batch_in(const tcx_circuit* circ, const tcx_pauli* pauli,
                             const double* theta, int64_t B, const void* psi0, double* E,
                             double* grad, void* ws, size_t ws_bytes, void* stream) {
  g_err.clear();
  if (!circ || !psi0) return fail(TCX_E_INVALID, "null circuit or input states");
  return run(const_cast<tcx_circuit*>(circ)->plan, pauli, theta, B, E, grad, nullptr, ws,
             ws_bytes, (cudaStream_t)stream, K_GRAD, nullptr, nullptr, psi0);
}

tcx_status tcx_state_batch_in(const tcx_circuit* circ, const double* theta, int64_t B,
                              const void* psi0, void* state, void* ws, size_t ws_bytes,
                              void* stream) {
  g_err.clear();
  if (!circ || !psi0) return fail(TCX_E_INVALID, "null circuit or input states");
  return run(const_cast<tcx_circuit*>(circ)->plan, nullptr, theta, B, nullptr, nullptr, state,
             ws, ws_bytes, (cudaStream_t)stream, K_STATE, nullptr, nullptr, psi0);
}

tcx_status tcx_expect_terms_batch(const tcx_circuit* circ, const tcx_pauli* pauli,
                                  const double* theta, int64_t B, const void* psi0,
                                  double* E_terms, void* ws, size_t ws_bytes, void* stream) {
  g_err.clear();
  if (!circ || !pauli || !E_terms) return fail(TCX_E_INVALID, "null argument");
  Plan& P = const_cast<tcx_circuit*>(circ)->plan;
  const Pauli& H = pauli->p;
  if (H.n != P.n) return fail(TCX_E_INVALID, "pauli n_qubits != circuit n_qubits");
  if (P.gbits > 0) return fail(TCX_E_UNSUPPORTED, "per-term values of a sharded state");
  if (B <= 0) return fail(TCX_E_INVALID, "B must be > 0");
  const int T = (int)H.weights.size();
  const WsLayout wl = ws_layout(P, nullptr, B, K_STATE, false, psi0 != nullptr);
  const size_t need = wl.total + terms_extra(P, B, T);
  if (!ws || ws_bytes < need)
    return fail(TCX_E_INVALID, "workspace too small: need " + std::to_string(need) + " bytes");
  cudaStream_t st = (cudaStream_t)stream;
  tcx_status s = run(P, nullptr, theta, B, nullptr, nullptr, nullptr, ws, ws_bytes, st, K_STATE,
                     &wl, nullptr, psi0, /*keep_state=*/true);
  if (s || T == 0) return s;
  // term masks in the final physical layout (SWAP relabels applied)
  std::vector<TTerm> tt(T);
  for (int j = 0; j < T; ++j) {
    TTerm t{};
    for (int q = 0; q < P.n; ++q) {
      const int c = H.codes[(size_t)j * P.n + q];
      const uint64_t m = 1ull << P.layout[q];
      if (c == 1 || c == 2) t.x |= m;
      if (c == 2 || c == 3) t.zy |= m;
      if (c == 2) t.ny++;
    }
    tt[j] = t;
  }
  char* W = (char*)ws;
  double* part = (double*)(W + wl.total);
  TTerm* dterms = (TTerm*)(W + wl.total + align256((size_t)B * terms_ctas(P) * std::max(T, 1) * 8));
  CUDA_TRY(cudaMemcpyAsync(dterms, tt.data(), sizeof(TTerm) * T, cudaMemcpyHostToDevice, st));
  const int S = terms_ctas(P);
  const int64_t kMaxRows = 65535;
  for (int64_t b0 = 0; b0 < B; b0 += kMaxRows) {
    const int64_t rows = std::min(kMaxRows, B - b0);
    if (P.dtype == TCX_C128)
      terms_kernel<double><<<dim3(S, (unsigned)rows), 256, 0, st>>>(
          (const Cx<double>*)(W + wl.psi), P.n, dterms, T, part, b0);
    else
      terms_kernel<float><<<dim3(S, (unsigned)rows), 256, 0, st>>>(
          (const Cx<float>*)(W + wl.psi), P.n, dterms, T, part, b0);
    CUDA_TRY(cudaGetLastError());
    terms_sum_kernel<<<dim3((T + 127) / 128, (unsigned)rows), 128, 0, st>>>(part, E_terms, S, T, b0);
    CUDA_TRY(cudaGetLastError());
  }
  return TCX_OK;
}

static tcx_status host_call(const tcx_circuit* circ, const tcx_pauli* pauli, const double* th,
                            int64_t B, double* E, double* grad, void* ws, size_t ws_bytes,
                            void* stream, int kind) {
  g_err.clear();
  if (!circ || !pauli) return fail(TCX_E_INVALID, "null circuit or pauli");
  if (B <= 0) return fail(TCX_E_INVALID, "B must be > 0");
  Plan& P = const_cast<tcx_circuit*>(circ)->plan;
  if (P.P > 0 && !th) return fail(TCX_E_INVALID, "null theta");
  if (!E || (kind == K_GRAD && P.P > 0 && !grad)) return fail(TCX_E_INVALID, "null output");
  std::shared_ptr<Binding> Bd;
  tcx_status s = binding_for(P, pauli, Bd, nullptr);
  if (s) return s;
  WsLayout wl = ws_layout(P, Bd.get(), B, kind, true);
  if (ws_bytes < wl.total)
    return fail(TCX_E_INVALID, "workspace too small: need " + std::to_string(wl.total));
  cudaStream_t st = (cudaStream_t)stream;
  char* W = (char*)ws;
  double* dth = (double*)(W + wl.theta);
  double* dE = (double*)(W + wl.E);
  double* dG = (double*)(W + wl.grad);
  if (P.P > 0)
    CUDA_TRY(cudaMemcpyAsync(dth, th, sizeof(double) * B * P.P, cudaMemcpyHostToDevice, st));
  s = run(P, pauli, dth, B, dE, dG, nullptr, ws, ws_bytes, st, kind, &wl);
  if (s) return s;
  CUDA_TRY(cudaMemcpyAsync(E, dE, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
  if (kind == K_GRAD && P.P > 0)
    CUDA_TRY(cudaMemcpyAsync(grad, dG, sizeof(double) * B * P.P, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return TCX_OK;
}

tcx_status tcx_expect_batch_host(const tcx_circuit* circ, const tcx_pauli* pauli,
                                 const double* theta_host, int64_t B, double* E_host, void* ws,
                                 size_t ws_bytes, void* stream) {
  return host_call(circ, pauli, theta_host, B, E_host, nullptr, ws, ws_bytes, stream, K_EXPECT);
}

tcx_status tcx_grad_batch_host(const tcx_circuit* circ, const tcx_pauli* pauli,
                               const double* theta_host, int64_t B, double* E_host,
                               double* grad_host, void* ws, size_t ws_bytes, void* stream) {
  return host_call(circ, pauli, theta_host, B, E_host, grad_host, ws, ws_bytes, stream, K_GRAD);
}

tcx_status tcx_circuit_jit(const tcx_circuit* circ, const tcx_pauli* pauli, int64_t B,
                           int32_t kind) {
  g_err.clear();
  if (!circ || B <= 0 || kind < 0 || kind > 2) return fail(TCX_E_INVALID, "bad argument");
  Plan& P = const_cast<tcx_circuit*>(circ)->plan;
  std::shared_ptr<Binding> Bd;
  if (kind != K_STATE) {
    if (!pauli) return fail(TCX_E_INVALID, "null pauli");
    tcx_status s = binding_for(P, pauli, Bd, nullptr);
    if (s) return s;
  }
  WsLayout wl = ws_layout(P, Bd.get(), B, kind, false);
  return jit_prepare(P, kind, wl.mega, Bd.get(), fuse_last_of(P, kind, wl.mega, Bd.get()));
}

tcx_status tcx_circuit_info(const tcx_circuit* circ, const tcx_pauli* pauli, tcx_plan_info* o) {
  g_err.clear();
  if (!circ || !o) return fail(TCX_E_INVALID, "null argument");
  Plan& P = const_cast<tcx_circuit*>(circ)->plan;
  std::memset(o, 0, sizeof(*o));
  o->n_qubits = P.n;
  o->n_params = P.P;
  o->dtype = P.dtype;
  o->tile_bits = P.t;
  o->reg_bits = P.r;
  o->coalesce_bits = P.c;
  o->threads_per_tile = 1 << P.h;
  o->n_ops = (int)P.ops.size();
  o->fwd_passes = (int)P.passes.size();
  o->bwd_passes = (int)P.passes.size();
  int st = 0;
  for (auto& p : P.passes) st += p.stage_count;
  o->stages = st;
  o->unitary = P.unitary;
  o->relabeled = P.relabeled;
  o->jit = P.jit_on ? 1 : 0;
  o->global_bits = P.gbits;
  o->segments = P.nseg;
  o->tiles_per_state = P.tiles;
  o->acc_slots = P.acc_total;
  o->mat_reals = P.mat_total;
  o->dense_k = P.dense_k;
  o->dense_blocks = (int)P.dblocks.size();
  o->init_h = __builtin_popcountll(P.init_hmask);
  o->cluster_bits = P.cluster ? P.gbits : 0;
  for (const auto& ps : P.passes) {
    const TmaDims td = tma_dims(P.nloc, ps.wmask, P.dtype == TCX_C128);
    if (td.rank > 0 && !ps.ops.empty()) (td.sub ? o->tma_multibox_passes : o->tma_passes)++;
  }
  for (size_t p = 1; p < P.passes.size(); ++p)
    if (P.passes[p].seg != P.passes[p - 1].seg)
      o->exchange_overlaps += pass_chunkable(P, P.passes[p]) + pass_chunkable(P, P.passes[p - 1]);
  if (!P.dblocks.empty()) {  // the trailing E / lambda pass has no gates: no backward launch
    int nb = 0;
    for (auto& p : P.passes) nb += p.ops.empty() ? 0 : 1;
    o->bwd_passes = nb;
  }
  o->lambda_passes = 0;
  if (pauli) {
    std::shared_ptr<Binding> Bd;
    tcx_status s = binding_for(P, pauli, Bd, nullptr);
    if (s) return s;
    o->lambda_passes = (int)Bd->units.size() - 1;
  }
  return TCX_OK;
}

tcx_status tcx_profile_enable(int32_t on) {
  g_err.clear();
  g_prof.on = on != 0;
  return TCX_OK;
}

tcx_status tcx_profile_read(tcx_kernel_time* out, int32_t cap, int32_t* n) {
  g_err.clear();
  if (!n) return fail(TCX_E_INVALID, "null n");
  int32_t k = 0;
  for (auto& e : g_prof.log) {
    float ms = 0.f;
    cudaEventSynchronize(e.b);
    cudaEventElapsedTime(&ms, e.a, e.b);
    if (out && k < cap) {
      out[k].phase = e.phase;
      out[k].index = e.index;
      out[k].ms = ms;
      out[k].pad = 0.f;
      out[k].flops = e.flops;
      out[k].bytes = e.bytes;
    }
    ++k;
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  g_prof.log.clear();
  *n = std::min(k, cap);
  return TCX_OK;
}

tcx_status tcx_shard_program(const tcx_circuit* circ, const tcx_pauli* pauli, int32_t want_grad,
                             tcx_shard_step* steps, int32_t cap, int32_t* n) {
  g_err.clear();
  if (!circ || !pauli || !n) return fail(TCX_E_INVALID, "null argument");
  Plan& P = const_cast<tcx_circuit*>(circ)->plan;
  std::shared_ptr<Binding> Bd;
  tcx_status s = binding_for(P, pauli, Bd, nullptr);
  if (s) return s;
  if (P.gbits == 0 || P.cluster) return fail(TCX_E_INVALID, "circuit is not sharded (global_bits = 0)");
  const std::vector<tcx_shard_step> v = shard_program(P, *Bd, want_grad != 0);
  *n = (int32_t)v.size();
  if (steps)
    for (int i = 0; i < std::min<int>(cap, (int)v.size()); ++i) steps[i] = v[i];
  return TCX_OK;
}

tcx_status tcx_shard_exec(const tcx_circuit* circ, const tcx_pauli* pauli, int32_t rank,
                          int32_t want_grad, const tcx_shard_step* step, const double* theta,
                          int64_t B, double* E_partial, double* grad_partial, void* ws,
                          size_t ws_bytes, void* stream) {
  g_err.clear();
  if (!circ || !step) return fail(TCX_E_INVALID, "null argument");
  Plan& P = const_cast<tcx_circuit*>(circ)->plan;
  if (P.gbits == 0 || P.cluster) return fail(TCX_E_INVALID, "circuit is not sharded (global_bits = 0)");
  if (rank < 0 || rank >= (1 << P.gbits)) return fail(TCX_E_INVALID, "rank out of range");
  if (step->kind == TCX_STEP_EXCHANGE) return fail(TCX_E_INVALID, "exchange steps run in the caller");
  OneStep one{step->kind, step->arg, rank, false};
  if (step->kind == TCX_STEP_LAMBDA) {  // the first lambda unit initialises lambda
    std::shared_ptr<Binding> Bd;
    if (!pauli) return fail(TCX_E_INVALID, "null pauli");
    tcx_status s = binding_for(P, pauli, Bd, nullptr);
    if (s) return s;
    int first = -1;
    for (int u = 0; u < (int)Bd->units.size() && first < 0; ++u)
      if (!Bd->units[u].swapped) first = u;
    if (first < 0) first = 0;
    one.first_lambda = step->arg == first;
  }
  return run(P, pauli, theta, B, E_partial, grad_partial, nullptr, ws, ws_bytes,
             (cudaStream_t)stream, want_grad ? K_GRAD : K_EXPECT, nullptr, &one);
}

tcx_status tcx_shard_buffers(const tcx_circuit* circ, const tcx_pauli* pauli, int64_t B,
                             int32_t want_grad, void* ws, void** psi, void** lam,
                             int64_t* local_amps) {
  g_err.clear();
  if (!circ || !pauli || !psi || !lam || !local_amps) return fail(TCX_E_INVALID, "null argument");
  Plan& P = const_cast<tcx_circuit*>(circ)->plan;
  std::shared_ptr<Binding> Bd;
  tcx_status s = binding_for(P, pauli, Bd, nullptr);
  if (s) return s;
  WsLayout wl = ws_layout(P, Bd.get(), B, want_grad ? K_GRAD : K_EXPECT, false);
  *psi = (char*)ws + wl.psi;
  *lam = want_grad ? (char*)ws + wl.lam : nullptr;
  *local_amps = (int64_t)1 << P.nloc;
  return TCX_OK;
}

tcx_status tcx_circuit_decode(const tcx_circuit* circ, tcx_gate* out, int64_t cap, int64_t* n) {
  g_err.clear();
  if (!circ || !n) return fail(TCX_E_INVALID, "null argument");
  const Plan& P = circ->plan;
  *n = (int64_t)P.gates.size();
  if (out)
    for (int64_t i = 0; i < std::min<int64_t>(cap, *n); ++i) out[i] = P.gates[i];
  return TCX_OK;
}

tcx_status tcx_circuit_layout(const tcx_circuit* circ, int32_t* out) {
  g_err.clear();
  if (!circ || !out) return fail(TCX_E_INVALID, "null argument");
  for (int q = 0; q < circ->plan.n; ++q) out[q] = circ->plan.layout[q];
  return TCX_OK;
}

tcx_status tcx_launch_count(const tcx_circuit* circ, const tcx_pauli* pauli, int64_t B,
                            int32_t want_grad, int32_t* launches) {
  g_err.clear();
  if (!circ || !pauli || !launches) return fail(TCX_E_INVALID, "null argument");
  if (B <= 0) return fail(TCX_E_INVALID, "B must be > 0");
  Plan& P = const_cast<tcx_circuit*>(circ)->plan;
  std::shared_ptr<Binding> Bd;
  tcx_status s = binding_for(P, pauli, Bd, nullptr);
  if (s) return s;
  const int kind = want_grad ? K_GRAD : K_EXPECT;
  WsLayout wl = ws_layout(P, Bd.get(), B, kind, false);
  auto chunks = [](int64_t rows) { return (rows + 65534) / 65535; };  // grid.y chunks
  if (P.cluster) {  // materialize, the cluster megakernel, finalize
    *launches = (int32_t)((P.mitems.empty() ? 0 : chunks(B)) + ((B + (1 << 24) - 1) >> 24) + chunks(B));
    return TCX_OK;
  }
  // mirrors run(): `once` launches, `perB` per row chunk of the whole batch, `perG` per row
  // chunk of every L2 row group (all rows when groups are off)
  int64_t once = 0, perB = 0, perG = 0;
  perB += P.mitems.empty() ? 0 : 1;  // materialize
  const bool dense = !P.dblocks.empty();
  if (dense) {
    int npb = 0;
    for (auto& d : P.dblocks) npb += d.has_param;
    once += P.dmat_shared > 0 ? 1 : 0;
    perB += P.dmat_row > 0 ? 1 : 0;
    perG += (int64_t)P.dblocks.size();  // forward blocks
    if (want_grad) {
      for (size_t i = 0; i < P.dblocks.size(); ++i) {
        const DBlock& d = P.dblocks[i];
        if ((i == 0 || d.first) && !d.has_param) continue;  // nothing left to compute
        perG += 1 + (d.has_param ? 1 : 0);                  // backward block (+ R' row sums)
      }
      perB += npb > 0 ? 1 : 0;  // dense_grad_kernel
    }
  }
  if (wl.mega) {
    perB += 1;
  } else {
    perG += (int64_t)P.passes.size() + (int64_t)Bd->units.size() - 1 -
            (fuse_last_of(P, kind, wl.mega, Bd.get()) ? 1 : 0);
    if (want_grad) {
      perG += (int64_t)P.passes.size();
      if (dense)
        for (auto& p : P.passes) perG -= p.ops.empty() ? 1 : 0;  // no backward of the E pass
    }
  }
  perB += 1;  // finalize
  const int64_t G = (P.l2_rows > 0 && P.gbits == 0 && !wl.mega) ? std::min<int64_t>(P.l2_rows, B) : B;
  int64_t gchunks = 0;
  for (int64_t g0 = 0; g0 < B; g0 += G) gchunks += chunks(std::min(B, g0 + G) - g0);
  *launches = (int32_t)(once + perB * chunks(B) + perG * gchunks);
  return TCX_OK;
}

}  // extern "C"

#include "comm.cuh"
