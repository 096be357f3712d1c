// kernels.cuh -- the window-pass kernel (sm_100a), included by pass_f32.cu / pass_f64.cu.
//
// One CTA owns `tiles_per_cta` tiles of one theta row.  A tile is the 2^t amplitudes whose
// index varies over the pass window W (t physical bits, always including the low
// `coalesce_bits` so global loads/stores are >= 64-byte runs) with the other bits fixed.
// Each of the 2^h threads holds 2^RB amplitudes in registers; a "stage" fixes which RB
// tile bits live in registers, so every gate on those bits is pure register FMA work.
// Between stages the tile is re-distributed through a swizzled shared-memory buffer.
// (SURVEY §8a rows a4, a6, a7.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "device_common.cuh"
#include "plan.h"

namespace tcx {
namespace dev {

// ---- the window pass kernel --------------------------------------------------
template <typename Real, int RB, int KM>
__global__ void __launch_bounds__(512, 1) pass_kernel(const PassArgs a) {
  using C = Cx<Real>;
  constexpr int NR = 1 << RB;
  constexpr bool kFwd = KM == KM_FWD || KM == KM_MEGA;
  constexpr bool kBwd = KM == KM_BWD || KM == KM_MEGA;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int8_t s_wpos[16];
  __shared__ uint32_t s_swb[16];
  const int t = a.t, h = a.h, tid = threadIdx.x, nthr = 1 << h;
  const int nw = (nthr + 31) >> 5, warp = tid >> 5, lane = tid & 31;
  const int width = nthr < 32 ? nthr : 32;
  const int mode = a.mode;
  const SmemLayout L = smem_layout(t, h, (int)sizeof(Real), a.mat_count, a.max_stage_acc,
                                   a.acc_count, a.nstages, kBwd);
  C* xp = reinterpret_cast<C*>(smem + L.xb_psi);
  C* xl = reinterpret_cast<C*>(smem + L.xb_lam);
  Real* mats = reinterpret_cast<Real*>(smem + L.mats);
  Real* wacc = reinterpret_cast<Real*>(smem + L.wacc);
  double* cacc = reinterpret_cast<double*>(smem + L.cacc);
  KStage* sst = reinterpret_cast<KStage*>(smem + L.stages);
  double* red = reinterpret_cast<double*>(smem + L.red);
  const int64_t b = a.b0 + blockIdx.y;
  const int64_t N = 1ll << a.n;

  for (int i = tid; i < 16; i += nthr) {
    s_wpos[i] = (int8_t)(i < t ? a.W[i] : 0);
    s_swb[i] = a.swb[i];
  }
  {
    const int* src = reinterpret_cast<const int*>(a.stages);
    int* dst = reinterpret_cast<int*>(sst);
    const int nint = a.nstages * (int)(sizeof(KStage) / 4);
    for (int i = tid; i < nint; i += nthr) dst[i] = src[i];
    const Real* gm = reinterpret_cast<const Real*>(a.mats) + b * a.mat_total + a.mat_begin;
    for (int i = tid; i < a.mat_count; i += nthr) mats[i] = gm[i];
    if (kBwd)
      for (int i = tid; i < a.acc_count; i += nthr) cacc[i] = 0.0;
  }
  __syncthreads();

  C* gpsi = reinterpret_cast<C*>(a.psi) + b * N;
  C* glam = reinterpret_cast<C*>(a.lam) + b * N;
  const KOp* ops = a.ops;
  const KTerm* terms = a.terms;
  const int msa = a.max_stage_acc;
  Real* wacc_w = wacc + warp * msa;
  double e_acc = 0.0;

  for (int it = 0; it < a.tiles_per_cta; ++it) {
    const int64_t tile = chunk_tile((int64_t)blockIdx.x * a.tiles_per_cta + it, a.chunk_pos, a.chunk_bits, a.chunk_val);
    uint64_t outer = 0;
    {
      int64_t tt = tile;
      for (int bit = 0; bit < a.n; ++bit)
        if (!((a.wmask >> bit) & 1ull)) {
          if (tt & 1) outer |= 1ull << bit;
          tt >>= 1;
        }
    }
    Map<RB> top;
    make_top<RB>(top, h, tid, outer, s_wpos, s_swb, a.gbase);
    C v[NR], l[NR];
    if (mode & M_INIT) {
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        v[j].x = ((gidx(top, j) | a.gbase) & ~a.init_hmask) == 0 ? Real(a.init_amp) : Real(0);
        v[j].y = 0;
      }
    } else if (mode & M_LOAD_PSI) {
#pragma unroll
      for (int j = 0; j < NR; ++j) v[j] = gpsi[gidx(top, j)];
    }
    if (mode & M_LOAD_LAM) {
#pragma unroll
      for (int j = 0; j < NR; ++j) l[j] = glam[gidx(top, j)];
    } else {
#pragma unroll
      for (int j = 0; j < NR; ++j) l[j].x = l[j].y = 0;
    }

    // ------------------------------------------------------------- forward
    if (kFwd && (mode & M_FWD)) {
      Map<RB> cur = top;
      for (int s = 0; s < a.nstages; ++s) {
        const KStage& st = sst[s];
        if (s > 0 && !st.same_as_prev) {
          Map<RB> nx;
          make_map<RB>(nx, st.R, st.T, h, tid, outer, s_wpos, s_swb, a.gbase);
          __syncthreads();
#pragma unroll
          for (int j = 0; j < NR; ++j) xp[sidx(cur, j)] = v[j];
          __syncthreads();
#pragma unroll
          for (int j = 0; j < NR; ++j) v[j] = xp[sidx(nx, j)];
          cur = nx;
        }
        for (int i = 0; i < st.op_count; ++i) {
          const KOp o = ops[st.op_begin + i];
          if (o.type == OP_U2F) {  // through shared memory
            __syncthreads();
#pragma unroll
            for (int j = 0; j < NR; ++j) xp[sidx(cur, j)] = v[j];
            __syncthreads();
            smem_u2<Real, false>(xp, t, o.a, o.b, mats + o.mat, s_swb, tid, nthr);
            __syncthreads();
#pragma unroll
            for (int j = 0; j < NR; ++j) v[j] = xp[sidx(cur, j)];
          } else {
            op_fwd<Real, RB>(o, v, cur, mats, terms);
          }
        }
      }
      if (!a.last_is_top) {
        __syncthreads();
#pragma unroll
        for (int j = 0; j < NR; ++j) xp[sidx(cur, j)] = v[j];
        __syncthreads();
#pragma unroll
        for (int j = 0; j < NR; ++j) v[j] = xp[sidx(top, j)];
      }
    }

    // ------------------------------------------- lambda = H psi, E partial
    if (kFwd && (mode & M_LAMBDA)) {
      const Real e = lambda_tile<Real, RB>(a, v, l, top, xp, gpsi, s_swb, t);
      e_acc += (double)e;
    }

    // ----------------------------------------------------------- backward
    if (kBwd && (mode & M_BWD)) {
      Map<RB> cur = top;
      int pending = -1;
      for (int s = a.nstages - 1; s >= 0; --s) {
        const KStage& st = sst[s];
        const bool same = (s == a.nstages - 1) ? (a.last_is_top != 0) : (sst[s + 1].same_as_prev != 0);
        Map<RB> nx = cur;
        if (!same) make_map<RB>(nx, st.R, st.T, h, tid, outer, s_wpos, s_swb, a.gbase);
        __syncthreads();
        if (pending >= 0) {
          const KStage& ps = sst[pending];
          for (int i = tid; i < ps.acc_count; i += nthr) {
            double sacc = 0.0;
            for (int w = 0; w < nw; ++w) sacc += (double)wacc[w * msa + i];
            cacc[ps.acc_begin + i] += sacc;
          }
        }
        if (!same) {
#pragma unroll
          for (int j = 0; j < NR; ++j) {
            const uint32_t si = sidx(cur, j);
            xp[si] = v[j];
            xl[si] = l[j];
          }
        }
        __syncthreads();
        if (!same) {
#pragma unroll
          for (int j = 0; j < NR; ++j) {
            const uint32_t si = sidx(nx, j);
            v[j] = xp[si];
            l[j] = xl[si];
          }
          cur = nx;
        }
        for (int i = st.op_count - 1; i >= 0; --i) {
          const KOp o = ops[st.op_begin + i];
          if (o.type == OP_U2F) {
            __syncthreads();
#pragma unroll
            for (int j = 0; j < NR; ++j) {
              const uint32_t si = sidx(cur, j);
              xp[si] = v[j];
              xl[si] = l[j];
            }
            __syncthreads();
            smem_u2<Real, true>(xp, t, o.a, o.b, mats + o.mat, s_swb, tid, nthr);
            smem_u2<Real, true>(xl, t, o.a, o.b, mats + o.mat, s_swb, tid, nthr);
            __syncthreads();
#pragma unroll
            for (int j = 0; j < NR; ++j) {
              const uint32_t si = sidx(cur, j);
              v[j] = xp[si];
              l[j] = xl[si];
            }
          } else {
            op_bwd<Real, RB>(o, v, l, cur, mats, terms, wacc_w, lane, width);
          }
        }
        pending = s;
      }
      __syncthreads();
      if (pending >= 0) {
        const KStage& ps = sst[pending];
        for (int i = tid; i < ps.acc_count; i += nthr) {
          double sacc = 0.0;
          for (int w = 0; w < nw; ++w) sacc += (double)wacc[w * msa + i];
          cacc[ps.acc_begin + i] += sacc;
        }
      }
      // stage 0 uses the load/store mapping: registers are back in `top` order
    }

    if (mode & M_STORE_PSI) {
#pragma unroll
      for (int j = 0; j < NR; ++j) gpsi[gidx(top, j)] = v[j];
    }
    if (mode & M_STORE_LAM) {
#pragma unroll
      for (int j = 0; j < NR; ++j) glam[gidx(top, j)] = l[j];
    }
  }

  // ------------------------------------------------------------- epilogue
  __syncthreads();
  const int64_t cta = b * a.cta_stride + a.cta_base + blockIdx.x;
  if (kBwd && (mode & M_BWD)) {
    double* dst = a.part + cta * a.acc_total + a.acc_begin;
    for (int i = tid; i < a.acc_count; i += nthr) dst[i] = cacc[i];
  }
  if (kFwd && (mode & M_LAMBDA)) {
    const double e = warp_sum(e_acc, width);
    if (lane == 0) red[warp] = e;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += red[w];
      a.epart[cta * a.e_units + a.e_index] = s;
    }
  }
}

template <typename Real, int RB, int KM>
cudaError_t launch_pass(const PassArgs& a, int64_t S, int64_t rows, size_t smem,
                        cudaStream_t st) {
  static size_t attr[64] = {0};  // dynamic smem opted in so far, per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && smem > 48 * 1024 && smem > attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(pass_kernel<Real, RB, KM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      return e;
    }
    attr[dev] = smem;
  }
  dim3 grid((unsigned)S, (unsigned)rows);
  pass_kernel<Real, RB, KM><<<grid, 1 << a.h, smem, st>>>(a);
  return cudaGetLastError();
}

// one translation unit per (precision, kernel mode): pass_inst.cu compiled with
// -DTCX_REAL=float|double -DTCX_KM=0|1|2 (parallel builds)
#define TCX_LAUNCH_DECL(NAME)                                                            \
  cudaError_t NAME(int rb, const PassArgs& a, int64_t S, int64_t rows, size_t smem,      \
                   cudaStream_t st);
TCX_LAUNCH_DECL(launch_f32_0)
TCX_LAUNCH_DECL(launch_f32_1)
TCX_LAUNCH_DECL(launch_f32_2)
TCX_LAUNCH_DECL(launch_f64_0)
TCX_LAUNCH_DECL(launch_f64_1)
TCX_LAUNCH_DECL(launch_f64_2)

}  // namespace dev
}  // namespace tcx
