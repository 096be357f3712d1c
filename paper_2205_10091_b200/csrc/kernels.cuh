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

#include "plan.h"

namespace tcx {
namespace dev {

template <typename Real>
struct alignas(2 * sizeof(Real)) Cx {
  Real x, y;
};

enum {
  M_INIT = 1, M_LOAD_PSI = 2, M_FWD = 4, M_LAMBDA = 8, M_LOAD_LAM = 16,
  M_STORE_PSI = 32, M_STORE_LAM = 64, M_BWD = 128
};
enum { KM_FWD = 0, KM_BWD = 1, KM_MEGA = 2 };

struct PassArgs {
  void* psi;
  void* lam;
  const void* mats;
  double* part;
  double* epart;
  const KStage* stages;
  const KOp* ops;
  const KTerm* terms;
  const KGroup* groups;
  const KPTerm* pterms;
  const uint32_t* swb;     // [16] swizzle images for this dtype
  uint64_t wmask;
  int W[16];
  int n, t, h;
  int nstages, mat_begin, mat_count, mat_total;
  int acc_begin, acc_count, acc_total, max_stage_acc;
  int group_count, e_units, e_index;
  int mode, tiles_per_cta, last_is_top;
  int64_t b0;
};

struct SmemLayout {
  int xb_psi, xb_lam, mats, wacc, cacc, stages, red, total;
};
__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }
__host__ __device__ inline SmemLayout smem_layout(int t, int h, int realsz, int mat_count,
                                                  int max_stage_acc, int acc_count,
                                                  int nstages, bool two) {
  SmemLayout L;
  int off = 0;
  const int csz = 2 * realsz;
  L.xb_psi = off;
  off = al16(off + (csz << t));
  L.xb_lam = off;
  if (two) off = al16(off + (csz << t));
  L.mats = off;
  off = al16(off + realsz * mat_count);
  const int nw = ((1 << h) + 31) / 32;
  L.wacc = off;
  off = al16(off + realsz * nw * max_stage_acc);
  L.cacc = off;
  off = al16(off + 8 * acc_count);
  L.stages = off;
  off = al16(off + (int)sizeof(KStage) * nstages);
  L.red = off;
  off = al16(off + 8 * 32);
  L.total = off;
  return L;
}

// Thread <-> amplitude mapping of one stage: thread tid holds the amplitudes whose
// tile-local index has bit T[m] = bit m of tid, bit R[k] = bit k of the slot j.
template <int RB>
struct Map {
  uint32_t sb;        // swizzled smem index of slot 0
  uint32_t so[RB];    // swizzle image of register bit k
  uint64_t g;         // global physical index of slot 0
  uint32_t gp;        // physical bit positions of register bits, 6 bits each
};
template <int RB>
__device__ __forceinline__ int gpos(const Map<RB>& m, int k) {
  return (m.gp >> (6 * k)) & 63;
}
template <int RB>
__device__ __forceinline__ void make_map(Map<RB>& m, const int8_t* R, const int8_t* T, int h,
                                         int tid, uint64_t outer, const int8_t* wpos,
                                         const uint32_t* swb) {
  m.sb = 0;
  m.g = outer;
  for (int i = 0; i < h; ++i)
    if (tid >> i & 1) {
      const int l = T[i];
      m.sb ^= swb[l];
      m.g |= 1ull << wpos[l];
    }
  m.gp = 0;
#pragma unroll
  for (int k = 0; k < RB; ++k) {
    const int l = R[k];
    m.so[k] = swb[l];
    m.gp |= (uint32_t)wpos[l] << (6 * k);
  }
}
template <int RB>
__device__ __forceinline__ void make_top(Map<RB>& m, int h, int tid, uint64_t outer,
                                         const int8_t* wpos, const uint32_t* swb) {
  m.sb = 0;
  m.g = outer;
  for (int i = 0; i < h; ++i)
    if (tid >> i & 1) {
      m.sb ^= swb[i];
      m.g |= 1ull << wpos[i];
    }
  m.gp = 0;
#pragma unroll
  for (int k = 0; k < RB; ++k) {
    m.so[k] = swb[h + k];
    m.gp |= (uint32_t)wpos[h + k] << (6 * k);
  }
}
template <int RB>
__device__ __forceinline__ uint32_t sidx(const Map<RB>& m, int j) {
  uint32_t s = m.sb;
#pragma unroll
  for (int k = 0; k < RB; ++k)
    if (j >> k & 1) s ^= m.so[k];
  return s;
}
template <int RB>
__device__ __forceinline__ uint64_t gidx(const Map<RB>& m, int j) {
  uint64_t s = m.g;
#pragma unroll
  for (int k = 0; k < RB; ++k)
    if (j >> k & 1) s |= 1ull << gpos(m, k);
  return s;
}
// register-slot image of a physical mask: bit k set iff register bit k is in mask
template <int RB>
__device__ __forceinline__ uint32_t regmask(const Map<RB>& m, uint64_t mask) {
  uint32_t r = 0;
#pragma unroll
  for (int k = 0; k < RB; ++k) r |= (uint32_t)((mask >> gpos(m, k)) & 1ull) << k;
  return r;
}

template <int N>
struct IC {
  static constexpr int value = N;
};
template <int RB, typename F>
__device__ __forceinline__ void dispatch_slot(int k, F&& f) {
  switch (k) {
    case 0: f(IC<0>{}); break;
    case 1: if constexpr (RB > 1) f(IC<1>{}); break;
    case 2: if constexpr (RB > 2) f(IC<2>{}); break;
    case 3: if constexpr (RB > 3) f(IC<3>{}); break;
    default: break;
  }
}

// ---- gate application on register slots -------------------------------------
// U = [[u00, u01], [u10, u11]] on slot K; m = (u00, u01, u10, u11) as (re, im).
template <int RB, int K, typename Real>
__device__ __forceinline__ void apply_u1(Cx<Real>* v, const Real (&m)[8]) {
#pragma unroll
  for (int j = 0; j < (1 << RB); ++j) {
    if (j & (1 << K)) continue;
    const int j1 = j | (1 << K);
    const Cx<Real> p = v[j], q = v[j1];
    v[j].x = m[0] * p.x - m[1] * p.y + m[2] * q.x - m[3] * q.y;
    v[j].y = m[0] * p.y + m[1] * p.x + m[2] * q.y + m[3] * q.x;
    v[j1].x = m[4] * p.x - m[5] * p.y + m[6] * q.x - m[7] * q.y;
    v[j1].y = m[4] * p.y + m[5] * p.x + m[6] * q.y + m[7] * q.x;
  }
}
// U^dagger on slot K from the same m (conj-transpose folded into operand signs).
template <int RB, int K, typename Real>
__device__ __forceinline__ void apply_u1_dag(Cx<Real>* v, const Real (&m)[8]) {
#pragma unroll
  for (int j = 0; j < (1 << RB); ++j) {
    if (j & (1 << K)) continue;
    const int j1 = j | (1 << K);
    const Cx<Real> p = v[j], q = v[j1];
    // out0 = conj(u00) p + conj(u10) q ; out1 = conj(u01) p + conj(u11) q
    v[j].x = m[0] * p.x + m[1] * p.y + m[4] * q.x + m[5] * q.y;
    v[j].y = m[0] * p.y - m[1] * p.x + m[4] * q.y - m[5] * q.x;
    v[j1].x = m[2] * p.x + m[3] * p.y + m[6] * q.x + m[7] * q.y;
    v[j1].y = m[2] * p.y - m[3] * p.x + m[6] * q.y - m[7] * q.x;
  }
}
// R'_ab += psi_a conj(lambda_b) over the pairs of slot K (a, b = value of the bit).
template <int RB, int K, typename Real>
__device__ __forceinline__ void accum_r(const Cx<Real>* v, const Cx<Real>* l, Real (&r)[8]) {
#pragma unroll
  for (int j = 0; j < (1 << RB); ++j) {
    if (j & (1 << K)) continue;
    const int j1 = j | (1 << K);
    const Cx<Real> p0 = v[j], p1 = v[j1], l0 = l[j], l1 = l[j1];
    r[0] = fma(p0.x, l0.x, fma(p0.y, l0.y, r[0]));
    r[1] = fma(p0.y, l0.x, fma(-p0.x, l0.y, r[1]));
    r[2] = fma(p0.x, l1.x, fma(p0.y, l1.y, r[2]));
    r[3] = fma(p0.y, l1.x, fma(-p0.x, l1.y, r[3]));
    r[4] = fma(p1.x, l0.x, fma(p1.y, l0.y, r[4]));
    r[5] = fma(p1.y, l0.x, fma(-p1.x, l0.y, r[5]));
    r[6] = fma(p1.x, l1.x, fma(p1.y, l1.y, r[6]));
    r[7] = fma(p1.y, l1.x, fma(-p1.x, l1.y, r[7]));
  }
}
// CNOT with target slot KT and control register slot KC: register swaps.
template <int RB, int KT, int KC, typename Real>
__device__ __forceinline__ void apply_cx_rr(Cx<Real>* v) {
#pragma unroll
  for (int j = 0; j < (1 << RB); ++j) {
    if ((j & (1 << KT)) || !(j & (1 << KC))) continue;
    const int j1 = j | (1 << KT);
    const Cx<Real> p = v[j];
    v[j] = v[j1];
    v[j1] = p;
  }
}
// CNOT with target slot KT and a control bit outside the registers (thread/tile bit
// `c`): warp-uniform controls branch, lane-varying ones select.  Self-inverse.
template <int RB, int KT, typename Real>
__device__ __forceinline__ void apply_cx_ext(Cx<Real>* v, bool c, bool uniform) {
  if (uniform) {
    if (c) {
#pragma unroll
      for (int j = 0; j < (1 << RB); ++j) {
        if (j & (1 << KT)) continue;
        const Cx<Real> p = v[j];
        v[j] = v[j | (1 << KT)];
        v[j | (1 << KT)] = p;
      }
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < (1 << RB); ++j) {
    if (j & (1 << KT)) continue;
    const int j1 = j | (1 << KT);
    const Cx<Real> p = v[j], q = v[j1];
    v[j].x = c ? q.x : p.x;
    v[j].y = c ? q.y : p.y;
    v[j1].x = c ? p.x : q.x;
    v[j1].y = c ? p.y : q.y;
  }
}
template <int RB, typename Real>
__device__ __forceinline__ void op_cx(const KOp& o, Cx<Real>* v, uint64_t g) {
  if (o.b == kExtCtrl) {
    const bool c = (g >> o.cbit) & 1;
    const bool uni = o.nterm != 0;  // plan: control is an outer or warp bit
    dispatch_slot<RB>(o.a, [&](auto KT) { apply_cx_ext<RB, decltype(KT)::value>(v, c, uni); });
  } else {
    if constexpr (RB >= 2) {
      dispatch_slot<RB>(o.a, [&](auto KT) {
        dispatch_slot<RB>(o.b, [&](auto KC) {
          if constexpr (decltype(KT)::value != decltype(KC)::value)
            apply_cx_rr<RB, decltype(KT)::value, decltype(KC)::value>(v);
        });
      });
    }
  }
}

// ---- warp reductions -----------------------------------------------------------
template <typename Real>
__device__ __forceinline__ Real warp_sum(Real x, int width) {
  const unsigned mask = width >= 32 ? 0xffffffffu : ((1u << width) - 1u);
  for (int o = (width >= 32 ? 16 : width >> 1); o > 0; o >>= 1) x += __shfl_xor_sync(mask, x, o);
  return x;
}
// Transposed butterfly: 8 values over 32 lanes in 9 shuffles; lane (l & 3) == 0 ends
// with value index 4*b4 + 2*b3 + b2 and writes it to dst[index].
template <typename Real>
__device__ __forceinline__ void warp_sum8(Real (&r)[8], int lane, int width, Real* dst) {
  if (width >= 32) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool hi = lane & 16;
      const Real send = hi ? r[k] : r[k + 4];
      const Real keep = hi ? r[k + 4] : r[k];
      r[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const bool hi = lane & 8;
      const Real send = hi ? r[k] : r[k + 2];
      const Real keep = hi ? r[k + 2] : r[k];
      r[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    {
      const bool hi = lane & 4;
      const Real send = hi ? r[0] : r[1];
      const Real keep = hi ? r[1] : r[0];
      r[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    r[0] += __shfl_xor_sync(0xffffffffu, r[0], 2);
    r[0] += __shfl_xor_sync(0xffffffffu, r[0], 1);
    if ((lane & 3) == 0) dst[((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1)] = r[0];
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = warp_sum(r[k], width);
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) dst[k] = r[k];
    }
  }
}

// ---- shared-memory 4x4 (fixed U2 payload; rare, no register-slot constraint) ----
template <typename Real, bool DAG>
__device__ void smem_u2(Cx<Real>* buf, int t, int la, int lb, const Real* m,
                        const uint32_t* swb, int tid, int nthr) {
  const int ngroups = 1 << (t - 2);
  const int lo = la < lb ? la : lb, hi = la < lb ? lb : la;
  for (int g = tid; g < ngroups; g += nthr) {
    uint32_t i = g;
    i = ((i >> lo) << (lo + 1)) | (i & ((1u << lo) - 1));
    i = ((i >> hi) << (hi + 1)) | (i & ((1u << hi) - 1));
    uint32_t id[4] = {i, i | (1u << lb), i | (1u << la), i | (1u << la) | (1u << lb)};
    Cx<Real> in[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t s = 0;
      for (int p = 0; p < t; ++p)
        if (id[k] >> p & 1) s ^= swb[p];
      id[k] = s;
      in[k] = buf[s];
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      Real ox = 0, oy = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const Real mr = DAG ? m[2 * (k * 4 + r)] : m[2 * (r * 4 + k)];
        const Real mi = DAG ? -m[2 * (k * 4 + r) + 1] : m[2 * (r * 4 + k) + 1];
        ox += mr * in[k].x - mi * in[k].y;
        oy += mr * in[k].y + mi * in[k].x;
      }
      buf[id[r]] = Cx<Real>{ox, oy};
    }
  }
}

// ---- diagonal phase op: prod_k exp(i w_k (-1)^popc(r & mask_k)) ------------------
template <typename Real, int RB, bool CONJ>
__device__ __forceinline__ void diag_term(Cx<Real>* v, const Map<RB>& mp, const KTerm& tm,
                                          const Real* mats) {
  const Real cw = mats[tm.wofs], sw = mats[tm.wofs + 1];
  const uint32_t tp = __popcll(mp.g & tm.mask) & 1u;
  const uint32_t mr = regmask<RB>(mp, tm.mask);
#pragma unroll
  for (int j = 0; j < (1 << RB); ++j) {
    const uint32_t s = tp ^ (__popc((uint32_t)j & mr) & 1u);
    const Real ss = (s ^ (CONJ ? 1u : 0u)) ? -sw : sw;
    const Cx<Real> p = v[j];
    v[j].x = p.x * cw - p.y * ss;
    v[j].y = p.x * ss + p.y * cw;
  }
}

template <typename Real, int RB>
__device__ __forceinline__ void op_fwd(const KOp& o, Cx<Real>* v, const Map<RB>& mp,
                                       const Real* mats, const KTerm* terms) {
  if (o.type == OP_U1) {
    Real m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = mats[o.mat + i];
    dispatch_slot<RB>(o.a, [&](auto K) { apply_u1<RB, decltype(K)::value>(v, m); });
  } else if (o.type == OP_CX) {
    op_cx<RB>(o, v, mp.g);
  } else if (o.type == OP_DIAG) {
    for (int k = 0; k < o.nterm; ++k) diag_term<Real, RB, false>(v, mp, terms[o.term + k], mats);
  }
}

template <typename Real, int RB>
__device__ __forceinline__ void op_bwd(const KOp& o, Cx<Real>* v, Cx<Real>* l,
                                       const Map<RB>& mp, const Real* mats, const KTerm* terms,
                                       Real* wacc_w, int lane, int width) {
  if (o.type == OP_U1) {
    Real m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = mats[o.mat + i];
    dispatch_slot<RB>(o.a, [&](auto K) {
      constexpr int k = decltype(K)::value;
      if (o.acc >= 0) {
        Real r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        accum_r<RB, k>(v, l, r);
        warp_sum8(r, lane, width, wacc_w + o.acc);
      }
      apply_u1_dag<RB, k>(v, m);
      apply_u1_dag<RB, k>(l, m);
    });
  } else if (o.type == OP_CX) {
    op_cx<RB>(o, v, mp.g);
    op_cx<RB>(o, l, mp.g);
  } else if (o.type == OP_DIAG) {
    // gradient: Im(conj(lambda) Z_mask psi) at the op output (all terms commute);
    // Im(conj(l) v) is invariant under the common phase, so order is free.
    int cur = -1;
    Real acc = 0;
    for (int k = 0; k < o.nterm; ++k) {
      const KTerm tm = terms[o.term + k];
      if (tm.acc >= 0) {
        if (tm.acc != cur) {
          if (cur >= 0) {
            acc = warp_sum(acc, width);
            if (lane == 0) wacc_w[cur] = acc;
          }
          cur = tm.acc;
          acc = 0;
        }
        const uint32_t tp = __popcll(mp.g & tm.mask) & 1u;
        const uint32_t mr = regmask<RB>(mp, tm.mask);
#pragma unroll
        for (int j = 0; j < (1 << RB); ++j) {
          const uint32_t s = tp ^ (__popc((uint32_t)j & mr) & 1u);
          const Real tj = fma(l[j].x, v[j].y, -l[j].y * v[j].x);
          acc += s ? -tj : tj;
        }
      }
      diag_term<Real, RB, true>(v, mp, tm, mats);
      diag_term<Real, RB, true>(l, mp, tm, mats);
    }
    if (cur >= 0) {
      acc = warp_sum(acc, width);
      if (lane == 0) wacc_w[cur] = acc;
    }
  }
}

// ---- the window pass kernel --------------------------------------------------
template <typename Real, int RB, int KM>
__global__ void __launch_bounds__(256, 2) pass_kernel(const PassArgs a) {
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
    const int64_t tile = (int64_t)blockIdx.x * a.tiles_per_cta + it;
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
    make_top<RB>(top, h, tid, outer, s_wpos, s_swb);
    C v[NR], l[NR];
    if (mode & M_INIT) {
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        v[j].x = gidx(top, j) == 0 ? Real(1) : Real(0);
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
          make_map<RB>(nx, st.R, st.T, h, tid, outer, s_wpos, s_swb);
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
      __syncthreads();
#pragma unroll
      for (int j = 0; j < NR; ++j) xp[sidx(top, j)] = v[j];
      __syncthreads();
      Real e = 0;
      for (int g = 0; g < a.group_count; ++g) {
        const KGroup G = a.groups[g];
        uint32_t swx = 0;
        for (int p = 0; p < t; ++p)
          if (G.xlocal >> p & 1u) swx ^= s_swb[p];
        Real cr[NR], ci[NR];
#pragma unroll
        for (int j = 0; j < NR; ++j) cr[j] = ci[j] = 0;
        for (int k = 0; k < G.term_count; ++k) {
          const KPTerm pt = a.pterms[G.term_begin + k];
          const uint32_t tp = __popcll(top.g & pt.zy) & 1u;
          const uint32_t mr = regmask<RB>(top, pt.zy);
          const Real re = (Real)pt.cre, im = (Real)pt.cim;
#pragma unroll
          for (int j = 0; j < NR; ++j) {
            const uint32_t s = tp ^ (__popc((uint32_t)j & mr) & 1u);
            cr[j] += s ? -re : re;
            ci[j] += s ? -im : im;
          }
        }
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          // partner amplitude psi[r ^ x]: from the tile in smem, or (flip mask not
          // inside the window) gathered from the stored state in global memory
          const C p = G.global ? gpsi[gidx(top, j) ^ G.xphys] : xp[sidx(top, j) ^ swx];
          const Real dx = cr[j] * p.x - ci[j] * p.y;
          const Real dy = cr[j] * p.y + ci[j] * p.x;
          e += v[j].x * dx + v[j].y * dy;
          l[j].x += dx;
          l[j].y += dy;
        }
      }
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
        if (!same) make_map<RB>(nx, st.R, st.T, h, tid, outer, s_wpos, s_swb);
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
  const int64_t cta = b * gridDim.x + blockIdx.x;
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
