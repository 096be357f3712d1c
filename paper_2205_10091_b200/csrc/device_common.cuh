// device_common.cuh -- device helpers of the window-pass kernels (register-slot gate
// application, reductions, diagonal phases).  Used by the precompiled interpreter
// (kernels.cuh) and embedded into the NVRTC-generated JIT kernels (jit.cpp).
#pragma once
#include "device_abi.h"

namespace tcx {
namespace dev {

template <typename Real>
struct alignas(2 * sizeof(Real)) Cx {
  Real x, y;
};

// Thread <-> amplitude mapping of one stage: thread tid holds the amplitudes whose
// tile-local index has bit T[m] = bit m of tid, bit R[k] = bit k of the slot j.
template <int RB>
struct Map {
  uint32_t sb;        // swizzled smem index of slot 0
  uint32_t so[RB];    // swizzle image of register bit k
  uint64_t g;         // physical index of slot 0 within this rank's (local) state
  uint64_t gb;        // sharded states: this rank's global index bits (0 otherwise)
  uint32_t gp;        // physical bit positions of register bits, 6 bits each
};
template <int RB>
__device__ __forceinline__ int gpos(const Map<RB>& m, int k) {
  return (m.gp >> (6 * k)) & 63;
}
template <int RB>
__device__ __forceinline__ void make_map(Map<RB>& m, const int8_t* R, const int8_t* T, int h,
                                         int tid, uint64_t outer, const int8_t* wpos,
                                         const uint32_t* swb, uint64_t gb = 0) {
  m.sb = 0;
  m.g = outer;
  m.gb = gb;
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
                                         const int8_t* wpos, const uint32_t* swb, uint64_t gb = 0) {
  m.sb = 0;
  m.g = outer;
  m.gb = gb;
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

// ---- packed FP32x2 arithmetic (sm_100a FFMA2/FMUL2): a complex64 amplitude (x, y) is one
// 64-bit register pair; broadcast / half-swapped / sign-alternated operands are free
// operand modifiers in SASS, so a complex multiply-add is 2 instructions instead of 4.
__device__ __forceinline__ unsigned long long f2u_(Cx<float> v) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
__device__ __forceinline__ Cx<float> u2f_(unsigned long long r) {
  Cx<float> v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ Cx<float> f2fma(Cx<float> a, Cx<float> b, Cx<float> c) {  // a*b+c
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u_(a)), "l"(f2u_(b)), "l"(f2u_(c)));
  return u2f_(d);
}
__device__ __forceinline__ Cx<float> f2mul(Cx<float> a, Cx<float> b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u_(a)), "l"(f2u_(b)));
  return u2f_(d);
}

// 64-bit packed complex64 (x in the low half, y in the high half): the operand form of
// FFMA2 / FMUL2.  Keeping amplitudes in aligned 64-bit registers avoids pair moves.
typedef unsigned long long q64;
__device__ __forceinline__ q64 qpk(float a, float b) {
  q64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float qx(q64 v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return a;
}
__device__ __forceinline__ float qy(q64 v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return b;
}
__device__ __forceinline__ q64 qsw(q64 v) { return qpk(qy(v), qx(v)); }
__device__ __forceinline__ q64 qneg(q64 v) { return qpk(-qx(v), -qy(v)); }
__device__ __forceinline__ q64 qfma(q64 a, q64 b, q64 c) {  // a * b + c, per half
  q64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ q64 qmul(q64 a, q64 b) {
  q64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// ---- TMA (cp.async.bulk.tensor) + mbarrier helpers for tile I/O -----------------------
// Opaque copy: the compiler cannot hoist values computed from it out of the tile loop, so
// per-transition shared-memory addresses are recomputed where used instead of being kept
// live (and spilled) across the whole straight-line pass body.
__device__ __forceinline__ uint32_t opq(uint32_t x) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred P1;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n}" ::"r"(smem_u32(b)), "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* tmap, const int* c, int rank,
                                         uint64_t* bar) {
  const uint64_t tm = (uint64_t)tmap;
  const uint32_t d = smem_u32(dst), br = smem_u32(bar);
  switch (rank) {
    case 2:
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(d), "l"(tm), "r"(c[0]), "r"(c[1]), "r"(br) : "memory");
      break;
    case 3:
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(d), "l"(tm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(br) : "memory");
      break;
    case 4:
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   ::"r"(d), "l"(tm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(br) : "memory");
      break;
    case 5:
      asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   ::"r"(d), "l"(tm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(br) : "memory");
      break;
  }
}
__device__ __forceinline__ void tma_store(const void* tmap, const int* c, int rank, const void* src) {
  const uint64_t tm = (uint64_t)tmap;
  const uint32_t s = smem_u32(src);
  switch (rank) {
    case 2:
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                   ::"l"(tm), "r"(c[0]), "r"(c[1]), "r"(s) : "memory");
      break;
    case 3:
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                   ::"l"(tm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(s) : "memory");
      break;
    case 4:
      asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                   ::"l"(tm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(s) : "memory");
      break;
    case 5:
      asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                   ::"l"(tm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(s) : "memory");
      break;
  }
}
// L2 prefetch of a tensor tile (no smem, no barrier): the next tile's HBM latency overlaps
// this tile's compute.
__device__ __forceinline__ void tma_prefetch(const void* tmap, const int* c, int rank) {
  const uint64_t tm = (uint64_t)tmap;
  switch (rank) {
    case 2:
      asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];"
                   ::"l"(tm), "r"(c[0]), "r"(c[1]) : "memory");
      break;
    case 3:
      asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];"
                   ::"l"(tm), "r"(c[0]), "r"(c[1]), "r"(c[2]) : "memory");
      break;
    case 4:
      asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];"
                   ::"l"(tm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory");
      break;
    case 5:
      asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];"
                   ::"l"(tm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
      break;
  }
}
__device__ __forceinline__ void tma_store_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// all but the most recently committed bulk group have read their shared memory
__device__ __forceinline__ void tma_store_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void tma_store_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// thread-block clusters (cluster-resident states): this CTA's rank, a full cluster barrier
// (release / acquire: shared-memory writes before it are visible to every CTA after it), and
// the generic address of the same shared-memory location in another CTA of the cluster
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void* cluster_map(void* p, uint32_t rank) {
  uint64_t r;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"((uint64_t)p), "r"(rank));
  return (void*)r;
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
// Pauli components of R' (R'_ab = sum psi_a conj(lambda_b) over the pairs of slot K):
// c[0] = Im(R'01 + R'10), c[1] = Re(R'01 - R'10), c[2] = Im(R'00 - R'11), so that
// Im Tr(B R') = bx c0 + by c1 + bz c2 for B = bx X + by Y + bz Z (finalize_kernel).
template <int RB, int K, typename Real>
__device__ __forceinline__ void accum_c3(const Cx<Real>* v, const Cx<Real>* l, Real (&c)[3]) {
#pragma unroll
  for (int j = 0; j < (1 << RB); ++j) {
    if (j & (1 << K)) continue;
    const int j1 = j | (1 << K);
    const Cx<Real> p0 = v[j], p1 = v[j1], l0 = l[j], l1 = l[j1];
    c[0] = fma(p0.y, l1.x, fma(-p0.x, l1.y, fma(p1.y, l0.x, fma(-p1.x, l0.y, c[0]))));
    c[1] = fma(p0.x, l1.x, fma(p0.y, l1.y, fma(-p1.x, l0.x, fma(-p1.y, l0.y, c[1]))));
    c[2] = fma(p0.y, l0.x, fma(-p0.x, l0.y, fma(-p1.y, l1.x, fma(p1.x, l1.y, c[2]))));
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
// Transposed butterfly for 3 values in 6 shuffles; lanes 0 / 16 / 8 end with the sums of
// r[0] / r[1] / r[2] and write dst[0..2].
template <typename Real>
__device__ __forceinline__ void warp_sum3(Real (&r)[3], int lane, int width, Real* dst) {
  if (width >= 32) {
    const bool h16 = lane & 16, h8 = lane & 8;
    const Real u = (h16 ? r[1] : r[0]) + __shfl_xor_sync(0xffffffffu, h16 ? r[0] : r[1], 16);
    const Real z = r[2] + __shfl_xor_sync(0xffffffffu, r[2], 16);
    Real w = (h8 ? z : u) + __shfl_xor_sync(0xffffffffu, h8 ? u : z, 8);
    w += __shfl_xor_sync(0xffffffffu, w, 4);
    w += __shfl_xor_sync(0xffffffffu, w, 2);
    w += __shfl_xor_sync(0xffffffffu, w, 1);
    if ((lane & 7) == 0 && lane != 24) dst[lane == 0 ? 0 : (lane == 16 ? 1 : 2)] = w;
  } else {
#pragma unroll
    for (int k = 0; k < 3; ++k) r[k] = warp_sum(r[k], width);
    if (lane == 0) {
      dst[0] = r[0];
      dst[1] = r[1];
      dst[2] = r[2];
    }
  }
}

// One value: lane 0 writes its warp sum (structured U1 classes keep one slot, plan.cpp op_accs).
template <typename Real>
__device__ __forceinline__ void warp_sum1s(Real x, int lane, int width, Real* dst) {
  x = warp_sum(x, width);
  if (lane == 0) dst[0] = x;
}
// One component K of the three (structured classes): lane 0 writes it and zeroes the rest.
template <int K, typename Real>
__device__ __forceinline__ void warp_sum1(Real x, int lane, int width, Real* dst) {
  x = warp_sum(x, width);
  if (lane == 0) {
    dst[0] = K == 0 ? x : Real(0);
    dst[1] = K == 1 ? x : Real(0);
    dst[2] = K == 2 ? x : Real(0);
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
  const uint32_t tp = __popcll((mp.g | mp.gb) & tm.mask) & 1u;
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

// one weight class (plan.cpp LUT op, KOp.a == 1): v[j] *= table[c(j)], c(j) = number of
// terms whose signed parity (KTerm.pad = weight sign) is odd at amplitude j
template <typename Real, int RB, bool CONJ>
__device__ __forceinline__ void diag_lut(Cx<Real>* v, Cx<Real>* l, const Map<RB>& mp, const KOp& o,
                                         const KTerm* terms, const Real* mats) {
  int c[1 << RB];
#pragma unroll
  for (int j = 0; j < (1 << RB); ++j) c[j] = 0;
  for (int k = 0; k < o.nterm; ++k) {
    const KTerm tm = terms[o.term + k];
    const uint32_t tp = (__popcll((mp.g | mp.gb) & tm.mask) & 1u) ^ (uint32_t)tm.pad;
    const uint32_t mr = regmask<RB>(mp, tm.mask);
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) c[j] += (int)(tp ^ (__popc((uint32_t)j & mr) & 1u));
  }
  const Cx<Real>* lut = reinterpret_cast<const Cx<Real>*>(mats + terms[o.term].wofs);
#pragma unroll
  for (int j = 0; j < (1 << RB); ++j) {
    const Cx<Real> ph = lut[c[j]];
    const Real sw = CONJ ? -ph.y : ph.y;
    Cx<Real> p = v[j];
    v[j].x = p.x * ph.x - p.y * sw;
    v[j].y = p.x * sw + p.y * ph.x;
    if (l) {
      p = l[j];
      l[j].x = p.x * ph.x - p.y * sw;
      l[j].y = p.x * sw + p.y * ph.x;
    }
  }
}

template <typename Real, int RB>
__device__ __forceinline__ void op_fwd(const KOp& o, Cx<Real>* v, const Map<RB>& mp,
                                       const Real* mats, const KTerm* terms) {
  if (o.type == OP_U1) {
    Real m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = mats[o.mat + (sizeof(Real) == 4 ? 2 * i + 1 : i)];
    dispatch_slot<RB>(o.a, [&](auto K) { apply_u1<RB, decltype(K)::value>(v, m); });
  } else if (o.type == OP_CX) {
    op_cx<RB>(o, v, mp.g | mp.gb);
  } else if (o.type == OP_DIAG) {
    if (o.a == 1)
      diag_lut<Real, RB, false>(v, nullptr, mp, o, terms, mats);
    else
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
    for (int i = 0; i < 8; ++i) m[i] = mats[o.mat + (sizeof(Real) == 4 ? 2 * i + 1 : i)];
    dispatch_slot<RB>(o.a, [&](auto K) {
      constexpr int k = decltype(K)::value;
      if (o.acc >= 0) {
        Real r[3] = {0, 0, 0};
        accum_c3<RB, k>(v, l, r);
        if (o.nterm & 3)  // structured class: one slot, the component its generators read
          warp_sum1s(r[(o.nterm & 3) - 1], lane, width, wacc_w + o.acc);
        else
          warp_sum3(r, lane, width, wacc_w + o.acc);
      }
      apply_u1_dag<RB, k>(v, m);
      apply_u1_dag<RB, k>(l, m);
    });
  } else if (o.type == OP_CX) {
    op_cx<RB>(o, v, mp.g | mp.gb);
    op_cx<RB>(o, l, mp.g | mp.gb);
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
        const uint32_t tp = __popcll((mp.g | mp.gb) & tm.mask) & 1u;
        const uint32_t mr = regmask<RB>(mp, tm.mask);
#pragma unroll
        for (int j = 0; j < (1 << RB); ++j) {
          const uint32_t s = tp ^ (__popc((uint32_t)j & mr) & 1u);
          const Real tj = fma(l[j].x, v[j].y, -l[j].y * v[j].x);
          acc += s ? -tj : tj;
        }
      }
      if (o.a != 1) {
        diag_term<Real, RB, true>(v, mp, tm, mats);
        diag_term<Real, RB, true>(l, mp, tm, mats);
      }
    }
    if (o.a == 1) diag_lut<Real, RB, true>(v, l, mp, o, terms, mats);
    if (cur >= 0) {
      acc = warp_sum(acc, width);
      if (lane == 0) wacc_w[cur] = acc;
    }
  }
}


// lambda += H psi on the tile (top mapping) and the E partial sum_r Re conj(psi_r) (H psi)_r
// (Eq. 2, structures :794-815).  Terms are grouped by X/Y flip mask x;
// (P psi)_r = i^nY (-1)^popc((r ^ x) & zy) psi_{r ^ x}; the sign of x & zy is folded into
// the host-side coefficient.  Partners come from the shared-memory tile, or from HBM when
// x leaves the window (KGroup::global).
// lambda = H psi over the groups [groups, groups + count) for a tile held in registers
// (T0 mapping), every flip mask inside the tile (cluster-resident megakernel)
template <typename Real, int RB>
__device__ __forceinline__ Real lambda_tile_g(const KGroup* groups, int count, const KPTerm* pterms,
                                              Cx<Real>* v, Cx<Real>* l, const Map<RB>& top,
                                              Cx<Real>* xp, const uint32_t* s_swb, int t) {
  using C = Cx<Real>;
  constexpr int NR = 1 << RB;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NR; ++j) xp[sidx(top, j)] = v[j];
  __syncthreads();
  Real e = 0;
  for (int g = 0; g < count; ++g) {
    const KGroup G = groups[g];
    uint32_t swx = 0;
    for (int p = 0; p < t; ++p)
      if (G.xlocal >> p & 1u) swx ^= s_swb[p];
    Real cr[NR], ci[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) cr[j] = ci[j] = 0;
    for (int k = 0; k < G.term_count; ++k) {
      const KPTerm pt = pterms[G.term_begin + k];
      const uint32_t tp = __popcll((top.g | top.gb) & pt.zy) & 1u;
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
      const C p = xp[sidx(top, j) ^ swx];
      const Real dx = cr[j] * p.x - ci[j] * p.y;
      const Real dy = cr[j] * p.y + ci[j] * p.x;
      e += v[j].x * dx + v[j].y * dy;
      l[j].x += dx;
      l[j].y += dy;
    }
  }
  return e;
}

template <typename Real, int RB>
__device__ __forceinline__ Real lambda_tile(const PassArgs& a, Cx<Real>* v, Cx<Real>* l,
                                            const Map<RB>& top, Cx<Real>* xp,
                                            const Cx<Real>* gpsi, const uint32_t* s_swb,
                                            int t) {
  using C = Cx<Real>;
  constexpr int NR = 1 << RB;
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
      const uint32_t tp = __popcll((top.g | top.gb) & pt.zy) & 1u;
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
  return e;
}

}  // namespace dev
}  // namespace tcx
