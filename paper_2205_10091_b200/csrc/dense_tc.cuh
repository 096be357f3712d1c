// dense_tc.cuh -- complex64 dense k-qubit blocks on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulator in TMEM), included by tcx.cu.
//
// North_star step 2: "fused k-qubit blocks run as small dense complex contractions, on
// tensor cores only where the fused block is large enough to leave the memory-bound
// regime".  A k = 5 complex64 block costs 8 * 32 = 256 flop per amplitude against 16 bytes
// (16 flop/B), above the FP32 CUDA-core ridge of 11.4 flop/B on B200, so on CUDA cores it
// is ALU-bound (dense_fwd_kernel); here it runs as a real GEMM on tensor cores instead:
//
//   D[m][n] = sum_k A[m][k] B[n][k]      (M = 128 state columns, N = K = 2 * 2^k)
//   A[m] = (Re psi_m[0..D), Im psi_m[0..D))        one state column per TMEM lane
//   B    = [[Re U, -Im U], [Im U, Re U]]            the real form of the block matrix
//
// so row m of D is the real form of U psi_m.  TF32 keeps 10 mantissa bits, too few for the
// 1e-5 complex64 tolerance, so every operand is split x = hi + lo with hi =
// x truncated to TF32 and lo = x - hi (exact in FP32), and D = A_hi B_hi + A_lo B_hi +
// A_hi B_lo (3xTF32, ~2^-21 relative; the dropped lo*lo term is ~2^-22).
//
// Per CTA (128 threads = 4 warps, one state column per thread and tile): the thread loads
// its column's 2^k amplitudes (coalesced across the warp over the non-block bits), splits
// them and writes the hi / lo rows of A into shared memory in the canonical K-major
// SWIZZLE_128B layout (8-row x 128-byte atoms, 16-byte chunk c of row r stored at c ^ (r & 7));
// one elected thread issues 3 * (2^(k+1) / 8) = 24 tcgen05.mma and commits to an mbarrier; while the
// tensor core runs, every thread already loads its column of the next tile; then each warp
// reads its 32 TMEM lanes back (tcgen05.ld 32x32b) and scatters the outputs in place.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "device_common.cuh"
#include "plan.h"

namespace tcx {
namespace dev {

// ---- tcgen05 / descriptor helpers (PTX ISA: tcgen05 matrix + instruction descriptors) --
// Shared-memory matrix descriptor: start address >> 4 (bits 0-13), leading byte offset >> 4
// (16-29), stride byte offset >> 4 (32-45), descriptor version 1 (46-47, sm_100), base
// offset 0 (49-51), layout type (61-63: 2 = SWIZZLE_128B).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(1) << 16;  // LBO (unused for swizzled K-major; 1 by convention)
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// Instruction descriptor, kind::tf32: D format F32 (bits 4-5 = 1), A / B format TF32
// (bits 7-9 / 10-12 = 2), both K-major (bits 15 / 16 = 0), N >> 3 (bits 17-22),
// M >> 4 (bits 24-28).
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// 32 lanes x 32 consecutive 32-bit TMEM columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* r) {
  uint32_t* u = reinterpret_cast<uint32_t*>(r);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
        "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]),
        "=r"(u[13]), "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]),
        "=r"(u[19]), "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]),
        "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]),
        "=r"(u[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// byte offset of element (row r, k) in a K-major SWIZZLE_128B tile of `rows` rows
// (atoms of 32 fp32 along K stacked after each other: [K/32][rows][128 B])
__device__ __forceinline__ uint32_t sw128_off(int r, int k, int rows) {
  const int atom = k >> 5, kk = k & 31;
  const int chunk = (kk >> 2) ^ (r & 7);
  return (uint32_t)(atom * rows * 128 + r * 128 + chunk * 16 + (kk & 3) * 4);
}

// 16-byte gathers: complex64 amplitudes are 8 bytes, so every global access moves a pair.
// Row pairs when index bit 0 is a block bit (amplitudes j, j+1 of a column are adjacent),
// else column pairs (columns 2p, 2p+1 are adjacent for every row).  Tile = 128 columns.
__device__ __forceinline__ void sts128(unsigned char* base, uint32_t off, float a, float b, float c,
                                       float d) {
  *reinterpret_cast<float4*>(base + off) = make_float4(a, b, c, d);
}
// write 4 consecutive K entries (k0 .. k0+3, k0 % 4 == 0) of row m as hi and lo
__device__ __forceinline__ void put4(unsigned char* sh, unsigned char* sl, int m, int k0, float a,
                                     float b, float c, float d) {
  const float ha = tf32_hi(a), hb = tf32_hi(b), hc = tf32_hi(c), hd = tf32_hi(d);
  const uint32_t off = sw128_off(m, k0, 128);
  sts128(sh, off, ha, hb, hc, hd);
  sts128(sl, off, a - ha, b - hb, c - hc, d - hd);
}

// K = 5 block qubits: D = 32 complex rows, real-form inner dimension and outputs 64.
template <int K>
__global__ void __launch_bounds__(128) dense_fwd_tc_kernel(const DenseArgs a) {
  static_assert(K == 5, "tensor-core dense blocks are k = 5 (16 flop/B, past the FP32 ridge)");
  constexpr int D = 1 << K, KD = 2 * D, N = 2 * D, M = 128;
  constexpr int A_BYTES = M * KD * 4, B_BYTES = N * KD * 4;
  constexpr uint32_t IDESC = umma_idesc_tf32(M, N);
  extern __shared__ __align__(1024) unsigned char tsm[];
  unsigned char* base = tsm + ((1024 - (smem_u32(tsm) & 1023)) & 1023);
  unsigned char* sAh = base;
  unsigned char* sAl = sAh + A_BYTES;
  unsigned char* sBh = sAl + A_BYTES;
  unsigned char* sBl = sBh + B_BYTES;
  __shared__ uint64_t mbar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t b = a.b0 + blockIdx.y;

  if (warp == 0) {  // TMEM: N fp32 columns x 128 lanes for the accumulator
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) mbar_init(&mbar, 1);
  // B = real form of U, split hi / lo; row n (output real index), column k (input)
  {
    const Cx<float>* U = reinterpret_cast<const Cx<float>*>(a.U) + b * a.u_stride;
    for (int e = tid; e < N * KD; e += blockDim.x) {
      const int n = e / KD, k = e % KD;
      const int i = n % D, j = k % D;
      const Cx<float> u = U[i * D + j];
      float v;
      if (n < D) v = k < D ? u.x : -u.y;   // Re out = Re U Re psi - Im U Im psi
      else v = k < D ? u.y : u.x;          // Im out = Im U Re psi + Re U Im psi
      const float h = tf32_hi(v);
      *reinterpret_cast<float*>(sBh + sw128_off(n, k, N)) = h;
      *reinterpret_cast<float*>(sBl + sw128_off(n, k, N)) = v - h;
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  int bits[K];
#pragma unroll
  for (int i = 0; i < K; ++i) bits[i] = a.bits[i];
  const bool rowpair = bits[0] == 0;
  const int64_t Nst = 1ll << a.n;
  const int64_t ncols = Nst >> K;
  const int64_t ntiles = (ncols + M - 1) / M;
  float* psi = reinterpret_cast<float*>(reinterpret_cast<Cx<float>*>(a.psi) + b * Nst);
  const uint32_t aH = smem_u32(sAh), aL = smem_u32(sAl), bH = smem_u32(sBh), bL = smem_u32(sBl);

  // per-thread load role: row pairs -> column t, 16 pairs (j, j+1) of rows;
  // column pairs -> columns (2p, 2p+1), p = t & 63, rows 16h .. 16h+15, h = t >> 6
  const int cp = tid & 63, hh = tid >> 6;
  float4 w[16];
  auto load = [&](int64_t tile) {
    if (rowpair) {
      const int64_t c = tile * M + tid;
      const bool ok = c < ncols;
      const uint64_t bs = dense_insert<K>(ok ? (uint64_t)c : 0ull, bits);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        if (a.init)
          w[q] = make_float4((ok && c == 0 && q == 0) ? 1.f : 0.f, 0.f, 0.f, 0.f);
        else
          w[q] = ok ? *reinterpret_cast<const float4*>(psi + 2 * (bs | dense_off<K>(2 * q, bits)))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    } else {
      const int64_t c = tile * M + 2 * cp;
      const bool ok = c < ncols;
      const uint64_t bs = dense_insert<K>(ok ? (uint64_t)c : 0ull, bits);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int j = 16 * hh + q;
        if (a.init)
          w[q] = make_float4((ok && c == 0 && j == 0) ? 1.f : 0.f, 0.f, 0.f, 0.f);
        else
          w[q] = ok ? *reinterpret_cast<const float4*>(psi + 2 * (bs | dense_off<K>(j, bits)))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  };
  uint32_t phase = 0;
  int64_t tile = blockIdx.x;
  if (tile < ntiles) load(tile);
  for (; tile < ntiles; tile += gridDim.x) {
    // A rows (hi / lo): K index = j for Re psi_j, D + j for Im psi_j
    if (rowpair) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {  // rows j = 4u .. 4u+3 live in w[2u] (j, j+1), w[2u+1]
        const float4 p0 = w[2 * u], p1 = w[2 * u + 1];
        put4(sAh, sAl, tid, 4 * u, p0.x, p0.z, p1.x, p1.z);
        put4(sAh, sAl, tid, D + 4 * u, p0.y, p0.w, p1.y, p1.w);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // rows j = 16h + 4u .. +3 of columns 2p (x, y) and 2p+1 (z, w)
        const float4 p0 = w[4 * u], p1 = w[4 * u + 1], p2 = w[4 * u + 2], p3 = w[4 * u + 3];
        const int k0 = 16 * hh + 4 * u;
        put4(sAh, sAl, 2 * cp, k0, p0.x, p1.x, p2.x, p3.x);
        put4(sAh, sAl, 2 * cp, D + k0, p0.y, p1.y, p2.y, p3.y);
        put4(sAh, sAl, 2 * cp + 1, k0, p0.z, p1.z, p2.z, p3.z);
        put4(sAh, sAl, 2 * cp + 1, D + k0, p0.w, p1.w, p2.w, p3.w);
      }
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      // K steps of 8 tf32 (32 bytes) inside each 128-byte swizzle atom
#pragma unroll
      for (int s = 0; s < KD / 8; ++s) {
        const uint32_t ao = (s >> 2) * (M * 128) + (s & 3) * 32;
        const uint32_t bo = (s >> 2) * (N * 128) + (s & 3) * 32;
        umma_tf32(tmem, umma_desc_sw128(aH + ao, 1024), umma_desc_sw128(bH + bo, 1024), IDESC, s > 0);
        umma_tf32(tmem, umma_desc_sw128(aL + ao, 1024), umma_desc_sw128(bH + bo, 1024), IDESC, 1);
        umma_tf32(tmem, umma_desc_sw128(aH + ao, 1024), umma_desc_sw128(bL + bo, 1024), IDESC, 1);
      }
      umma_commit(&mbar);
    }
    // next tile's loads overlap the tensor-core work
    if (tile + gridDim.x < ntiles) load(tile + gridDim.x);
    mbar_wait(&mbar, phase);
    phase ^= 1;
    tc_fence_after();
    // D row m = TMEM lane m = column tile*128 + m: Re out[0..D) then Im out[0..D)
    float o[N];
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
    for (int h = 0; h < N / 32; ++h) tmem_ld32(trow + h * 32, o + 32 * h);
    tmem_ld_wait();
    const int64_t c = tile * M + tid;
    if (rowpair) {
      const bool ok = c < ncols;
      const uint64_t bs = dense_insert<K>(ok ? (uint64_t)c : 0ull, bits);
      if (ok) {
#pragma unroll
        for (int q = 0; q < 16; ++q)
          *reinterpret_cast<float4*>(psi + 2 * (bs | dense_off<K>(2 * q, bits))) =
              make_float4(o[2 * q], o[D + 2 * q], o[2 * q + 1], o[D + 2 * q + 1]);
      }
    } else {
      // lanes 2i / 2i+1 hold adjacent columns; the even lane stores rows 0..15 of both,
      // the odd lane rows 16..31 (16-byte pairs), exchanging the other half by shuffles
      const bool odd = lane & 1;
      const int64_t ce = c & ~1ll;
      const bool ok = ce < ncols;
      const uint64_t bs = dense_insert<K>(ok ? (uint64_t)ce : 0ull, bits);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        // compile-time register indices only (a lane-dependent index would spill o[])
        const float lo_r = o[q], lo_i = o[D + q], hi_r = o[16 + q], hi_i = o[D + 16 + q];
        const float sr = __shfl_xor_sync(0xffffffffu, odd ? lo_r : hi_r, 1);  // what this lane sends
        const float si = __shfl_xor_sync(0xffffffffu, odd ? lo_i : hi_i, 1);
        const int j = odd ? 16 + q : q;   // what this lane stores
        const float4 v = odd ? make_float4(sr, si, hi_r, hi_i) : make_float4(lo_r, lo_i, sr, si);
        if (ok) *reinterpret_cast<float4*>(psi + 2 * (bs | dense_off<K>(j, bits))) = v;
      }
    }
    tc_fence_before();
    __syncthreads();  // TMEM and the A tiles are free for the next tile
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(N));
}

inline constexpr int dense_tc_smem(int K) {
  return 2 * 128 * (2 << K) * 4 + 2 * (2 << K) * (2 << K) * 4 + 1024;
}

}  // namespace dev
}  // namespace tcx
