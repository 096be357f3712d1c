// device_abi.h -- POD tables and kernel arguments shared by the host plan, the
// precompiled kernels and the NVRTC-generated (JIT) kernels.  Byte-identical layout
// on every side; no host-only headers (it is also fed to NVRTC).
#pragma once
#ifdef __CUDACC_RTC__
typedef signed char int8_t;
typedef short int16_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
#else
#include <stdint.h>
#endif
#if defined(__CUDACC__) || defined(__CUDACC_RTC__)
#define TCX_HD __host__ __device__
#else
#define TCX_HD
#endif

namespace tcx {

enum : uint8_t { OP_U1 = 1, OP_U2F = 2, OP_CX = 3, OP_DIAG = 4 };
constexpr uint8_t kExtCtrl = 0xFF;

// ---- kernel tables (POD, copied to the device as-is) ----
struct KOp {       // 16 bytes
  uint8_t type, a, b, cbit;  // slots / external control bit
  int16_t mat;     // offset (Reals) into the pass's smem matrix table
  int16_t nterm;   // DIAG terms
  int32_t acc;     // stage-local acc slot base, -1 none
  int32_t term;    // DIAG: first KTerm (pass-relative)
};
struct KTerm {     // 16 bytes
  uint64_t mask;   // physical bits
  int16_t wofs;    // (cos, sin) pair offset in the pass matrix table
  int16_t acc;     // stage-local acc slot, -1 none
  int32_t pad;
};
struct KStage {    // 48 bytes
  int8_t R[8];     // local positions of register slots k < r
  int8_t T[16];    // local positions of thread bits m < h (lanes first)
  int32_t op_begin, op_count;      // pass-relative KOp range
  int32_t acc_begin, acc_count;    // pass-relative slot range
  int32_t same_as_prev, pad;       // 1: identical mapping to the previous stage
};
struct KGroup {    // Pauli terms sharing one X/Y flip mask
  uint64_t xphys;     // flip mask, physical bits
  uint32_t xlocal;    // flip mask in tile-local bits (global == 0)
  int32_t term_begin, term_count;
  int32_t global;     // 1: partner amplitudes gathered from global memory
};
struct KPTerm {    // 24 bytes: coefficient alpha_j * i^nY * (-1)^popc(x & zy)
  uint64_t zy;     // physical Y|Z mask
  double cre, cim;
};

namespace dev {

enum {
  M_INIT = 1, M_LOAD_PSI = 2, M_FWD = 4, M_LAMBDA = 8, M_LOAD_LAM = 16,
  M_STORE_PSI = 32, M_STORE_LAM = 64, M_BWD = 128
};
enum { KM_FWD = 0, KM_BWD = 1, KM_MEGA = 2 };

struct PassArgs {
  alignas(64) unsigned char tmap[2][128];  // CUtensorMap of psi / lambda (TMA tile I/O)
  int use_tma;                             // 1: tmap valid for this launch
  uint64_t gbase;                          // sharded state: rank << n_local (else 0)
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
  uint64_t init_hmask;     // M_INIT: leading H gates folded into the initial state |+> on
  double init_amp;         //   these bits, amplitude init_amp = 2^(-popc/2) (plan.cpp)
  int fold_active;         // 1: the call starts from |0..0>, so leading U1 ops folded into
                           //   the product initial state are skipped in forward passes (JIT)
  const uint8_t* cut[15];  // LUT cut tables: c(r) per local index (plan.cpp, JIT kernels)
  // chunked launches (sharded exchange overlapped with the next pass): this launch covers the
  // tiles whose tile-index bits [chunk_pos, chunk_pos + chunk_bits) equal chunk_val; the CTA's
  // partial slot is b * cta_stride + cta_base + blockIdx.x (cta_stride = CTAs per full launch)
  int chunk_pos, chunk_bits, chunk_val, cta_base;
  int64_t cta_stride;
  // tile order of the JIT pass kernels: 0 blocked (CTA x takes tiles [x*tpc, (x+1)*tpc)),
  // 1 interleaved (CTA x takes tiles it*gridDim.x + x; tcx.cu picks it when a row's CTAs are
  // co-resident, so the two halves of a line shared by neighbouring tiles are read together)
  int tile_ilv, pad_ilv;
};
// tile index of a (possibly chunked) launch: the chunk value inserted at chunk_pos
TCX_HD inline int64_t chunk_tile(int64_t t, int pos, int bits, int val) {
  if (!bits) return t;
  const int64_t lo = t & ((1ll << pos) - 1);
  return ((t >> pos) << (pos + bits)) | ((int64_t)val << pos) | lo;
}

struct SmemLayout {
  int xb_psi, xb_lam, mats, wacc, cacc, stages, red, pb, total;
};
TCX_HD inline int al16(int x) { return (x + 15) & ~15; }
TCX_HD inline SmemLayout smem_layout(int t, int h, int realsz, int mat_count,
                                     int max_stage_acc, int acc_count, int nstages, bool two,
                                     int nsub = 1, int pipe = 0) {
  // nsub lock-stepped sub-tiles per CTA (JIT kernels): one exchange buffer each
  SmemLayout L;
  int off = 0;
  const int csz = 2 * realsz;
  L.xb_psi = off;
  off = al16(off + nsub * (csz << t));
  L.xb_lam = off;
  if (two) off = al16(off + nsub * (csz << t));
  L.mats = off;
  off = al16(off + realsz * mat_count);
  const int nw = nsub * (((1 << h) + 31) / 32);
  L.wacc = off;
  off = al16(off + realsz * nw * max_stage_acc);
  L.cacc = off;
  off = al16(off + 8 * acc_count);
  L.stages = off;
  off = al16(off + (int)sizeof(KStage) * nstages);
  L.red = off;
  off = al16(off + 8 * 32);
  // pipelined TMA passes: the next tile (psi, and lambda in two-state kernels) lands here
  // while this one is computed (128-byte aligned TMA destination); pipe == 2 (two-state
  // kernels, "half" pipeline) prefetches psi only, so two CTAs still fit one SM
  L.pb = 0;
  if (pipe) {
    off = (off + 127) & ~127;
    L.pb = off;
    off += (((two && pipe == 1) || pipe == 3) ? 2 : 1) * (csz << t);  // 3: two one-state buffers
  }
  L.total = off;
  return L;
}

}  // namespace dev
}  // namespace tcx
