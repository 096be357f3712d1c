// plan.h -- host-side circuit compiler for the tcx engine (the K.jit analog,
// PAPER.md:492-496).  Lowers a gate list to fused kernel ops on physical index bits,
// schedules light-cone window passes and register stages, and lays out the tables
// the sm_100a kernels execute.  Pure host code: no CUDA calls here.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tcx.h"

#include "device_abi.h"

namespace tcx {

constexpr int kMaxQubits = 40;
constexpr int kMaxTileBits = 15;
constexpr int kMaxRegBits = 4;
constexpr int kMaxCutBits = 26;  // cut tables (bytes per amplitude index) up to 64 MB

// One original 1-qubit gate folded into a fused U1 op (applied in list order).
struct Constituent {
  int32_t kind;     // tcx_gate_kind of a 1-qubit gate
  int32_t param;    // theta column or -1
  double coeff;     // rotation: angle multiplier (param>=0) or fixed angle
  int64_t payload;  // complex offset into Plan::fixed for TCX_U1, else -1
  int32_t contrib;  // gradient contribution index (param >= 0), else -1
};

// Diagonal op term: phase(r) *= exp(i * w_eff * (-1)^popc(r & mask)), where
// w_eff = w (param < 0) or w * theta[param].  R_Z-type gates exp(-i a Z_m / 2) with
// a = coeff*theta give w = -coeff/2.
struct DiagTerm {
  uint64_t mask;
  int32_t param;      // theta column, -1 fixed, <= -2 derived: the diagonal phase Phi of the
                      // kind-3 U1 op (-2 - param) (mask 0: its global part, else its Z part)
  double w;
  int32_t slot = -1;  // op-local gradient slot (param terms sharing (param, w))
};

struct Op {
  uint8_t type = 0;
  uint64_t bits = 0;  // every physical bit the op reads (dependencies)
  uint64_t need = 0;  // bits that must be inside the tile / register set
  int b0 = -1, b1 = -1;  // U1: bit; U2F: (hi=q0, lo=q1); CX: (target, control)
  std::vector<Constituent> cons;  // U1
  int64_t u2_payload = -1;        // U2F
  std::vector<DiagTerm> terms;    // DIAG
  int nslots = 0;                 // DIAG: distinct gradient slots
  bool has_param = false;
  bool fold_init = false;  // U1: the first op on a |0> bit; the JIT's first pass writes the
                           // product state it produces (column 0 of its 2x2 per theta row)
  bool skip_udag = false;  // backward: no op executed before it touches its bits, so U^dagger
                           // on psi and lambda can be skipped (plan.cpp, stage emission)
  int tan = 0;       // U1 applied as (I + K) with a deferred real factor (plan.cpp tan_kind_of):
                     // 1 RX only, 2 RY only (u00 = u11 real), 3 general unitary run, whose
                     // diagonal phase Phi = diag(u00, u11) / |u00| follows as a derived DIAG op
  int tan_idx = -1;  // index of its u00 in the per-row fp64 factor table
  bool lut = false;  // DIAG: one weight class (param, |w|); phase from a (T+1)-entry table
  int ngroups = 0;   // DIAG (not LUT): distinct register-slot masks of its terms = complex
                     // multiplies per amplitude in the kernels (cost model)
  // layout (filled by the scheduler)
  int pass = -1;
  int mat_off = 0, mat_len = 0;  // Reals in the per-theta table
  int acc_off = -1, acc_len = 0; // global partial slots
};


// materialize items (per theta): U1 product, U2F copy, diag (cos, sin)
struct MItem {
  int32_t type;      // OP_U1 / OP_U2F / OP_DIAG(term)
  int32_t mat_off;   // Reals
  int32_t cons_begin, cons_count;
  int64_t payload;
  int32_t param, pad;
  double w;
  int32_t tan, tan_idx;  // U1: deferred-factor rotation (Op::tan) and its factor-table index
};
// Deferred rotation factors (Op::tan): per pass, the forward list of factor ops (execution
// order) and the backward walk (reverse execution order) that the scan kernel (tcx.cu) runs
// per theta row to choose fast/exact per op, write the pass-end scales into the pass header
// and the gradient-slot corrections S^2.
struct SPass {
  int32_t hdr;             // absolute offset (Reals) of the pass header [S_fwd, S_bwd, plain, pad]
  int32_t fbeg, fcnt, bbeg, bcnt, pad;
};
struct SFwd {
  int32_t idx, flag;       // factor index, absolute offset (Reals) of the op's exact flag
};
struct SBwd {
  int32_t kind, a, b, pad; // 0: gradient slots [a, a + b); 1: factor a (flag at b)
};
struct DCons {       // device copy of Constituent
  int32_t kind, param;
  double coeff;
  int64_t payload;
  int32_t contrib, pad;
};
struct GItem {       // finalize items
  int32_t type;      // OP_U1: R' -> constituent contributions; OP_DIAG: scalar slot
  int32_t acc;       // global slot (U1: 3 Im components, + 3 Re components with q_grad)
  int32_t cons_begin, cons_count;
  double factor;     // DIAG: -2 * w
  int32_t contrib;
  int32_t re_acc;    // q_grad: slot of the real-part sums (U1: acc + 3, structured acc + 1), else -1
  int32_t phase;     // U1 kind 3 (Op::tan): R' was taken before its diagonal phase, so the
                     //   generators are conjugated B' = Phi^dagger B Phi (finalize_kernel)
  int32_t cls;       // U1 structured class (u1_class): 0 three slots (cX, cY, cZ), else the
                     //   one component the class needs (1 cX, 2 cY, 3 cZ) in one slot
};

// Dense k-qubit block (north_star step 2): a run of gates fused into one
// 2^k x 2^k unitary U = G_m ... G_1 on k physical bits; applied as Psi' = U Psi with Psi
// the state viewed as [2^k x 2^(n-k)].  Block-local index j: bit i of j <-> bits[i].
constexpr int kMaxDenseK = 5;
struct DGate {       // device: one gate of a dense block, on block-local bits
  int32_t kind, a, b, param;  // a: local bit of q0, b: local bit of q1 (-1: 1-qubit)
  double coeff;
  int64_t payload;            // complex offset into Plan::fixed (U1: 4, U2: 16), else -1
  int32_t contrib, pad;       // gradient contribution index (param >= 0), else -1
};
struct DBlock {
  int32_t k;
  int32_t bits[kMaxDenseK];   // ascending physical bits
  int32_t gate_begin, gate_count;
  int32_t shared;             // 1: no parameters -> U in the row-independent table
  int32_t mat_off;            // complex offset of U (row-major 2^k x 2^k) in its table
  int32_t acc_off;            // backward: offset of the block's Q partials (2^(2k) reals)
  int32_t has_param;
  int32_t first;              // 1: no earlier block touches these bits -> the backward needs
                              // only R' here, not U^dagger on psi / lambda (plan.cpp)
};

struct PassInfo {
  int seg = 0;                      // sharded: segment (layout) this pass runs in
  uint64_t wmask = 0;
  int W[kMaxTileBits + 1] = {0};   // local -> physical bit
  std::vector<int> ops;             // plan op indices in program order
  int stage_begin = 0, stage_count = 0;  // into Plan::kstages
  int kop_begin = 0, kop_count = 0;      // into Plan::kops
  int kterm_begin = 0, kterm_count = 0;  // into Plan::kterms
  int mat_begin = 0, mat_count = 0;
  int acc_begin = 0, acc_count = 0;
  int max_stage_acc = 0;
  int last_is_top = 1;   // last stage uses the load/store mapping
  int tan_hdr = -1;      // >= 0: pass-relative offset of [S_fwd, S_bwd, plain, pad] (deferred factors)
};

struct Pauli {
  int n = 0;
  std::vector<uint8_t> codes;  // [T][n]
  std::vector<double> weights;
  uint64_t hash = 0;           // content hash (binding cache key; handles may be reused)
};

// Lambda evaluation unit: a window pass computing some Pauli groups.
struct LamUnit {
  int swapped = 0;      // sharded: computed after the global <-> top-local exchange
  uint64_t wmask = 0;
  int W[kMaxTileBits + 1] = {0};
  int group_begin = 0, group_count = 0;  // into Binding::groups
  int fwd_pass = -1;   // >= 0: fused into this forward pass (the last one)
};

struct Binding {        // (circuit, pauli) specific lambda schedule
  uint64_t hash = 0;    // Pauli::hash this binding was built from
  std::vector<KGroup> groups;
  std::vector<KPTerm> pterms;
  std::vector<LamUnit> units;
  bool xmask_ok = true;
  std::string err;
  // device copies (per device), released by the destructor (tcx.cu)
  std::map<int, std::pair<void*, void*>> dev;  // device -> (groups, pterms)
  Binding() = default;
  Binding(const Binding&) = delete;
  Binding& operator=(const Binding&) = delete;
  ~Binding();
};

struct DeviceTables;

struct JitKernel {      // NVRTC-compiled specialisation (jit.cpp)
  std::string key, name;
  std::string cache_key;  // disk cache entry it came from / went to ("" = none)
  std::vector<char> cubin;
};

struct Plan {
  int n = 0, P = 0;
  tcx_dtype dtype = TCX_C64;
  int t = 0, r = 0, c = 0, h = 0;
  int max_ops_per_pass = 0;
  int gbits = 0, nloc = 0;       // sharded state: global index bits, local bits (= n if not)
  int nseg = 1;                  // sharded: layouts separated by global<->top-local exchanges
  std::vector<int> init_pos;     // sharded: initial physical bit of each qubit (empty: n-1-q)
  std::vector<tcx_gate> gates;  // validated input (decode)
  std::vector<double> mats_in;  // input payloads
  std::vector<double> fixed;    // complex (re, im) payloads referenced by ops
  std::vector<Op> ops;
  std::vector<PassInfo> passes;
  std::vector<KOp> kops;
  std::vector<KTerm> kterms;
  std::vector<KStage> kstages;
  std::vector<MItem> mitems;
  int ntan = 0;                  // deferred-factor rotation ops (Op::tan)
  std::vector<SPass> spass;      // scan program (tan_scan_kernel), empty if ntan == 0
  std::vector<SFwd> sfwd;
  std::vector<SBwd> sbwd;
  std::vector<DCons> dcons;
  std::vector<GItem> gitems;
  std::vector<int32_t> param_ptr, param_list;  // CSR param -> contrib indices
  int n_contrib = 0;
  int mat_total = 0;
  int acc_total = 0;
  int layout[kMaxQubits] = {0};  // final physical bit of each qubit
  bool relabeled = false;
  bool unitary = true;
  int64_t tiles = 1;             // 2^(n - t)
  int tpc = 1;                   // tiles per CTA (depends on the tile count only, never on B)
  int jit_nsub = 1;              // lock-stepped sub-tiles per CTA in JIT kernels
  std::vector<std::vector<std::pair<uint64_t, int>>> cut_sets;  // LUT cut tables (mask, sign)
  int jit_pipe = -1;             // JIT TMA passes prefetch the next tile: 1 on, 0 off, 2 forward, -1 auto
  bool xchunk_forbid = false;     // sharded planning keeps the chunk bits out of post-exchange windows
  int xchunk_bits = 0;           // sharded: exchange column chunks = 2^xchunk_bits (overlap)
  bool cluster = false;          // cluster-resident: gbits = log2(CTAs per row), t = nloc

  uint64_t init_hmask = 0;         // leading H gates folded into the initial state (bits)
  uint64_t fold_mask = 0;          // bits whose leading U1 op is folded into the initial state
  double init_amp = 1.0;           // 2^(-popc(init_hmask)/2)
  int dense_k = 0;                 // > 0: gates run as dense k-qubit blocks (tcx_build_opts)
  bool q_grad = false;             // window plan also accumulates Re R' components
  int64_t l2_rows = 0;             // > 0: theta rows per L2-resident group (run())
  std::vector<DBlock> dblocks;     // in execution order (before the window passes)
  std::vector<DGate> dgates;
  int dmat_row = 0;                // complex entries per theta row (parameterised blocks)
  int dmat_shared = 0;             // complex entries of the row-independent table
  int dacc_total = 0;              // backward Q partial reals per CTA slot

  bool jit_on = false;             // per-circuit specialised kernels (compiled lazily)
  std::map<std::string, JitKernel> jit;  // key (jit.h) -> compiled CUBIN
  std::string jit_note;            // why JIT is off, if it is
  std::mutex jit_mu;

  std::mutex mu;
  std::map<uint64_t, std::shared_ptr<Binding>> bindings;  // keyed by Pauli::hash
  std::map<uint64_t, uint64_t> binding_use;  // Pauli::hash -> last use (LRU eviction)
  uint64_t use_clock = 0;
  std::map<int, std::shared_ptr<DeviceTables>> dev;
};

// TMA view of a pass window: the state [B][2^n] of 8-byte elements
// (complex64 = 1, complex128 = 2 per amplitude) as a rank <= 5 tensor whose dims are the
// runs of window / non-window index bits; the box is the tile (window dims full, others 1).
struct TmaDims {
  int rank = 0;         // 0: the window does not fit a rank-5 box (plain loads are used)
  int start[5];         // first element-index bit of each dim (element = amp * epa + half)
  int bits[5];          // dim size 2^bits (the last dim also spans the batch: bits = -1)
  int inwin[5];         // 1: dim lies inside the window (box = full dim)
  int epa;              // 8-byte elements per amplitude
  // multi-box windows (more runs than a rank-5 box holds): the box covers the first four runs,
  // the window bits above them (inside dim 4) are iterated -- 2^sub boxes per tile, box j the
  // contiguous chunk j << kel (elements) of the tile in shared memory
  int sub = 0;          // iterated window bits
  int kel = 0;          // element-index bits one box covers
  int sub_pos[8];       // element-index positions of the iterated bits (increasing)
};
TmaDims tma_dims(int n, uint64_t wmask, bool c128);

// Build; returns TCX_OK or an error with message.
int u1_class(const std::vector<Constituent>& cons);  // plan.cpp: 0 general, 1 XT, 2 RE, 3 DG
tcx_status build_plan(int n, int P, const tcx_gate* gates, int64_t G, const double* mats,
                      int64_t nmat, tcx_dtype dtype, const tcx_build_opts* opts, Plan& plan,
                      std::string& err);
// The step list of a sharded (or cluster-resident) program, identical on every rank
std::vector<tcx_shard_step> shard_program(const Plan& P, const Binding& B, bool want_grad);
tcx_status build_pauli(int n, int T, const uint8_t* codes, const double* w, Pauli& p,
                       std::string& err);
std::shared_ptr<Binding> bind(Plan& plan, const Pauli& pauli);

// swizzled shared-memory bit table: sw(1 << p) for local position p
uint32_t swizzle_bit(int p, bool c128);

}  // namespace tcx
