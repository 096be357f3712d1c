// plan.cpp -- circuit compiler: validation, lowering to fused ops on physical bits,
// light-cone window scheduling, register-stage scheduling, table layout.
//
// Method references:
//  * gate semantics: PAPER.md:343-386 (§3.2 gates, exp1, unitary), SURVEY §8 conventions.
//  * "fuses runs of gates on low qubits into one pass" (north_star step 1): every pass
//    runs all remaining ops whose non-diagonal bits lie in its window and that are not
//    blocked by an earlier unrun op on a shared bit (SURVEY §8a "Window scheduling").
//  * the reverse sweep replays the same passes/stages backwards (SURVEY §8a-7, R = F).
#include "plan.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <array>
#include <functional>
#include <set>

namespace tcx {
namespace {

using cd = std::complex<double>;

bool is_rot(int k) {
  return k == TCX_RX || k == TCX_RY || k == TCX_RZ || k == TCX_RXX || k == TCX_RYY ||
         k == TCX_RZZ || k == TCX_RROT;
}
bool is_2q(int k) {
  return k == TCX_CNOT || k == TCX_CZ || k == TCX_SWAP || k == TCX_RXX || k == TCX_RYY ||
         k == TCX_RZZ || k == TCX_U2;
}
bool is_diag1(int k) {
  return k == TCX_I || k == TCX_Z || k == TCX_S || k == TCX_SDG || k == TCX_T ||
         k == TCX_TDG || k == TCX_RZ;
}
inline int popc64(uint64_t x) { return __builtin_popcountll(x); }

bool unitary_check(const double* m, int d) {
  double worst = 0;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      cd s = 0;
      for (int k = 0; k < d; ++k)
        s += std::conj(cd(m[2 * (k * d + i)], m[2 * (k * d + i) + 1])) *
             cd(m[2 * (k * d + j)], m[2 * (k * d + j) + 1]);
      if (i == j) s -= 1.0;
      worst = std::max(worst, std::abs(s));
    }
  return worst < 1e-9;
}

// ------------------------------------------------------------------ lowering
int tan_kind_of(const Op& o);  // deferred-factor kind (below)
struct Lowerer {
  Plan& P;
  struct Run {
    bool open = false, diag = true;
    std::vector<Constituent> cons;
  };
  Run runs[kMaxQubits];
  int last_on_bit[kMaxQubits];
  int last_diag = -1;
  bool fold = false;              // fold leading U1 ops into the product initial state
  bool pristine[kMaxQubits];      // physical bit still |0> (no op emitted, not H-folded)
  explicit Lowerer(Plan& p) : P(p) {
    std::fill(last_on_bit, last_on_bit + kMaxQubits, -1);
    std::fill(pristine, pristine + kMaxQubits, true);
  }

  void emit(Op&& op) {
    int idx = (int)P.ops.size();
    if (fold && op.type == OP_U1 && pristine[op.b0]) {
      op.fold_init = true;
      P.fold_mask |= 1ull << op.b0;
    }
    for (int b = 0; b < P.n; ++b)
      if (op.bits >> b & 1) pristine[b] = false;
    for (int b = 0; b < P.n; ++b)
      if (op.bits >> b & 1) last_on_bit[b] = idx;
    if (op.type == OP_DIAG) last_diag = idx;
    const bool derive = op.type == OP_U1 && tan_kind_of(op) == 3;
    const int bit = op.b0;
    P.ops.push_back(std::move(op));
    if (derive) {
      // U = |u00| Phi (I + K): the kernels apply (I + K) (scale deferred); Phi = diag(u00, u11)
      // / |u00| = e^{i gamma} e^{i w Z} follows as this diagonal op (materialize_kernel writes
      // gamma and w from the same fused 2x2), free to move and merge like any other
      Op d;
      d.type = OP_DIAG;
      d.bits = 1ull << bit;
      d.need = 0;
      d.terms.push_back({0, -2 - idx, 0.0});
      d.terms.push_back({1ull << bit, -2 - idx, 0.0});
      emit(std::move(d));
    }
  }
  void emit_diag(const std::vector<DiagTerm>& terms, uint64_t bits) {
    if (terms.empty()) return;
    int lastS = -1;
    for (int b = 0; b < P.n; ++b)
      if (bits >> b & 1) lastS = std::max(lastS, last_on_bit[b]);
    bool par = false;
    for (auto& t : terms) par |= t.param >= 0;
    // Diagonal gates stay separate ops here (a merged op would carry the union of their
    // bits as false light-cone dependencies); runs of consecutive diagonal ops inside one
    // pass are merged after pass scheduling (merge_pass_diagonals).
    static const bool merge = getenv("TCX_DIAG_EARLY_MERGE") != nullptr;
    if (merge && last_diag >= 0 && last_diag >= lastS) {
      Op& d = P.ops[last_diag];
      d.terms.insert(d.terms.end(), terms.begin(), terms.end());
      d.bits |= bits;
      d.has_param |= par;
      for (int b = 0; b < P.n; ++b)
        if (bits >> b & 1) last_on_bit[b] = last_diag;
      return;
    }
    Op op;
    op.type = OP_DIAG;
    op.bits = bits;
    op.need = 0;
    op.terms = terms;
    op.has_param = par;
    emit(std::move(op));
  }
  // exp(i w (-1)^{b}) factors of the diagonal 1-qubit gates (global phase kept so
  // that state-level parity holds): Z = e^{i pi/2 (1 - Z)}, S = e^{i pi/4 (1 - Z)},
  // T = e^{i pi/8 (1 - Z)}, RZ(a) = e^{-i a/2 Z}.
  void diag_terms_of(const Constituent& c, int bit, std::vector<DiagTerm>& out) {
    const uint64_t m = 1ull << bit;
    auto fixed2 = [&](double w) {
      out.push_back({0, -1, w});
      out.push_back({m, -1, -w});
    };
    switch (c.kind) {
      case TCX_I: break;
      case TCX_Z: fixed2(M_PI / 2); break;
      case TCX_S: fixed2(M_PI / 4); break;
      case TCX_SDG: fixed2(-M_PI / 4); break;
      case TCX_T: fixed2(M_PI / 8); break;
      case TCX_TDG: fixed2(-M_PI / 8); break;
      case TCX_RZ: out.push_back({m, c.param, -c.coeff / 2}); break;
      default: break;
    }
  }
  void add1(int bit, const Constituent& c, bool diag) {
    Run& R = runs[bit];
    R.open = true;
    R.diag = R.diag && diag;
    R.cons.push_back(c);
  }
  void close(int bit) {
    Run& R = runs[bit];
    if (!R.open) return;
    if (R.diag) {
      std::vector<DiagTerm> terms;
      for (auto& c : R.cons) diag_terms_of(c, bit, terms);
      emit_diag(terms, 1ull << bit);
    } else {
      Op op;
      op.type = OP_U1;
      op.bits = op.need = 1ull << bit;
      op.b0 = bit;
      op.cons = R.cons;
      for (auto& c : op.cons) op.has_param |= c.param >= 0 && is_rot(c.kind);
      emit(std::move(op));
    }
    R = Run();
  }
};

void normalize_diag(Op& op) {
  // combine fixed terms by mask and param terms by (param, mask)
  std::map<std::pair<int, uint64_t>, double> acc;
  for (auto& t : op.terms) acc[{t.param, t.mask}] += t.w;
  std::vector<DiagTerm> fixed, par;
  for (auto& kv : acc) {
    DiagTerm t{kv.first.second, kv.first.first, kv.second, -1};
    if (t.param <= -2) {
      fixed.push_back(t);  // derived phase (kind-3 U1): its value comes from materialize
    } else if (t.param < 0) {
      if (t.w != 0.0) fixed.push_back(t);
    } else {
      par.push_back(t);
    }
  }
  // gradient slots: distinct (param, w)
  std::map<std::pair<int, double>, int> slots;
  for (auto& t : par) {
    auto key = std::make_pair(t.param, t.w);
    auto it = slots.find(key);
    if (it == slots.end()) it = slots.emplace(key, (int)slots.size()).first;
    t.slot = it->second;
  }
  std::stable_sort(par.begin(), par.end(),
                   [](const DiagTerm& a, const DiagTerm& b) { return a.slot < b.slot; });
  op.terms = fixed;
  op.terms.insert(op.terms.end(), par.begin(), par.end());
  op.nslots = (int)slots.size();
  op.has_param = !par.empty();
}

// Regroup the diagonal ops of one pass (program-ordered op list).  Lowering emits a fused
// 1-qubit op when the next multi-qubit gate reaches its qubit, so a QAOA cost layer arrives
// interleaved with the previous mixer's rotations (U q1, U q2, D e1, U q3, D e2, ...) and
// every term would become a phase multiply of its own.  Diagonal ops commute with each other
// and with every op on other bits, and pass CNOTs by conjugation, so each may sink to any gap
// before the first later U1 / U2F op of the pass touching its (conjugated) bits.  The
// non-diagonal ops keep their order; the diagonal ops of one weight class (param, |w|) are
// placed by greedy interval stabbing (fewest gaps = fewest LUT ops after the merge below).
void regroup_diag(Plan& P, std::vector<int>& ops) {
  std::vector<int> nd;                 // non-diagonal ops, in order
  struct DI { int op, hi, orig; std::pair<int, double> key; };
  std::vector<DI> di;
  for (int i : ops) {
    const Op& o = P.ops[i];
    if (o.type != OP_DIAG) { nd.push_back(i); continue; }
    DI d{i, 0, (int)nd.size(), {-3, (double)i}};
    bool one = !o.terms.empty(), derived = !o.terms.empty();
    for (auto& tm : o.terms) {
      one = one && tm.param == o.terms[0].param && std::fabs(tm.w) == std::fabs(o.terms[0].w);
      derived = derived && tm.param <= -2;
    }
    if (derived) d.key = {-2, 0.0};  // kind-3 phases: one class for placement
    else if (one) d.key = {o.terms[0].param, std::fabs(o.terms[0].w)};
    di.push_back(d);
  }
  if (di.empty()) return;
  const int m = (int)nd.size();
  // Sinking a diagonal past a CNOT conjugates it: a term on the target t picks up the control
  // c (Z_t -> Z_c Z_t); a term on the control alone commutes.  Only U1 / U2F ops on a term's
  // bits stop it.
  auto pass_over = [&](std::vector<uint64_t>& masks, const Op& x) {
    if (x.type == OP_CX) {
      for (auto& mk : masks)
        if (mk >> x.b0 & 1) mk ^= 1ull << x.b1;
      return true;
    }
    uint64_t u = 0;
    for (auto mk : masks) u |= mk;
    return (x.bits & u) == 0;
  };
  for (auto& d : di) {
    std::vector<uint64_t> masks;
    for (auto& tm : P.ops[d.op].terms) masks.push_back(tm.mask);
    d.hi = m;
    for (int k = d.orig; k < m; ++k)
      if (!pass_over(masks, P.ops[nd[k]])) { d.hi = k; break; }
  }
  std::map<std::pair<int, double>, std::vector<int>> bykey;
  for (int i = 0; i < (int)di.size(); ++i) bykey[di[i].key].push_back(i);
  std::vector<int> gap(di.size(), -1);
  for (auto& kv : bykey) {
    std::vector<int> v = kv.second;
    std::sort(v.begin(), v.end(), [&](int a, int b) {
      return di[a].hi < di[b].hi || (di[a].hi == di[b].hi && a < b);
    });
    for (int a : v) {
      if (gap[a] >= 0) continue;
      const int pt = di[a].hi;
      for (int b2 : v)
        if (gap[b2] < 0 && di[b2].orig <= pt && di[b2].hi >= pt) gap[b2] = pt;
    }
  }
  std::vector<std::vector<int>> at(m + 1);
  for (int i = 0; i < (int)di.size(); ++i) {
    Op& o = P.ops[di[i].op];
    std::vector<uint64_t> masks;
    for (auto& tm : o.terms) masks.push_back(tm.mask);
    for (int k = di[i].orig; k < gap[i]; ++k) pass_over(masks, P.ops[nd[k]]);
    o.bits = 0;
    for (size_t t2 = 0; t2 < masks.size(); ++t2) {
      o.terms[t2].mask = masks[t2];
      o.bits |= masks[t2];
    }
    at[gap[i]].push_back(di[i].op);  // original order kept
  }
  std::vector<int> out;
  out.reserve(ops.size());
  for (int g = 0; g <= m; ++g) {
    for (int i : at[g]) out.push_back(i);
    if (g < m) out.push_back(nd[g]);
  }
  ops.swap(out);
}

// Structured 2x2 class of a fused 1-qubit run (KOp.nterm of a U1 op; the JIT skips the
// identically-zero coefficients and, in the adjoint, the R' entries the generator never
// reads).  Each class is closed under products:
//   1 XT  [[re, i re], [i re, re]]: I, Z, Y, RX      generator X -> B = +-X (R'01, R'10)
//   2 RE  real:                     I, Z, X, H, RY   generator Y -> B = det(S) Y (R'01, R'10)
//   3 DG  diagonal:                 I, Z, S, T, RZ   generator Z -> B = Z (R'00, R'11)
// 0 = general (any TCX_U1 payload or mixed classes).  TCX_U1_STRUCT=0 disables.
int u1_class_of(const std::vector<Constituent>& cons) {
  static const int off = [] {
    const char* e = std::getenv("TCX_U1_STRUCT");
    return e && e[0] == '0';
  }();
  if (off) return 0;
  unsigned m = 7;  // bit k-1: class k possible
  for (const auto& c : cons) {
    unsigned k = 0;
    switch (c.kind) {
      case TCX_I: case TCX_Z: k = 7; break;
      case TCX_RX: case TCX_Y: k = 1; break;
      case TCX_RY: case TCX_X: case TCX_H: k = 2; break;
      case TCX_RZ: case TCX_S: case TCX_SDG: case TCX_T: case TCX_TDG: k = 4; break;
      default: k = 0; break;
    }
    m &= k;
  }
  if (m & 4) return 3;
  if (m & 2) return 2;
  if (m & 1) return 1;
  return 0;
}

// ------------------------------------------------------------- scheduling
double op_weight(const Op& o) {
  switch (o.type) {
    case OP_U1: return 8.0;
    case OP_U2F: return 16.0;
    case OP_CX: return 1.0;
    default: return 2.0 + 4.0 * (double)o.terms.size();
  }
}
// Per-theta table entries (Reals).  complex64 U1 ops store the 2x2 as 16 packed FP32x2
// coefficient pairs (forward and adjoint forms) so the FFMA2 operands
// load straight into aligned register pairs; complex128 stores the plain 8 Reals.
thread_local bool g_packed_u1 = false;
// Deferred-factor rotations (DESIGN.md §Kernels "Deferred rotation factors"): a fused run of
// RX gates only (XT, u00 = u11 real) or RY gates only (RE, u00 = u11 real) is applied as
// U = u00 (I + K), K off-diagonal; the kernels apply I + K (one FFMA2 per output amplitude
// instead of an FMUL2 + FFMA2) and multiply the pass's product of the u00 back at its end.
// Runs folded into the product initial state keep the plain form.  TCX_NO_TAN=1 turns it off.
thread_local bool g_tan_on = false;
thread_local bool g_tan_general = false;  // kind 3 (TCX_TAN_GENERAL=1)
int u1_class_of(const std::vector<Constituent>& cons);
int tan_kind_of(const Op& o) {
  if (!g_tan_on || o.type != OP_U1 || o.fold_init || o.cons.empty()) return 0;
  bool rx = true, ry = true, any = false, unit = true;
  for (auto& c : o.cons) {
    switch (c.kind) {  // unitary constituents only (payload U1, noise and structure gates excluded)
      case TCX_I: case TCX_X: case TCX_Y: case TCX_Z: case TCX_H: case TCX_S: case TCX_SDG:
      case TCX_T: case TCX_TDG: case TCX_RX: case TCX_RY: case TCX_RZ: break;
      default: unit = false; break;
    }
    if (c.kind == TCX_I) continue;
    any = true;
    rx = rx && c.kind == TCX_RX;
    ry = ry && c.kind == TCX_RY;
  }
  if (!any || !unit) return 0;
  if (rx) return 1;
  if (ry) return 2;
  // general runs (the structured classes already cost 2 FFMA2 per output amplitude): opt-in,
  // measured slower -- the derived phases merge into diagonal ops that stall the stage
  // schedule (cfg2: 44 -> 58 register stages, 3572 -> 3490 circuits/s; cfg1 330k -> 216k)
  return (g_tan_general && u1_class_of(o.cons) == 0) ? 3 : 0;
}
int op_mats(const Op& o) {
  switch (o.type) {
    // complex128 deferred-factor ops append [k0, k1, exact flag, pad]; complex64 ops keep
    // them in adjoint-half coefficient pairs the structured class never reads (materialize_kernel)
    // kind 3 appends the four coefficient pairs of K (forward) and K^dagger (adjoint):
    // 8 packed pairs + 1 spare (complex64) / [k01, k10] complex (complex128)
    case OP_U1: {
      const int tk = tan_kind_of(o);
      if (g_packed_u1) return tk == 3 ? 50 : 32;
      return tk == 3 ? 14 : (tk ? 12 : 8);
    }
    case OP_U2F: return 32;
    case OP_CX: return 0;
    default: return 2 * ((int)o.terms.size() + (o.lut ? 1 : 0));
  }
}
thread_local bool g_q_grad = false;  // set per build_plan (this thread's plan)
int op_accs(const Op& o) {
  if (!o.has_param) return 0;
  // U1: Pauli components (cX, cY, cZ) of R' (Im parts), + (rX, rY, rZ) real parts with
  // q_grad -- structured classes need one component (XT cX, RE cY, DG cZ); DIAG: one
  // Im(lambda* psi) sum per slot, + one Re sum per slot
  const int base = o.type == OP_U1 ? (u1_class_of(o.cons) ? 1 : 3) : o.nslots;
  return g_q_grad ? 2 * base : base;
}

struct Budget {
  int mats, accs, ops;
};

struct Scheduler {
  Plan& P;
  std::vector<char> done;
  int first = 0;
  uint64_t full;
  int nl;  // local index bits (windows live there; sharded states keep the top bits global)
  Budget pass_budget;
  explicit Scheduler(Plan& p) : P(p), done(p.ops.size(), 0) {
    full = (P.n >= 64) ? ~0ull : ((1ull << P.n) - 1);
    nl = P.nloc;
  }
  // light-cone closure under tile mask W (physical)
  double closure(uint64_t W, std::vector<int>* out) {
    uint64_t blocked = 0;
    double score = 0;
    int mats = 0, accs = 0, nops = 0;
    for (int i = first; i < (int)P.ops.size(); ++i) {
      if (done[i]) continue;
      const Op& o = P.ops[i];
      bool ok = !(o.bits & blocked) && !(o.need & ~W);
      if (ok) {
        int m2 = mats + op_mats(o), a2 = accs + op_accs(o);
        if (m2 > pass_budget.mats || a2 > pass_budget.accs ||
            (pass_budget.ops > 0 && nops + 1 > pass_budget.ops))
          ok = false;
        else {
          mats = m2;
          accs = a2;
          nops++;
          score += op_weight(o);
          if (out) out->push_back(i);
        }
      }
      if (!ok) {
        blocked |= o.bits;
        if ((blocked & full) == full) break;
      }
    }
    return score;
  }
  // first not-runnable op's needed bits (guides window growth)
  uint64_t first_missing(uint64_t W) {
    uint64_t blocked = 0;
    for (int i = first; i < (int)P.ops.size(); ++i) {
      if (done[i]) continue;
      const Op& o = P.ops[i];
      if (!(o.bits & blocked) && (o.need & ~W)) return o.need & ~W;
      if ((o.bits & blocked) || (o.need & ~W)) blocked |= o.bits;
    }
    return 0;
  }
  // Window for the next pass.  Candidates come from three greedy families (score growth,
  // earliest need, contiguous runs); with lookahead each of the best few is rolled out with
  // the greedy choice to the end of the schedule and the one finishing in the fewest passes
  // wins (ties: more work now).
  bool lookahead = false;
  uint64_t forbid = 0;  // bits the next window must leave out (exchange chunk bits)
  bool tma_ok(uint64_t W) const { return tma_dims(nl, W, P.dtype == TCX_C128).rank > 0; }
  uint64_t choose_window() {
    std::vector<std::pair<double, uint64_t>> cand;
    uint64_t W0 = candidates(&cand);
    if (!lookahead || cand.size() < 2) return W0;
    std::sort(cand.begin(), cand.end(), [](const std::pair<double, uint64_t>& a,
                                           const std::pair<double, uint64_t>& b) {
      return a.first > b.first || (a.first == b.first && a.second < b.second);
    });
    cand.erase(std::unique(cand.begin(), cand.end(),
                           [](const std::pair<double, uint64_t>& a, const std::pair<double, uint64_t>& b) {
                             return a.second == b.second;
                           }),
               cand.end());
    const size_t K = std::min<size_t>(cand.size(), 6);
    const std::vector<char> done0 = done;
    const int first0 = first;
    int bestp = 1 << 30;
    uint64_t bestW = W0;
    for (size_t k = 0; k < K; ++k) {
      uint64_t W = cand[k].second;
      int passes = 0;
      bool ok = true, finished = false;
      for (;;) {
        std::vector<int> list;
        closure(W, &list);
        if (list.empty()) {
          ok = false;
          break;
        }
        for (int i : list) done[i] = 1;
        while (first < (int)P.ops.size() && done[first]) first++;
        ++passes;
        finished = first >= (int)P.ops.size();
        if (finished || passes >= bestp) break;
        W = candidates(nullptr);
      }
      done = done0;
      first = first0;
      // ties in the pass count go to windows whose tile is a TMA box (<= 5 contiguous index
      // runs): those passes move tiles with cp.async.bulk.tensor (and prefetch the next one)
      if (ok && finished &&
          (passes < bestp || (passes == bestp && tma_ok(cand[k].second) && !tma_ok(bestW)))) {
        bestp = passes;
        bestW = cand[k].second;
      }
    }
    return bestW;
  }
  uint64_t candidates(std::vector<std::pair<double, uint64_t>>* all) {
    const int n = nl, t = P.t, c = P.c;
    if (n <= t) return (n >= 64) ? ~0ull : ((1ull << n) - 1);
    const uint64_t base = (1ull << c) - 1;
    uint64_t bestW = 0;
    double best = -1;
    auto consider = [&](uint64_t W) {
      double s = closure(W, nullptr);
      if (all) all->push_back({s, W});
      if (s > best) {
        best = s;
        bestW = W;
      }
    };
    auto fill = [&](uint64_t W) {  // pad with lowest unused bits
      for (int b = 0; b < n && popc64(W) < t; ++b)
        if (!(forbid >> b & 1)) W |= 1ull << b;
      return W;
    };
    // (a) greedy growth by score
    {
      uint64_t W = base;
      while (popc64(W) < t) {
        double cur = closure(W, nullptr), bs = -1;
        int bb = -1;
        for (int b = 0; b < n; ++b) {
          if ((W >> b & 1) || (forbid >> b & 1)) continue;
          double s = closure(W | (1ull << b), nullptr);
          if (s > bs) {
            bs = s;
            bb = b;
          }
        }
        if (bs <= cur) {
          uint64_t miss = first_missing(W);
          uint64_t add = 0;
          for (int b = 0; b < n; ++b)
            if ((miss >> b & 1) && !(forbid >> b & 1)) {
              add = 1ull << b;
              break;
            }
          if (!add) {
            W = fill(W);
            break;
          }
          W |= add;
        } else {
          W |= 1ull << bb;
        }
      }
      consider(W);
    }
    // (b) earliest-need-first
    {
      uint64_t W = base;
      const uint64_t lmask = (n >= 64) ? ~0ull : ((1ull << n) - 1);
      for (int i = first; i < (int)P.ops.size() && popc64(W) < t; ++i) {
        if (done[i] || (P.ops[i].need & ~lmask) || (P.ops[i].need & forbid)) continue;  // global bits never enter a window
        uint64_t nw = W | P.ops[i].need;
        if (popc64(nw) <= t) W = nw;
      }
      consider(fill(W));
    }
    // (c) contiguous runs above the coalescing bits
    for (int s = c; s + (t - c) <= n; ++s) {
      uint64_t W = base;
      for (int b = s; b < s + (t - c); ++b) W |= 1ull << b;
      if (!(W & forbid)) consider(W);
    }
    return bestW;
  }
};

// combinations helper
void combos(int t, int r, std::vector<uint32_t>& out) {
  for (uint32_t m = 0; m < (1u << t); ++m)
    if (__builtin_popcount(m) == r) out.push_back(m);
}

struct StageOut {
  uint32_t Rloc;                 // local register-bit mask
  std::vector<int> ops;          // plan op indices
};

// Stage scheduling inside one pass: ops run in the stage whose register set covers
// their non-diagonal bits (relaxed locality for CX controls and diagonals).
static const double g_cx_bonus = getenv("TCX_CX_BONUS") ? atof(getenv("TCX_CX_BONUS")) : 1.0;
void schedule_stages(Plan& P, const PassInfo& pass, std::vector<StageOut>& stages) {
  const int t = P.t, r = P.r, h = P.h;
  std::vector<int> loc(P.n, -1);
  for (int l = 0; l < t; ++l) loc[pass.W[l]] = l;
  auto lneed = [&](const Op& o) {  // register-slot need (U2F runs through smem)
    uint32_t m = 0;
    if (o.type == OP_U2F) return m;
    for (int b = 0; b < P.n; ++b)
      if (o.need >> b & 1) m |= 1u << loc[b];
    return m;
  };
  std::vector<uint32_t> need(pass.ops.size());
  for (size_t i = 0; i < pass.ops.size(); ++i) need[i] = lneed(P.ops[pass.ops[i]]);
  std::vector<char> done(pass.ops.size(), 0);
  size_t remaining = pass.ops.size();
  const int kStageAccMax = 256;
  auto closure_d = [&](const std::vector<char>& dn, uint32_t R, std::vector<int>* out) {
    uint64_t blocked = 0;
    double s = 0;
    int accs = 0;
    for (size_t i = 0; i < pass.ops.size(); ++i) {
      if (dn[i]) continue;
      const Op& o = P.ops[pass.ops[i]];
      bool ok = !(o.bits & blocked) && !(need[i] & ~R);
      if (ok && accs + op_accs(o) > kStageAccMax) ok = false;
      if (ok) {
        accs += op_accs(o);
        s += op_weight(o);
        // a CNOT whose control is also a register slot is a free rename; with an outside
        // control it becomes predicated register swaps (TCX_CX_BONUS tunes the preference)
        if (o.type == OP_CX && loc[o.b1] >= 0 && (R >> loc[o.b1] & 1)) s += g_cx_bonus;
        if (out) out->push_back((int)i);
      } else {
        blocked |= o.bits;
      }
    }
    return s;
  };
  std::vector<uint32_t> cand;
  combos(t, r, cand);
  const uint32_t top = ((1u << t) - 1) & ~((1u << h) - 1);
  auto greedy_pick = [&](const std::vector<char>& dn, double* score) {
    double best = -1;
    uint32_t R = top;
    for (uint32_t m : cand) {
      double sc = closure_d(dn, m, nullptr);
      if (sc > best) {
        best = sc;
        R = m;
      }
    }
    if (score) *score = best;
    return R;
  };
  // Stage lookahead (round 2): each stage boundary costs a shared-memory exchange of the tile
  // (plus two barriers), so among the best few greedy choices take the one whose greedy
  // completion needs the fewest register-set changes, counting the return to the load/store
  // set at the end.  TCX_STAGE_LOOKAHEAD=K candidates (0: plain greedy); big passes stay greedy.
  static const int kLook = getenv("TCX_STAGE_LOOKAHEAD") ? atoi(getenv("TCX_STAGE_LOOKAHEAD")) : 4;
  const bool look = kLook > 1 && pass.ops.size() <= 160;
  auto finish_cost = [&](std::vector<char> dn, size_t rem, uint32_t R) {
    int changes = 0;
    uint32_t cur = R;
    for (int guard = 0; rem > 0 && guard < 256; ++guard) {
      const uint32_t nx = greedy_pick(dn, nullptr);
      std::vector<int> idx;
      closure_d(dn, nx, &idx);
      if (idx.empty()) break;
      for (int i : idx) dn[i] = 1;
      rem -= idx.size();
      if (nx != cur) ++changes;
      cur = nx;
    }
    return changes + (cur != top ? 1 : 0);
  };
  bool first = true;
  uint32_t curR = top;
  while (remaining > 0 || first) {
    uint32_t R = top;
    if (!first) {
      if (!look) {
        R = greedy_pick(done, nullptr);
      } else {
        std::vector<std::pair<double, uint32_t>> sc;
        for (uint32_t m : cand) sc.push_back({closure_d(done, m, nullptr), m});
        std::sort(sc.begin(), sc.end(), [](const std::pair<double, uint32_t>& a, const std::pair<double, uint32_t>& b) {
          return a.first > b.first || (a.first == b.first && a.second < b.second);
        });
        int bestc = 1 << 30;
        double bests = -1;
        for (int k = 0; k < (int)sc.size() && k < kLook; ++k) {
          if (sc[k].first <= 0) break;
          std::vector<char> dn = done;
          std::vector<int> idx;
          closure_d(dn, sc[k].second, &idx);
          for (int i : idx) dn[i] = 1;
          const int c = (sc[k].second != curR ? 1 : 0) + finish_cost(dn, remaining - idx.size(), sc[k].second);
          if (c < bestc || (c == bestc && sc[k].first > bests)) {
            bestc = c;
            bests = sc[k].first;
            R = sc[k].second;
          }
        }
        if (bests < 0) R = sc.empty() ? top : sc[0].second;
      }
    }
    std::vector<int> idx;
    closure_d(done, R, &idx);
    StageOut so;
    so.Rloc = R;
    for (int i : idx) {
      done[i] = 1;
      so.ops.push_back(pass.ops[i]);
    }
    remaining -= idx.size();
    if (!first && idx.empty()) break;  // cannot happen (r >= arity); guard
    stages.push_back(std::move(so));
    curR = R;
    first = false;
  }
}

// thread-bit order: lanes first, chosen so the lane bits' bank vectors are independent
void thread_order(uint32_t Rloc, int t, bool c128, int8_t* T) {
  const int lg = c128 ? 3 : 4;
  std::vector<int> nr;
  for (int l = 0; l < t; ++l)
    if (!(Rloc >> l & 1)) nr.push_back(l);
  std::vector<int> lanes, rest;
  // greedy GF(2) basis over bank bits
  std::vector<uint32_t> basis;
  auto bankvec = [&](int l) { return swizzle_bit(l, c128) & ((1u << lg) - 1); };
  auto indep = [&](uint32_t v) {
    for (uint32_t b : basis) v = std::min(v, v ^ b);
    return v != 0 ? v : 0u;
  };
  for (int l : nr) {
    if ((int)lanes.size() < lg) {
      uint32_t v = indep(bankvec(l));
      if (v) {
        // keep basis reduced
        basis.push_back(v);
        std::sort(basis.rbegin(), basis.rend());
        lanes.push_back(l);
        continue;
      }
    }
    rest.push_back(l);
  }
  int m = 0;
  for (int l : lanes) T[m++] = (int8_t)l;
  for (int l : rest) T[m++] = (int8_t)l;
}

}  // namespace

int u1_class(const std::vector<Constituent>& cons) { return u1_class_of(cons); }

// Swizzle of the tile-local element index in shared memory: the low lg bits (bank
// group within a 128-byte row) are XORed with a GF(2)-linear image of the higher bits,
// chosen so that any (t - r) positions span the bank space.
uint32_t swizzle_bit(int p, bool c128) {
  static const uint32_t col64[] = {3, 5, 6, 9, 10, 12, 7, 11, 13, 14, 15, 3, 5};
  static const uint32_t col128[] = {3, 5, 6, 7, 1, 2, 4, 3, 5, 6, 7, 1, 2};
  const int lg = c128 ? 3 : 4;
  if (p < lg) return 1u << p;
  return (1u << p) ^ (c128 ? col128[p - lg] : col64[p - lg]);
}

TmaDims tma_dims(int n, uint64_t wmask, bool c128) {
  TmaDims d{};
  d.epa = c128 ? 2 : 1;
  // element-index bits: for complex128 bit 0 is the (re,im)-half, inside the window
  const int eb = c128 ? 1 : 0;
  std::vector<std::pair<int, int>> runs;  // (start element-bit, nbits), alternating in/out
  std::vector<int> in;
  int bit = 0;
  const int nbits = n + eb;
  auto win = [&](int e) { return e < eb ? true : ((wmask >> (e - eb)) & 1) != 0; };
  while (bit < nbits) {
    const bool w = win(bit);
    int len = 0;
    while (bit + len < nbits && win(bit + len) == w) ++len;
    // window runs longer than 8 bits split (box dims <= 256)
    for (int o = 0; o < len;) {
      int l = w ? std::min(8, len - o) : len - o;
      runs.push_back({bit + o, l});
      in.push_back(w ? 1 : 0);
      o += l;
    }
    bit += len;
  }
  // batch: merged into a trailing out-of-window run, else its own dim
  if (in.back() == 0) {
    runs.back().second = -1;
  } else {
    runs.push_back({nbits, -1});
    in.push_back(0);
  }
  // multi-box windows (opt-in, TCX_TMA_MULTIBOX=1): measured slower on cfg3, whose scattered
  // windows then move 8 boxes of 4 KB per tile (541 vs 584 circuits/s), so such windows keep
  // plain coalesced loads by default
  if (runs.size() > 5 && !getenv("TCX_TMA_MULTIBOX")) return d;  // rank 0: plain loads
  if (runs.size() > 5) {
    // multi-box: the first four runs form the box, dim 4 (box extent 1) is everything above;
    // its window bits are iterated (at most 2^6 boxes per tile)
    std::vector<int> sp;
    for (size_t i = 4; i < runs.size(); ++i)
      if (in[i])
        for (int k = 0; k < runs[i].second; ++k) sp.push_back(runs[i].first + k);
    if (sp.size() > 6) return d;  // rank 0: plain loads
    const int s4 = runs[4].first;
    runs.resize(4);
    in.resize(4);
    runs.push_back({s4, -1});
    in.push_back(0);
    d.sub = (int)sp.size();
    for (int k = 0; k < d.sub; ++k) d.sub_pos[k] = sp[k];
  }
  d.rank = (int)runs.size();
  for (int i = 0; i < d.rank; ++i) {
    d.start[i] = runs[i].first;
    d.bits[i] = runs[i].second;
    d.inwin[i] = in[i];
  }
  // innermost box >= 16 bytes
  if (!d.inwin[0] || (1 << d.bits[0]) * 8 < 16) d.rank = 0;
  for (int i = 0; i < d.rank; ++i)
    if (d.inwin[i]) d.kel += d.bits[i];
  // multi-box: every box lands at a 128-byte aligned shared-memory address
  if (d.sub && (8 << d.kel) < 128) d.rank = 0;
  return d;
}

tcx_status build_pauli(int n, int T, const uint8_t* codes, const double* w, Pauli& p,
                       std::string& err) {
  if (n < 1 || n > kMaxQubits) {
    err = "pauli: n_qubits out of range";
    return TCX_E_INVALID;
  }
  if (T < 0 || (T > 0 && (!codes || !w))) {
    err = "pauli: bad term arrays";
    return TCX_E_INVALID;
  }
  p.n = n;
  p.codes.assign(codes, codes + (size_t)T * n);
  p.weights.assign(w, w + T);
  uint64_t h = 1469598103934665603ull ^ (uint64_t)n;
  auto mix = [&](const void* d, size_t len) {
    const unsigned char* c = (const unsigned char*)d;
    for (size_t i = 0; i < len; ++i) h = (h ^ c[i]) * 1099511628211ull;
  };
  mix(p.codes.data(), p.codes.size());
  mix(p.weights.data(), p.weights.size() * sizeof(double));
  p.hash = h;
  for (int j = 0; j < T; ++j) {
    if (!std::isfinite(w[j])) {
      err = "pauli: term " + std::to_string(j) + " has a non-finite weight";
      return TCX_E_INVALID;
    }
    for (int q = 0; q < n; ++q)
      if (codes[(size_t)j * n + q] > 3) {
        err = "pauli: term " + std::to_string(j) + " qubit " + std::to_string(q) +
              " has code > 3";
        return TCX_E_INVALID;
      }
  }
  return TCX_OK;
}

namespace {
uint64_t remap_mask(uint64_t m, const int* perm, int n) {
  uint64_t r = 0;
  for (int b = 0; b < n; ++b)
    if (m >> b & 1) r |= 1ull << perm[b];
  return r;
}
void remap_op(Op& o, const int* perm, int n) {
  o.bits = remap_mask(o.bits, perm, n);
  o.need = remap_mask(o.need, perm, n);
  if (o.b0 >= 0) o.b0 = perm[o.b0];
  if (o.b1 >= 0) o.b1 = perm[o.b1];
  for (auto& t : o.terms) t.mask = remap_mask(t.mask, perm, n);
}
}  // namespace

// Sharded layout exchange: global bits L+i <-> top local bits L-g+i (i < g), so each rank's
// outgoing data for rank k is the contiguous chunk whose top local bits equal k.
void shard_swap_perm(int n, int g, int* perm) {
  const int L = n - g;
  for (int b = 0; b < n; ++b) perm[b] = b;
  for (int i = 0; i < g; ++i) {
    perm[L + i] = L - g + i;
    perm[L - g + i] = L + i;
  }
}

// Dense k-qubit block fusion (north_star step 2 "fused k-qubit blocks run
// as small dense complex contractions").  Greedy, in program order: every open block owns
// a disjoint set of physical bits; a gate joins (merging every open block it touches) when
// the union stays within k bits, else the blocks it touches are closed and emitted and
// the gate opens a new block (at k = 1 a 2-qubit gate is a block of its own; the cfg4
// brick circuit gives 8702 / 2999 / 2696 / 1500 / 1137 blocks for k = 1..5).  Per bit, blocks are emitted in program order,
// and blocks on disjoint bits commute, so the emitted sequence equals the gate list.
// SWAP stays a relabel of the qubit -> bit map (as in the window lowering).
void build_dense(Plan& P, const tcx_gate* gates, int64_t G, int* pos,
                 const std::function<int64_t(int64_t, int)>& payload_copy,
                 const std::function<int64_t(int64_t, int)>& payload_copy_raw) {
  struct Open {
    std::vector<int64_t> g;
    uint64_t mask = 0;
    int64_t order = 0;
  };
  std::vector<Open> open;
  std::vector<std::array<int, 2>> gp((size_t)G);  // physical bits of each gate when it ran
  auto pos_at = [&](int64_t gi) { return gp[(size_t)gi].data(); };
  auto emit = [&](const Open& o) {
    DBlock d{};
    bool theta_dep = false;
    d.k = popc64(o.mask);
    int loc[64];
    int i = 0;
    for (int b = 0; b < P.n; ++b)
      if (o.mask >> b & 1) {
        loc[b] = i;
        d.bits[i++] = b;
      }
    d.gate_begin = (int)P.dgates.size();
    d.gate_count = (int)o.g.size();
    for (int64_t gi : o.g) {
      const tcx_gate& x = gates[gi];
      DGate dg{};
      dg.kind = x.kind;
      dg.a = loc[pos_at(gi)[0]];
      dg.b = is_2q(x.kind) ? loc[pos_at(gi)[1]] : -1;
      dg.param = (is_rot(x.kind) || x.kind == TCX_DEPOL) ? x.param : -1;
      dg.coeff = x.coeff;
      dg.payload = -1;
      if (x.kind == TCX_U1) dg.payload = payload_copy(x.payload, 2);
      if (x.kind == TCX_U2) dg.payload = payload_copy(x.payload, 4);
      if (x.kind == TCX_DEPOL) dg.payload = payload_copy_raw(x.payload, 2);
      if (x.kind == TCX_RROT) dg.payload = payload_copy_raw(x.payload, 1);
      dg.contrib = -1;
      d.has_param |= dg.param >= 0 && is_rot(x.kind);  // gradient slots
      theta_dep |= dg.param >= 0 || x.kind == TCX_RROT;  // U depends on the theta row
      P.dgates.push_back(dg);
    }
    d.shared = theta_dep ? 0 : 1;
    const int m = 1 << (2 * d.k);
    if (d.shared) {
      d.mat_off = P.dmat_shared;
      P.dmat_shared += m;
    } else {
      d.mat_off = P.dmat_row;
      P.dmat_row += m;
    }
    d.acc_off = -1;
    if (d.has_param) {  // R' = sum psi_out lam_out^dagger: 2^(2k) complex (re, im)
      d.acc_off = P.dacc_total;
      P.dacc_total += 2 * m;
    }
    P.dblocks.push_back(d);
  };
  int64_t order = 0;
  for (int64_t gi = 0; gi < G; ++gi) {
    const tcx_gate& x = gates[gi];
    if (x.kind == TCX_I) continue;
    if (x.kind == TCX_SWAP) {
      std::swap(pos[x.q0], pos[x.q1]);
      P.relabeled = true;
      continue;
    }
    const int ar = is_2q(x.kind) ? 2 : 1;
    int* pp = pos_at(gi);
    pp[0] = pos[x.q0];
    pp[1] = ar == 2 ? pos[x.q1] : -1;
    const uint64_t Q = (1ull << pp[0]) | (ar == 2 ? (1ull << pp[1]) : 0ull);
    uint64_t U = Q;
    std::vector<size_t> touch;
    for (size_t i = 0; i < open.size(); ++i)
      if (open[i].mask & Q) {
        touch.push_back(i);
        U |= open[i].mask;
      }
    std::sort(touch.begin(), touch.end(),
              [&](size_t a, size_t b) { return open[a].order < open[b].order; });
    if (popc64(U) <= P.dense_k) {
      Open m;
      m.order = touch.empty() ? order++ : open[touch[0]].order;
      for (size_t i : touch) m.g.insert(m.g.end(), open[i].g.begin(), open[i].g.end());
      m.g.push_back(gi);
      m.mask = U;
      std::vector<Open> keep;
      for (size_t i = 0; i < open.size(); ++i)
        if (!(open[i].mask & Q)) keep.push_back(std::move(open[i]));
      keep.push_back(std::move(m));
      open.swap(keep);
      continue;
    }
    for (size_t i : touch) emit(open[i]);
    std::vector<Open> keep;
    for (size_t i = 0; i < open.size(); ++i)
      if (!(open[i].mask & Q)) keep.push_back(std::move(open[i]));
    Open nb;
    nb.g.push_back(gi);
    nb.mask = Q;
    nb.order = order++;
    keep.push_back(std::move(nb));
    open.swap(keep);
  }
  std::sort(open.begin(), open.end(), [](const Open& a, const Open& b) { return a.order < b.order; });
  for (auto& o : open) emit(o);
  // adjoint shortcut (as for window ops): later-processed blocks read only partial traces
  // over their complement, invariant under a unitary on bits no earlier block touches
  uint64_t touched = 0;
  for (auto& d : P.dblocks) {
    uint64_t m = 0;
    for (int i = 0; i < d.k; ++i) m |= 1ull << d.bits[i];
    d.first = (m & touched) == 0 ? 1 : 0;
    touched |= m;
  }
}

tcx_status build_plan(int n, int Pn, const tcx_gate* gates, int64_t G, const double* mats,
                      int64_t nmat, tcx_dtype dtype, const tcx_build_opts* opts, Plan& P,
                      std::string& err) {
  const int gb_req = opts ? std::max(0, opts->global_bits) : 0;
  if (n < 1 || n - gb_req > 34 || n > kMaxQubits) {
    err = "n_qubits must be in [1, 34] per rank (n - global_bits <= 34)";
    return TCX_E_INVALID;
  }
  if (Pn < 0 || G < 0 || (G > 0 && !gates) || nmat < 0 || (nmat > 0 && !mats)) {
    err = "bad sizes or null arrays";
    return TCX_E_INVALID;
  }
  if (dtype != TCX_C64 && dtype != TCX_C128) {
    err = "dtype must be TCX_C64 or TCX_C128";
    return TCX_E_INVALID;
  }
  P.n = n;
  P.P = Pn;
  P.dtype = dtype;
  P.gates.assign(gates, gates + G);
  P.mats_in.assign(mats, mats + 2 * nmat);
  // ---- validate (SPEC.md:301 "arity mismatch; qubit out of range", :422 op index)
  for (int64_t g = 0; g < G; ++g) {
    const tcx_gate& x = gates[g];
    auto bad = [&](const char* why) {
      err = "gate " + std::to_string(g) + ": " + why;
      return TCX_E_INVALID;
    };
    if (x.kind < 0 || x.kind >= TCX_NKINDS) return bad("unknown kind");
    if (x.q0 < 0 || x.q0 >= n) return bad("q0 out of range");
    if (is_2q(x.kind)) {
      if (x.q1 < 0 || x.q1 >= n) return bad("q1 out of range");
      if (x.q1 == x.q0) return bad("q0 == q1");
    } else if (x.q1 != -1) {
      return bad("q1 must be -1 for a 1-qubit gate");
    }
    if (is_rot(x.kind)) {
      if (x.param < -1 || x.param >= Pn) return bad("param out of range");
      if (!std::isfinite(x.coeff)) return bad("non-finite coeff");
    } else if (x.kind == TCX_DEPOL) {
      if (x.param < 0 || x.param >= Pn) return bad("depolarizing status column out of range");
      if (x.payload < 0 || x.payload + 2 > nmat) return bad("payload out of range");
      const double px = mats[2 * x.payload], py = mats[2 * x.payload + 1],
                   pz = mats[2 * x.payload + 2];
      if (!(px >= 0 && py >= 0 && pz >= 0 && px + py + pz <= 1.0 + 1e-12))
        return bad("depolarizing probabilities must be >= 0 with px + py + pz <= 1");
      continue;
    } else if (x.param != -1) {
      return bad("param must be -1 for a non-rotation gate");
    }
    if (x.kind == TCX_RROT) {
      if (x.payload < 0 || x.payload + 1 > nmat) return bad("payload out of range");
      const double sc = mats[2 * x.payload];
      if (!(sc >= 0 && sc < Pn && sc == std::floor(sc)))
        return bad("random-axis rotation: status column out of range");
      continue;
    }
    if (x.kind == TCX_U1 || x.kind == TCX_U2) {
      int64_t need = x.kind == TCX_U1 ? 4 : 16;
      if (x.payload < 0 || x.payload + need > nmat) return bad("payload out of range");
      for (int64_t e = 0; e < 2 * need; ++e)
        if (!std::isfinite(mats[2 * x.payload + e])) return bad("non-finite payload");
    } else if (x.payload != -1) {
      return bad("payload must be -1 for this kind");
    }
  }
  // ---- options
  const bool c128 = dtype == TCX_C128;
  int gb = opts ? std::max(0, opts->global_bits) : 0;
  if (gb > 0 && (gb > 6 || n - gb < 2 * gb + 2)) {
    err = "global_bits must be in [1, 6] with n - g >= 2g + 2 local bits";
    return TCX_E_INVALID;
  }
  // Cluster-resident states: the plan of a state "sharded" over the 2^g_c
  // CTAs of one thread-block cluster, one tile per CTA (t = n - g_c), run by one JIT
  // megakernel per batch whose registers hold psi and lambda (jit.cpp cluster_kernel).
  const int cb = opts ? std::max(0, opts->cluster_bits) : 0;
  if (cb > 0) {
    if (gb > 0) {
      err = "cluster_bits and global_bits are exclusive";
      return TCX_E_INVALID;
    }
    if (cb > 4 || n - cb < 2 * cb + 2 || n - cb > (c128 ? 12 : 13)) {
      err = "cluster_bits must be in [1, 4] with 2 cluster_bits + 2 <= n - cluster_bits <= 13 "
            "(complex64) / 12 (complex128)";
      return TCX_E_INVALID;
    }
    if (opts && opts->dense_k > 0) {
      err = "dense_k is not supported with cluster_bits";
      return TCX_E_UNSUPPORTED;
    }
    gb = cb;
    P.cluster = true;
  }
  P.gbits = gb;
  P.nloc = n - gb;
  int tdef = c128 ? 11 : 12;
  int t = opts && opts->tile_bits > 0 ? opts->tile_bits : tdef;
  int c = opts && opts->coalesce_bits > 0 ? opts->coalesce_bits : (c128 ? 2 : 3);
  t = std::min(t, kMaxTileBits);
  if (t >= n - gb) t = n - gb;
  // register bits per stage: 4 for full tiles; small single-tile states use more threads per
  // tile (latency-bound: cfg1 n=10 c128 measured 255k -> 287k circuits/s with r = 2)
  if (P.cluster) t = n - gb;  // the whole local state is one tile
  int r = opts && opts->reg_bits > 0 ? opts->reg_bits : (t < tdef ? (n - gb <= 10 ? 2 : 3) : 4);
  if (P.cluster) r = std::max(r, gb);  // the exchange moves register slots (top local bits)
  r = std::min(r, kMaxRegBits);
  if (r > t) r = t;
  if (t - r > 9) r = t - 9;  // at most 512 threads per tile (kernel launch bounds)
  if (r > kMaxRegBits) {
    err = "tile_bits too large: needs reg_bits <= 4 with <= 512 threads (t <= 13)";
    return TCX_E_INVALID;
  }
  if (c > t) c = t;
  if (n - gb > t && t - c < 2) {
    err = "tile_bits - coalesce_bits must be >= 2";
    return TCX_E_INVALID;
  }
  P.t = t;
  P.r = r;
  P.c = c;
  P.h = t - r;
  P.max_ops_per_pass = opts ? std::max(0, opts->max_ops_per_pass) : 0;
  P.dense_k = opts ? opts->dense_k : 0;
  P.q_grad = opts && opts->q_grad != 0 && gb == 0;
  if (opts && opts->l2_rows > 0) {
    P.l2_rows = opts->l2_rows;
  } else if (opts && opts->l2_rows < 0) {  // psi + lambda of a group within ~96 MB of L2
    const double row = 2.0 * (double)((int64_t)1 << (n - gb)) * (dtype == TCX_C128 ? 16.0 : 8.0);
    P.l2_rows = std::max<int64_t>(1, (int64_t)(96.0e6 / row));
  }
  if (P.dense_k < 0 || P.dense_k > kMaxDenseK) {
    err = "dense_k must be in [0, 5]";
    return TCX_E_INVALID;
  }
  if (P.dense_k > 0 && gb > 0) {
    err = "dense_k is not supported with global_bits (sharded state)";
    return TCX_E_UNSUPPORTED;
  }
  if (P.dense_k > 0 && n < 2) {
    err = "dense_k needs n_qubits >= 2";
    return TCX_E_INVALID;
  }
  P.tiles = 1ll << (n - gb - t);
  P.tpc = (int)std::min<int64_t>(64, std::max<int64_t>(1, P.tiles / 32));
  // two lock-stepped sub-tiles (512 threads) share one instruction stream in the JIT
  // kernels when tiles pair up and a sub-tile has whole warps
  // software-pipelined TMA tiles (prefetch of tile i+1 into its own buffer while tile i is
  // computed; the store of tile i drains while tile i+1 runs)
  P.jit_pipe = getenv("TCX_JIT_PIPE") ? std::min(2, std::max(0, atoi(getenv("TCX_JIT_PIPE")))) : -1;
  P.jit_nsub = 1;  // 2 = lock-stepped sub-tiles (measured slower with FFMA2 code; opt-in via TCX_JIT_NSUB)
  if (const char* e = getenv("TCX_JIT_NSUB"))
    if (atoi(e) == 2 && P.tpc % 2 == 0 && P.h >= 5) P.jit_nsub = 2;
  // ---- lower
  int pos[kMaxQubits];
  for (int q = 0; q < n; ++q) pos[q] = n - 1 - q;  // PAPER.md:249 qubit 0 = MSB
  if ((int)P.init_pos.size() == n)  // sharded layout search (tcx_circuit_build)
    for (int q = 0; q < n; ++q) pos[q] = P.init_pos[q];
  g_packed_u1 = dtype == TCX_C64;
  g_tan_on = getenv("TCX_NO_TAN") == nullptr && !P.cluster && P.dense_k == 0;  // cluster kernels: no plain variant
  g_tan_general = getenv("TCX_TAN_GENERAL") != nullptr;
  Lowerer L(P);
  auto payload_copy_raw = [&](int64_t off, int elems) {  // complex elements, no checks
    int64_t at = (int64_t)P.fixed.size() / 2;
    for (int64_t e = 0; e < 2 * elems; ++e) P.fixed.push_back(mats[2 * off + e]);
    return at;
  };
  auto payload_copy = [&](int64_t off, int d) {
    int64_t at = (int64_t)P.fixed.size() / 2;
    for (int64_t e = 0; e < 2 * d * d; ++e) P.fixed.push_back(mats[2 * off + e]);
    if (!unitary_check(mats + 2 * off, d)) P.unitary = false;
    return at;
  };
  if (P.dense_k > 0) build_dense(P, gates, G, pos, payload_copy, payload_copy_raw);
  // Leading H gates (the first gate on a still-|0> qubit) fold into the initial state: the
  // first pass writes |+> on those bits (amplitude 2^(-m/2)) instead of applying them, as
  // QAOA's H^n layer (PAPER.md:391 default input, SURVEY §8d cfg3 "H layer folded into a
  // write-only init").  The _in entries (caller input states) apply them explicitly.
  static const bool hfold = getenv("TCX_NO_HFOLD") == nullptr;
  // Leading U1 runs on |0> bits fold into a product initial state in the JIT's first pass
  // (the op stays in the plan for the backward's gradient term; with caller input states
  // the forward applies it as usual): amplitude(r) = prod over folded bits b of U_b[r_b][0].
  L.fold = gb == 0 && getenv("TCX_NO_UFOLD") == nullptr;
  std::vector<char> touched(n, 0);
  for (int64_t g = 0; g < G && P.dense_k == 0; ++g) {
    const tcx_gate& x = gates[g];
    if (hfold && x.kind == TCX_H && !touched[x.q0]) {
      P.init_hmask |= 1ull << pos[x.q0];
      L.pristine[pos[x.q0]] = false;
      touched[x.q0] = 1;
      continue;
    }
    if (x.kind == TCX_SWAP) {  // the qubits exchange states (a relabel below)
      std::swap(touched[x.q0], touched[x.q1]);
    } else if (x.kind != TCX_I) {
      touched[x.q0] = 1;
      if (is_2q(x.kind)) touched[x.q1] = 1;
    }
    if (!is_2q(x.kind)) {
      if (x.kind == TCX_I) continue;
      Constituent cn{x.kind, (is_rot(x.kind) || x.kind == TCX_DEPOL) ? x.param : -1, x.coeff, -1, -1};
      if (x.kind == TCX_U1) cn.payload = payload_copy(x.payload, 2);
      if (x.kind == TCX_DEPOL) cn.payload = payload_copy_raw(x.payload, 2);
      if (x.kind == TCX_RROT) cn.payload = payload_copy_raw(x.payload, 1);
      L.add1(pos[x.q0], cn, is_diag1(x.kind));
      continue;
    }
    const int a = pos[x.q0], b = pos[x.q1];
    const uint64_t ab = (1ull << a) | (1ull << b);
    switch (x.kind) {
      case TCX_SWAP:
        std::swap(pos[x.q0], pos[x.q1]);
        P.relabeled = true;
        break;
      case TCX_CNOT: {
        L.close(a);
        L.close(b);
        Op op;
        op.type = OP_CX;
        op.bits = ab;
        op.need = 1ull << b;
        op.b0 = b;  // target
        op.b1 = a;  // control
        L.emit(std::move(op));
        break;
      }
      case TCX_CZ:
        L.close(a);
        L.close(b);
        // CZ = exp(i pi/4 (1 - Z_a - Z_b + Z_a Z_b))
        L.emit_diag({{0, -1, M_PI / 4},
                     {1ull << a, -1, -M_PI / 4},
                     {1ull << b, -1, -M_PI / 4},
                     {ab, -1, M_PI / 4}},
                    ab);
        break;
      case TCX_RZZ:
        L.close(a);
        L.close(b);
        L.emit_diag({{ab, x.param, -x.coeff / 2}}, ab);
        break;
      case TCX_RXX:
      case TCX_RYY: {
        // R_XX(a) = (H x H) R_ZZ(a) (H x H);  R_YY(a) = (V^+ x V^+) R_ZZ(a) (V x V),
        // V = R_X(pi/2) (V^+ Z V = Y).
        Constituent pre{TCX_H, -1, 0.0, -1, -1}, post{TCX_H, -1, 0.0, -1, -1};
        if (x.kind == TCX_RYY) {
          pre = {TCX_RX, -1, M_PI / 2, -1, -1};
          post = {TCX_RX, -1, -M_PI / 2, -1, -1};
        }
        L.add1(a, pre, false);
        L.add1(b, pre, false);
        L.close(a);
        L.close(b);
        L.emit_diag({{ab, x.param, -x.coeff / 2}}, ab);
        L.add1(a, post, false);
        L.add1(b, post, false);
        break;
      }
      case TCX_U2: {
        L.close(a);
        L.close(b);
        Op op;
        op.type = OP_U2F;
        op.bits = op.need = ab;
        op.b0 = a;  // index 2*b_q0 + b_q1
        op.b1 = b;
        op.u2_payload = payload_copy(x.payload, 4);
        L.emit(std::move(op));
        break;
      }
    }
  }
  for (int b = 0; b < n; ++b) L.close(b);
  P.init_amp = std::pow(2.0, -0.5 * (double)popc64(P.init_hmask));
  for (auto& op : P.ops)
    if (op.type == OP_DIAG) normalize_diag(op);
  for (int q = 0; q < n; ++q) P.layout[q] = pos[q];

  // ---- pass scheduling
  g_packed_u1 = dtype == TCX_C64;
  g_q_grad = P.q_grad && P.dense_k == 0;
  Scheduler S(P);
  S.lookahead = gb == 0 && P.ops.size() <= 4096 && !(getenv("TCX_PLAN_GREEDY"));
  const int rb = c128 ? 8 : 4;  // bytes per Real
  S.pass_budget.mats = (24 * 1024) / rb;
  S.pass_budget.accs = 2048;
  S.pass_budget.ops = P.max_ops_per_pass;
  size_t left = P.ops.size();
  int seg = 0;
  bool swapped_last = false;
  // exchange chunks (overlap of an exchange with the next pass, comm.cuh): the 2 local bits
  // below the exchanged top g, kept out of the first window after each exchange when possible
  P.xchunk_bits = (gb > 0 && !P.cluster && P.nloc - gb - 2 >= P.c + 2 && !getenv("TCX_NO_XCHUNK")) ? 2 : 0;
  const uint64_t xmask = (P.xchunk_bits && P.xchunk_forbid)
      ? (((1ull << P.xchunk_bits) - 1) << (P.nloc - gb - P.xchunk_bits)) : 0;
  while (left > 0) {
    S.forbid = swapped_last ? xmask : 0;
    uint64_t W = S.choose_window();
    std::vector<int> list;
    S.closure(W, &list);
    if (list.empty() && S.forbid) {  // nothing runs without the chunk bits: plain window
      S.forbid = 0;
      W = S.choose_window();
      S.closure(W, &list);
    }
    S.forbid = 0;
    if (list.empty() && gb > 0 && !swapped_last) {
      // blocked on global qubits: exchange global <-> top-local bits, relabel what is left
      int perm[64];
      shard_swap_perm(n, gb, perm);
      for (size_t i = 0; i < P.ops.size(); ++i)
        if (!S.done[i]) remap_op(P.ops[i], perm, n);
      // no pass has run yet: the first pass (which writes the initial state) runs in the
      // new layout, so the folded-H bits move with the qubits
      if (P.passes.empty()) P.init_hmask = remap_mask(P.init_hmask, perm, n);
      for (int q = 0; q < n; ++q) pos[q] = perm[pos[q]];
      ++seg;
      swapped_last = true;
      continue;
    }
    if (list.empty()) {
      err = gb > 0 ? "sharded schedule stuck (a 4x4 payload spans a global and a top-local qubit)"
                   : "internal scheduler error (no progress)";
      return gb > 0 ? TCX_E_UNSUPPORTED : TCX_E_INVALID;
    }
    swapped_last = false;
    PassInfo pi;
    pi.seg = seg;
    pi.wmask = W;
    int l = 0;
    for (int b = 0; b < n; ++b)
      if (W >> b & 1) pi.W[l++] = b;
    pi.ops = list;
    for (int i : list) {
      S.done[i] = 1;
      P.ops[i].pass = (int)P.passes.size();
    }
    while (S.first < (int)P.ops.size() && S.done[S.first]) S.first++;
    left -= list.size();
    if (getenv("TCX_PLAN_DEBUG"))
      fprintf(stderr, "tcx plan: pass %zu seg %d window %llx ops %zu\n", P.passes.size(), seg,
              (unsigned long long)W, list.size());
    P.passes.push_back(std::move(pi));
  }
  static const bool lut_off = getenv("TCX_DIAG_NOLUT") != nullptr;
  static const bool regroup_off = getenv("TCX_NO_DIAG_REGROUP") != nullptr;
  for (auto& pass : P.passes)
    if (!regroup_off) regroup_diag(P, pass.ops);
  // merge runs of consecutive diagonal ops within each pass (they commute, and no op of
  // the pass sits between them; ops of other passes keep their order relative to the pass)
  for (auto& pass : P.passes) {
    std::vector<int> kept;
    for (int i : pass.ops) {
      Op& o = P.ops[i];
      if (o.type == OP_DIAG && !kept.empty() && P.ops[kept.back()].type == OP_DIAG) {
        Op& d = P.ops[kept.back()];
        d.terms.insert(d.terms.end(), o.terms.begin(), o.terms.end());
        d.bits |= o.bits;
        d.has_param |= o.has_param;
        o.terms.clear();
        o.has_param = false;
        o.nslots = 0;
        o.pass = -1;
        continue;
      }
      kept.push_back(i);
    }
    // split each merged diagonal into weight classes (param, |w|): a class of T >= 2 terms
    // becomes a LUT op (its phase is exp(i W (T - 2c)), c = number of terms whose signed
    // parity is odd: one table read and one complex multiply per amplitude); the rest
    // stays a grouped op
    std::vector<int> out;
    for (int i : kept) {
      if (P.ops[i].type != OP_DIAG || lut_off) {
        if (P.ops[i].type == OP_DIAG) normalize_diag(P.ops[i]);
        out.push_back(i);
        continue;
      }
      normalize_diag(P.ops[i]);
      std::map<std::pair<int, double>, std::vector<DiagTerm>> cls;
      for (auto& tm : P.ops[i].terms) cls[{tm.param, std::fabs(tm.w)}].push_back(tm);
      std::vector<DiagTerm> rest;
      std::vector<Op> luts;
      for (auto& kv : cls) {
        if (kv.second.size() < 2 || kv.first.second == 0.0) {
          rest.insert(rest.end(), kv.second.begin(), kv.second.end());
          continue;
        }
        Op L;
        L.type = OP_DIAG;
        L.lut = true;
        L.need = 0;
        L.pass = P.ops[i].pass;
        for (auto& tm : kv.second) L.bits |= tm.mask;
        L.terms = kv.second;
        normalize_diag(L);
        luts.push_back(std::move(L));
      }
      if (!rest.empty()) {
        Op& d = P.ops[i];
        d.terms = rest;
        d.bits = 0;
        for (auto& tm : rest) d.bits |= tm.mask;
        normalize_diag(d);
        out.push_back(i);
      } else {
        P.ops[i].terms.clear();
        P.ops[i].has_param = false;
        P.ops[i].nslots = 0;
        P.ops[i].pass = -1;
      }
      for (auto& L : luts) {
        out.push_back((int)P.ops.size());
        P.ops.push_back(std::move(L));
      }
    }
    pass.ops = out;
    if (const char* dbg = getenv("TCX_PLAN_DEBUG"))
      if (dbg[0] == '3') {
        fprintf(stderr, "pass-list %d:", (int)(&pass - &P.passes[0]));
        for (int oi : pass.ops) {
          const Op& o = P.ops[oi];
          if (o.type == OP_U1) fprintf(stderr, " U%d", o.b0);
          else if (o.type == OP_DIAG) fprintf(stderr, " D%s%zu", o.lut ? "L" : "", o.terms.size());
          else fprintf(stderr, " O");
        }
        fprintf(stderr, "\n");
      }
  }
  if (P.passes.empty() || P.passes.back().seg != seg) {  // init / trailing-layout pass
    PassInfo pi;
    pi.seg = seg;
    pi.wmask = (t >= 64) ? ~0ull : ((1ull << t) - 1);
    for (int l = 0; l < t; ++l) pi.W[l] = l;
    P.passes.push_back(pi);
  }
  P.nseg = seg + 1;
  for (int q = 0; q < n; ++q) P.layout[q] = pos[q];

  // ---- stages, kernel tables, matrix and accumulator layout
  int mat = 0, acc = 0;
  // Adjoint shortcut: the reverse sweep needs psi and lambda only through quantities that
  // are invariant under the same unitary applied to both on bits no later-processed op
  // touches (partial traces over those bits, inner products).  So an op that no earlier op
  // (in execution order) touches -- e.g. the first rotation layer -- takes its gradient
  // term in the backward but skips U^dagger on psi and lambda.  Execution order = passes,
  // stages, ops as emitted below; off for sharded plans (exchanges move data across bits).
  uint64_t touched_exec = 0;
  static const bool no_skip = getenv("TCX_NO_UDAG_SKIP") != nullptr;
  for (auto& pass : P.passes) {
    std::vector<StageOut> stages;
    schedule_stages(P, pass, stages);
    pass.stage_begin = (int)P.kstages.size();
    pass.kop_begin = (int)P.kops.size();
    pass.kterm_begin = (int)P.kterms.size();
    pass.mat_begin = mat;
    pass.acc_begin = acc;
    std::vector<int> loc(n, -1);
    for (int l = 0; l < t; ++l) loc[pass.W[l]] = l;
    int pass_acc = 0;
    uint32_t prevR = 0xFFFFFFFFu;
    // deferred-factor ops in this pass: header [S_fwd, S_bwd, plain, pad] at the start of its
    // table (plain = 1: this row runs the pass's plain-form variant)
    pass.tan_hdr = -1;
    for (auto& st : stages)
      for (int oi : st.ops)
        if (tan_kind_of(P.ops[oi]) && pass.tan_hdr < 0) pass.tan_hdr = 0;
    if (pass.tan_hdr == 0) mat += 4;
    std::vector<int> pass_kops_ops;  // plan op index of each kop of this pass (scan program)
    for (auto& st : stages) {
      KStage ks;
      std::memset(&ks, 0, sizeof(ks));
      int k = 0;
      for (int l = 0; l < t; ++l)
        if (st.Rloc >> l & 1) ks.R[k++] = (int8_t)l;
      if (st.Rloc == (((1u << t) - 1) & ~((1u << P.h) - 1)) && &st == &stages[0]) {
        for (int m = 0; m < P.h; ++m) ks.T[m] = (int8_t)m;  // load/store mapping
      } else {
        thread_order(st.Rloc, t, c128, ks.T);
      }
      ks.same_as_prev = 0;
      if (!P.kstages.empty() && (int)P.kstages.size() > pass.stage_begin) {
        const KStage& pv = P.kstages.back();
        ks.same_as_prev = (std::memcmp(pv.R, ks.R, sizeof(ks.R)) == 0 &&
                           std::memcmp(pv.T, ks.T, sizeof(ks.T)) == 0) ? 1 : 0;
      }
      (void)prevR;
      ks.op_begin = (int)P.kops.size() - pass.kop_begin;
      ks.acc_begin = pass_acc;
      int stage_acc = 0;
      auto slot_of = [&](int bit) {
        int l = loc[bit];
        for (int j = 0; j < P.r; ++j)
          if (ks.R[j] == l) return j;
        return -1;
      };
      for (int oi : st.ops) {
        Op& o = P.ops[oi];
        KOp ko;
        std::memset(&ko, 0, sizeof(ko));
        ko.type = o.type;
        o.skip_udag = !no_skip && gb == 0 && (o.type == OP_U1 || o.type == OP_DIAG) &&
                      (o.bits & touched_exec) == 0;
        touched_exec |= o.bits;
        ko.acc = -1;
        ko.term = -1;
        pass_kops_ops.push_back(oi);
        o.tan = tan_kind_of(o);
        o.tan_idx = o.tan ? P.ntan++ : -1;
        o.mat_off = mat;
        o.mat_len = op_mats(o);
        ko.mat = (int16_t)(mat - pass.mat_begin);
        if (o.type == OP_U1) {
          ko.a = (uint8_t)slot_of(o.b0);
          ko.nterm = (int16_t)u1_class_of(o.cons);
          ko.cbit = o.skip_udag ? 1 : 0;  // U1 / DIAG: backward skips U^dagger
          ko.b = (uint8_t)((o.fold_init ? 1 : 0) |  // U1: folded into the first pass's initial state
                           (o.tan << 1));           //     deferred-factor rotation kind
        } else if (o.type == OP_U2F) {  // tile-local positions (shared-memory op)
          ko.a = (uint8_t)loc[o.b0];
          ko.b = (uint8_t)loc[o.b1];
        } else if (o.type == OP_CX) {
          ko.a = (uint8_t)slot_of(o.b0);
          int cs = loc[o.b1] >= 0 ? slot_of(o.b1) : -1;
          ko.b = cs >= 0 ? (uint8_t)cs : kExtCtrl;
          ko.cbit = (uint8_t)o.b1;
          if (cs < 0) {  // uniform across a warp unless the control is a lane bit
            bool lane_bit = false;
            if (loc[o.b1] >= 0)
              for (int m = 0; m < std::min(P.h, 5); ++m) lane_bit |= ks.T[m] == loc[o.b1];
            ko.nterm = lane_bit ? 0 : 1;
          }
        } else {
          ko.nterm = (int16_t)o.terms.size();
          ko.term = (int)P.kterms.size() - pass.kterm_begin;
          ko.a = o.lut ? 1 : 0;  // JIT: table-driven phase (one weight class)
          ko.cbit = o.skip_udag ? 1 : 0;
          {
            std::set<uint32_t> rm;  // register-slot masks (the kernels' phase groups)
            for (auto& tm : o.terms) {
              uint32_t m = 0;
              for (int b = 0; b < P.n; ++b)
                if (tm.mask >> b & 1) {
                  const int sl = loc[b] >= 0 ? slot_of(b) : -1;
                  if (sl >= 0) m |= 1u << sl;
                }
              rm.insert(m);
            }
            o.ngroups = (int)rm.size();
          }
          for (size_t i = 0; i < o.terms.size(); ++i) {
            KTerm kt;
            std::memset(&kt, 0, sizeof(kt));
            kt.mask = o.terms[i].mask;
            kt.wofs = (int16_t)(mat - pass.mat_begin + (o.lut ? 0 : 2 * (int)i));
            kt.acc = o.terms[i].param >= 0 ? (int16_t)(stage_acc + o.terms[i].slot) : -1;
            kt.pad = o.lut && o.terms[i].w < 0 ? 1 : 0;  // LUT: sign of the term's weight
            P.kterms.push_back(kt);
          }
          // Cut table: a LUT op's odd-parity count c(r) depends only on the index r and the
          // op's (mask, sign) set -- theta- and row-independent -- so the JIT kernels read it
          // from a per-plan byte table (2^n entries, L2-resident for n <= 26) instead of a
          // popcount per term (QAOA: every cost layer shares one table)
          // Measured slower on cfg3 (424 -> 352 circuits/s: the byte reads follow the stage
          // mapping, so a warp's 32 lanes hit 32 L2 sectors per load), hence opt-in.
          static const bool cut_on = getenv("TCX_CUT_TABLE") != nullptr;
          if (o.lut && cut_on && P.gbits == 0 && P.nloc <= kMaxCutBits && o.terms.size() < 256) {
            std::vector<std::pair<uint64_t, int>> key;
            for (size_t i = 0; i < o.terms.size(); ++i)
              key.push_back({o.terms[i].mask, o.terms[i].w < 0 ? 1 : 0});
            std::sort(key.begin(), key.end());
            int id = -1;
            for (size_t c2 = 0; c2 < P.cut_sets.size(); ++c2)
              if (P.cut_sets[c2] == key) id = (int)c2;
            // at most 15 tables (4 bits in KOp::cbit) and 1 GB of them
            const size_t max_tabs = std::min<size_t>(15, ((size_t)1 << 30) >> P.nloc);
            if (id < 0 && P.cut_sets.size() < max_tabs) {
              id = (int)P.cut_sets.size();
              P.cut_sets.push_back(key);
            }
            if (id >= 0) ko.cbit |= (uint8_t)((id + 1) << 4);
          }
        }
        int na = op_accs(o);
        if (na > 0) {
          ko.acc = stage_acc;
          o.acc_off = pass.acc_begin + pass_acc + stage_acc;
          o.acc_len = na;
          stage_acc += na;
        }
        mat += o.mat_len;
        P.kops.push_back(ko);
      }
      ks.op_count = (int)P.kops.size() - pass.kop_begin - ks.op_begin;
      ks.acc_count = stage_acc;
      pass_acc += stage_acc;
      pass.max_stage_acc = std::max(pass.max_stage_acc, stage_acc);
      P.kstages.push_back(ks);
    }
    pass.stage_count = (int)P.kstages.size() - pass.stage_begin;
    if (pass.tan_hdr >= 0) {  // scan program: forward factors, backward walk (reverse order)
      const bool c128p = !g_packed_u1;
      auto flag_of = [&](const Op& o) { return o.mat_off + (c128p ? 10 : 30); };
      SPass sp{};
      sp.hdr = pass.mat_begin + pass.tan_hdr;
      sp.fbeg = (int)P.sfwd.size();
      for (int oi : pass_kops_ops)
        if (P.ops[oi].tan) P.sfwd.push_back(SFwd{P.ops[oi].tan_idx, flag_of(P.ops[oi])});
      sp.fcnt = (int)P.sfwd.size() - sp.fbeg;
      sp.bbeg = (int)P.sbwd.size();
      for (int k = (int)pass_kops_ops.size() - 1; k >= 0; --k) {
        const Op& o = P.ops[pass_kops_ops[k]];
        if (o.acc_off >= 0 && o.acc_len > 0 && o.pass >= 0) P.sbwd.push_back(SBwd{0, o.acc_off, o.acc_len, 0});
        if (o.tan && !o.skip_udag) P.sbwd.push_back(SBwd{1, o.tan_idx, flag_of(o), 0});
      }
      sp.bcnt = (int)P.sbwd.size() - sp.bbeg;
      P.spass.push_back(sp);
    }
    if (const char* dbg = getenv("TCX_PLAN_DEBUG"))
      if (dbg[0] == '2') {  // stage-level op listing: U1 q / X t.c / D(nterms)
        fprintf(stderr, "pass %d:", (int)(&pass - &P.passes[0]));
        for (auto& st : stages) {
          fprintf(stderr, " |");
          for (int oi : st.ops) {
            const Op& o = P.ops[oi];
            if (o.type == OP_U1) fprintf(stderr, " U%d", o.b0);
            else if (o.type == OP_CX) fprintf(stderr, " X%d.%d", o.b0, o.b1);
            else if (o.type == OP_DIAG) fprintf(stderr, " D%s%zu", o.lut ? "L" : "", o.terms.size());
            else fprintf(stderr, " F");
          }
        }
        fprintf(stderr, "\n");
      }
    {
      const KStage& ls = P.kstages.back();
      bool top = true;
      for (int k = 0; k < P.r; ++k) top &= ls.R[k] == P.h + k;
      for (int m = 0; m < P.h; ++m) top &= ls.T[m] == m;
      pass.last_is_top = top ? 1 : 0;
    }
    pass.kop_count = (int)P.kops.size() - pass.kop_begin;
    pass.kterm_count = (int)P.kterms.size() - pass.kterm_begin;
    pass.mat_count = mat - pass.mat_begin;
    pass.acc_count = pass_acc;
    acc += pass_acc;
  }
  P.mat_total = mat;
  P.acc_total = acc;

  // ---- materialize / finalize tables
  int contrib = 0;
  std::vector<int> contrib_param;
  for (auto& o : P.ops) {
    if (o.type == OP_U1) {
      MItem mi{};
      mi.type = OP_U1;
      mi.mat_off = o.mat_off;
      mi.cons_begin = (int)P.dcons.size();
      mi.cons_count = (int)o.cons.size();
      mi.param = -1;
      mi.tan = o.pass >= 0 ? o.tan : 0;
      mi.tan_idx = o.pass >= 0 ? o.tan_idx : -1;
      for (auto& cn : o.cons) {
        DCons d{};
        d.kind = cn.kind;
        d.param = cn.param;
        d.coeff = cn.coeff;
        d.payload = cn.payload;
        d.contrib = -1;
        if (cn.param >= 0 && is_rot(cn.kind)) {
          d.contrib = contrib++;
          contrib_param.push_back(cn.param);
        }
        P.dcons.push_back(d);
      }
      P.mitems.push_back(mi);
      if (o.has_param) {
        GItem gi{};
        gi.type = OP_U1;
        gi.acc = o.acc_off;
        gi.cls = u1_class_of(o.cons);
        gi.re_acc = g_q_grad ? o.acc_off + (gi.cls ? 1 : 3) : -1;
        gi.cons_begin = mi.cons_begin;
        gi.cons_count = mi.cons_count;
        gi.contrib = -1;
        gi.phase = o.tan == 3 ? 1 : 0;
        P.gitems.push_back(gi);
      }
    } else if (o.type == OP_U2F) {
      MItem mi{};
      mi.type = OP_U2F;
      mi.mat_off = o.mat_off;
      mi.payload = o.u2_payload;
      mi.param = -1;
      P.mitems.push_back(mi);
    } else if (o.type == OP_DIAG && o.lut) {
      // table entry c = exp(i W (T - 2c)) for c odd-signed terms, W = |w| of the class
      const int T = (int)o.terms.size();
      const double W = std::fabs(o.terms[0].w);
      for (int cnt = 0; cnt <= T; ++cnt) {
        MItem mi{};
        mi.type = OP_DIAG;
        mi.mat_off = o.mat_off + 2 * cnt;
        mi.param = o.terms[0].param;
        mi.w = W * (double)(T - 2 * cnt);
        mi.payload = -1;
        P.mitems.push_back(mi);
      }
    } else if (o.type == OP_DIAG) {
      for (size_t i = 0; i < o.terms.size(); ++i) {
        MItem mi{};
        mi.type = OP_DIAG;
        mi.mat_off = o.mat_off + 2 * (int)i;
        mi.param = o.terms[i].param;
        mi.w = o.terms[i].w;
        mi.payload = -1;
        if (mi.param <= -2) {  // derived phase of a kind-3 U1: recomputed from its constituents
          const Op& src = P.ops[-2 - mi.param];
          mi.cons_begin = (int)P.dcons.size();
          mi.cons_count = (int)src.cons.size();
          for (auto& cn : src.cons) {
            DCons d{};
            d.kind = cn.kind;
            d.param = cn.param;
            d.coeff = cn.coeff;
            d.payload = cn.payload;
            d.contrib = -1;
            P.dcons.push_back(d);
          }
          mi.tan = 4;
          mi.tan_idx = o.terms[i].mask ? 1 : 0;  // 0: global part gamma, 1: Z part w
        }
        P.mitems.push_back(mi);
      }
    }
    if (o.type == OP_DIAG) {
      // one finalize item per gradient slot
      std::vector<int> seen(o.nslots, 0);
      for (auto& tm : o.terms) {
        if (tm.param < 0 || seen[tm.slot]) continue;
        seen[tm.slot] = 1;
        GItem gi{};
        gi.type = OP_DIAG;
        gi.acc = o.acc_off + tm.slot;
        gi.re_acc = g_q_grad ? o.acc_off + o.nslots + tm.slot : -1;
        gi.factor = -2.0 * tm.w;
        gi.contrib = contrib++;
        contrib_param.push_back(tm.param);
        P.gitems.push_back(gi);
      }
    }
  }
  for (auto& dg : P.dgates)
    if (dg.param >= 0 && is_rot(dg.kind)) {
      dg.contrib = contrib++;
      contrib_param.push_back(dg.param);
    }
  P.n_contrib = contrib;
  P.param_ptr.assign(Pn + 1, 0);
  for (int p : contrib_param) P.param_ptr[p + 1]++;
  for (int p = 0; p < Pn; ++p) P.param_ptr[p + 1] += P.param_ptr[p];
  P.param_list.assign(contrib, 0);
  {
    std::vector<int> fill(P.param_ptr.begin(), P.param_ptr.end() - 1);
    for (int ci = 0; ci < contrib; ++ci) P.param_list[fill[contrib_param[ci]]++] = ci;
  }
  return TCX_OK;
}

// ---------------------------------------------------------------- binding
std::shared_ptr<Binding> bind(Plan& P, const Pauli& H) {
  auto B = std::make_shared<Binding>();
  B->hash = H.hash;
  const int n = P.n, t = P.t, c = P.c;
  // group terms by X/Y flip mask (physical bits through the final layout)
  std::map<uint64_t, std::vector<KPTerm>> groups;
  const int T = (int)H.weights.size();
  for (int j = 0; j < T; ++j) {
    uint64_t x = 0, zy = 0;
    int ny = 0;
    for (int q = 0; q < n; ++q) {
      int code = H.codes[(size_t)j * n + q];
      uint64_t bit = 1ull << P.layout[q];
      if (code == 1 || code == 2) x |= bit;
      if (code == 2 || code == 3) zy |= bit;
      if (code == 2) ny++;
    }
    // (P psi)_r = i^nY (-1)^popc((r ^ x) & zy) psi_{r ^ x}   (SURVEY §8 conventions)
    double re = 0, im = 0;
    switch (ny & 3) {
      case 0: re = 1; break;
      case 1: im = 1; break;
      case 2: re = -1; break;
      case 3: im = -1; break;
    }
    double s = (popc64(x & zy) & 1) ? -1.0 : 1.0;
    groups[x].push_back({zy, H.weights[j] * re * s, H.weights[j] * im * s});
  }
  // units: the last forward pass, then greedy windows for the remaining groups
  std::vector<std::pair<uint64_t, std::vector<KPTerm>>> left(groups.begin(), groups.end());
  // windows live in the local bits; sharded states keep their top g bits global
  const int nl = P.nloc;
  const uint64_t lfull = (nl >= 64) ? ~0ull : ((1ull << nl) - 1);
  const bool sharded = P.gbits > 0;
  bool gather_all = false;
  int swapped = 0;
  auto add_unit = [&](uint64_t W, int fwd_pass) {
    LamUnit u;
    u.wmask = W;
    u.swapped = swapped;
    int l = 0;
    int loc[64];
    for (int b = 0; b < nl; ++b)
      if (W >> b & 1) {
        loc[b] = l;
        u.W[l++] = b;
      }
    u.fwd_pass = fwd_pass;
    u.group_begin = (int)B->groups.size();
    std::vector<std::pair<uint64_t, std::vector<KPTerm>>> rest;
    for (auto& g : left) {
      const bool global = fwd_pass < 0 && gather_all;
      if (global || (g.first & ~W) == 0) {
        KGroup kg{};
        uint32_t xl = 0;
        if (!global)
          for (int b = 0; b < nl; ++b)
            if (g.first >> b & 1) xl |= 1u << loc[b];
        kg.xlocal = xl;
        kg.xphys = g.first;
        kg.global = global ? 1 : 0;
        kg.term_begin = (int)B->pterms.size();
        kg.term_count = (int)g.second.size();
        B->pterms.insert(B->pterms.end(), g.second.begin(), g.second.end());
        B->groups.push_back(kg);
      } else {
        rest.push_back(g);
      }
    }
    u.group_count = (int)B->groups.size() - u.group_begin;
    left.swap(rest);
    B->units.push_back(u);
  };
  // lambda-unit windows use the default run width (64-byte runs) whatever the passes use: the
  // units read psi and read-modify-write lambda in blocked tile order, where 32-byte runs waste
  // DRAM bursts (cfg5: 238 -> 139 ms of lambda units), and 128-byte runs leave fewer free
  // window bits (cfg2: two units instead of one)
  const int cl = (P.gbits == 0 && !getenv("TCX_LAM_SAME_C")) ? (P.dtype == TCX_C128 ? 2 : 3) : c;
  auto greedy_units = [&]() {
    while (!left.empty()) {
      uint64_t W = (1ull << std::min(cl, t)) - 1;
      bool grew = true;  // admit groups in order of fewest extra bits
      while (grew) {
        grew = false;
        int best = -1, bestc = 1 << 30;
        for (size_t i = 0; i < left.size(); ++i) {
          uint64_t nw = W | left[i].first;
          int cnt = popc64(nw);
          if ((left[i].first & ~W) == 0 || cnt > t || (left[i].first & ~lfull)) continue;
          if (cnt < bestc) {
            bestc = cnt;
            best = (int)i;
          }
        }
        if (best >= 0) {
          W |= left[best].first;
          grew = true;
        }
      }
      for (int b = 0; b < nl && popc64(W) < t; ++b) W |= 1ull << b;
      size_t before = left.size();
      add_unit(W, -1);
      if (left.size() == before) {
        B->units.pop_back();
        if (sharded) return;  // partners on another rank: handled after an exchange
        // flip masks wider than a window: one more unit gathers partners from HBM
        gather_all = true;
        add_unit(W, -1);
      }
    }
  };
  if (!sharded) {
    const PassInfo& last = P.passes.back();
    add_unit(nl <= t ? lfull : last.wmask, (int)P.passes.size() - 1);
    greedy_units();
  } else {
    // groups flipping a global qubit run after the global <-> top-local exchange
    std::vector<std::pair<uint64_t, std::vector<KPTerm>>> glob, loc0;
    for (auto& g : left) ((g.first & ~lfull) ? glob : loc0).push_back(g);
    left = loc0;
    greedy_units();
    if (!left.empty()) {
      B->xmask_ok = false;
      B->err = "sharded: a Pauli flip mask does not fit one local window";
      return B;
    }
    if (!glob.empty()) {
      int perm[64];
      shard_swap_perm(n, P.gbits, perm);
      for (auto& g : glob) {
        g.first = remap_mask(g.first, perm, n);
        for (auto& pt : g.second) pt.zy = remap_mask(pt.zy, perm, n);
      }
      left = glob;
      swapped = 1;
      greedy_units();
      if (!left.empty()) {
        B->xmask_ok = false;
        B->err = "sharded: a Pauli term flips qubits that are global in both layouts";
        return B;
      }
    }
  }
  return B;
}

// The fixed step list of a sharded program (identical on every rank): materialise, forward
// passes with an EXCHANGE between segments, lambda units (those flipping global qubits run
// after an exchange), backward passes mirrored, finalise.
std::vector<tcx_shard_step> shard_program(const Plan& P, const Binding& Bdr, bool want_grad) {
  const Binding* Bd = &Bdr;
  std::vector<tcx_shard_step> v;
  auto add = [&](int k, int a) { v.push_back({k, a}); };
  const int nP = (int)P.passes.size();
  add(TCX_STEP_MATERIALIZE, 0);
  for (int p = 0; p < nP; ++p) {
    if (p > 0 && P.passes[p].seg != P.passes[p - 1].seg) add(TCX_STEP_EXCHANGE, 1);
    add(TCX_STEP_FWD, p);
  }
  const int x = want_grad ? 3 : 1;  // exchange psi (+ lambda once it exists)
  bool any_lam = false;
  for (int u = 0; u < (int)Bd->units.size(); ++u)
    if (!Bd->units[u].swapped) {
      add(TCX_STEP_LAMBDA, u);
      any_lam = true;
    }
  bool sw = false;
  for (int u = 0; u < (int)Bd->units.size(); ++u)
    if (Bd->units[u].swapped) {
      if (!sw) add(TCX_STEP_EXCHANGE, any_lam ? x : 1);
      sw = true;
      add(TCX_STEP_LAMBDA, u);
    }
  if (sw && want_grad) add(TCX_STEP_EXCHANGE, x);  // back to the backward's layout
  if (want_grad)
    for (int p = nP - 1; p >= 0; --p) {
      add(TCX_STEP_BWD, p);
      if (p > 0 && P.passes[p].seg != P.passes[p - 1].seg) add(TCX_STEP_EXCHANGE, 3);
    }
  add(TCX_STEP_FINALIZE, 0);
  return v;
}

}  // namespace tcx
