/*
 * tcx.h -- C ABI of the B200-native batched <H> + grad engine (libtcx.so).
 *
 * The operation (arXiv 2205.10091, TensorCircuit):
 *   psi_b = U_L(theta_b) ... U_1(theta_b) |0...0>          PAPER.md:391 (§3.3 default
 *           input), :268-280 (§3.2 circuit + state()), north_star "contracting the
 *           circuit's gate tensors into the 2^n-amplitude state tensor".
 *   E_b   = Re sum_j alpha_j <psi_b|P_j|psi_b>              PAPER.md:79-91 (Eq. 1-2),
 *           Pauli structures PAPER.md:794-815 (§6.2.1).
 *   grad_b = dE_b/dtheta_b (per row)                        PAPER.md:487-492 (§4
 *           value_and_grad), batched with argnums = vectorized_argnums = 0 as in the
 *           batched-VQE example PAPER.md:1121-1139 (§6.3.5); obtained by an adjoint
 *           reverse sweep (north_star step 4).
 *
 * Conventions (SURVEY.md §8 conventions):
 *   - qubit 0 is the most significant bit of the amplitude index:
 *     r = sum_q b_q 2^(n-1-q).
 *   - rotations R_P(a) = exp(-i a P / 2), P in {X,Y,Z,XX,YY,ZZ}; a = coeff*theta[param]
 *     when param >= 0, a = coeff when param == -1 (fixed angle).  PAPER.md:362's
 *     exp1(theta, G) = e^{+i theta G} is R_GG with coeff = -2.
 *   - two-qubit matrices on (q0, q1) use row/column index 2*b_q0 + b_q1
 *     (PAPER.md:368-374); CNOT control = q0, target = q1.
 *   - Pauli codes 0=I 1=X 2=Y 3=Z per qubit in paper order; weights real
 *     ("alpha_j are real coefficients").
 *   - complex amplitudes are interleaved (re, im): float2 for TCX_C64, double2 for
 *     TCX_C128 (complex64 default / complex128).
 *   - theta, E and grad are float64 for both dtypes.
 *
 * Ownership: the caller owns every buffer (theta, E, grad, state, workspace); the
 * library owns the opaque handles.  Handles are immutable after build and may be
 * shared across threads and streams.  All device work is enqueued on the caller's
 * CUDA stream (cudaStream_t passed as void*; NULL = legacy default stream); no call
 * synchronizes the device except the *_host variants, which synchronize the stream
 * before returning.
 *
 * Errors: every entry returns a tcx_status; the library never aborts.  On failure
 * tcx_last_error() (thread-local) names the offending argument / gate / term index.
 * There is no CPU fallback: every compute step runs in the library's sm_100a kernels;
 * without a usable CUDA device the compute entries return TCX_E_CUDA.
 */
#ifndef TCX_ABI_H_
#define TCX_ABI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TCX_OK = 0,
    TCX_E_INVALID = 1,      /* bad argument, gate, term, size, or workspace too small */
    TCX_E_UNSUPPORTED = 2,  /* valid input outside this build's scope (e.g. grad of a
                               non-unitary payload, C11 in DESIGN.md) */
    TCX_E_OOM = 3,          /* host allocation failed */
    TCX_E_CUDA = 4,         /* CUDA runtime error / no device */
    TCX_E_NCCL = 5
} tcx_status;

typedef enum { TCX_C64 = 0, TCX_C128 = 1 } tcx_dtype;

typedef enum {
    /* fixed 1-qubit */
    TCX_I = 0, TCX_X, TCX_Y, TCX_Z, TCX_H, TCX_S, TCX_SDG, TCX_T, TCX_TDG,
    /* fixed 2-qubit */
    TCX_CNOT, TCX_CZ, TCX_SWAP,
    /* rotations R_P(coeff*theta[param]) */
    TCX_RX, TCX_RY, TCX_RZ, TCX_RXX, TCX_RYY, TCX_RZZ,
    /* fixed payload matrices (PAPER.md:355-360 c.unitary): 2x2 / 4x4 */
    TCX_U1, TCX_U2,
    /* Monte Carlo trajectory of a depolarizing channel (PAPER.md:652-700 unitary_kraus with an
     * external `status`): 1 qubit, param = the theta column holding the row's
     * status x in [0, 1), payload = 2 complex elements (px + i py, pz + 0i).  [0, 1) is split
     * in the paper's Kraus order I, X, Y, Z: x < 1-px-py-pz -> I, < 1-py-pz -> X, < 1-pz -> Y,
     * else Z.  Not differentiable: its status column gets no gradient contribution. */
    TCX_DEPOL,
    /* Random-axis rotation (Table VII "vmap over circuit structures":
     * unitary_kraus over [Rx, Ry, Rz] with probabilities 1/3 and an external status): 1 qubit,
     * angle = coeff * theta[param] as for rotations, payload = 1 complex element whose real
     * part is the index s of the theta column holding the row's status x in [0, 1);
     * x < 1/3 -> R_X, x < 2/3 -> R_Y, else R_Z.  Differentiable in the angle. */
    TCX_RROT,
    TCX_NKINDS
} tcx_gate_kind;

/* One gate of the input list (32 bytes).
 *   kind    tcx_gate_kind
 *   q0, q1  qubits (q1 = -1 for 1-qubit gates); distinct, in [0, n)
 *   param   theta column for rotations, -1 = fixed angle (then coeff is the angle);
 *           must be -1 for non-rotation kinds
 *   coeff   angle multiplier (rotations); ignored otherwise
 *   payload offset in complex elements into `matrices` for TCX_U1 (4) / TCX_U2 (16),
 *           -1 otherwise */
typedef struct {
    int32_t kind, q0, q1, param;
    double coeff;
    int64_t payload;
} tcx_gate;

/* Build options; zero-initialised = defaults chosen per dtype and n. */
typedef struct {
    int32_t tile_bits;      /* t: amplitudes per tile = 2^t (default 12 c64 / 11 c128; n if n<t) */
    int32_t reg_bits;       /* r: amplitudes per thread per stage = 2^r (default 4, 3 if n<=t) */
    int32_t coalesce_bits;  /* c: low index bits present in every tile (default: 64 B runs) */
    int32_t max_ops_per_pass; /* fusion depth cap: 0 = light-cone (unlimited), 1 = unfused */
    int32_t jit;            /* 0 = per-circuit specialised kernels (NVRTC, sm_100a) when
                               available, -1 = the precompiled generic kernels */
    int32_t global_bits;    /* g > 0: the state is sharded over 2^g ranks on its top g index
                               bits (qubits 0..g-1); run with tcx_shard_* (north_star
                               "shards on its top log2(G) global qubits") */
    int32_t dense_k;        /* k in [1, 5]: fuse the gate list greedily into dense k-qubit
                               blocks (2-qubit gates make at least 2-qubit blocks) and apply
                               each as one 2^k x 2^k complex contraction over the state
                               (north_star step 2); 0 = window passes only.
                               Not with global_bits; grad needs k <= 4. */
    int32_t q_grad;         /* 1: window plans also accumulate the real parts of the R' Pauli
                               components, so tcx_grad_batch_q works on them (per-circuit
                               kernels only); 0 = off (dense plans always support it) */
    int32_t l2_rows;        /* L2-resident row groups: > 0 runs all passes for
                               groups of this many theta rows in turn, so a group's psi and
                               lambda stay in L2 between passes; -1 = auto (groups whose psi +
                               lambda fit ~96 MB); 0 = off (every pass over all rows) */
    int32_t cluster_bits;   /* cluster-resident states: g_c in [1, 4] runs each
                               theta row on one thread-block cluster of 2^g_c CTAs (one per SM)
                               whose REGISTERS hold the whole psi and lambda (2^(n-g_c)
                               amplitudes per CTA, at most 2^13 complex64 / 2^12 complex128);
                               gates on the top g_c qubits trade places through distributed
                               shared memory, so HBM carries only theta in and E / grad out;
                               one launch per batch.  tcx_expect_batch / tcx_grad_batch only;
                               0 = off */
} tcx_build_opts;

/* Executed-plan summary (for reports and tests). */
typedef struct {
    int32_t n_qubits, n_params, dtype;
    int32_t tile_bits, reg_bits, coalesce_bits, threads_per_tile;
    int32_t n_ops;            /* fused kernel ops after lowering */
    int32_t fwd_passes;       /* F: forward window passes */
    int32_t lambda_passes;    /* extra passes to complete lambda = H psi (excl. the last fwd) */
    int32_t bwd_passes;       /* R */
    int32_t stages;           /* register stages summed over forward passes */
    int32_t unitary;          /* 1 if every payload is unitary (grad allowed) */
    int32_t relabeled;        /* 1 if SWAP gates were applied as qubit relabels */
    int32_t jit;              /* 1 if the passes run per-circuit specialised kernels */
    int32_t global_bits;      /* sharded: g (2^g ranks), else 0 */
    int32_t segments;         /* sharded: forward segments (exchanges = segments - 1) */
    int64_t tiles_per_state;  /* 2^(n-t) */
    int64_t acc_slots;        /* gradient partial slots per tile */
    int64_t mat_reals;        /* per-theta materialised matrix entries */
    int32_t dense_k;          /* dense block size cap (0: no dense blocks) */
    int32_t dense_blocks;     /* dense k-qubit block passes (each one read+write of psi) */
    int32_t init_h;           /* leading H gates folded into the initial |+> state */
    int32_t cluster_bits;     /* cluster-resident plan: CTAs per theta row = 2^cluster_bits */
    int32_t exchange_overlaps; /* sharded: exchanges whose next pass (forward or backward) runs
                                  chunk by chunk as the exchange lands (overlap) */
    int32_t tma_passes;       /* window passes whose tiles move by TMA (one box per tile) */
    int32_t tma_multibox_passes; /* ... by TMA in 2^k boxes per tile (windows of > 5 runs) */
} tcx_plan_info;

typedef struct tcx_circuit tcx_circuit;
typedef struct tcx_pauli tcx_pauli;

/* Compile a gate list into an executable plan (host only; the analog of K.jit,
 * PAPER.md:492-496; excluded from timings as the paper excludes JIT).
 * matrices: n_matrix_elems complex numbers as interleaved (re, im) float64, row-major,
 * index order of the conventions above.  TCX_E_INVALID names the first bad gate. */
tcx_status tcx_circuit_build(int32_t n_qubits, int32_t n_params,
                             const tcx_gate* gates, int64_t n_gates,
                             const double* matrices, int64_t n_matrix_elems,
                             tcx_dtype dtype, const tcx_build_opts* opts,
                             tcx_circuit** out);

/* Pauli sum H = sum_j weights[j] P_j.  codes: [n_terms][n_qubits]
 * uint8 in {0,1,2,3}, paper qubit order.  The identity string is allowed. */
tcx_status tcx_pauli_build(int32_t n_qubits, int32_t n_terms, const uint8_t* codes,
                           const double* weights, tcx_pauli** out);

enum { TCX_WS_GRAD = 1, TCX_WS_HOST_IO = 2, TCX_WS_STATE = 4, TCX_WS_INPUTS = 8,
       TCX_WS_TERMS = 16 };

/* Device workspace bytes for a batch of B rows.  mode: TCX_WS_GRAD for tcx_grad_batch
 * (psi and lambda), 0 for tcx_expect_batch, TCX_WS_STATE for tcx_state_batch; OR
 * TCX_WS_HOST_IO for the *_host entries (adds device room for theta/E/grad), and
 * TCX_WS_INPUTS for the *_in entries (input states); TCX_WS_TERMS (| TCX_WS_INPUTS) for
 * tcx_expect_terms_batch. */
tcx_status tcx_workspace_bytes(const tcx_circuit* circ, const tcx_pauli* pauli, int64_t B,
                               int32_t mode, size_t* bytes);

/* E[b] = Re sum_j alpha_j <psi(theta_b)|P_j|psi(theta_b)> for b < B.
 * theta: device [B][n_params] float64 row-major; E: device [B] float64;
 * ws: device workspace of >= tcx_workspace_bytes(..., 0) bytes. */
tcx_status tcx_expect_batch(const tcx_circuit* circ, const tcx_pauli* pauli,
                            const double* theta, int64_t B, double* E,
                            void* ws, size_t ws_bytes, void* cuda_stream);

/* E as above and grad[b][p] = dE_b/dtheta_{b,p} (per row).
 * grad: device [B][n_params] float64.  TCX_E_UNSUPPORTED if a payload is not unitary
 * (the adjoint sweep applies U^dagger). */
tcx_status tcx_grad_batch(const tcx_circuit* circ, const tcx_pauli* pauli,
                          const double* theta, int64_t B, double* E, double* grad,
                          void* ws, size_t ws_bytes, void* cuda_stream);

/* psi(theta_b) for b < B into state: device [B][2^n] complex (dtype of the circuit),
 * paper index order (qubit 0 most significant), for parity tests. */
tcx_status tcx_state_batch(const tcx_circuit* circ, const double* theta, int64_t B,
                           void* state, void* ws, size_t ws_bytes, void* cuda_stream);

/* Batched input states (`inputs` vmapped together with the weights,
 * SURVEY §8f f2).  As tcx_expect_batch / tcx_grad_batch / tcx_state_batch, but row b
 * starts from psi0[b] instead of |0...0>.  psi0: device [B][2^n] complex in the circuit
 * dtype (complex64 / complex128, interleaved re, im), paper index order (qubit 0 most
 * significant); read only, caller-owned; need not be normalised (E is then
 * <psi|H|psi> of the unnormalised state).  ws sized with TCX_WS_INPUTS (| TCX_WS_GRAD /
 * TCX_WS_STATE).  TCX_E_INVALID on a null psi0, TCX_E_UNSUPPORTED for sharded circuits. */
tcx_status tcx_expect_batch_in(const tcx_circuit* circ, const tcx_pauli* pauli,
                               const double* theta, int64_t B, const void* psi0, double* E,
                               void* ws, size_t ws_bytes, void* cuda_stream);
tcx_status tcx_grad_batch_in(const tcx_circuit* circ, const tcx_pauli* pauli,
                             const double* theta, int64_t B, const void* psi0, double* E,
                             double* grad, void* ws, size_t ws_bytes, void* cuda_stream);
tcx_status tcx_state_batch_in(const tcx_circuit* circ, const double* theta, int64_t B,
                              const void* psi0, void* state, void* ws, size_t ws_bytes,
                              void* cuda_stream);

/* <psi|H|d psi/d theta>: its real part is grad / 2, its
 * imaginary part is written to q_im[b][p] (device [B][n_params] float64); E and grad as in
 * tcx_grad_batch.  Needs the real parts of R' = sum psi lambda^dagger: dense plans
 * (dense_k in 1..4, full 2^k x 2^k R') or window plans built with q_grad = 1 (three more
 * Pauli components per fused op, per-circuit kernels); else TCX_E_UNSUPPORTED.  ws sized
 * with TCX_WS_GRAD. */
tcx_status tcx_grad_batch_q(const tcx_circuit* circ, const tcx_pauli* pauli,
                            const double* theta, int64_t B, double* E, double* grad,
                            double* q_im, void* ws, size_t ws_bytes, void* cuda_stream);

/* Per-term values (vvag over Pauli structures returns
 * f(w, v_j) for every term next to the summed gradient, which is tcx_grad_batch with unit
 * weights): E_terms[b][j] = Re <psi_b|P_j|psi_b> (weights ignored), device [B][n_terms]
 * float64.  psi0: NULL (|0...0>) or device input states as for the _in entries.  ws sized
 * with TCX_WS_TERMS (| TCX_WS_INPUTS).  Fixed-order fp64 reductions. */
tcx_status tcx_expect_terms_batch(const tcx_circuit* circ, const tcx_pauli* pauli,
                                  const double* theta, int64_t B, const void* psi0,
                                  double* E_terms, void* ws, size_t ws_bytes,
                                  void* cuda_stream);

/* End-to-end variants: theta/E/grad are HOST pointers (pinned memory recommended);
 * the call copies theta host->device, runs the same kernels, copies E/grad back and
 * synchronizes the stream.  ws must be sized with TCX_WS_HOST_IO. */
tcx_status tcx_expect_batch_host(const tcx_circuit* circ, const tcx_pauli* pauli,
                                 const double* theta_host, int64_t B, double* E_host,
                                 void* ws, size_t ws_bytes, void* cuda_stream);
tcx_status tcx_grad_batch_host(const tcx_circuit* circ, const tcx_pauli* pauli,
                               const double* theta_host, int64_t B, double* E_host,
                               double* grad_host, void* ws, size_t ws_bytes,
                               void* cuda_stream);

/* Ahead-of-time specialisation: generate and compile (NVRTC, host only) the per-circuit
 * kernels a call of `kind` (0 expect, 1 grad, 2 state) needs for B rows; otherwise this
 * happens on the first compute call.  No-op when the plan runs the generic kernels. */
tcx_status tcx_circuit_jit(const tcx_circuit* circ, const tcx_pauli* pauli, int64_t B,
                           int32_t kind);

/* Plan summary. */
tcx_status tcx_circuit_info(const tcx_circuit* circ, const tcx_pauli* pauli,
                            tcx_plan_info* out);

/* Decoded, validated gate table exactly as the plan stores it (bit-exact round trip
 * of the input list; parse parity test).  Writes min(cap, n_gates) gates. */
tcx_status tcx_circuit_decode(const tcx_circuit* circ, tcx_gate* out, int64_t cap,
                              int64_t* n_gates);

/* Physical index bit of each qubit at the end of the circuit (after SWAP relabels);
 * out: [n_qubits].  Identity layout is bit = n-1-q. */
tcx_status tcx_circuit_layout(const tcx_circuit* circ, int32_t* out);

/* Kernel launches one tcx_grad_batch / tcx_expect_batch call enqueues for B rows. */
tcx_status tcx_launch_count(const tcx_circuit* circ, const tcx_pauli* pauli, int64_t B,
                            int32_t want_grad, int32_t* launches);

/* ---- Sharded single state (circuit built with tcx_build_opts.global_bits = g > 0) ----
 * north_star: "A single large state shards on its top log2(G) global qubits, and gates on
 * global qubits are handled by NCCL all-to-all qubit swaps."  Rank r (of G = 2^g) holds the
 * 2^(n-g) amplitudes whose top g index bits equal r.  Diagonal phases and CNOT controls on
 * global qubits are rank-dependent constants; a gate that needs a global qubit inside a
 * window is preceded by an EXCHANGE of the g global bits with the top g local bits: every
 * rank sends chunk k (the 2^(n-2g) amplitudes whose top local bits equal k, contiguous,
 * per theta row) to rank k and receives chunk r from it -- an all-to-all the CALLER runs
 * (NCCL via torch.distributed, or device copies between virtual ranks).
 * The program is a fixed list of steps identical on all ranks; tcx_shard_exec enqueues
 * one non-exchange step for one rank on the caller's stream; FINALIZE writes this rank's
 * partial E[B] and grad[B][P], which the caller all-reduces (sum) over ranks. */
enum { TCX_STEP_MATERIALIZE = 0, TCX_STEP_FWD = 1, TCX_STEP_LAMBDA = 2, TCX_STEP_BWD = 3,
       TCX_STEP_FINALIZE = 4, TCX_STEP_EXCHANGE = 5 /* arg: 1 = psi, 3 = psi and lambda */ };
typedef struct { int32_t kind, arg; } tcx_shard_step;
tcx_status tcx_shard_program(const tcx_circuit* circ, const tcx_pauli* pauli, int32_t want_grad,
                             tcx_shard_step* steps, int32_t cap, int32_t* n_steps);
tcx_status tcx_shard_exec(const tcx_circuit* circ, const tcx_pauli* pauli, int32_t rank,
                          int32_t want_grad, const tcx_shard_step* step, const double* theta,
                          int64_t B, double* E_partial, double* grad_partial, void* ws,
                          size_t ws_bytes, void* cuda_stream);
/* Device pointers of this rank's psi / lambda ([B][2^(n-g)] complex) inside ws, for the
 * caller's exchanges; local_amps = 2^(n-g). */
tcx_status tcx_shard_buffers(const tcx_circuit* circ, const tcx_pauli* pauli, int64_t B,
                             int32_t want_grad, void* ws, void** psi, void** lambda,
                             int64_t* local_amps);

/* ---- Library-owned communicator for the sharded state (north_star "gates on
 * global qubits are handled by NCCL all-to-all qubit swaps over NVLink"; PAPER.md:1788 outlook,
 * "distributed quantum circuit simulation").  tcx_grad_sharded runs the whole program of
 * tcx_shard_program for this process's rank(s): every compute step in the library's kernels,
 * every EXCHANGE in the library's transport on its own streams (ordered after / before the
 * caller's stream with events), then the sum of E / grad over ranks, so E and grad come back
 * complete (identical on every rank).
 *   TCX_COMM_NCCL     one process per GPU; tcx_comm_init bootstraps an NCCL communicator from
 *                     an ncclUniqueId (NCCL_UNIQUE_ID_BYTES = 128 bytes, made by
 *                     tcx_comm_unique_id on one rank and broadcast by the caller, e.g. with
 *                     torch.distributed).  libnccl.so.2 is resolved at run time (the copy
 *                     already loaded in the process first).  The exchange: XOR-pairwise steps,
 *                     grouped ncclSend straight from the contiguous [B][G][C] blocks (no pack
 *                     kernel) and ncclRecv into two staging chunks (TCX_XCHG_CHUNK_MB, default
 *                     256 MiB each, inside ws) copied into place on a second stream while the
 *                     next chunk is on the wire; E/grad: ncclAllReduce(sum).
 *   TCX_COMM_VIRTUAL  all 2^g ranks in this process on the current device (one-GPU runs and
 *                     parity tests): ws holds every rank's workspace; the exchange is an
 *                     in-place swap kernel (no staging); E/grad: fixed-order sum over ranks.
 *   TCX_COMM_HOST     tests with several processes on one device: each exchange goes block ->
 *                     pinned host -> fn -> block synchronously; fn(user, peer, send, recv,
 *                     bytes) must send `bytes` host bytes to rank `peer` and receive as many
 *                     from it (return 0 on success); E/grad: recursive doubling through fn.
 * A comm is bound to the device current at init; it must not be used by two calls at once.
 * Errors: TCX_E_INVALID (world not a power of two in [1, 64], rank out of range, world !=
 * 2^global_bits of the circuit, workspace too small), TCX_E_NCCL (library missing, NCCL or
 * callback failure). */
typedef struct tcx_comm tcx_comm;
enum { TCX_COMM_VIRTUAL = 0, TCX_COMM_NCCL = 1, TCX_COMM_HOST = 2 };
typedef int32_t (*tcx_host_exchange_fn)(void* user, int32_t peer, const void* send_host,
                                        void* recv_host, size_t bytes);
tcx_status tcx_comm_unique_id(void* nccl_unique_id_out /* 128 bytes */);
tcx_status tcx_comm_init(const void* nccl_unique_id, int32_t world, int32_t rank, tcx_comm** out);
tcx_status tcx_comm_init_virtual(int32_t world, tcx_comm** out);
tcx_status tcx_comm_init_host(int32_t world, int32_t rank, tcx_host_exchange_fn fn, void* user,
                              tcx_comm** out);
tcx_status tcx_comm_info(const tcx_comm* comm, int32_t* kind, int32_t* world, int32_t* rank);
void tcx_comm_free(tcx_comm* comm);
/* Device workspace for one tcx_grad_sharded (want_grad = 1) / tcx_expect_sharded call with
 * this comm: per local rank the psi (+ lambda) [B][2^(n-g)] complex buffers and partials,
 * plus the staging chunks (NCCL).  A circuit with global_bits = 0 and a world of 1 is the
 * ordinary single-GPU program (then the all-reduce is a no-op). */
tcx_status tcx_sharded_workspace_bytes(const tcx_circuit* circ, const tcx_pauli* pauli,
                                       const tcx_comm* comm, int64_t B, int32_t want_grad,
                                       size_t* bytes);
/* E[b] and grad[b][p] of the full (2^n-amplitude) state for theta rows b < B; theta: device
 * [B][n_params] float64, identical on every rank; E: device [B], grad: device [B][n_params]
 * float64, complete on return (summed over ranks).  Enqueued on cuda_stream except the host
 * transport, which synchronizes it. */
tcx_status tcx_grad_sharded(const tcx_circuit* circ, const tcx_pauli* pauli, tcx_comm* comm,
                            const double* theta, int64_t B, double* E, double* grad, void* ws,
                            size_t ws_bytes, void* cuda_stream);
tcx_status tcx_expect_sharded(const tcx_circuit* circ, const tcx_pauli* pauli, tcx_comm* comm,
                              const double* theta, int64_t B, double* E, void* ws,
                              size_t ws_bytes, void* cuda_stream);

/* Per-launch device timing (bench.py roofline).  When enabled on the calling thread,
 * every kernel a compute entry enqueues is bracketed by CUDA events recorded on the
 * call's stream.  tcx_profile_read waits for the recorded events, returns up to cap
 * entries (oldest first) and clears the log.  flops / bytes are the launch's
 * ALGORITHMIC floating-point operations and HBM bytes. */
typedef struct {
    int32_t phase;   /* 0 materialize, 1 forward pass, 2 lambda pass, 3 backward pass,
                        4 finalize, 5 fused single pass (forward + lambda + backward),
                        6 dense block, 7 dense block backward, 8 sharded-state exchange
                        (bytes = data that changes rank; virtual ranks: HBM read + write),
                        9 last forward pass fused with lambda and its backward,
                        10 cluster-resident megakernel (whole program; bytes = HBM in/out) */
    int32_t index;   /* pass / lambda-unit index */
    float ms;
    float pad;
    double flops;
    double bytes;
} tcx_kernel_time;
tcx_status tcx_profile_enable(int32_t on);
tcx_status tcx_profile_read(tcx_kernel_time* out, int32_t cap, int32_t* n);

void tcx_circuit_free(tcx_circuit* circ);
void tcx_pauli_free(tcx_pauli* pauli);

/* Thread-local message for the last failing call on this thread ("" if none). */
const char* tcx_last_error(void);

/* Library version string. */
const char* tcx_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TCX_ABI_H_ */
