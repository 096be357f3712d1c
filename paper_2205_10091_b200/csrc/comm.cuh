// comm.cuh -- the sharded single state's communicator and exchange.
//
// Included once, at the end of tcx.cu (it drives run() one program step at a time).
//
// north_star: "A single large state shards on its top log2(G) global qubits, and gates on
// global qubits are handled by NCCL all-to-all qubit swaps over NVLink" (outlook
// PAPER.md:1788, "distributed quantum circuit simulation").  Rank r of G = 2^g holds the
// amplitudes whose top g index bits equal r, as [B][G][C] (C = 2^(n-2g)): block k of a row
// is the contiguous run whose top g LOCAL bits equal k.  An EXCHANGE swaps the g global bits
// with the top g local bits, i.e. rank r's block k <-> rank k's block r for every r != k.
// The library owns that data movement on its own streams:
//
//   * NCCL (one process per GPU): XOR-pairwise steps s = 1..G-1, peer = rank ^ s; grouped
//     ncclSend of block `peer` straight from the state (no pack kernel: one send per row,
//     each contiguous) and ncclRecv into a double-buffered staging area, which a second
//     stream copies into block `peer` while the next chunk is on the wire.
//   * virtual (G ranks in this process on one device; parity tests / one-GPU runs): one
//     in-place swap kernel per XOR step over the G/2 rank pairs, 16-byte vectors, no
//     staging (the data never leaves HBM).
//   * host (tests: several processes sharing one GPU): block -> pinned host -> caller's
//     callback (e.g. a gloo send/recv) -> block, synchronously.
//
// E and grad partials are summed over ranks: ncclAllReduce (NCCL), a fixed-order sum kernel
// over the virtual ranks, or recursive doubling through the callback (host).
#include <dlfcn.h>
#include <nccl.h>  // types only: the functions are resolved with dlsym at tcx_comm_init

namespace {

constexpr int kXChunksMax = 8;  // column chunks of an exchange overlapped with the next pass

// ---- NCCL entry points (torch's libnccl when already loaded in the process, else the system one)
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*getUniqueId)(ncclUniqueId*);
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*commDestroy)(ncclComm_t);
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*groupStart)();
  ncclResult_t (*groupEnd)();
  const char* (*errorString)(ncclResult_t);
};
NcclApi& nccl() {
  static NcclApi A;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD))) break;  // the copy torch already loaded
    if (!h)
      for (const char* nm : names)
        if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      A.err = "libnccl.so.2 not found";
      return;
    }
    bool ok = true;
    auto sym = [&](const char* nm, void** fp) {
      *fp = dlsym(h, nm);
      ok = ok && *fp;
    };
    sym("ncclGetUniqueId", (void**)&A.getUniqueId);
    sym("ncclCommInitRank", (void**)&A.commInitRank);
    sym("ncclCommDestroy", (void**)&A.commDestroy);
    sym("ncclSend", (void**)&A.send);
    sym("ncclRecv", (void**)&A.recv);
    sym("ncclAllReduce", (void**)&A.allReduce);
    sym("ncclGroupStart", (void**)&A.groupStart);
    sym("ncclGroupEnd", (void**)&A.groupEnd);
    sym("ncclGetErrorString", (void**)&A.errorString);
    A.ok = ok;
    if (!ok) A.err = "libnccl.so.2 lacks a required symbol";
  });
  return A;
}

#define NCCL_TRY(x)                                                                        \
  do {                                                                                     \
    ncclResult_t r_ = (x);                                                                 \
    if (r_ != ncclSuccess)                                                                 \
      return fail(TCX_E_NCCL, std::string(#x) + ": " + nccl().errorString(r_));            \
  } while (0)

// ---- virtual ranks: rank r's block k <-> rank k's block r for the G/2 pairs of XOR step s,
// restricted to the byte columns [col_off, col_off + col_bytes) of each block (a chunk)
struct SwapArgs {
  char* base[64];  // each rank's psi (or lambda) buffer, [B][G][C] amplitudes
  int64_t row_bytes;    // N * amplitude bytes
  int64_t block_bytes;  // C * amplitude bytes
  int64_t col_off, col_bytes;  // chunk of each block (multiples of 16)
  int64_t B;
  int s;      // XOR step
  int hbit;   // highest set bit of s
};
__global__ void virtual_swap_kernel(const SwapArgs a) {
  const int64_t vecs = a.col_bytes >> 4;
  const int64_t per_pair = vecs * a.B;
  const int pair = blockIdx.y;
  // the pair's lower rank: insert a zero at bit hbit of the pair index
  const int lo = pair & ((1 << a.hbit) - 1);
  const int r = ((pair >> a.hbit) << (a.hbit + 1)) | lo;
  const int k = r ^ a.s;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < per_pair;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = u / vecs, v = u - b * vecs;
    uint4* x = reinterpret_cast<uint4*>(a.base[r] + b * a.row_bytes + k * a.block_bytes + a.col_off) + v;
    uint4* y = reinterpret_cast<uint4*>(a.base[k] + b * a.row_bytes + r * a.block_bytes + a.col_off) + v;
    const uint4 tx = *x, ty = *y;
    *x = ty;
    *y = tx;
  }
}

// fixed-order sum of the per-rank partials (virtual ranks): out[i] = sum_r part[r][i]
__global__ void rank_sum_kernel(const double* part, int64_t stride, int G, int64_t M, double* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < G; ++r) s += part[r * stride + i];
    out[i] = s;
  }
}

}  // namespace

struct tcx_comm {
  int kind = TCX_COMM_VIRTUAL;
  int world = 1, rank = 0, device = 0;
  ncclComm_t nc = nullptr;
  tcx_host_exchange_fn fn = nullptr;
  void* user = nullptr;
  cudaStream_t cs = nullptr, ks = nullptr;  // exchange stream, staging-copy stream
  cudaEvent_t ev_go = nullptr, ev_done = nullptr, ev_recv[2] = {nullptr, nullptr},
              ev_copy[2] = {nullptr, nullptr};
  size_t chunk = (size_t)256 << 20;  // staging chunk (bytes); two are resident
  cudaEvent_t ev_chunk[kXChunksMax] = {};  // overlapped exchanges: chunk c has landed
  void* hsend = nullptr;             // host transport: pinned staging
  void* hrecv = nullptr;
  size_t hbytes = 0;
  ~tcx_comm() {
    if (nc) nccl().commDestroy(nc);
    for (cudaEvent_t e : {ev_go, ev_done, ev_recv[0], ev_recv[1], ev_copy[0], ev_copy[1]})
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_chunk)
      if (e) cudaEventDestroy(e);
    if (cs) cudaStreamDestroy(cs);
    if (ks) cudaStreamDestroy(ks);
    if (hsend) cudaFreeHost(hsend);
    if (hrecv) cudaFreeHost(hrecv);
  }
};

namespace {

tcx_status comm_streams(tcx_comm* c) {
  CUDA_TRY(cudaGetDevice(&c->device));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->ks, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&c->ev_go, &c->ev_done, &c->ev_recv[0], &c->ev_recv[1], &c->ev_copy[0],
                         &c->ev_copy[1]})
    CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  for (cudaEvent_t& e : c->ev_chunk) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (const char* e = getenv("TCX_XCHG_CHUNK_MB")) c->chunk = (size_t)std::max(1, atoi(e)) << 20;
  return TCX_OK;
}

// Per-call workspace of a sharded run: [local ranks][per-rank ws] then the virtual ranks'
// E / grad partials, then (NCCL) two staging chunks.
struct ShardWs {
  size_t per_rank, parts, stage, total;
  int local;  // ranks this process runs
};
ShardWs shard_ws(const Plan& P, const Binding* Bd, const tcx_comm* c, int64_t B, int kind) {
  ShardWs s{};
  s.local = c->kind == TCX_COMM_VIRTUAL ? c->world : 1;
  s.per_rank = align256(ws_layout(P, Bd, B, kind, false).total);
  size_t off = s.per_rank * s.local;
  s.parts = off;
  if (c->kind == TCX_COMM_VIRTUAL && s.local > 1)
    off += align256((size_t)s.local * B * (1 + std::max(P.P, 1)) * 8);
  s.stage = off;
  if (c->kind == TCX_COMM_NCCL && c->world > 1) off += 2 * align256(c->chunk);
  s.total = off;
  return s;
}

// EXCHANGE of the buffers at byte offset `boff` inside each rank's workspace, for the byte
// columns [c0, c1) of every block (the whole block, or one chunk of an exchange that overlaps
// the next pass).  xchg_begin orders the exchange streams after everything already queued on
// the caller's stream; xchg_cols enqueues the data movement on them (virtual: swap kernels on
// the exchange stream; NCCL: grouped send / recv on it and staging copies on the copy stream;
// host: synchronous on the caller's stream); xchg_mark records `ev` once the columns landed.
tcx_status xchg_begin(tcx_comm* c, cudaStream_t st) {
  if (c->kind == TCX_COMM_HOST) return TCX_OK;
  CUDA_TRY(cudaEventRecord(c->ev_go, st));
  CUDA_TRY(cudaStreamWaitEvent(c->cs, c->ev_go, 0));
  CUDA_TRY(cudaStreamWaitEvent(c->ks, c->ev_go, 0));
  return TCX_OK;
}
tcx_status xchg_mark(tcx_comm* c, cudaEvent_t ev, cudaStream_t st) {
  if (c->kind == TCX_COMM_HOST) return TCX_OK;  // already complete on st
  // both streams: the exchange stream (swaps / sends and receives) and the copy stream
  CUDA_TRY(cudaEventRecord(c->ev_done, c->cs));
  CUDA_TRY(cudaStreamWaitEvent(c->ks, c->ev_done, 0));
  CUDA_TRY(cudaEventRecord(ev, c->ks));
  (void)st;
  return TCX_OK;
}
tcx_status xchg_cols(tcx_comm* c, const Plan& P, char* W, const ShardWs& sw, size_t boff, int64_t B,
                     int64_t c0, int64_t c1, int& it, cudaStream_t st) {
  const int G = 1 << P.gbits;
  const size_t esz = P.dtype == TCX_C128 ? 16 : 8;
  const int64_t N = (int64_t)1 << P.nloc;
  const int64_t Cb = (N / G) * (int64_t)esz;  // block bytes
  if (c->kind == TCX_COMM_VIRTUAL) {
    SwapArgs a{};
    for (int r = 0; r < G; ++r) a.base[r] = W + r * sw.per_rank + boff;
    a.row_bytes = N * (int64_t)esz;
    a.block_bytes = Cb;
    a.col_off = c0;
    a.col_bytes = c1 - c0;
    a.B = B;
    for (int s = 1; s < G; ++s) {
      a.s = s;
      a.hbit = 31 - __builtin_clz(s);
      const int64_t per_pair = (a.col_bytes >> 4) * B;
      const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((per_pair + 255) / 256,
                                                                           148 * 8 / std::max(1, G / 2)));
      virtual_swap_kernel<<<dim3(gx, G / 2), 256, 0, c->cs>>>(a);
      CUDA_TRY(cudaGetLastError());
    }
    return TCX_OK;
  }
  char* buf = W + boff;
  const int r = c->rank;
  // rows of one staging chunk: the whole column range when it fits, else a sub-range
  const int64_t cols = std::max<int64_t>(16, std::min<int64_t>(c1 - c0, (int64_t)c->chunk / B) & ~(int64_t)15);
  if (c->kind == TCX_COMM_HOST) {
    const size_t need = (size_t)B * cols;
    if (c->hbytes < need) {
      if (c->hsend) cudaFreeHost(c->hsend);
      if (c->hrecv) cudaFreeHost(c->hrecv);
      c->hsend = c->hrecv = nullptr;
      c->hbytes = 0;
      CUDA_TRY(cudaMallocHost(&c->hsend, need));
      CUDA_TRY(cudaMallocHost(&c->hrecv, need));
      c->hbytes = need;
    }
    for (int s = 1; s < G; ++s) {
      const int peer = r ^ s;
      for (int64_t x0 = c0; x0 < c1; x0 += cols) {
        const int64_t w = std::min(cols, c1 - x0);
        CUDA_TRY(cudaMemcpy2DAsync(c->hsend, w, buf + peer * Cb + x0, N * esz, w, B,
                                   cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        if (c->fn(c->user, peer, c->hsend, c->hrecv, (size_t)(w * B)) != 0)
          return fail(TCX_E_NCCL, "host exchange callback failed");
        CUDA_TRY(cudaMemcpy2DAsync(buf + peer * Cb + x0, N * esz, c->hrecv, w, w, B,
                                   cudaMemcpyHostToDevice, st));
      }
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    return TCX_OK;
  }
  // NCCL: sends straight from the state, receives into two staging chunks; the copy stream
  // moves chunk i into place while chunk i+1 is on the wire.
  NcclApi& A = nccl();
  char* stage[2] = {W + sw.stage, W + sw.stage + align256(c->chunk)};
  for (int s = 1; s < G; ++s) {
    const int peer = r ^ s;
    for (int64_t x0 = c0; x0 < c1; x0 += cols, ++it) {
      const int64_t w = std::min(cols, c1 - x0);
      const int sb = it & 1;
      if (it >= 2) CUDA_TRY(cudaStreamWaitEvent(c->cs, c->ev_copy[sb], 0));  // staging free
      NCCL_TRY(A.groupStart());
      for (int64_t b = 0; b < B; ++b) {
        NCCL_TRY(A.send(buf + b * N * esz + peer * Cb + x0, (size_t)w, ncclUint8, peer, c->nc, c->cs));
        NCCL_TRY(A.recv(stage[sb] + b * w, (size_t)w, ncclUint8, peer, c->nc, c->cs));
      }
      NCCL_TRY(A.groupEnd());
      CUDA_TRY(cudaEventRecord(c->ev_recv[sb], c->cs));
      CUDA_TRY(cudaStreamWaitEvent(c->ks, c->ev_recv[sb], 0));
      // the copy overwrites the block range just sent: ev_recv completes with the whole
      // group, sends included
      CUDA_TRY(cudaMemcpy2DAsync(buf + peer * Cb + x0, N * esz, stage[sb], w, w, B,
                                 cudaMemcpyDeviceToDevice, c->ks));
      CUDA_TRY(cudaEventRecord(c->ev_copy[sb], c->ks));
    }
  }
  return TCX_OK;
}

// One whole EXCHANGE (every column of every block), joined back into the caller's stream.
tcx_status exchange(tcx_comm* c, const Plan& P, char* W, const ShardWs& sw, size_t boff, int64_t B,
                    cudaStream_t st) {
  const int64_t Cb = ((int64_t)1 << (P.nloc - P.gbits)) * (P.dtype == TCX_C128 ? 16 : 8);
  int it = 0;
  tcx_status s;
  if ((s = xchg_begin(c, st)) || (s = xchg_cols(c, P, W, sw, boff, B, 0, Cb, it, st)) ||
      (s = xchg_mark(c, c->ev_chunk[0], st)))
    return s;
  if (c->kind != TCX_COMM_HOST) CUDA_TRY(cudaStreamWaitEvent(st, c->ev_chunk[0], 0));
  return TCX_OK;
}

// Sum E[B] and grad[B][P] over the ranks (in place on every rank).
tcx_status allreduce(tcx_comm* c, double* E, double* grad, int64_t B, int P, cudaStream_t st) {
  if (c->world == 1) return TCX_OK;
  if (c->kind == TCX_COMM_NCCL) {
    NcclApi& A = nccl();
    NCCL_TRY(A.groupStart());
    NCCL_TRY(A.allReduce(E, E, (size_t)B, ncclFloat64, ncclSum, c->nc, st));
    if (grad && P > 0) NCCL_TRY(A.allReduce(grad, grad, (size_t)B * P, ncclFloat64, ncclSum, c->nc, st));
    NCCL_TRY(A.groupEnd());
    return TCX_OK;
  }
  // host: recursive doubling; each step adds the partner's vector in rank order (lower
  // rank's term first), so every rank ends with bitwise the same sums
  const size_t M = (size_t)B * (1 + (grad ? P : 0));
  std::vector<double> mine(M), other(M);
  CUDA_TRY(cudaMemcpyAsync(mine.data(), E, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
  if (grad && P > 0)
    CUDA_TRY(cudaMemcpyAsync(mine.data() + B, grad, sizeof(double) * B * P, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (int s = 1; s < c->world; s <<= 1) {
    const int peer = c->rank ^ s;
    if (c->fn(c->user, peer, mine.data(), other.data(), M * sizeof(double)) != 0)
      return fail(TCX_E_NCCL, "host exchange callback failed (all-reduce)");
    for (size_t i = 0; i < M; ++i)
      mine[i] = c->rank < peer ? mine[i] + other[i] : other[i] + mine[i];
  }
  CUDA_TRY(cudaMemcpyAsync(E, mine.data(), sizeof(double) * B, cudaMemcpyHostToDevice, st));
  if (grad && P > 0)
    CUDA_TRY(cudaMemcpyAsync(grad, mine.data() + B, sizeof(double) * B * P, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return TCX_OK;
}

// The whole sharded program (tcx_shard_program's steps) for the ranks this process runs.
tcx_status run_sharded(Plan& P, const tcx_pauli* H, tcx_comm* c, const double* theta, int64_t B,
                       double* E, double* grad, void* ws, size_t ws_bytes, cudaStream_t st, int kind) {
  if (!H || !c) return fail(TCX_E_INVALID, "null pauli or comm");
  if (B <= 0) return fail(TCX_E_INVALID, "B must be > 0");
  if (!E || (kind == K_GRAD && P.P > 0 && !grad)) return fail(TCX_E_INVALID, "null output");
  if (P.cluster) return fail(TCX_E_INVALID, "cluster-resident plans run on one GPU (tcx_grad_batch)");
  if (c->world != (1 << P.gbits))
    return fail(TCX_E_INVALID, "comm world size " + std::to_string(c->world) +
                                   " != 2^global_bits = " + std::to_string(1 << P.gbits));
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev != c->device) return fail(TCX_E_INVALID, "comm was created on another device");
  if (P.gbits == 0) {  // one rank: the ordinary program, then the (trivial) reduction
    tcx_status s = run(P, H, theta, B, E, grad, nullptr, ws, ws_bytes, st, kind, nullptr);
    return s ? s : allreduce(c, E, grad, B, P.P, st);
  }
  std::shared_ptr<Binding> Bd;
  tcx_status s = binding_for(P, H, Bd, nullptr);
  if (s) return s;
  const ShardWs sw = shard_ws(P, Bd.get(), c, B, kind);
  if (!ws || ws_bytes < sw.total)
    return fail(TCX_E_INVALID, "workspace too small: need " + std::to_string(sw.total) +
                                   " bytes (tcx_sharded_workspace_bytes), got " + std::to_string(ws_bytes));
  const WsLayout wl = ws_layout(P, Bd.get(), B, kind, false);
  const std::vector<tcx_shard_step> prog = shard_program(P, *Bd, kind == K_GRAD);
  int first_lambda = -1;
  for (int u = 0; u < (int)Bd->units.size() && first_lambda < 0; ++u)
    if (!Bd->units[u].swapped) first_lambda = u;
  if (first_lambda < 0) first_lambda = 0;
  char* W = (char*)ws;
  const int Pp = std::max(P.P, 1);
  double* parts = (double*)(W + sw.parts);
  auto Ep = [&](int li) { return sw.local > 1 ? parts + (size_t)li * B * (1 + Pp) : E; };
  auto Gp = [&](int li) { return sw.local > 1 ? parts + (size_t)li * B * (1 + Pp) + B : grad; };
  const bool no_overlap = getenv("TCX_XCHG_NO_OVERLAP") != nullptr;  // A/B switch, read per call
  const int64_t Cb = ((int64_t)1 << (P.nloc - P.gbits)) * (P.dtype == TCX_C128 ? 16 : 8);
  for (size_t si = 0; si < prog.size(); ++si) {
    const tcx_shard_step& stp = prog[si];
    if (stp.kind == TCX_STEP_EXCHANGE) {
      const bool both = (stp.arg & 2) && wl.lam;
      // the next pass can start on chunk q while chunks q+1.. are still moving when its window
      // leaves the chunk bits out (tcx.cu pass_chunkable; planned for by the layout search)
      const tcx_shard_step* nx = si + 1 < prog.size() ? &prog[si + 1] : nullptr;
      const bool overlap = !no_overlap && nx && (nx->kind == TCX_STEP_FWD || nx->kind == TCX_STEP_BWD) &&
                           pass_chunkable(P, P.passes[nx->arg]) && c->kind != TCX_COMM_HOST;
      ProfEntry pe{};
      cudaStream_t ps = c->kind == TCX_COMM_HOST ? st : c->cs;  // the exchange's own timeline
      if (g_prof.on) {
        CUDA_TRY(cudaEventCreate(&pe.a));
        CUDA_TRY(cudaEventCreate(&pe.b));
      }
      if (!overlap) {
        if (g_prof.on) CUDA_TRY(cudaEventRecord(pe.a, st));
        if ((s = exchange(c, P, W, sw, wl.psi, B, st))) return s;
        if (both && (s = exchange(c, P, W, sw, wl.lam, B, st))) return s;
        if (g_prof.on) CUDA_TRY(cudaEventRecord(pe.b, st));
      } else {
        const int nc = 1 << P.xchunk_bits;
        int it = 0;
        if ((s = xchg_begin(c, st))) return s;
        if (g_prof.on) CUDA_TRY(cudaEventRecord(pe.a, ps));
        for (int q = 0; q < nc; ++q) {
          const int64_t c0 = Cb * q / nc, c1 = Cb * (q + 1) / nc;
          if ((s = xchg_cols(c, P, W, sw, wl.psi, B, c0, c1, it, st))) return s;
          if (both && (s = xchg_cols(c, P, W, sw, wl.lam, B, c0, c1, it, st))) return s;
          if ((s = xchg_mark(c, c->ev_chunk[q], st))) return s;
          if (g_prof.on && q == nc - 1) CUDA_TRY(cudaEventRecord(pe.b, c->ks));
          CUDA_TRY(cudaStreamWaitEvent(st, c->ev_chunk[q], 0));
          for (int li = 0; li < sw.local; ++li) {  // the next pass on chunk q of every rank
            const int rank = sw.local > 1 ? li : c->rank;
            OneStep one{nx->kind, nx->arg, rank, false, q};
            if ((s = run(P, H, theta, B, Ep(li), Gp(li), nullptr, W + (size_t)li * sw.per_rank,
                         sw.per_rank, st, kind, &wl, &one)))
              return s;
          }
        }
        ++si;  // that pass ran
      }
      if (g_prof.on) {
        // bytes that change rank: (G-1)/G of every local state moved; virtual ranks read and
        // write each of them in HBM (swap kernel), a real rank sends its share over the link
        const double moved = (double)B * (double)((int64_t)1 << P.nloc) * (P.dtype == TCX_C128 ? 16 : 8) *
                             (double)(c->world - 1) / c->world * (both ? 2 : 1);
        pe.phase = 8;
        pe.index = stp.arg | (overlap ? 4 : 0);
        pe.flops = 0;
        pe.bytes = sw.local > 1 ? 2.0 * moved * sw.local : moved;
        g_prof.log.push_back(pe);
      }
      continue;
    }
    for (int li = 0; li < sw.local; ++li) {
      const int rank = sw.local > 1 ? li : c->rank;
      OneStep one{stp.kind, stp.arg, rank, stp.kind == TCX_STEP_LAMBDA && stp.arg == first_lambda};
      if ((s = run(P, H, theta, B, Ep(li), Gp(li), nullptr, W + (size_t)li * sw.per_rank, sw.per_rank,
                   st, kind, &wl, &one)))
        return s;
    }
  }
  if (sw.local > 1) {  // virtual ranks: fixed-order sums of the partials
    rank_sum_kernel<<<(unsigned)std::min<int64_t>(1024, (B + 255) / 256), 256, 0, st>>>(
        parts, B * (1 + Pp), sw.local, B, E);
    CUDA_TRY(cudaGetLastError());
    if (kind == K_GRAD && P.P > 0) {
      // grad rows are [B][Pp] with Pp == P when P > 0
      rank_sum_kernel<<<(unsigned)std::min<int64_t>(4096, (B * P.P + 255) / 256), 256, 0, st>>>(
          parts + B, B * (1 + Pp), sw.local, B * (int64_t)P.P, grad);
      CUDA_TRY(cudaGetLastError());
    }
    return TCX_OK;
  }
  return allreduce(c, E, kind == K_GRAD ? grad : nullptr, B, P.P, st);
}

}  // namespace

extern "C" {

tcx_status tcx_comm_unique_id(void* id_out) {
  g_err.clear();
  if (!id_out) return fail(TCX_E_INVALID, "null id");
  NcclApi& A = nccl();
  if (!A.ok) return fail(TCX_E_NCCL, A.err);
  ncclUniqueId id;
  NCCL_TRY(A.getUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return TCX_OK;
}

tcx_status tcx_comm_init(const void* nccl_unique_id, int32_t world, int32_t rank, tcx_comm** out) {
  g_err.clear();
  if (!out || !nccl_unique_id) return fail(TCX_E_INVALID, "null argument");
  *out = nullptr;
  if (world < 1 || world > 64 || (world & (world - 1)) || rank < 0 || rank >= world)
    return fail(TCX_E_INVALID, "world must be a power of two in [1, 64] and 0 <= rank < world");
  NcclApi& A = nccl();
  if (!A.ok) return fail(TCX_E_NCCL, A.err);
  std::unique_ptr<tcx_comm> c(new (std::nothrow) tcx_comm());
  if (!c) return fail(TCX_E_OOM, "out of host memory");
  c->kind = TCX_COMM_NCCL;
  c->world = world;
  c->rank = rank;
  tcx_status s = comm_streams(c.get());
  if (s) return s;
  ncclUniqueId id;
  std::memcpy(&id, nccl_unique_id, sizeof(id));
  NCCL_TRY(A.commInitRank(&c->nc, world, id, rank));
  *out = c.release();
  return TCX_OK;
}

tcx_status tcx_comm_init_virtual(int32_t world, tcx_comm** out) {
  g_err.clear();
  if (!out) return fail(TCX_E_INVALID, "null out");
  *out = nullptr;
  if (world < 1 || world > 64 || (world & (world - 1)))
    return fail(TCX_E_INVALID, "world must be a power of two in [1, 64]");
  std::unique_ptr<tcx_comm> c(new (std::nothrow) tcx_comm());
  if (!c) return fail(TCX_E_OOM, "out of host memory");
  c->kind = TCX_COMM_VIRTUAL;
  c->world = world;
  tcx_status s = comm_streams(c.get());
  if (s) return s;
  *out = c.release();
  return TCX_OK;
}

tcx_status tcx_comm_init_host(int32_t world, int32_t rank, tcx_host_exchange_fn fn, void* user,
                              tcx_comm** out) {
  g_err.clear();
  if (!out || !fn) return fail(TCX_E_INVALID, "null argument");
  *out = nullptr;
  if (world < 1 || world > 64 || (world & (world - 1)) || rank < 0 || rank >= world)
    return fail(TCX_E_INVALID, "world must be a power of two in [1, 64] and 0 <= rank < world");
  std::unique_ptr<tcx_comm> c(new (std::nothrow) tcx_comm());
  if (!c) return fail(TCX_E_OOM, "out of host memory");
  c->kind = TCX_COMM_HOST;
  c->world = world;
  c->rank = rank;
  c->fn = fn;
  c->user = user;
  tcx_status s = comm_streams(c.get());
  if (s) return s;
  *out = c.release();
  return TCX_OK;
}

void tcx_comm_free(tcx_comm* c) { delete c; }

tcx_status tcx_comm_info(const tcx_comm* c, int32_t* kind, int32_t* world, int32_t* rank) {
  g_err.clear();
  if (!c) return fail(TCX_E_INVALID, "null comm");
  if (kind) *kind = c->kind;
  if (world) *world = c->world;
  if (rank) *rank = c->rank;
  return TCX_OK;
}

tcx_status tcx_sharded_workspace_bytes(const tcx_circuit* circ, const tcx_pauli* pauli,
                                       const tcx_comm* comm, int64_t B, int32_t want_grad,
                                       size_t* bytes) {
  g_err.clear();
  if (!circ || !pauli || !comm || !bytes) return fail(TCX_E_INVALID, "null argument");
  if (B <= 0) return fail(TCX_E_INVALID, "B must be > 0");
  Plan& P = const_cast<tcx_circuit*>(circ)->plan;
  std::shared_ptr<Binding> Bd;
  tcx_status s = binding_for(P, pauli, Bd, nullptr);
  if (s) return s;
  const int kind = want_grad ? K_GRAD : K_EXPECT;
  if (P.gbits == 0) {
    *bytes = ws_layout(P, Bd.get(), B, kind, false).total;
    return TCX_OK;
  }
  *bytes = shard_ws(P, Bd.get(), comm, B, kind).total;
  return TCX_OK;
}

tcx_status tcx_grad_sharded(const tcx_circuit* circ, const tcx_pauli* pauli, tcx_comm* comm,
                            const double* theta, int64_t B, double* E, double* grad, void* ws,
                            size_t ws_bytes, void* stream) {
  g_err.clear();
  if (!circ) return fail(TCX_E_INVALID, "null circuit");
  Plan& P = const_cast<tcx_circuit*>(circ)->plan;
  if (!P.unitary) return fail(TCX_E_UNSUPPORTED, "grad needs unitary payloads (adjoint applies U^dagger)");
  return run_sharded(P, pauli, comm, theta, B, E, grad, ws, ws_bytes, (cudaStream_t)stream, K_GRAD);
}

tcx_status tcx_expect_sharded(const tcx_circuit* circ, const tcx_pauli* pauli, tcx_comm* comm,
                              const double* theta, int64_t B, double* E, void* ws, size_t ws_bytes,
                              void* stream) {
  g_err.clear();
  if (!circ) return fail(TCX_E_INVALID, "null circuit");
  return run_sharded(const_cast<tcx_circuit*>(circ)->plan, pauli, comm, theta, B, E, nullptr, ws,
                     ws_bytes, (cudaStream_t)stream, K_EXPECT);
}

}  // extern "C"
