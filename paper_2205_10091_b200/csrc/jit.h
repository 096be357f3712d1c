// jit.h -- per-circuit kernel specialisation (see jit.cpp).
#pragma once
#include <string>
#include <cstdint>
#include <vector>

namespace tcx {
struct Plan;
bool jit_available(std::string* why);
// Kernel keys: "p<pass>k<km>" (km 0 forward, 1 backward, 2 fused single pass) and
// "L<pauli hash>u<unit>" (lambda = H psi unit of a Pauli binding).
std::string jit_key_pass(int pass, int km);
// pass kernel with the lambda = H psi of a Pauli binding's unit 0 specialised in ("p..k..h<hash>")
std::string jit_key_pass_lam(int pass, int km, uint64_t pauli_hash);
std::string jit_key_lambda(uint64_t pauli_hash, int unit);
// "C<pauli hash>g<grad>": the cluster-resident megakernel of a plan built with cluster_bits
std::string jit_key_cluster(uint64_t pauli_hash, int grad);
int jit_cluster_smem(const Plan& P);  // its dynamic shared memory (bytes)
// compile (or fetch from the disk cache) the kernels not yet built
bool jit_build(Plan& P, const std::vector<std::string>& keys, std::string& err);
std::string jit_source(const Plan& P, const std::string& key);  // generated CUDA C++
// drop a built kernel and its disk-cache entry (the driver rejected the cubin): the next
// jit_build of the key compiles it afresh
void jit_evict(Plan& P, const std::string& key);
std::string jit_kernel_name(const std::string& key);
// software-pipelined TMA tiles (Plan::jit_pipe) for pass p's kernel with (bwd = two-state)
// or without the backward: on when the plan asks for it, the window is a TMA box and the
// prefetch buffer still fits the 227 KB of shared memory
struct PassInfo;
int jit_pipe_on(const Plan& P, const PassInfo& p, bool bwd);
}  // namespace tcx
