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
std::string jit_key_lambda(uint64_t pauli_hash, int unit);
// compile (or fetch from the disk cache) the kernels not yet built
bool jit_build(Plan& P, const std::vector<std::string>& keys, std::string& err);
std::string jit_source(const Plan& P, const std::string& key);  // generated CUDA C++
std::string jit_kernel_name(const std::string& key);
}  // namespace tcx
