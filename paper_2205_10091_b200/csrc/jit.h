// jit.h -- per-circuit kernel specialisation (see jit.cpp).
#pragma once
#include <string>
#include <vector>

namespace tcx {
struct Plan;
bool jit_available(std::string* why);
// compile (or fetch from the disk cache) the kernels keys = pass*4 + km not yet built
bool jit_build(Plan& P, const std::vector<int>& keys, std::string& err);
std::string jit_source(const Plan& P, int pass, int km);  // generated CUDA C++ (debug/tests)
std::string jit_kernel_name(int pass, int km);
}  // namespace tcx
