// Dense contraction kernels on the 5th-generation tensor cores (tcgen05 / TMEM / TMA).
#include "../registry.hpp"

namespace mtb {

void register_matmul_kernels(kernel_table&) {}

} // namespace mtb
