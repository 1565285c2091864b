// inst_hermitian.cu — kernel instantiations for hermitian data (split per symmetry for parallel builds).
#include "registry.cuh"
namespace hc {
void registry_sym2(KernelEntry* out, int* count) { build_registry<2>(out, count); }
}  // namespace hc
