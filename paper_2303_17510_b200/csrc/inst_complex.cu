// inst_complex.cu — kernel instantiations for complex data (split per symmetry for parallel builds).
#include "registry.cuh"
namespace hc {
void registry_sym0(KernelEntry* out, int* count) { build_registry<0>(out, count); }
}  // namespace hc
