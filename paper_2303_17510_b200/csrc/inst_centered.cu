// inst_centered.cu — kernel instantiations for centered data (split per symmetry for parallel builds).
#include "registry.cuh"
namespace hc {
void registry_sym1(KernelEntry* out, int* count) { build_registry<1>(out, count); }
}  // namespace hc
