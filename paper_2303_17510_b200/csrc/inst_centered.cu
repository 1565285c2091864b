// inst_centered.cu — kernel instantiations for centered data, blocks up to 3072 points (the registry of a
// symmetry is split over two translation units for parallel builds; inst_centered_long.cu has the rest).
#include "registry.cuh"
namespace hc {
void registry_sym1_a(KernelEntry* out, int* count) { build_registry<1, 0>(out, count); }
}  // namespace hc
