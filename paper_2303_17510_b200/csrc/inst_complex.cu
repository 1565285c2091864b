// inst_complex.cu — kernel instantiations for complex data, blocks up to 3072 points (the registry of a
// symmetry is split over two translation units for parallel builds; inst_complex_long.cu has the rest).
#include "registry.cuh"
namespace hc {
void registry_sym0_a(KernelEntry* out, int* count) { build_registry<0, 0>(out, count); }
}  // namespace hc
