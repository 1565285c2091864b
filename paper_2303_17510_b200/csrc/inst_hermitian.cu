// inst_hermitian.cu — kernel instantiations for hermitian data, blocks up to 3072 points (the registry of a
// symmetry is split over two translation units for parallel builds; inst_hermitian_long.cu has the rest).
#include "registry.cuh"
namespace hc {
void registry_sym2_a(KernelEntry* out, int* count) { build_registry<2, 0>(out, count); }
}  // namespace hc
