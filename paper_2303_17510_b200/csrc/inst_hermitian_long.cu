// inst_hermitian_long.cu — kernel instantiations for hermitian data: the long blocks (4096 points and more) and
// the direct-sum entry (appended after inst_hermitian.cu's part of the table).
#include "registry.cuh"
namespace hc {
void registry_sym2_b(KernelEntry* out, int* count) { build_registry<2, 1>(out, count); }
}  // namespace hc
