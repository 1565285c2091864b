// inst_complex_long.cu — kernel instantiations for complex data: the long blocks (4096 points and more) and
// the direct-sum entry (appended after inst_complex.cu's part of the table).
#include "registry.cuh"
namespace hc {
void registry_sym0_b(KernelEntry* out, int* count) { build_registry<0, 1>(out, count); }
}  // namespace hc
