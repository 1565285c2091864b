// inst_centered_long.cu — kernel instantiations for centered data: the long blocks (4096 points and more) and
// the direct-sum entry (appended after inst_centered.cu's part of the table).
#include "registry.cuh"
namespace hc {
void registry_sym1_b(KernelEntry* out, int* count) { build_registry<1, 1>(out, count); }
}  // namespace hc
