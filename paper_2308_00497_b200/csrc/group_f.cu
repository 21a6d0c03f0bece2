// K3 group-kernel instances, direction=-1.
#include "group_instances.cuh"
namespace fftgen_b200 {
FFTGEN_GROUP_INSTANCES(f, -1)
}  // namespace fftgen_b200
