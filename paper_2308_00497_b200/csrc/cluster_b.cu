// K5 cluster-kernel instances, direction=1.
#include "cluster_instances.cuh"
namespace fftgen_b200 {
FFTGEN_CLUSTER_INSTANCES(b, 1)
}  // namespace fftgen_b200
