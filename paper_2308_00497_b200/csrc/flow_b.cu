// K3 dataflow-kernel instances, direction=1.
#include "flow_instances.cuh"
namespace fftgen_b200 {
FFTGEN_FLOW_INSTANCES(b, 1)
}  // namespace fftgen_b200
