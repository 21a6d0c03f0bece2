// K6 phased-kernel instances, direction=-1.
#include "phased_instances.cuh"
namespace fftgen_b200 {
FFTGEN_PHASED_INSTANCES(f, -1)
}  // namespace fftgen_b200
