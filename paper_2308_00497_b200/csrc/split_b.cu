// K7 split-cluster kernel instances, direction=+1.
#include "split_instances.cuh"
namespace fftgen_b200 {
FFTGEN_SPLIT_INSTANCES(b, 1)
}  // namespace fftgen_b200
