// K2 instances: layout=LAYOUT_SPLIT, direction=1.
#include "block_instances.cuh"
namespace fftgen_b200 {
FFTGEN_BLOCK_INSTANCES(s_b, LAYOUT_SPLIT, 1)
}  // namespace fftgen_b200
