// K2 instances: layout=LAYOUT_INTERLEAVED, direction=1.
#include "block_instances.cuh"
namespace fftgen_b200 {
FFTGEN_BLOCK_INSTANCES(i_b, LAYOUT_INTERLEAVED, 1)
}  // namespace fftgen_b200
