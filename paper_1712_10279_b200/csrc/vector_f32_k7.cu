// Instantiation: k = 7 vector payload, float (its own unit keeps the build parallel).
#include "instantiate.cuh"

namespace otfx {

const Ops<float>* ops_vector_f32_k7() {
  return OpsFor<VecPolicy<float, 7, true>, float>::table(KIND_VECTOR);
}

}  // namespace otfx
