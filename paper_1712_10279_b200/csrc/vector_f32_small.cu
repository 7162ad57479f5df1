// Instantiations: scalar and k = 2, 3 vector payloads, float.
#include "instantiate.cuh"

namespace otfx {

const Ops<float>* ops_vector_f32_small(int K, bool has_w) {
  if (!has_w) return K == 1 ? OpsFor<VecPolicy<float, 1, false>, float>::table(KIND_SCALAR) : nullptr;
  switch (K) {
    case 2: return OpsFor<VecPolicy<float, 2, true>, float>::table(KIND_VECTOR);
    case 3: return OpsFor<VecPolicy<float, 3, true>, float>::table(KIND_VECTOR);
    default: return nullptr;
  }
}

}  // namespace otfx
