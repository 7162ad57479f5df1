// Instantiations: scalar and vector payloads, float.
#include "instantiate.cuh"

namespace otfx {

const Ops<float>* ops_vector_f32(int K, bool has_w) {
  if (!has_w) return K == 1 ? OpsFor<VecPolicy<float, 1, false>, float>::table(KIND_SCALAR) : nullptr;
  switch (K) {
    case 2: return OpsFor<VecPolicy<float, 2, true>, float>::table(KIND_VECTOR);
    case 3: return OpsFor<VecPolicy<float, 3, true>, float>::table(KIND_VECTOR);
    case 4: return OpsFor<VecPolicy<float, 4, true>, float>::table(KIND_VECTOR);
    case 5: return OpsFor<VecPolicy<float, 5, true>, float>::table(KIND_VECTOR);
    case 6: return OpsFor<VecPolicy<float, 6, true>, float>::table(KIND_VECTOR);
    case 8: return OpsFor<VecPolicy<float, 8, true>, float>::table(KIND_VECTOR);
    default: return nullptr;
  }
}

}  // namespace otfx
