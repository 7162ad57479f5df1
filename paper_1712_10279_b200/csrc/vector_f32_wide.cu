// Instantiations: k = 4, 5, 6, 8 (7 in vector_f32_k7.cu) vector payloads, float.
#include "instantiate.cuh"

namespace otfx {

const Ops<float>* ops_vector_f32_k7();

const Ops<float>* ops_vector_f32_wide(int K) {
  switch (K) {
    case 4: return OpsFor<VecPolicy<float, 4, true>, float>::table(KIND_VECTOR);
    case 5: return OpsFor<VecPolicy<float, 5, true>, float>::table(KIND_VECTOR);
    case 6: return OpsFor<VecPolicy<float, 6, true>, float>::table(KIND_VECTOR);
    case 7: return ops_vector_f32_k7();
    case 8: return OpsFor<VecPolicy<float, 8, true>, float>::table(KIND_VECTOR);
    default: return nullptr;
  }
}

}  // namespace otfx
