// Instantiations: sparse graphs (ell <= k edges) on k = 4, 5 channels, float.
#include "instantiate.cuh"

namespace otfx {

const Ops<float>* ops_vector_f32_sparse_k45(int K) {
  switch (K) {
    case 4: return OpsFor<VecPolicy<float, 4, true, 4>, float>::table(KIND_VECTOR);
    case 5: return OpsFor<VecPolicy<float, 5, true, 5>, float>::table(KIND_VECTOR);
    default: return nullptr;
  }
}

}  // namespace otfx
