// Instantiations: sparse graphs (ell <= k edges) on k = 7 channels, float.
#include "instantiate.cuh"

namespace otfx {

const Ops<float>* ops_vector_f32_sparse_k7(int K) {
  switch (K) {
    case 7: return OpsFor<VecPolicy<float, 7, true, 7>, float>::table(KIND_VECTOR);
    default: return nullptr;
  }
}

}  // namespace otfx
