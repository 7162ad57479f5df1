// Instantiations: sparse graphs (ell <= k edges) on k = 8 channels, float.
#include "instantiate.cuh"

namespace otfx {

const Ops<float>* ops_vector_f32_sparse_k8(int K) {
  switch (K) {
    case 8: return OpsFor<VecPolicy<float, 8, true, 8>, float>::table(KIND_VECTOR);
    default: return nullptr;
  }
}

}  // namespace otfx
