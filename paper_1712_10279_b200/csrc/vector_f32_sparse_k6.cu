// Instantiations: sparse graphs (ell <= k edges) on k = 6 channels, float.
#include "instantiate.cuh"

namespace otfx {

const Ops<float>* ops_vector_f32_sparse_k6(int K) {
  switch (K) {
    case 6: return OpsFor<VecPolicy<float, 6, true, 6>, float>::table(KIND_VECTOR);
    default: return nullptr;
  }
}

}  // namespace otfx
