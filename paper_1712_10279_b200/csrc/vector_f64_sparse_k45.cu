// Instantiations: sparse graphs (ell <= k edges) on k = 4, 5 channels, double.
#include "instantiate.cuh"

namespace otfx {

const Ops<double>* ops_vector_f64_sparse_k45(int K) {
  switch (K) {
    case 4: return OpsFor<VecPolicy<double, 4, true, 4>, double>::table(KIND_VECTOR);
    case 5: return OpsFor<VecPolicy<double, 5, true, 5>, double>::table(KIND_VECTOR);
    default: return nullptr;
  }
}

}  // namespace otfx
