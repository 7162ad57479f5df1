// Instantiations: sparse graphs (ell <= k edges) on k = 7 channels, double.
#include "instantiate.cuh"

namespace otfx {

const Ops<double>* ops_vector_f64_sparse_k7(int K) {
  switch (K) {
    case 7: return OpsFor<VecPolicy<double, 7, true, 7>, double>::table(KIND_VECTOR);
    default: return nullptr;
  }
}

}  // namespace otfx
