// Instantiations: sparse graphs (ell <= k edges) on k = 8 channels, double.
#include "instantiate.cuh"

namespace otfx {

const Ops<double>* ops_vector_f64_sparse_k8(int K) {
  switch (K) {
    case 8: return OpsFor<VecPolicy<double, 8, true, 8>, double>::table(KIND_VECTOR);
    default: return nullptr;
  }
}

}  // namespace otfx
