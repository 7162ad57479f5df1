// Instantiations: sparse graphs (ell <= k edges) on k = 6 channels, double.
#include "instantiate.cuh"

namespace otfx {

const Ops<double>* ops_vector_f64_sparse_k6(int K) {
  switch (K) {
    case 6: return OpsFor<VecPolicy<double, 6, true, 6>, double>::table(KIND_VECTOR);
    default: return nullptr;
  }
}

}  // namespace otfx
