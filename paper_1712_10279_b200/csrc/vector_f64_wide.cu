// Instantiations: k = 4, 5, 6, 8 (7 in vector_f64_k7.cu) vector payloads, double.
#include "instantiate.cuh"

namespace otfx {

const Ops<double>* ops_vector_f64_k7();

const Ops<double>* ops_vector_f64_wide(int K) {
  switch (K) {
    case 4: return OpsFor<VecPolicy<double, 4, true>, double>::table(KIND_VECTOR);
    case 5: return OpsFor<VecPolicy<double, 5, true>, double>::table(KIND_VECTOR);
    case 6: return OpsFor<VecPolicy<double, 6, true>, double>::table(KIND_VECTOR);
    case 7: return ops_vector_f64_k7();
    case 8: return OpsFor<VecPolicy<double, 8, true>, double>::table(KIND_VECTOR);
    default: return nullptr;
  }
}

}  // namespace otfx
