// Instantiations: scalar and k = 2, 3 vector payloads, double.
#include "instantiate.cuh"

namespace otfx {

const Ops<double>* ops_vector_f64_small(int K, bool has_w) {
  if (!has_w) return K == 1 ? OpsFor<VecPolicy<double, 1, false>, double>::table(KIND_SCALAR) : nullptr;
  switch (K) {
    case 2: return OpsFor<VecPolicy<double, 2, true>, double>::table(KIND_VECTOR);
    case 3: return OpsFor<VecPolicy<double, 3, true>, double>::table(KIND_VECTOR);
    default: return nullptr;
  }
}

}  // namespace otfx
