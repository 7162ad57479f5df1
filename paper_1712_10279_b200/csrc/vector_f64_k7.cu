// Instantiation: k = 7 vector payload, double (its own unit keeps the build parallel).
#include "instantiate.cuh"

namespace otfx {

const Ops<double>* ops_vector_f64_k7() {
  return OpsFor<VecPolicy<double, 7, true>, double>::table(KIND_VECTOR);
}

}  // namespace otfx
