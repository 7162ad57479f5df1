// Instantiations: real-symmetric and complex-Hermitian matrix payloads, double.
#include "instantiate.cuh"

namespace otfx {

const Ops<double>* ops_matrix_f64(int kind, int K) {
  if (kind == KIND_MATRIX_REAL) {
    switch (K) {
      case 2: return OpsFor<SymPolicy<double, 2>, double>::table(kind);
      case 3: return OpsFor<SymPolicy<double, 3>, double>::table(kind);
      case 4: return OpsFor<SymPolicy<double, 4>, double>::table(kind);
      default: return nullptr;
    }
  }
  switch (K) {
    case 2: return OpsFor<HermPolicy<double, 2>, double>::table(kind);
    case 3: return OpsFor<HermPolicy<double, 3>, double>::table(kind);
    case 4: return OpsFor<HermPolicy<double, 4>, double>::table(kind);
    default: return nullptr;
  }
}

}  // namespace otfx
