// Instantiations: real-symmetric and complex-Hermitian matrix payloads, float.
#include "instantiate.cuh"

namespace otfx {

const Ops<float>* ops_matrix_f32(int kind, int K) {
  if (kind == KIND_MATRIX_REAL) {
    switch (K) {
      case 2: return OpsFor<SymPolicy<float, 2>, float>::table(kind);
      case 3: return OpsFor<SymPolicy<float, 3>, float>::table(kind);
      case 4: return OpsFor<SymPolicy<float, 4>, float>::table(kind);
      default: return nullptr;
    }
  }
  switch (K) {
    case 2: return OpsFor<HermPolicy<float, 2>, float>::table(kind);
    case 3: return OpsFor<HermPolicy<float, 3>, float>::table(kind);
    case 4: return OpsFor<HermPolicy<float, 4>, float>::table(kind);
    default: return nullptr;
  }
}

}  // namespace otfx
