// Instantiations: 3x3 real-symmetric and complex-Hermitian payloads, float,
// Lindblad capacity 2 (the common case) or 4.
#include "instantiate.cuh"

namespace otfx {

const Ops<float>* ops_matrix_f32_k3(int kind, int lmax) {
  if (kind == KIND_MATRIX_REAL)
    return lmax <= 2 ? OpsFor<SymPolicy<float, 3, 2>, float>::table(kind)
                     : OpsFor<SymPolicy<float, 3, 4>, float>::table(kind);
  return lmax <= 2 ? OpsFor<HermPolicy<float, 3, 2>, float>::table(kind)
                   : OpsFor<HermPolicy<float, 3, 4>, float>::table(kind);
}

}  // namespace otfx
