// Instantiations: Lindblad capacity 8 (ell = 5..8; e.g. the eight Gell-Mann
// matrices of su(3)) for 2x2 and 3x3 payloads, float.
#include "instantiate.cuh"

namespace otfx {

const Ops<float>* ops_matrix_f32_l8(int kind, int K) {
  switch (K) {
    case 2: return kind == KIND_MATRIX_REAL ? OpsFor<SymPolicy<float, 2, 8>, float>::table(kind)
                                            : OpsFor<HermPolicy<float, 2, 8>, float>::table(kind);
    case 3: return kind == KIND_MATRIX_REAL ? OpsFor<SymPolicy<float, 3, 8>, float>::table(kind)
                                            : OpsFor<HermPolicy<float, 3, 8>, float>::table(kind);
    default: return nullptr;
  }
}

}  // namespace otfx
