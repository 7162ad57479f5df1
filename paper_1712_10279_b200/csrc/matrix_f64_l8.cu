// Instantiations: Lindblad capacity 8 (ell = 5..8; e.g. the eight Gell-Mann
// matrices of su(3)) for 2x2 and 3x3 payloads, double.
#include "instantiate.cuh"

namespace otfx {

const Ops<double>* ops_matrix_f64_l8(int kind, int K) {
  switch (K) {
    case 2: return kind == KIND_MATRIX_REAL ? OpsFor<SymPolicy<double, 2, 8>, double>::table(kind)
                                            : OpsFor<HermPolicy<double, 2, 8>, double>::table(kind);
    case 3: return kind == KIND_MATRIX_REAL ? OpsFor<SymPolicy<double, 3, 8>, double>::table(kind)
                                            : OpsFor<HermPolicy<double, 3, 8>, double>::table(kind);
    default: return nullptr;
  }
}

}  // namespace otfx
