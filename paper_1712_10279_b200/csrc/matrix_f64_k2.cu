// Instantiations: 2x2 real-symmetric and complex-Hermitian payloads, double,
// Lindblad capacity 2 (the common case) or 4.
#include "instantiate.cuh"

namespace otfx {

const Ops<double>* ops_matrix_f64_k2(int kind, int lmax) {
  if (kind == KIND_MATRIX_REAL)
    return lmax <= 2 ? OpsFor<SymPolicy<double, 2, 2>, double>::table(kind)
                     : OpsFor<SymPolicy<double, 2, 4>, double>::table(kind);
  return lmax <= 2 ? OpsFor<HermPolicy<double, 2, 2>, double>::table(kind)
                   : OpsFor<HermPolicy<double, 2, 4>, double>::table(kind);
}

}  // namespace otfx
