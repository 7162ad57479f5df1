// Dispatch of the matrix payload instantiations (float); one unit per k keeps
// the build parallel.
#include "ops.h"

namespace otfx {

const Ops<float>* ops_matrix_f32_k2(int kind, int lmax);
const Ops<float>* ops_matrix_f32_k3(int kind, int lmax);
const Ops<float>* ops_matrix_f32_k4(int kind, int lmax);
const Ops<float>* ops_matrix_f32_l8(int kind, int K);

const Ops<float>* ops_matrix_f32(int kind, int K, int ell) {
  // Lindblad capacity classes: 2, 4, and 8 for k <= 3 (k^2 - 1 = 8 matrices
  // span su(3), e.g. the Gell-Mann set)
  if (ell > 4) return ell <= 8 ? ops_matrix_f32_l8(kind, K) : nullptr;
  const int lmax = ell <= 2 ? 2 : 4;
  switch (K) {
    case 2: return ops_matrix_f32_k2(kind, lmax);
    case 3: return ops_matrix_f32_k3(kind, lmax);
    case 4: return ops_matrix_f32_k4(kind, lmax);
    default: return nullptr;
  }
}

}  // namespace otfx
