// Dispatch of the matrix payload instantiations (float); one unit per k keeps
// the build parallel.
#include "ops.h"

namespace otfx {

const Ops<float>* ops_matrix_f32_k2(int kind, int lmax);
const Ops<float>* ops_matrix_f32_k3(int kind, int lmax);
const Ops<float>* ops_matrix_f32_k4(int kind, int lmax);

const Ops<float>* ops_matrix_f32(int kind, int K, int ell) {
  const int lmax = ell <= 2 ? 2 : 4;
  if (ell > 4) return nullptr;
  switch (K) {
    case 2: return ops_matrix_f32_k2(kind, lmax);
    case 3: return ops_matrix_f32_k3(kind, lmax);
    case 4: return ops_matrix_f32_k4(kind, lmax);
    default: return nullptr;
  }
}

}  // namespace otfx
