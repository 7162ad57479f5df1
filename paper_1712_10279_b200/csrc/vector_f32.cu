// Dispatch of the scalar / vector payload instantiations (float).
#include "ops.h"

namespace otfx {

const Ops<float>* ops_vector_f32_small(int K, bool has_w);
const Ops<float>* ops_vector_f32_wide(int K);
const Ops<float>* ops_vector_f32_sparse(int K);

const Ops<float>* ops_vector_f32(int K, bool has_w, int ell) {
  if (!has_w || K <= 3) return ops_vector_f32_small(K, has_w);
  if (ell >= 1 && ell <= K && K <= 8) return ops_vector_f32_sparse(K);
  const Ops<float>* o = ops_vector_f32_wide(K);
  return o ? o : ops_vector_dyn_f32(K);
}

}  // namespace otfx
