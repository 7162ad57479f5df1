// Dispatch of the scalar / vector payload instantiations (double).
#include "ops.h"

namespace otfx {

const Ops<double>* ops_vector_f64_small(int K, bool has_w);
const Ops<double>* ops_vector_f64_wide(int K);
const Ops<double>* ops_vector_f64_sparse(int K);

const Ops<double>* ops_vector_f64(int K, bool has_w, int ell) {
  if (!has_w || K <= 3) return ops_vector_f64_small(K, has_w);
  if (ell >= 1 && ell <= K && K <= 8) return ops_vector_f64_sparse(K);
  const Ops<double>* o = ops_vector_f64_wide(K);
  return o ? o : ops_vector_dyn_f64(K);
}

}  // namespace otfx
