// Dispatch of the sparse-graph vector instantiations (edge capacity k), double.
#include "ops.h"

namespace otfx {

const Ops<double>* ops_vector_f64_sparse_k45(int K);
const Ops<double>* ops_vector_f64_sparse_k6(int K);
const Ops<double>* ops_vector_f64_sparse_k7(int K);
const Ops<double>* ops_vector_f64_sparse_k8(int K);

const Ops<double>* ops_vector_f64_sparse(int K) {
  if (K <= 5) return ops_vector_f64_sparse_k45(K);
  if (K == 6) return ops_vector_f64_sparse_k6(K);
  if (K == 7) return ops_vector_f64_sparse_k7(K);
  return ops_vector_f64_sparse_k8(K);
}

}  // namespace otfx
