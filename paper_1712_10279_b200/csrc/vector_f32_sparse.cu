// Dispatch of the sparse-graph vector instantiations (edge capacity k), float.
#include "ops.h"

namespace otfx {

const Ops<float>* ops_vector_f32_sparse_k45(int K);
const Ops<float>* ops_vector_f32_sparse_k6(int K);
const Ops<float>* ops_vector_f32_sparse_k7(int K);
const Ops<float>* ops_vector_f32_sparse_k8(int K);

const Ops<float>* ops_vector_f32_sparse(int K) {
  if (K <= 5) return ops_vector_f32_sparse_k45(K);
  if (K == 6) return ops_vector_f32_sparse_k6(K);
  if (K == 7) return ops_vector_f32_sparse_k7(K);
  return ops_vector_f32_sparse_k8(K);
}

}  // namespace otfx
