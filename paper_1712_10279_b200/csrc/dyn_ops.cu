// Ops tables of the runtime-size payloads (dyn.cuh): graphs wider than the
// compiled vector instantiations (k > 8, up to DYN_KMAX channels and DYN_LMAX
// edges) and matrix payloads beyond the compiled (k, ell) capacities (k up to
// DYN_MKMAX, ell * block reals up to DYN_MNWMAX).  One table per (payload,
// precision, k), built on first use; the kernels read k, ell and the channel
// operator from their arguments.  No TMA ring and no cluster solve: the engine
// runs the register-sweep schedule with these kernels.
#include <map>
#include <memory>
#include <mutex>

#include "dyn.cuh"
#include "ops.h"

namespace otfx {

template <class D, typename T>
struct DynOps {
  static cudaError_t prepare() { return cudaSuccess; }
  static cudaError_t sweep(const SweepArgs<T>& a, dim3 g, dim3 b, size_t, cudaStream_t s,
                           bool check) {
    // the payload lives in local memory: no dynamic shared memory
    if (check)
      dyn_sweep_kernel<D, T, true><<<g, b, 0, s>>>(a);
    else
      dyn_sweep_kernel<D, T, false><<<g, b, 0, s>>>(a);
    return cudaGetLastError();
  }
  static cudaError_t evaluate(const SweepArgs<T>& a, dim3 g, dim3 b, cudaStream_t s) {
    dyn_evaluate_kernel<D, T><<<g, b, 0, s>>>(a);
    return cudaGetLastError();
  }
  static cudaError_t residual(const SweepArgs<T>& a, dim3 g, dim3 b, cudaStream_t s) {
    dyn_residual_kernel<D, T><<<g, b, 0, s>>>(a);
    return cudaGetLastError();
  }
  static int regs(bool check) {
    cudaFuncAttributes at;
    if (check) cudaFuncGetAttributes(&at, dyn_sweep_kernel<D, T, true>);
    else cudaFuncGetAttributes(&at, dyn_sweep_kernel<D, T, false>);
    return at.numRegs;
  }
  static int no_regs(bool) { return 0; }
  static int no_occupancy(int, size_t) { return 0; }
  static int sweep_occupancy(int threads, size_t) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dyn_sweep_kernel<D, T, false>, threads, 0);
    return nb;
  }
  static size_t no_cluster_smem(int, int) { return ~size_t(0); }
  static int no_cluster(int, int, size_t) { return 0; }

  static const Ops<T>* table(int kind, int K, int NP, int NWS, int LMAX) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<Ops<T>>> tables;
    std::lock_guard<std::mutex> lock(mu);
    auto it = tables.find(K);
    if (it != tables.end()) return it->second.get();
    auto o = std::make_unique<Ops<T>>();
    o->kind = kind;
    o->K = K;
    o->NP = NP;
    o->NWS = NWS;
    o->LMAX = LMAX;
    o->has_w = true;
    o->prepare = &prepare;
    o->sweep = &sweep;
    o->evaluate = &evaluate;
    o->residual = &residual;
    o->sweep_tma = nullptr;
    o->sweep_regs = &regs;
    o->tma_regs = &no_regs;
    o->wide_cw = 4;
    o->wide_threads = 160;
    o->narrow_threads = 160;
    o->tma_occupancy = &no_occupancy;
    o->sweep_occupancy = &sweep_occupancy;
    o->cluster_run = nullptr;
    o->cluster_smem = &no_cluster_smem;
    o->cluster_fits = &no_cluster;
    o->dynamic = true;
    return tables.emplace(K, std::move(o)).first->second.get();
  }
};

const Ops<double>* ops_vector_dyn_f64(int K) {
  return K >= 2 && K <= DYN_KMAX ? DynOps<DynVec<double>, double>::table(KIND_VECTOR, K, K, 1, DYN_LMAX)
                                 : nullptr;
}
const Ops<float>* ops_vector_dyn_f32(int K) {
  return K >= 2 && K <= DYN_KMAX ? DynOps<DynVec<float>, float>::table(KIND_VECTOR, K, K, 1, DYN_LMAX)
                                 : nullptr;
}

template <typename T>
static const Ops<T>* matrix_dyn(int kind, int K) {
  if (K < 2 || K > DYN_MKMAX) return nullptr;
  if (kind == KIND_MATRIX_REAL) {
    const int nws = K * (K - 1) / 2;
    return DynOps<DynMat<T, false>, T>::table(kind, K, K * (K + 1) / 2, nws, DYN_MNWMAX / nws);
  }
  return DynOps<DynMat<T, true>, T>::table(kind, K, K * K, K * K, DYN_MNWMAX / (K * K));
}
const Ops<double>* ops_matrix_dyn_f64(int kind, int K) { return matrix_dyn<double>(kind, K); }
const Ops<float>* ops_matrix_dyn_f32(int kind, int K) { return matrix_dyn<float>(kind, K); }

}  // namespace otfx
