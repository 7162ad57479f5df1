// Host-side dispatch table: one Ops<T> per (payload policy, precision).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"
#include "sweep_tma.cuh"
#include "cluster.cuh"

namespace otfx {

template <typename T>
struct Ops {
  int kind;
  int K;      // channels / matrix dimension
  int NP;     // reals per potential (and per flux direction)
  int NWS;    // reals per channel block (edge / Lindblad matrix)
  int LMAX;   // channel-block capacity of the instantiation
  bool has_w;
  cudaError_t (*prepare)();  // raise dynamic smem limits once
  cudaError_t (*sweep)(const SweepArgs<T>& a, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       bool check);
  cudaError_t (*evaluate)(const SweepArgs<T>& a, dim3 grid, dim3 block, cudaStream_t s);
  cudaError_t (*residual)(const SweepArgs<T>& a, dim3 grid, dim3 block, cudaStream_t s);
  // fl bit 0: check sweep (R^k + primal/feasibility), bit 1: dual-norm sweep
  cudaError_t (*sweep_tma)(const TmaSweepArgs<T>& a, const TmaSet& m, dim3 grid, dim3 block,
                           cudaStream_t s, int fl);
  int (*sweep_regs)(bool check);
  int (*tma_regs)(bool check);
  int wide_cw;  // consumer warps of the wide TMA sweep instantiation (8, or 4 if none)
  int wide_threads;  // threads per CTA of the wide TMA sweep (consumers + producer warp)
  int narrow_threads;  // threads per CTA of the 4-consumer-warp TMA sweep
  // resident CTAs per SM of the plain TMA sweep at this width / shared memory
  int (*tma_occupancy)(int cw, size_t smem);
  // resident CTAs per SM of the plain register-streamed sweep
  int (*sweep_occupancy)(int threads, size_t smem);
  // on-chip solve of small grids in one thread-block cluster (graph / scalar
  // payloads; nullptr for the matrix payloads)
  cudaError_t (*cluster_run)(const ClusterArgs<T>& a, int ctas, int threads, size_t smem,
                             cudaStream_t s);
  size_t (*cluster_smem)(int rows_max, int n);
  int (*cluster_fits)(int ctas, int threads, size_t smem);  // 1 if such a cluster can launch
  // runtime-size payload (dyn.cuh): k and the graph D/c come from the kernel
  // arguments (nchan, chan_dev), no TMA sweep
  bool dynamic = false;
};

// registries, one per instantiation unit
// ell: edges of the graph (k >= 4 graphs with ell <= k take the sparse
// instantiation, edge capacity k)
const Ops<double>* ops_vector_f64(int K, bool has_w, int ell = 0);
const Ops<float>* ops_vector_f32(int K, bool has_w, int ell = 0);
const Ops<double>* ops_vector_dyn_f64(int K);  // k beyond the compiled policies
const Ops<float>* ops_vector_dyn_f32(int K);
const Ops<double>* ops_matrix_dyn_f64(int kind, int K);  // (k, ell) beyond the compiled ones
const Ops<float>* ops_matrix_dyn_f32(int kind, int K);
const Ops<double>* ops_matrix_f64(int kind, int K, int ell);
const Ops<float>* ops_matrix_f32(int kind, int K, int ell);

template <typename T>
const Ops<T>* find_ops(int kind, int K, int ell);

}  // namespace otfx
