// Builds an Ops<T> table entry for one payload policy.
#pragma once

#include "ops.h"
#include "sweep.cuh"
#include "sweep_tma.cuh"
#include "sweep_tb2.cuh"

namespace otfx {

template <class P, typename T>
struct OpsFor {
  static cudaError_t prepare() {
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<P, T, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(sweep_kernel<P, T, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    const void* tk[4] = {(const void*)sweep_tma_kernel<P, T, 0>, (const void*)sweep_tma_kernel<P, T, 1>,
                         (const void*)sweep_tma_kernel<P, T, 2>, (const void*)sweep_tma_kernel<P, T, 3>};
    for (int q = 0; q < 4; ++q) {
      e = cudaFuncSetAttribute(tk[q], cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (e != cudaSuccess) return e;
    }
    if constexpr (TB2) {
      return cudaFuncSetAttribute(sweep_tb2_kernel<P, T>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    }
    return cudaSuccess;
  }
  // temporal blocking is instantiated for the graph payloads with k <= 4
  // (the matrix payloads would spill the two register-resident levels)
  static constexpr bool TB2 = (P::NCOEF > 0 || !P::HAS_W) && P::K <= 4;
  static cudaError_t sweep_tb2(const TmaSweepArgs<T>& a, const TmaSet& m, dim3 g, dim3 b,
                               cudaStream_t s) {
    if constexpr (TB2) {
      sweep_tb2_kernel<P, T><<<g, b, a.L.total, s>>>(a, m);
      return cudaGetLastError();
    }
    return cudaErrorNotSupported;
  }
  static int tb2_regs() {
    if constexpr (TB2) {
      cudaFuncAttributes at;
      cudaFuncGetAttributes(&at, sweep_tb2_kernel<P, T>);
      return at.numRegs;
    }
    return 0;
  }
  static cudaError_t sweep_tma(const TmaSweepArgs<T>& a, const TmaSet& m, dim3 g, dim3 b,
                               cudaStream_t s, int fl) {
    switch (fl & 3) {
      case 0: sweep_tma_kernel<P, T, 0><<<g, b, a.L.total, s>>>(a, m); break;
      case 1: sweep_tma_kernel<P, T, 1><<<g, b, a.L.total, s>>>(a, m); break;
      case 2: sweep_tma_kernel<P, T, 2><<<g, b, a.L.total, s>>>(a, m); break;
      default: sweep_tma_kernel<P, T, 3><<<g, b, a.L.total, s>>>(a, m); break;
    }
    return cudaGetLastError();
  }
  static int tma_regs(bool check) {
    cudaFuncAttributes at;
    if (check) cudaFuncGetAttributes(&at, sweep_tma_kernel<P, T, 1>);
    else cudaFuncGetAttributes(&at, sweep_tma_kernel<P, T, 0>);
    return at.numRegs;
  }
  static cudaError_t sweep(const SweepArgs<T>& a, dim3 g, dim3 b, size_t smem, cudaStream_t s,
                           bool check) {
    if (check)
      sweep_kernel<P, T, true><<<g, b, smem, s>>>(a);
    else
      sweep_kernel<P, T, false><<<g, b, smem, s>>>(a);
    return cudaGetLastError();
  }
  static cudaError_t evaluate(const SweepArgs<T>& a, dim3 g, dim3 b, cudaStream_t s) {
    evaluate_kernel<P, T><<<g, b, 0, s>>>(a);
    return cudaGetLastError();
  }
  static cudaError_t residual(const SweepArgs<T>& a, dim3 g, dim3 b, cudaStream_t s) {
    residual_kernel<P, T><<<g, b, 0, s>>>(a);
    return cudaGetLastError();
  }
  static int regs(bool check) {
    cudaFuncAttributes at;
    if (check) cudaFuncGetAttributes(&at, sweep_kernel<P, T, true>);
    else cudaFuncGetAttributes(&at, sweep_kernel<P, T, false>);
    return at.numRegs;
  }
  static const Ops<T>* table(int kind) {
    static const Ops<T> o = {kind,     P::K,     P::NP,    P::NWS,   P::LMAX,
                             P::HAS_W, &prepare, &sweep,   &evaluate, &residual, &sweep_tma,
                             TB2 ? &sweep_tb2 : nullptr, &regs, &tma_regs, &tb2_regs};
    return &o;
  }
};

}  // namespace otfx
