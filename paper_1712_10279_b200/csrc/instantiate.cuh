// Builds an Ops<T> table entry for one payload policy.
#pragma once

#include <utility>

#include "ops.h"
#include "sweep.cuh"
#include "sweep_tma.cuh"

namespace otfx {

// sweep launch with the programmatic-dependent-launch attribute (common.cuh
// pdl_wait): the sweep's launch and prologue overlap the previous kernel's
// tail -- the graph-node gap that dominates small grids
template <typename... KArgs, typename... Args>
static cudaError_t launch_sweep_pdl(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem,
                                    cudaStream_t s, Args&&... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

template <class P, typename T>
struct OpsFor {
  static cudaError_t prepare() {
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<P, T, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(sweep_kernel<P, T, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    const void* tk[8] = {(const void*)sweep_tma_kernel<P, T, 0, 4>, (const void*)sweep_tma_kernel<P, T, 1, 4>,
                         (const void*)sweep_tma_kernel<P, T, 2, 4>, (const void*)sweep_tma_kernel<P, T, 3, 4>,
                         (const void*)sweep_tma_kernel<P, T, 0, WIDE>, (const void*)sweep_tma_kernel<P, T, 1, WIDE>,
                         (const void*)sweep_tma_kernel<P, T, 2, WIDE>, (const void*)sweep_tma_kernel<P, T, 3, WIDE>};
    for (int q = 0; q < 8; ++q) {
      e = cudaFuncSetAttribute(tk[q], cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  // wide CTAs (8 consumer warps, 248 columns) for the graph payloads.  The
  // fp64 complex-Hermitian payloads with K >= 3 need 226-255 registers, so at
  // most 8 warps fit an SM (two per sub-partition register file): they run 8
  // consumer warps with no producer warp (the last warp to release a ring slot
  // refills it, TmaRoles) on a 2-stage ring, one CTA per SM -- 3x3 complex
  // 2048^2 0.743 -> 0.648 ms (l2/l1) / 0.662 ms (l1nuc), profiles/
  // r02_heavy_self8.md (6 consumer warps + producer before).  The other
  // matrix payloads keep 4.
  static constexpr bool HEAVY = TmaRoles<P, T, 4>::HEAVY;
#ifndef OTFX_HEAVY_CW
#define OTFX_HEAVY_CW 8
#endif
  // (Lindblad capacity 4: a 72-plane stage fits a 2-stage ring only at 6
  // consumer warps, which keep their producer warp)
  static constexpr int WIDE =
      (P::NCOEF > 0 || !P::HAS_W) ? 8 : (HEAVY ? (P::LMAX <= 2 ? OTFX_HEAVY_CW : 6) : 4);
  template <int CW>
  static void launch_tma(const TmaSweepArgs<T>& a, const TmaSet& m, dim3 g, dim3 b,
                         cudaStream_t s, int fl) {
    const size_t sm = a.L.total;
    switch (fl & 3) {
      case 0: launch_sweep_pdl(sweep_tma_kernel<P, T, 0, CW>, g, b, sm, s, a, m); break;
      case 1: launch_sweep_pdl(sweep_tma_kernel<P, T, 1, CW>, g, b, sm, s, a, m); break;
      case 2: launch_sweep_pdl(sweep_tma_kernel<P, T, 2, CW>, g, b, sm, s, a, m); break;
      default: launch_sweep_pdl(sweep_tma_kernel<P, T, 3, CW>, g, b, sm, s, a, m); break;
    }
  }
  static cudaError_t sweep_tma(const TmaSweepArgs<T>& a, const TmaSet& m, dim3 g, dim3 b,
                               cudaStream_t s, int fl) {
    if (a.L.cw == WIDE) {
      launch_tma<WIDE>(a, m, g, b, s, fl);
    } else if (a.L.cw == 4) {
      launch_tma<4>(a, m, g, b, s, fl);
    } else {
      return cudaErrorNotSupported;
    }
    return cudaGetLastError();
  }
  static int tma_regs(bool check) {
    cudaFuncAttributes at;
    if (check) cudaFuncGetAttributes(&at, sweep_tma_kernel<P, T, 1, WIDE>);
    else cudaFuncGetAttributes(&at, sweep_tma_kernel<P, T, 0, WIDE>);
    return at.numRegs;
  }
  static constexpr int wide_cw() { return WIDE; }
  static int tma_occupancy(int cw, size_t smem) {
    int nb = 0;
    if (cw == WIDE)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sweep_tma_kernel<P, T, 0, WIDE>,
                                                    TmaRoles<P, T, WIDE>::THREADS, smem);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sweep_tma_kernel<P, T, 0, 4>,
                                                    TmaRoles<P, T, 4>::THREADS, smem);
    return nb;
  }
  static int sweep_occupancy(int threads, size_t smem) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sweep_kernel<P, T, false>, threads, smem);
    return nb;
  }
  static cudaError_t sweep(const SweepArgs<T>& a, dim3 g, dim3 b, size_t smem, cudaStream_t s,
                           bool check) {
    if (check) return launch_sweep_pdl(sweep_kernel<P, T, true>, g, b, smem, s, a);
    return launch_sweep_pdl(sweep_kernel<P, T, false>, g, b, smem, s, a);
  }
  // the on-chip cluster solve is instantiated for the graph / scalar payloads
  static constexpr bool CLUSTER = (P::NCOEF > 0 || !P::HAS_W);
  static cudaLaunchConfig_t cluster_cfg(int ctas, int threads, size_t smem, cudaStream_t s,
                                        cudaLaunchAttribute* at) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ctas;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cfg;
  }
  static cudaError_t cluster_prepare() {
    if constexpr (CLUSTER) {
      cudaError_t e = cudaFuncSetAttribute(cluster_run_kernel<P, T>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (e != cudaSuccess) return e;
      return cudaFuncSetAttribute(cluster_run_kernel<P, T>,
                                  cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    return cudaSuccess;
  }
  static cudaError_t cluster_run(const ClusterArgs<T>& a, int ctas, int threads, size_t smem,
                                 cudaStream_t s) {
    if constexpr (CLUSTER) {
      cudaLaunchAttribute at[1];
      cudaLaunchConfig_t cfg = cluster_cfg(ctas, threads, smem, s, at);
      return cudaLaunchKernelEx(&cfg, cluster_run_kernel<P, T>, a);
    }
    return cudaErrorNotSupported;
  }
  static size_t cluster_smem(int rows_max, int n) { return cluster_smem_bytes<P, T>(rows_max, n); }
  static int cluster_fits(int ctas, int threads, size_t smem) {
    if constexpr (CLUSTER) {
      if (cluster_prepare() != cudaSuccess) return 0;
      cudaLaunchAttribute at[1];
      cudaLaunchConfig_t cfg = cluster_cfg(ctas, threads, smem, nullptr, at);
      int num = 0;
      if (cudaOccupancyMaxActiveClusters(&num, cluster_run_kernel<P, T>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
      }
      return num > 0 ? 1 : 0;
    }
    return 0;
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
                             &regs, &tma_regs,
                             WIDE,     TmaRoles<P, T, WIDE>::THREADS, TmaRoles<P, T, 4>::THREADS, &tma_occupancy, &sweep_occupancy,
                             CLUSTER ? &cluster_run : nullptr, &cluster_smem, &cluster_fits};
    return &o;
  }
};

}  // namespace otfx
