// Standalone TMA probe: one 3-D box load per configuration, data checked on
// the host.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tma_probe tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../../paper_1712_10279_b200/csrc/tma.cuh"

using namespace otfx;

template <typename T>
__global__ void probe(const __grid_constant__ CUtensorMap m, int c0, int r, int bytes, T* out,
                      int n_out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  T* buf = reinterpret_cast<T*>(sm + 128);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, bytes);
    tma_load_3d(buf, &m, bar, c0, r, 0);
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < n_out; i += blockDim.x) out[i] = buf[i];
}

template <typename T>
int run(int n, int pitch, int rows, int planes, int tw, int c0) {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  size_t plane = size_t(rows) * pitch;
  std::vector<T> h(plane * planes);
  for (size_t i = 0; i < h.size(); ++i) h[i] = T(i % 100000);
  T* d;
  cudaMalloc(&d, h.size() * sizeof(T));
  cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  CUtensorMap m;
  cuuint64_t dims[3] = {cuuint64_t(n), cuuint64_t(rows), cuuint64_t(planes)};
  cuuint64_t str[2] = {cuuint64_t(pitch) * sizeof(T), cuuint64_t(plane) * sizeof(T)};
  cuuint32_t box[3] = {cuuint32_t(tw), 1u, cuuint32_t(planes)};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", int(r));
    return 1;
  }
  int nout = tw * planes;
  T* dout;
  cudaMalloc(&dout, nout * sizeof(T));
  int bytes = nout * sizeof(T);
  probe<T><<<1, 128, 128 + bytes + 128>>>(m, c0, 1, bytes, dout, nout);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("elem=%zu tw=%d planes=%d c0=%d: %s\n", sizeof(T), tw, planes, c0, cudaGetErrorString(e));
    return 2;
  }
  std::vector<T> o(nout);
  cudaMemcpy(o.data(), dout, nout * sizeof(T), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int p = 0; p < planes; ++p)
    for (int c = 0; c < tw; ++c) {
      int col = c0 + c;
      T want = (col >= 0 && col < n) ? h[p * plane + 1 * pitch + col] : T(0);
      if (o[p * tw + c] != want) ++bad;
    }
  printf("elem=%zu tw=%d planes=%d c0=%d: %s (%d bad)\n", sizeof(T), tw, planes, c0,
         bad ? "MISMATCH" : "ok", bad);
  cudaFree(d);
  cudaFree(dout);
  return bad ? 3 : 0;
}

int main(int argc, char** argv) {
  int which = argc > 1 ? atoi(argv[1]) : 0;
  switch (which) {
    case 0: return run<double>(256, 256, 8, 6, 128, -2);
    case 1: return run<float>(256, 256, 8, 6, 128, -2);
    case 2: return run<float>(256, 256, 8, 6, 128, 0);
    case 3: return run<float>(256, 256, 8, 6, 128, 2);
    case 4: return run<float>(256, 256, 8, 3, 132, 30);
    case 5: return run<double>(256, 256, 8, 3, 132, 30);
    case 6: return run<float>(256, 256, 8, 6, 64, -4);
    case 7: return run<float>(256, 256, 8, 1, 32, 0);
  }
  return 0;
}
