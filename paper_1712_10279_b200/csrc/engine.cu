// Host runtime of the otfx engine: device memory, layout conversion, the
// iteration / check / run loops (CUDA graphs), halo exchange (local copies or
// NCCL over NVLink), and the extern "C" ABI of include/otfx.h.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <omp.h>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/otfx.h"
#include "ops.h"

namespace otfx {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      throw Error(e_ == cudaErrorMemoryAllocation ? OTFX_ENOMEM : OTFX_ECUDA,                 \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                        \
  } while (0)

// NVTX ranges (header-only NVTX 3: free unless a profiler attaches) around the
// host-side phases of a solve, so an nsys / ncu timeline shows the run loop,
// the check periods, the halo exchanges and the host <-> device conversions
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
  Range(const Range&) = delete;
  Range& operator=(const Range&) = delete;
};

static void require(bool ok, int code, const std::string& msg) {
  if (!ok) throw Error(code, msg);
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

template <>
const Ops<double>* find_ops<double>(int kind, int K, int ell) {
  if (kind == KIND_SCALAR) return ops_vector_f64(1, false);
  if (kind == KIND_VECTOR) return ops_vector_f64(K, true, ell);
  const Ops<double>* o = ops_matrix_f64(kind, K, ell);
  return o ? o : ops_matrix_dyn_f64(kind, K);
}
template <>
const Ops<float>* find_ops<float>(int kind, int K, int ell) {
  if (kind == KIND_SCALAR) return ops_vector_f32(1, false);
  if (kind == KIND_VECTOR) return ops_vector_f32(K, true, ell);
  const Ops<float>* o = ops_matrix_f32(kind, K, ell);
  return o ? o : ops_matrix_dyn_f32(kind, K);
}

// ---------------------------------------------------------------------------
// NCCL, loaded at run time so the library has no hard NCCL dependency
// ---------------------------------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  if (api.h) return api;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    api.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL);  // reuses an already-loaded copy (torch)
    if (api.h) break;
  }
  require(api.h != nullptr, OTFX_ENCCL, "NCCL library (libnccl.so.2) not found");
#define SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(api.h, name))
  SYM(GetUniqueId, "ncclGetUniqueId");
  SYM(CommInitRank, "ncclCommInitRank");
  SYM(CommDestroy, "ncclCommDestroy");
  SYM(Send, "ncclSend");
  SYM(Recv, "ncclRecv");
  SYM(AllReduce, "ncclAllReduce");
  SYM(GroupStart, "ncclGroupStart");
  SYM(GroupEnd, "ncclGroupEnd");
  SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
  require(api.GetUniqueId && api.CommInitRank && api.Send && api.Recv && api.AllReduce &&
              api.GroupStart && api.GroupEnd,
          OTFX_ENCCL, "NCCL library lacks required symbols");
  return api;
}

#define NK(call)                                                                        \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      throw Error(OTFX_ENCCL, std::string(#call) + ": " +                               \
                                  (nccl().GetErrorString ? nccl().GetErrorString(r_) : "")); \
  } while (0)

// ---------------------------------------------------------------------------
// layout conversion kernels (reference AoS <-> device planes)
// ---------------------------------------------------------------------------
// record reals of one cell: up to the runtime-size matrix payload's w record
// (real path ell * k^2 <= 1024 at k = 2, complex 2 * ell * k^2 <= 512)
constexpr int MAXMAP = 1024;

struct PackMap {
  int np;                 // planes written
  int rec;                // doubles per cell record in the source
  int src[MAXMAP];        // record index per plane (-1: zero)
  double wt[MAXMAP];      // plane weight for the sum of squares
  int nmass;              // record indices summed into the mass
  int mass[64];            // (up to DYN_KMAX channels)
};

struct UnpackMap {
  int rec;                // doubles per cell record in the destination
  int plane[MAXMAP];      // source plane per record element (-1: zero)
  signed char sign[MAXMAP];
};

// planes[p] = T(src0[rec*cell + map] (- src1[...])), rows [0, nrows) of the chunk
// written to local rows lrow0 + r.  Per-block partials: mass0, mass1, sumsq.
template <typename T>
__global__ void pack_kernel(const double* __restrict__ s0, const double* __restrict__ s1,
                            int64_t ncell, int n, T* planes, int64_t plane, int pitch, int lrow0,
                            const __grid_constant__ PackMap m, double* part) {
  __shared__ double sred[32 * 3];
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < ncell;
       c += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(c / n), j = int(c % n);
    const double* a = s0 + c * m.rec;
    const double* b = s1 ? s1 + c * m.rec : nullptr;
    const int64_t o = int64_t(lrow0 + r) * pitch + j;
    for (int p = 0; p < m.np; ++p) {
      double v = 0.0;
      if (m.src[p] >= 0) v = b ? (a[m.src[p]] - b[m.src[p]]) : a[m.src[p]];
      planes[p * plane + o] = T(v);
      acc[2] += m.wt[p] * v * v;
    }
    for (int q = 0; q < m.nmass; ++q) {
      acc[0] += a[m.mass[q]];
      if (b) acc[1] += b[m.mass[q]];
    }
  }
  block_sum<3>(acc, sred);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 3 + 0] = acc[0];
    part[blockIdx.x * 3 + 1] = acc[1];
    part[blockIdx.x * 3 + 2] = acc[2];
  }
}

template <typename T>
__global__ void unpack_kernel(const T* __restrict__ planes, int64_t plane, int pitch, int lrow0,
                              int64_t ncell, int n, const __grid_constant__ UnpackMap m,
                              double* dst) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < ncell;
       c += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(c / n), j = int(c % n);
    const int64_t o = int64_t(lrow0 + r) * pitch + j;
    double* d = dst + c * m.rec;
    for (int q = 0; q < m.rec; ++q) {
      const int p = m.plane[q];
      d[q] = p >= 0 ? double(m.sign[q]) * double(planes[p * plane + o]) : 0.0;
    }
  }
}

// Deterministic final reduction of the per-block partials into raw[OTFX_NRAW].
__global__ void reduce_raw_kernel(const double* __restrict__ pe, const double* __restrict__ me,
                                  int nbe, const double* __restrict__ ps, int nbs, int with_res,
                                  double* raw) {
  __shared__ double sred[32 * 14];
  double v[14];
  for (int q = 0; q < 14; ++q) v[q] = 0.0;
  for (int b = threadIdx.x; b < nbe; b += blockDim.x) {
    for (int q = 0; q < 8; ++q) v[q] += pe[b * 8 + q];
  }
  if (with_res) {
    for (int b = threadIdx.x; b < nbs; b += blockDim.x) {
      for (int q = 0; q < 4; ++q) v[8 + q] += ps[b * 10 + q];
    }
  }
  double mx[2] = {0.0, 0.0};
  for (int b = threadIdx.x; b < nbe; b += blockDim.x) {
    mx[0] = dmax(mx[0], me[b * 2]);
    mx[1] = dmax(mx[1], me[b * 2 + 1]);
  }
  double s12[12];
  for (int q = 0; q < 12; ++q) s12[q] = v[q];
  block_sum<12>(s12, sred);
  block_max<2>(mx, sred);
  if (threadIdx.x == 0) {
    for (int q = 0; q < 12; ++q) raw[q] = s12[q];
    raw[R_GU] = mx[0];
    raw[R_GW] = mx[1];
  }
}

// Fused check: R^k partials of the check sweep ([nb][10], slots 0..3) and the
// evaluate partials of the following sweep ([nb][10]: PU PW SU2 SW2 SCON SPHID
// PENU PENW | GU GW), reduced in block order.
__global__ void reduce_fused_kernel(const double* __restrict__ pc, const double* __restrict__ pd,
                                    int nb, double* raw) {
  __shared__ double sred[32 * 12];
  double v[12], mx[2] = {0.0, 0.0};
  for (int q = 0; q < 12; ++q) v[q] = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const double* c = pc + size_t(b) * 10;
    const double* d = pd + size_t(b) * 10;
    v[R_SDU] += c[0];
    v[R_SDW] += c[1];
    v[R_SDPHI] += c[2];
    v[R_SCROSS] += c[3];
    v[R_PU] += d[0];
    v[R_PW] += d[1];
    v[R_SU2] += d[2];
    v[R_SW2] += d[3];
    v[R_SCON] += d[4];
    v[R_SPHID] += d[5];
    v[R_PENU] += d[6];
    v[R_PENW] += d[7];
    mx[0] = dmax(mx[0], d[8]);
    mx[1] = dmax(mx[1], d[9]);
  }
  block_sum<12>(v, sred);
  block_max<2>(mx, sred);
  if (threadIdx.x == 0) {
    for (int q = 0; q < 12; ++q) raw[q] = v[q];
    raw[R_GU] = mx[0];
    raw[R_GW] = mx[1];
  }
}

// ---------------------------------------------------------------------------
// the engine
// ---------------------------------------------------------------------------
constexpr int kPackBlocks = 296;

}  // namespace otfx

struct otfx_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
};

struct otfx_engine {
  otfx_engine_desc d{};
  std::vector<double> chan;
  int elem = 8;
  int K = 1, NP = 1, NWS = 0, LMAX = 0, NWact = 0;
  bool has_w = false;
  int rows = 0, rows_alloc = 0, pitch = 0;
  int64_t plane = 0;
  size_t state_bytes = 0, total_bytes = 0;
  unsigned char* mem = nullptr;
  bool pooled = false;  // mem came from the library's device pool
  void* u[2]{};
  void* w[2]{};
  void* phi[2]{};
  void* diff = nullptr;
  int cur = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // sweep geometry
  int TX = 128, R = 64, gx = 1, gy = 1;
  size_t smem_plain = 0, smem_check = 0;
  // reductions
  double* d_part_sweep = nullptr;  // [gx*gy][10] check-sweep partials
  double* d_part_dual = nullptr;   // [gx*gy][10] dual-sweep partials
  double* d_part_eval = nullptr;   // [ex*ey][8]
  double* d_max_eval = nullptr;    // [ex*ey][2]
  double* d_raw = nullptr;         // [OTFX_NRAW]
  double* h_raw = nullptr;         // pinned
  int ex = 1, ey = 1;
  bool residual_valid = false;
  double diff_norm = 0.0;       // ||diff|| of the whole grid (allreduced across ranks)
  double diff_norm_own = 0.0;   // ||diff|| of this slab's own rows
  // staging for host <-> device conversions
  double* d_stage = nullptr;
  size_t stage_bytes = 0;
  double* d_pack_part = nullptr;
  double* h_pack_part = nullptr;
  // device-side timing of the plain-iteration graphs (for the bench roofline)
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
  std::vector<std::pair<int, int64_t>> ev_pending;  // (pool index, sweeps)
  double plain_ms = 0.0;
  int64_t plain_sweeps = 0;
  // graphs
  bool use_graphs = true;
  std::map<std::pair<int, int64_t>, cudaGraphExec_t> graphs;
  // NCCL
  ncclComm_t comm = nullptr;
  bool own_comm = false;  // created by attach_nccl (destroyed with the engine)
  int nranks = 1, rank = 0;
  void* d_halo = nullptr;  // send/recv buffers
  // overlapped halo exchange: edge bands + exchange on a high-priority stream
  cudaStream_t edge_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_hand = nullptr;  // caller-stream ordering of the device hand-off
  // TMA-streamed sweep
  bool use_tma = false;
  bool narrow = false;  // 4 consumer warps although the payload has a wide instantiation
  // history of the last run() (the caller's buffer may be smaller: it gets
  // the first `capacity` rows, otfx_engine_history returns all of them)
  std::vector<otfx_history_point> history;
  otfx::StageLayout L{};
  otfx::TmaSet maps[2];
  // on-chip cluster solve (small single-slab grids)
  bool use_cluster = false;
  int cl_ctas = 0, cl_threads = 0, cl_rows = 0;
  size_t cl_smem = 0;
  long long* d_result = nullptr;  // [4] iterations, history points, converged
  // policy dispatch
  const otfx::Ops<double>* ops64 = nullptr;
  const otfx::Ops<float>* ops32 = nullptr;
  // the channel operator in device memory (runtime-size payloads, dyn.cuh)
  double* d_chan = nullptr;
  // device-side run loop (run_loop_device): loop control block
  void* d_loop = nullptr;
  bool dynamic() const { return ops64 ? ops64->dynamic : (ops32 && ops32->dynamic); }
};

namespace otfx {

static int pair_index_rt(int K, int a, int b) { return a * K - a * (a + 1) / 2 + (b - a - 1); }

template <typename T>
static SweepArgs<T> make_args(otfx_engine* e, int from) {
  SweepArgs<T> a;
  memset(&a, 0, sizeof(a));
  const int to = from ^ 1;
  a.a = {static_cast<T*>(e->u[from]), static_cast<T*>(e->w[from]), static_cast<T*>(e->phi[from])};
  a.b = {static_cast<T*>(e->u[to]), static_cast<T*>(e->w[to]), static_cast<T*>(e->phi[to])};
  a.diff = static_cast<const T*>(e->diff);
  a.plane = e->plane;
  a.pitch = e->pitch;
  a.n = e->d.n;
  a.row_begin = e->d.row_begin;
  a.row_end = e->d.row_end;
  a.rows_per_block = e->R;
  a.band0 = 0;
  a.band_step = 1;
  a.ell = e->d.ell;
  a.norm_u = e->d.norm_u;
  a.norm_w = e->d.norm_w;
  const double mu = e->d.mu, nu = e->d.nu, alpha = e->d.alpha, eps = e->d.eps_reg;
  const double thr_w = alpha * nu;  // S/solver.py:213
  a.mu = T(mu);
  a.nu = T(nu);
  a.thr_w = T(thr_w);
  a.tau = T(e->d.tau);
  a.inv_dx = T(e->d.inv_dx);
  a.has_eps = eps > 0 ? 1 : 0;
  // S/shrink.py:240 divides by (1 + 2 mu eps); w uses eps/alpha (S/solver.py:215-217)
  a.den_u = T(eps > 0 ? 1.0 + 2.0 * mu * eps : 1.0);
  a.den_w = T(eps > 0 ? 1.0 + 2.0 * thr_w * (eps / alpha) : 1.0);
  a.alpha = alpha;
  a.eps = eps;
  a.partials = e->d_part_sweep;
  a.maxes = nullptr;
  a.dualp = e->d_part_dual;
  const int K = e->K;
  a.nchan = K;
  a.chan_dev = e->d_chan;
  if (e->dynamic()) {
    // the kernels read the graph from d_chan
  } else if (e->d.kind == OTFX_KIND_VECTOR) {
    const int L = e->LMAX;
    for (int c = 0; c < K; ++c)
      for (int q = 0; q < e->d.ell; ++q) a.coef[c * L + q] = e->chan[size_t(c) * e->d.ell + q];
  } else if (e->d.kind != OTFX_KIND_SCALAR) {
    for (size_t q = 0; q < e->chan.size(); ++q) a.coef[q] = e->chan[q];
    if (e->d.kind == OTFX_KIND_MATRIX_COMPLEX) {
      // real Lindblad stacks (the DTI and Pauli-x sets) skip the imaginary
      // multiply-adds of the commutators (HermPolicy lmac / macl)
      a.real_l = env_int("OTFX_REAL_L", 1) != 0 ? 1 : 0;
      for (size_t q = 1; q < e->chan.size(); q += 2)
        if (e->chan[q] != 0.0) a.real_l = 0;
    }
  }
  return a;
}

template <typename T>
static const Ops<T>* ops_of(otfx_engine* e);
template <>
const Ops<double>* ops_of<double>(otfx_engine* e) { return e->ops64; }
template <>
const Ops<float>* ops_of<float>(otfx_engine* e) { return e->ops32; }

// threads per TMA sweep CTA: the 4-warp instantiation has a producer warp;
// the wide one says (TmaRoles)
static int tma_threads(const otfx_engine* e) {
  const int wide = e->ops64 ? e->ops64->wide_cw : e->ops32->wide_cw;
  if (e->L.cw != wide) return e->ops64 ? e->ops64->narrow_threads : e->ops32->narrow_threads;
  return e->ops64 ? e->ops64->wide_threads : e->ops32->wide_threads;
}

// fl bit 0: check sweep; bit 1: dual-norm accumulation (TMA sweep only).
// One launch over nb bands (band0, band0 + step, ...) of the slab on stream s;
// the iterate index is not advanced.
template <typename T>
static void launch_bands(otfx_engine* e, int fl, int band0, int step, int nb, cudaStream_t s) {
  if (e->use_tma) {
    TmaSweepArgs<T> g;
    g.s = make_args<T>(e, e->cur);
    g.s.band0 = band0;
    g.s.band_step = step;
    g.L = e->L;
    CK(ops_of<T>(e)->sweep_tma(g, e->maps[e->cur], dim3(e->gx, nb), dim3(tma_threads(e)), s,
                               fl));
  } else {
    require((fl & 2) == 0, OTFX_EINVAL, "dual accumulation needs the TMA sweep");
    const bool check = (fl & 1) != 0;
    SweepArgs<T> a = make_args<T>(e, e->cur);
    a.band0 = band0;
    a.band_step = step;
    CK(ops_of<T>(e)->sweep(a, dim3(e->gx, nb), dim3(e->TX),
                           check ? e->smem_check : e->smem_plain, s, check));
  }
}

static void launch_bands(otfx_engine* e, int fl, int band0, int step, int nb, cudaStream_t s) {
  if (e->elem == 8) launch_bands<double>(e, fl, band0, step, nb, s);
  else launch_bands<float>(e, fl, band0, step, nb, s);
}

template <typename T>
static void launch_sweep(otfx_engine* e, int fl) {
  launch_bands<T>(e, fl, 0, 1, e->gy, e->stream);
  e->cur ^= 1;
}

// ---- TMA descriptors ------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    require(q == cudaDriverEntryPointSuccess && p != nullptr, OTFX_ECUDA,
            "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D view (cols = n, rows = rows_alloc, planes) of a group of planes; one box
// = L.tw columns x 1 row x all planes; columns outside [0, n) read as zero
static void make_map(otfx_engine* e, CUtensorMap* m, void* base, int planes, int tw) {
  memset(m, 0, sizeof(*m));
  if (planes <= 0) return;
  require(planes <= 256, OTFX_EUNSUPPORTED, "too many planes for one TMA box");
  cuuint64_t dims[3] = {cuuint64_t(e->d.n), cuuint64_t(e->rows_alloc), cuuint64_t(planes)};
  cuuint64_t strides[2] = {cuuint64_t(e->pitch) * e->elem, cuuint64_t(e->plane) * e->elem};
  cuuint32_t box[3] = {cuuint32_t(tw), 1u, cuuint32_t(planes)};
  cuuint32_t es[3] = {1u, 1u, 1u};
  CUresult r = tensor_map_encoder()(
      m, e->elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base,
      dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, OTFX_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

static int round_up(int x, int a) { return (x + a - 1) / a * a; }

// shared-memory plan of the TMA sweep; returns false when it cannot fit
static bool plan_stages(otfx_engine* e, int S) {
  StageLayout& L = e->L;
  // consumer warps per CTA: the payload's wide instantiation (8 warps, 248
  // columns, half the halo re-reads, for graph payloads; 8 without a
  // producer warp for the heavy complex matrices, 6 + producer at Lindblad
  // capacity 4), else 4; OTFX_TMA_WARPS=4 overrides.  31 * cw columns of fp64
  // must stay a multiple of 16 bytes (TMA box starts): cw even.
  const int wide = e->ops64 ? e->ops64->wide_cw : e->ops32->wide_cw;
  L.cw = (!e->narrow && env_int("OTFX_TMA_WARPS", wide) == wide) ? wide : 4;
  // the consumers hold stages q and q+1, so 2 is the minimum ring; only the
  // 8-warp heavy payloads use it (their stage is released before the W half
  // of the row, whose eigensolves cover the next load)
  require(S >= 2 && S <= 8, OTFX_EINVAL, "TMA ring depth out of range");
  L.tile = 31 * L.cw;  // a multiple of 16 bytes' worth of columns for fp32 and fp64
  L.h = 16 / e->elem;
  L.tw = round_up(L.tile + 2 * L.h, L.h);  // = StageShape::TW
  L.S = S;
  const int row = L.tw * e->elem;
  const int bu = 2 * e->NP * row, bw = e->NWact * row, bd = e->NP * row, bp = e->NP * row;
  // same layout as StageShape<P,T> (w sub-block sized for the policy capacity)
  const int nwcap = e->has_w ? e->LMAX * e->NWS : 1;
  L.off_w = round_up(bu, 128);
  L.off_d = L.off_w + round_up(nwcap * row, 128);
  L.off_p = L.off_d + round_up(bd, 128);
  L.stage_bytes = L.off_p + round_up(bp, 128);
  L.bytes_full = bu + bw + bd + bp;
  L.bytes_flux = bu + bp;
  L.bytes_phi = bp;
  L.off_stages = 128;
  L.off_xchg = L.off_stages + S * L.stage_bytes;
  L.off_red = round_up(L.off_xchg, 16);
  L.total = L.off_red + 32 * 10 * 8;
  return L.total <= 227 * 1024;
}

static void launch_sweep(otfx_engine* e, int fl) {
  if (e->elem == 8) launch_sweep<double>(e, fl);
  else launch_sweep<float>(e, fl);
}

template <typename T>
static void launch_evaluate(otfx_engine* e) {
  SweepArgs<T> a = make_args<T>(e, e->cur);
  a.partials = e->d_part_eval;
  a.maxes = e->d_max_eval;
  CK(ops_of<T>(e)->evaluate(a, dim3(e->ex, e->ey), dim3(128), e->stream));
}

static void launch_evaluate(otfx_engine* e) {
  if (e->elem == 8) launch_evaluate<double>(e);
  else launch_evaluate<float>(e);
}

// ---- halo exchange: pack -> transport -> unpack ----------------------------
// One layout for every transport.  e->d_halo holds four contiguous buffers of
// n-element rows ([row][n], the planes of one grid row stacked):
//   send_top  NP rows   phi of the first owned row          -> previous slab
//   send_bot  3NP rows  phi, u (2NP planes) of the last row  -> next slab
//   recv_top  3NP rows  <- previous slab's send_bot  (unpacked into local row 0)
//   recv_bot  NP rows   <- next slab's send_top      (unpacked into row rows+1)
// Rows [0, rows+1] of a slab: 0 and rows+1 are the ghost rows the stencils
// read (S/spatial.py:30-37 needs ubar_x(i-1); S/spatial.py:80-86 phi(i+1)).
// pack/unpack are one kernel each; the transport is NCCL send/recv between
// ranks (exchange_nccl) or device copies between the slabs of one process
// (exchange_local_impl), so the single-GPU slab groups run the exact buffer
// layout and kernels the NCCL ranks run.
struct RowSeg {
  const char* src;
  char* dst;
  long long src_stride, dst_stride;  // bytes between consecutive planes / rows
  int planes;
};
struct RowSegs {
  RowSeg s[3];
  int nseg = 0;
  int planes = 0;  // total
};

template <typename W>
__global__ void row_copy_kernel(const __grid_constant__ RowSegs m, int n) {
  int p = blockIdx.y, q = 0;
  while (q + 1 < m.nseg && p >= m.s[q].planes) p -= m.s[q++].planes;
  const W* src = reinterpret_cast<const W*>(m.s[q].src + p * m.s[q].src_stride);
  W* dst = reinterpret_cast<W*>(m.s[q].dst + p * m.s[q].dst_stride);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    dst[j] = src[j];
}

struct HaloBufs {
  char *send_top, *send_bot, *recv_top, *recv_bot;
};

static HaloBufs halo_bufs(const otfx_engine* e) {
  const size_t wb = size_t(e->d.n) * e->elem;
  char* b = static_cast<char*>(e->d_halo);
  HaloBufs h;
  h.send_top = b;
  h.send_bot = h.send_top + e->NP * wb;
  h.recv_top = h.send_bot + 3 * e->NP * wb;
  h.recv_bot = h.recv_top + 3 * e->NP * wb;
  return h;
}

static void add_seg(RowSegs& m, const void* src, long long ss, void* dst, long long ds, int planes) {
  m.s[m.nseg++] = {static_cast<const char*>(src), static_cast<char*>(dst), ss, ds, planes};
  m.planes += planes;
}

static void launch_row_copy(const otfx_engine* e, const RowSegs& m, cudaStream_t st) {
  if (!m.planes) return;
  const int n = e->d.n;
  dim3 grid(std::min((n + 255) / 256, 16), m.planes);
  if (e->elem == 8) row_copy_kernel<double><<<grid, 256, 0, st>>>(m, n);
  else row_copy_kernel<float><<<grid, 256, 0, st>>>(m, n);
  CK(cudaGetLastError());
}

static char* row_of(const otfx_engine* e, void* base, int lrow) {
  return static_cast<char*>(base) + size_t(lrow) * e->pitch * e->elem;
}

// boundary rows of the current iterate -> send buffers
static void halo_pack(const otfx_engine* e, bool has_prev, bool has_next, cudaStream_t st) {
  const HaloBufs h = halo_bufs(e);
  const long long pb = (long long)e->plane * e->elem, wb = (long long)e->d.n * e->elem;
  const int c = e->cur, NP = e->NP;
  RowSegs m;
  if (has_prev) add_seg(m, row_of(e, e->phi[c], 1), pb, h.send_top, wb, NP);
  if (has_next) {
    add_seg(m, row_of(e, e->phi[c], e->rows), pb, h.send_bot, wb, NP);
    add_seg(m, row_of(e, e->u[c], e->rows), pb, h.send_bot + NP * wb, wb, 2 * NP);
  }
  launch_row_copy(e, m, st);
}

// receive buffers -> ghost rows of the current iterate
static void halo_unpack(const otfx_engine* e, bool has_prev, bool has_next, cudaStream_t st) {
  const HaloBufs h = halo_bufs(e);
  const long long pb = (long long)e->plane * e->elem, wb = (long long)e->d.n * e->elem;
  const int c = e->cur, NP = e->NP;
  RowSegs m;
  if (has_prev) {
    add_seg(m, h.recv_top, wb, row_of(e, e->phi[c], 0), pb, NP);
    add_seg(m, h.recv_top + NP * wb, wb, row_of(e, e->u[c], 0), pb, 2 * NP);
  }
  if (has_next) add_seg(m, h.recv_bot, wb, row_of(e, e->phi[c], e->rows + 1), pb, NP);
  launch_row_copy(e, m, st);
}

static void exchange_nccl(otfx_engine* e, cudaStream_t st) {
  if (!e->comm || e->nranks == 1) return;
  Range nv("otfx.halo_exchange_nccl");
  NcclApi& N = nccl();
  const bool has_prev = e->rank > 0, has_next = e->rank + 1 < e->nranks;
  const size_t w = size_t(e->d.n);
  const int NP = e->NP;
  const HaloBufs h = halo_bufs(e);
  halo_pack(e, has_prev, has_next, st);
  const ncclDataType_t dt = e->elem == 8 ? ncclFloat64 : ncclFloat32;
  NK(N.GroupStart());
  if (has_prev) {
    NK(N.Send(h.send_top, NP * w, dt, e->rank - 1, e->comm, st));
    NK(N.Recv(h.recv_top, 3 * NP * w, dt, e->rank - 1, e->comm, st));
  }
  if (has_next) {
    NK(N.Send(h.send_bot, 3 * NP * w, dt, e->rank + 1, e->comm, st));
    NK(N.Recv(h.recv_bot, NP * w, dt, e->rank + 1, e->comm, st));
  }
  NK(N.GroupEnd());
  halo_unpack(e, has_prev, has_next, st);
}

static void exchange_nccl(otfx_engine* e) { exchange_nccl(e, e->stream); }

// ---- halo exchange overlapped with the interior -------------------------------
// Every iteration of a decomposed slab: the two edge bands (first and last
// row band, which produce the rows the neighbours need and read the ghost
// rows) run on a high-priority edge stream, followed there by the halo
// exchange; the interior bands run concurrently on the engine stream.  Both
// halves read iterate k and write disjoint rows of iterate k+1; the exchange
// reads the edge bands' boundary rows of k+1 and writes its ghost rows, which
// no interior band touches.  The engine stream then joins the edge stream, so
// the exchange of iteration k is hidden behind the interior of iteration k.
static bool overlap_ready(const otfx_engine* e) {
  return e->gy >= 3 && env_int("OTFX_OVERLAP", 1) != 0;
}

static void ensure_overlap(otfx_engine* e) {
  if (e->edge_stream) return;
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CK(cudaStreamCreateWithPriority(&e->edge_stream, cudaStreamNonBlocking, hi));
  CK(cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming));
}

// one overlapped iteration of the engines es[0..count) (one rank's slab, or a
// local group sharing es[0]'s stream); `exchange` runs on the edge stream
template <class X>
static void overlapped_sweep(otfx_engine* const* es, int count, int fl, X&& exchange) {
  otfx_engine* L = es[0];
  ensure_overlap(L);
  CK(cudaEventRecord(L->ev_fork, L->stream));
  CK(cudaStreamWaitEvent(L->edge_stream, L->ev_fork, 0));
  for (int q = 0; q < count; ++q) launch_bands(es[q], fl, 0, es[q]->gy - 1, 2, L->edge_stream);
  for (int q = 0; q < count; ++q) launch_bands(es[q], fl, 1, 1, es[q]->gy - 2, L->stream);
  for (int q = 0; q < count; ++q) es[q]->cur ^= 1;
  exchange(L->edge_stream);
  CK(cudaEventRecord(L->ev_join, L->edge_stream));
  CK(cudaStreamWaitEvent(L->stream, L->ev_join, 0));
}

// one iteration of a rank's slab followed by its halo exchange
static void sweep_exchange(otfx_engine* e, int fl) {
  if (e->comm && e->nranks > 1 && overlap_ready(e)) {
    otfx_engine* const one[1] = {e};
    overlapped_sweep(one, 1, fl, [&](cudaStream_t st) { exchange_nccl(e, st); });
    return;
  }
  launch_sweep(e, fl);
  exchange_nccl(e);
}

static void enqueue_plain(otfx_engine* e, int64_t count) {
  for (int64_t q = 0; q < count; ++q) sweep_exchange(e, 0);
}

// device-time bracket (CUDA events on the engine stream) around a run of
// plain iterations, folded into plain_ms by collect_timing
static int timing_begin(otfx_engine* e) {
  if (!e->timing) return -1;
  const int slot = int(e->ev_pending.size());
  while (int(e->ev_pool.size()) <= slot) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    e->ev_pool.emplace_back(a, b);
  }
  CK(cudaEventRecord(e->ev_pool[slot].first, e->stream));
  return slot;
}

static void timing_end(otfx_engine* e, int slot, int64_t count) {
  if (slot < 0) return;
  CK(cudaEventRecord(e->ev_pool[slot].second, e->stream));
  e->ev_pending.emplace_back(slot, count);
}

static void run_plain(otfx_engine* e, int64_t count) {
  if (count <= 0) return;
  Range nv("otfx.plain_iterations");
  // NCCL halo exchanges stay outside graph capture unless explicitly enabled
  const bool graphs = e->use_graphs && (e->nranks == 1 || env_int("OTFX_NCCL_GRAPHS", 0) != 0);
  if (!graphs || count < 3) {
    // (timed too: a decomposed slab runs here, its iterations including the
    // overlapped halo exchange)
    const int slot = timing_begin(e);
    enqueue_plain(e, count);
    timing_end(e, slot, count);
    return;
  }
  auto key = std::make_pair(e->cur, count);
  auto it = e->graphs.find(key);
  if (it == e->graphs.end()) {
    const int saved = e->cur;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_plain(e, count);
    } catch (...) {
      cudaStreamEndCapture(e->stream, &g);
      e->cur = saved;
      throw;
    }
    CK(cudaStreamEndCapture(e->stream, &g));
    e->cur = saved;
    cudaGraphExec_t ge;
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    it = e->graphs.emplace(key, ge).first;
  }
  const int slot = timing_begin(e);
  CK(cudaGraphLaunch(it->second, e->stream));
  timing_end(e, slot, count);
  e->cur ^= int(count & 1);
}

// fold the timed graph launches into plain_ms once the stream has caught up
static void collect_timing(otfx_engine* e) {
  for (auto& pr : e->ev_pending) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e->ev_pool[pr.first].first, e->ev_pool[pr.first].second));
    e->plain_ms += ms;
    e->plain_sweeps += pr.second;
  }
  e->ev_pending.clear();
}

// SUM over the 12 sums, MAX over the two dual-norm maxima of d_raw, across
// the ranks of `comm` (the engine's own communicator, or for a local slab
// group the one-rank loopback communicator that exercises the same calls)
static void allreduce_raw(otfx_engine* e, ncclComm_t comm) {
  if (!comm) return;
  NcclApi& N = nccl();
  NK(N.GroupStart());
  NK(N.AllReduce(e->d_raw, e->d_raw, OTFX_NRAW_SUM, ncclFloat64, ncclSum, comm, e->stream));
  NK(N.AllReduce(e->d_raw + OTFX_NRAW_SUM, e->d_raw + OTFX_NRAW_SUM, OTFX_NRAW - OTFX_NRAW_SUM,
                 ncclFloat64, ncclMax, comm, e->stream));
  NK(N.GroupEnd());
}

static ncclComm_t rank_comm(const otfx_engine* e) {
  return e->comm && e->nranks > 1 ? e->comm : nullptr;
}

static void raw_download(otfx_engine* e) {
  CK(cudaMemcpyAsync(e->h_raw, e->d_raw, OTFX_NRAW * sizeof(double), cudaMemcpyDeviceToHost,
                     e->stream));
  CK(cudaStreamSynchronize(e->stream));
  collect_timing(e);
}

// raw scalars of the current iterate into d_raw (and h_raw after sync),
// allreduced over `ar` (nullptr: this engine's rows only)
static void raw_to_host(otfx_engine* e, bool with_res, ncclComm_t ar) {
  launch_evaluate(e);
  reduce_raw_kernel<<<1, 256, 0, e->stream>>>(e->d_part_eval, e->d_max_eval, e->ex * e->ey,
                                               e->d_part_sweep, e->gx * e->gy, with_res ? 1 : 0,
                                               e->d_raw);
  CK(cudaGetLastError());
  allreduce_raw(e, ar);
  raw_download(e);
}

// fused check: the check sweep already wrote R^k + primal/feasibility
// partials, the speculative sweep after it the dual-norm partials
static void raw_fused_to_host(otfx_engine* e, ncclComm_t ar) {
  reduce_fused_kernel<<<1, 256, 0, e->stream>>>(e->d_part_sweep, e->d_part_dual, e->gx * e->gy,
                                                 e->d_raw);
  CK(cudaGetLastError());
  allreduce_raw(e, ar);
  raw_download(e);
}

// ---- device memory pool ------------------------------------------------------
static std::mutex g_pool_mu;
static std::map<int, cudaMemPool_t> g_pools;

static cudaMemPool_t device_pool(int device) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  auto it = g_pools.find(device);
  if (it != g_pools.end()) return it->second;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  cudaMemPool_t pool;
  CK(cudaMemPoolCreate(&pool, &props));
  uint64_t keep = UINT64_MAX;
  CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  g_pools.emplace(device, pool);
  return pool;
}

// ---- on-chip cluster solve --------------------------------------------------
static bool cluster_ok(const otfx_engine* e) { return e->use_cluster && e->nranks == 1; }

template <typename T>
static void launch_cluster(otfx_engine* e, const otfx_run_config* cfg, int64_t plain_iters) {
  ClusterArgs<T> g;
  memset(&g, 0, sizeof(g));
  g.s = make_args<T>(e, e->cur);
  g.tol_gap = cfg ? cfg->tol_gap : 0.0;
  g.tol_feas = cfg ? cfg->tol_feas : 0.0;
  g.diff_norm = e->diff_norm;
  g.mu = e->d.mu;
  g.nu = e->d.nu;
  g.tau = e->d.tau;
  g.max_iters = cfg ? cfg->max_iters : plain_iters;
  g.check_every = cfg ? cfg->check_every : 1;
  g.checks = cfg ? 1 : 0;
  g.ctas = e->cl_ctas;
  g.rows_max = e->cl_rows;
  g.has_w = e->has_w ? 1 : 0;
  g.hist = e->d_stage;
  g.hist_cap = (long long)(e->stage_bytes / (6 * sizeof(double)));
  g.result = e->d_result;
  CK(ops_of<T>(e)->cluster_run(g, e->cl_ctas, e->cl_threads, e->cl_smem, e->stream));
}

static void launch_cluster(otfx_engine* e, const otfx_run_config* cfg, int64_t plain_iters) {
  if (e->elem == 8) launch_cluster<double>(e, cfg, plain_iters);
  else launch_cluster<float>(e, cfg, plain_iters);
}

// S/solver.py:242-291 scalar algebra, same operation order
static void finalize(const otfx_engine* e, const double* raw, double out[5], double diff_norm);
static void finalize(const otfx_engine* e, const double* raw, double out[5]) {
  finalize(e, raw, out, e->diff_norm);
}
static void finalize(const otfx_engine* e, const double* raw, double out[5], double diff_norm) {
  const bool has_w = e->has_w;
  const double alpha = e->d.alpha, eps = e->d.eps_reg;
  double p = raw[R_PU];
  if (has_w) p += alpha * raw[R_PW];
  if (eps > 0) {
    p += eps * raw[R_SU2];
    if (has_w) p += eps * raw[R_SW2];
  }
  const double rawd = -raw[R_SPHID];
  double dual;
  if (eps == 0) {
    double s = std::max(1.0, raw[R_GU]);
    if (has_w) s = std::max(s, raw[R_GW] / alpha);
    dual = rawd / s;
  } else {
    double pen = raw[R_PENU] / (4.0 * eps);
    if (has_w) pen += raw[R_PENW] / (4.0 * eps);
    dual = rawd - pen;
  }
  const double gap = (p - dual) / std::max(p, 1e-30);
  const double tiny = 2.2250738585072014e-308;
  const double feas = std::sqrt(raw[R_SCON]) / std::max(diff_norm, tiny);
  double r = raw[R_SDU] / e->d.mu + raw[R_SDPHI] / e->d.tau;
  if (has_w) r += raw[R_SDW] / e->d.nu;
  r = r - 2.0 * raw[R_SCROSS];
  out[0] = p;
  out[1] = dual;
  out[2] = gap;
  out[3] = feas;
  out[4] = r;
}

// ---- maps -----------------------------------------------------------------
static void add_mass(PackMap& m, int idx) {
  require(m.nmass < 64, OTFX_EUNSUPPORTED, "mass map overflow");
  m.mass[m.nmass++] = idx;
}

// record layout of a potential-type payload (phi, diff, one u direction)
// complex_rec: record holds complex128 entries
static PackMap potential_pack(const otfx_engine* e, bool complex_rec) {
  PackMap m;
  memset(&m, 0, sizeof(m));
  const int K = e->K;
  m.np = e->NP;
  switch (e->d.kind) {
    case OTFX_KIND_SCALAR:
      m.rec = 1;
      m.src[0] = 0;
      m.wt[0] = 1.0;
      add_mass(m, 0);
      break;
    case OTFX_KIND_VECTOR:
      m.rec = K;
      for (int c = 0; c < K; ++c) {
        m.src[c] = c;
        m.wt[c] = 1.0;
      }
      break;
    case OTFX_KIND_MATRIX_REAL: {
      const int cs = complex_rec ? 2 : 1;
      m.rec = cs * K * K;
      for (int a = 0; a < K; ++a) {
        m.src[a] = cs * (a * K + a);
        m.wt[a] = 1.0;
      }
      for (int a = 0; a < K; ++a)
        for (int b = a + 1; b < K; ++b) {
          const int p = K + pair_index_rt(K, a, b);
          m.src[p] = cs * (a * K + b);
          m.wt[p] = 2.0;
        }
      break;
    }
    default: {
      m.rec = 2 * K * K;
      for (int a = 0; a < K; ++a) {
        m.src[a] = 2 * (a * K + a);
        m.wt[a] = 1.0;
      }
      for (int a = 0; a < K; ++a)
        for (int b = a + 1; b < K; ++b) {
          const int p = K + 2 * pair_index_rt(K, a, b);
          m.src[p] = 2 * (a * K + b);
          m.src[p + 1] = 2 * (a * K + b) + 1;
          m.wt[p] = m.wt[p + 1] = 2.0;
        }
    }
  }
  return m;
}

}  // namespace otfx

namespace otfx {

static UnpackMap potential_unpack(const otfx_engine* e) {
  UnpackMap m;
  memset(&m, 0, sizeof(m));
  const int K = e->K;
  for (int q = 0; q < MAXMAP; ++q) {
    m.plane[q] = -1;
    m.sign[q] = 1;
  }
  switch (e->d.kind) {
    case OTFX_KIND_SCALAR:
      m.rec = 1;
      m.plane[0] = 0;
      break;
    case OTFX_KIND_VECTOR:
      m.rec = K;
      for (int c = 0; c < K; ++c) m.plane[c] = c;
      break;
    case OTFX_KIND_MATRIX_REAL:
      m.rec = K * K;
      for (int a = 0; a < K; ++a)
        for (int b = 0; b < K; ++b)
          m.plane[a * K + b] = a == b ? a : K + pair_index_rt(K, std::min(a, b), std::max(a, b));
      break;
    default:
      m.rec = 2 * K * K;
      for (int a = 0; a < K; ++a)
        for (int b = 0; b < K; ++b) {
          const int q = 2 * (a * K + b);
          if (a == b) {
            m.plane[q] = a;
          } else {
            const int p = K + 2 * pair_index_rt(K, std::min(a, b), std::max(a, b));
            m.plane[q] = p;
            m.plane[q + 1] = p + 1;
            m.sign[q + 1] = a < b ? 1 : -1;
          }
        }
  }
  return m;
}

static PackMap flux_w_pack(const otfx_engine* e) {
  PackMap m;
  memset(&m, 0, sizeof(m));
  const int K = e->K, ell = e->d.ell;
  m.np = e->NWact;
  if (e->d.kind == OTFX_KIND_VECTOR) {
    m.rec = ell;
    for (int q = 0; q < ell; ++q) {
      m.src[q] = q;
      m.wt[q] = 1.0;
    }
    return m;
  }
  // real path: w is a float64 (ell, K, K) record, as the reference's real
  // engine holds it (S/solver.py:414-432); complex path: complex128
  const int cs = e->d.kind == OTFX_KIND_MATRIX_REAL ? 1 : 2;
  m.rec = cs * ell * K * K;
  require(m.rec <= MAXMAP && m.np <= MAXMAP, OTFX_EUNSUPPORTED, "channel flux record too large");
  const int NWS = e->NWS;
  for (int s = 0; s < ell; ++s) {
    const int base = cs * s * K * K;
    if (e->d.kind == OTFX_KIND_MATRIX_REAL) {
      for (int a = 0; a < K; ++a)
        for (int b = a + 1; b < K; ++b) {
          const int p = s * NWS + pair_index_rt(K, a, b);
          m.src[p] = base + (a * K + b);
          m.wt[p] = 2.0;
        }
    } else {
      for (int a = 0; a < K; ++a) {
        m.src[s * NWS + a] = base + 2 * (a * K + a) + 1;
        m.wt[s * NWS + a] = 1.0;
      }
      for (int a = 0; a < K; ++a)
        for (int b = a + 1; b < K; ++b) {
          const int p = s * NWS + K + 2 * pair_index_rt(K, a, b);
          m.src[p] = base + 2 * (a * K + b);
          m.src[p + 1] = base + 2 * (a * K + b) + 1;
          m.wt[p] = m.wt[p + 1] = 2.0;
        }
    }
  }
  return m;
}

static UnpackMap flux_w_unpack(const otfx_engine* e) {
  UnpackMap m;
  memset(&m, 0, sizeof(m));
  for (int q = 0; q < MAXMAP; ++q) {
    m.plane[q] = -1;
    m.sign[q] = 1;
  }
  const int K = e->K, ell = e->d.ell;
  if (e->d.kind == OTFX_KIND_VECTOR) {
    m.rec = ell;
    for (int q = 0; q < ell; ++q) m.plane[q] = q;
    return m;
  }
  const int cs = e->d.kind == OTFX_KIND_MATRIX_REAL ? 1 : 2;
  m.rec = cs * ell * K * K;
  require(m.rec <= MAXMAP, OTFX_EUNSUPPORTED, "channel flux record too large");
  const int NWS = e->NWS;
  for (int s = 0; s < ell; ++s) {
    const int base = cs * s * K * K;
    for (int a = 0; a < K; ++a)
      for (int b = 0; b < K; ++b) {
        const int q = base + cs * (a * K + b);
        if (e->d.kind == OTFX_KIND_MATRIX_REAL) {
          if (a == b) continue;
          m.plane[q] = s * NWS + pair_index_rt(K, std::min(a, b), std::max(a, b));
          m.sign[q] = a < b ? 1 : -1;
        } else if (a == b) {
          m.plane[q + 1] = s * NWS + a;
        } else {
          const int p = s * NWS + K + 2 * pair_index_rt(K, std::min(a, b), std::max(a, b));
          m.plane[q] = p;
          m.sign[q] = a < b ? 1 : -1;
          m.plane[q + 1] = p + 1;
        }
      }
  }
  return m;
}

// ---- host <-> device transfers -------------------------------------------
template <typename T>
static void pack_chunk(otfx_engine* e, const double* s0, const double* s1, int64_t ncell,
                       void* planes, int lrow0, const PackMap& m) {
  pack_kernel<T><<<kPackBlocks, 256, 0, e->stream>>>(s0, s1, ncell, e->d.n, static_cast<T*>(planes),
                                                     e->plane, e->pitch, lrow0, m, e->d_pack_part);
  CK(cudaGetLastError());
}

// ---- pinned staging pool shared by all engines of the process -------------
// Host <-> device transfers go through two pinned slots per direction so the
// multi-threaded host memcpy of chunk k overlaps the DMA of chunk k-1.
// The slot-reuse events are recorded on the engine's stream, so they are
// created per device (an event recorded on another device's stream is an
// error): ev_of(device) is called with the pool lock held and the engine's
// device current.
struct PinnedPool {
  static constexpr size_t kSlot = size_t(32) << 20;  // bytes per slot
  unsigned char* buf = nullptr;                        // 4 slots: 2 x (in0, in1)
  std::map<int, std::pair<cudaEvent_t, cudaEvent_t>> ev;
  std::mutex mu;
  cudaEvent_t* ev_of(int device) {
    auto it = ev.find(device);
    if (it == ev.end()) {
      std::pair<cudaEvent_t, cudaEvent_t> pr{};
      CK(cudaEventCreateWithFlags(&pr.first, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&pr.second, cudaEventDisableTiming));
      it = ev.emplace(device, pr).first;
    }
    return &it->second.first;
  }
};

static PinnedPool& pinned_pool() {
  static PinnedPool* p = [] {
    PinnedPool* q = new PinnedPool();
    CK(cudaMallocHost(&q->buf, 4 * PinnedPool::kSlot));
    return q;
  }();
  return *p;
}

static void par_copy(void* dst, const void* src, size_t bytes) {
  // ~2 blocks per host thread (first-touch page faults of fresh NumPy
  // arrays are part of the cost, so every core should take a share)
  static const int nthr = std::max(1, omp_get_max_threads());
  const size_t grain = std::max<size_t>(size_t(1) << 20, (bytes / (2 * nthr) + 4095) & ~size_t(4095));
  const long nblk = long((bytes + grain - 1) / grain);
#pragma omp parallel for schedule(static) if (nblk > 1)
  for (long b = 0; b < nblk; ++b) {
    const size_t o = size_t(b) * grain;
    memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
           std::min(grain, bytes - o));
  }
}

// upload rows of host records (reference layout) into planes; returns the
// summed block partials {mass0, mass1, weighted sumsq}
static void host_to_planes(otfx_engine* e, const double* h0, const double* h1, const PackMap& m,
                           void* planes, double sums[3]) {
  Range nv("otfx.upload");
  PinnedPool& P = pinned_pool();
  std::lock_guard<std::mutex> lock(P.mu);
  cudaEvent_t ev[2] = {P.ev_of(e->d.device)[0], P.ev_of(e->d.device)[1]};
  const int n = e->d.n;
  const size_t row_bytes = size_t(n) * m.rec * sizeof(double);
  const size_t slot = std::min(PinnedPool::kSlot, e->stage_bytes / 4);
  int chunk = int(std::max<size_t>(1, slot / row_bytes));
  chunk = std::min(chunk, e->rows);
  require(size_t(chunk) * row_bytes <= slot, OTFX_EUNSUPPORTED,
          "grid row too large for the staging buffer");
  const int nchunks = (e->rows + chunk - 1) / chunk;
  std::vector<double> part(size_t(nchunks) * kPackBlocks * 3);
  double* hp;
  CK(cudaMallocHost(&hp, part.size() * sizeof(double)));
  for (int k = 0; k < nchunks; ++k) {
    const int b = k & 1;
    const int r0 = k * chunk;
    const int nr = std::min(chunk, e->rows - r0);
    const size_t off = size_t(r0) * n * m.rec;
    const size_t bytes = size_t(nr) * row_bytes;
    unsigned char* pin0 = P.buf + size_t(2 * b) * PinnedPool::kSlot;
    unsigned char* pin1 = pin0 + PinnedPool::kSlot;
    double* st0 = e->d_stage + size_t(b) * (e->stage_bytes / 2 / sizeof(double));
    double* st1 = st0 + slot / sizeof(double);
    if (k >= 2) CK(cudaEventSynchronize(ev[b]));  // slot b free again
    par_copy(pin0, h0 + off, bytes);
    if (h1) par_copy(pin1, h1 + off, bytes);
    CK(cudaMemcpyAsync(st0, pin0, bytes, cudaMemcpyHostToDevice, e->stream));
    if (h1) CK(cudaMemcpyAsync(st1, pin1, bytes, cudaMemcpyHostToDevice, e->stream));
    CK(cudaEventRecord(ev[b], e->stream));
    if (e->elem == 8) pack_chunk<double>(e, st0, h1 ? st1 : nullptr, int64_t(nr) * n, planes, 1 + r0, m);
    else pack_chunk<float>(e, st0, h1 ? st1 : nullptr, int64_t(nr) * n, planes, 1 + r0, m);
    CK(cudaMemcpyAsync(hp + size_t(k) * kPackBlocks * 3, e->d_pack_part,
                       kPackBlocks * 3 * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
  }
  CK(cudaStreamSynchronize(e->stream));
  sums[0] = sums[1] = sums[2] = 0.0;
  for (size_t q = 0; q < part.size(); q += 3) {
    sums[0] += hp[q];
    sums[1] += hp[q + 1];
    sums[2] += hp[q + 2];
  }
  cudaFreeHost(hp);
}

static void planes_to_host(otfx_engine* e, const void* planes, const UnpackMap& m, double* h) {
  Range nv("otfx.download");
  PinnedPool& P = pinned_pool();
  std::lock_guard<std::mutex> lock(P.mu);
  cudaEvent_t ev[2] = {P.ev_of(e->d.device)[0], P.ev_of(e->d.device)[1]};
  const int n = e->d.n;
  const size_t row_bytes = size_t(n) * m.rec * sizeof(double);
  const size_t slot = std::min(PinnedPool::kSlot, e->stage_bytes / 4);
  int chunk = int(std::max<size_t>(1, slot / row_bytes));
  chunk = std::min(chunk, e->rows);
  require(size_t(chunk) * row_bytes <= slot, OTFX_EUNSUPPORTED,
          "grid row too large for the staging buffer");
  const int nchunks = (e->rows + chunk - 1) / chunk;
  auto launch = [&](int k) {
    const int b = k & 1;
    const int r0 = k * chunk;
    const int nr = std::min(chunk, e->rows - r0);
    const int64_t ncell = int64_t(nr) * n;
    double* st = e->d_stage + size_t(b) * (e->stage_bytes / 2 / sizeof(double));
    unsigned char* pin = P.buf + size_t(2 * b) * PinnedPool::kSlot;
    if (e->elem == 8)
      unpack_kernel<double><<<kPackBlocks, 256, 0, e->stream>>>(
          static_cast<const double*>(planes), e->plane, e->pitch, 1 + r0, ncell, n, m, st);
    else
      unpack_kernel<float><<<kPackBlocks, 256, 0, e->stream>>>(
          static_cast<const float*>(planes), e->plane, e->pitch, 1 + r0, ncell, n, m, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(pin, st, size_t(nr) * row_bytes, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaEventRecord(ev[b], e->stream));
  };
  launch(0);
  for (int k = 0; k < nchunks; ++k) {
    if (k + 1 < nchunks) launch(k + 1);  // next chunk's DMA overlaps this chunk's memcpy
    const int b = k & 1;
    CK(cudaEventSynchronize(ev[b]));
    const int r0 = k * chunk;
    const int nr = std::min(chunk, e->rows - r0);
    par_copy(h + size_t(r0) * n * m.rec, P.buf + size_t(2 * b) * PinnedPool::kSlot,
             size_t(nr) * row_bytes);
  }
}

// ---- device-pointer hand-off (torch-owned tensors) ----------
// The caller's arrays live on the engine's device in the reference layout;
// they are read / written in place by the pack / unpack kernels, ordered
// against the caller's stream with events (no host synchronisation unless a
// host-side scalar is needed).
static void stream_wait(cudaStream_t waiter, cudaStream_t on, cudaEvent_t ev) {
  if (waiter == on) return;
  CK(cudaEventRecord(ev, on));
  CK(cudaStreamWaitEvent(waiter, ev, 0));
}

static void check_device_ptr(const otfx_engine* e, const void* p) {
  if (!p) return;
  cudaPointerAttributes a{};
  CK(cudaPointerGetAttributes(&a, p));
  require(a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged, OTFX_EINVAL,
          "expected a device pointer");
  require(a.device == e->d.device, OTFX_EINVAL, "device pointer on another device");
}

static void device_to_planes(otfx_engine* e, const double* d0, const double* d1, const PackMap& m,
                             void* planes, double sums[3]) {
  const int64_t ncell = int64_t(e->rows) * e->d.n;
  if (e->elem == 8) pack_chunk<double>(e, d0, d1, ncell, planes, 1, m);
  else pack_chunk<float>(e, d0, d1, ncell, planes, 1, m);
  if (!sums) return;
  CK(cudaMemcpyAsync(e->h_pack_part, e->d_pack_part, kPackBlocks * 3 * sizeof(double),
                     cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  sums[0] = sums[1] = sums[2] = 0.0;
  for (int q = 0; q < kPackBlocks * 3; q += 3) {
    sums[0] += e->h_pack_part[q];
    sums[1] += e->h_pack_part[q + 1];
    sums[2] += e->h_pack_part[q + 2];
  }
}

static void planes_to_device(otfx_engine* e, const void* planes, const UnpackMap& m, double* d) {
  const int64_t ncell = int64_t(e->rows) * e->d.n;
  if (e->elem == 8)
    unpack_kernel<double><<<kPackBlocks, 256, 0, e->stream>>>(
        static_cast<const double*>(planes), e->plane, e->pitch, 1, ncell, e->d.n, m, d);
  else
    unpack_kernel<float><<<kPackBlocks, 256, 0, e->stream>>>(
        static_cast<const float*>(planes), e->plane, e->pitch, 1, ncell, e->d.n, m, d);
  CK(cudaGetLastError());
}

static void* plane_ptr(otfx_engine* e, void* base, int p) {
  return static_cast<char*>(base) + size_t(p) * e->plane * e->elem;
}

static void allreduce_host(otfx_engine* e, double* v, int count) {
  if (!e->comm || e->nranks == 1) return;
  CK(cudaMemcpyAsync(e->d_raw, v, count * sizeof(double), cudaMemcpyHostToDevice, e->stream));
  NK(nccl().AllReduce(e->d_raw, e->d_raw, count, ncclFloat64, ncclSum, e->comm, e->stream));
  CK(cudaMemcpyAsync(v, e->d_raw, count * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
}

static void drop_graphs(otfx_engine* e) {
  for (auto& kv : e->graphs) cudaGraphExecDestroy(kv.second);
  e->graphs.clear();
}


static void create(const otfx_engine_desc* d, otfx_engine* e) {
  Range nv("otfx.create");
  require(d != nullptr, OTFX_EINVAL, "null descriptor");
  e->d = *d;
  const int kind = d->kind;
  require(kind >= 0 && kind <= 3, OTFX_EINVAL, "unknown kind");
  require(d->dtype == OTFX_F64 || d->dtype == OTFX_F32, OTFX_EINVAL, "unknown dtype");
  require(d->n >= 2, OTFX_EINVAL, "grid needs n >= 2");
  require(d->row_begin >= 0 && d->row_end <= d->n && d->row_begin < d->row_end, OTFX_EINVAL,
          "bad slab rows");
  require(d->tau > 0 && d->mu > 0, OTFX_EINVAL, "step sizes must be positive");
  require(d->norm_u >= 0 && d->norm_u <= 3 && d->norm_w >= 0 && d->norm_w <= 3, OTFX_EINVAL,
          "unknown norm family");
  e->elem = d->dtype == OTFX_F64 ? 8 : 4;
  e->K = kind == OTFX_KIND_SCALAR ? 1 : d->k;
  if (d->dtype == OTFX_F64) e->ops64 = find_ops<double>(kind, e->K, d->ell);
  else e->ops32 = find_ops<float>(kind, e->K, d->ell);
  const bool found = e->ops64 || e->ops32;
  require(found, OTFX_EUNSUPPORTED,
          "no sm_100a instantiation for kind=" + std::to_string(kind) + " k=" + std::to_string(e->K));
  const int NP = e->ops64 ? e->ops64->NP : e->ops32->NP;
  const int NWS = e->ops64 ? e->ops64->NWS : e->ops32->NWS;
  const int LMAX = e->ops64 ? e->ops64->LMAX : e->ops32->LMAX;
  e->has_w = e->ops64 ? e->ops64->has_w : e->ops32->has_w;
  e->NP = NP;
  e->NWS = NWS;
  e->LMAX = LMAX;
  if (e->has_w) {
    require(d->ell >= 1 && d->ell <= LMAX, OTFX_EUNSUPPORTED,
            "channel count ell=" + std::to_string(d->ell) + " exceeds the instantiation capacity " +
                std::to_string(LMAX));
    require(d->nu > 0 && d->alpha > 0, OTFX_EINVAL, "nu and alpha must be positive");
    require(d->chan != nullptr, OTFX_EINVAL, "channel operator missing");
    const size_t nc = kind == OTFX_KIND_VECTOR ? size_t(e->K) * d->ell : size_t(d->ell) * e->K * e->K * 2;
    require(e->dynamic() || nc <= size_t(MAX_CHAN_COEF), OTFX_EUNSUPPORTED,
            "channel operator too large");
    e->chan.assign(d->chan, d->chan + nc);
    e->NWact = d->ell * NWS;
  } else {
    e->d.ell = 0;
    e->NWact = 0;
  }
  if (kind == OTFX_KIND_VECTOR || kind == OTFX_KIND_SCALAR)
    require(d->norm_u != OTFX_NORM_L1NUC && d->norm_w != OTFX_NORM_L1NUC, OTFX_EUNSUPPORTED,
            "nuclear norm requires a matrix payload");
  if (kind == OTFX_KIND_MATRIX_REAL)
    require(d->norm_u != OTFX_NORM_L1NUC && d->norm_w != OTFX_NORM_L1NUC, OTFX_EINVAL,
            "nuclear norms run on the complex path");
  require(!(e->has_w && d->norm_w == OTFX_NORM_L12), OTFX_EUNSUPPORTED,
          "row-grouped norm applies only to spatial fluxes");
  require(!(d->eps_reg > 0 && (d->norm_u == OTFX_NORM_L1NUC || d->norm_w == OTFX_NORM_L1NUC)),
          OTFX_EUNSUPPORTED, "eps_reg > 0 has no closed-form prox for the nuclear family");

  CK(cudaSetDevice(d->device));
  if (d->stream) {
    e->stream = static_cast<cudaStream_t>(d->stream);
  } else {
    CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    e->own_stream = true;
  }
  e->rows = d->row_end - d->row_begin;
  e->rows_alloc = e->rows + 2;
  e->pitch = (d->n + 31) / 32 * 32;
  e->plane = int64_t(e->rows_alloc) * e->pitch;
  const int per_state = 3 * NP + e->NWact;
  const size_t pb = size_t(e->plane) * e->elem;
  e->state_bytes = size_t(per_state) * pb;

  // sweep geometry: TX columns per CTA, R rows per CTA, >= ~4 CTAs per SM
  const int n = d->n;
  e->TX = env_int("OTFX_TILE_COLS", n > 64 ? 128 : (n > 32 ? 64 : 32));
  require(e->TX % 32 == 0 && e->TX >= 32 && e->TX <= 128, OTFX_EINVAL,
          "tile columns must be 32, 64, 96 or 128");
  e->gx = (n + e->TX - 1) / e->TX;
  const int want = 148 * 4;
  int gy = (want + e->gx - 1) / e->gx;
  int R = (e->rows + gy - 1) / gy;
  // small slabs are latency-bound (one CTA walks R rows in sequence): spread
  // them over ~4 CTAs per SM with as few rows per CTA as possible
  const bool small = int64_t(n) * e->rows <= int64_t(512) * 512;
  R = small ? std::max(1, std::min(64, R)) : std::max(4, std::min(64, R));
  R = env_int("OTFX_TILE_ROWS", R);
  e->R = R;
  e->gy = (e->rows + R - 1) / R;
  const size_t sw = size_t(e->TX + 1) * NP * 2 * e->elem;
  e->smem_plain = ((2 * sw + 15) & ~size_t(15)) + 32 * 4 * sizeof(double);
  e->smem_check = ((3 * sw + 15) & ~size_t(15)) + 32 * 4 * sizeof(double);
  // small slabs: one wave -- grow the rows per CTA until every CTA of the
  // register sweep is resident at once (measured on B200: 3x3 real matrix
  // 256^2, 232 registers, 2 CTAs/SM: 14.1 -> 11.2 us / iteration)
  if (small && env_int("OTFX_TILE_ROWS", 0) == 0) {
    CK(e->ops64 ? e->ops64->prepare() : e->ops32->prepare());
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device));
    const int occ = e->ops64 ? e->ops64->sweep_occupancy(e->TX, e->smem_plain)
                             : e->ops32->sweep_occupancy(e->TX, e->smem_plain);
    const int64_t gy_max = std::max<int64_t>(1, int64_t(std::max(occ, 1)) * sms / e->gx);
    if (e->gy > gy_max) {
      e->R = int((e->rows + gy_max - 1) / gy_max);
      e->gy = (e->rows + e->R - 1) / e->R;
    }
  }
  e->ex = (n + 127) / 128;
  e->ey = std::min(e->rows, std::max(1, 2048 / e->ex));
  // TMA-streamed sweep: ring depth 4 (3 if that keeps two CTAs per SM)
  // the TMA ring pays off once rows are long enough to pipeline; small slabs
  // run the register-streamed sweep (measured: 4.4 vs 8.9 us/iteration at 64^2)
  const bool want_tma = env_int("OTFX_TMA", small ? 0 : 1) != 0 && !e->dynamic();
  e->use_tma = want_tma;
  // a wide (6 / 8-warp) plan that does not fit shared memory at any ring depth
  // is retried with 4 consumer warps before falling back to the register
  // sweep (4x4 complex, ell = 2: 1.45 -> 0.77 ms / iteration at 1024^2,
  // profiles/r02_stage_depth.txt)
  for (int attempt = 0; want_tma && attempt < 2; ++attempt) {
    e->narrow = attempt == 1;
    if (e->narrow && (e->ops64 ? e->ops64->wide_cw : e->ops32->wide_cw) == 4) break;
    // ring depth: 3 or 4 stages, whichever keeps more CTAs resident per SM
    // (registers and shared memory both count); on a tie the deeper ring
    // (measured on B200: 2x2 complex l1nuc 75 % -> 88 % of the HBM roofline at
    // 3 stages / 3 CTAs vs 4 stages / 2 CTAs; fp32 vector, 3 CTAs either way:
    // 96 % at 4 stages vs 92 % at 3)
    // (2 stages: the 8-warp heavy payloads, and see below)
    const int wide = e->ops64 ? e->ops64->wide_cw : e->ops32->wide_cw;
    // (and for payloads whose 3-stage ring does not fit shared memory)
    // (2 stages are also a candidate for the real-symmetric matrix payloads,
    // where the shallower ring buys a third resident CTA: C4 family 2048^2
    // 92.2 -> 94.0 % of the roofline; profiles/r02_stage_depth.txt)
    const bool heavy = kind == OTFX_KIND_MATRIX_COMPLEX && e->K >= 3 && e->elem == 8;
    int smin = (heavy && !e->narrow && env_int("OTFX_TMA_WARPS", wide) == wide) ? 2 : 3;
    if (d->kind == OTFX_KIND_MATRIX_REAL) smin = 2;
    // (self-producing 4-warp CTAs: a 2-stage ring buys the fourth resident CTA)
    if ((e->ops64 ? e->ops64->narrow_threads : e->ops32->narrow_threads) == 128) smin = 2;
    if (smin == 3 && !plan_stages(e, 3)) smin = 2;
    int S = env_int("OTFX_STAGES", 0);
    if (S <= 0) {
      CK(e->ops64 ? e->ops64->prepare() : e->ops32->prepare());
      int best = -1;
      for (int cand = 4; cand >= smin; --cand) {
        if (!plan_stages(e, cand)) continue;
        const int occ = e->ops64 ? e->ops64->tma_occupancy(e->L.cw, e->L.total)
                                 : e->ops32->tma_occupancy(e->L.cw, e->L.total);
        if (occ > best) {
          best = occ;
          S = cand;
        }
      }
      if (S <= 0) S = smin;
    }
    // (an explicit OTFX_STAGES >= 2 is honoured as given: measurement knob)
    e->use_tma = plan_stages(e, env_int("OTFX_STAGES", 0) >= 2 ? S : std::max(smin, S));
    if (e->use_tma) break;
  }
  if (e->use_tma) {
    e->gx = (n + e->L.tile - 1) / e->L.tile;
    // Row split.  Short CTAs (16 rows) keep the set of CTAs resident at any
    // moment on a compact band of rows, so the ~300 concurrent TMA streams hit
    // few DRAM pages and the one-row halo re-reads hit L2; measured on B200
    // (tools/wave_sweep.py, profiles/README.md): 8192^2 fp64 vector 93 % of
    // the HBM peak at 119-row CTAs -> 98 % at 16, 4096^2 91 % -> 95 %, 3x3
    // matrix 2048^2 81 % -> 92 %.  When that leaves only a few waves, rows per
    // CTA grow just enough for the CTA count to fill integral waves (a
    // partial last wave runs on a few SMs only).
    CK(e->ops64 ? e->ops64->prepare() : e->ops32->prepare());
    int dev_sms = 148;
    CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, d->device));
    const int per_sm = std::max(1, e->ops64 ? e->ops64->tma_occupancy(e->L.cw, e->L.total)
                                            : e->ops32->tma_occupancy(e->L.cw, e->L.total));
    const long slots = (long)dev_sms * per_sm;
    // (8 rows for the 2x2 complex payload: twice the CTAs, a smaller last
    // wave -- C3 family 2048^2 0.2536 -> 0.2479 ms; 16 is best for the vector
    // and real-symmetric ones, profiles/r02_stage_depth.txt)
    const int r0 = (kind == OTFX_KIND_MATRIX_COMPLEX && e->K == 2) ? 8 : 16;
    int R = std::min(r0, e->rows);
    const long ctas = (long)e->gx * ((e->rows + R - 1) / R);
    const long waves = (ctas + slots - 1) / slots;
    if (per_sm == 1) {
      // one resident CTA per SM (the heavy payloads): nothing back-fills a
      // partial wave, and every CTA re-derives its halo row's flux, so the
      // sweep costs ~ (waves, rounded up) x (R + 1) row steps; take the R in
      // [8, 32] that minimises it (3x3 complex 1024^2: R = 12, 3 whole waves;
      // 2048^2: R = 32, 3.9 waves: l2/l1 0.645 -> 0.636 ms, l1nuc 0.659 ->
      // 0.642 ms vs R = 16; profiles/r02_heavy_self8.md)
      long best = -1;
      for (int r = 8; r <= std::min(32, e->rows); ++r) {
        const long w = (e->gx * ((e->rows + r - 1) / r) + slots - 1) / slots;
        const long cost = w * (r + 1);
        if (best < 0 || cost < best) {
          best = cost;
          R = r;
        }
      }
    } else if (waves <= 8) {
      const long gyw = std::max(1L, std::min<long>(waves * slots / e->gx, e->rows));
      const int Rw = (int)((e->rows + gyw - 1) / gyw);
      R = std::max(R, Rw);
    }
    e->R = env_int("OTFX_TILE_ROWS", R);
    e->gy = (e->rows + e->R - 1) / e->R;
  }

  // On-chip solve: a small single-slab grid whose state fits in the shared
  // memory of one cluster of up to 16 CTAs runs the whole run loop in one
  // launch (cluster.cuh).  Measured on B200, vector 3-channel 64^2 fp64:
  // see DESIGN.md section 4.
  {
    const bool inst = e->ops64 ? e->ops64->cluster_run != nullptr : e->ops32->cluster_run != nullptr;
    if (inst && !e->use_tma && d->row_begin == 0 && d->row_end == n && n >= 2 &&
        int64_t(n) * n <= int64_t(128) * 128 && env_int("OTFX_CLUSTER", 1) != 0) {
      const int want = env_int("OTFX_CLUSTER_CTAS", 16);
      for (int C = std::min(want, n); C >= 2 && !e->use_cluster; C /= 2) {
        const int rmax = (n + C - 1) / C;
        // one thread per cell of the band plus one per cell of the halo row
        const int thr = (rmax * n + n + 31) / 32 * 32;
        const size_t sm = e->ops64 ? e->ops64->cluster_smem(rmax, n) : e->ops32->cluster_smem(rmax, n);
        if (thr > kClusterThreads || sm > 227 * 1024) break;  // fewer CTAs: taller bands
        const int fits = e->ops64 ? e->ops64->cluster_fits(C, thr, sm) : e->ops32->cluster_fits(C, thr, sm);
        if (fits) {
          e->use_cluster = true;
          e->cl_ctas = C;
          e->cl_threads = thr;
          e->cl_rows = rmax;
          e->cl_smem = sm;
        }
      }
    }
  }

  // staging: up to 64 MB, at least two grid rows of the widest record
  const int max_rec = (kind == OTFX_KIND_VECTOR || kind == OTFX_KIND_SCALAR)
                          ? std::max(std::max(2 * e->K, int(d->ell)), 16)
                          : std::max(2 * e->K * e->K * std::max(1, d->ell) * 2, 16);
  e->stage_bytes = std::max<size_t>(size_t(128) << 20, size_t(4) * n * max_rec * sizeof(double));

  const size_t n_sweep = size_t(e->gx) * e->gy * 10, n_pe = size_t(e->ex) * e->ey * 8,
               n_me = size_t(e->ex) * e->ey * 2, n_du = size_t(e->gx) * e->gy * 10;
  const size_t halo = size_t(8) * NP * n * e->elem;
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_state0 = carve(e->state_bytes), o_state1 = carve(e->state_bytes);
  const size_t o_diff = carve(size_t(NP) * pb);
  const size_t o_ps = carve(n_sweep * 8), o_pe = carve(n_pe * 8), o_me = carve(n_me * 8);
  const size_t o_du = carve(n_du * 8);
  const size_t o_raw = carve(64 * 8);
  const size_t o_pack = carve(kPackBlocks * 3 * 8);
  const size_t o_halo = carve(halo);
  const size_t o_result = carve(4 * sizeof(long long));
  const size_t o_chan = carve(e->chan.size() * sizeof(double));
  const size_t o_loop = carve(256);
  const size_t o_stage = carve(e->stage_bytes);
  e->total_bytes = off;
  // stream-ordered allocation from the library's per-device pool: freed
  // blocks stay cached (release threshold = max), so a solve that follows
  // another one of the same size skips cudaMalloc / cudaFree (hundreds of ms
  // at 8192^2); otfx_release_cached_memory() trims the pool
  if (env_int("OTFX_POOL", 1) != 0) {
    CK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&e->mem), off, device_pool(d->device),
                               e->stream));
    e->pooled = true;
  } else {
    CK(cudaMalloc(&e->mem, off));
  }
  CK(cudaMemsetAsync(e->mem, 0, o_stage, e->stream));
  for (int s = 0; s < 2; ++s) {
    unsigned char* b = e->mem + (s ? o_state1 : o_state0);
    e->u[s] = b;
    e->phi[s] = b + size_t(2 * NP) * pb;
    e->w[s] = b + size_t(3 * NP) * pb;
  }
  e->diff = e->mem + o_diff;
  e->d_part_sweep = reinterpret_cast<double*>(e->mem + o_ps);
  e->d_part_dual = reinterpret_cast<double*>(e->mem + o_du);
  e->d_part_eval = reinterpret_cast<double*>(e->mem + o_pe);
  e->d_max_eval = reinterpret_cast<double*>(e->mem + o_me);
  e->d_raw = reinterpret_cast<double*>(e->mem + o_raw);
  e->d_pack_part = reinterpret_cast<double*>(e->mem + o_pack);
  e->d_halo = e->mem + o_halo;
  e->d_result = reinterpret_cast<long long*>(e->mem + o_result);
  e->d_loop = e->mem + o_loop;
  if (e->dynamic()) {
    e->d_chan = reinterpret_cast<double*>(e->mem + o_chan);
    CK(cudaMemcpyAsync(e->d_chan, e->chan.data(), e->chan.size() * sizeof(double),
                       cudaMemcpyHostToDevice, e->stream));
  }
  e->d_stage = reinterpret_cast<double*>(e->mem + o_stage);
  if (e->use_tma) {
    for (int st = 0; st < 2; ++st) {
      make_map(e, &e->maps[st].u, e->u[st], 2 * NP, e->L.tw);
      make_map(e, &e->maps[st].w, e->w[st], e->NWact, e->L.tw);
      make_map(e, &e->maps[st].phi, e->phi[st], NP, e->L.tw);
      make_map(e, &e->maps[st].diff, e->diff, NP, e->L.tw);
    }
  }
  CK(cudaMallocHost(&e->h_raw, 64 * sizeof(double)));
  CK(cudaMallocHost(&e->h_pack_part, kPackBlocks * 3 * sizeof(double)));
  CK(cudaEventCreateWithFlags(&e->ev_hand, cudaEventDisableTiming));
  CK(e->ops64 ? e->ops64->prepare() : e->ops32->prepare());
  e->use_graphs = env_int("OTFX_GRAPHS", 1) != 0;
  CK(cudaStreamSynchronize(e->stream));
}

static void destroy(otfx_engine* e) {
  if (!e) return;
  drop_graphs(e);
  for (auto& pr : e->ev_pool) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  if (e->stream) cudaStreamSynchronize(e->stream);
  if (e->edge_stream) {
    cudaStreamSynchronize(e->edge_stream);
    cudaStreamDestroy(e->edge_stream);
  }
  if (e->ev_fork) cudaEventDestroy(e->ev_fork);
  if (e->ev_join) cudaEventDestroy(e->ev_join);
  if (e->ev_hand) cudaEventDestroy(e->ev_hand);
  if (e->comm && e->own_comm && nccl().CommDestroy) nccl().CommDestroy(e->comm);
  if (e->mem) {
    if (e->pooled) {
      cudaFreeAsync(e->mem, e->stream);
      cudaStreamSynchronize(e->stream);  // the block is reusable from any stream
    } else {
      cudaFree(e->mem);
    }
  }
  if (e->h_raw) cudaFreeHost(e->h_raw);
  if (e->h_pack_part) cudaFreeHost(e->h_pack_part);
  if (e->own_stream && e->stream) cudaStreamDestroy(e->stream);
}

static void zero_state(otfx_engine* e) {
  for (int s = 0; s < 2; ++s) {
    CK(cudaMemsetAsync(e->u[s], 0, e->state_bytes, e->stream));
  }
  e->cur = 0;
  e->residual_valid = false;
  CK(cudaStreamSynchronize(e->stream));
}

}  // namespace otfx

// ===========================================================================
// extern "C" ABI
// ===========================================================================
using namespace otfx;

namespace otfx {

// The engines the run loop drives: one engine (a whole grid, or this rank's
// slab of an NCCL-connected decomposition), or the P slabs of one grid on one
// device stepped in lockstep with local halo copies -- the single-GPU stand-in
// for the NCCL transport, which runs the same loop (tests/test_gpu_solver.py).
struct SlabGroup {
  otfx_engine* const* es;
  int count;
  ncclComm_t loop = nullptr;  // one-rank NCCL loopback transport (local groups)
  bool local() const { return count > 1; }
  otfx_engine* lead() const { return es[0]; }
};

// the slabs of one grid in one process: same pack / unpack as exchange_nccl,
// the transport is a device copy of each send buffer into the neighbour's
// receive buffer (what ncclSend/ncclRecv move between ranks)
static void exchange_local_impl(otfx_engine* const* es, int count, cudaStream_t st,
                                ncclComm_t loop = nullptr) {
  Range nv("otfx.halo_exchange_local");
  for (int s = 0; s + 1 < count; ++s) {
    otfx_engine* a = es[s];
    otfx_engine* b = es[s + 1];
    require(a->stream == b->stream, OTFX_EINVAL, "local exchange needs one shared stream");
    require(a->d.row_end == b->d.row_begin && a->d.n == b->d.n && a->elem == b->elem &&
                a->NP == b->NP && a->pitch == b->pitch,
            OTFX_EINVAL, "engines are not adjacent slabs of one grid");
    require(a->cur == b->cur, OTFX_EINVAL, "engines are at different iterations");
  }
  for (int s = 0; s < count; ++s) halo_pack(es[s], s > 0, s + 1 < count, st);
  if (loop) {
    // NCCL loopback: the same ncclSend / ncclRecv calls (buffers, counts,
    // datatype, one group) exchange_nccl posts between ranks, addressed to
    // this process's own rank; sends and receives to one peer match in
    // posting order, so each boundary posts (a -> b), then (b -> a)
    NcclApi& N = nccl();
    const ncclDataType_t dt = es[0]->elem == 8 ? ncclFloat64 : ncclFloat32;
    NK(N.GroupStart());
    for (int s = 0; s + 1 < count; ++s) {
      const HaloBufs ha = halo_bufs(es[s]), hb = halo_bufs(es[s + 1]);
      const size_t w = size_t(es[s]->d.n);
      const int NP = es[s]->NP;
      NK(N.Send(ha.send_bot, 3 * NP * w, dt, 0, loop, st));
      NK(N.Recv(hb.recv_top, 3 * NP * w, dt, 0, loop, st));
      NK(N.Send(hb.send_top, NP * w, dt, 0, loop, st));
      NK(N.Recv(ha.recv_bot, NP * w, dt, 0, loop, st));
    }
    NK(N.GroupEnd());
  } else {
    for (int s = 0; s + 1 < count; ++s) {
      const HaloBufs ha = halo_bufs(es[s]), hb = halo_bufs(es[s + 1]);
      const size_t wb = size_t(es[s]->d.n) * es[s]->elem;
      const int NP = es[s]->NP;
      CK(cudaMemcpyAsync(hb.recv_top, ha.send_bot, 3 * NP * wb, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(ha.recv_bot, hb.send_top, NP * wb, cudaMemcpyDeviceToDevice, st));
    }
  }
  for (int s = 0; s < count; ++s) halo_unpack(es[s], s > 0, s + 1 < count, st);
}

// one iteration of every slab, then the halo exchange (overlapped with the
// interior bands when the slabs are tall enough)
static void group_sweep(const SlabGroup& g, int fl) {
  if (!g.local()) {
    sweep_exchange(g.lead(), fl);
    return;
  }
  bool ov = true;
  for (int q = 0; q < g.count; ++q) ov = ov && overlap_ready(g.es[q]);
  if (ov) {
    overlapped_sweep(g.es, g.count, fl,
                     [&](cudaStream_t st) { exchange_local_impl(g.es, g.count, st, g.loop); });
    return;
  }
  for (int q = 0; q < g.count; ++q) launch_sweep(g.es[q], fl);
  exchange_local_impl(g.es, g.count, g.lead()->stream, g.loop);
}

static void group_plain(const SlabGroup& g, int64_t count) {
  if (!g.local()) {
    run_plain(g.lead(), count);
    return;
  }
  for (int64_t q = 0; q < count; ++q) group_sweep(g, 0);
}

// raw check scalars of the group: NCCL-allreduced for a rank, summed / maxed
// over the slabs (in slab order) for a local group
static void group_raw(const SlabGroup& g, bool fused, bool with_res, double raw[OTFX_NRAW]) {
  Range nv("otfx.check_reduce");
  for (int q = 0; q < OTFX_NRAW; ++q) raw[q] = 0.0;
  for (int s = 0; s < g.count; ++s) {
    otfx_engine* e = g.es[s];
    const ncclComm_t ar = g.local() ? g.loop : rank_comm(e);
    if (fused) raw_fused_to_host(e, ar);
    else raw_to_host(e, with_res, ar);
    for (int q = 0; q < R_NSUM; ++q) raw[q] += e->h_raw[q];
    for (int q = R_NSUM; q < OTFX_NRAW; ++q) raw[q] = s ? std::max(raw[q], e->h_raw[q]) : e->h_raw[q];
  }
}

// the _run loop (S/solver.py:294-337) over a slab group
// the first `capacity` rows of the engine's history into the caller's buffer;
// n_history = all rows (more than capacity: fetch them with otfx_engine_history)
static void copy_history(const otfx_engine* e, otfx_history_point* hist, int64_t capacity,
                         int64_t* n_history) {
  const int64_t nh = int64_t(e->history.size());
  if (hist && capacity > 0)
    std::copy(e->history.begin(), e->history.begin() + std::min(nh, capacity), hist);
  *n_history = nh;
}

// ---- device-side run loop ----------------------------------------------------
// Small grids spend a host round trip per check (check sweep -> evaluate ->
// reduce -> copy -> stream sync -> host finalize -> next graph launch): ~40 us
// per 100 iterations at 256^2, 6-8 % of the run (tools/check_overhead.py).
// Here the check periods run inside ONE CUDA graph: a WHILE conditional node
// whose body is a period -- ce - 1 plain sweeps, the check sweep, evaluate,
// the fixed-order reduction and loop_check_kernel, which applies the
// reference's finalize algebra (S/solver.py:242-291, finalize_dev), appends the
// history row on the device, takes the stopping decision (:315-316) and sets
// the loop condition.  Same kernels and reductions as the host loop, so the
// iterates and history are identical; the host syncs once per run.
struct LoopCtl {
  double tol_gap, tol_feas, diff_norm;
  long long it, ce, periods_left, nh, hist_cap;
  int conv;
};

__global__ void loop_check_kernel(const double* raw, LoopCtl* c, double* hist, double mu, double nu,
                                  double tau, double alpha, double eps, int has_w,
                                  cudaGraphConditionalHandle h) {
  if (threadIdx.x != 0) return;
  double out[5];
  finalize_dev(raw, has_w != 0, alpha, eps, c->diff_norm, mu, nu, tau, out);
  c->it += c->ce;
  const bool conv = out[2] <= c->tol_gap && out[3] <= c->tol_feas;
  double* r = hist + c->nh * 6;
  r[0] = double(c->it);
  r[1] = out[0];
  r[2] = out[1];
  r[3] = out[2];
  r[4] = out[3];
  r[5] = out[4];
  c->nh += 1;
  c->periods_left -= 1;
  c->conv = conv ? 1 : 0;
  cudaGraphSetConditional(h, (!conv && c->periods_left > 0 && c->nh < c->hist_cap) ? 1u : 0u);
}

static cudaGraphExec_t loop_graph(otfx_engine* e, int64_t ce) {
  const auto key = std::make_pair(e->cur, -ce);  // plain graphs use positive counts
  auto it = e->graphs.find(key);
  if (it != e->graphs.end()) return it->second;
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, nullptr, 0, &p));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  const int saved = e->cur;
  CK(cudaStreamBeginCaptureToGraph(e->stream, body, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  try {
    for (int64_t q = 0; q + 1 < ce; ++q) launch_sweep(e, 0);
    launch_sweep(e, 1);
    launch_evaluate(e);
    reduce_raw_kernel<<<1, 256, 0, e->stream>>>(e->d_part_eval, e->d_max_eval, e->ex * e->ey,
                                                 e->d_part_sweep, e->gx * e->gy, 1, e->d_raw);
    CK(cudaGetLastError());
    loop_check_kernel<<<1, 32, 0, e->stream>>>(e->d_raw, static_cast<LoopCtl*>(e->d_loop),
                                               e->d_stage, e->d.mu, e->d.nu, e->d.tau, e->d.alpha,
                                               e->d.eps_reg, e->has_w ? 1 : 0, h);
    CK(cudaGetLastError());
  } catch (...) {
    cudaStreamEndCapture(e->stream, &body);
    e->cur = saved;
    cudaGraphDestroy(g);
    throw;
  }
  CK(cudaStreamEndCapture(e->stream, &body));
  e->cur = saved;  // ce is even: the period ends on the iterate parity it started from
  cudaGraphExec_t ge;
  CK(cudaGraphInstantiate(&ge, g, 0));
  cudaGraphDestroy(g);
  return e->graphs.emplace(key, ge).first->second;
}

static bool device_loop_ok(const SlabGroup& g, int64_t ce, bool fused) {
  const otfx_engine* e = g.lead();
  return !g.local() && e->nranks == 1 && !fused && e->use_graphs && !e->timing && ce >= 2 &&
         ce % 2 == 0 && env_int("OTFX_DEVICE_LOOP", 1) != 0;
}

// the run's full check periods from iteration `it` (a multiple of ce) on the
// device; appends their history rows, returns false if the loop did not run
static bool run_loop_device(otfx_engine* e, const otfx_run_config* cfg, double dn, int64_t& it,
                            bool& conv) {
  const int64_t ce = cfg->check_every;
  const int64_t periods = (cfg->max_iters - it) / ce;
  if (periods < 1) return false;
  LoopCtl c = {};
  c.tol_gap = cfg->tol_gap;
  c.tol_feas = cfg->tol_feas;
  c.diff_norm = dn;
  c.it = it;
  c.ce = ce;
  c.periods_left = periods;
  c.hist_cap = (long long)(e->stage_bytes / (6 * sizeof(double)));
  cudaGraphExec_t ge = loop_graph(e, ce);
  CK(cudaMemcpyAsync(e->d_loop, &c, sizeof(c), cudaMemcpyHostToDevice, e->stream));
  CK(cudaGraphLaunch(ge, e->stream));
  CK(cudaMemcpyAsync(&c, e->d_loop, sizeof(c), cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  const size_t h0 = e->history.size();
  e->history.resize(h0 + size_t(c.nh));
  static_assert(sizeof(otfx_history_point) == 6 * sizeof(double), "history row layout");
  CK(cudaMemcpyAsync(e->history.data() + h0, e->d_stage, size_t(c.nh) * sizeof(otfx_history_point),
                     cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  it = c.it;
  conv = c.conv != 0;
  return true;
}

static void run_loop(const SlabGroup& g, const otfx_run_config* cfg, otfx_history_point* hist,
                     int64_t capacity, int64_t* n_history, int64_t* iterations, int* converged) {
  Range nv("otfx.run");
  otfx_engine* e = g.lead();
  // ||diff|| of the whole grid: the engine's (allreduced under NCCL), or for a
  // local slab group the root of the slabs' summed squares, combined here
  // from every slab's own-row norm (S/solver.py:185)
  double dn = e->diff_norm;
  if (g.local()) {
    double s2 = 0.0;
    for (int q = 0; q < g.count; ++q) s2 += g.es[q]->diff_norm_own * g.es[q]->diff_norm_own;
    dn = std::sqrt(s2);
  }
  std::vector<otfx_history_point>& H = e->history;
  H.clear();
  auto push = [&](int64_t it, const double* r, double rk) {
    H.push_back({double(it), r[0], r[1], r[2], r[3], rk});
  };
  double r[5], raw[OTFX_NRAW];
  group_raw(g, false, false, raw);
  finalize(e, raw, r, dn);
  push(0, r, std::nan(""));
  bool conv = r[2] <= cfg->tol_gap && r[3] <= cfg->tol_feas;
  int64_t it = 0;
  const int64_t ce = cfg->check_every, mx = cfg->max_iters;
  bool fused_ok = env_int("OTFX_FUSED_CHECK", 1) != 0;
  for (int q = 0; q < g.count; ++q) fused_ok = fused_ok && g.es[q]->use_tma;
  if (!conv && device_loop_ok(g, ce, fused_ok)) {
    Range nv("otfx.device_loop");
    run_loop_device(e, cfg, dn, it, conv);
  }
  while (!conv && it < mx) {
    const int64_t next = std::min((it / ce + 1) * ce, mx);
    group_plain(g, next - it - 1);
    it = next - 1;
    // Fused check: the iteration after the check runs speculatively and
    // accumulates the dual norms of the checked iterate; it is kept when the
    // run continues and dropped (ping-pong buffer flipped back) when it stops.
    // It must not itself be a check iteration.
    const bool fuse = fused_ok && next + 1 < mx && (next + 1) % ce != 0;
    group_sweep(g, 1);
    if (fuse) group_sweep(g, 2);
    group_raw(g, fuse, true, raw);
    finalize(e, raw, r, dn);
    it = next;
    push(it, r, r[4]);
    conv = r[2] <= cfg->tol_gap && r[3] <= cfg->tol_feas;
    if (fuse) {
      if (conv) {
        for (int q = 0; q < g.count; ++q) g.es[q]->cur ^= 1;  // drop the speculative iterate
      } else {
        ++it;  // keep it: iteration next+1 is done
      }
    }
  }
  copy_history(e, hist, capacity, n_history);
  *iterations = it;
  *converged = conv ? 1 : 0;
}

}  // namespace otfx

#define API_BEGIN try {
#define API_END                        \
  }                                    \
  catch (const Error& ex) {            \
    g_err = ex.what();                 \
    return ex.code;                    \
  }                                    \
  catch (const std::exception& ex) {   \
    g_err = ex.what();                 \
    return OTFX_ECUDA;                 \
  }                                    \
  return OTFX_OK;

extern "C" {

int otfx_abi_version(void) { return OTFX_ABI_VERSION; }

const char* otfx_last_error(void) { return g_err.c_str(); }

int otfx_release_cached_memory(void) {
  API_BEGIN
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (auto& pr : g_pools) {
    CK(cudaSetDevice(pr.first));
    CK(cudaDeviceSynchronize());
    CK(cudaMemPoolTrimTo(pr.second, 0));
  }
  API_END
}

int otfx_host_prefault(void* p, size_t bytes) {
  API_BEGIN
  require(p != nullptr || bytes == 0, OTFX_EINVAL, "null buffer");
  const long pages = long((bytes + 4095) / 4096);
  volatile char* c = static_cast<volatile char*>(p);
#pragma omp parallel for schedule(static) if (pages > 256)
  for (long q = 0; q < pages; ++q) c[size_t(q) * 4096] = 0;
  API_END
}

int otfx_device_count(int* count) {
  API_BEGIN
  require(count != nullptr, OTFX_EINVAL, "null pointer");
  int c = 0;
  cudaError_t err = cudaGetDeviceCount(&c);
  if (err != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *count = c;
  API_END
}

int otfx_engine_create(const otfx_engine_desc* desc, otfx_engine** out) {
  API_BEGIN
  require(out != nullptr, OTFX_EINVAL, "null output pointer");
  *out = nullptr;
  std::unique_ptr<otfx_engine> e(new otfx_engine());
  try {
    create(desc, e.get());
  } catch (...) {
    destroy(e.get());
    throw;
  }
  *out = e.release();
  API_END
}

int otfx_engine_destroy(otfx_engine* e) {
  API_BEGIN
  if (e) {
    destroy(e);
    delete e;
  }
  API_END
}

int otfx_engine_get_info(otfx_engine* e, otfx_engine_info* info) {
  API_BEGIN
  require(e && info, OTFX_EINVAL, "null pointer");
  info->state_bytes = int64_t(e->state_bytes);
  info->total_bytes = int64_t(e->total_bytes);
  info->np = e->NP;
  info->nws = e->NWS;
  info->lmax = e->LMAX;
  info->pitch = e->pitch;
  info->tile_cols = e->use_tma ? e->L.tile : e->TX;
  info->tile_rows = e->R;
  info->grid_x = e->gx;
  info->grid_y = e->gy;
  info->regs_plain = e->ops64 ? e->ops64->sweep_regs(false) : e->ops32->sweep_regs(false);
  info->regs_check = e->ops64 ? e->ops64->sweep_regs(true) : e->ops32->sweep_regs(true);
  info->graphs = e->use_graphs ? 1 : 0;
  info->tma_stages = e->use_tma ? e->L.S : 0;
  info->smem_bytes = e->use_tma ? e->L.total : int(e->smem_plain);
  info->cluster_ctas = cluster_ok(e) ? e->cl_ctas : 0;
  info->halo_overlap = overlap_ready(e) ? 1 : 0;
  if (e->use_tma) {
    info->regs_plain = e->ops64 ? e->ops64->tma_regs(false) : e->ops32->tma_regs(false);
    info->regs_check = e->ops64 ? e->ops64->tma_regs(true) : e->ops32->tma_regs(true);
  }
  API_END
}

static PackMap marginals_map(const otfx_engine* e) {
  PackMap m = potential_pack(e, e->d.kind >= OTFX_KIND_MATRIX_REAL);
  if (e->d.kind == OTFX_KIND_VECTOR) {
    for (int c = 0; c < e->K; ++c) add_mass(m, c);
  } else if (e->d.kind >= OTFX_KIND_MATRIX_REAL) {
    for (int a = 0; a < e->K; ++a) add_mass(m, 2 * (a * e->K + a));
  }
  return m;
}

static void take_marginal_sums(otfx_engine* e, double sums[3], double masses[2]) {
  e->diff_norm_own = std::sqrt(sums[2]);
  allreduce_host(e, sums, 3);
  e->diff_norm = std::sqrt(sums[2]);
  if (masses) {
    masses[0] = sums[0];
    masses[1] = sums[1];
  }
}

int otfx_engine_set_marginals(otfx_engine* e, const double* l0, const double* l1, double masses[2]) {
  API_BEGIN
  require(e && l0 && l1, OTFX_EINVAL, "null pointer");
  CK(cudaSetDevice(e->d.device));
  double sums[3];
  host_to_planes(e, l0, l1, marginals_map(e), e->diff, sums);
  take_marginal_sums(e, sums, masses);
  API_END
}

int otfx_engine_set_marginals_device(otfx_engine* e, const double* l0, const double* l1,
                                     double masses[2], void* stream) {
  API_BEGIN
  require(e && l0 && l1, OTFX_EINVAL, "null pointer");
  CK(cudaSetDevice(e->d.device));
  check_device_ptr(e, l0);
  check_device_ptr(e, l1);
  stream_wait(e->stream, static_cast<cudaStream_t>(stream), e->ev_hand);
  double sums[3];
  device_to_planes(e, l0, l1, marginals_map(e), e->diff, sums);  // synchronises e->stream
  take_marginal_sums(e, sums, masses);
  API_END
}

int otfx_engine_set_state_device(otfx_engine* e, const double* ux, const double* uy,
                                 const double* w, const double* phi, void* stream) {
  API_BEGIN
  require(e && ux && uy && phi, OTFX_EINVAL, "null pointer");
  require(!e->has_w || w, OTFX_EINVAL, "channel flux missing");
  CK(cudaSetDevice(e->d.device));
  for (const double* p : {ux, uy, w, phi}) check_device_ptr(e, p);
  zero_state(e);
  const cudaStream_t caller = static_cast<cudaStream_t>(stream);
  stream_wait(e->stream, caller, e->ev_hand);
  const int c = e->cur;
  PackMap pm = potential_pack(e, e->d.kind == OTFX_KIND_MATRIX_COMPLEX);
  device_to_planes(e, ux, nullptr, pm, e->u[c], nullptr);
  device_to_planes(e, uy, nullptr, pm, plane_ptr(e, e->u[c], e->NP), nullptr);
  device_to_planes(e, phi, nullptr, pm, e->phi[c], nullptr);
  if (e->has_w) device_to_planes(e, w, nullptr, flux_w_pack(e), e->w[c], nullptr);
  exchange_nccl(e);
  stream_wait(caller, e->stream, e->ev_hand);
  API_END
}

int otfx_engine_get_state_device(otfx_engine* e, double* ux, double* uy, double* w, double* phi,
                                 void* stream) {
  API_BEGIN
  require(e, OTFX_EINVAL, "null engine");
  CK(cudaSetDevice(e->d.device));
  for (const double* p : {ux, uy, w, phi}) check_device_ptr(e, p);
  const cudaStream_t caller = static_cast<cudaStream_t>(stream);
  stream_wait(e->stream, caller, e->ev_hand);
  const int c = e->cur;
  UnpackMap pm = potential_unpack(e);
  if (ux) planes_to_device(e, e->u[c], pm, ux);
  if (uy) planes_to_device(e, plane_ptr(e, e->u[c], e->NP), pm, uy);
  if (phi) planes_to_device(e, e->phi[c], pm, phi);
  if (w && e->has_w) planes_to_device(e, e->w[c], flux_w_unpack(e), w);
  stream_wait(caller, e->stream, e->ev_hand);
  API_END
}

int otfx_engine_set_diff(otfx_engine* e, const double* diff) {
  API_BEGIN
  require(e && diff, OTFX_EINVAL, "null pointer");
  CK(cudaSetDevice(e->d.device));
  PackMap m = potential_pack(e, e->d.kind == OTFX_KIND_MATRIX_COMPLEX);
  double sums[3];
  host_to_planes(e, diff, nullptr, m, e->diff, sums);
  e->diff_norm_own = std::sqrt(sums[2]);
  allreduce_host(e, sums, 3);
  e->diff_norm = std::sqrt(sums[2]);
  API_END
}

int otfx_engine_diff_norm(otfx_engine* e, double* get, const double* set) {
  API_BEGIN
  require(e, OTFX_EINVAL, "null engine");
  if (get) *get = e->diff_norm;
  if (set) e->diff_norm = *set;
  API_END
}

int otfx_engine_zero_state(otfx_engine* e) {
  API_BEGIN
  require(e, OTFX_EINVAL, "null engine");
  CK(cudaSetDevice(e->d.device));
  zero_state(e);
  API_END
}

int otfx_engine_set_state(otfx_engine* e, const double* ux, const double* uy, const double* w,
                          const double* phi) {
  API_BEGIN
  require(e && ux && uy && phi, OTFX_EINVAL, "null pointer");
  require(!e->has_w || w, OTFX_EINVAL, "channel flux missing");
  CK(cudaSetDevice(e->d.device));
  zero_state(e);
  const int c = e->cur;
  PackMap pm = potential_pack(e, e->d.kind == OTFX_KIND_MATRIX_COMPLEX);
  double sums[3];
  host_to_planes(e, ux, nullptr, pm, e->u[c], sums);
  host_to_planes(e, uy, nullptr, pm, plane_ptr(e, e->u[c], e->NP), sums);
  host_to_planes(e, phi, nullptr, pm, e->phi[c], sums);
  if (e->has_w) host_to_planes(e, w, nullptr, flux_w_pack(e), e->w[c], sums);
  exchange_nccl(e);
  CK(cudaStreamSynchronize(e->stream));
  API_END
}

int otfx_engine_get_state(otfx_engine* e, double* ux, double* uy, double* w, double* phi) {
  API_BEGIN
  require(e, OTFX_EINVAL, "null engine");
  CK(cudaSetDevice(e->d.device));
  const int c = e->cur;
  UnpackMap pm = potential_unpack(e);
  if (ux) planes_to_host(e, e->u[c], pm, ux);
  if (uy) planes_to_host(e, plane_ptr(e, e->u[c], e->NP), pm, uy);
  if (phi) planes_to_host(e, e->phi[c], pm, phi);
  if (w && e->has_w) planes_to_host(e, e->w[c], flux_w_unpack(e), w);
  API_END
}

int otfx_engine_step(otfx_engine* e, int64_t iters) {
  API_BEGIN
  require(e, OTFX_EINVAL, "null engine");
  require(iters >= 0, OTFX_EINVAL, "negative iteration count");
  CK(cudaSetDevice(e->d.device));
  if (cluster_ok(e) && iters > 0 && iters < (int64_t(1) << 30)) launch_cluster(e, nullptr, iters);
  else run_plain(e, iters);
  e->residual_valid = false;
  API_END
}

int otfx_engine_sweep(otfx_engine* e, int check) {
  API_BEGIN
  require(e, OTFX_EINVAL, "null engine");
  CK(cudaSetDevice(e->d.device));
  launch_sweep(e, check != 0 ? 1 : 0);
  e->residual_valid = check != 0;
  API_END
}

int otfx_engine_evaluate(otfx_engine* e, double out[4]) {
  API_BEGIN
  require(e && out, OTFX_EINVAL, "null pointer");
  CK(cudaSetDevice(e->d.device));
  raw_to_host(e, false, rank_comm(e));
  double r[5];
  finalize(e, e->h_raw, r);
  for (int q = 0; q < 4; ++q) out[q] = r[q];
  API_END
}

int otfx_engine_step_check(otfx_engine* e, double out[5]) {
  API_BEGIN
  require(e && out, OTFX_EINVAL, "null pointer");
  CK(cudaSetDevice(e->d.device));
  sweep_exchange(e, 1);
  raw_to_host(e, true, rank_comm(e));
  finalize(e, e->h_raw, out);
  API_END
}

int otfx_engine_raw(otfx_engine* e, int with_residual, double raw[OTFX_NRAW]) {
  API_BEGIN
  require(e && raw, OTFX_EINVAL, "null pointer");
  require(!with_residual || e->residual_valid, OTFX_EINVAL, "no check sweep since the last step");
  CK(cudaSetDevice(e->d.device));
  raw_to_host(e, with_residual != 0, nullptr);
  for (int q = 0; q < OTFX_NRAW; ++q) raw[q] = e->h_raw[q];
  API_END
}

int otfx_engine_finalize(otfx_engine* e, const double raw[OTFX_NRAW], double out[5]) {
  API_BEGIN
  require(e && raw && out, OTFX_EINVAL, "null pointer");
  finalize(e, raw, out);
  API_END
}

int otfx_engine_run(otfx_engine* e, const otfx_run_config* cfg, otfx_history_point* hist,
                    int64_t capacity, int64_t* n_history, int64_t* iterations, int* converged,
                    double* wall_seconds) {
  API_BEGIN
  require(e && cfg && n_history && iterations && converged, OTFX_EINVAL, "null pointer");
  require(cfg->max_iters >= 1 && cfg->check_every >= 1, OTFX_EINVAL,
          "max_iters and check_every must be >= 1");
  CK(cudaSetDevice(e->d.device));
  const auto t0 = std::chrono::steady_clock::now();
  if (cluster_ok(e) && cfg->check_every < (int64_t(1) << 30) &&
      cfg->max_iters / cfg->check_every + 2 <=
                           int64_t(e->stage_bytes / (6 * sizeof(double)))) {
    // the whole run loop on the device, one launch
    launch_cluster(e, cfg, 0);
    long long res[4];
    CK(cudaMemcpyAsync(res, e->d_result, sizeof(res), cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    require(res[1] >= 1, OTFX_ECUDA, "on-chip solve returned no history");
    e->history.resize(size_t(res[1]));
    static_assert(sizeof(otfx_history_point) == 6 * sizeof(double), "history row layout");
    CK(cudaMemcpyAsync(e->history.data(), e->d_stage, e->history.size() * sizeof(otfx_history_point),
                       cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    copy_history(e, hist, capacity, n_history);
    *iterations = res[0];
    *converged = int(res[2]);
    e->residual_valid = false;
    if (wall_seconds)
      *wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return OTFX_OK;
  }
  run_loop(SlabGroup{&e, 1}, cfg, hist, capacity, n_history, iterations, converged);
  if (wall_seconds)
    *wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  API_END
}

int otfx_engines_run_local(otfx_engine* const* es, int count, const otfx_run_config* cfg,
                           otfx_history_point* hist, int64_t capacity, int64_t* n_history,
                           int64_t* iterations, int* converged) {
  return otfx_engines_run_local_nccl(es, count, nullptr, cfg, hist, capacity, n_history,
                                     iterations, converged);
}

int otfx_engines_run_local_nccl(otfx_engine* const* es, int count, otfx_comm* loop,
                                const otfx_run_config* cfg, otfx_history_point* hist,
                                int64_t capacity, int64_t* n_history, int64_t* iterations,
                                int* converged) {
  API_BEGIN
  if (loop)
    require(loop->nranks == 1 && loop->device == es[0]->d.device, OTFX_EINVAL,
            "the loopback communicator must be a one-rank communicator on the slabs' device");
  require(es && count >= 1 && cfg && n_history && iterations && converged, OTFX_EINVAL,
          "null pointer");
  require(cfg->max_iters >= 1 && cfg->check_every >= 1, OTFX_EINVAL,
          "max_iters and check_every must be >= 1");
  for (int q = 0; q < count; ++q) {
    require(es[q]->nranks == 1, OTFX_EINVAL, "local slab groups cannot carry a communicator");
    require(es[q]->d.row_begin == (q ? es[q - 1]->d.row_end : 0) &&
                (q + 1 < count || es[q]->d.row_end == es[q]->d.n),
            OTFX_EINVAL, "engines must be the slabs of one grid, in order");
  }
  CK(cudaSetDevice(es[0]->d.device));
  run_loop(SlabGroup{es, count, loop ? loop->comm : nullptr}, cfg, hist, capacity, n_history,
           iterations, converged);
  API_END
}

int otfx_engine_history(otfx_engine* e, otfx_history_point* hist, int64_t capacity,
                        int64_t* n_history) {
  API_BEGIN
  require(e && n_history, OTFX_EINVAL, "null pointer");
  copy_history(e, hist, capacity, n_history);
  API_END
}

int otfx_engine_residual_between(otfx_engine* e, const double* ux0, const double* uy0,
                                 const double* w0, const double* phi0, const double* ux1,
                                 const double* uy1, const double* w1, const double* phi1,
                                 double* out) {
  API_BEGIN
  require(e && ux0 && uy0 && phi0 && ux1 && uy1 && phi1 && out, OTFX_EINVAL, "null pointer");
  require(!e->has_w || (w0 && w1), OTFX_EINVAL, "channel flux missing");
  require(e->rows == e->d.n, OTFX_EINVAL, "residual_between needs a whole-grid engine");
  CK(cudaSetDevice(e->d.device));
  zero_state(e);
  PackMap pm = potential_pack(e, e->d.kind == OTFX_KIND_MATRIX_COMPLEX);
  double sums[3];
  const double* src[2][4] = {{ux0, uy0, w0, phi0}, {ux1, uy1, w1, phi1}};
  for (int s = 0; s < 2; ++s) {
    host_to_planes(e, src[s][0], nullptr, pm, e->u[s], sums);
    host_to_planes(e, src[s][1], nullptr, pm, plane_ptr(e, e->u[s], e->NP), sums);
    host_to_planes(e, src[s][3], nullptr, pm, e->phi[s], sums);
    if (e->has_w) host_to_planes(e, src[s][2], nullptr, flux_w_pack(e), e->w[s], sums);
  }
  if (e->elem == 8) {
    SweepArgs<double> a = make_args<double>(e, 0);
    a.partials = e->d_part_eval;
    a.maxes = e->d_max_eval;
    CK(e->ops64->residual(a, dim3(e->ex, e->ey), dim3(128), e->stream));
  } else {
    SweepArgs<float> a = make_args<float>(e, 0);
    a.partials = e->d_part_eval;
    a.maxes = e->d_max_eval;
    CK(e->ops32->residual(a, dim3(e->ex, e->ey), dim3(128), e->stream));
  }
  reduce_raw_kernel<<<1, 256, 0, e->stream>>>(e->d_part_eval, e->d_max_eval, e->ex * e->ey,
                                               e->d_part_sweep, 0, 0, e->d_raw);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(e->h_raw, e->d_raw, OTFX_NRAW * sizeof(double), cudaMemcpyDeviceToHost,
                     e->stream));
  CK(cudaStreamSynchronize(e->stream));
  const double* r = e->h_raw;
  double v = r[0] / e->d.mu + r[2] / e->d.tau;
  if (e->has_w) v += r[1] / e->d.nu;
  *out = v - 2.0 * r[3];
  zero_state(e);
  API_END
}

int otfx_engine_exchange_local(otfx_engine* const* es, int count) {
  API_BEGIN
  require(es && count >= 1, OTFX_EINVAL, "no engines");
  CK(cudaSetDevice(es[0]->d.device));
  exchange_local_impl(es, count, es[0]->stream);
  API_END
}

int otfx_nccl_unique_id(unsigned char id[128]) {
  API_BEGIN
  require(id, OTFX_EINVAL, "null pointer");
  ncclUniqueId u;
  NK(nccl().GetUniqueId(&u));
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  memcpy(id, &u, 128);
  API_END
}

int otfx_engine_attach_nccl(otfx_engine* e, const unsigned char id[128], int nranks, int rank) {
  API_BEGIN
  require(e && id, OTFX_EINVAL, "null pointer");
  require(nranks >= 1 && rank >= 0 && rank < nranks, OTFX_EINVAL, "bad rank");
  CK(cudaSetDevice(e->d.device));
  ncclUniqueId u;
  memcpy(&u, id, 128);
  require(!e->comm, OTFX_EINVAL, "engine already has a communicator");
  NK(nccl().CommInitRank(&e->comm, nranks, u, rank));
  e->own_comm = true;
  e->nranks = nranks;
  e->rank = rank;
  drop_graphs(e);
  API_END
}

int otfx_comm_create(const unsigned char id[128], int nranks, int rank, int device,
                     otfx_comm** out) {
  API_BEGIN
  require(id && out, OTFX_EINVAL, "null pointer");
  require(nranks >= 1 && rank >= 0 && rank < nranks, OTFX_EINVAL, "bad rank");
  CK(cudaSetDevice(device));
  ncclUniqueId u;
  memcpy(&u, id, 128);
  auto* c = new otfx_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  try {
    NK(nccl().CommInitRank(&c->comm, nranks, u, rank));
  } catch (...) {
    delete c;
    throw;
  }
  *out = c;
  API_END
}

int otfx_comm_destroy(otfx_comm* c) {
  API_BEGIN
  if (c) {
    if (c->comm && nccl().CommDestroy) nccl().CommDestroy(c->comm);
    delete c;
  }
  API_END
}

int otfx_engine_attach_comm(otfx_engine* e, otfx_comm* c) {
  API_BEGIN
  require(e && c, OTFX_EINVAL, "null pointer");
  require(!e->comm, OTFX_EINVAL, "engine already has a communicator");
  require(c->device == e->d.device, OTFX_EINVAL, "communicator and engine on different devices");
  e->comm = c->comm;
  e->own_comm = false;
  e->nranks = c->nranks;
  e->rank = c->rank;
  drop_graphs(e);
  API_END
}

int otfx_engine_timing(otfx_engine* e, int enable, double* plain_ms, int64_t* plain_sweeps) {
  API_BEGIN
  require(e, OTFX_EINVAL, "null engine");
  CK(cudaStreamSynchronize(e->stream));
  collect_timing(e);
  // report what was accumulated so far, then (enable >= 0) reset and start/stop
  if (plain_ms) *plain_ms = e->plain_ms;
  if (plain_sweeps) *plain_sweeps = e->plain_sweeps;
  if (enable >= 0) {
    e->timing = enable != 0;
    e->plain_ms = 0.0;
    e->plain_sweeps = 0;
  }
  API_END
}

int otfx_engine_sync(otfx_engine* e) {
  API_BEGIN
  require(e, OTFX_EINVAL, "null engine");
  CK(cudaStreamSynchronize(e->stream));
  API_END
}

void* otfx_engine_stream(otfx_engine* e) { return e ? static_cast<void*>(e->stream) : nullptr; }

}  // extern "C"
