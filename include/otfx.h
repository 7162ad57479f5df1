/*
 * otfx -- C ABI of the B200 (sm_100a) PDHG engine for vector- and
 * matrix-valued W1 optimal transport (arXiv 1712.10279).
 *
 * The reference (otflux, pure Python) has no FFI.  Its only plug point for the
 * hot path is the private engine protocol consumed by the run loop:
 *
 *   _Engine.__init__        /root/reference/pkg/src/otflux/solver.py:179-201
 *   _Engine.set_channel_bound                               solver.py:203-205
 *   _Engine.step            (one PDHG iteration)            solver.py:220-240
 *   _Engine.evaluate        (primal, dual, gap, feas)       solver.py:276-280
 *   _Engine.residual_from   (fixed-point residual R^k)      solver.py:282-291
 *   _run                    (check cadence, history, stop)  solver.py:294-337
 *   _load_state             (evaluate a given state)        solver.py:477-482
 *
 * Every entry point below replaces one of those; the Python host layer
 * (paper_1712_10279_b200/solver.py) keeps the reference's public solve_*
 * signatures and calls through this ABI with ctypes.
 *
 * Conventions: plain pointers and sizes only.  Host arrays are C-contiguous
 * float64 in the reference layout; complex arrays are complex128 (interleaved
 * re, im doubles).  A slab engine (row_begin, row_end) takes and returns only
 * its own rows.  Return value 0 = success, negative = error code below;
 * otfx_last_error() gives the message (thread-local).
 */
#ifndef OTFX_H_
#define OTFX_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OTFX_ABI_VERSION 2

/* error codes; the Python layer maps them onto the reference's exceptions
 * (S/errors.py:4-21) */
#define OTFX_OK 0
#define OTFX_EINVAL (-1)       /* ValidationError */
#define OTFX_EUNSUPPORTED (-2) /* UnsupportedNormError / unsupported size */
#define OTFX_ECUDA (-3)        /* NumericalError (device failure) */
#define OTFX_ENCCL (-4)        /* NumericalError (collective failure) */
#define OTFX_ENOMEM (-5)       /* NumericalError (device memory) */

/* payload kinds: S/solver.py:359-435 (the matrix kind splits into the real
 * and complex paths of solver.py:412-426) */
#define OTFX_KIND_SCALAR 0
#define OTFX_KIND_VECTOR 1
#define OTFX_KIND_MATRIX_REAL 2
#define OTFX_KIND_MATRIX_COMPLEX 3

/* norm families, S/shrink.py:33-37 */
#define OTFX_NORM_L2 0
#define OTFX_NORM_L12 1
#define OTFX_NORM_L1 2
#define OTFX_NORM_L1NUC 3

/* arithmetic precision of the device iterates */
#define OTFX_F64 0
#define OTFX_F32 1

/* raw per-slab check scalars (summed / maxed across slabs by the caller or
 * by the NCCL allreduce inside the engine) */
#define OTFX_NRAW 14
#define OTFX_NRAW_SUM 12

typedef struct otfx_engine otfx_engine;

/* Engine construction parameters (replaces _Engine.__init__ +
 * set_channel_bound, S/solver.py:179-205).  mu, nu, tau and inv_dx are the
 * host-computed step sizes, exactly as the reference computes them. */
typedef struct {
  int32_t kind;      /* OTFX_KIND_* */
  int32_t dtype;     /* OTFX_F64 / OTFX_F32 */
  int32_t n;         /* global grid side */
  int32_t k;         /* channels (vector) or matrix dimension; 1 for scalar */
  int32_t ell;       /* edges (vector) or Lindblad matrices; 0 for scalar */
  int32_t norm_u;    /* OTFX_NORM_* of the spatial flux */
  int32_t norm_w;    /* OTFX_NORM_* of the channel flux */
  int32_t device;    /* CUDA device ordinal */
  int32_t row_begin; /* owned global rows [row_begin, row_end) */
  int32_t row_end;
  double tau, mu, nu, alpha, eps_reg, inv_dx;
  /* channel operator: vector -> k x ell row-major D/c (S/graph.py:69);
   * matrix -> ell x k x k complex128 Lindblad stack (S/lindblad.py:87-129) */
  const double* chan;
  void* stream; /* cudaStream_t to run on; NULL = engine-owned stream */
} otfx_engine_desc;

/* one HistoryPoint (S/solver.py:133-141) */
typedef struct {
  double iteration, primal, dual, gap_ratio, feas_residual, residual;
} otfx_history_point;

/* run-loop controls (SolverConfig fields used by _run, S/solver.py:97-130) */
typedef struct {
  double tol_gap;
  double tol_feas;
  int64_t max_iters;
  int64_t check_every;
} otfx_run_config;

typedef struct {
  int64_t state_bytes;   /* device bytes of one iterate (u, w, phi) */
  int64_t total_bytes;   /* all device allocations */
  int32_t np, nws, lmax; /* reals per potential, per channel block, block capacity */
  int32_t pitch;         /* plane row pitch (elements) */
  int32_t tile_cols, tile_rows, grid_x, grid_y; /* sweep launch geometry */
  int32_t regs_plain, regs_check;               /* registers per thread */
  int32_t graphs;        /* CUDA graphs in use */
  int32_t tma_stages;    /* TMA ring depth of the streamed sweep (0: register sweep) */
  int32_t smem_bytes;    /* dynamic shared memory per sweep CTA */
  int32_t cluster_ctas;  /* > 0: run()/step() execute on chip in one cluster of this many CTAs */
  int32_t halo_overlap;  /* slab halo exchange overlapped with the interior bands when decomposed */
} otfx_engine_info;

int otfx_abi_version(void);
const char* otfx_last_error(void);
int otfx_device_count(int* count);
/* Engine memory comes from a per-device stream-ordered pool that keeps freed
 * blocks cached for the next engine (no reference counterpart: NumPy's
 * allocator plays this role in S/solver.py:179-201).  Returns the cached
 * blocks of every device to the driver. */
int otfx_release_cached_memory(void);

/* Payload sizes: scalar; vector k = 2..8 (compiled, any edge count) and
 * k = 9..32 with up to 128 edges (runtime-size kernels); matrix k = 2..4 with
 * ell <= 4 and k = 2, 3 with ell <= 8 (compiled), k <= 8 with ell * block
 * reals <= 256 beyond that (runtime-size).  Anything else returns
 * OTFX_EUNSUPPORTED before any device work. */
int otfx_engine_create(const otfx_engine_desc* desc, otfx_engine** out);
int otfx_engine_destroy(otfx_engine* e);
int otfx_engine_get_info(otfx_engine* e, otfx_engine_info* info);

/* diff = lambda0 - lambda1 formed on the device (S/solver.py:367, 384, 410),
 * plus the total masses used by _check_pair (S/solver.py:351-355).
 * scalar (rows,n) / vector (rows,n,k) float64 / matrix (rows,n,k,k) complex128 */
int otfx_engine_set_marginals(otfx_engine* e, const double* l0, const double* l1,
                              double masses[2]);
/* diff given directly, in the engine's payload layout (matrix real path:
 * float64 (rows,n,k,k); complex path: complex128) */
int otfx_engine_set_diff(otfx_engine* e, const double* diff);

/* Device-pointer hand-off (SURVEY §8(b) ownership row: torch owns the
 * tensors, the library reads / writes them in place and keeps no reference).
 * Same layouts and dtypes as the host calls, arrays resident on the engine's
 * device (e.g. torch.Tensor.data_ptr() of a contiguous float64 / complex128
 * CUDA tensor).  `stream` is the caller's cudaStream_t (NULL = legacy default
 * stream): the engine's work is ordered after the caller's prior work on it,
 * and the caller's later work after the engine's reads / writes (CUDA events,
 * no host synchronisation; set_marginals_device synchronises once to return
 * the masses and ||diff||).  Replace the host-array versions of
 * _Engine.__init__'s diff (S/solver.py:179-185), _load_state
 * (S/solver.py:477-482) and the state packing (S/solver.py:318-336). */
int otfx_engine_set_marginals_device(otfx_engine* e, const double* l0, const double* l1,
                                     double masses[2], void* stream);
int otfx_engine_set_state_device(otfx_engine* e, const double* ux, const double* uy,
                                 const double* w, const double* phi, void* stream);
int otfx_engine_get_state_device(otfx_engine* e, double* ux, double* uy, double* w, double* phi,
                                 void* stream);

/* ||diff|| used by the feasibility residual (S/solver.py:185, 246): read the
 * engine's value (its own rows, or the global one under NCCL) and/or
 * override it (local multi-slab drivers combine the slabs' values) */
int otfx_engine_diff_norm(otfx_engine* e, double* get, const double* set);

/* state I/O (S/solver.py:318-336 packing and :477-482 loading).
 * ux, uy, phi: payload layout as diff; w: vector (rows,n,ell) float64,
 * matrix (rows,n,ell,k,k) complex128 (QuantumFlux, S/fields.py:276-289).
 * w may be NULL for the scalar kind. */
int otfx_engine_zero_state(otfx_engine* e);
int otfx_engine_set_state(otfx_engine* e, const double* ux, const double* uy, const double* w,
                          const double* phi);
int otfx_engine_get_state(otfx_engine* e, double* ux, double* uy, double* w, double* phi);

/* Host helper for the state download: touch every page of a freshly
 * allocated host buffer (one write per 4 KiB page, OpenMP) so the page faults
 * are taken before otfx_engine_get_state writes it.  The Python drop-in runs
 * it on the output arrays of SolverState (S/solver.py:318-336) from a second
 * host thread while otfx_engine_run keeps the device busy (8192^2 vector,
 * 6.4 GB: download 0.217 s into fresh arrays, 0.129 s into faulted ones). */
int otfx_host_prefault(void* p, size_t bytes);

/* iterations (S/solver.py:220-240), halo exchange included when a
 * communicator is attached */
int otfx_engine_step(otfx_engine* e, int64_t iters);
/* primal, dual, gap_ratio, feas of the current iterate (S/solver.py:276-280) */
int otfx_engine_evaluate(otfx_engine* e, double out[4]);
/* one iteration followed by R^k and evaluate (S/solver.py:305-313):
 * out = primal, dual, gap_ratio, feas, residual */
int otfx_engine_step_check(otfx_engine* e, double out[5]);
/* the whole _run loop (S/solver.py:294-337) on the device.  The engine keeps
 * the run's whole history (the reference grows its list as it goes,
 * S/solver.py:300-333); the first `capacity` points are copied to `history`
 * (which may be NULL when capacity is 0) and n_history is the total, so a
 * caller whose buffer was too small fetches the rest with
 * otfx_engine_history. */
int otfx_engine_run(otfx_engine* e, const otfx_run_config* cfg, otfx_history_point* history,
                    int64_t capacity, int64_t* n_history, int64_t* iterations, int* converged,
                    double* wall_seconds);
/* the same run loop over the row slabs of one grid held by `count` engines on
 * one device and one stream (in row order), stepped in lockstep: the
 * single-GPU stand-in for the NCCL-connected ranks (same check cadence, fused
 * checks and stopping rule, and the same halo pack -> transport -> unpack as
 * exchange over NCCL, the transport being device copies between the slabs'
 * send / receive buffers).  The whole-grid ||diff|| is combined from the
 * slabs' own-row norms (overrides set with otfx_engine_diff_norm are not
 * used here). */
int otfx_engines_run_local(otfx_engine* const* engines, int count, const otfx_run_config* cfg,
                           otfx_history_point* history, int64_t capacity, int64_t* n_history,
                           int64_t* iterations, int* converged);

/* the same local slab group with the halo transport and the check-scalar
 * allreduces going through NCCL: `loopback` is a one-rank communicator
 * (otfx_comm_create with nranks = 1) on the slabs' device, and every halo
 * send / receive of exchange_nccl is posted to that rank itself -- the same
 * ncclSend / ncclRecv / ncclAllReduce calls, buffers, counts and datatypes the
 * multi-GPU ranks post, executed on a one-GPU machine.  NULL = device copies
 * (otfx_engines_run_local). */
typedef struct otfx_comm otfx_comm;
int otfx_engines_run_local_nccl(otfx_engine* const* engines, int count, otfx_comm* loopback,
                                const otfx_run_config* cfg, otfx_history_point* history,
                                int64_t capacity, int64_t* n_history, int64_t* iterations,
                                int* converged);

/* the history of the engine's last run (for a local slab group: the lead
 * engine's): the first `capacity` points into `history`, n_history = total */
int otfx_engine_history(otfx_engine* e, otfx_history_point* history, int64_t capacity,
                        int64_t* n_history);

/* fixed-point residual between two given iterates (residual_Rk,
 * S/solver.py:501-526), using the engine's mu, nu, tau; whole-grid engines */
int otfx_engine_residual_between(otfx_engine* e, const double* ux0, const double* uy0,
                                 const double* w0, const double* phi0, const double* ux1,
                                 const double* uy1, const double* w1, const double* phi1,
                                 double* out);

/* --- lower-level pieces used to drive several slabs from one process ---- */
/* one iteration kernel without halo exchange; check != 0 also accumulates
 * the R^k partial sums */
int otfx_engine_sweep(otfx_engine* e, int check);
/* per-slab raw scalars of the current iterate (with_residual: include the
 * R^k sums of the last check sweep) */
int otfx_engine_raw(otfx_engine* e, int with_residual, double raw[OTFX_NRAW]);
/* raw scalars (already combined across slabs) -> primal, dual, gap, feas, R^k */
int otfx_engine_finalize(otfx_engine* e, const double raw[OTFX_NRAW], double out[5]);
/* copy halo rows between engines of one process sharing one stream */
int otfx_engine_exchange_local(otfx_engine* const* engines, int count);

/* --- multi-GPU row slabs over NCCL (NVLink / NVSwitch) ------------------ */
int otfx_nccl_unique_id(unsigned char id[128]);
/* attach a communicator: ranks are slabs in row order (rank r owns the r-th
 * slab); the engine then exchanges halo rows after every iteration and
 * allreduces the check scalars */
int otfx_engine_attach_nccl(otfx_engine* e, const unsigned char id[128], int nranks, int rank);
/* a communicator that outlives engines: created once per process and rank,
 * attached (non-owning) to every engine of a series of solves, so the NCCL
 * setup is paid once rather than per solve */
int otfx_comm_create(const unsigned char id[128], int nranks, int rank, int device,
                     otfx_comm** out);
int otfx_comm_destroy(otfx_comm* c);
int otfx_engine_attach_comm(otfx_engine* e, otfx_comm* c);

/* device time of the plain-iteration graph launches (CUDA events on the
 * engine stream): returns the time / sweep count accumulated so far, then
 * enable = 1 resets and starts, 0 resets and stops, -1 leaves it running */
int otfx_engine_timing(otfx_engine* e, int enable, double* plain_ms, int64_t* plain_sweeps);

/* enqueue-side helpers for timing */
int otfx_engine_sync(otfx_engine* e);
void* otfx_engine_stream(otfx_engine* e);

#ifdef __cplusplus
}
#endif

#endif /* OTFX_H_ */
