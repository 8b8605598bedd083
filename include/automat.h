/*
 * automat.h -- C ABI of the B200 AutoMat library (libautomat.so).
 *
 * Plain C types only: pointers, sizes, POD structs.  This is the boundary
 * the reference's Python API sits on (the ctypes shim in
 * paper_2006_04391_b200/_lib.py binds exactly these symbols).  Every entry
 * point names the reference routine it replaces.
 *
 * Layouts
 *   SoA ("component-major"): element (c, b) of a batch of B items with k
 *   components lives at p[c * B + b].  Device entry points take SoA device
 *   pointers; *_host entry points take the reference's AoS host arrays
 *   ((B, 6), (B, m), (B, 6, 6) row-major, exactly what
 *   gsmkit.evaluator.evaluate_arrays receives and returns).
 *   Fields of the basic-scheme solver are component-first (6, Nx, Ny, Nz)
 *   like gsmkit.homogenize (homogenize.py:12-13).
 *
 * Errors: every function returns an am_status; am_last_error() gives a
 * thread-local message for the last failure on the calling thread.
 */
#ifndef AUTOMAT_H
#define AUTOMAT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- codes */
typedef enum am_status {
    AM_OK = 0,
    AM_ERR_CONFIG = 1,            /* evaluator.ConfigError (evaluator.py:31) */
    AM_ERR_NEWTON = 2,            /* odeint.NewtonDivergenceError (odeint.py:34, 415-416) */
    AM_ERR_SINGULAR = 3,          /* linalg.SingularMatrixError (linalg.py:20, 103-104) */
    AM_ERR_NOT_CONVERGED = 4,     /* homogenize.SolverError (homogenize.py:29-34, 466-471) */
    AM_ERR_CUDA = 5,
    AM_ERR_NCCL = 6,
    AM_ERR_ARG = 7,               /* ValueError on bad arguments */
    AM_ERR_NONFINITE = 8,         /* reference_update: non-finite tangent (homogenize.py:316-317) */
    AM_ERR_INTEGRATION = 9,       /* odeint.IntegrationError: substep cap / step underflow (odeint.py:30-31) */
    AM_ERR_RADIAL = 10            /* gsm.NewtonError: conventional radial return stalled (gsm.py:40, 377-378) */
} am_status;

/* per-voxel status bits written by the material kernel */
#define AM_VOXEL_NEWTON_FAILED 1u
#define AM_VOXEL_SINGULAR 2u
#define AM_VOXEL_NONFINITE 4u
#define AM_VOXEL_INTEGRATION 8u
#define AM_VOXEL_RADIAL 16u

/* ---------------------------------------------------------------- laws
 * A law is its two potentials; the potentials live on the device.
 * kind: AM_LAW_LINEAR_ELASTIC -> gsm.LinearElastic(E, nu)      (gsm.py:100-153)
 *       AM_LAW_MICHEL_SUQUET  -> gsm.MichelSuquet(params)      (gsm.py:210-256)
 */
enum { AM_LAW_LINEAR_ELASTIC = 0, AM_LAW_MICHEL_SUQUET = 1 };

typedef struct am_law {
    int32_t kind;
    int32_t reserved;
    double E, nu;                              /* both laws */
    double sigma_Y, H, eps0_dot, sigma_d, n;   /* MichelSuquetParams (gsm.py:156-174) */
} am_law;

/* ---------------------------------------------------------------- config
 * StrategyConfig (evaluator.py:35-74).  Order of the enums follows
 * STRATEGIES / INTEGRATORS / ERROR_MEASURES (evaluator.py:26-28).  This
 * build implements every combination the reference accepts: the automatic
 * and semi-automatic strategies with implicit-euler, ode12 and ode23,
 * ode23s (Rosenbrock) with the semi-automatic strategy, and the
 * conventional (radial return) implicit-Euler route.
 */
enum { AM_STRATEGY_CONVENTIONAL = 0, AM_STRATEGY_AUTOMATIC = 1, AM_STRATEGY_SEMI_AUTOMATIC = 2 };
enum { AM_INTEGRATOR_IMPLICIT_EULER = 0, AM_INTEGRATOR_ODE12 = 1, AM_INTEGRATOR_ODE23 = 2, AM_INTEGRATOR_ODE23S = 3 };
enum { AM_NEWTON_INTERNAL = 0, AM_NEWTON_STRESS = 1 };

typedef struct am_cfg {
    int32_t strategy;
    int32_t integrator;
    int32_t newton_mode;     /* resolved_newton_mode (evaluator.py:69-71) */
    int32_t max_newton;      /* 50 (odeint.py:371) */
    double newton_tol;       /* 1e-10 (odeint.py:404) */
    /* adaptive integrators (StepController, odeint.py:198-214) */
    int32_t error_measure;   /* 0 internal, 1 stress (evaluator.py:28) */
    int32_t max_substeps;    /* 10000 */
    double atol, rtol;       /* 1e-6, 1e-3 */
} am_cfg;

/* ---------------------------------------------------------------- library */
const char *am_last_error(void);
const char *am_version(void);
int am_device_count(int *count);
int am_set_device(int device);

/* Page-locked host memory for result arrays (cached pool; no reference
 * counterpart): the Python shim returns evaluate_arrays' outputs in such
 * blocks so the D2H copies land in them directly.  am_host_free returns a
 * block to the pool. */
int am_host_alloc(int64_t bytes, void **out);
int am_host_free(void *p);

/* ---------------------------------------------------------------- material points
 * am_eval_batch -- replaces gsmkit.evaluator.evaluate_arrays
 * (evaluator.py:206-248) for the automatic implicit-Euler route.
 * Device pointers, SoA, asynchronous on `stream` (cudaStream_t or NULL).
 *   eps_n, eps_np1: 6*B      a_n, a_out: m*B (m = 7 Michel-Suquet, 0 elastic)
 *   dt: B values, or NULL to use dt_scalar for every item
 *   sigma: 6*B   C: 36*B (C[(i*6+j)*B + b] = dsigma_i/deps_j) or NULL
 *   newton_iters (int32, B): implicit Euler: the per-point Newton count;
 *   adaptive integrators: accepted substeps (EvalResult.substeps)
 *   rejected (int32, B): rejected attempts of the adaptive integrators (0 for
 *   implicit Euler) / status (uint8, B) / flags (one uint32 that receives
 *   the OR of all status bits): each optional (NULL).
 * Returns AM_OK once the work is enqueued; per-voxel failures are reported
 * through status / flags (NewtonDivergenceError / SingularMatrixError are
 * raised from them by the caller, see am_eval_batch_host).
 */
int am_eval_batch(const am_law *law, const am_cfg *cfg, int64_t B,
                  const double *eps_n, const double *a_n, const double *eps_np1,
                  const double *dt, double dt_scalar, int want_tangent,
                  double *sigma, double *a_out, double *C,
                  int32_t *newton_iters, int32_t *rejected, uint8_t *status, uint32_t *flags, void *stream);

/* Per-kernel device time of the stress + tangent route (Newton kernel,
 * tangent kernel), from CUDA events on the launching stream around each
 * kernel (synchronises after every launch while on: a measurement mode).
 * enable 1 = on (reset), 0 = off, -1 = query; out (3, optional) = Newton
 * ms, tangent ms, launches.  No reference counterpart (roofline evidence). */
int am_k1_timing(int enable, double *out);

/*
 * am_eval_batch_host -- same as evaluate_arrays with the reference's host
 * AoS arrays: eps_n/eps_np1 (B,6), a_n/a_out (B,m), dt (B), sigma (B,6),
 * C (B,6,6) or NULL.  Pinned or pageable memory.  Synchronous.  The batch is
 * pipelined through the GPU in chunks over two streams (H2D | kernel | D2H).
 * Returns AM_ERR_NEWTON if any voxel's Newton failed (odeint.py:415-416),
 * AM_ERR_INTEGRATION if an adaptive integration hit a cap (odeint.py:
 * 690-691, 740-744), else AM_ERR_SINGULAR if any tangent LU was singular
 * (odeint.py:424), else AM_OK.  Outputs are written for every voxel.
 */
int am_eval_batch_host(const am_law *law, const am_cfg *cfg, int64_t B,
                       const double *eps_n, const double *a_n, const double *eps_np1,
                       const double *dt, int want_tangent,
                       double *sigma, double *a_out, double *C,
                       int32_t *newton_iters, int32_t *rejected, uint8_t *status);

/*
 * am_eval_batch_record_host -- evaluate_arrays with record_steps=True for the
 * adaptive integrators (EvalResult.steps, odeint.py:725-727): as
 * am_eval_batch_host (host AoS arrays, one launch), plus every attempt's
 * (step size, accepted) of point b at rec_h / rec_acc [offsets[b],
 * offsets[b+1]).  offsets (B + 1 entries) are the prefix sums of the
 * substeps + rejected counts of a previous evaluation of the same inputs
 * (results are deterministic).
 */
int am_eval_batch_record_host(const am_law *law, const am_cfg *cfg, int64_t B,
                              const double *eps_n, const double *a_n, const double *eps_np1,
                              const double *dt, int want_tangent,
                              double *sigma, double *a_out, double *C, int32_t *substeps, int32_t *rejected,
                              const int64_t *offsets, double *rec_h, uint8_t *rec_acc);

/*
 * am_constitutive_host -- module-level constitutive operations at B points
 * (gsm.stress / generalized_stress / evolution_rhs / rhs_jacobian /
 * rhs_strain_jacobian, gsm.py:574-602), evaluated by the same device AD
 * routines as the material kernel.  AoS host arrays: eps (B,6), a (B,m);
 * outputs sigma (B,6), A (B,m), f (B,m), dfda (B,m,m), dfde (B,m,6); any
 * output may be NULL.  Automatic strategy only; am_lawops_host (below)
 * covers every strategy and the tangents and is what the Python shim uses.
 */
int am_constitutive_host(const am_law *law, int64_t B, const double *eps, const double *a,
                         double *sigma, double *A, double *f, double *dfda, double *dfde);

/* ---------------------------------------------------------------- basic scheme
 * am_solver -- replaces gsmkit.homogenize.Homogenizer (homogenize.py:345-480)
 * on one GPU: the fields, per-phase internal states, cuFFT plans and
 * workspaces live on the device for the solver's lifetime.  A handle is
 * single-threaded (like Homogenizer).  Host field layout is component-first
 * (6, nx, ny, nz), C order, exactly the reference's.
 */
typedef struct am_solver am_solver;

typedef struct am_stepinfo {       /* homogenize.StepInfo (homogenize.py:337-342) */
    int32_t iterations;
    int32_t converged;
    double residual;               /* last history entry max(res, res_bc) */
    double mean_substeps;
    double ebar[6];                /* voxel mean of the returned (last evaluated) strain field,
                                      eps.mean() of homogenize.py:503 (sums per x plane, added in
                                      plane order: independent of the slab / GPU count) */
    double sig_bar[6];             /* voxel mean of the returned stress field (same order) */
} am_stepinfo;

enum { AM_FIELD_EPS = 0, AM_FIELD_EPS_N = 1, AM_FIELD_SIGMA = 2 };

/* Homogenizer.__init__ minus the reference (set with am_solver_set_reference):
 * ids (nx*ny*nz uint8, C order) index `laws`; state starts at zero
 * (VoxelGrid, homogenize.py:85-99). */
int am_solver_create(int nx, int ny, int nz, const uint8_t *ids, int nmat, const am_law *laws,
                     const am_cfg *cfg, am_solver **out);
/* The same solver over nslabs x-slabs driven from this process on the
 * current device (the distributed algorithm -- 2-D FFTs, all-to-all
 * transposes, 1-D FFTs over x -- with device copies as the transport; used to
 * test the multi-GPU code path on one GPU).  nslabs must divide nx and ny. */
int am_solver_create_slabs(int nx, int ny, int nz, const uint8_t *ids, int nmat, const am_law *laws,
                           const am_cfg *cfg, int nslabs, am_solver **out);
/* One x-slab per process (rank of nranks) on the current device, transposes
 * and reductions over an NCCL communicator (NVLink / NVSwitch).  `id128` is
 * an ncclUniqueId from am_nccl_unique_id on rank 0, broadcast by the caller.
 * Every rank passes the full ids array.  Host fields / states of this
 * handle are the rank's slab (6, nx/nranks, ny, nz). */
int am_nccl_unique_id(void *id128);
int am_solver_create_nccl(int nx, int ny, int nz, const uint8_t *ids, int nmat, const am_law *laws,
                          const am_cfg *cfg, const void *id128, int rank, int nranks, am_solver **out);
/* Fused transposes over NVLink for am_solver_create_nccl handles: export
 * this rank's spectrum buffers (128 bytes of CUDA IPC handles), gather them
 * from every rank (caller's transport, rank order) and import them; the
 * forward transpose then packs straight into the peers' buffers and the
 * inverse unpacks straight from them (one kernel each, no all-to-all).
 * Handles from am_solver_create_slabs use the same kernels on their
 * sibling slabs automatically. */
int am_solver_ipc_export(am_solver *h, void *out128);
int am_solver_ipc_import(am_solver *h, const void *all, int nranks);
/* slab decomposition of a handle: global slab count, first local slab, local slabs */
int am_solver_layout(am_solver *h, int *nslabs, int *first, int *nlocal);
int am_solver_destroy(am_solver *h);
/* Homogenizer.set_reference / .reference (homogenize.py:378-380) */
int am_solver_set_reference(am_solver *h, double lam, double mu);
int am_solver_get_reference(am_solver *h, double *lam, double *mu);
/* Homogenizer.ebar_n (homogenize.py:355) */
int am_solver_set_mean(am_solver *h, const double *ebar_n);
/* Homogenizer.solve_step (homogenize.py:425-472): converges the basic
 * scheme for one loading step; `history` (optional, history_cap entries)
 * receives max(res, res_bc) per iteration.  AM_ERR_NOT_CONVERGED after
 * max_iterations (SolverError), AM_ERR_NEWTON if a voxel's Newton failed.
 * The converged fields stay on the device (am_solver_get_field). */
int am_solver_solve_step(am_solver *h, const double *ebar_target, double dt, const uint8_t *free_mask,
                         double tol, int max_iterations, am_stepinfo *info, double *history, int history_cap);
/* Newton warm start inside solve_step (implicit Euler only; default off):
 * from the second basic-scheme iteration of a step on, each voxel's
 * Newton starts at its previous iterate's state instead of a_n.  Same
 * equations and tolerance (odeint.py:357-401), fewer iterations; results
 * agree with the cold start to round-off, not bit for bit.  No reference
 * counterpart (the reference always starts at a_n, odeint.py:371). */
int am_solver_set_warm_start(am_solver *h, int on);
/* Bits of *on: 1 if the solver's inverse transform reads the carried
 * spectrum through a cuFFT load callback (the 3-D inverse on one slab, every
 * slab's inverse x transform on x slabs; power-of-two voxel counts), 2 if
 * sigma's slab transposes ride on the 2-D transforms' store / load callbacks
 * (x slabs).  Both for power-of-two voxel counts from 128^3 on, or
 * AM_FFT_CALLBACK=1; fields bitwise those of the copy / pack-kernel paths.  No
 * reference counterpart (implementation detail of homogenize.py:458-460). */
int am_solver_fft_callback(const am_solver *h, int *on);
/* Homogenizer.commit_step (homogenize.py:474-480) for the solver's eps:
 * eps_n <- eps, ebar_n <- ebar and, if a solve_step converged since the
 * last commit, the internal state <- that step's state (evaluations in
 * between do not change what is committed) */
int am_solver_commit(am_solver *h, const double *ebar);
/* Homogenizer.evaluate_field (homogenize.py:389-421) of the device eps,
 * without tangent: sigma field; states to the evaluation slot
 * (am_solver_get_state pending = 2) */
int am_solver_evaluate(am_solver *h, double dt);
/* evaluate_field(want_tangent=True) fused with reference_update
 * (homogenize.py:509-513): Cbar (36, optional) = voxel mean of C,
 * lam_mu (2, optional) = reference_update(C field); C_out (optional, host
 * (N, 6, 6)) receives the tangent field itself.  C is reduced per (phase,
 * x plane, part) and summed in that order: Cbar does not depend on the slab
 * or GPU count.  States go to the evaluation slot. */
int am_solver_tangent_sweep(am_solver *h, double dt, double *Cbar, double *lam_mu, double *C_out);
/* host (6, nx_local, ny, nz): the whole grid for handles from
 * am_solver_create[_slabs], the rank's slab for am_solver_create_nccl */
int am_solver_get_field(am_solver *h, int which, double *out);
int am_solver_set_field(am_solver *h, int which, const double *in);
/* per-phase internal state, host (count, m); pending = 0 for the committed
 * state (VoxelGrid.state), 1 for the state of the last converged
 * solve_step, 2 for the state of the last am_solver_evaluate /
 * am_solver_tangent_sweep */
int am_solver_get_state(am_solver *h, int phase, int pending, double *out);
int am_solver_set_state(am_solver *h, int phase, const double *in);
int am_solver_phase_count(am_solver *h, int phase, int64_t *count);
int am_solver_synchronize(am_solver *h);
/* per-phase device time of solve_step iterations: out[0..4] = ms in the
 * material sweeps, D2Z, Fourier kernel + reduction, origin + Z2D, and the
 * iteration count; enable 1 = on (reset), 0 = off, -1 = query */
int am_solver_timing(am_solver *h, int enable, double *out);
int am_solver_stream(am_solver *h, void **stream);

/* ---------------------------------------------------------------- field operators (host arrays) */
/* GreenOperator(dims, ReferenceMaterial(lam, mu)).apply(tau) (homogenize.py:174-233) */
int am_green_apply_host(int nx, int ny, int nz, double lam, double mu, const double *tau, double *out);
/* equilibrium_residual(sig) (homogenize.py:241-267) */
int am_equilibrium_residual_host(int nx, int ny, int nz, const double *sig, double *res);
/* apply_isotropic(ref, eps) (homogenize.py:270-281), fields (6, N) */
int am_apply_isotropic_host(int64_t N, double lam, double mu, const double *eps, double *out);
/* reference_update(C_field) (homogenize.py:307-329), C (n, 6, 6) */
int am_reference_update_host(int64_t n, const double *C, double *lam, double *mu);

/*
 * am_lawops_host -- gsm.LawOps(law, strategy) (gsm.py:412-566) at B points:
 * strategy AM_STRATEGY_AUTOMATIC (device AD) or SEMI_AUTOMATIC /
 * CONVENTIONAL (hand partials, gsm.py:258-328; _ops_for maps conventional
 * to semi-automatic, gsm.py:574-577).  AoS host arrays: eps (B,6), a (B,m),
 * da (B,m,6) or NULL (frozen state: elastic tangent); outputs sigma (B,6),
 * A (B,m), f (B,m), dfda (B,m,m), dfde (B,m,6), C (B,6,6), any NULL.
 */
int am_lawops_host(const am_law *law, int strategy, int64_t B, const double *eps, const double *a,
                   const double *da, double *sigma, double *A, double *f, double *dfda, double *dfde,
                   double *C);

/* ---------------------------------------------------------------- diagnostics
 * am_probe_fp64_tflops -- sustained fp64 FMA throughput of the current
 * device (the roofline denominator of the material kernel; no reference
 * counterpart).
 */
int am_probe_fp64_tflops(int reps, double *tflops);

#ifdef __cplusplus
}
#endif
#endif /* AUTOMAT_H */
