/* =====================================================================================
 * include/pbe.h — C ABI of libpbe: the batched, B200-native explicit finite-volume
 * time-march of the 1D crystal population balance (PBE) coupled to the solute mass
 * balance, with fused forward-mode tangent lanes.
 *
 * Problem statement (arXiv 2411.00742, reference/PAPER.md):
 *   PBE                dn/dt + d(G n)/dL = 0               eq-PBE_batch_2d, L257-266 (1D reading)
 *   mass balance       dc/dt = -rho_c k_v d(mu_3)/dt        eq-mass_balance, L268-273
 *   IC / BC            n(t=0) = n0, n(L=0) = n(L=inf) = 0   L275-283
 *   supersaturation    S = c / c*(T)                        L285
 *   solubility         c* = a exp(b T)                      Eq. A.1
 *   growth             G = k1 exp(-k2/(T+273.15)) (S-1)^k3  Eq. A.2
 *                      G = sum_j a_j (S-1)^j                eq-poly_growth_rate, L565-571
 *   FVM update         eq-highRes_growth (L292-298) + van Leer limiter (SI L849-856)
 *   time step          dt = nu dL / |G|, nu = 0.9           SI L857-861, L301
 *   discrete balance   c^{n+1} = c^n - rho_c k_v (mu3^{n+1} - mu3^n)   L304-312
 *   moments            mu_k = sum_i dL L_i^k n_i            SI eq-moment2D L871-875
 *   forward-mode AD    tangents alongside primals           L341, L908-913
 *   loss               residual sum of squares              eq-loss L551-557, L764
 * Readings where the paper is silent are numbered R-1..R-25 in DESIGN.md.
 *
 * Units: um, min, degC, g/kg.  All physics is IEEE binary64.
 *
 * Conventions (all calls):
 *   - Ownership: the caller owns every pointer it passes; libpbe copies what it needs
 *     (kinetics, c0, sample times, targets, host n0) into context-owned device memory and
 *     keeps no caller pointer after a call returns, except that device output pointers
 *     passed to pbe_run_batch must stay valid until the stream reaches that point.
 *   - Errors: argument errors return PBE_ERR_ARG synchronously, with a message from
 *     pbe_last_error(ctx).  CUDA failures return PBE_ERR_CUDA; allocation failures
 *     PBE_ERR_NOMEM.  Numerical failures are PER SIMULATION (status codes below) and do
 *     not abort the batch: a failed simulation stops at the failing step (its recorded
 *     samples up to then are valid, later samples are NaN, its loss is NaN).
 *   - Threading: one host thread per context; a context is bound to one CUDA device.
 *   - Determinism: a simulation's results depend only on its own inputs, never on batch
 *     composition, scheduling or the number of GPUs (bitwise).
 * ===================================================================================== */
#ifndef PBE_H_
#define PBE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pbe_ctx_s* pbe_ctx;

typedef enum {
    PBE_OK = 0,
    PBE_ERR_ARG = 1,         /* invalid argument (synchronous) */
    PBE_ERR_CFL = 2,         /* per sim: fixed dt gave |C| > 1 */
    PBE_ERR_NEGATIVE = 3,    /* per sim: n < -1e-12 max(n0) after a step (R-17) */
    PBE_ERR_INFEASIBLE = 4,  /* per sim: c < 0 after a step */
    PBE_ERR_MAXSTEPS = 5,    /* per sim: max_steps reached before the last sample */
    PBE_ERR_CUDA = 6,        /* CUDA runtime failure */
    PBE_ERR_NOMEM = 7,       /* device allocation failure */
    PBE_ERR_STATE = 8        /* call out of order (e.g. run before set_kinetics) */
} pbe_status;

enum { PBE_LIM_UPWIND = 0, PBE_LIM_VANLEER = 1,         /* phi = 0 / van Leer (SI L855), the paper's */
       PBE_LIM_MINMOD = 2, PBE_LIM_SUPERBEE = 3, PBE_LIM_MC = 4 };  /* NEXT-4 extras (R-31) */
enum {
    PBE_LAW_CONST = 0,         /* G = theta0 (size- and S-independent; config C1)         */
    PBE_LAW_ARRHENIUS_GD = 1,  /* theta = (kg, Eg, g[, kd, Ed, d]): Eq. A.2 for S > 1;   */
                               /* S < 1: -kd exp(-Ed/(T+273.15)) (1-S)^d if 6 params (R-12) */
    PBE_LAW_POLY = 2           /* theta = (a1..ak): sum_j a_j (S-1)^j for S > 1, else 0    */
};
enum { PBE_SOL_EXP = 0 /* (a, b): a exp(bT) */, PBE_SOL_POLY = 1 /* (s0,s1,s2) (R-13) */ };
enum { PBE_MAX_PARAMS = 4096 };  /* kinetic parameters per simulation (POLY terms) */
enum {
    PBE_KERNEL_AUTO = 0,      /* choose by N and lanes              */
    PBE_KERNEL_RESIDENT = 1,  /* one CTA per sim, state in registers across all steps     */
    PBE_KERNEL_CLUSTER = 2,   /* thread-block cluster per sim, DSMEM halo + reduction     */
    PBE_KERNEL_STREAM = 3,    /* grid-wide persistent kernel, HBM streaming, grid barrier */
    PBE_KERNEL_2D = 4,        /* 2D model (set by n_bins2 > 0): grid-wide split-sweep kernel */
    PBE_KERNEL_ADJOINT = 5    /* reported by pbe_last_run_info after pbe_run_adjoint (NEXT-3) */
};

typedef struct {
    int32_t n_bins;      /* N >= 3 */
    double  L_lo;        /* bin i has center L_lo + (i + 1/2) dL (R-2) */
    double  dL;          /* > 0 */
    int32_t limiter;     /* PBE_LIM_*: phi(theta) of eq-highRes_growth; van Leer in the paper (L299-300) */
    double  courant;     /* nu in (0, 1]; the paper uses 0.9 (L301) */
    double  dt_fixed;    /* > 0: fixed-dt mode (|C| <= 1 checked per step); 0: CFL mode */
    double  dt_max;      /* CFL cap (> 0); INFINITY = the paper's uncapped CFL step */
    int64_t max_steps;   /* runaway guard (> 0) */
    int64_t n_steps;     /* > 0: steps mode: exactly n_steps steps, no sample landing, one
                            final record (config C4); 0: march to the last sample time */
    double  rho_c;       /* crystal density, g/um^3 (Table 1: 1.11e-12) */
    double  k_v;         /* shape factor (Table 1: pi/4) */
    int32_t n_samples;   /* M >= 1 sample times (must be 1 in steps mode) */
    int32_t n_tangents;  /* 0..10 forward-mode tangent lanes */
    int32_t max_sims;    /* capacity (>= n_sims of every later call) */
    int32_t kernel;      /* PBE_KERNEL_* (AUTO unless forcing a variant) */
    /* --- 2D model (NEXT-1; eq-PBE_batch_2d L257-266, Godunov splitting L291) ----------
     * n_bins2 > 0 selects the paper's 2D model: f(L1, L2) on n_bins x n_bins2 cells, L2 bin j
     * centered at L2_lo + (j + 1/2) dL2; each step sweeps every row along L1 then every
     * column along L2 (eq-highRes_growth), dt = nu min(dL1/|G1|, dL2/|G2|) (SI L859), mass
     * balance on mu_12 = sum dL1 dL2 L1 L2^2 f (L271, L304-312).  In 2D mode: kinetics theta
     * = [dimension-1 law | dimension-2 law] (n_params even), n_tangents must be 0, n0 /
     * n_final are [sims][n_bins2][n_bins] (L1 fastest), and pbe_moments records are
     * [sims][M][8] = (t, c, mu00, mu10, mu01, mu11, mu02, mu12).  0 = 1D. */
    int32_t n_bins2;
    double  L2_lo;
    double  dL2;
} pbe_config;

/* Creates a context on CUDA device `device` and allocates its device scratch for
 * max_sims simulations.  Returns PBE_ERR_ARG for an invalid config (message available
 * through pbe_last_error(NULL) on this thread), PBE_ERR_CUDA / PBE_ERR_NOMEM otherwise. */
pbe_status pbe_create(const pbe_config* cfg, int device, pbe_ctx* out);

/* Frees every device allocation of the context.  NULL is a no-op. */
void pbe_destroy(pbe_ctx ctx);

/* Last error message of the context (or of this thread's last pbe_create if ctx is
 * NULL).  Valid until the next call on the same context/thread. */
const char* pbe_last_error(pbe_ctx ctx);

/* Kinetics of the next runs (row a1).
 *   theta        host [n_sims][n_params]   per-simulation kinetic parameters; n_params is 1
 *                (CONST), 3 or 6 (ARRHENIUS_GD), 1..PBE_MAX_PARAMS (POLY: the paper grows
 *                the polynomial to scale the parameter count, L565-572, L599)
 *   sol_params   host [n_sol]              solubility parameters (shared)
 *   knot_t       host [n_knots]            temperature-profile times (strictly increasing)
 *   knot_T       host [n_knots] or [n_sims][n_knots] (knot_T_per_sim = 0 / 1); T(t) is
 *                piecewise linear through the knots, constant outside (R-14)
 *   tangent_seed host [n_tangents][n_params + n_sol] or NULL (= unit vectors e_0..e_{P-1}
 *                over theta).  Lane p differentiates along seed[p] (R-20).
 * Copied to the device (synchronously); the pointers are not retained.  If a run is still in
 * flight, this call first waits for it (cudaStreamSynchronize of the last run's stream), so
 * kinetics are never replaced under a running kernel. */
pbe_status pbe_set_kinetics(pbe_ctx ctx, int32_t law, int32_t n_params, int32_t n_sims,
                            const double* theta, int32_t sol_kind, int32_t n_sol,
                            const double* sol_params, int32_t n_knots, const double* knot_t,
                            const double* knot_T, int32_t knot_T_per_sim,
                            const double* tangent_seed);

/* Enqueues the whole march of n_sims simulations on `cuda_stream` (a cudaStream_t; NULL =
 * legacy default stream) and returns (rows a1-a8).
 *   n0          [n_sims][N] (n0_stride = N) or one shared row (n0_stride = 0); device
 *               memory if n0_on_device, else host memory (copied H2D on the stream)
 *   c0          host [n_sims] initial concentrations (>= 0)
 *   t_samples   host [n_samples] strictly increasing, > 0 (ignored in steps mode)
 *   target      host [n_sims][n_samples][2] = measured (c, mean length mu1/mu0) for the
 *               RSS loss (R-23), or NULL (no loss; must be NULL for the 2D model: PBE_ERR_ARG)
 *   n_final     device [n_sims][N] final distributions, or NULL
 *   ndot_final  device [n_sims][n_tangents][N] final tangent distributions, or NULL
 * Validates n0 only for shape/pointers (non-negativity of device n0 is the caller's).
 * The context's input/output buffers are reused: a run enqueued on a different stream than
 * the previous run first waits (cudaStreamWaitEvent) for the previous run's kernel. */
pbe_status pbe_run_batch(pbe_ctx ctx, int32_t n_sims, const double* n0, int64_t n0_stride,
                         int32_t n0_on_device, const double* c0, const double* t_samples,
                         const double* target, double* n_final, double* ndot_final,
                         void* cuda_stream);

/* Synchronizes the last run's stream and copies its records (rows a5-a7):
 *   moments   [n_sims][M][6] = (t, c, mu0, mu1, mu2, mu3) at each sample (NaN if not reached)
 *   status    [n_sims] int32 pbe_status per simulation
 *   steps     [n_sims] int64 time steps taken
 *   loss      [n_sims] RSS objective, or NULL (NaN when no target was given)
 * on_device != 0: the destinations are device pointers (same device), else host. */
pbe_status pbe_moments(pbe_ctx ctx, double* moments, int32_t* sim_status, int64_t* sim_steps,
                       double* loss, int32_t on_device);

/* Tangent records of the last run (row a8):
 *   tangents  [n_sims][M][n_tangents][5] = d(c, mu0, mu1, mu2, mu3)/d(seed direction)
 *   grad      [n_sims][n_tangents] = d loss / d(seed direction), or NULL */
pbe_status pbe_tangents(pbe_ctx ctx, double* tangents, double* grad, int32_t on_device);

/* Reverse-mode gradient (NEXT-3; jax.grad with checkpointing, "for
 * 1000 parameters specifically, jax-AD is 40x faster than jax-ND"): d loss / d theta for ALL
 * n_params kinetic parameters of every simulation at the cost of about four primal marches,
 * independent of n_params (tangent lanes cost one lane per direction).  The discrete adjoint
 * of exactly the march pbe_run_batch performs: same steps, same branch decisions (sample
 * landing, dt cap, clip), derivatives equal to pbe_tangents' up to rounding.
 *   n0, n0_stride, n0_on_device, c0, t_samples: as pbe_run_batch
 *   target            host [n_sims][n_samples][2] (required: the loss R-23 is differentiated)
 *   checkpoint_every  store the distribution every K steps (0: K = ceil(sqrt(max_steps))); K is
 *                     capped so that a segment's trace rows (and, when they fit, its K + 1
 *                     states) are staged in shared memory; device memory per simulation =
 *                     8 B x (16 max_steps + N ceil(max_steps / K) [+ N (K + 1) if the states
 *                     do not fit shared memory]) -- max_steps bounds the trace
 * Restrictions (PBE_ERR_ARG): 1D model, sample mode (n_steps = 0), N <= 6144.  The gradient is
 * w.r.t. theta only (not the solubility parameters).  Launches k_adjoint (one CTA per simulation)
 * and k_adjoint_theta (dL/dtheta from the per-step trace, grid over parameters x simulations).
 * Records, status, steps and loss of the forward pass are read with pbe_moments. */
pbe_status pbe_run_adjoint(pbe_ctx ctx, int32_t n_sims, const double* n0, int64_t n0_stride,
                           int32_t n0_on_device, const double* c0, const double* t_samples,
                           const double* target, int32_t checkpoint_every, void* cuda_stream);

/* Result of the last pbe_run_adjoint (synchronizes its stream):
 *   grad  [n_sims][n_params] d loss / d theta (NaN for a simulation whose march failed)
 *   loss  [n_sims] or NULL */
pbe_status pbe_adjoint_gradient(pbe_ctx ctx, double* grad, double* loss, int32_t on_device);

/* Introspection for tests and the benchmark harness. */
typedef struct {
    int32_t kernel;          /* PBE_KERNEL_* variant that ran */
    int32_t launches;        /* number of libpbe kernels launched by the last pbe_run_batch */
    int32_t threads_per_cta; /* CTA size of the main kernel */
    int32_t ctas;            /* grid size of the main kernel */
    int32_t cluster;         /* cluster size (1 if none) */
    int32_t bins_per_thread; /* register-resident bins per thread (0 if streaming) */
    double  main_ms;         /* CUDA-event duration of the main kernel of the last run
                                (measured on the launch stream; valid after pbe_moments) */
    int32_t steps_per_pass;  /* time steps fused per HBM pass (k_stream temporal blocking, NEXT-4;
                                1 otherwise) */
    int32_t warp_specialized;/* 1: k_resident_ws (primal warps + tangent warps), 0 otherwise */
} pbe_run_info;
pbe_status pbe_last_run_info(pbe_ctx ctx, pbe_run_info* info);

/* Library version string. */
const char* pbe_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PBE_H_ */
