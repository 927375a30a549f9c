/*
 * osam.h -- C ABI of the B200 (sm_100a) O-SAM FOM/OpInf coupled time loop.
 *
 * Implements the online stage of arXiv 2511.20687 ("Hybrid coupling with operator
 * inference and the overlapping Schwarz alternating method"): Algorithm 1
 * with subdomain-local full-order models (hex8 linear-elastic FE, explicit Newmark
 * beta=0/gamma=1/2 with lumped mass, A.1 P:L1934-1947) and linear
 * OpInf ROMs (eq:opinf_model_schwarz P:L550-583, online coupling P:L617-722), coupled by
 * pointwise (trilinear) Schwarz transfer and stopped by the relative
 * convergence test eq:conv_criterion.  P:L### = /root/reference/PAPER.md line.
 *
 * All arithmetic is IEEE fp64.  Every step of the time loop runs in CUDA kernels of
 * libosam.so; there is no CPU fallback (a missing GPU makes every call return OSAM_ECUDA).
 *
 * Conventions
 *   - Box mesh [lo,hi] with nel[d] hex8 elements per axis; node id p = i + (nx+1)(j + (ny+1)k).
 *   - Physical fields exchanged through this ABI are SoA per sample: u[c*n + p], c in {x,y,z},
 *     n = number of nodes; batched fields are sample-major: u[b*3n + c*n + p].
 *   - Faces are numbered 0:x-, 1:x+, 2:y-, 3:y+, 4:z-, 5:z+.
 *   - A face of subdomain i that lies strictly inside another subdomain's box (normal
 *     direction) and is laterally covered by it is a Schwarz face fed by the first such
 *     subdomain in the osam_step list (d_S Omega_i = d Omega_i cap Omega_j).
 *     All three components of its closed-face nodes are Schwarz DOFs, except components held
 *     by a Dirichlet face (Dirichlet > Schwarz > free).  A node on two Schwarz faces takes its
 *     value from the lower-numbered face.
 *   - Free DOFs are ordered by ascending canonical DOF id 3p+c; Schwarz DOFs likewise.
 *
 * Ownership: the caller owns every pointer it passes.  Host arrays in the descriptor are
 * copied by osam_create_subdomain.  Field pointers (osam_set_ic / osam_get_state /
 * osam_get_accel) may be host or device pointers (detected with cudaPointerGetAttributes);
 * device pointers are accessed only on the subdomain's stream and only during the call.
 * The library owns its device buffers and frees them in osam_destroy.  Handles are not
 * thread-safe.  Functions never abort and never print; on error they return a negative
 * code and osam_last_error() describes it (thread-local string, valid until the next call).
 */
#ifndef OSAM_H
#define OSAM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct osam_subdomain osam_subdomain; /* opaque handle */

enum { OSAM_FOM = 0, OSAM_ROM = 1 };

/* Time integrator of a subdomain (Newmark-beta, gamma = 1/2, eq:schwarz_opinf_discrete
 * P:L617-722, reading R32): explicit (beta = 0, central difference) or, for a ROM, implicit average
 * acceleration (beta = 1/4): linear OpInf (I + beta dt_i^2 e_b Kbar) a^' = e_b (-Kbar u~ + Bbar g^);
 * QOpInf / COpInf by Newton per sample with the exact Jacobian (reading R37; OSAM_EUNSTABLE if it does
 * not converge in 50 steps; OSAM_EINVAL at create if the per-sample system exceeds 200 KB of shared
 * memory).  The FOM is explicit.                                                                      */
enum { OSAM_EXPLICIT = 0, OSAM_IMPLICIT = 1 };

/* FOM material (App. A; readings R35, R36): linear elasticity (A.1, the merged-stencil kernel K1), or the
 * nonlinear Saint Venant-Kirchhoff (A.2: P = F S, S = lambda tr(E) I + 2 mu E, E = (F^T F - I)/2) and
 * Neohookean (A.3: S = kappa/2 (det C - 1) C^-1 + mu (det C)^(-1/3) (I - tr(C)/3 C^-1), kappa = lambda +
 * 2 mu/3) hex8 forces with 2x2x2 Gauss points (kernel NL1).  lambda, mu from (E, nu).                 */
enum { OSAM_LINEAR = 0, OSAM_SVK = 1, OSAM_NEOHOOKEAN = 2 };

enum {
  OSAM_OK = 0,
  OSAM_WNOTCONVERGED = 1, /* some controller step hit max_iters; last iterate kept */
  OSAM_EINVAL = -1,       /* bad sizes/pointers, hi <= lo, nel < 1, r > n_free, dt <= 0 ...   */
  OSAM_ENOMEM = -2,       /* device allocation failed                                           */
  OSAM_ECUDA = -3,        /* a CUDA runtime call failed (message names it)                      */
  OSAM_EOVERLAP = -4,     /* a Schwarz node lies outside its source box by > 1e-8 h             */
  OSAM_EUNSTABLE = -5     /* non-finite convergence norm (state blew up)                       */
};

typedef struct {
  int32_t kind;         /* OSAM_FOM | OSAM_ROM                                                  */
  double lo[3], hi[3];  /* box [lo,hi] in metres                                                */
  int32_t nel[3];       /* hex8 elements per axis (>= 1)                                        */
  double E, nu, rho;    /* Pa, -, kg/m^3 (ROM: E0 the operators were trained at)                */
  uint8_t dirichlet[6]; /* per face, bitmask of displacement components held at 0 (1:x 2:y 4:z) */
  /* ROM only (ignored for a FOM).  Host pointers, column-major, copied at create.            */
  int32_t r, r_b, batch;  /* POD rank, Schwarz-boundary POD rank, samples (FOM: must be 1)      */
  int64_t n_free, n_s;    /* rows of Phi and Phi_s; checked against the geometric DOF split at the
                             first osam_step (OSAM_EINVAL on mismatch)                            */
  const double *Phi;      /* n_free x r   POD basis Phi (rows = free DOFs)  */
  const double *Phi_s;    /* n_s x r_b    Schwarz boundary basis Phi_dS (rows = Schwarz DOFs)   */
  const double *Kbar;     /* r x r        inferred linear operator      */
  const double *Bbar;     /* r x r_b      inferred boundary operator  */
  const double *e_scale;  /* batch factors e_b = E_b/E0 applied to every reduced operator (NULL -> 1) */
  /* Polynomial OpInf (QOpInf / COpInf, eq:quadratic_opinf P:L263-272), NULL = absent.  Compressed
   * Khatri-Rao powers (P:L167 footnote): u^*2 = [u_i u_j, i <= j], u^*3 = [u_i u_j u_l, i <= j <= l],
   * lexicographic; the reduced model is a^ = e_b (-Kbar u^ - Hbar u^*2 - Cbar u^*3 + Bbar g^).      */
  const double *Hbar;     /* r x r(r+1)/2        column-major                                         */
  const double *Cbar;     /* r x r(r+1)(r+2)/6   column-major                                         */
  /* Time discretisation of this subdomain (footnote: dt_i divides the controller step):
   * n_substeps steps of dt_i = cfg.dt / n_substeps per controller step (0 or 1: one step).  When the
   * subdomains of a step differ in n_substeps, Schwarz values at a destination substep come from the
   * source's iterate trace through the temporal interpolant Xi: linear in time between the
   * two bracketing source substeps, the interval start being the source's checkpoint (reading R31);
   * the convergence norm is evaluated at the interval end with dt_i (reading R33).                    */
  int32_t n_substeps;     /* 0/1 .. 4096                                                              */
  int32_t integrator;     /* OSAM_EXPLICIT (FOM: required) | OSAM_IMPLICIT (ROM)                      */
  int32_t material;       /* FOM: OSAM_LINEAR | OSAM_SVK | OSAM_NEOHOOKEAN (ROM: must be OSAM_LINEAR) */
  /* ROM only, optional: Phi given on a subset of its rows.  The online loop reads Phi only where the
   * Schwarz transfer lifts the ROM's field to a neighbour's Schwarz nodes ("Phi restricted to the relevant
   * boundary DoFs") and, in osam_set_ic, to restrict a full field.  phi_rows (host, copied at
   * create): n_phi_rows strictly ascending free-row indices in [0, n_free); Phi is then n_phi_rows x r
   * column-major (its row q = free row phi_rows[q]).  NULL: Phi has all n_free rows.  The first osam_step
   * returns OSAM_EINVAL if the transfer needs a row that is not given; osam_set_ic returns OSAM_EINVAL
   * (use osam_set_ic_reduced).                                                                         */
  const int64_t *phi_rows;
  int64_t n_phi_rows;
} osam_subdomain_desc;

typedef struct {
  double dt;         /* controller step (> 0); subdomain i steps with dt / n_substeps_i           */
  double tol_rel;    /* delta_rel of eq:conv_criterion                                          */
  double tol_abs;    /* delta_abs; <= 0 disables the absolute test                              */
  int32_t max_iters; /* Schwarz iteration cap (>= 1)                                             */
  int32_t min_iters; /* first iteration at which convergence is tested (2)                      */
} osam_schwarz_cfg;

/* Create a subdomain on `cuda_stream` (a cudaStream_t; NULL = legacy default stream): one subdomain
 * Omega_i of the coupled problem with its mesh, material and Dirichlet boundary (the inputs
 * of Algorithm 1); a FOM (hex8 linear/SVK/Neohookean FE, App. A) or an OpInf
 * ROM with its operators (eq:opinf_model_schwarz P:L550-583).  Validates the descriptor (every check
 * before the first CUDA call), copies the host arrays, allocates the double-buffered state.
 * Returns OSAM_OK and *out, or a negative code (then *out = NULL and nothing is leaked). */
int osam_create_subdomain(const osam_subdomain_desc* d, void* cuda_stream, osam_subdomain** out);

/* Initial condition from full-mesh physical fields (batch x 3n doubles each; v0 may be NULL = 0).
 * FOM: Dirichlet DOFs := 0, Schwarz DOFs keep u0, v := 0 on constrained DOFs, a0 = -f(u0)/m.
 * ROM: u^0 = Phi^T u0[free], v^0 = Phi^T v0[free], s0 = u0[Schwarz DOFs],
 *      a^0 = e_b (-Kbar u^0 + Bbar Phi_dS^T s0)  (SURVEY c.1 step 10). */
int osam_set_ic(osam_subdomain* s, const double* u0, const double* v0);

/* Reduced initial condition of a ROM (the restriction step of SURVEY c.1 step 10 / S:L558-565 done by the
 * caller, e.g. when Phi is given on a row subset): u^0 = uh0, v^0 = vh0 (NULL = 0), both r x batch
 * (uh0[b*r + i]); s0 = the Schwarz-DOF values of the initial field (n_s x batch, s0[b*n_s + q], Schwarz
 * DOFs in ascending DOF id; NULL only if the ROM has no Schwarz DOF); a^0 = e_b(-Kbar u^0 + Bbar
 * Phi_dS^T s0) is computed at the first osam_step.  Host or device pointers, read only during the call.
 * OSAM_EINVAL for a FOM. */
int osam_set_ic_reduced(osam_subdomain* s, const double* uh0, const double* vh0, const double* s0);

/* Advance `n_steps` controller steps of Algorithm 1 over the subdomains `sds` (sweep order =
 * array order).  Schwarz maps are built on the first call (n_steps = 0 only builds them).
 * iters_out (host, may be NULL): n_steps x max(batch) Schwarz iteration counts, step-major.
 * Synchronises the stream once at the end. Returns OSAM_OK, OSAM_WNOTCONVERGED or an error. */
int osam_step(osam_subdomain* const* sds, int32_t n_sd, const osam_schwarz_cfg* cfg, int32_t n_steps,
              int32_t* iters_out);

/* Current converged state phi_i(t_k) of the subdomain (the output of Algorithm 1).
 * FOM: u (all DOFs) and v as physical fields, 3n doubles each (constrained v = 0, reading R10).
 * ROM: u^ and v^ as r x batch column-major (u_out[b*r + i]).  Either pointer may be NULL.  Host or
 * device pointers; synchronises the stream.  OSAM_EINVAL before the first osam_step. */
int osam_get_state(const osam_subdomain* s, double* u_out, double* v_out);

/* Diagnostic: acceleration (FOM: 3n physical field; ROM: a^, r x batch). */
int osam_get_accel(const osam_subdomain* s, double* a_out);

/* Counts: nodes, free DOFs, Schwarz DOFs, batch (any pointer may be NULL). */
int osam_get_sizes(const osam_subdomain* s, int64_t* n_nodes, int64_t* n_free, int64_t* n_schwarz,
                   int32_t* batch);

/* Release a subdomain and every device buffer the library allocated for it (the end of the online stage,
 * Algorithm 2); waits for its stream.  Step groups that contain it are forgotten.  NULL: no-op. */
void osam_destroy(osam_subdomain* s);

const char* osam_last_error(void);

/* ---- regularisation selection (offline stage, grid P:L808) --------------------
 * Batched subdomain-local replay: n_models candidate OpInf ROMs of one subdomain (typically one per
 * lambda of the grid 1e-4 * 10^(4(j-1)/(n-1))), each with its own operator
 *     O_b = [-Kbar | Bbar | -Hbar | -Cbar]     (r x (r + r_b + nf), column-major, nf as in the descriptor
 *                                               for order 1 / 2 / 3),
 * are advanced alone with explicit Newmark over the n_steps of the training run, from u^_0 = Ubar[:, 0]
 * and v^_0 = vh0 (NULL: 0), with the Schwarz boundary data of the training run g^_k = Ghat[:, k]
 * (the OpInf part of eq:schwarz_opinf_discrete with the boundary "taken from training data"), and
 * scored by err_b = ||Ubar - U^hat_b||_F / ||Ubar||_F in reduced coordinates (reading R34).
 * best = first argmin over the finite errors (-1 if none).  All models run in one launch (one CTA
 * per model).  Inputs may be host or device pointers; outputs too (traj_out: n_models x n_steps x r,
 * may be NULL; best_out may be NULL).  Synchronises `cuda_stream` before returning.               */
typedef struct {
  int32_t r, r_b, order, n_models, n_steps;
  double dt;
  const double *O;     /* n_models blocks of r x (r + r_b + nf), column-major                       */
  const double *Ubar;  /* r x n_steps   reduced training trajectory (column k = step k)            */
  const double *Ghat;  /* r_b x n_steps reduced Schwarz data of the training run                   */
  const double *vh0;   /* r             initial reduced velocity, NULL = 0                          */
} osam_replay_desc;

int osam_opinf_replay(const osam_replay_desc* d, double* err_out, int32_t* best_out, double* traj_out,
                      void* cuda_stream);

/* ---- measurement helpers (not part of the method) --------------------------------------
 * When profiling is on, osam_step records a CUDA event pair around every FOM-advance
 * launch (kernel K1) on the subdomain's stream and accumulates their durations; the
 * convergence check then synchronises once per iteration.  osam_get_profile returns the
 * accumulated K1 milliseconds, the number of K1 launches, the algorithmic bytes those
 * launches moved (32 B per FOM DOF per launch + 8 B per DOF when the launch tests convergence,
 * DESIGN.md section 6),
 * and the total number of kernels this library launched since the last reset. */
void osam_set_profiling(int32_t on);

/* Convergence trace (diagnostics of eq:conv_criterion): with max_n > 0, every later osam_step
 * records, for each controller step k, each tested Schwarz iteration n <= max_n and each sample b, the
 * (num, den) pair K3 compared (num = sum_i ||du_i + dt dv_i||^2, den = sum_i ||u_i + dt v_i||^2 over
 * unconstrained DOFs, ROM terms in reduced coordinates); untested entries are NaN.  0 disables.
 * osam_get_conv_trace copies the trace of the last osam_step call on the list `sds` (same order) into out
 * ([n_steps][max_n][batch][2] doubles, host or device; may be NULL to query the sizes). */
void osam_set_conv_trace(int32_t max_n);

/* In-schedule timeline of the FOM advance K1 (measurement, not part of the method): every tiled K1 launch of
 * a sweep records its first CTA start and last CTA end (%globaltimer) and K3 folds them per sweep, in the
 * timed schedule itself (CUDA graph, concurrent branches).  out[6] (host) for the group `sds`, accumulated
 * since its first osam_step or the last reset: [0] ms during which some K1 ran (the union of the sweep's K1
 * intervals), [1] ms summed over K1 launches, [2] K1 launches, [3] sweeps, [4] sweeps with the convergence
 * test (n >= 2), [5] algorithmic bytes of those launches (32 B per DOF per sweep + 8 B per DOF within one
 * layer of a Schwarz face per tested sweep).  reset != 0 zeroes the accumulators. */
int osam_get_k1_timeline(osam_subdomain* const* sds, int32_t n_sd, int32_t reset, double* out);
int osam_get_conv_trace(osam_subdomain* const* sds, int32_t n_sd, double* out, int32_t* n_steps, int32_t* max_n,
                        int32_t* batch);
void osam_reset_profile(void);
void osam_get_profile(double* k1_ms, int64_t* k1_launches, double* k1_bytes, int64_t* kernel_launches);

#ifdef __cplusplus
}
#endif

#endif /* OSAM_H */
