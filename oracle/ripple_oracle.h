/*
 * ripple_oracle.h -- CPU ORACLE for the Ripple (arXiv 2104.08571) finite-volume step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (include/, paper_2104_08571_b200/).
 *
 * What it computes (PAPER.md = P:, SPEC.md = S:, SURVEY.md readings S1..S22):
 *   one time step = Listing 8: for each sweep direction d = x, y, z
 *   in order: set_boundary (fill every ghost layer),
 *   FORCE flux on every face normal to d ("the FORCE method of Toro",
 *   S:587), conservative update U' = U - dt/dx (F_{i+1/2} - F_{i-1/2})
 *   (P:1270-1271 flux difference, applied per direction = split scheme, S1).
 *   Euler equations with ideal-gas EOS p = (gamma-1)(E - 1/2 |m|^2 / rho)
 *   (reading S5), conserved components [rho, m_0..m_{D-1}, E] (S6).
 *
 * Data layout at this interface: dense AoS interior, index
 *   ((k*n[1] + j)*n[0] + i)*C + c,   C = ndim + 2,  x fastest.
 * The oracle allocates its own padded copy internally.
 *
 * Order 2 (the paper is silent on reconstruction order, Listing 8 is
 * order 1): per sweep, per cell, minmod-limited slopes of the conserved variables,
 * boundary-extrapolated values, a half-step (dt/2) evolution with the physical
 * flux, FORCE at every face between the evolved values (Toro's SLIC scheme).
 *
 * Return codes: 0 = ok, -7 = numerical-domain error (rho<=0, p<=0 or non-finite
 * after a sweep; order 2 also: rho<=0 or p<=0 in an extrapolated or
 * evolved boundary value), -1 = invalid argument.
 */
#ifndef RIPPLE_ORACLE_H
#define RIPPLE_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_BC_TRANSMISSIVE = 0, ORC_BC_PERIODIC = 1, ORC_BC_REFLECTIVE = 2 };
enum { ORC_OK = 0, ORC_E_INVALID = -1, ORC_E_DOMAIN = -7 };

typedef struct {
  int ndim;          /* 1, 2 or 3 */
  long n[3];         /* interior cells per dim (unused dims: 1) */
  int pad;           /* ghost width p >= 1 */
  double dx[3];      /* cell widths */
  double gamma;      /* ratio of specific heats (1.4) */
  int bc_lo[3];      /* boundary kind on the low face of each dim */
  int bc_hi[3];      /* boundary kind on the high face of each dim */
  int order;         /* 1: piecewise constant (reading S7; 0 also means 1);
                      * 2: MUSCL-Hancock + FORCE = Toro's SLIC (SURVEY f3,
                      *    DESIGN.md readings F3a-F3d), needs pad >= 2 */
} orc_grid;

/* nsteps split FORCE steps with fixed dt (reading D3).  U in/out. */
int orc_step_f64(const orc_grid* g, double* U, double dt, int nsteps);
int orc_step_f32(const orc_grid* g, float* U, double dt, int nsteps);

/* One sweep along direction d only (ghost fill + faces + update), for tests. */
int orc_sweep_f64(const orc_grid* g, double* U, double dt, int d);

/* Ghost fill of a padded AoS array P (extent n[d]+2*pad in each used dim),
 * dims in order 0..ndim-1 over the full padded extent. For tests. */
void orc_fill_ghosts_f64(const orc_grid* g, double* P);

/* Flux difference (paper sec. 7.3): R = sum_d (F_{i+1/2} - F_{i-1/2})
 * with FORCE at step dt on every face of every interior cell (one ghost fill). */
int orc_flux_difference_f64(const orc_grid* g, const double* U, double dt, double* R);
int orc_flux_difference_f32(const orc_grid* g, const float* U, double dt, float* R);

/* S = max over interior cells of |u| + c, c = sqrt(gamma p / rho). */
double orc_max_wavespeed_f64(const orc_grid* g, const double* U);
double orc_max_wavespeed_f32(const orc_grid* g, const float* U);

/* CFL-driven run to t_end (Listing 8 set_wavespeeds -> reduce Max -> set_dt,
 * P:1343-1350): dt = cfl_n * min_d dx_d / S, cfl_n = cfl * reduce for the
 * first n_reduced steps (reading S8), last step clipped to land on t_end.
 * Returns steps taken in *nsteps_out. */
int orc_run_cfl_f64(const orc_grid* g, double* U, double t_end, double cfl,
                    int n_reduced, double reduce, int max_steps, int* nsteps_out);

/* Exact solution of the 1-D Riemann problem for the Euler equations
 * (Toro's exact solver: two-wave pressure function, Newton iteration from
 * the PVRS guess, sampling at xi = x/t).  Left/right primitive states
 * (rho, u, p).  Writes star state (p*, u*, rho*L, rho*R) to star[4] and
 * samples (rho, u, p) at each xi[i] into out[3*i..3*i+2]. Returns Newton
 * iterations, or -1 on vacuum generation. */
int orc_riemann_exact(double rl, double ul, double pl, double rr, double ur,
                      double pr, double gamma, const double* xi, long nxi,
                      double* star, double* out);

/* OpenMP threads of the line loops of step/sweep/flux_difference (default 1).
 * Lines are independent, so results are bitwise the same for any count.
 * Returns the count set (1 when built without OpenMP). */
int orc_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
