/*
 * ripple_oracle.c -- CPU ORACLE for the Ripple (arXiv 2104.08571) FORCE step.
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
 * bench.py cpu_baseline / --impl reference legs, never by the product path.
 * Shares no code with paper_2104_08571_b200/ or include/.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared (oracle/__init__.py build()).
 * -ffp-contract=off keeps every a*b+c as two rounded operations, exactly as
 * written below (reading S21).
 *
 * Pins for every function live in tests/test_oracle_*.py.
 */
#include "ripple_oracle.h"

#include <math.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Threads of the line loops (OpenMP; 1 unless set).  The bench's cpu_baseline times
 * the oracle at 1 thread and at all host cores; results are identical either way. */
int orc_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n < 1 ? 1 : n);
  return n < 1 ? 1 : n;
#else
  (void)n;
  return 1;
#endif
}

#define REAL double
#define SFX f64
#include "oracle_scheme.inc"
#undef REAL
#undef SFX

#define REAL float
#define SFX f32
#include "oracle_scheme.inc"
#undef REAL
#undef SFX

int orc_sweep_f64(const orc_grid* g, double* U, double dt, int d) {
  if (!g || d < 0 || d >= g->ndim) return ORC_E_INVALID;
  if (g->order == 2 && g->pad < 2) return ORC_E_INVALID;
  int C = g->ndim + 2;
  size_t n = padded_cells_f64(g) * (size_t)C;
  double* a = (double*)calloc(n, sizeof(double));
  double* b = (double*)calloc(n, sizeof(double));
  to_padded_f64(g, U, a);
  int rc = sweep_padded_f64(g, a, b, dt, d);
  from_padded_f64(g, b, U);
  free(a);
  free(b);
  return rc;
}

void orc_fill_ghosts_f64(const orc_grid* g, double* P) { fill_ghosts_f64(g, P); }

/* CFL loop = Listing 8 set_wavespeeds -> then_reduce(Max) -> set_dt,
 * with the caller-side dt of reading D3 and the first-step reduction of S8. */
int orc_run_cfl_f64(const orc_grid* g, double* U, double t_end, double cfl, int n_reduced,
                    double reduce, int max_steps, int* nsteps_out) {
  double dxmin = g->dx[0];
  for (int d = 1; d < g->ndim; ++d)
    if (g->dx[d] < dxmin) dxmin = g->dx[d];
  double t = 0.0;
  int n = 0;
  int rc = ORC_OK;
  while (t < t_end && n < max_steps) {
    double S = orc_max_wavespeed_f64(g, U);
    if (!(S > 0) || !isfinite(S)) {
      rc = ORC_E_DOMAIN;
      break;
    }
    double c = (n < n_reduced) ? cfl * reduce : cfl;
    double dt = c * dxmin / S;
    int last = 0;
    if (t + dt >= t_end) {
      dt = t_end - t;
      last = 1;
    }
    rc = orc_step_f64(g, U, dt, 1);
    ++n;
    if (rc != ORC_OK) break;
    t = last ? t_end : t + dt;
  }
  if (nsteps_out) *nsteps_out = n;
  return rc;
}

/* ---------------------------------------------------------------------------
 * Exact Riemann solver for the 1-D Euler equations, ideal gas (Toro, "Riemann
 * Solvers and Numerical Methods for Fluid Dynamics", ch. 4; the paper cites
 * Toro for FORCE).  Used only to check the scheme's convergence
 * (SURVEY pins P1, P2); it is not part of the scheme.
 * ------------------------------------------------------------------------- */

typedef struct {
  double r, u, p, c;
} prim_t;

/* Pressure function f_K(p) and its derivative for one side K (Toro eq. 4.6-4.7). */
static void pfun(double p, const prim_t* K, double g, double* f, double* fd) {
  if (p > K->p) { /* shock */
    double A = 2.0 / ((g + 1.0) * K->r);
    double B = (g - 1.0) / (g + 1.0) * K->p;
    double q = sqrt(A / (B + p));
    *f = (p - K->p) * q;
    *fd = q * (1.0 - 0.5 * (p - K->p) / (B + p));
  } else { /* rarefaction */
    double pr = p / K->p;
    *f = 2.0 * K->c / (g - 1.0) * (pow(pr, (g - 1.0) / (2.0 * g)) - 1.0);
    *fd = 1.0 / (K->r * K->c) * pow(pr, -(g + 1.0) / (2.0 * g));
  }
}

/* Sample the self-similar solution at xi = x/t (Toro sec. 4.5). */
static void sample(double xi, const prim_t* L, const prim_t* R, double ps, double us, double g,
                   double* r, double* u, double* p) {
  double g6 = (g - 1.0) / (g + 1.0);
  if (xi <= us) { /* left of the contact */
    if (ps > L->p) {
      double SL = L->u - L->c * sqrt((g + 1.0) / (2.0 * g) * ps / L->p + (g - 1.0) / (2.0 * g));
      if (xi <= SL) {
        *r = L->r; *u = L->u; *p = L->p;
      } else {
        *r = L->r * (ps / L->p + g6) / (g6 * ps / L->p + 1.0); *u = us; *p = ps;
      }
    } else {
      double SHL = L->u - L->c;
      if (xi <= SHL) {
        *r = L->r; *u = L->u; *p = L->p;
      } else {
        double cml = L->c * pow(ps / L->p, (g - 1.0) / (2.0 * g));
        double STL = us - cml;
        if (xi > STL) {
          *r = L->r * pow(ps / L->p, 1.0 / g); *u = us; *p = ps;
        } else { /* inside the left fan */
          double c = 2.0 / (g + 1.0) * (L->c + 0.5 * (g - 1.0) * (L->u - xi));
          *u = 2.0 / (g + 1.0) * (L->c + 0.5 * (g - 1.0) * L->u + xi);
          *r = L->r * pow(c / L->c, 2.0 / (g - 1.0));
          *p = L->p * pow(c / L->c, 2.0 * g / (g - 1.0));
        }
      }
    }
  } else { /* right of the contact */
    if (ps > R->p) {
      double SR = R->u + R->c * sqrt((g + 1.0) / (2.0 * g) * ps / R->p + (g - 1.0) / (2.0 * g));
      if (xi >= SR) {
        *r = R->r; *u = R->u; *p = R->p;
      } else {
        *r = R->r * (ps / R->p + g6) / (g6 * ps / R->p + 1.0); *u = us; *p = ps;
      }
    } else {
      double SHR = R->u + R->c;
      if (xi >= SHR) {
        *r = R->r; *u = R->u; *p = R->p;
      } else {
        double cmr = R->c * pow(ps / R->p, (g - 1.0) / (2.0 * g));
        double STR = us + cmr;
        if (xi <= STR) {
          *r = R->r * pow(ps / R->p, 1.0 / g); *u = us; *p = ps;
        } else { /* inside the right fan */
          double c = 2.0 / (g + 1.0) * (R->c - 0.5 * (g - 1.0) * (R->u - xi));
          *u = 2.0 / (g + 1.0) * (-R->c + 0.5 * (g - 1.0) * R->u + xi);
          *r = R->r * pow(c / R->c, 2.0 / (g - 1.0));
          *p = R->p * pow(c / R->c, 2.0 * g / (g - 1.0));
        }
      }
    }
  }
}

int orc_riemann_exact(double rl, double ul, double pl, double rr, double ur, double pr,
                      double gamma, const double* xi, long nxi, double* star, double* out) {
  prim_t L = {rl, ul, pl, sqrt(gamma * pl / rl)};
  prim_t R = {rr, ur, pr, sqrt(gamma * pr / rr)};
  if (2.0 / (gamma - 1.0) * (L.c + R.c) <= R.u - L.u) return -1; /* vacuum */
  /* PVRS initial guess (Toro eq. 4.47) */
  double ppv = 0.5 * (pl + pr) - 0.125 * (ur - ul) * (rl + rr) * (L.c + R.c);
  double p = ppv > 1e-12 ? ppv : 1e-12;
  int it = 0;
  for (it = 1; it <= 200; ++it) {
    double fl, fld, fr, frd;
    pfun(p, &L, gamma, &fl, &fld);
    pfun(p, &R, gamma, &fr, &frd);
    double pn = p - (fl + fr + (ur - ul)) / (fld + frd);
    if (pn < 1e-14) pn = 1e-14;
    double ch = 2.0 * fabs(pn - p) / (pn + p);
    p = pn;
    if (ch < 1e-14) break;
  }
  double fl, fld, fr, frd;
  pfun(p, &L, gamma, &fl, &fld);
  pfun(p, &R, gamma, &fr, &frd);
  double us = 0.5 * (ul + ur) + 0.5 * (fr - fl);
  double g6 = (gamma - 1.0) / (gamma + 1.0);
  double rsl = (p > pl) ? rl * (p / pl + g6) / (g6 * p / pl + 1.0) : rl * pow(p / pl, 1.0 / gamma);
  double rsr = (p > pr) ? rr * (p / pr + g6) / (g6 * p / pr + 1.0) : rr * pow(p / pr, 1.0 / gamma);
  if (star) {
    star[0] = p;
    star[1] = us;
    star[2] = rsl;
    star[3] = rsr;
  }
  for (long i = 0; i < nxi; ++i)
    sample(xi[i], &L, &R, p, us, gamma, &out[3 * i], &out[3 * i + 1], &out[3 * i + 2]);
  return it;
}
