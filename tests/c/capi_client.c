/* Plain C99 client of include/hps_b200.h (the C-ABI boundary), mirroring the
 * reference's proj/tests/capi_smoke.c:12-44: the header must be valid C and
 * the shared library must link and run from a C program.
 *
 * BASELINE cfg0 (4 x 4 elements, N = 8): seeded sample -> element stage ->
 * skeleton -> merge hierarchy -> MG preconditioner with the reference's
 * default MgConfig (depth 2 on the full hierarchy, gamma 1, 4 coarse steps)
 * -> FGMRES with the reference's default KrylovConfig (restart 60, tol 1e-8,
 * single MGS pass) and the right-preconditioned GMRES.
 * Exit 0: ok; 77: no usable sm_100 device (context_create failed); 1: error. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hps_b200.h"

#define CHECK(call)                                                        \
  do {                                                                     \
    hpsb_status st_ = (call);                                              \
    if (st_ != HPSB_OK) {                                                  \
      fprintf(stderr, "%s failed (%d): %s\n", #call, (int)st_, hpsb_last_error()); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

int main(void) {
  int n = 0, order = 0, nrhs = 0, restart = 0;
  double kappa = 0, tol = 0;
  CHECK(hpsb_problem_dims(2, 0, 0, 0, &n, &order, &nrhs, &kappa, &restart, &tol));
  const size_t ne = (size_t)n * n, np = (size_t)order + 1, m = (size_t)order - 1;
  double* coeff = malloc(sizeof(double) * ne * np * np);
  double* source = malloc(2 * sizeof(double) * ne * m * m);
  double* tside = malloc(2 * sizeof(double) * (size_t)nrhs * ne * 4 * m);
  int source_zero = 0;
  CHECK(hpsb_problem_sample(2, 0, 0, 0, 0, 0.0, coeff, source, tside, &source_zero));

  hpsb_context ctx = NULL;
  if (hpsb_context_create(0, &ctx) != HPSB_OK) {
    fprintf(stderr, "no device: %s\n", hpsb_last_error());
    return 77;
  }
  hpsb_elements el = NULL;
  hpsb_skeleton sk = NULL;
  hpsb_hierarchy h = NULL;
  hpsb_precond pc = NULL;
  CHECK(hpsb_elements_build(ctx, n, order, kappa, coeff, source_zero ? NULL : source, &el));
  CHECK(hpsb_skeleton_create(el, tside, nrhs, &sk));
  CHECK(hpsb_hierarchy_build(sk, 0, 0, &h));
  hpsb_mg_config mg = {2, 1, 4, 0}; /* MgConfig{} (multigrid.hpp:12-18) */
  CHECK(hpsb_precond_create(h, mg, &pc));

  const int64_t dim = hpsb_skeleton_dim(sk);
  double* rhs = malloc(2 * sizeof(double) * (size_t)dim);
  double* x = malloc(2 * sizeof(double) * (size_t)dim);
  double* y = malloc(2 * sizeof(double) * (size_t)dim);
  CHECK(hpsb_skeleton_rhs(sk, 0, rhs));
  hpsb_krylov_config kc = {60, 1e-8, 2000, 1, 0}; /* KrylovConfig{} (krylov.hpp:15-21) */
  hpsb_solve_report rep;
  memset(&rep, 0, sizeof rep);
  CHECK(hpsb_fgmres(sk, pc, rhs, x, kc, &rep));
  /* true residual through the interface operator */
  CHECK(hpsb_skeleton_apply(sk, x, y));
  double r2 = 0, b2 = 0;
  for (int64_t i = 0; i < 2 * dim; ++i) {
    r2 += (rhs[i] - y[i]) * (rhs[i] - y[i]);
    b2 += rhs[i] * rhs[i];
  }
  const double res = sqrt(r2 / b2);
  /* plain modified Gram-Schmidt (reorthogonalize 0): the reference bounds the
     basis orthogonality by 1e-5 (test_krylov.cpp:88) */
  if (!rep.converged || res > 1e-8 || rep.basis_orthogonality > 1e-5 || rep.precond_memory <= 0) {
    fprintf(stderr, "unexpected fgmres result: converged=%d iterations=%d residual=%g "
            "orthogonality=%g precond_memory=%lld\n", rep.converged, rep.iterations, res,
            rep.basis_orthogonality, (long long)rep.precond_memory);
    return 1;
  }
  hpsb_solve_report rep2;
  CHECK(hpsb_gmres(sk, pc, rhs, x, kc, &rep2));
  if (!rep2.converged) {
    fprintf(stderr, "right-preconditioned gmres did not converge\n");
    return 1;
  }
  CHECK(hpsb_precond_destroy(pc));
  CHECK(hpsb_hierarchy_destroy(h));
  CHECK(hpsb_skeleton_destroy(sk));
  CHECK(hpsb_elements_destroy(el));
  CHECK(hpsb_context_destroy(ctx));
  if (strlen(hpsb_version()) == 0) return 1;
  printf("c client ok: fgmres %d iterations (residual %.2e), gmres %d iterations\n",
         rep.iterations, res, rep2.iterations);
  free(coeff), free(source), free(tside), free(rhs), free(x), free(y);
  return 0;
}
