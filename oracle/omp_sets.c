/* ORACLE / CPU BASELINE -- TEST INFRASTRUCTURE ONLY (see oracle/README.md).
 *
 * The strongest CPU figure for batched evaluation (SURVEY.md §8(d) CPU reference item 4): the
 * reference has no batch API, so value sets are independent sg_run calls
 * (/root/reference/pkg/src/sparsegen/emit.py:190) -- here one OpenMP thread per value set, each
 * sg_run serial (the emitted kernels' own `#pragma omp parallel for` regions are nested inside
 * this one and run on one thread).  Linked with the reference's emitted source for the plan.
 */
void sg_run(double *x, const double *c, const unsigned *p);

void sg_run_sets(int n_sets, double **xs, const double *c, const unsigned *p) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < n_sets; ++i) sg_run(xs[i], c, p);
}
