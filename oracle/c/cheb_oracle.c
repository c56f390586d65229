/*
 * CPU ORACLE -- test infrastructure and timed CPU baseline only; never the
 * product path.  Plain-C restatement of the reference's Chebyshev moment
 * recurrence (/root/reference/pkg/src/specdens/kpm.py:96-107, :174-189) on a
 * CSR matrix, with SciPy csr_matvec semantics for A x (row sums in storage
 * order, matrix.py:101-102) and the MappedOperator form (A x - c x)/d
 * (matrix.py:125-126).  Probes are independent, so they run in parallel on a
 * pthread pool (the reference's own probe-level thread pool,
 * stochastic.py:64-74, without the GIL).
 *
 *   mode 0 (direct):   zeta_k = v0 . w_k, degree matvecs per probe
 *   mode 1 (doubling): zeta_{2k} = 2<w_k,w_k> - zeta_0,
 *                      zeta_{2k+1} = 2<w_{k+1},w_k> - zeta_1,
 *                      (degree+1)/2 matvecs per probe, no stored history
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static void mapped_matvec(int64_t n, const int64_t* indptr, const int32_t* indices, const double* data, double c,
                          double d, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) s += data[k] * x[indices[k]];
    y[i] = (s - c * x[i]) / d;
  }
}

static double dot(int64_t n, const double* a, const double* b) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

static void one_probe(int64_t n, const int64_t* indptr, const int32_t* indices, const double* data, double c, double d,
                      int64_t degree, int mode, const double* v0, double* zeta, double* wa, double* wb, double* t) {
  zeta[0] = dot(n, v0, v0);
  if (degree == 0) return;
  /* w_prev = v0, w = B v0 */
  mapped_matvec(n, indptr, indices, data, c, d, v0, wa);
  const double* wprev = v0;
  double* w = wa;
  double* spare = wb;
  if (mode == 0) {
    zeta[1] = dot(n, v0, w);
    for (int64_t k = 2; k <= degree; ++k) {
      mapped_matvec(n, indptr, indices, data, c, d, w, t);
      for (int64_t i = 0; i < n; ++i) spare[i] = 2.0 * t[i] - wprev[i];
      zeta[k] = dot(n, v0, spare);
      wprev = w;
      double* tmp = w;
      w = spare;
      spare = (tmp == wa || tmp == wb) ? tmp : wa;
      if (spare == w) spare = (w == wa) ? wb : wa;
    }
    return;
  }
  /* doubling: step k produces w_{k+1}; slots 2k+1, 2k+2 */
  const double* wk = v0;
  double* wn = wa;
  int64_t k = 0;
  for (;;) {
    if (2 * k + 1 <= degree) {
      double r = dot(n, wn, wk);
      zeta[2 * k + 1] = (k == 0) ? r : 2.0 * r - zeta[1];
    }
    if (2 * k + 2 <= degree) zeta[2 * k + 2] = 2.0 * dot(n, wn, wn) - zeta[0];
    ++k;
    if (2 * k + 1 > degree) break;
    /* w_{k+1} = 2 B w_k - w_{k-1}; current (wk, wn) = (w_{k-1}, w_k) */
    double* out = (wn == wa) ? wb : wa;
    mapped_matvec(n, indptr, indices, data, c, d, wn, t);
    for (int64_t i = 0; i < n; ++i) out[i] = 2.0 * t[i] - wk[i];
    wk = wn;
    wn = out;
    if (wk == out) break; /* unreachable */
  }
}

struct job {
  int64_t n, degree, n_vec;
  const int64_t* indptr;
  const int32_t* indices;
  const double* data;
  double c, d;
  int mode;
  const double* probes;
  double* zeta_pp;
  int64_t next; /* next probe to claim */
  int err;
  pthread_mutex_t mu;
};

static void* worker(void* arg) {
  struct job* j = (struct job*)arg;
  double* buf = (double*)malloc(sizeof(double) * 3 * (size_t)j->n);
  if (!buf) {
    pthread_mutex_lock(&j->mu);
    j->err = 2;
    pthread_mutex_unlock(&j->mu);
    return NULL;
  }
  for (;;) {
    pthread_mutex_lock(&j->mu);
    int64_t l = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (l >= j->n_vec) break;
    one_probe(j->n, j->indptr, j->indices, j->data, j->c, j->d, j->degree, j->mode, j->probes + l * j->n,
              j->zeta_pp + l * (j->degree + 1), buf, buf + j->n, buf + 2 * j->n);
  }
  free(buf);
  return NULL;
}

int oracle_max_threads(void) {
  long v = sysconf(_SC_NPROCESSORS_ONLN);
  return v > 0 ? (int)v : 1;
}

int oracle_cheb_moments(int64_t n, const int64_t* indptr, const int32_t* indices, const double* data, double c,
                        double d, int64_t degree, int mode, int64_t n_vec, const double* probes, double* zeta_pp,
                        int threads) {
  if (n < 1 || degree < 0 || n_vec < 1 || (mode != 0 && mode != 1)) return 1;
  if (threads < 1) threads = oracle_max_threads();
  if (threads > n_vec) threads = (int)n_vec;
  struct job j = {n, degree, n_vec, indptr, indices, data, c, d, mode, probes, zeta_pp, 0, 0};
  pthread_mutex_init(&j.mu, NULL);
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  int started = 0;
  for (int t = 0; t < threads; ++t)
    if (pthread_create(&tid[t], NULL, worker, &j) == 0) ++started;
  if (started == 0) worker(&j);
  for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
  free(tid);
  pthread_mutex_destroy(&j.mu);
  return j.err;
}
