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
 * The same recurrence also runs on a periodic constant-coefficient stencil
 * (the StencilOperator form of BASELINE configs 2 and 5, whose CSR at 256^3
 * would be 5.4 GB of host arrays): oracle_stencil_moments.  Its row sum runs
 * over the terms in the column order of an interior row's CSR form (sorted by
 * the flat offset dz*nx*ny + dy*nx + dx, the diagonal at offset 0); tests pin
 * it against the CSR path on the stencil's own CSR (24^3, 32^3).
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

/* operator: CSR (indptr != NULL) or periodic stencil */
struct oper {
  int64_t n;
  const int64_t* indptr;
  const int32_t* indices;
  const double* data;
  int64_t nx, ny, nz;
  int nt;                 /* terms incl. the diagonal, sorted by flat offset */
  int off[27][3];
  double w[27];           /* weight per term; the diagonal's comes from diag */
  int center;             /* index of the diagonal term */
  const double* diag;
};

static int64_t wrap(int64_t v, int64_t m) { return v < 0 ? v + m : (v >= m ? v - m : v); }

static void mapped_matvec(const struct oper* A, double c, double d, const double* x, double* y) {
  const int64_t n = A->n;
  if (A->indptr) {
    for (int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (int64_t k = A->indptr[i]; k < A->indptr[i + 1]; ++k) s += A->data[k] * x[A->indices[k]];
      y[i] = (s - c * x[i]) / d;
    }
    return;
  }
  const int64_t nx = A->nx, ny = A->ny, nz = A->nz;
  for (int64_t iz = 0; iz < nz; ++iz)
    for (int64_t iy = 0; iy < ny; ++iy)
      for (int64_t ix = 0; ix < nx; ++ix) {
        const int64_t i = (iz * ny + iy) * nx + ix;
        double s = 0.0;
        for (int t = 0; t < A->nt; ++t) {
          const int64_t j = (wrap(iz + A->off[t][2], nz) * ny + wrap(iy + A->off[t][1], ny)) * nx +
                            wrap(ix + A->off[t][0], nx);
          s += (t == A->center ? A->diag[i] : A->w[t]) * x[j];
        }
        y[i] = (s - c * x[i]) / d;
      }
}

static double dot(int64_t n, const double* a, const double* b) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

static void one_probe(const struct oper* A, double c, double d, int64_t degree, int mode, const double* v0,
                      double* zeta, double* wa, double* wb, double* t) {
  const int64_t n = A->n;
  zeta[0] = dot(n, v0, v0);
  if (degree == 0) return;
  /* w_prev = v0, w = B v0 */
  mapped_matvec(A, c, d, v0, wa);
  const double* wprev = v0;
  double* w = wa;
  double* spare = wb;
  if (mode == 0) {
    zeta[1] = dot(n, v0, w);
    for (int64_t k = 2; k <= degree; ++k) {
      mapped_matvec(A, c, d, w, t);
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
    mapped_matvec(A, c, d, wn, t);
    for (int64_t i = 0; i < n; ++i) out[i] = 2.0 * t[i] - wk[i];
    wk = wn;
    wn = out;
    if (wk == out) break; /* unreachable */
  }
}

struct job {
  int64_t n, degree, n_vec;
  const struct oper* A;
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
    one_probe(j->A, j->c, j->d, j->degree, j->mode, j->probes + l * j->n, j->zeta_pp + l * (j->degree + 1), buf,
              buf + j->n, buf + 2 * j->n);
  }
  free(buf);
  return NULL;
}

int oracle_max_threads(void) {
  long v = sysconf(_SC_NPROCESSORS_ONLN);
  return v > 0 ? (int)v : 1;
}

static int run_jobs(const struct oper* A, double c, double d, int64_t degree, int mode, int64_t n_vec,
                    const double* probes, double* zeta_pp, int threads) {
  const int64_t n = A->n;
  if (n < 1 || degree < 0 || n_vec < 1 || (mode != 0 && mode != 1)) return 1;
  if (threads < 1) threads = oracle_max_threads();
  if (threads > n_vec) threads = (int)n_vec;
  struct job j = {n, degree, n_vec, A, c, d, mode, probes, zeta_pp, 0, 0};
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

int oracle_cheb_moments(int64_t n, const int64_t* indptr, const int32_t* indices, const double* data, double c,
                        double d, int64_t degree, int mode, int64_t n_vec, const double* probes, double* zeta_pp,
                        int threads) {
  struct oper A;
  memset(&A, 0, sizeof(A));
  A.n = n;
  A.indptr = indptr;
  A.indices = indices;
  A.data = data;
  return run_jobs(&A, c, d, degree, mode, n_vec, probes, zeta_pp, threads);
}

/* offsets: n_off x 3 (dx, dy, dz) in [-1, 1], weights: n_off, diag: nx*ny*nz */
int oracle_stencil_moments(int64_t nx, int64_t ny, int64_t nz, int n_off, const int32_t* offsets,
                           const double* weights, const double* diag, double c, double d, int64_t degree, int mode,
                           int64_t n_vec, const double* probes, double* zeta_pp, int threads) {
  if (n_off < 0 || n_off > 26 || nx < 1 || ny < 1 || nz < 1) return 1;
  struct oper A;
  memset(&A, 0, sizeof(A));
  A.n = nx * ny * nz;
  A.nx = nx;
  A.ny = ny;
  A.nz = nz;
  A.diag = diag;
  A.nt = n_off + 1;
  int64_t key[27];
  for (int t = 0; t < n_off; ++t) {
    for (int a = 0; a < 3; ++a) A.off[t][a] = offsets[3 * t + a];
    A.w[t] = weights[t];
    key[t] = (int64_t)offsets[3 * t + 2] * nx * ny + (int64_t)offsets[3 * t + 1] * nx + offsets[3 * t];
  }
  A.off[n_off][0] = A.off[n_off][1] = A.off[n_off][2] = 0;
  A.w[n_off] = 0.0;
  key[n_off] = 0;
  /* insertion sort of the terms by flat offset (stable; the diagonal sorts at 0) */
  for (int i = 1; i < A.nt; ++i)
    for (int k = i; k > 0 && key[k] < key[k - 1]; --k) {
      int64_t tk = key[k];
      key[k] = key[k - 1];
      key[k - 1] = tk;
      double tw = A.w[k];
      A.w[k] = A.w[k - 1];
      A.w[k - 1] = tw;
      for (int a = 0; a < 3; ++a) {
        int to = A.off[k][a];
        A.off[k][a] = A.off[k - 1][a];
        A.off[k - 1][a] = to;
      }
    }
  A.center = -1;
  for (int t = 0; t < A.nt; ++t)
    if (A.off[t][0] == 0 && A.off[t][1] == 0 && A.off[t][2] == 0) A.center = t;
  return run_jobs(&A, c, d, degree, mode, n_vec, probes, zeta_pp, threads);
}
