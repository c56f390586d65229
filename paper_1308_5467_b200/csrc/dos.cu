// dos.cu — K3 (Jackson damping, coefficients, Clenshaw DOS) and the Lanczos
// quadrature back end: K6 batched tridiagonal eigensolver (first-row QL),
// node pooling, and K7 Gaussian blur.
#include <vector>

#include "common.cuh"

namespace sdb {

// ---- K3 -----------------------------------------------------------------------
// jackson_damping (kpm.py:84-93):
//   g_k = [(1 - k/(M+2)) sin(a) cos(k a) + sin(k a) cos(a)/(M+2)] / sin(a),  a = pi/(M+2)
__global__ void jackson_kernel(int64_t degree, double* __restrict__ g) {
  const double mp2 = (double)(degree + 2);
  const double a = M_PI / mp2;
  const double sa = sin(a), ca = cos(a);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= degree; k += (int64_t)gridDim.x * blockDim.x) {
    const double kd = (double)k;
    g[k] = ((1.0 - kd / mp2) * sa * cos(kd * a) + sin(kd * a) * ca / mp2) / sa;
  }
}

// moments_to_coefficients (kpm.py:201-208): mu_k = prefactor_k * zeta_k * g_k,
// prefactor = 2/(n pi) for k >= 1 and 1/(n pi) for k = 0.
__global__ void coefficients_kernel(const double* __restrict__ zeta, int64_t degree, int64_t n, int damping,
                                    double* __restrict__ mu) {
  const double npi = (double)n * M_PI;
  const double mp2 = (double)(degree + 2);
  const double a = M_PI / mp2;
  const double sa = sin(a), ca = cos(a);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= degree; k += (int64_t)gridDim.x * blockDim.x) {
    const double pref = (k == 0 ? 1.0 : 2.0) / npi;
    double g = 1.0;
    if (damping == SDB_DAMP_JACKSON) {
      const double kd = (double)k;
      g = ((1.0 - kd / mp2) * sa * cos(kd * a) + sin(kd * a) * ca / mp2) / sa;
    }
    mu[k] = pref * zeta[k] * g;
  }
}

// evaluate_chebyshev_series (kpm.py:211-217) by Clenshaw, one grid point per
// thread, coefficients staged through shared memory in tiles; then the
// Chebyshev weight 1/sqrt(1-t^2) (kpm.py:247) and the 1/d unmapping
// (density.py:124-136).
__global__ void series_kernel(const double* __restrict__ mu, int64_t degree, const double* __restrict__ t,
                              int64_t n_pts, int edge_weight, double divisor, double* __restrict__ values,
                              double* __restrict__ density) {
  constexpr int TILE = 1024;
  __shared__ double cs[TILE];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = i < n_pts;
  const double ti = live ? t[i] : 0.0;
  const double t2 = 2.0 * ti;
  double b1 = 0.0, b2 = 0.0;
  // coefficients M..1, walked downwards in tiles of TILE
  for (int64_t hi = degree; hi >= 1; hi -= TILE) {
    const int64_t lo = hi - TILE + 1 < 1 ? 1 : hi - TILE + 1;
    __syncthreads();
    for (int64_t k = lo + threadIdx.x; k <= hi; k += blockDim.x) cs[k - lo] = mu[k];
    __syncthreads();
    for (int64_t k = hi; k >= lo; --k) {
      const double nb1 = t2 * b1 - b2 + cs[k - lo];
      b2 = b1;
      b1 = nb1;
    }
  }
  if (!live) return;
  double v = ti * b1 - b2 + mu[0];
  if (edge_weight) v = v / sqrt(1.0 - ti * ti);
  values[i] = v;
  if (density) density[i] = v / divisor;
}

// KPML evaluation (kpm.py:220-231, :298-308): sum_k c_k L_k(t) by the forward
// recurrence L_{k+1} = ((2k+1) t L_k - k L_{k-1}) / (k+1), one grid point per
// thread, in the reference's expression order; density = values / divisor.
__global__ void legendre_series_kernel(const double* __restrict__ c, int64_t degree, const double* __restrict__ t,
                                       int64_t n_pts, double divisor, double* __restrict__ values,
                                       double* __restrict__ density) {
  constexpr int TILE = 1024;
  __shared__ double cs[TILE];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = i < n_pts;
  const double ti = live ? t[i] : 0.0;
  double acc = c[0] * 1.0;
  double lp = 1.0, lc = ti;
  if (degree >= 1) acc = acc + c[1] * lc;
  // coefficients 2..M in tiles; step k produces L_{k+1}
  for (int64_t lo = 2; lo <= degree; lo += TILE) {
    const int64_t hi = lo + TILE - 1 < degree ? lo + TILE - 1 : degree;
    __syncthreads();
    for (int64_t k = lo + threadIdx.x; k <= hi; k += blockDim.x) cs[k - lo] = c[k];
    __syncthreads();
    for (int64_t k1 = lo; k1 <= hi; ++k1) {
      const int64_t k = k1 - 1;
      const double ln = ((double)(2 * k + 1) * ti * lc - (double)k * lp) / ((double)k + 1.0);
      lp = lc;
      lc = ln;
      acc += cs[k1 - lo] * lc;
    }
  }
  if (!live) return;
  values[i] = acc;
  if (density) density[i] = acc / divisor;
}

// ---- K6: batched first-row implicit QL ---------------------------------------------
// ritz_quadrature (lanczos.py:152-159) takes theta, y = eigh_tridiagonal(alpha,
// beta) and tau^2 = y[0,:]^2.  Only the first row of the eigenvector matrix is
// needed (Golub-Welsch), so the implicit-shift QL sweep applies each plane
// rotation to a single row vector z (initialised to e_0) instead of a matrix.
// One block per probe; the serial sweep runs on one thread with d, e, z in
// shared memory.
// With resid != NULL the last row zl is rotated as well (initialised to
// e_{m-1}) and resid = |beta_next| |zl| -- ritz_residual_bounds
// (lanczos.py:162-167), beta_next read from beta[l][steps_done-1].
__global__ void ritz_ql_kernel(const double* __restrict__ alpha, const double* __restrict__ beta,
                               const int32_t* __restrict__ steps_done, int64_t m, double* __restrict__ theta,
                               double* __restrict__ tau2, double* __restrict__ resid, int* failed) {
  extern __shared__ double sh[];
  double* d = sh;
  double* e = sh + m;
  double* z = sh + 2 * m;
  double* zl = sh + 3 * m;
  const bool last = resid != nullptr;
  const int64_t l = blockIdx.x;
  const int64_t mm = steps_done[l];
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    d[i] = i < mm ? alpha[l * m + i] : 0.0;
    e[i] = (i + 1 < mm) ? beta[l * m + i] : 0.0;
    z[i] = (i == 0) ? 1.0 : 0.0;
    if (last) zl[i] = (i == mm - 1) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t nn = mm;
    for (int64_t lo = 0; lo < nn; ++lo) {
      int iter = 0;
      int64_t hi;
      do {
        // find the first negligible off-diagonal at or after lo
        for (hi = lo; hi < nn - 1; ++hi) {
          const double dd = fabs(d[hi]) + fabs(d[hi + 1]);
          if (fabs(e[hi]) <= 2.220446049250313e-16 * dd) break;
        }
        if (hi != lo) {
          if (++iter > 60) {
            atomicExch(failed, 1);
            break;
          }
          // Wilkinson-type shift from the leading 2x2 block
          double g = (d[lo + 1] - d[lo]) / (2.0 * e[lo]);
          double r = hypot(g, 1.0);
          g = d[hi] - d[lo] + e[lo] / (g + copysign(r, g));
          double s = 1.0, c = 1.0, p = 0.0;
          int64_t i;
          bool deflated = false;
          for (i = hi - 1; i >= lo; --i) {
            double f = s * e[i];
            const double b = c * e[i];
            r = hypot(f, g);
            e[i + 1] = r;
            if (r == 0.0) {  // underflow: split the problem here
              d[i + 1] -= p;
              e[hi] = 0.0;
              deflated = true;
              break;
            }
            s = f / r;
            c = g / r;
            g = d[i + 1] - p;
            r = (d[i] - g) * s + 2.0 * c * b;
            p = s * r;
            d[i + 1] = g + p;
            g = c * r - b;
            // rotate columns i, i+1 of the (first row of the) eigenvector matrix
            f = z[i + 1];
            z[i + 1] = s * z[i] + c * f;
            z[i] = c * z[i] - s * f;
            if (last) {
              f = zl[i + 1];
              zl[i + 1] = s * zl[i] + c * f;
              zl[i] = c * zl[i] - s * f;
            }
          }
          if (deflated) continue;
          d[lo] -= p;
          e[lo] = g;
          e[hi] = 0.0;
        }
      } while (hi != lo);
    }
    // ascending order (LAPACK convention), insertion sort carrying z
    for (int64_t i = 1; i < nn; ++i) {
      const double dv = d[i], zv = z[i], lv = last ? zl[i] : 0.0;
      int64_t j = i - 1;
      while (j >= 0 && d[j] > dv) {
        d[j + 1] = d[j];
        z[j + 1] = z[j];
        if (last) zl[j + 1] = zl[j];
        --j;
      }
      d[j + 1] = dv;
      z[j + 1] = zv;
      if (last) zl[j + 1] = lv;
    }
  }
  __syncthreads();
  const double bn = (last && mm >= 1) ? fabs(beta[l * m + mm - 1]) : 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    theta[l * m + i] = i < mm ? d[i] : 0.0;
    if (tau2) tau2[l * m + i] = i < mm ? z[i] * z[i] : 0.0;
    if (last) resid[l * m + i] = i < mm ? bn * fabs(zl[i]) : 0.0;
  }
}

// ---- Haydock resolvent (lanczos.py:222-293), SURVEY §8(f)-3 ---------------------------
// Complex arithmetic on (re, im) pairs.
struct cplx {
  double re, im;
};
__device__ __forceinline__ cplx cmk(double r, double i) { return cplx{r, i}; }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return cplx{a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cplx{a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return cplx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
__device__ __forceinline__ cplx cscale(double s, cplx a) { return cplx{s * a.re, s * a.im}; }
// a / b, Smith's algorithm (the scaling NumPy's complex division uses)
__device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
  if (fabs(b.re) >= fabs(b.im)) {
    if (b.re == 0.0 && b.im == 0.0) return cplx{a.re / fabs(b.re), a.im / fabs(b.im)};
    const double r = b.im / b.re, den = b.re + b.im * r;
    return cplx{(a.re + a.im * r) / den, (a.im - a.re * r) / den};
  }
  const double r = b.re / b.im, den = b.im + b.re * r;
  return cplx{(a.re * r + a.im) / den, (a.im * r - a.re) / den};
}
__device__ __forceinline__ double cabs_(cplx a) { return hypot(a.re, a.im); }

// e1^T (zI - T)^{-1} e1 by the bottom-up continued fraction (lanczos.py:222-227).
__device__ cplx cf_resolvent(const double* a, const double* b, int64_t mm, cplx z) {
  const cplx one = cmk(1.0, 0.0);
  cplx f = cdiv(one, csub(z, cmk(a[mm - 1], 0.0)));
  for (int64_t j = mm - 2; j >= 0; --j) f = cdiv(one, csub(csub(z, cmk(a[j], 0.0)), cscale(b[j] * b[j], f)));
  return f;
}

// Last entry of the Thomas solve of (zI - T) w = e1 (lanczos.py:230-260, forward sweep).
__device__ cplx thomas_last(const double* a, const double* b, int64_t mm, cplx z) {
  const cplx one = cmk(1.0, 0.0);
  if (mm == 1) return cdiv(one, csub(z, cmk(a[0], 0.0)));
  cplx denom = csub(z, cmk(a[0], 0.0));
  cplx cp = cdiv(cmk(-b[0], 0.0), denom);
  cplx dp = cdiv(one, denom);
  for (int64_t j = 1; j < mm; ++j) {
    denom = cadd(csub(z, cmk(a[j], 0.0)), cscale(b[j - 1], cp));
    const cplx cpn = (j < mm - 1) ? cdiv(cmk(-b[j], 0.0), denom) : cp;
    dp = cdiv(cscale(b[j - 1], dp), denom);
    cp = cpn;
  }
  return dp;
}

// haydock_dos (lanczos.py:263-293): density(x) = mean_l -Im f_l(x + i eta)/pi in
// probe order; trunc[i] = max_l beta_next_l |w_last,l(x_i + i eta)|.  One grid
// point per thread, every probe's tridiagonal walked in order.
__global__ void haydock_kernel(const double* __restrict__ alpha, const double* __restrict__ beta,
                               const int32_t* __restrict__ steps_done, const int32_t* __restrict__ status,
                               int64_t n_vec, int64_t m, const double* __restrict__ grid, int64_t n_pts, double eta,
                               double* __restrict__ density, double* __restrict__ trunc) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_pts) return;
  const cplx z = cmk(grid[i], eta);
  double sum = 0.0, tmax = 0.0;
  for (int64_t l = 0; l < n_vec; ++l) {
    const int64_t mm = steps_done[l];
    const double* a = alpha + l * m;
    const double* b = beta + l * m;
    const cplx f = cf_resolvent(a, b, mm, z);
    sum += -f.im / M_PI;
    const cplx wl = thomas_last(a, b, mm, z);
    const double bn = status[l] == SDB_LZ_BREAKDOWN ? 0.0 : b[mm - 1];
    const double tv = bn * cabs_(wl);
    tmax = tv > tmax ? tv : tmax;
  }
  density[i] = sum / (double)n_vec;
  if (trunc) trunc[i] = tmax;
}

// continued_fraction_resolvent / tridiagonal_resolvent_first for one
// tridiagonal at arbitrary complex points (z interleaved re, im).  The back
// substitution for w_0 keeps cp, dp per point in scratch (2 m complex each).
__global__ void tridiag_resolvent_kernel(const double* __restrict__ alpha, const double* __restrict__ beta,
                                         int64_t m, const double* __restrict__ zs, int64_t nz,
                                         double* __restrict__ cf, double* __restrict__ wfirst,
                                         double* __restrict__ wlast, double* __restrict__ scratch) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nz) return;
  const cplx z = cmk(zs[2 * i], zs[2 * i + 1]);
  const cplx one = cmk(1.0, 0.0);
  if (cf) {
    const cplx f = cf_resolvent(alpha, beta, m, z);
    cf[2 * i] = f.re;
    cf[2 * i + 1] = f.im;
  }
  if (!wfirst && !wlast) return;
  cplx w0, wl;
  if (m == 1) {
    w0 = wl = cdiv(one, csub(z, cmk(alpha[0], 0.0)));
  } else {
    cplx* cpa = reinterpret_cast<cplx*>(scratch) + i * 2 * m;
    cplx* dpa = cpa + m;
    cplx denom = csub(z, cmk(alpha[0], 0.0));
    cpa[0] = cdiv(cmk(-beta[0], 0.0), denom);
    dpa[0] = cdiv(one, denom);
    for (int64_t j = 1; j < m; ++j) {
      denom = cadd(csub(z, cmk(alpha[j], 0.0)), cscale(beta[j - 1], cpa[j - 1]));
      if (j < m - 1) cpa[j] = cdiv(cmk(-beta[j], 0.0), denom);
      dpa[j] = cdiv(cscale(beta[j - 1], dpa[j - 1]), denom);
    }
    wl = dpa[m - 1];
    cplx w = wl;
    for (int64_t j = m - 2; j >= 0; --j) w = csub(dpa[j], cmul(cpa[j], w));
    w0 = w;
  }
  if (wfirst) {
    wfirst[2 * i] = w0.re;
    wfirst[2 * i + 1] = w0.im;
  }
  if (wlast) {
    wlast[2 * i] = wl.re;
    wlast[2 * i + 1] = wl.im;
  }
}

__global__ void max_reduce_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  __shared__ double red[256];
  double v = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v = x[i] > v ? x[i] : v;
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s && red[threadIdx.x + s] > red[threadIdx.x]) red[threadIdx.x] = red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// ---- Delta-Gauss-Legendre (dgl.py:42-132) -------------------------------------------
// One expansion centre per thread: the gamma_k / psi_k recurrence seeded by the
// erf formula, halted at the first k >= 1 with |gamma_{k-1}| + |gamma_k| <= k tol
// (later gammas are zero), accumulating sum_k w_k gamma_k with w_k =
// (k + 1/2) zeta_k when w is given.  gamma/psi tables ((M+1) x n_pts,
// row-major) are optional outputs (compute_dgl_coefficients).
__global__ void dgl_kernel(const double* __restrict__ w, int64_t degree, const double* __restrict__ t, int64_t n_pts,
                           double sigma, double tol, double divisor, double* __restrict__ values,
                           double* __restrict__ gamma_out, double* __restrict__ psi_out, int32_t* __restrict__ eff,
                           int32_t* failed) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_pts) return;
  const double ti = t[i];
  const double s2 = sqrt(2.0) * sigma;
  const double g0 = sigma * sqrt(M_PI / 2.0) * (erf((1.0 - ti) / s2) + erf((1.0 + ti) / s2));
  const double exp_lo = exp(-0.5 * ((1.0 - ti) / sigma) * ((1.0 - ti) / sigma));
  const double exp_hi = exp(-0.5 * ((1.0 + ti) / sigma) * ((1.0 + ti) / sigma));
  double gk = g0, gprev = 0.0;           // gamma_k, gamma_{k-1}
  double psi_k = 0.0, psi_next = g0;     // psi_k, psi_{k+1}
  double acc = w ? w[0] * g0 : 0.0;
  int64_t effective = degree;
  if (gamma_out) {
    for (int64_t k = 0; k <= degree; ++k) {
      gamma_out[k * n_pts + i] = 0.0;
      if (psi_out) psi_out[k * n_pts + i] = 0.0;
    }
    gamma_out[i] = g0;
    if (psi_out && degree >= 1) psi_out[n_pts + i] = psi_next;
  }
  for (int64_t k = 0; k < degree; ++k) {
    if (k >= 1 && fabs(gprev) + fabs(gk) <= (double)k * tol) {
      effective = k;
      break;
    }
    // NumPy's operation order with no FMA contraction: the recurrence
    // amplifies rounding differences once the gammas have decayed
    const double boundary = __dsub_rn(exp_lo, __dmul_rn((k & 1) ? -1.0 : 1.0, exp_hi));
    const double inner = __dadd_rn(__dmul_rn(__dmul_rn(sigma, sigma), __dsub_rn(psi_k, boundary)), __dmul_rn(ti, gk));
    const double nxt = __dsub_rn(__dmul_rn((double)(2 * k + 1) / ((double)k + 1.0), inner),
                                 __dmul_rn((double)k / ((double)k + 1.0), gprev));
    if (!isfinite(nxt)) {
      atomicExch(failed, (int32_t)(k + 1));
      effective = k;
      break;
    }
    gprev = gk;
    gk = nxt;
    const int64_t j = k + 1;
    if (w) acc = __dadd_rn(acc, __dmul_rn(w[j], gk));
    const double pn = __dadd_rn(__dmul_rn((double)(2 * j + 1), gk), psi_k);
    psi_k = psi_next;
    psi_next = pn;
    if (gamma_out) {
      gamma_out[j * n_pts + i] = gk;
      if (psi_out && j + 1 <= degree) psi_out[(j + 1) * n_pts + i] = psi_next;
    }
  }
  if (values) values[i] = acc / divisor;
  if (eff) eff[i] = (int32_t)effective;
}

// ---- node pooling (lanczos.py:170-177) ---------------------------------------------
// Stable rank sort of the concatenated nodes: rank(i) = #{j : th_j < th_i} +
// #{j < i : th_j == th_i}.  O(N^2) compares on a tile of theta staged in
// shared memory; N = probes x steps is small (12,800 at config 4).
__global__ void compact_kernel(const double* __restrict__ theta, const double* __restrict__ tau2,
                               const int64_t* __restrict__ offsets, const int32_t* __restrict__ steps_done,
                               int64_t n_rows, int64_t m, double* __restrict__ flat_th, double* __restrict__ flat_w) {
  const int64_t total = n_rows * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = idx / m, k = idx % m;
    if (k >= steps_done[l]) continue;
    flat_th[offsets[l] + k] = theta[idx];
    flat_w[offsets[l] + k] = tau2[idx];
  }
}

__global__ void rank_sort_kernel(const double* __restrict__ th, const double* __restrict__ w, int64_t count,
                                 double divisor, double* __restrict__ nodes, double* __restrict__ weights) {
  constexpr int TILE = 1024;
  __shared__ double tile[TILE];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double x = i < count ? th[i] : 0.0;
  int64_t rank = 0;
  for (int64_t t0 = 0; t0 < count; t0 += TILE) {
    __syncthreads();
    for (int64_t k = threadIdx.x; k < TILE && t0 + k < count; k += blockDim.x) tile[k] = th[t0 + k];
    __syncthreads();
    const int64_t lim = (count - t0) < TILE ? (count - t0) : TILE;
    for (int64_t k = 0; k < lim; ++k) {
      const double y = tile[k];
      rank += (y < x) || (y == x && t0 + k < i);
    }
  }
  if (i < count) {
    nodes[rank] = x;
    weights[rank] = w[i] / divisor;
  }
}

// ---- K7: blur (lanczos.py:180-187, density.py:58-76) ---------------------------------
// One block per grid point; threads stride over the nodes, then a fixed-order
// shared-memory tree reduce (deterministic).
__global__ void blur_kernel(const double* __restrict__ theta, const double* __restrict__ w, int64_t count,
                            double scale, int kind, double width, const double* __restrict__ grid, int64_t n_pts,
                            double* __restrict__ density) {
  __shared__ double red[256];
  const double gnorm = sqrt(2.0 * M_PI * width * width);
  const double lnum = width / M_PI, w2 = width * width;
  for (int64_t gi = blockIdx.x; gi < n_pts; gi += gridDim.x) {
    const double x = grid[gi];
    double s = 0.0;
    for (int64_t k = threadIdx.x; k < count; k += blockDim.x) {
      const double dx = x - theta[k];
      double kv;
      if (kind == SDB_KERNEL_GAUSSIAN) {
        const double u = dx / width;
        kv = exp(-0.5 * (u * u)) / gnorm;
      } else {
        kv = lnum / (dx * dx + w2);
      }
      s += kv * w[k];
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int off = blockDim.x / 2; off > 0; off >>= 1) {
      if ((int)threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
      __syncthreads();
    }
    if (threadIdx.x == 0) density[gi] = scale * red[0];
    __syncthreads();
  }
}

}  // namespace sdb

using namespace sdb;

// ---- CDOS: monotone spline through the pooled cumulative staircase -----------------
// cdos_refine (lanczos.py:296-349).  Stage 1 (one thread: the merge is a
// running weighted mean, inherently sequential; <= a few 10^4 nodes): merge
// sorted nodes closer than tol, stair midpoints cumsum - w/2, anchor points
// (lo, 0) and (hi, total).  Stage 2: PCHIP derivatives (SciPy
// PchipInterpolator._find_derivatives, same operation order).  Stage 3: the
// cubic Hermite pieces evaluated at the clipped cell edges as SciPy's PPoly
// does (power series c3 + c2 s + c1 s^2 + c0 s^3 accumulated in that order,
// interval by bisection), then density = max(diff(cdf)/diff(edges), 0).
// Explicit _rn intrinsics: no FMA contraction, like the host evaluation.
__global__ void cdos_merge_kernel(const double* __restrict__ th, const double* __restrict__ tw, int64_t count,
                                  double tol, double lb, double ub, double* __restrict__ nodes,
                                  double* __restrict__ weights, double* __restrict__ xs, double* __restrict__ ys,
                                  int64_t* __restrict__ kout) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t k = 0;
  for (int64_t i = 0; i < count; ++i) {
    const double t = th[i], w = tw[i];
    if (k > 0 && __dsub_rn(t, nodes[k - 1]) <= tol) {
      const double total = __dadd_rn(weights[k - 1], w);
      nodes[k - 1] = __ddiv_rn(__dadd_rn(__dmul_rn(nodes[k - 1], weights[k - 1]), __dmul_rn(t, w)), total);
      weights[k - 1] = total;
    } else {
      nodes[k] = t;
      weights[k] = w;
      ++k;
    }
  }
  *kout = k;
  if (k < 2) return;
  double cum = 0.0;
  for (int64_t i = 0; i < k; ++i) {
    cum = __dadd_rn(cum, weights[i]);
    xs[i + 1] = nodes[i];
    ys[i + 1] = __dsub_rn(cum, __dmul_rn(0.5, weights[i]));
  }
  const double tiny = 2.2250738585072014e-308;  // np.finfo(float).tiny
  const double a = __dsub_rn(__dsub_rn(nodes[0], tol), tiny);
  const double b = __dadd_rn(__dadd_rn(nodes[k - 1], tol), tiny);
  xs[0] = a < lb ? a : lb;  // min(lambda_lb, ...): the first argument on ties
  xs[k + 1] = b > ub ? b : ub;
  ys[0] = 0.0;
  ys[k + 1] = cum;
}

__device__ __forceinline__ double sgn_(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

__device__ double pchip_edge(double h0, double h1, double m0, double m1) {
  double d = __ddiv_rn(__dsub_rn(__dmul_rn(__dadd_rn(__dmul_rn(2.0, h0), h1), m0), __dmul_rn(h0, m1)),
                       __dadd_rn(h0, h1));
  const bool mask = sgn_(d) != sgn_(m0);
  const bool mask2 = (sgn_(m0) != sgn_(m1)) && (fabs(d) > __dmul_rn(3.0, fabs(m0)));
  if (mask) d = 0.0;
  else if (mask2) d = __dmul_rn(3.0, m0);
  return d;
}

__global__ void cdos_slopes_kernel(const double* __restrict__ xs, const double* __restrict__ ys,
                                   const int64_t* __restrict__ kin, double* __restrict__ dk) {
  const int64_t np_ = *kin + 2;  // spline points
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np_; i += (int64_t)gridDim.x * blockDim.x) {
    auto h = [&](int64_t j) { return __dsub_rn(xs[j + 1], xs[j]); };
    auto m = [&](int64_t j) { return __ddiv_rn(__dsub_rn(ys[j + 1], ys[j]), h(j)); };
    double d;
    if (i == 0) {
      d = pchip_edge(h(0), h(1), m(0), m(1));
    } else if (i == np_ - 1) {
      d = pchip_edge(h(np_ - 2), h(np_ - 3), m(np_ - 2), m(np_ - 3));
    } else {
      const double h0 = h(i - 1), h1 = h(i), m0 = m(i - 1), m1 = m(i);
      if (sgn_(m1) != sgn_(m0) || m1 == 0.0 || m0 == 0.0) {
        d = 0.0;
      } else {
        const double w1 = __dadd_rn(__dmul_rn(2.0, h1), h0);
        const double w2 = __dadd_rn(h1, __dmul_rn(2.0, h0));
        const double whmean = __ddiv_rn(__dadd_rn(__ddiv_rn(w1, m0), __ddiv_rn(w2, m1)), __dadd_rn(w1, w2));
        d = __ddiv_rn(1.0, whmean);
      }
    }
    dk[i] = d;
  }
}

// value (deriv = 0) or first derivative (deriv = 1) of the PCHIP spline at x
__device__ double pchip_eval(const double* __restrict__ xs, const double* __restrict__ ys,
                             const double* __restrict__ dk, int64_t np_, double x, int deriv) {
  int64_t lo = 0, hi = np_ - 1;  // find i with xs[i] <= x < xs[i+1]; x == xs[last] -> last piece
  if (x >= xs[np_ - 1]) {
    lo = np_ - 2;
  } else {
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) / 2;
      if (x < xs[mid]) hi = mid; else lo = mid;
    }
  }
  const int64_t i = lo;
  const double dx = __dsub_rn(xs[i + 1], xs[i]);
  const double slope = __ddiv_rn(__dsub_rn(ys[i + 1], ys[i]), dx);
  const double t = __ddiv_rn(__dsub_rn(__dadd_rn(dk[i], dk[i + 1]), __dmul_rn(2.0, slope)), dx);
  const double c0 = __ddiv_rn(t, dx);
  const double c1 = __dsub_rn(__ddiv_rn(__dsub_rn(slope, dk[i]), dx), t);
  const double c2 = dk[i], c3 = ys[i];
  const double sv = __dsub_rn(x, xs[i]);
  if (deriv == 0) {
    double res = 0.0, z = 1.0;
    res = __dadd_rn(res, __dmul_rn(c3, z));
    z = __dmul_rn(z, sv);
    res = __dadd_rn(res, __dmul_rn(c2, z));
    z = __dmul_rn(z, sv);
    res = __dadd_rn(res, __dmul_rn(c1, z));
    z = __dmul_rn(z, sv);
    res = __dadd_rn(res, __dmul_rn(c0, z));
    return res;
  }
  double res = 0.0, z = 1.0;
  res = __dadd_rn(res, __dmul_rn(__dmul_rn(c2, z), 1.0));
  z = __dmul_rn(z, sv);
  res = __dadd_rn(res, __dmul_rn(__dmul_rn(c1, z), 2.0));
  z = __dmul_rn(z, sv);
  res = __dadd_rn(res, __dmul_rn(__dmul_rn(c0, z), 3.0));
  return res;
}

__global__ void cdos_density_kernel(const double* __restrict__ xs, const double* __restrict__ ys,
                                    const double* __restrict__ dk, const int64_t* __restrict__ kin,
                                    const double* __restrict__ grid, int64_t n_pts, double* __restrict__ density) {
  const int64_t np_ = *kin + 2;
  if (np_ < 4) return;  // fewer than 2 nodes: reported by the host
  const double lo = xs[0], hi = xs[np_ - 1];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_pts; g += (int64_t)gridDim.x * blockDim.x) {
    double v;
    if (n_pts < 2) {
      v = pchip_eval(xs, ys, dk, np_, grid[g], 1);
    } else {
      // edges (lanczos.py:336-340) of cell g: left and right
      const double el = g == 0 ? __dsub_rn(grid[0], __dmul_rn(0.5, __dsub_rn(grid[1], grid[0])))
                               : __dmul_rn(0.5, __dadd_rn(grid[g], grid[g - 1]));
      const double er = g == n_pts - 1
                            ? __dadd_rn(grid[n_pts - 1], __dmul_rn(0.5, __dsub_rn(grid[n_pts - 1], grid[n_pts - 2])))
                            : __dmul_rn(0.5, __dadd_rn(grid[g + 1], grid[g]));
      const double cl = pchip_eval(xs, ys, dk, np_, fmin(fmax(el, lo), hi), 0);
      const double cr = pchip_eval(xs, ys, dk, np_, fmin(fmax(er, lo), hi), 0);
      v = __ddiv_rn(__dsub_rn(cr, cl), __dsub_rn(er, el));
    }
    density[g] = v > 0.0 ? v : 0.0;  // np.clip(..., 0.0, None)
  }
}

extern "C" {

int sdb_jackson_damping(int64_t degree, double* g, void* stream) {
  SDB_REQUIRE(g != nullptr, "NULL argument");
  SDB_REQUIRE(degree >= 0, "degree must be non-negative");
  int blocks = (int)((degree + 256) / 256);
  jackson_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(degree, g);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int sdb_kpm_coefficients(const double* zeta, int64_t degree, int64_t n, int damping, double* mu, void* stream) {
  SDB_REQUIRE(zeta && mu, "NULL argument");
  SDB_REQUIRE(degree >= 0 && n >= 1, "bad degree or dimension");
  SDB_REQUIRE(damping == SDB_DAMP_NONE || damping == SDB_DAMP_JACKSON, "unknown damping kind %d", damping);
  int blocks = (int)((degree + 256) / 256);
  coefficients_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(zeta, degree, n, damping, mu);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int sdb_chebyshev_series(const double* mu, int64_t degree, const double* t, int64_t n_pts, int edge_weight,
                         double divisor, double* values, double* density, void* stream) {
  SDB_REQUIRE(mu && t && values, "NULL argument");
  SDB_REQUIRE(degree >= 0, "degree must be non-negative");
  if (n_pts <= 0) return SDB_OK;
  SDB_REQUIRE(density == nullptr || divisor != 0.0, "divisor must be non-zero");
  int blocks = (int)((n_pts + 127) / 128);
  series_kernel<<<blocks, 128, 0, (cudaStream_t)stream>>>(mu, degree, t, n_pts, edge_weight, divisor, values,
                                                          density);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int sdb_legendre_series(const double* c, int64_t degree, const double* t, int64_t n_pts, double divisor,
                        double* values, double* density, void* stream) {
  SDB_REQUIRE(c && t && values, "NULL argument");
  SDB_REQUIRE(degree >= 0, "degree must be non-negative");
  if (n_pts <= 0) return SDB_OK;
  SDB_REQUIRE(density == nullptr || divisor != 0.0, "divisor must be non-zero");
  int blocks = (int)((n_pts + 127) / 128);
  legendre_series_kernel<<<blocks, 128, 0, (cudaStream_t)stream>>>(c, degree, t, n_pts, divisor, values, density);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int sdb_haydock(const double* alpha, const double* beta, const int32_t* steps_done, const int32_t* status,
                int64_t n_vec, int64_t m, const double* grid, int64_t n_pts, double eta, double* density,
                double* trunc_pts, double* trunc, void* stream) {
  SDB_REQUIRE(alpha && beta && steps_done && status && grid && density, "NULL argument");
  SDB_REQUIRE(n_vec >= 1 && m >= 1, "bad shape");
  SDB_REQUIRE(eta > 0.0, "eta must be positive");
  SDB_REQUIRE(trunc == nullptr || trunc_pts != nullptr, "trunc needs the per-point buffer");
  if (n_pts <= 0) return SDB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  haydock_kernel<<<(unsigned)((n_pts + 127) / 128), 128, 0, s>>>(alpha, beta, steps_done, status, n_vec, m, grid,
                                                                  n_pts, eta, density, trunc_pts);
  SDB_CHECK_LAUNCH();
  if (trunc) {
    max_reduce_kernel<<<1, 256, 0, s>>>(trunc_pts, n_pts, trunc);
    SDB_CHECK_LAUNCH();
  }
  return SDB_OK;
}

int sdb_dgl(const double* weights, int64_t degree, const double* t, int64_t n_pts, double sigma, double tol,
            double divisor, double* values, double* gamma, double* psi, int32_t* effective, int32_t* failed,
            void* stream) {
  SDB_REQUIRE(t && failed, "NULL argument");
  SDB_REQUIRE(degree >= 0, "max degree must be non-negative");
  SDB_REQUIRE(sigma > 0.0, "sigma must be positive");
  SDB_REQUIRE(tol > 0.0, "tol must be positive");
  SDB_REQUIRE(values == nullptr || weights != nullptr, "values need the weights");
  if (n_pts <= 0) return SDB_OK;
  dgl_kernel<<<(unsigned)((n_pts + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      weights, degree, t, n_pts, sigma, tol, divisor, values, gamma, psi, effective, failed);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int sdb_tridiag_resolvent(const double* alpha, const double* beta, int64_t m, const double* z, int64_t nz,
                          double* cf, double* w_first, double* w_last, double* scratch, void* stream) {
  SDB_REQUIRE(alpha && z, "NULL argument");
  SDB_REQUIRE(m >= 1, "bad shape");
  SDB_REQUIRE(m == 1 || (beta != nullptr && (scratch != nullptr || (!w_first && !w_last))),
              "beta / scratch required");
  if (nz <= 0) return SDB_OK;
  tridiag_resolvent_kernel<<<(unsigned)((nz + 127) / 128), 128, 0, (cudaStream_t)stream>>>(alpha, beta, m, z, nz, cf,
                                                                                           w_first, w_last, scratch);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

static int ritz_ql(const double* alpha, const double* beta, const int32_t* steps_done, int64_t n_vec, int64_t m,
                   double* theta, double* tau2, double* resid, void* stream);

int sdb_ritz_quadrature(const double* alpha, const double* beta, const int32_t* steps_done, int64_t n_vec,
                        int64_t m, double* theta, double* tau2, void* stream) {
  SDB_REQUIRE(alpha && beta && steps_done && theta && tau2, "NULL argument");
  return ritz_ql(alpha, beta, steps_done, n_vec, m, theta, tau2, nullptr, stream);
}

int sdb_ritz_residual_bounds(const double* alpha, const double* beta, const int32_t* steps_done, int64_t n_vec,
                             int64_t m, double* theta, double* resid, void* stream) {
  SDB_REQUIRE(alpha && beta && steps_done && theta && resid, "NULL argument");
  return ritz_ql(alpha, beta, steps_done, n_vec, m, theta, nullptr, resid, stream);
}

static int ritz_ql(const double* alpha, const double* beta, const int32_t* steps_done, int64_t n_vec, int64_t m,
                   double* theta, double* tau2, double* resid, void* stream) {
  SDB_REQUIRE(n_vec >= 1 && m >= 1, "bad shape");
  size_t shmem = sizeof(double) * 4 * (size_t)m;
  SDB_REQUIRE(shmem <= 200 * 1024, "tridiagonal order %lld too large for the on-chip eigensolver", (long long)m);
  cudaStream_t s = (cudaStream_t)stream;
  if (shmem > 48 * 1024) SDB_CUDA(cudaFuncSetAttribute(ritz_ql_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem));
  int* failed = nullptr;
  SDB_CUDA(cudaMallocAsync(&failed, sizeof(int), s));
  SDB_CUDA(cudaMemsetAsync(failed, 0, sizeof(int), s));
  ritz_ql_kernel<<<(unsigned)n_vec, 64, shmem, s>>>(alpha, beta, steps_done, m, theta, tau2, resid, failed);
  cudaError_t le = cudaGetLastError();
  int hf = 0;
  cudaError_t e = le;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hf, failed, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(failed, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "ritz_ql_kernel", __FILE__, __LINE__);
  if (hf) return fail(SDB_ENUMERIC, "tridiagonal eigensolver did not converge");
  return SDB_OK;
}

int sdb_pool_nodes(const double* theta, const double* tau2, const int32_t* steps_done, int64_t n_rows, int64_t m,
                   double divisor, double* nodes, double* weights, int64_t* count, void* stream) {
  SDB_REQUIRE(theta && tau2 && steps_done && nodes && weights && count, "NULL argument");
  SDB_REQUIRE(n_rows >= 1 && m >= 1, "bad shape");
  SDB_REQUIRE(divisor != 0.0, "divisor must be non-zero");
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<int32_t> sd((size_t)n_rows);
  SDB_CUDA(cudaMemcpyAsync(sd.data(), steps_done, sizeof(int32_t) * n_rows, cudaMemcpyDeviceToHost, s));
  SDB_CUDA(cudaStreamSynchronize(s));
  std::vector<int64_t> off((size_t)n_rows);
  int64_t total = 0;
  for (int64_t l = 0; l < n_rows; ++l) {
    SDB_REQUIRE(sd[l] >= 0 && sd[l] <= m, "steps_done out of range");
    off[l] = total;
    total += sd[l];
  }
  *count = total;
  if (total == 0) return SDB_OK;
  int64_t* d_off = nullptr;
  double* flat = nullptr;
  SDB_CUDA(cudaMallocAsync(&d_off, sizeof(int64_t) * n_rows, s));
  SDB_CUDA(cudaMallocAsync(&flat, sizeof(double) * 2 * total, s));
  SDB_CUDA(cudaMemcpyAsync(d_off, off.data(), sizeof(int64_t) * n_rows, cudaMemcpyHostToDevice, s));
  int64_t work = n_rows * m;
  compact_kernel<<<(int)((work + 255) / 256), 256, 0, s>>>(theta, tau2, d_off, steps_done, n_rows, m, flat,
                                                           flat + total);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    rank_sort_kernel<<<(int)((total + 255) / 256), 256, 0, s>>>(flat, flat + total, total, divisor, nodes, weights);
    e = cudaGetLastError();
  }
  cudaFreeAsync(d_off, s);
  cudaFreeAsync(flat, s);
  // the host offsets vector dies here: make sure the async upload finished
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_fail(e, "sdb_pool_nodes", __FILE__, __LINE__);
  return SDB_OK;
}

int sdb_blur_nodes(const double* theta, const double* w, int64_t count, double scale, int kind, double width,
                   const double* grid, int64_t n_pts, double* density, void* stream) {
  SDB_REQUIRE(grid && density, "NULL argument");
  SDB_REQUIRE(count == 0 || (theta && w), "NULL argument");
  SDB_REQUIRE(kind == SDB_KERNEL_GAUSSIAN || kind == SDB_KERNEL_LORENTZIAN, "unknown kernel kind %d", kind);
  SDB_REQUIRE(width > 0.0, "kernel width must be positive");
  if (n_pts <= 0) return SDB_OK;
  int blocks = (int)(n_pts < 65535 ? n_pts : 65535);
  blur_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(theta, w, count, scale, kind, width, grid, n_pts, density);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}


int sdb_cdos_refine(const double* theta, const double* weights, int64_t count, double merge_tol, double lambda_lb,
                    double lambda_ub, const double* grid, int64_t n_pts, double* density, double* nodes_out,
                    double* weights_out, double* spline_x, double* spline_y, double* spline_d, int64_t* n_nodes,
                    void* stream) {
  SDB_REQUIRE(theta && weights && nodes_out && weights_out && spline_x && spline_y && spline_d && n_nodes,
              "NULL argument");
  SDB_REQUIRE(n_pts == 0 || (grid && density), "NULL argument");
  SDB_REQUIRE(count >= 0, "bad shape");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t* dk = nullptr;
  SDB_CUDA(cudaMallocAsync(&dk, sizeof(int64_t), s));
  SDB_CUDA(cudaMemsetAsync(dk, 0, sizeof(int64_t), s));
  if (count > 0) {
    cdos_merge_kernel<<<1, 32, 0, s>>>(theta, weights, count, merge_tol, lambda_lb, lambda_ub, nodes_out, weights_out,
                                      spline_x, spline_y, dk);
    SDB_CHECK_LAUNCH();
  }
  SDB_CUDA(cudaMemcpyAsync(n_nodes, dk, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SDB_CUDA(cudaStreamSynchronize(s));
  if (*n_nodes < 2) {
    cudaFreeAsync(dk, s);
    return fail(SDB_EINVAL, "need at least 2 distinct Ritz nodes for the spline");
  }
  const int64_t np_ = *n_nodes + 2;
  cdos_slopes_kernel<<<(unsigned)((np_ + 255) / 256), 256, 0, s>>>(spline_x, spline_y, dk, spline_d);
  SDB_CHECK_LAUNCH();
  if (n_pts > 0) {
    cdos_density_kernel<<<(unsigned)((n_pts + 255) / 256), 256, 0, s>>>(spline_x, spline_y, spline_d, dk, grid, n_pts,
                                                                        density);
    SDB_CHECK_LAUNCH();
  }
  SDB_CUDA(cudaFreeAsync(dk, s));
  return SDB_OK;
}

}  // extern "C"
