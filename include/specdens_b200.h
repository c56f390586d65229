/*
 * specdens_b200.h — C ABI of the B200-native Chebyshev / Lanczos moment engine.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `specdens` (arXiv 1308.5467).  Every entry point is `extern "C"`, takes plain
 * pointers and sizes, and knows nothing about PyTorch.  Device buffers
 * (probe blocks, moment outputs, workspaces, Lanczos bases) are owned by the
 * caller; the library owns only the opaque matrix handles it creates.
 *
 * Conventions
 *   - Return value: SDB_OK (0) or one of the SDB_E* codes below; the message
 *     of the last failure on the calling thread is sdb_last_error().
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  All work is stream-ordered; functions that must return host
 *     values synchronise the stream and say so.
 *   - A "probe block" is n rows x ldv columns of fp64, row-major: row i holds
 *     entry i of probe vectors 0..n_vec-1 followed by zero padding.  ldv comes
 *     from sdb_block_ldv(n_vec).  Probe l lives in column l.
 *   - Results are deterministic: no floating-point atomics; every reduction
 *     has a fixed shape and order for a given (matrix, n_vec, device model).
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/specdens):
 *   matrix.py:35-109    SparseSymmetricMatrix (CSR, both triangles)  -> sdb_matrix_create_csr
 *   matrix.py:112-126   MappedOperator (A - cI)/d                     -> (c, d) arguments
 *   kpm.py:96-107,143   _chebyshev_probe_moments / compute_chebyshev_moments -> sdb_cheb_moments(mode=DIRECT)
 *   kpm.py:157-198      moments_via_product_formula                   -> sdb_cheb_moments(mode=DOUBLING)
 *   kpm.py:127-140      _average_moments (mean over probes)           -> sdb_moments_mean
 *   kpm.py:84-93        jackson_damping                               -> sdb_jackson_damping
 *   kpm.py:201-208      moments_to_coefficients                       -> sdb_kpm_coefficients
 *   kpm.py:211-217,244-250 evaluate_chebyshev_series / evaluate_kpm_dos -> sdb_chebyshev_series
 *   lanczos.py:67-131   lanczos_factorize (batched over probes)       -> sdb_lanczos
 *   lanczos.py:152-159  ritz_quadrature (eigh_tridiagonal, tau = y[0,:]^2) -> sdb_ritz_quadrature
 *   lanczos.py:170-177  pool_ritz_quadratures                         -> sdb_pool_nodes
 *   lanczos.py:180-187  blur_nodes (kernels of density.py:58-76)      -> sdb_blur_nodes
 *   lanczos.py:296-349  cdos_refine (monotone spline CDOS)            -> sdb_cdos_refine
 */
#ifndef SPECDENS_B200_H
#define SPECDENS_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SDB_API __attribute__((visibility("default")))
#else
#define SDB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define SDB_OK 0
#define SDB_EINVAL 1     /* bad argument            -> ValueError          */
#define SDB_ECUDA 2      /* CUDA runtime failure     -> RuntimeError        */
#define SDB_ENUMERIC 3   /* non-finite numbers       -> NumericalFailure    */
#define SDB_ENOMEM 4     /* device allocation failed -> MemoryError         */
#define SDB_EUNSUPPORTED 5 /* shape/format not handled -> TypeError         */

/* Chebyshev moment modes */
#define SDB_CHEB_DIRECT 0   /* zeta_k = v0 . w_k, degree matvecs / probe (kpm.py:96-107)     */
#define SDB_CHEB_DOUBLING 1 /* zeta_{2k}=2<w_k,w_k>-zeta_0, zeta_{2k+1}=2<w_{k+1},w_k>-zeta_1;
                               (degree+1)/2 matvecs / probe (kpm.py:157-198)                  */
#define SDB_LEGENDRE 2      /* zeta_k = v0 . L_k(B) v0, (k+1)L_{k+1} = (2k+1)B L_k - k L_{k-1}
                             (kpm.py:110-124, :150-154); direct-mode kernels                    */

/* damping kinds (kpm.py:62-93) */
#define SDB_DAMP_NONE 0
#define SDB_DAMP_JACKSON 1

/* Lanczos reorthogonalisation modes (lanczos.py:30) */
#define SDB_REORTH_FULL 0
#define SDB_REORTH_SELECTIVE 1
#define SDB_REORTH_NONE 2

/* per-probe Lanczos status (lanczos.py:111-125) */
#define SDB_LZ_OK 0
#define SDB_LZ_BREAKDOWN 1   /* invariant subspace: truncated, beta_next = 0      */
#define SDB_LZ_NONFINITE 2   /* non-finite alpha/beta: reference raises            */
#define SDB_LZ_ZERO_START 3  /* zero starting vector: reference raises ValueError */

/* matrix storage formats */
#define SDB_FMT_CSR 0
#define SDB_FMT_STENCIL 1

typedef struct sdb_matrix sdb_matrix;

typedef struct sdb_matrix_info {
    int64_t n;          /* dimension                                        */
    int64_t nnz;        /* stored entries (stencil: points x offsets)       */
    int32_t format;     /* SDB_FMT_*                                        */
    int32_t device;     /* CUDA ordinal the handle lives on                 */
    int64_t bytes;      /* device bytes one full matrix pass streams (M_A)  */
} sdb_matrix_info;

/* Constant-coefficient stencil on a periodic 3-D grid (nx fastest):
 *   (A x)_p = diag[p] * x_p + sum_o weight[o] * x_{p + offset[o]}
 * offsets are (dx,dy,dz) triples in [-1,1]; the centre is carried by diag.
 * z_ghost = 1 makes the operator a z-slab of a larger grid (row partition):
 * z is not wrapped; the neighbours of plane 0 / nz-1 are read from ghost
 * planes the caller stores immediately before / after the slab's rows in
 * every block passed as x (i.e. at x - nx*ny*ldv and x + nz*nx*ny*ldv). */
typedef struct sdb_stencil_desc {
    int64_t nx, ny, nz;
    int32_t n_offsets;          /* <= 26 off-centre points                  */
    int32_t offsets[26][3];
    double weights[26];
    int32_t z_ghost;
    int32_t reserved;
} sdb_stencil_desc;

/* ---- library ----------------------------------------------------------- */
SDB_API const char* sdb_last_error(void);
SDB_API int sdb_version(void);
/* Probe-block row stride (padded column count) the kernels use for n_vec probes,
 * n_vec in [1, SDB_MAX_BATCH]; larger probe counts are processed in batches. */
#define SDB_MAX_BATCH 256
SDB_API int64_t sdb_block_ldv(int64_t n_vec);

/* ---- matrix layer (matrix.py:35-109) ------------------------------------ */
/* Upload a CSR matrix from HOST arrays (indptr int64[n+1], indices int32 or
 * int64 [nnz] per index_bits, values fp64[nnz]).  Column indices are checked
 * to lie in [0,n).  Row order and in-row entry order are kept, so row sums
 * accumulate in the reference's csr_matvec order. */
SDB_API int sdb_matrix_create_csr(int device, int64_t n, int64_t nnz, const int64_t* indptr,
                          const void* indices, int index_bits, const double* values,
                          void* stream, sdb_matrix** out);
/* Upload a periodic stencil operator; diag is HOST fp64[nx*ny*nz]. */
SDB_API int sdb_matrix_create_stencil(int device, const sdb_stencil_desc* desc, const double* diag,
                              void* stream, sdb_matrix** out);
SDB_API int sdb_matrix_get_info(const sdb_matrix* m, sdb_matrix_info* info);
/* Band + far split of a CSR handle (done at upload when the matrix has a dense
 * symmetric band, e.g. BASELINE config 3; matrix.py:35-109 storage, read by
 * the probe-sliced step kernel): half_width = 0 when the matrix is not split;
 * far_entries = stored off-band entries (pair-padded); bytes_per_pass = bytes
 * one probe slice streams (band diagonals + far pairs + row pointers). */
SDB_API int sdb_matrix_band_info(const sdb_matrix* m, int32_t* half_width, int64_t* far_entries,
                                 int64_t* bytes_per_pass);
SDB_API void sdb_matrix_destroy(sdb_matrix* m);

/* Deterministic device-side pack: probes_t is n_vec x n (probe-major, device),
 * block is n x ldv (row-major, device; padding columns zeroed). */
SDB_API int sdb_pack_probes(const double* probes_t, int64_t n_vec, int64_t n, int64_t ldv,
                    double* block, void* stream);
/* Rademacher probes (stochastic.py:54: rng.integers(0, 2, dim) * 2.0 - 1.0) are
 * exactly +-1: stage them as sign bits.  bits: device, n_vec rows of
 * ceil(n/8) bytes, bit i of row l = (i >> 3, i & 7) little-endian (NumPy
 * packbits bitorder='little'); 1 -> +1.0, 0 -> -1.0.  Writes the n x ldv
 * block (padding columns zeroed). */
SDB_API int sdb_unpack_signs(const uint8_t* bits, int64_t n_vec, int64_t n, int64_t ldv, double* block,
                     void* stream);
/* Inverse of sdb_pack_probes for the first n_vec columns. */
SDB_API int sdb_unpack_block(const double* block, int64_t n, int64_t ldv, int64_t n_vec,
                     double* out_t, void* stream);

/* ---- KPM moments (kpm.py:96-198) ---------------------------------------- */
/* Workspace bytes for sdb_cheb_moments with this matrix / probe count / degree. */
SDB_API int sdb_cheb_workspace_size(const sdb_matrix* m, int64_t n_vec, int64_t degree, int mode,
                            size_t* bytes);
/* Per-probe Chebyshev moments of B = (A - cI)/d.
 *   probes:  device block n x ldv (const; padding columns must be zero)
 *   zeta_pp: device out, n_vec x (degree+1), probe-major
 *   step_ms: optional HOST out — CUDA-event time of the recurrence kernels
 *            only (synchronises the stream when non-NULL). */
SDB_API int sdb_cheb_moments(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree,
                     int mode, const double* probes, double* zeta_pp, void* workspace,
                     size_t workspace_bytes, void* stream, float* step_ms);
/* Name of the step kernel sdb_cheb_moments runs for this matrix / probe count /
 * mode ("cheb_step_zmarch", "cheb_step_grid", "cheb_step_tile",
 * "cheb_step_stencil" or "cheb_step_csr"); "" for invalid arguments. */
SDB_API const char* sdb_cheb_kernel(const sdb_matrix* m, int64_t n_vec, int mode);
/* Step-level form of sdb_cheb_moments for callers that exchange data between
 * steps (row-partitioned multi-GPU: halo planes).  Step k reads x = w_k,
 * prev = w_{k-1} (k >= 1), v0 (direct mode), writes next = w_{k+1} (may alias
 * prev) and its moment partials; sdb_cheb_reduce turns the partials of all
 * steps into per-probe moments (linear in the rows, so per-rank results of a
 * row partition add up).  degree = 0: step 0 only computes zeta_0. */
SDB_API int sdb_cheb_partials_size(const sdb_matrix* m, int64_t n_vec, int64_t degree, int mode, size_t* bytes);
SDB_API int sdb_cheb_step(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree, int mode,
                  int64_t k, const double* x, const double* prev, double* next, const double* v0,
                  double* partials, size_t partial_bytes, void* stream);
/* sdb_cheb_step for a z-slab stencil handle (row partition) that also pushes
 * the halo: the first own plane of `next` is stored to halo_lo (the lower
 * neighbour slab's upper ghost plane, nx*ny x ldv), the last own plane to
 * halo_hi (the upper neighbour's lower ghost plane), from the same kernel
 * epilogue that stores them locally -- peer-device memory over NVLink (P2P
 * enabled, sdb_enable_peer_access) or this device; either may be NULL.  The
 * caller orders step k+1 after the neighbours' step k (same stream, or events). */
SDB_API int sdb_cheb_step_halo(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree, int mode,
                       int64_t k, const double* x, const double* prev, double* next, const double* v0,
                       double* partials, size_t partial_bytes, double* halo_lo, double* halo_hi, void* stream);
/* cudaDeviceEnablePeerAccess(peer) from `device` (already-enabled is success);
 * returns SDB_EUNSUPPORTED if the pair cannot access each other. */
SDB_API int sdb_enable_peer_access(int device, int peer);
SDB_API int sdb_cheb_reduce(const sdb_matrix* m, int64_t n_vec, int64_t degree, int mode, const double* partials,
                    double* zeta_pp, void* stream);
/* Plane-range steps on the z-march layout (row partition of a periodic 7/27-
 * point grid): every rank holds full-size ghost-padded blocks
 * [nz][ny+2][nx+2][ldv] of the whole grid but computes only its own planes
 * [z_lo, z_hi) of w_{k+1}, reading x = w_k on planes z_lo-1 .. z_hi (periodic;
 * the two neighbour planes are the halo the caller exchanged) -- the TMA
 * z-march kernel of sdb_cheb_moments restricted to a plane range.
 * sdb_zm_block_info: doubles per padded plane and bytes per block (0 and 0
 * when the z-march layout does not apply: then use sdb_cheb_step on z-slab
 * handles).  sdb_zm_pad_probes: n x ldv probe block -> padded block.
 * sdb_cheb_step_planes: step k on the planes [z_lo, z_hi) (x/prev/next/v0 are
 * padded blocks; next may alias prev); sdb_cheb_reduce_planes: the partials
 * of all steps of that same range -> per-probe moments (linear in the planes,
 * so ranges and ranks add up).  partial_bytes as sdb_cheb_partials_size. */
SDB_API int sdb_zm_block_info(const sdb_matrix* m, int64_t n_vec, int mode, int64_t* plane_doubles,
                              size_t* block_bytes);
SDB_API int sdb_zm_pad_probes(const sdb_matrix* m, int64_t n_vec, const double* probes, double* padded, void* stream);
SDB_API int sdb_cheb_step_planes(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree, int mode,
                                 int64_t k, int64_t z_lo, int64_t z_hi, const double* x, const double* prev,
                                 double* next, const double* v0, double* partials, size_t partial_bytes,
                                 void* stream);
/* sdb_cheb_step_planes that also pushes the halo from the kernel epilogue:
 * plane z_lo of w_{k+1} is stored at the same offset into halo_lo (the lower
 * neighbour slab's full-size `next` block; peer device memory over NVLink or
 * this device), plane z_hi-1 into halo_hi; either may be NULL.  The caller
 * orders step k+1 of a slab after its neighbours' step k. */
SDB_API int sdb_cheb_step_planes_halo(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree,
                                      int mode, int64_t k, int64_t z_lo, int64_t z_hi, const double* x,
                                      const double* prev, double* next, const double* v0, double* partials,
                                      size_t partial_bytes, double* halo_lo, double* halo_hi, void* stream);
SDB_API int sdb_cheb_reduce_planes(const sdb_matrix* m, int64_t n_vec, int64_t degree, int mode, int64_t z_lo,
                                   int64_t z_hi, const double* partials, double* zeta_pp, void* stream);
/* zeta[k] = (1/n_vec) sum_l zeta_pp[l][k], probes summed in index order
 * (kpm.py:135, :193).  nonfinite (device int32, may be NULL) is set to 1 if
 * any zeta[k] is not finite. */
SDB_API int sdb_moments_mean(const double* zeta_pp, int64_t n_vec, int64_t degree, double* zeta,
                     int32_t* nonfinite, void* stream);

/* ---- KPM density (kpm.py:84-93, 201-217, 244-250) ----------------------- */
SDB_API int sdb_jackson_damping(int64_t degree, double* g, void* stream);
/* mu_k = (2 - delta_k0)/(n pi) * zeta_k * g_k  (all device pointers) */
SDB_API int sdb_kpm_coefficients(const double* zeta, int64_t degree, int64_t n, int damping,
                         double* mu, void* stream);
/* values[i] = sum_k mu_k T_k(t_i) (Clenshaw) [/ sqrt(1 - t_i^2) if edge_weight];
 * density[i] = values[i] / divisor (density may be NULL; divisor = interval
 * halfwidth d, density.py:124-136).  Device pointers. */
SDB_API int sdb_chebyshev_series(const double* mu, int64_t degree, const double* t, int64_t n_pts,
                         int edge_weight, double divisor, double* values, double* density,
                         void* stream);
/* values[i] = sum_k c_k L_k(t_i) (Legendre forward recurrence, kpm.py:220-231);
 * density[i] = values[i] / divisor (density may be NULL).  Device pointers. */
SDB_API int sdb_legendre_series(const double* c, int64_t degree, const double* t, int64_t n_pts,
                        double divisor, double* values, double* density, void* stream);

/* ---- Lanczos quadrature (lanczos.py:67-219) ----------------------------- */
SDB_API int sdb_lanczos_workspace_size(const sdb_matrix* m, int64_t n_vec, int64_t steps,
                               size_t* bytes);
/* Batched lock-step Lanczos, one independent run per probe column, on the
 * operator (A - cI)/d (c = 0, d = 1 for the plain matrix, lanczos.py:198-204).
 *   v0:        device block n x ldv (unnormalised starting vectors; a zero
 *              vector is flagged SDB_LZ_ZERO_START, lanczos.py:83-85)
 *   basis:     device, steps x n x ldv (the Lanczos vectors, step-major)
 *   alpha:     device out n_vec x steps
 *   beta:      device out n_vec x steps: beta[l][j] for j < steps_done-1 and
 *              beta_next at index steps_done-1
 *   steps_done:device out int32 n_vec (M, or j+1 at breakdown)
 *   status:    device out int32 n_vec (SDB_LZ_*); for SDB_LZ_NONFINITE,
 *              steps_done holds the 1-based failing step */
SDB_API int sdb_lanczos(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t steps, int reorth,
                const double* v0, double* basis, double* alpha, double* beta,
                int32_t* steps_done, int32_t* status, void* workspace, size_t workspace_bytes,
                void* stream);
/* Ritz values/weights of each probe's tridiagonal (alpha, beta) of order
 * steps_done[l] (<= m): theta ascending, tau2 = squared first eigenvector
 * components.  Outputs n_vec x m; unused tail entries are set to 0. */
SDB_API int sdb_ritz_quadrature(const double* alpha, const double* beta, const int32_t* steps_done,
                        int64_t n_vec, int64_t m, double* theta, double* tau2, void* stream);
/* ritz_residual_bounds (lanczos.py:162-167): theta as above and
 * resid[l][i] = |beta_next| |y[last, i]| (beta_next = beta[l][steps_done[l]-1],
 * the sdb_lanczos layout).  Outputs n_vec x m; tails zeroed. */
SDB_API int sdb_ritz_residual_bounds(const double* alpha, const double* beta, const int32_t* steps_done,
                             int64_t n_vec, int64_t m, double* theta, double* resid, void* stream);
/* haydock_dos (lanczos.py:263-293): per grid point x_i,
 * density[i] = (1/n_vec) sum_l -Im f_l(x_i + i eta)/pi with f_l the (1,1)
 * resolvent of probe l's tridiagonal (continued fraction, lanczos.py:222-227),
 * probes summed in index order; trunc_pts[i] = max_l beta_next_l |w_last|
 * (Thomas forward sweep, lanczos.py:230-260; beta_next = 0 for probes with
 * status SDB_LZ_BREAKDOWN) and *trunc = max_i trunc_pts[i] (device scalars;
 * both may be NULL).  alpha/beta/steps_done/status in the sdb_lanczos layout. */
SDB_API int sdb_haydock(const double* alpha, const double* beta, const int32_t* steps_done,
                const int32_t* status, int64_t n_vec, int64_t m, const double* grid, int64_t n_pts,
                double eta, double* density, double* trunc_pts, double* trunc, void* stream);
/* Delta-Gauss-Legendre (dgl.py:42-132), one expansion centre t_i per thread:
 * gamma_k(t_i) by the erf-seeded recurrence with psi_k partial sums, halted at
 * the first k >= 1 with |gamma_{k-1}| + |gamma_k| <= k tol (effective[i] = k;
 * later gammas are 0).  values[i] = sum_k weights[k] gamma_k(t_i) / divisor
 * (weights = (k + 1/2) zeta_k; values/weights may be NULL); gamma, psi
 * ((degree+1) x n_pts row-major) and effective (int32 n_pts) are optional
 * device outputs; *failed (device int32, caller-zeroed) gets the first
 * non-finite step.  sigma in unit coordinates. */
SDB_API int sdb_dgl(const double* weights, int64_t degree, const double* t, int64_t n_pts, double sigma,
            double tol, double divisor, double* values, double* gamma, double* psi, int32_t* effective,
            int32_t* failed, void* stream);
/* continued_fraction_resolvent / tridiagonal_resolvent_first (lanczos.py:222-260)
 * for one tridiagonal (alpha m, beta m-1) at nz complex points z (interleaved
 * re, im); outputs interleaved complex, each may be NULL.  scratch: 4*m*nz
 * doubles when w_first or w_last is requested and m > 1. */
SDB_API int sdb_tridiag_resolvent(const double* alpha, const double* beta, int64_t m, const double* z,
                          int64_t nz, double* cf, double* w_first, double* w_last, double* scratch,
                          void* stream);
/* pool_ritz_quadratures (lanczos.py:170-177): concatenate the first
 * steps_done[l] entries of every row l of theta/tau2 (n_rows x m), divide the
 * weights by `divisor` (the number of probes) and sort by theta (stable: ties
 * keep concatenation order).  nodes/weights: device out, capacity n_rows*m;
 * count: HOST out.  Synchronises the stream (reads steps_done). */
SDB_API int sdb_pool_nodes(const double* theta, const double* tau2, const int32_t* steps_done,
                   int64_t n_rows, int64_t m, double divisor, double* nodes, double* weights,
                   int64_t* count, void* stream);
/* blur_nodes (lanczos.py:180-187) with RegularizationKernel (density.py:58-76):
 * density[g] = scale * sum_k w_k K(x_g - theta_k), K Gaussian
 * exp(-x^2/(2 s^2))/sqrt(2 pi s^2) (kind 0) or Lorentzian (s/pi)/(x^2+s^2)
 * (kind 1).  Device pointers. */
/* cdos_refine (lanczos.py:296-349): theta (sorted ascending) / weights of the
 * pooled quadrature (count, device); nodes closer than merge_tol are merged at
 * their weighted mean; a PCHIP spline through (lo, 0), (node_k, cum_k - w_k/2),
 * (hi, total) is averaged over each grid cell: density[g] = max((cdf(e_{g+1})
 * - cdf(e_g)) / (e_{g+1} - e_g), 0) with cell edges at grid midpoints (n_pts
 * == 1: the spline derivative).  Outputs (device): merged nodes/weights
 * (capacity count), spline_x/y/d (capacity count + 2); n_nodes: HOST out.
 * Fewer than 2 merged nodes -> SDB_EINVAL.  Synchronises the stream. */
SDB_API int sdb_cdos_refine(const double* theta, const double* weights, int64_t count, double merge_tol,
                            double lambda_lb, double lambda_ub, const double* grid, int64_t n_pts,
                            double* density, double* nodes_out, double* weights_out, double* spline_x,
                            double* spline_y, double* spline_d, int64_t* n_nodes, void* stream);
#define SDB_KERNEL_GAUSSIAN 0
#define SDB_KERNEL_LORENTZIAN 1
SDB_API int sdb_blur_nodes(const double* theta, const double* w, int64_t count, double scale,
                   int kind, double width, const double* grid, int64_t n_pts, double* density,
                   void* stream);

/* ---- Matrix Market ingestion (matrix.py:247-304) --------- */
/* Host-side reader (no CUDA calls): parses a real/integer coordinate file with a
 * symmetric or general header into an expanded CSR (both triangles, columns
 * sorted per row, duplicates summed in file order), checks exact symmetry;
 * errors are SDB_EINVAL with the reference's ValueError messages.  The CSR is
 * copied out with sdb_mm_export and uploaded like any other matrix. */
typedef struct sdb_mm sdb_mm;
SDB_API int sdb_mm_read(const char* path, sdb_mm** out);
SDB_API int sdb_mm_info(const sdb_mm* mm, int64_t* n, int64_t* nnz, int32_t* symmetric_storage);
SDB_API int sdb_mm_export(const sdb_mm* mm, int64_t* indptr, int32_t* indices, double* values);
SDB_API void sdb_mm_free(sdb_mm* mm);

#ifdef __cplusplus
}
#endif
#endif /* SPECDENS_B200_H */
