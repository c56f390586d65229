// cheb.cu — K1 fused Chebyshev SpMM step and K2 deterministic moment reduce.
//
// Reference hot loop (kpm.py:96-107, kpm.py:174-189): per probe,
//     v_1 = B v_0,  v_{k+1} = 2 B v_k - v_{k-1},  B x = (A x - c x)/d  (matrix.py:125-126)
// with one dot product per step.  Here all n_vec probes advance together as
// an n x ldv row-major block, so every matrix entry is read once per step for
// the whole block and each gathered x-row is a contiguous, coalesced run of
// ldv doubles.  The spectral map, the 2*(.) - w_{k-1} update and the moment
// dot products are fused into the same pass:
//   DIRECT   (compute_chebyshev_moments):  slot k+1 <- <v_0, w_{k+1}>
//   DOUBLING (moments_via_product_formula): slot 2k+1 <- <w_{k+1}, w_k>,
//                                           slot 2k+2 <- <w_{k+1}, w_{k+1}>
// and zeta_k = 2 r_k - zeta_{k mod 2} (k >= 2) in the reduce (the identity
// T_{a+b} = 2 T_a T_b - T_{a-b} of kpm.py:185-188 with a-b in {0,1}).
//
// Each block owns a contiguous row range (persistent row-range blocks, fixed
// count per matrix), accumulates its dot partials in registers, reduces them
// warp -> block in a fixed order and writes one partial per (slot, block,
// column).  K2 sums those partials over blocks in index order: no atomics, so
// results are bitwise reproducible.
#include "rowgroup.cuh"

namespace sdb {

constexpr int kStepThreads = kRowThreads;
constexpr int kStepWarps = kRowWarps;

struct StepArgs {
  const double* x;     // w_k                      (gathered)
  const double* prev;  // w_{k-1}                  (row-local; may alias next)
  double* next;        // w_{k+1}
  const double* v0;    // probes (direct mode dots)
  double c;            // spectral centre
  double inv_d;        // 1/halfwidth
  int first;           // k == 0: w_1 = B w_0
  int64_t n;
  int64_t ldv;
  int64_t nblocks;
  double* partials;    // [(M+1)][nblocks][ldv]
  int slotA;           // doubling: <w+,w+>, direct: <v0,w+>   (-1: none)
  int slotB;           // doubling: <w+,w>                       (-1: none)
  int slot0;           // step 0: <w0,w0>                        (-1: none)
};

// Epilogue shared by the CSR and stencil steps: spectral map, recurrence,
// store, and the fused dot products for one row.
template <int L, int VPL, int MODE>
__device__ __forceinline__ void step_epilogue(const StepArgs& a, int64_t row, int q, double2 (&y)[VPL],
                                              double2 (&accA)[VPL], double2 (&accB)[VPL],
                                              double2 (&acc0)[VPL]) {
  const double* xr = a.x + row * a.ldv + 2 * q;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int off = 2 * L * v;
    double2 xi = ld_d2(xr + off);
    // t = (A x - c x)/d  (matrix.py:126); w+ = t (k = 0) or 2 t - w- (kpm.py:105)
    double tx = (y[v].x - a.c * xi.x) * a.inv_d;
    double ty = (y[v].y - a.c * xi.y) * a.inv_d;
    double2 wn;
    if (a.first) {
      wn.x = tx;
      wn.y = ty;
    } else {
      double2 wp = *reinterpret_cast<const double2*>(a.prev + row * a.ldv + 2 * q + off);
      wn.x = 2.0 * tx - wp.x;
      wn.y = 2.0 * ty - wp.y;
    }
    st_d2(a.next + row * a.ldv + 2 * q + off, wn);
    if (MODE == SDB_CHEB_DOUBLING) {
      accA[v].x += wn.x * wn.x;
      accA[v].y += wn.y * wn.y;
      accB[v].x += wn.x * xi.x;
      accB[v].y += wn.y * xi.y;
      acc0[v].x += xi.x * xi.x;
      acc0[v].y += xi.y * xi.y;
    } else {
      double2 p = ld_d2(a.v0 + row * a.ldv + 2 * q + off);
      accA[v].x += p.x * wn.x;
      accA[v].y += p.y * wn.y;
      acc0[v].x += p.x * p.x;
      acc0[v].y += p.y * p.y;
    }
  }
}

template <int L, int VPL, int MODE>
__device__ __forceinline__ void step_finish(const StepArgs& a, double2 (&accA)[VPL], double2 (&accB)[VPL],
                                            double2 (&acc0)[VPL]) {
  __shared__ double smem[kStepWarps * SDB_MAX_BATCH];
  if (a.slotA >= 0) block_partial<L, VPL>(accA, smem, a.partials, a.slotA, a.nblocks, a.ldv);
  if (MODE == SDB_CHEB_DOUBLING && a.slotB >= 0) block_partial<L, VPL>(accB, smem, a.partials, a.slotB, a.nblocks, a.ldv);
  if (a.slot0 >= 0) block_partial<L, VPL>(acc0, smem, a.partials, a.slot0, a.nblocks, a.ldv);
}

// ---- K1: one recurrence step for the whole probe block ----------------------------
// Persistent row-range blocks: block b owns rows [n*b/B, n*(b+1)/B) and walks
// them RPB rows at a time, so the +-1 / +-nx neighbours of a stencil-like
// pattern are re-read from L1 within the block.
template <class View, int L, int VPL, int MODE>
__global__ void __launch_bounds__(kStepThreads, VPL <= 1 ? 4 : (VPL == 2 ? 3 : 2)) cheb_step_kernel(View A, StepArgs a) {
  constexpr int RPW = 32 / L;            // rows per warp
  constexpr int RPB = RPW * kStepWarps;  // rows per block iteration
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / L, q = lane % L;
  const int64_t rs = a.n * blockIdx.x / a.nblocks;
  const int64_t re = a.n * (blockIdx.x + 1) / a.nblocks;

  double2 accA[VPL], accB[VPL], acc0[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) accA[v] = accB[v] = acc0[v] = make_double2(0.0, 0.0);

  for (int64_t base = rs; base < re; base += RPB) {
    const int64_t row = base + warp * RPW + g;
    const bool valid = row < re;
    double2 y[VPL];
    spmv_row<L, VPL>(A, row, valid, valid ? (int)row : (int)rs, a.x, a.ldv, q, y);
    if (valid) step_epilogue<L, VPL, MODE>(a, row, q, y, accA, accB, acc0);
  }
  step_finish<L, VPL, MODE>(a, accA, accB, acc0);
}

// Degree 0: only zeta_0 = <v0, v0>.
template <int L, int VPL>
__global__ void __launch_bounds__(kStepThreads) self_dot_kernel(StepArgs a) {
  constexpr int RPW = 32 / L;
  constexpr int RPB = RPW * kStepWarps;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / L, q = lane % L;
  const int64_t rs = a.n * blockIdx.x / a.nblocks;
  const int64_t re = a.n * (blockIdx.x + 1) / a.nblocks;
  double2 acc[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) acc[v] = make_double2(0.0, 0.0);
  for (int64_t base = rs; base < re; base += RPB) {
    const int64_t row = base + warp * RPW + g;
    if (row < re) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        double2 p = ld_d2(a.v0 + row * a.ldv + 2 * q + 2 * L * v);
        acc[v].x += p.x * p.x;
        acc[v].y += p.y * p.y;
      }
    }
  }
  __shared__ double smem[kStepWarps * SDB_MAX_BATCH];
  block_partial<L, VPL>(acc, smem, a.partials, 0, a.nblocks, a.ldv);
}

// ---- K2: partials -> per-probe moments ------------------------------------------
__global__ void cheb_reduce_kernel(const double* __restrict__ partials, int64_t nblocks, int64_t ldv, int64_t n_vec,
                                   int64_t degree, int mode, double* __restrict__ zeta_pp) {
  const int64_t total = n_vec * (degree + 1);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx / n_vec, l = idx % n_vec;
    double r = sum_blocks(partials, k, nblocks, ldv, l);
    if (mode == SDB_CHEB_DOUBLING && k >= 2) r = 2.0 * r - sum_blocks(partials, k & 1, nblocks, ldv, l);
    zeta_pp[l * (degree + 1) + k] = r;
  }
}

__global__ void moments_mean_kernel(const double* __restrict__ zeta_pp, int64_t n_vec, int64_t degree,
                                    double* __restrict__ zeta, int32_t* nonfinite) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= degree; k += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t l = 0; l < n_vec; ++l) s += zeta_pp[l * (degree + 1) + k];
    double z = s / (double)n_vec;
    zeta[k] = z;
    if (nonfinite && !isfinite(z)) *nonfinite = 1;
  }
}

// ---- host dispatch ------------------------------------------------------------------
template <int MODE>
static int launch_step(const sdb_matrix* m, const Geometry& g, const StencilView* st, const StepArgs& a,
                       cudaStream_t s) {
  dim3 grid((unsigned)a.nblocks), block(kStepThreads);
  if (m->format == SDB_FMT_CSR) {
    const CsrView A = make_csr_view(m);
#define SDB_STEP_CASE(LL, VV) cheb_step_kernel<CsrView, LL, VV, MODE><<<grid, block, 0, s>>>(A, a)
    SDB_GEOMETRY_DISPATCH(g, SDB_STEP_CASE);
#undef SDB_STEP_CASE
  } else {
#define SDB_STEP_CASE(LL, VV) cheb_step_kernel<StencilView, LL, VV, MODE><<<grid, block, 0, s>>>(*st, a)
    SDB_GEOMETRY_DISPATCH(g, SDB_STEP_CASE);
#undef SDB_STEP_CASE
  }
  return SDB_OK;
}

static int launch_self_dot(const Geometry& g, const StepArgs& a, cudaStream_t s) {
#define SDB_SD_CASE(LL, VV) self_dot_kernel<LL, VV><<<(unsigned)a.nblocks, kStepThreads, 0, s>>>(a)
  SDB_GEOMETRY_DISPATCH(g, SDB_SD_CASE);
#undef SDB_SD_CASE
  return SDB_OK;
}

StencilView make_stencil_view(const sdb_matrix* m) {
  StencilView s{};
  s.nx = m->st.nx;
  s.ny = m->st.ny;
  s.nz = m->st.nz;
  s.n_off = m->st.n_off;
  s.diag = m->diag;
  // order the off-centre points by the flattened offset dz*nx*ny + dy*nx + dx
  int idx[26];
  for (int o = 0; o < s.n_off; ++o) idx[o] = o;
  auto flat = [&](int o) {
    return (int64_t)m->st.off[o][2] * s.nx * s.ny + (int64_t)m->st.off[o][1] * s.nx + m->st.off[o][0];
  };
  for (int i = 1; i < s.n_off; ++i)
    for (int j = i; j > 0 && flat(idx[j]) < flat(idx[j - 1]); --j) {
      int t = idx[j];
      idx[j] = idx[j - 1];
      idx[j - 1] = t;
    }
  s.center_pos = 0;
  for (int o = 0; o < s.n_off; ++o) {
    s.dx[o] = m->st.off[idx[o]][0];
    s.dy[o] = m->st.off[idx[o]][1];
    s.dz[o] = m->st.off[idx[o]][2];
    s.w[o] = m->st.w[idx[o]];
    if (flat(idx[o]) < 0) s.center_pos = o + 1;
  }
  return s;
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

static void cheb_layout(const sdb_matrix* m, int64_t ldv, int64_t degree, size_t* block_bytes,
                        size_t* partial_bytes) {
  *block_bytes = align256(sizeof(double) * (size_t)m->n * (size_t)ldv);
  *partial_bytes = align256(sizeof(double) * (size_t)(degree + 1) * (size_t)row_blocks(m) * (size_t)ldv);
}

}  // namespace sdb

using namespace sdb;

extern "C" {

int sdb_cheb_workspace_size(const sdb_matrix* m, int64_t n_vec, int64_t degree, int mode, size_t* bytes) {
  SDB_REQUIRE(m && bytes, "NULL argument");
  SDB_REQUIRE(n_vec >= 1 && n_vec <= SDB_MAX_BATCH, "n_vec must lie in [1, %d] per batch", SDB_MAX_BATCH);
  SDB_REQUIRE(degree >= 0, "degree must be non-negative");
  SDB_REQUIRE(mode == SDB_CHEB_DIRECT || mode == SDB_CHEB_DOUBLING, "unknown moment mode %d", mode);
  Geometry g = choose_geometry(n_vec);
  size_t bb, pb;
  cheb_layout(m, g.ldv, degree, &bb, &pb);
  *bytes = 2 * bb + pb;
  return SDB_OK;
}

int sdb_cheb_moments(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree, int mode,
                     const double* probes, double* zeta_pp, void* workspace, size_t workspace_bytes, void* stream,
                     float* step_ms) {
  SDB_REQUIRE(m && probes && zeta_pp, "NULL argument");
  size_t need = 0;
  int rc = sdb_cheb_workspace_size(m, n_vec, degree, mode, &need);
  if (rc) return rc;
  SDB_REQUIRE(workspace != nullptr && workspace_bytes >= need, "workspace too small (%zu < %zu bytes)",
              workspace_bytes, need);
  SDB_REQUIRE(d != 0.0, "spectral halfwidth must be non-zero");
  DeviceGuard dg(m->device);
  if (!dg.ok) return fail(SDB_ECUDA, "cannot select CUDA device %d", m->device);
  cudaStream_t s = (cudaStream_t)stream;
  Geometry g = choose_geometry(n_vec);
  size_t bb, pb;
  cheb_layout(m, g.ldv, degree, &bb, &pb);
  double* bufA = (double*)workspace;
  double* bufB = (double*)((char*)workspace + bb);
  double* partials = (double*)((char*)workspace + 2 * bb);

  StepArgs a{};
  a.v0 = probes;
  a.c = c;
  a.inv_d = 1.0 / d;
  a.n = m->n;
  a.ldv = g.ldv;
  a.nblocks = row_blocks(m);
  a.partials = partials;
  StencilView st{};
  if (m->format == SDB_FMT_STENCIL) st = make_stencil_view(m);

  const int64_t steps = (mode == SDB_CHEB_DOUBLING) ? (degree + 1) / 2 : degree;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (step_ms) {
    SDB_CUDA(cudaEventCreate(&e0));
    SDB_CUDA(cudaEventCreate(&e1));
    SDB_CUDA(cudaEventRecord(e0, s));
  }
  if (steps == 0) {
    a.slot0 = 0;
    rc = launch_self_dot(g, a, s);
    if (rc) return rc;
    SDB_CHECK_LAUNCH();
  }
  const double* cur = probes;
  const double* prev = nullptr;
  for (int64_t k = 0; k < steps; ++k) {
    double* next = (k == 0) ? bufA : (k == 1 ? bufB : const_cast<double*>(prev));
    a.x = cur;
    a.prev = prev;
    a.next = next;
    a.first = (k == 0);
    a.slot0 = (k == 0) ? 0 : -1;
    if (mode == SDB_CHEB_DOUBLING) {
      a.slotB = (2 * k + 1 <= degree) ? (int)(2 * k + 1) : -1;
      a.slotA = (2 * k + 2 <= degree) ? (int)(2 * k + 2) : -1;
      rc = launch_step<SDB_CHEB_DOUBLING>(m, g, &st, a, s);
    } else {
      a.slotA = (int)(k + 1);
      a.slotB = -1;
      rc = launch_step<SDB_CHEB_DIRECT>(m, g, &st, a, s);
    }
    if (rc) return rc;
    SDB_CHECK_LAUNCH();
    prev = cur;
    cur = next;
  }
  if (step_ms) SDB_CUDA(cudaEventRecord(e1, s));
  {
    int64_t total = n_vec * (degree + 1);
    int blocks = (int)((total + 255) / 256);
    if (blocks > 4096) blocks = 4096;
    cheb_reduce_kernel<<<blocks, 256, 0, s>>>(partials, a.nblocks, g.ldv, n_vec, degree, mode, zeta_pp);
    SDB_CHECK_LAUNCH();
  }
  if (step_ms) {
    SDB_CUDA(cudaEventSynchronize(e1));
    SDB_CUDA(cudaEventElapsedTime(step_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return SDB_OK;
}

int sdb_moments_mean(const double* zeta_pp, int64_t n_vec, int64_t degree, double* zeta, int32_t* nonfinite,
                     void* stream) {
  SDB_REQUIRE(zeta_pp && zeta, "NULL argument");
  SDB_REQUIRE(n_vec >= 1 && degree >= 0, "bad shape");
  int blocks = (int)((degree + 1 + 255) / 256);
  moments_mean_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(zeta_pp, n_vec, degree, zeta, nonfinite);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

}  // extern "C"
