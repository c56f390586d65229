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
#include "stepargs.cuh"

namespace sdb {

constexpr int kStepThreads = kRowThreads;
constexpr int kStepWarps = kRowWarps;

// Resident blocks per SM the step kernels are compiled for (register cap).
// (compile-time tunables: -DSDB_MINB_V1=.. -DSDB_MINB_V2=.. -DSDB_U_V1=..)
#ifndef SDB_MINB_V1
#define SDB_MINB_V1 5
#endif
#ifndef SDB_MINB_V2
#define SDB_MINB_V2 2
#endif
#ifndef SDB_U_V1
#define SDB_U_V1 4
#endif
#ifndef SDB_U_V2
#define SDB_U_V2 8
#endif
__host__ __device__ constexpr int step_min_blocks(int l, int vpl) {
  return l < 8 ? (vpl == 1 ? 4 : 2) : (vpl == 1 ? SDB_MINB_V1 : (vpl == 2 ? SDB_MINB_V2 : 2));
}



// Epilogue shared by the CSR and stencil steps, split in two so the row's own
// operands (x_i for the spectral shift, w_{k-1}, v_0) are requested before
// the gathers and arrive while they are in flight.  FIRST (k = 0) has no
// w_{k-1} and additionally accumulates zeta_0 = <v0, v0>.
template <int VPL>
struct EpiIn {
  double2 xi[VPL];
  double2 wp[VPL];
  double2 p0[VPL];
};

template <int L, int VPL, int MODE, bool FIRST>
__device__ __forceinline__ void epi_load(const StepArgs& a, int64_t row, int q, uint64_t pol, EpiIn<VPL>& e) {
  const int64_t o = row * a.ldv + 2 * q;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    e.xi[v] = ld_d2(a.x + o + 2 * L * v);
    if (!FIRST) e.wp[v] = ld_d2_once(a.prev + o + 2 * L * v, pol);
    if (MODE == SDB_CHEB_DIRECT && !FIRST) e.p0[v] = ld_d2_once(a.v0 + o + 2 * L * v, pol);
  }
}

template <int L, int VPL, int MODE, bool FIRST>
__device__ __forceinline__ void epi_finish(const StepArgs& a, int64_t row, int q, const double2 (&y)[VPL],
                                           const EpiIn<VPL>& e, double2 (&accA)[VPL], double2 (&accB)[VPL],
                                           double2 (&accZ)[VPL], uint64_t pol) {
  const int64_t o = row * a.ldv + 2 * q;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const double2 xi = e.xi[v];
    // t = (A x - c x)/d  (matrix.py:126); w+ = t (k = 0) or 2 t - w- (kpm.py:105)
    const double tx = (y[v].x - a.c * xi.x) * a.inv_d;
    const double ty = (y[v].y - a.c * xi.y) * a.inv_d;
    double2 wn;
    if (FIRST) {
      wn = make_double2(tx, ty);
    } else if (MODE == SDB_CHEB_DIRECT && a.legendre) {
      wn.x = (a.la * tx - a.lb * e.wp[v].x) / a.lc;
      wn.y = (a.la * ty - a.lb * e.wp[v].y) / a.lc;
    } else {
      wn.x = 2.0 * tx - e.wp[v].x;
      wn.y = 2.0 * ty - e.wp[v].y;
    }
    st_d2_once(a.next + o + 2 * L * v, wn, pol);
    halo_push(a, row, 2 * q + 2 * L * v, wn);
    if (MODE == SDB_CHEB_DOUBLING) {
      accA[v].x += wn.x * wn.x;
      accA[v].y += wn.y * wn.y;
      if constexpr (MODE == SDB_CHEB_DOUBLING) {
        accB[v].x += wn.x * xi.x;
        accB[v].y += wn.y * xi.y;
      }
    } else {
      const double2 p = FIRST ? xi : e.p0[v];  // at k = 0 the gathered block is v0
      accA[v].x += p.x * wn.x;
      accA[v].y += p.y * wn.y;
    }
    if constexpr (FIRST) {
      accZ[v].x += xi.x * xi.x;
      accZ[v].y += xi.y * xi.y;
    }
  }
}

template <int L, int VPL, int MODE, bool FIRST>
__device__ __forceinline__ void step_finish(const StepArgs& a, double2 (&accA)[VPL], double2 (&accB)[VPL],
                                            double2 (&accZ)[VPL]) {
  __shared__ double smem[kStepWarps * SDB_MAX_BATCH];
  if (a.slotA >= 0) block_partial<L, VPL>(accA, smem, a.partials, a.slotA, a.nblocks, a.ldv);
  if constexpr (MODE == SDB_CHEB_DOUBLING) {
    if (a.slotB >= 0) block_partial<L, VPL>(accB, smem, a.partials, a.slotB, a.nblocks, a.ldv);
  }
  if constexpr (FIRST) {
    if (a.slot0 >= 0) block_partial<L, VPL>(accZ, smem, a.partials, a.slot0, a.nblocks, a.ldv);
  }
}

// Issue U gathers x[col[u]] (this lane's columns), then accumulate them in
// order: y += w[u] * x[col[u]].
template <int L, int VPL, int U>
__device__ __forceinline__ void gather_fma(const double* __restrict__ x, int64_t ldv, int q, const int (&col)[U],
                                           const double (&w)[U], double2 (&y)[VPL]) {
  double2 xv[U][VPL];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const double* xr = x + (int64_t)col[u] * ldv + 2 * q;
#pragma unroll
    for (int v = 0; v < VPL; ++v) xv[u][v] = ld_d2(xr + 2 * L * v);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      y[v].x = fma(w[u], xv[u][v].x, y[v].x);
      y[v].y = fma(w[u], xv[u][v].y, y[v].y);
    }
  }
}

// ---- K1, CSR form ---------------------------------------------------------------
// Rows follow the phased-panel schedule (rowgroup.cuh).  The L lanes of a row
// group load up to L (col, value) pairs of their row cooperatively and
// broadcast them with shuffles; U gathers are in flight per lane; the row's
// own operands are requested before the gathers.  Entries are accumulated in
// storage order (csr_matvec order, matrix.py:101-102).
template <int L, int VPL, int MODE, bool FIRST>
__global__ void __launch_bounds__(kStepThreads, step_min_blocks(L, VPL)) cheb_step_csr(CsrView A, StepArgs a) {
  pdl_wait();
  pdl_trigger();
  constexpr int RPW = 32 / L;
  constexpr int RPB = RPW * kStepWarps;
  constexpr int U = L < 4 ? L : (VPL == 1 ? SDB_U_V1 : (VPL == 2 ? SDB_U_V2 : 2));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / L, q = lane % L;
  const uint64_t pol = policy_evict_first();
  double2 accA[VPL], accB[VPL], accZ[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) accA[v] = accB[v] = accZ[v] = make_double2(0.0, 0.0);
  for (int64_t ph = 0;; ++ph) {
    const int64_t p0 = (ph * a.nblocks + blockIdx.x) * a.panel;
    if (p0 >= a.n) break;
    const int64_t pend = p0 + a.panel < a.n ? p0 + a.panel : a.n;
    for (int64_t base = p0; base < pend; base += RPB) {
    const int64_t row = base + warp * RPW + g;
    const bool valid = row < pend;
    const int safe = valid ? (int)row : (int)base;
    const int beg = valid ? __ldg(A.rowptr + row) : 0;
    const int cnt = valid ? __ldg(A.rowptr + row + 1) - beg : 0;
    EpiIn<VPL> e;
    if (valid) epi_load<L, VPL, MODE, FIRST>(a, row, q, pol, e);
    double2 y[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) y[v] = make_double2(0.0, 0.0);
    const int maxcnt = __reduce_max_sync(0xffffffffu, cnt);
    for (int k0 = 0; k0 < maxcnt; k0 += L) {
      const int kk = k0 + q;
      int colc = safe;
      double valc = 0.0;
      if (kk < cnt) {
        colc = __ldg(A.colidx + beg + kk);
        valc = __ldg(A.vals + beg + kk);
      }
      const int nloc = min(L, maxcnt - k0);
      for (int t0 = 0; t0 < nloc; t0 += U) {
        int ct[U];
        double at[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          ct[u] = __shfl_sync(0xffffffffu, colc, t0 + u, L);
          at[u] = __shfl_sync(0xffffffffu, valc, t0 + u, L);
        }
        gather_fma<L, VPL, U>(a.x, a.ldv, q, ct, at, y);
      }
    }
    if (valid) epi_finish<L, VPL, MODE, FIRST>(a, row, q, y, e, accA, accB, accZ, pol);
    }
  }
  step_finish<L, VPL, MODE, FIRST>(a, accA, accB, accZ);
}

// ---- K1, periodic stencil form -------------------------------------------------------
// Terms (off-centre points + diagonal) are ordered by the column index they
// produce for an interior point; interior rows use the precomputed deltas,
// rows on a periodic face recompute wrapped coordinates.
template <int L, int VPL, int MODE, bool FIRST>
__global__ void __launch_bounds__(kStepThreads, step_min_blocks(L, VPL)) cheb_step_stencil(StencilView S, StepArgs a) {
  pdl_wait();
  pdl_trigger();
  constexpr int RPW = 32 / L;
  constexpr int RPB = RPW * kStepWarps;
  constexpr int U = VPL == 1 ? 8 : (VPL == 2 ? 4 : 2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / L, q = lane % L;
  const uint64_t pol = policy_evict_first();
  const int nx = S.nx, ny = S.ny, nz = S.nz;
  double2 accA[VPL], accB[VPL], accZ[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) accA[v] = accB[v] = accZ[v] = make_double2(0.0, 0.0);
  for (int64_t ph = 0;; ++ph) {
    const int64_t p0 = (ph * a.nblocks + blockIdx.x) * a.panel;
    if (p0 >= a.n) break;
    const int64_t pend = p0 + a.panel < a.n ? p0 + a.panel : a.n;
    for (int64_t base = p0; base < pend; base += RPB) {
    const int64_t row = base + warp * RPW + g;
    if (row >= pend) continue;
    EpiIn<VPL> e;
    epi_load<L, VPL, MODE, FIRST>(a, row, q, pol, e);
    const int r32 = (int)row;
    const int ix = r32 % nx, t = r32 / nx;
    const int iy = t % ny, iz = t / ny;
    const bool interior = (!S.mx || (ix > 0 && ix < nx - 1)) && (!S.my || (iy > 0 && iy < ny - 1)) &&
                          (S.zghost || !S.mz || (iz > 0 && iz < nz - 1));
    const double dg = __ldg(S.diag + row);
    double2 y[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) y[v] = make_double2(0.0, 0.0);
    for (int o0 = 0; o0 < S.nterms; o0 += U) {
      int col[U];
      double w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int o = o0 + u;
        col[u] = r32;
        w[u] = 0.0;
        if (o < S.nterms) {
          const int4 tm = __ldg(S.term + o);
          w[u] = (o == S.center_pos) ? dg : __ldg(S.tw + o);
          if (interior) {
            col[u] = r32 + tm.w;
          } else {
            int jx = ix + tm.x, jy = iy + tm.y, jz = iz + tm.z;
            jx = jx < 0 ? jx + nx : (jx >= nx ? jx - nx : jx);
            jy = jy < 0 ? jy + ny : (jy >= ny ? jy - ny : jy);
            if (!S.zghost) jz = jz < 0 ? jz + nz : (jz >= nz ? jz - nz : jz);
            col[u] = (jz * ny + jy) * nx + jx;
          }
        }
      }
      gather_fma<L, VPL, U>(a.x, a.ldv, q, col, w, y);
    }
    epi_finish<L, VPL, MODE, FIRST>(a, row, q, y, e, accA, accB, accZ, pol);
    }
  }
  step_finish<L, VPL, MODE, FIRST>(a, accA, accB, accZ);
}

// ---- K1, structured-grid forms (7-point faces, 27-point box) -----------------------
// The term order is fixed at compile time: lexicographic in (dz, dy, dx), which
// is the sorted-column order of the stencil's CSR form for nx, ny >= 3.  Per
// row the wrapped neighbour offsets along each axis are computed once; a
// term's column is then row + xo + yo + zo.
struct GridShapeTable {
  int nt;
};
inline GridShapeTable grid_shape_table(int shape) {
  return GridShapeTable{shape == SDB_SHAPE_FACE7 ? 7 : 27};
}

template <int SHAPE, int L, int VPL, int MODE, bool FIRST>
__global__ void __launch_bounds__(kStepThreads, step_min_blocks(L, VPL)) cheb_step_grid(StencilView S, StepArgs a0) {
  pdl_wait();
  pdl_trigger();
  using G = GridShape<SHAPE>;
  // column slices of one panel are adjacent blocks (slice fastest)
  const int slice = blockIdx.x % a0.slices;
  const int64_t sb = blockIdx.x / a0.slices;
  const int cs = (int)(a0.ldv / a0.slices);
  StepArgs a = a0;
  a.x += slice * cs;
  a.prev += slice * cs;
  a.next += slice * cs;
  a.v0 += slice * cs;
  if (a.halo_lo) a.halo_lo += slice * cs;
  if (a.halo_hi) a.halo_hi += slice * cs;
  constexpr int RPW = 32 / L;
  constexpr int RPB = RPW * kStepWarps;
  constexpr int U = VPL == 1 ? SDB_U_V1 : 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / L, q = lane % L;
  const uint64_t pol = policy_evict_first();
  const int nx = S.nx, ny = S.ny, nz = S.nz, nxy = nx * ny;
  double2 accA[VPL], accB[VPL], accZ[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) accA[v] = accB[v] = accZ[v] = make_double2(0.0, 0.0);
  for (int64_t ph = 0;; ++ph) {
    const int64_t p0 = (ph * a.nblocks + sb) * a.panel;
    if (p0 >= a.n) break;
    const int64_t pend = p0 + a.panel < a.n ? p0 + a.panel : a.n;
    for (int64_t base = p0; base < pend; base += RPB) {
      const int64_t row = base + warp * RPW + g;
      if (row >= pend) continue;
      EpiIn<VPL> e;
      epi_load<L, VPL, MODE, FIRST>(a, row, q, pol, e);
      const double dg = __ldg(S.diag + row);
      const int r32 = (int)row;
      const int ix = r32 % nx, t = r32 / nx;
      const int iy = t % ny, iz = t / ny;
      // wrapped offsets for d = -1, +1 along each axis
      const int xm = ix == 0 ? nx - 1 : -1, xp = ix == nx - 1 ? 1 - nx : 1;
      const int ym = iy == 0 ? (ny - 1) * nx : -nx, yp = iy == ny - 1 ? (1 - ny) * nx : nx;
      const int zm = (iz == 0 && !S.zghost) ? (nz - 1) * nxy : -nxy;
      const int zp = (iz == nz - 1 && !S.zghost) ? (1 - nz) * nxy : nxy;
      double2 y[VPL];
#pragma unroll
      for (int v = 0; v < VPL; ++v) y[v] = make_double2(0.0, 0.0);
#pragma unroll
      for (int o0 = 0; o0 < G::NT; o0 += U) {
        int col[U];
        double w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int o = o0 + u;
          if (o < G::NT) {
            const int ox = G::dx(o) < 0 ? xm : (G::dx(o) > 0 ? xp : 0);
            const int oy = G::dy(o) < 0 ? ym : (G::dy(o) > 0 ? yp : 0);
            const int oz = G::dz(o) < 0 ? zm : (G::dz(o) > 0 ? zp : 0);
            col[u] = r32 + ox + oy + oz;
            w[u] = (G::dx(o) == 0 && G::dy(o) == 0 && G::dz(o) == 0) ? dg : S.wc[o];
          } else {
            col[u] = r32;
            w[u] = 0.0;
          }
        }
        gather_fma<L, VPL, U>(a.x, a.ldv, q, col, w, y);
      }
      epi_finish<L, VPL, MODE, FIRST>(a, row, q, y, e, accA, accB, accZ, pol);
    }
  }
  if (a0.slices == 1) {
    step_finish<L, VPL, MODE, FIRST>(a, accA, accB, accZ);
  } else {
    __shared__ double smem[kStepWarps * SDB_MAX_BATCH];
    auto part = [&](double2 (&acc)[VPL], int slot) {
      block_partial_cols<L, VPL>(acc, smem, a0.partials, slot, a0.nblocks, a0.ldv, sb, slice * cs, cs);
    };
    if (a.slotA >= 0) part(accA, a.slotA);
    if constexpr (MODE == SDB_CHEB_DOUBLING) {
      if (a.slotB >= 0) part(accB, a.slotB);
    }
    if constexpr (FIRST) {
      if (a.slot0 >= 0) part(accZ, a.slot0);
    }
  }
}

#include "tile25d.cuh"

// Degree 0: only zeta_0 = <v0, v0>.
template <int L, int VPL>
__global__ void __launch_bounds__(kStepThreads) self_dot_kernel(StepArgs a) {
  constexpr int RPW = 32 / L;
  constexpr int RPB = RPW * kStepWarps;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / L, q = lane % L;
  double2 acc[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) acc[v] = make_double2(0.0, 0.0);
  const PanelSched sched{a.n, a.nblocks, a.panel};
  for_each_panel_chunk<RPB>(sched, [&](int64_t base, int64_t pend) {
    const int64_t row = base + warp * RPW + g;
    if (row < pend) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        double2 p = ld_d2(a.v0 + row * a.ldv + 2 * q + 2 * L * v);
        acc[v].x += p.x * p.x;
        acc[v].y += p.y * p.y;
      }
    }
  });
  __shared__ double smem[kStepWarps * SDB_MAX_BATCH];
  block_partial<L, VPL>(acc, smem, a.partials, 0, a.nblocks, a.ldv);
}

// ---- K2: partials -> per-probe moments ------------------------------------------
// Two fixed-order stages: (1) sums of kReduceChunk consecutive blocks per
// (slot, chunk, column), coalesced over columns; (2) per (slot, probe) the sum
// of the chunk sums in chunk order, then the doubling transform.  Deterministic.
constexpr int kReduceChunk = 64;

__global__ void cheb_reduce_stage1(const double* __restrict__ partials, int64_t nblocks, int64_t ldv, int64_t slots,
                                   int64_t nchunks, double* __restrict__ stage) {
  const int64_t total = slots * nchunks * ldv;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = idx % ldv, rest = idx / ldv;
    const int64_t ch = rest % nchunks, k = rest / nchunks;
    const int64_t b0 = ch * kReduceChunk, b1 = b0 + kReduceChunk < nblocks ? b0 + kReduceChunk : nblocks;
    const double* p = partials + (k * nblocks + b0) * ldv + l;
    double s = 0.0;
    for (int64_t b = b0; b < b1; ++b, p += ldv) s += *p;
    stage[idx] = s;
  }
}

__global__ void cheb_reduce_stage2(const double* __restrict__ stage, int64_t nchunks, int64_t ldv, int64_t n_vec,
                                   int64_t degree, int mode, double* __restrict__ zeta_pp) {
  const int64_t total = n_vec * (degree + 1);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx / n_vec, l = idx % n_vec;
    auto sum = [&](int64_t slot) {
      const double* p = stage + slot * nchunks * ldv + l;
      double s = 0.0;
      for (int64_t ch = 0; ch < nchunks; ++ch) s += p[ch * ldv];
      return s;
    };
    double r = sum(k);
    if (mode == SDB_CHEB_DOUBLING && k >= 2) r = 2.0 * r - sum(k & 1);
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
template <int MODE, bool FIRST>
static int launch_step(const sdb_matrix* m, const Geometry& g, const StencilView* st, const StepArgs& a,
                       cudaStream_t s) {
  dim3 grid((unsigned)(a.nblocks * a.slices)), block(kStepThreads);
  cudaError_t err = cudaSuccess;
  StepArgs aa = a;
  if (m->format == SDB_FMT_CSR) {
    CsrView A = make_csr_view(m);
    void* args[] = {(void*)&A, (void*)&aa};
#define SDB_STEP_CASE(LL, VV) err = launch_maybe_pdl((const void*)cheb_step_csr<LL, VV, MODE, FIRST>, grid, block, args, 0, s)
    SDB_GEOMETRY_DISPATCH(g, SDB_STEP_CASE);
#undef SDB_STEP_CASE
  } else if (m->shape == SDB_SHAPE_FACE7) {
    StencilView sv = *st;
    void* args[] = {(void*)&sv, (void*)&aa};
#define SDB_STEP_CASE(LL, VV) err = launch_maybe_pdl((const void*)cheb_step_grid<SDB_SHAPE_FACE7, LL, VV, MODE, FIRST>, grid, block, args, 0, s)
    SDB_GEOMETRY_DISPATCH(g, SDB_STEP_CASE);
#undef SDB_STEP_CASE
  } else if (m->shape == SDB_SHAPE_BOX27) {
    StencilView sv = *st;
    void* args[] = {(void*)&sv, (void*)&aa};
#define SDB_STEP_CASE(LL, VV) err = launch_maybe_pdl((const void*)cheb_step_grid<SDB_SHAPE_BOX27, LL, VV, MODE, FIRST>, grid, block, args, 0, s)
    SDB_GEOMETRY_DISPATCH(g, SDB_STEP_CASE);
#undef SDB_STEP_CASE
  } else {
    StencilView sv = *st;
    void* args[] = {(void*)&sv, (void*)&aa};
#define SDB_STEP_CASE(LL, VV) err = launch_maybe_pdl((const void*)cheb_step_stencil<LL, VV, MODE, FIRST>, grid, block, args, 0, s)
    SDB_GEOMETRY_DISPATCH(g, SDB_STEP_CASE);
#undef SDB_STEP_CASE
  }
  SDB_CUDA(err);
  return SDB_OK;
}

// Blocks for a moment run: every block of the phased schedule must be
// resident at once (a second wave would break the sliding window), so the
// count is SMs x (resident blocks per SM of the step kernels), capped by the
// number of row iterations.  Fixed per (matrix, geometry, GPU model).
static int64_t step_blocks(const sdb_matrix* m, const Geometry& g, int64_t rpb) {
  int occ = 0;
  const void* fns[4] = {};
  int nf = 0;
  if (m->format == SDB_FMT_CSR) {
#define SDB_OCC_CASE(LL, VV)                                                                \
  fns[0] = (const void*)cheb_step_csr<LL, VV, SDB_CHEB_DOUBLING, true>;                      \
  fns[1] = (const void*)cheb_step_csr<LL, VV, SDB_CHEB_DOUBLING, false>;                     \
  fns[2] = (const void*)cheb_step_csr<LL, VV, SDB_CHEB_DIRECT, true>;                        \
  fns[3] = (const void*)cheb_step_csr<LL, VV, SDB_CHEB_DIRECT, false>;                       \
  nf = 4
    [&]() -> int { SDB_GEOMETRY_DISPATCH(g, SDB_OCC_CASE); return 0; }();
#undef SDB_OCC_CASE
  } else if (m->shape == SDB_SHAPE_FACE7) {
#define SDB_OCC_CASE(LL, VV)                                                                 \
  fns[0] = (const void*)cheb_step_grid<SDB_SHAPE_FACE7, LL, VV, SDB_CHEB_DOUBLING, true>;     \
  fns[1] = (const void*)cheb_step_grid<SDB_SHAPE_FACE7, LL, VV, SDB_CHEB_DOUBLING, false>;    \
  fns[2] = (const void*)cheb_step_grid<SDB_SHAPE_FACE7, LL, VV, SDB_CHEB_DIRECT, true>;       \
  fns[3] = (const void*)cheb_step_grid<SDB_SHAPE_FACE7, LL, VV, SDB_CHEB_DIRECT, false>;      \
  nf = 4
    [&]() -> int { SDB_GEOMETRY_DISPATCH(g, SDB_OCC_CASE); return 0; }();
#undef SDB_OCC_CASE
  } else if (m->shape == SDB_SHAPE_BOX27) {
#define SDB_OCC_CASE(LL, VV)                                                                 \
  fns[0] = (const void*)cheb_step_grid<SDB_SHAPE_BOX27, LL, VV, SDB_CHEB_DOUBLING, true>;     \
  fns[1] = (const void*)cheb_step_grid<SDB_SHAPE_BOX27, LL, VV, SDB_CHEB_DOUBLING, false>;    \
  fns[2] = (const void*)cheb_step_grid<SDB_SHAPE_BOX27, LL, VV, SDB_CHEB_DIRECT, true>;       \
  fns[3] = (const void*)cheb_step_grid<SDB_SHAPE_BOX27, LL, VV, SDB_CHEB_DIRECT, false>;      \
  nf = 4
    [&]() -> int { SDB_GEOMETRY_DISPATCH(g, SDB_OCC_CASE); return 0; }();
#undef SDB_OCC_CASE
  } else {
#define SDB_OCC_CASE(LL, VV)                                                                \
  fns[0] = (const void*)cheb_step_stencil<LL, VV, SDB_CHEB_DOUBLING, true>;                  \
  fns[1] = (const void*)cheb_step_stencil<LL, VV, SDB_CHEB_DOUBLING, false>;                 \
  fns[2] = (const void*)cheb_step_stencil<LL, VV, SDB_CHEB_DIRECT, true>;                    \
  fns[3] = (const void*)cheb_step_stencil<LL, VV, SDB_CHEB_DIRECT, false>;                   \
  nf = 4
    [&]() -> int { SDB_GEOMETRY_DISPATCH(g, SDB_OCC_CASE); return 0; }();
#undef SDB_OCC_CASE
  }
  occ = 1 << 20;
  for (int i = 0; i < nf; ++i) {
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fns[i], kStepThreads, 0) != cudaSuccess || o < 1) o = 1;
    occ = o < occ ? o : occ;
  }
  if (nf == 0) occ = 4;
  if (const char* env = getenv("SDB_BLOCKS_PER_SM")) {
    int v = atoi(env);
    if (v > 0) occ = v;
  }
  int64_t b = (int64_t)occ * num_sms(m->device);
  const int64_t iters = (m->n + rpb - 1) / rpb;
  if (iters < b) b = iters;
  return b < 1 ? 1 : b;
}

static int launch_self_dot(const Geometry& g, const StepArgs& a, cudaStream_t s) {
#define SDB_SD_CASE(LL, VV) self_dot_kernel<LL, VV><<<(unsigned)a.nblocks, kStepThreads, 0, s>>>(a)
  SDB_GEOMETRY_DISPATCH(g, SDB_SD_CASE);
#undef SDB_SD_CASE
  return SDB_OK;
}

// ---- 2.5-D tile path (tile25d.cuh) ------------------------------------------------
struct TilePlan {
  bool on = false;
  int CS = 8, TY = 2, PD = 2;
  int slices = 0;
  int64_t nblocks = 0;  // spatial blocks (partials rows)
  TileArgs t{};
  size_t smem = 0;
};

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

static TilePlan plan_tile(const sdb_matrix* m, int64_t ldv, int mode) {
  TilePlan p;
  if (mode != SDB_CHEB_DOUBLING || m->format != SDB_FMT_STENCIL) return p;
  if (m->shape != SDB_SHAPE_FACE7 && m->shape != SDB_SHAPE_BOX27) return p;
  // Measured (profiles/r01_tile_sweep.txt): the tile path wins for the
  // 27-point box (C5: 8.8 -> 4.8 ms/step) but not for the 7-point star at 64
  // probes, where the row-panel grid kernel is faster; SDB_TILE=1 forces it.
  const int dflt = m->shape == SDB_SHAPE_BOX27 ? 1 : 0;
  if (!env_int("SDB_TILE", dflt)) return p;
  p.CS = env_int("SDB_TILE_CS", ldv % 16 == 0 ? 16 : 8);
  p.TY = env_int("SDB_TILE_TY", 2);
  p.PD = env_int("SDB_TILE_PD", 1);
  if (!((p.CS == 8 || p.CS == 16) && (p.TY == 2 || p.TY == 4) && (p.PD >= 1 && p.PD <= 3))) return p;
  if (ldv % p.CS != 0) return p;
  const int nx = (int)m->st.nx, ny = (int)m->st.ny, nz = (int)m->st.nz;
  p.t.nx = nx;
  p.t.ny = ny;
  p.t.nz = nz;
  p.t.TX = nx < kTileMaxX ? nx : kTileMaxX;
  p.t.n_xt = (nx + p.t.TX - 1) / p.t.TX;
  p.t.n_yt = (ny + p.TY - 1) / p.TY;
  p.slices = (int)(ldv / p.CS);
  p.t.slices = p.slices;
  const int64_t base = (int64_t)p.t.n_xt * p.t.n_yt * p.slices;
  const int64_t want = 4LL * num_sms(m->device);
  int nzs = (int)((want + base - 1) / base);
  if (const char* e = getenv("SDB_TILE_ZSEG")) nzs = atoi(e);
  nzs = nzs < 1 ? 1 : nzs;
  if (nzs > nz / 4) nzs = nz / 4 > 0 ? nz / 4 : 1;
  p.t.ZS = (nz + nzs - 1) / nzs;
  p.t.n_zs = (nz + p.t.ZS - 1) / p.t.ZS;
  {
    const size_t px = kTileMaxX + 2, R = 3 + p.PD, RP = p.PD + 1;
    p.smem = sizeof(double) * (R * (p.TY + 2) * px * p.CS + RP * p.TY * kTileMaxX * p.CS + RP * p.TY * kTileMaxX);
    if (p.smem > 227 * 1024) return p;  // does not fit: grid kernel instead
  }
  p.t.diag = m->diag;
  p.t.zghost = m->zghost;
  // weights in lexicographic (dz, dy, dx) order = sorted term order
  for (int o = 0; o < 27; ++o) p.t.wc[o] = 0.0;
  const GridShapeTable tab = grid_shape_table(m->shape);
  for (int o = 0; o < tab.nt; ++o) p.t.wc[o] = o < m->nterms ? m->term_w_host[o] : 0.0;
  p.nblocks = (int64_t)p.t.n_xt * p.t.n_yt * p.t.n_zs;
  if (p.nblocks > 8LL * num_sms(m->device)) return p;  // partials sized for <= 8 blocks per SM
  p.on = true;
  return p;
}

template <int SHAPE, int CS, int TY, int PD, bool FIRST>
static int launch_tile_t(const TilePlan& p, const StepArgs& a, cudaStream_t s) {
  auto fn = cheb_step_tile<SHAPE, CS, TY, PD, FIRST>;
  constexpr size_t smem = TileSmem<CS, TY, PD>::bytes;
  static bool configured = false;  // per instantiation
  if (!configured) {
    SDB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  dim3 grid((unsigned)(p.nblocks * p.slices));
  TileArgs tt = p.t;
  StepArgs aa = a;
  void* args[] = {(void*)&tt, (void*)&aa};
  SDB_CUDA(launch_maybe_pdl((const void*)fn, grid, dim3(kTileThreads), args, smem, s));
  return SDB_OK;
}

template <bool FIRST>
static int launch_tile(const sdb_matrix* m, const TilePlan& p, const StepArgs& a, cudaStream_t s) {
#define SDB_TILE_PD(SH, CS_, TY_)                                                                  \
  if (p.CS == CS_ && p.TY == TY_) {                                                                \
    if (p.PD == 1) return launch_tile_t<SH, CS_, TY_, 1, FIRST>(p, a, s);                          \
    if (p.PD == 2) return launch_tile_t<SH, CS_, TY_, 2, FIRST>(p, a, s);                          \
    if (p.PD == 3) return launch_tile_t<SH, CS_, TY_, 3, FIRST>(p, a, s);                          \
  }
#define SDB_TILE_CASE(SH) SDB_TILE_PD(SH, 8, 2) SDB_TILE_PD(SH, 8, 4) SDB_TILE_PD(SH, 16, 2) SDB_TILE_PD(SH, 16, 4)
  if (m->shape == SDB_SHAPE_FACE7) {
    SDB_TILE_CASE(SDB_SHAPE_FACE7)
  } else {
    SDB_TILE_CASE(SDB_SHAPE_BOX27)
  }
#undef SDB_TILE_CASE
#undef SDB_TILE_PD
  return fail(SDB_EUNSUPPORTED, "no tile kernel for CS=%d TY=%d PD=%d", p.CS, p.TY, p.PD);
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

static void cheb_layout(const sdb_matrix* m, int64_t ldv, int64_t degree, size_t* block_bytes,
                        size_t* partial_bytes) {
  // partial_bytes covers the block partials plus the stage-1 reduce buffer
  *block_bytes = align256(sizeof(double) * (size_t)m->n * (size_t)ldv);
  // upper bound on step_blocks(): 8 resident 256-thread blocks per SM
  const int64_t bmax = 8LL * num_sms(m->device);
  const int64_t cmax = (bmax + kReduceChunk - 1) / kReduceChunk;
  *partial_bytes = align256(sizeof(double) * (size_t)(degree + 1) * (size_t)(bmax + cmax) * (size_t)ldv);
}

// ---- step planning shared by the moment driver and the step-level ABI ------------
struct StepPlan {
  Geometry g;   // block geometry (ldv)
  Geometry gk;  // geometry of the launched kernel (per column slice)
  TilePlan tp;
  StepArgs a;   // n, ldv, nblocks, panel, slices, c, inv_d filled
  StencilView st;
  int device;
};

static int plan_steps(const sdb_matrix* m, int64_t n_vec, int mode, double c, double d, StepPlan* P) {
  SDB_REQUIRE(n_vec >= 1 && n_vec <= SDB_MAX_BATCH, "n_vec must lie in [1, %d] per batch", SDB_MAX_BATCH);
  SDB_REQUIRE(mode == SDB_CHEB_DIRECT || mode == SDB_CHEB_DOUBLING, "unknown moment mode %d", mode);
  StepPlan& p = *P;
  p.device = m->device;
  p.g = choose_geometry(n_vec);
  p.gk = p.g;
  p.a = StepArgs{};
  p.a.c = c;
  p.a.inv_d = 1.0 / d;
  p.a.n = m->n;
  p.a.ldv = p.g.ldv;
  p.tp = plan_tile(m, p.g.ldv, mode);
  p.a.slices = 1;
  if (!p.tp.on && m->format == SDB_FMT_STENCIL && (m->shape == SDB_SHAPE_FACE7 || m->shape == SDB_SHAPE_BOX27)) {
    const int sl = env_int("SDB_GRID_SLICES", 1);
    if (sl > 1 && p.g.ldv % (2 * sl) == 0) {
      Geometry gs = choose_geometry(p.g.ldv / sl);
      if (gs.ldv == p.g.ldv / sl) {
        p.a.slices = sl;
        p.gk = gs;
      }
    }
  }
  const int rpbk = (32 / p.gk.L) * kStepWarps;
  p.a.nblocks = p.tp.on ? p.tp.nblocks : step_blocks(m, p.gk, rpbk) / p.a.slices;
  if (p.a.nblocks < 1) p.a.nblocks = 1;
  p.a.panel = panel_rows(m, p.g.ldv, rpbk);
  p.st = StencilView{};
  if (m->format == SDB_FMT_STENCIL) p.st = make_stencil_view(m);
  return SDB_OK;
}

static int launch_plan_step(const sdb_matrix* m, const StepPlan& P, int64_t degree, int mode, int64_t k,
                            const double* x, const double* prev, double* next, const double* v0, double* partials,
                            cudaStream_t s) {
  StepArgs a = P.a;
  a.partials = partials;
  a.v0 = v0;
  int rc;
  const int64_t steps = (mode == SDB_CHEB_DOUBLING) ? (degree + 1) / 2 : degree;
  if (steps == 0) {  // degree 0: only zeta_0 = <v0, v0>
    a.v0 = x;
    a.slot0 = 0;
    if ((rc = launch_self_dot(P.g, a, s))) return rc;
    SDB_CHECK_LAUNCH();
    return SDB_OK;
  }
  a.x = x;
  a.prev = prev;
  a.next = next;
  a.slot0 = (k == 0) ? 0 : -1;
  set_step_scalars(a, k);
  if (mode == SDB_CHEB_DOUBLING) {
    a.slotB = (2 * k + 1 <= degree) ? (int)(2 * k + 1) : -1;
    a.slotA = (2 * k + 2 <= degree) ? (int)(2 * k + 2) : -1;
    if (P.tp.on)
      rc = k == 0 ? launch_tile<true>(m, P.tp, a, s) : launch_tile<false>(m, P.tp, a, s);
    else
      rc = k == 0 ? launch_step<SDB_CHEB_DOUBLING, true>(m, P.gk, &P.st, a, s)
                  : launch_step<SDB_CHEB_DOUBLING, false>(m, P.gk, &P.st, a, s);
  } else {
    a.slotA = (int)(k + 1);
    a.slotB = -1;
    rc = k == 0 ? launch_step<SDB_CHEB_DIRECT, true>(m, P.gk, &P.st, a, s)
                : launch_step<SDB_CHEB_DIRECT, false>(m, P.gk, &P.st, a, s);
  }
  if (rc) return rc;
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

static int launch_reduce(const StepPlan& P, int64_t n_vec, int64_t degree, int mode, const double* partials,
                         double* zeta_pp, cudaStream_t s, int64_t ldv_override = 0) {
  const int64_t nb = P.a.nblocks, ldv = ldv_override > 0 ? ldv_override : P.g.ldv, slots = degree + 1;
  const int64_t nch = (nb + kReduceChunk - 1) / kReduceChunk;
  // stage buffer sits behind the largest possible partials array (cheb_layout)
  const int64_t bmax = 8LL * num_sms(P.device);
  double* stage = const_cast<double*>(partials) + slots * bmax * ldv;
  const int64_t t1 = slots * nch * ldv;
  int b1 = (int)((t1 + 255) / 256);
  if (b1 > 65535) b1 = 65535;
  cheb_reduce_stage1<<<b1, 256, 0, s>>>(partials, nb, ldv, slots, nch, stage);
  SDB_CHECK_LAUNCH();
  const int64_t t2 = n_vec * slots;
  int b2 = (int)((t2 + 255) / 256);
  if (b2 > 65535) b2 = 65535;
  cheb_reduce_stage2<<<b2, 256, 0, s>>>(stage, nch, ldv, n_vec, degree, mode, zeta_pp);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

// Moment run on the probe-sliced band + far path (band.cu): slice-major copy
// of the probes, PDL-chained step launches, K2 over the band kernel's partial
// rows.  Timed from the probe copy, like the z-march padding.
static int band_moments(const sdb_matrix* m, const StepPlan& P0, const BandPlan& bp, int64_t n_vec, int64_t degree,
                        int mode, const double* probes, double* zeta_pp, void* workspace, cudaStream_t s,
                        float* step_ms) {
  double* v0b = (double*)workspace;
  double* bufA = (double*)((char*)workspace + bp.block_bytes);
  double* bufB = (double*)((char*)workspace + 2 * bp.block_bytes);
  double* partials = (double*)((char*)workspace + 3 * bp.block_bytes);
  const int64_t steps = (mode == SDB_CHEB_DOUBLING) ? (degree + 1) / 2 : degree;
  PdlScope pdl_scope;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (step_ms) {
    SDB_CUDA(cudaEventCreate(&e0));
    SDB_CUDA(cudaEventCreate(&e1));
    SDB_CUDA(cudaEventRecord(e0, s));
  }
  int rc = band_pack(m, bp, probes, P0.g.ldv, v0b, bufA, bufB, s);
  if (rc) return rc;
  const double* cur = v0b;
  const double* prev = nullptr;
  for (int64_t k = 0; k < steps; ++k) {
    double* next = k == 0 ? bufA : (k == 1 ? bufB : const_cast<double*>(prev));
    StepArgs a = P0.a;
    a.partials = partials;
    a.v0 = v0b;
    a.x = cur;
    a.prev = prev;
    a.next = next;
    a.slot0 = (k == 0) ? 0 : -1;
    set_step_scalars(a, k);
    if (mode == SDB_CHEB_DOUBLING) {
      a.slotB = (2 * k + 1 <= degree) ? (int)(2 * k + 1) : -1;
      a.slotA = (2 * k + 2 <= degree) ? (int)(2 * k + 2) : -1;
    } else {
      a.slotA = (int)(k + 1);
      a.slotB = -1;
    }
    if ((rc = band_launch_step(m, bp, a, k == 0, mode, s))) return rc;
    prev = cur;
    cur = next;
  }
  if (step_ms) SDB_CUDA(cudaEventRecord(e1, s));
  StepPlan P = P0;
  P.a.nblocks = bp.grid;
  if ((rc = launch_reduce(P, n_vec, degree, mode, partials, zeta_pp, s, bp.ldvb))) return rc;
  if (step_ms) {
    SDB_CUDA(cudaEventSynchronize(e1));
    SDB_CUDA(cudaEventElapsedTime(step_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return SDB_OK;
}

// Moment run on the cluster-resident path (resident.cu): every step in one
// launch, K2 over its per-warp partial rows.  The recurrence blocks of the
// workspace are not used; the partials sit at its start.
static int resident_moments(const sdb_matrix* m, const StepPlan& P0, const ResPlan& rp, int64_t n_vec,
                            int64_t degree, int mode, const double* probes, double* zeta_pp, void* workspace,
                            cudaStream_t s, float* step_ms) {
  double* partials = (double*)workspace;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (step_ms) {
    SDB_CUDA(cudaEventCreate(&e0));
    SDB_CUDA(cudaEventCreate(&e1));
    SDB_CUDA(cudaEventRecord(e0, s));
  }
  int rc = res_launch(m, rp, P0.a, degree, mode, probes, partials, s);
  if (rc) return rc;
  if (step_ms) SDB_CUDA(cudaEventRecord(e1, s));
  StepPlan P = P0;
  P.a.nblocks = rp.nblocks;
  if ((rc = launch_reduce(P, n_vec, degree, mode, partials, zeta_pp, s))) return rc;
  if (step_ms) {
    SDB_CUDA(cudaEventSynchronize(e1));
    SDB_CUDA(cudaEventElapsedTime(step_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return SDB_OK;
}

}  // namespace sdb

using namespace sdb;

extern "C" {

int sdb_cheb_workspace_size(const sdb_matrix* m, int64_t n_vec, int64_t degree, int mode, size_t* bytes) {
  int leg_;
  mode = split_mode(mode, &leg_);
  SDB_REQUIRE(m && bytes, "NULL argument");
  SDB_REQUIRE(n_vec >= 1 && n_vec <= SDB_MAX_BATCH, "n_vec must lie in [1, %d] per batch", SDB_MAX_BATCH);
  SDB_REQUIRE(degree >= 0, "degree must be non-negative");
  SDB_REQUIRE(mode == SDB_CHEB_DIRECT || mode == SDB_CHEB_DOUBLING, "unknown moment mode %d", mode);
  Geometry g = choose_geometry(n_vec);
  size_t bb, pb;
  BandPlan bp;
  int rc = band_plan(m, n_vec, mode, &bp);
  if (rc) return rc;
  if (bp.on) {  // slice-major probe copy + two recurrence blocks + partials
    cheb_layout(m, bp.ldvb, degree, &bb, &pb);
    *bytes = 3 * bp.block_bytes + pb;
    return SDB_OK;
  }
  cheb_layout(m, g.ldv, degree, &bb, &pb);
  ZmPlan zp;
  rc = zm_plan(m, g.ldv, mode, &zp);
  if (rc) return rc;
  // z-march path: padded probe copy + two padded recurrence buffers (fused
  // pairs: + a third and the padded diagonal)
  *bytes = !zp.on ? 2 * bb + pb : (zp.fuse ? 4 * zp.block_bytes + zp.diag_bytes + pb : 3 * zp.block_bytes + pb);
  return SDB_OK;
}

const char* sdb_cheb_kernel(const sdb_matrix* m, int64_t n_vec, int mode) {
  int leg_;
  mode = split_mode(mode, &leg_);
  if (!m || n_vec < 1 || n_vec > SDB_MAX_BATCH) return "";
  const Geometry g = choose_geometry(n_vec);
  BandPlan bp;
  if (band_plan(m, n_vec, mode, &bp) == SDB_OK && bp.on) return "cheb_step_band";
  ZmPlan zp;
  if (zm_plan(m, g.ldv, mode, &zp) == SDB_OK && zp.on) return zp.name;
  ResPlan rp;
  if (res_plan(m, n_vec, mode, &rp) == SDB_OK && rp.on) return "cheb_resident";
  if (m->format == SDB_FMT_CSR) return "cheb_step_csr";
  if (plan_tile(m, g.ldv, mode).on) return "cheb_step_tile";
  if (m->shape == SDB_SHAPE_FACE7 || m->shape == SDB_SHAPE_BOX27) return "cheb_step_grid";
  return "cheb_step_stencil";
}

int sdb_cheb_moments(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree, int mode,
                     const double* probes, double* zeta_pp, void* workspace, size_t workspace_bytes, void* stream,
                     float* step_ms) {
  SDB_REQUIRE(m && probes && zeta_pp, "NULL argument");
  int legendre;
  mode = split_mode(mode, &legendre);
  size_t need = 0;
  int rc = sdb_cheb_workspace_size(m, n_vec, degree, mode, &need);
  if (rc) return rc;
  SDB_REQUIRE(workspace != nullptr && workspace_bytes >= need, "workspace too small (%zu < %zu bytes)",
              workspace_bytes, need);
  SDB_REQUIRE(d != 0.0, "spectral halfwidth must be non-zero");
  DeviceGuard dg(m->device);
  if (!dg.ok) return fail(SDB_ECUDA, "cannot select CUDA device %d", m->device);
  cudaStream_t s = (cudaStream_t)stream;
  StepPlan P;
  if ((rc = plan_steps(m, n_vec, mode, c, d, &P))) return rc;
  P.a.legendre = legendre;
  {
    const int64_t steps_b = (mode == SDB_CHEB_DOUBLING) ? (degree + 1) / 2 : degree;
    BandPlan bp;
    if ((rc = band_plan(m, n_vec, mode, &bp))) return rc;
    if (bp.on && steps_b > 0)
      return band_moments(m, P, bp, n_vec, degree, mode, probes, zeta_pp, workspace, (cudaStream_t)stream,
                          step_ms);
    ResPlan rp;
    if ((rc = res_plan(m, n_vec, mode, &rp))) return rc;
    if (rp.on && steps_b > 0)
      return resident_moments(m, P, rp, n_vec, degree, mode, probes, zeta_pp, workspace, (cudaStream_t)stream,
                              step_ms);
  }
  size_t bb, pb;
  cheb_layout(m, P.g.ldv, degree, &bb, &pb);
  ZmPlan zp;
  if ((rc = zm_plan(m, P.g.ldv, mode, &zp))) return rc;
  const int64_t steps = (mode == SDB_CHEB_DOUBLING) ? (degree + 1) / 2 : degree;
  if (steps == 0) zp.on = false;  // degree 0: only <v0, v0>
  const size_t blk = zp.on ? zp.block_bytes : bb;
  double* bufA = (double*)workspace;
  double* bufB = (double*)((char*)workspace + blk);
  double* padded = zp.on ? (double*)((char*)workspace + 2 * blk) : nullptr;
  double* bufC = zp.fuse ? (double*)((char*)workspace + 3 * blk) : nullptr;
  double* diag_padded = zp.fuse ? (double*)((char*)workspace + 4 * blk) : nullptr;
  double* partials = (double*)((char*)workspace + (zp.fuse ? 4 * blk + zp.diag_bytes : (zp.on ? 3 : 2) * blk));

  PdlScope pdl_scope;  // step kernels of this loop overlap their launch with the previous step's tail
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (step_ms) {
    SDB_CUDA(cudaEventCreate(&e0));
    SDB_CUDA(cudaEventCreate(&e1));
    SDB_CUDA(cudaEventRecord(e0, s));
  }
  const double* v0 = probes;
  if (zp.on) {  // ghost-padded copy of the probes (counted in the step time)
    if ((rc = zm_pad(m, zp, probes, P.g.ldv, padded, s))) return rc;
    v0 = padded;
  }
  const double* cur = v0;
  const double* prev = nullptr;
  int64_t k0 = 0;
  if (zp.on && zp.fuse) {
    // fused pairs of steps; buffers rotate over {padded, A, B, C} (each pair
    // writes two buffers distinct from its x and prev)
    if ((rc = zm_pad_diag(m, diag_padded, s))) return rc;
    double* pool[4] = {padded, bufA, bufB, bufC};
    auto clip = [&](int64_t slot) { return slot <= degree ? (int)slot : -1; };
    for (; k0 + 1 < steps; k0 += 2) {
      double* outs[2];
      int no = 0;
      for (int i = 0; i < 4 && no < 2; ++i)
        if (pool[i] != cur && pool[i] != prev) outs[no++] = pool[i];
      StepArgs a = P.a;
      a.partials = partials;
      a.v0 = v0;
      a.x = cur;
      a.prev = prev;
      a.next = outs[0];
      a.next2 = outs[1];
      a.slot0 = (k0 == 0) ? 0 : -1;
      a.slotB = clip(2 * k0 + 1);
      a.slotA = clip(2 * k0 + 2);
      a.slotB2 = clip(2 * k0 + 3);
      a.slotA2 = clip(2 * k0 + 4);
      if ((rc = zm_launch_pair(m, zp, a, diag_padded, k0 == 0, s))) return rc;
      prev = outs[0];
      cur = outs[1];
    }
    if (k0 < steps) {  // odd step count: one single step, written over a free buffer
      double* out = nullptr;
      for (int i = 0; i < 4 && !out; ++i)
        if (pool[i] != cur && pool[i] != prev) out = pool[i];
      bufA = out;  // picked up as `next` by the loop below (k0 >= 1 -> k0 != 1 handled there)
    }
  }
  for (int64_t k = k0; k < (steps > 0 ? steps : 1); ++k) {
    double* next = (k == 0 || (zp.fuse && k == k0 && k0 > 0)) ? bufA
                   : (k == 1 ? bufB : const_cast<double*>(prev));
    if (zp.on) {
      StepArgs a = P.a;
      a.partials = partials;
      a.v0 = v0;
      a.x = cur;
      a.prev = prev;
      a.next = next;
      a.slot0 = (k == 0) ? 0 : -1;
      set_step_scalars(a, k);
      if (mode == SDB_CHEB_DOUBLING) {
        a.slotB = (2 * k + 1 <= degree) ? (int)(2 * k + 1) : -1;
        a.slotA = (2 * k + 2 <= degree) ? (int)(2 * k + 2) : -1;
      } else {
        a.slotA = (int)(k + 1);
        a.slotB = -1;
      }
      if ((rc = zm_launch_step(m, zp, a, k == 0, mode, s))) return rc;
    } else if ((rc = launch_plan_step(m, P, degree, mode, k, cur, prev, next, probes, partials, s))) {
      return rc;
    }
    prev = cur;
    cur = next;
  }
  if (zp.on) P.a.nblocks = zp.nbp;  // partial rows the reduce sums
  if (step_ms) SDB_CUDA(cudaEventRecord(e1, s));
  if ((rc = launch_reduce(P, n_vec, degree, mode, partials, zeta_pp, s))) return rc;
  if (step_ms) {
    SDB_CUDA(cudaEventSynchronize(e1));
    SDB_CUDA(cudaEventElapsedTime(step_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return SDB_OK;
}

int sdb_cheb_partials_size(const sdb_matrix* m, int64_t n_vec, int64_t degree, int mode, size_t* bytes) {
  SDB_REQUIRE(m && bytes, "NULL argument");
  size_t need = 0;
  int rc = sdb_cheb_workspace_size(m, n_vec, degree, mode, &need);
  if (rc) return rc;
  size_t bb, pb;
  cheb_layout(m, choose_geometry(n_vec).ldv, degree, &bb, &pb);
  *bytes = pb;
  return SDB_OK;
}

static int cheb_step_impl(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree, int mode,
                          int64_t k, const double* x, const double* prev, double* next, const double* v0,
                          double* partials, size_t partial_bytes, double* halo_lo, double* halo_hi, void* stream);

int sdb_cheb_step(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree, int mode, int64_t k,
                  const double* x, const double* prev, double* next, const double* v0, double* partials,
                  size_t partial_bytes, void* stream) {
  return cheb_step_impl(m, c, d, n_vec, degree, mode, k, x, prev, next, v0, partials, partial_bytes, nullptr,
                        nullptr, stream);
}

int sdb_cheb_step_halo(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree, int mode, int64_t k,
                       const double* x, const double* prev, double* next, const double* v0, double* partials,
                       size_t partial_bytes, double* halo_lo, double* halo_hi, void* stream) {
  SDB_REQUIRE(m && m->format == SDB_FMT_STENCIL, "halo push needs a stencil slab handle");
  return cheb_step_impl(m, c, d, n_vec, degree, mode, k, x, prev, next, v0, partials, partial_bytes, halo_lo,
                        halo_hi, stream);
}

static int cheb_step_impl(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree, int mode,
                          int64_t k, const double* x, const double* prev, double* next, const double* v0,
                          double* partials, size_t partial_bytes, double* halo_lo, double* halo_hi, void* stream) {
  SDB_REQUIRE(m && x && partials, "NULL argument");
  int legendre;
  mode = split_mode(mode, &legendre);
  size_t pb = 0;
  int rc = sdb_cheb_partials_size(m, n_vec, degree, mode, &pb);
  if (rc) return rc;
  SDB_REQUIRE(partial_bytes >= pb, "partials buffer too small (%zu < %zu bytes)", partial_bytes, pb);
  const int64_t steps = (mode == SDB_CHEB_DOUBLING) ? (degree + 1) / 2 : degree;
  SDB_REQUIRE(k >= 0 && (k < steps || (steps == 0 && k == 0)), "step %lld outside [0, %lld)", (long long)k,
              (long long)steps);
  SDB_REQUIRE(steps == 0 || next != nullptr, "next must not be NULL");
  SDB_REQUIRE(k == 0 || prev != nullptr, "prev must not be NULL after the first step");
  SDB_REQUIRE(mode != SDB_CHEB_DIRECT || v0 != nullptr || k == 0, "direct mode needs v0");
  SDB_REQUIRE(d != 0.0, "spectral halfwidth must be non-zero");
  DeviceGuard dg(m->device);
  if (!dg.ok) return fail(SDB_ECUDA, "cannot select CUDA device %d", m->device);
  StepPlan P;
  if ((rc = plan_steps(m, n_vec, mode, c, d, &P))) return rc;
  P.a.legendre = legendre;
  if (halo_lo || halo_hi) {
    P.a.halo_lo = halo_lo;
    P.a.halo_hi = halo_hi;
    P.a.halo_rows = m->st.nx * m->st.ny;
    P.a.last_row0 = (m->st.nz - 1) * P.a.halo_rows;
  }
  return launch_plan_step(m, P, degree, mode, k, x, prev, next, v0 ? v0 : x, partials, (cudaStream_t)stream);
}

int sdb_cheb_reduce(const sdb_matrix* m, int64_t n_vec, int64_t degree, int mode, const double* partials,
                    double* zeta_pp, void* stream) {
  int leg_;
  mode = split_mode(mode, &leg_);
  SDB_REQUIRE(m && partials && zeta_pp, "NULL argument");
  SDB_REQUIRE(n_vec >= 1 && n_vec <= SDB_MAX_BATCH && degree >= 0, "bad shape");
  DeviceGuard dg(m->device);
  if (!dg.ok) return fail(SDB_ECUDA, "cannot select CUDA device %d", m->device);
  StepPlan P;
  int rc = plan_steps(m, n_vec, mode, 0.0, 1.0, &P);
  if (rc) return rc;
  return launch_reduce(P, n_vec, degree, mode, partials, zeta_pp, (cudaStream_t)stream);
}

int sdb_zm_block_info(const sdb_matrix* m, int64_t n_vec, int mode, int64_t* plane_doubles, size_t* block_bytes) {
  SDB_REQUIRE(m && plane_doubles && block_bytes, "NULL argument");
  SDB_REQUIRE(n_vec >= 1 && n_vec <= SDB_MAX_BATCH, "n_vec must lie in [1, %d] per batch", SDB_MAX_BATCH);
  int leg_;
  mode = split_mode(mode, &leg_);
  const int64_t ldv = choose_geometry(n_vec).ldv;
  ZmPlan zp;
  int rc = zm_plan(m, ldv, mode, &zp);
  if (rc) return rc;
  *plane_doubles = 0;
  *block_bytes = 0;
  if (!zp.on || zp.fuse) return SDB_OK;
  *plane_doubles = (m->st.ny + 2 * zp.G) * (m->st.nx + 2 * zp.G) * ldv;
  *block_bytes = zp.block_bytes;
  return SDB_OK;
}

int sdb_zm_pad_probes(const sdb_matrix* m, int64_t n_vec, const double* probes, double* padded, void* stream) {
  SDB_REQUIRE(m && probes && padded, "NULL argument");
  SDB_REQUIRE(n_vec >= 1 && n_vec <= SDB_MAX_BATCH, "n_vec must lie in [1, %d] per batch", SDB_MAX_BATCH);
  const int64_t ldv = choose_geometry(n_vec).ldv;
  ZmPlan zp;
  int rc = zm_plan(m, ldv, SDB_CHEB_DOUBLING, &zp);
  if (rc) return rc;
  SDB_REQUIRE(zp.on && !zp.fuse, "the z-march layout does not apply to this matrix");
  DeviceGuard dg(m->device);
  if (!dg.ok) return fail(SDB_ECUDA, "cannot select CUDA device %d", m->device);
  return zm_pad(m, zp, probes, ldv, padded, (cudaStream_t)stream);
}

static int step_planes_impl(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree, int mode,
                            int64_t k, int64_t z_lo, int64_t z_hi, const double* x, const double* prev, double* next,
                            const double* v0, double* partials, size_t partial_bytes, double* halo_lo,
                            double* halo_hi, void* stream);

int sdb_cheb_step_planes(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree, int mode, int64_t k,
                         int64_t z_lo, int64_t z_hi, const double* x, const double* prev, double* next,
                         const double* v0, double* partials, size_t partial_bytes, void* stream) {
  return step_planes_impl(m, c, d, n_vec, degree, mode, k, z_lo, z_hi, x, prev, next, v0, partials, partial_bytes,
                          nullptr, nullptr, stream);
}

int sdb_cheb_step_planes_halo(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree, int mode,
                              int64_t k, int64_t z_lo, int64_t z_hi, const double* x, const double* prev,
                              double* next, const double* v0, double* partials, size_t partial_bytes,
                              double* halo_lo, double* halo_hi, void* stream) {
  return step_planes_impl(m, c, d, n_vec, degree, mode, k, z_lo, z_hi, x, prev, next, v0, partials, partial_bytes,
                          halo_lo, halo_hi, stream);
}

static int step_planes_impl(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t degree, int mode,
                            int64_t k, int64_t z_lo, int64_t z_hi, const double* x, const double* prev, double* next,
                            const double* v0, double* partials, size_t partial_bytes, double* halo_lo,
                            double* halo_hi, void* stream) {
  SDB_REQUIRE(m && x && next && partials, "NULL argument");
  int legendre;
  mode = split_mode(mode, &legendre);
  size_t pb = 0;
  int rc = sdb_cheb_partials_size(m, n_vec, degree, mode, &pb);
  if (rc) return rc;
  SDB_REQUIRE(partial_bytes >= pb, "partials buffer too small (%zu < %zu bytes)", partial_bytes, pb);
  const int64_t steps = (mode == SDB_CHEB_DOUBLING) ? (degree + 1) / 2 : degree;
  SDB_REQUIRE(k >= 0 && k < steps, "step %lld outside [0, %lld)", (long long)k, (long long)steps);
  SDB_REQUIRE(k == 0 || prev != nullptr, "prev must not be NULL after the first step");
  SDB_REQUIRE(mode != SDB_CHEB_DIRECT || v0 != nullptr || k == 0, "direct mode needs v0");
  SDB_REQUIRE(d != 0.0, "spectral halfwidth must be non-zero");
  DeviceGuard dg(m->device);
  if (!dg.ok) return fail(SDB_ECUDA, "cannot select CUDA device %d", m->device);
  StepPlan P;
  if ((rc = plan_steps(m, n_vec, mode, c, d, &P))) return rc;
  ZmPlan zp;
  if ((rc = zm_plan_range(m, P.g.ldv, mode, z_lo, z_hi, &zp))) return rc;
  SDB_REQUIRE(zp.on, "no z-march plan for planes [%lld, %lld) of this matrix", (long long)z_lo, (long long)z_hi);
  StepArgs a = P.a;
  a.legendre = legendre;
  a.partials = partials;
  a.v0 = v0 ? v0 : x;
  a.x = x;
  a.prev = prev;
  a.next = next;
  a.halo_lo = halo_lo;
  a.halo_hi = halo_hi;
  a.slot0 = (k == 0) ? 0 : -1;
  set_step_scalars(a, k);
  if (mode == SDB_CHEB_DOUBLING) {
    a.slotB = (2 * k + 1 <= degree) ? (int)(2 * k + 1) : -1;
    a.slotA = (2 * k + 2 <= degree) ? (int)(2 * k + 2) : -1;
  } else {
    a.slotA = (int)(k + 1);
    a.slotB = -1;
  }
  return zm_launch_step(m, zp, a, k == 0, mode, (cudaStream_t)stream);
}

int sdb_cheb_reduce_planes(const sdb_matrix* m, int64_t n_vec, int64_t degree, int mode, int64_t z_lo, int64_t z_hi,
                           const double* partials, double* zeta_pp, void* stream) {
  int leg_;
  mode = split_mode(mode, &leg_);
  SDB_REQUIRE(m && partials && zeta_pp, "NULL argument");
  SDB_REQUIRE(n_vec >= 1 && n_vec <= SDB_MAX_BATCH && degree >= 0, "bad shape");
  DeviceGuard dg(m->device);
  if (!dg.ok) return fail(SDB_ECUDA, "cannot select CUDA device %d", m->device);
  StepPlan P;
  int rc = plan_steps(m, n_vec, mode, 0.0, 1.0, &P);
  if (rc) return rc;
  ZmPlan zp;
  if ((rc = zm_plan_range(m, P.g.ldv, mode, z_lo, z_hi, &zp))) return rc;
  SDB_REQUIRE(zp.on, "no z-march plan for planes [%lld, %lld) of this matrix", (long long)z_lo, (long long)z_hi);
  P.a.nblocks = zp.nbp;
  return launch_reduce(P, n_vec, degree, mode, partials, zeta_pp, (cudaStream_t)stream);
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
