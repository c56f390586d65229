// rowgroup.cuh — the row-group thread mapping shared by the block kernels.
//
// A probe block is n x ldv fp64, row-major.  A "row group" is L lanes of one
// warp (L a power of two <= 32) that together hold one row: lane q owns the
// double2 columns 2*(q + v*L), v < VPL, so every load of a row is one
// coalesced run of 16*L bytes per v.  32/L rows share a warp.
#pragma once
#include "common.cuh"

namespace sdb {

constexpr int kRowThreads = 256;
constexpr int kRowWarps = kRowThreads / 32;

// ---- phased-panel row schedule ------------------------------------------------
// Block b processes, in phase t, the panel of P consecutive rows starting at
// (t*B + b)*P.  At any moment the whole grid works on one contiguous window
// of B*P rows, so the far neighbours of a row (e.g. +-nx*ny on a 3-D grid)
// are touched by other blocks within a short time and hit in L2, while the
// near neighbours (+-1, +-nx) are re-read from the block's own L1.  The
// schedule depends only on (n, B, P): the reduction tree is fixed.
struct PanelSched {
  int64_t n;
  int64_t nblocks;
  int64_t panel;
};

// Iterate the rows of this block: calls f(base) for every block iteration
// whose first row is base (rows base .. base+RPB-1, clipped to [.., pend)).
template <int RPB, class F>
__device__ __forceinline__ void for_each_panel_chunk(const PanelSched& s, F&& f) {
  for (int64_t ph = 0;; ++ph) {
    const int64_t p0 = (ph * s.nblocks + blockIdx.x) * s.panel;
    if (p0 >= s.n) break;
    const int64_t p1 = p0 + s.panel < s.n ? p0 + s.panel : s.n;
    for (int64_t base = p0; base < p1; base += RPB) f(base, p1);
  }
}

// Cache-policy helpers: data streamed once per pass (w_{k-1} reads, w_{k+1}
// writes) is marked evict-first in L2 so it does not push out the gathered
// x rows that other blocks are about to reuse.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_d2_once(const double* ptr, uint64_t pol) {
  double2 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y)
               : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_d2_once(double* ptr, double2 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(ptr), "d"(v.x),
               "d"(v.y), "l"(pol)
               : "memory");
}

// Sum per-thread column accumulators over every row the block touched and
// write one partial row (ldv doubles) at partials[(slot*nblocks + block)*ldv].
// Lanes sharing q hold the same columns: xor-shuffle them together, then add
// the warps in warp order through shared memory (fixed order, deterministic).
// Must be called by every thread of the block.
template <int L, int VPL>
__device__ __forceinline__ void block_partial(double2 (&acc)[VPL], double* smem, double* partials, int64_t slot,
                                              int64_t nblocks, int64_t ldv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, q = lane % L;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
#pragma unroll
    for (int off = L; off < 32; off <<= 1) {
      acc[v].x += __shfl_xor_sync(0xffffffffu, acc[v].x, off);
      acc[v].y += __shfl_xor_sync(0xffffffffu, acc[v].y, off);
    }
  }
  if (lane < L) {
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      int col = 2 * (q + v * L);
      smem[warp * ldv + col] = acc[v].x;
      smem[warp * ldv + col + 1] = acc[v].y;
    }
  }
  __syncthreads();
  for (int col = threadIdx.x; col < ldv; col += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kRowWarps; ++w) s += smem[w * ldv + col];
    partials[(slot * nblocks + blockIdx.x) * ldv + col] = s;
  }
  __syncthreads();
}

// Same, for a block that owns columns [col0, col0 + ncols) of row `bidx`.
template <int L, int VPL>
__device__ __forceinline__ void block_partial_cols(double2 (&acc)[VPL], double* smem, double* partials, int64_t slot,
                                                   int64_t nblocks, int64_t ldv, int64_t bidx, int col0, int ncols) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, q = lane % L;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
#pragma unroll
    for (int off = L; off < 32; off <<= 1) {
      acc[v].x += __shfl_xor_sync(0xffffffffu, acc[v].x, off);
      acc[v].y += __shfl_xor_sync(0xffffffffu, acc[v].y, off);
    }
  }
  if (lane < L) {
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      int col = 2 * (q + v * L);
      smem[warp * ncols + col] = acc[v].x;
      smem[warp * ncols + col + 1] = acc[v].y;
    }
  }
  __syncthreads();
  for (int col = threadIdx.x; col < ncols; col += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kRowWarps; ++w) s += smem[w * ncols + col];
    partials[(slot * nblocks + bidx) * ldv + col0 + col] = s;
  }
  __syncthreads();
}

// Sum one partial slot over blocks in block order.
__device__ __forceinline__ double sum_blocks(const double* __restrict__ partials, int64_t slot, int64_t nblocks,
                                             int64_t ldv, int64_t l) {
  const double* p = partials + slot * nblocks * ldv + l;
  double s = 0.0;
  for (int64_t b = 0; b < nblocks; ++b) s += p[b * ldv];
  return s;
}

// ---- matrix views: y[row] = sum_k a_{row,k} x[k] for the lane's columns ------
// CSR: the row's entries are summed in storage order (SciPy csr_matvec order,
// matrix.py:101-102).  The L lanes of a row group load up to L (col, value)
// pairs cooperatively and broadcast them with shuffles; U gathers per lane
// are issued before they are consumed.  Every lane of the warp must call
// this (rows past the end pass valid = false).
struct CsrView {
  const int32_t* __restrict__ rowptr;
  const int32_t* __restrict__ colidx;
  const double* __restrict__ vals;
};

template <int L, int VPL>
__device__ __forceinline__ void spmv_row(const CsrView& A, int64_t row, bool valid, int safe,
                                         const double* __restrict__ x, int64_t ldv, int q, double2 (&y)[VPL]) {
  constexpr int U = L < 4 ? L : (VPL >= 3 ? 2 : 4);
  const int beg = valid ? A.rowptr[row] : 0;
  const int cnt = valid ? A.rowptr[row + 1] - beg : 0;
  const int maxcnt = __reduce_max_sync(0xffffffffu, cnt);
#pragma unroll
  for (int v = 0; v < VPL; ++v) y[v] = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < maxcnt; k0 += L) {
    const int kk = k0 + q;
    int col = safe;
    double av = 0.0;
    if (kk < cnt) {
      col = __ldg(A.colidx + beg + kk);
      av = __ldg(A.vals + beg + kk);
    }
    const int nloc = min(L, maxcnt - k0);
    for (int t0 = 0; t0 < nloc; t0 += U) {
      int ct[U];
      double at[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ct[u] = __shfl_sync(0xffffffffu, col, t0 + u, L);
        at[u] = __shfl_sync(0xffffffffu, av, t0 + u, L);
      }
      double2 xv[U][VPL];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double* xr = x + (int64_t)ct[u] * ldv + 2 * q;
#pragma unroll
        for (int v = 0; v < VPL; ++v) xv[u][v] = ld_d2(xr + 2 * L * v);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          y[v].x = fma(at[u], xv[u][v].x, y[v].x);
          y[v].y = fma(at[u], xv[u][v].y, y[v].y);
        }
      }
    }
  }
}

// Periodic constant-coefficient stencil, (A x)_p = diag[p] x_p + sum_o w_o x_{p+o}
// on an nx*ny*nz torus (nx fastest).  Terms are summed in the order of the
// column index each offset produces for an interior point, the diagonal at
// its sorted place -- the storage order the CSR form of the same operator
// would have away from the periodic wrap.
struct StencilView {
  int nx, ny, nz;
  int nterms;          // off-centre points + 1
  int center_pos;      // index of the diagonal term
  int mx, my, mz;      // does any offset move along x / y / z
  int zghost;          // z-slab: no z wrap (ghost planes next to the slab)
  const int4* term;    // (dx, dy, dz, interior column delta), device, nterms
  const double* tw;    // term weights (the diagonal's comes from diag[])
  const double* diag;
  double wc[27];       // the same weights by value: compile-time indexed by the
                       // grid kernels, read straight from the constant bank
};

template <int L, int VPL>
__device__ __forceinline__ void spmv_row(const StencilView& S, int64_t row, bool valid, int safe,
                                         const double* __restrict__ x, int64_t ldv, int q, double2 (&y)[VPL]) {
#pragma unroll
  for (int v = 0; v < VPL; ++v) y[v] = make_double2(0.0, 0.0);
  if (!valid) return;
  const int r32 = (int)row;
  const int ix = r32 % S.nx, t = r32 / S.nx;
  const int iy = t % S.ny, iz = t / S.ny;
  const double dg = __ldg(S.diag + row);
  for (int o = 0; o < S.nterms; ++o) {
    const int4 tm = __ldg(S.term + o);
    int jx = ix + tm.x, jy = iy + tm.y, jz = iz + tm.z;
    jx = jx < 0 ? jx + S.nx : (jx >= S.nx ? jx - S.nx : jx);
    jy = jy < 0 ? jy + S.ny : (jy >= S.ny ? jy - S.ny : jy);
    if (!S.zghost) jz = jz < 0 ? jz + S.nz : (jz >= S.nz ? jz - S.nz : jz);
    const int64_t col = ((int64_t)jz * S.ny + jy) * S.nx + jx;
    const double wt = (o == S.center_pos) ? dg : __ldg(S.tw + o);
    const double* xr = x + col * ldv + 2 * q;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      double2 xv = ld_d2(xr + 2 * L * v);
      y[v].x = fma(wt, xv.x, y[v].x);
      y[v].y = fma(wt, xv.y, y[v].y);
    }
  }
}

// 7-point-face / 27-point-box grids with compile-time term order
// (lexicographic in (dz, dy, dx) = sorted-column order) and weights in the
// kernel-parameter constant bank.
template <int SHAPE>
struct GridView {
  int nx, ny, nz, zghost;
  const double* diag;
  double wc[27];
};

template <int SHAPE>
struct GridTerms;
template <>
struct GridTerms<SDB_SHAPE_FACE7> {
  static constexpr int NT = 7;
  __host__ __device__ static constexpr int dx(int o) { return o == 2 ? -1 : (o == 4 ? 1 : 0); }
  __host__ __device__ static constexpr int dy(int o) { return o == 1 ? -1 : (o == 5 ? 1 : 0); }
  __host__ __device__ static constexpr int dz(int o) { return o == 0 ? -1 : (o == 6 ? 1 : 0); }
};
template <>
struct GridTerms<SDB_SHAPE_BOX27> {
  static constexpr int NT = 27;
  __host__ __device__ static constexpr int dx(int o) { return o % 3 - 1; }
  __host__ __device__ static constexpr int dy(int o) { return (o / 3) % 3 - 1; }
  __host__ __device__ static constexpr int dz(int o) { return o / 9 - 1; }
};

template <int L, int VPL, int SHAPE>
__device__ __forceinline__ void spmv_row(const GridView<SHAPE>& S, int64_t row, bool valid, int safe,
                                         const double* __restrict__ x, int64_t ldv, int q, double2 (&y)[VPL]) {
  using G = GridTerms<SHAPE>;
#pragma unroll
  for (int v = 0; v < VPL; ++v) y[v] = make_double2(0.0, 0.0);
  if (!valid) return;
  const int nx = S.nx, ny = S.ny, nz = S.nz, nxy = nx * ny;
  const int r32 = (int)row;
  const int ix = r32 % nx, t = r32 / nx;
  const int iy = t % ny, iz = t / ny;
  const int xm = ix == 0 ? nx - 1 : -1, xp = ix == nx - 1 ? 1 - nx : 1;
  const int ym = iy == 0 ? (ny - 1) * nx : -nx, yp = iy == ny - 1 ? (1 - ny) * nx : nx;
  const int zm = (iz == 0 && !S.zghost) ? (nz - 1) * nxy : -nxy;
  const int zp = (iz == nz - 1 && !S.zghost) ? (1 - nz) * nxy : nxy;
  const double dg = __ldg(S.diag + row);
  constexpr int U = VPL == 1 ? 4 : 2;
#pragma unroll
  for (int o0 = 0; o0 < G::NT; o0 += U) {
    double2 xv[U][VPL];
    double w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int o = o0 + u;
      int col = r32;
      w[u] = 0.0;
      if (o < G::NT) {
        col = r32 + (G::dx(o) < 0 ? xm : (G::dx(o) > 0 ? xp : 0)) + (G::dy(o) < 0 ? ym : (G::dy(o) > 0 ? yp : 0)) +
              (G::dz(o) < 0 ? zm : (G::dz(o) > 0 ? zp : 0));
        w[u] = (G::dx(o) == 0 && G::dy(o) == 0 && G::dz(o) == 0) ? dg : S.wc[o];
      }
      const double* xr = x + (int64_t)col * ldv + 2 * q;
#pragma unroll
      for (int v = 0; v < VPL; ++v) xv[u][v] = ld_d2(xr + 2 * L * v);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        y[v].x = fma(w[u], xv[u][v].x, y[v].x);
        y[v].y = fma(w[u], xv[u][v].y, y[v].y);
      }
  }
}

template <int SHAPE>
inline GridView<SHAPE> make_grid_view(const sdb_matrix* m) {
  GridView<SHAPE> g{};
  g.nx = (int)m->st.nx;
  g.ny = (int)m->st.ny;
  g.nz = (int)m->st.nz;
  g.zghost = m->zghost;
  g.diag = m->diag;
  for (int o = 0; o < 27; ++o) g.wc[o] = o < m->nterms ? m->term_w_host[o] : 0.0;
  return g;
}

inline StencilView make_stencil_view(const sdb_matrix* m) {
  StencilView s{};
  s.nx = (int)m->st.nx;
  s.ny = (int)m->st.ny;
  s.nz = (int)m->st.nz;
  s.nterms = m->nterms;
  s.center_pos = m->center_pos;
  s.mx = m->mx;
  s.my = m->my;
  s.mz = m->mz;
  s.zghost = m->zghost;
  s.term = m->terms;
  s.tw = m->term_w;
  s.diag = m->diag;
  for (int o = 0; o < 27; ++o) s.wc[o] = o < m->nterms ? m->term_w_host[o] : 0.0;
  return s;
}

inline CsrView make_csr_view(const sdb_matrix* m) { return CsrView{m->rowptr, m->colidx, m->values}; }

// Instantiate F<L, VPL> for the runtime geometry.
#define SDB_GEOMETRY_DISPATCH(g, CASE)                                                                  \
  do {                                                                                                  \
    switch ((g).L * 8 + (g).VPL) {                                                                      \
      case 32 * 8 + 1: CASE(32, 1); break;                                                              \
      case 32 * 8 + 2: CASE(32, 2); break;                                                              \
      case 32 * 8 + 3: CASE(32, 3); break;                                                              \
      case 32 * 8 + 4: CASE(32, 4); break;                                                              \
      case 16 * 8 + 1: CASE(16, 1); break;                                                              \
      case 16 * 8 + 2: CASE(16, 2); break;                                                              \
      case 16 * 8 + 3: CASE(16, 3); break;                                                              \
      case 16 * 8 + 4: CASE(16, 4); break;                                                              \
      case 8 * 8 + 1: CASE(8, 1); break;                                                                \
      case 8 * 8 + 2: CASE(8, 2); break;                                                                \
      case 8 * 8 + 3: CASE(8, 3); break;                                                                \
      case 8 * 8 + 4: CASE(8, 4); break;                                                                \
      case 4 * 8 + 1: CASE(4, 1); break;                                                                \
      case 4 * 8 + 2: CASE(4, 2); break;                                                                \
      case 4 * 8 + 3: CASE(4, 3); break;                                                                \
      case 4 * 8 + 4: CASE(4, 4); break;                                                                \
      case 2 * 8 + 1: CASE(2, 1); break;                                                                \
      case 2 * 8 + 2: CASE(2, 2); break;                                                                \
      case 2 * 8 + 3: CASE(2, 3); break;                                                                \
      case 2 * 8 + 4: CASE(2, 4); break;                                                                \
      case 1 * 8 + 1: CASE(1, 1); break;                                                                \
      case 1 * 8 + 2: CASE(1, 2); break;                                                                \
      case 1 * 8 + 3: CASE(1, 3); break;                                                                \
      case 1 * 8 + 4: CASE(1, 4); break;                                                                \
      default: return fail(SDB_EUNSUPPORTED, "no kernel for row geometry L=%d VPL=%d", (g).L, (g).VPL); \
    }                                                                                                   \
  } while (0)

}  // namespace sdb
