// lanczos.cu — batched lock-step Lanczos with full reorthogonalisation.
//
// Reference: lanczos_factorize (lanczos.py:67-131), one probe at a time:
//   basis[:,0] = v0/||v0||
//   for j: w = A v_j - beta_{j-1} v_{j-1};  alpha_j = v_j . w;  w -= alpha_j v_j
//          full: 2x  w -= V (V^T w)          (classical Gram-Schmidt, twice)
//          selective: h = V^T w; w -= V[:, |h| > sqrt(eps)||w||] h[...]
//          beta_j = ||w||; non-finite -> NumericalFailure; breakdown if
//          beta_j <= 1e-13 max(tscale, 1) -> truncate; v_{j+1} = w / beta_j
// Here all probes of a batch run the same step together on an n x ldv block.
// Each probe keeps its own basis V_l (the basis is stored step-major,
// basis[t][i][l]), so the CGS projections are batched GEMVs, not a GEMM: no
// operand is shared across probes, and the passes are HBM-bound.  Per step:
//   K4  lz_spmm    w = A v_j - beta v_{j-1}, v_j = w_prev/beta written to the
//                  basis on the fly, alpha partials
//   K5a lz_proj    h = V_{0..j}^T w (one warp per basis vector t streaming its
//                  rows; the first projection also applies w -= alpha v_j)
//   K5b lz_update  w -= V_{0..j} h, optional ||w||^2 partials
//   K5c lz_update_proj  full reorth: pass 1's update and pass 2's projection
//                  in one basis read (3 basis passes per step instead of 4)
//   two-pass full reorth (default for n >= 16384, steps <= n / 64): lz_proj also yields the
//                  Gram column V^T v_j; h = 2 h1 - G h1 (lz_gram_correct)
//                  stands in for the second projection, one lz_update follows
//                  (2 basis passes per step; see lz_gram_correct)
// and small fixed-order reduce kernels between them (deterministic).  A probe
// that breaks down is frozen (1/beta = 0) while the others continue.
#include <cmath>

#include "rowgroup.cuh"

namespace sdb {

constexpr int kProjWarps = 8;
#ifndef SDB_PROJ_UNROLL
#define SDB_PROJ_UNROLL 2
#endif
constexpr int kProjUnroll = SDB_PROJ_UNROLL;  // rows in flight per warp in lz_proj
#ifndef SDB_UPD_TU
#define SDB_UPD_TU 4
#endif
constexpr int kUpdTU = SDB_UPD_TU;  // basis vectors per load batch in lz_update

struct LzState {       // per-probe device state, each an ldv-long array
  double* inv_beta;    // 1/beta_{j-1} (0 once frozen)
  double* beta_prev;   // beta_{j-1}
  double* tscale;      // max |alpha|, beta seen so far (lanczos.py:114)
  double* alpha_cur;   // alpha_j
};

// Column sums of a [slot][nblocks][ldv] partials array, block-parallel in a
// fixed order: the block is 32 columns x SEGS segments; segment k sums rows
// k, k+SEGS, ... in order, then segment 0 adds the SEGS segment sums in order.
// Deterministic (the same tree every launch).  The serial per-column loop it
// replaces left ~ldv threads walking nblocks rows each (the reduce kernels ran
// at a few hundred GB/s on 28 MB of partials late in a 100-step run).
// Every thread of the block must call it; the result is valid for seg == 0.
template <int SEGS>
__device__ __forceinline__ double block_col_sum(const double* __restrict__ partials, int64_t slot, int64_t nblocks,
                                                int64_t ldv, int64_t l) {
  __shared__ double red[SEGS][32];
  const int lane = threadIdx.x & 31, seg = threadIdx.x >> 5;
  double s = 0.0;
  if (l < ldv) {
    const double* p = partials + slot * nblocks * ldv + l;
#pragma unroll 4
    for (int64_t b = seg; b < nblocks; b += SEGS) s += p[b * ldv];
  }
  red[seg][lane] = s;
  __syncthreads();
  double tot = 0.0;
  if (seg == 0) {
#pragma unroll
    for (int k = 0; k < SEGS; ++k) tot += red[k][lane];
  }
  __syncthreads();
  return tot;
}
constexpr int kRedSegs = 16;

// ---- start: ||v0|| --------------------------------------------------------------
template <int L, int VPL>
__global__ void __launch_bounds__(kRowThreads) lz_start_norm(const double* __restrict__ v0, int64_t n, int64_t ldv,
                                                             int64_t nblocks, int64_t panel, double* partials) {
  constexpr int RPW = 32 / L, RPB = RPW * kRowWarps;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane / L, q = lane % L;
  double2 acc[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) acc[v] = make_double2(0.0, 0.0);
  for_each_panel_chunk<RPB>(PanelSched{n, nblocks, panel}, [&](int64_t base, int64_t pend) {
    const int64_t row = base + warp * RPW + g;
    if (row < pend) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        double2 p = ld_d2(v0 + row * ldv + 2 * q + 2 * L * v);
        acc[v].x += p.x * p.x;
        acc[v].y += p.y * p.y;
      }
    }
  });
  __shared__ double smem[kRowWarps * SDB_MAX_BATCH];
  block_partial<L, VPL>(acc, smem, partials, 0, nblocks, ldv);
}

__global__ void lz_start_reduce(const double* __restrict__ partials, int64_t nblocks, int64_t ldv, int64_t n_vec,
                                LzState st, int32_t* __restrict__ steps_done, int32_t* __restrict__ status) {
  const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (l >= ldv) return;
  const double nrm = sqrt(sum_blocks(partials, 0, nblocks, ldv, l));
  const bool live = l < n_vec && nrm != 0.0 && isfinite(nrm);
  st.inv_beta[l] = live ? 1.0 / nrm : 0.0;
  st.beta_prev[l] = 0.0;
  st.tscale[l] = 0.0;
  st.alpha_cur[l] = 0.0;
  if (l < n_vec) {
    steps_done[l] = 0;
    status[l] = (nrm == 0.0) ? SDB_LZ_ZERO_START : (isfinite(nrm) ? SDB_LZ_OK : SDB_LZ_NONFINITE);
  }
}

// ---- K4: w = A v_j - beta_{j-1} v_{j-1}, v_j = w_prev * inv_beta, alpha partials ----
#ifndef SDB_SPMM_MINB
#define SDB_SPMM_MINB 4
#endif
template <class View, int L, int VPL>
__global__ void __launch_bounds__(kRowThreads, VPL <= 2 ? SDB_SPMM_MINB : 2)
    lz_spmm(View A, const double* __restrict__ wprev, const double* __restrict__ vprev, double* __restrict__ vj,
            double* __restrict__ wout, LzState st, int first, double c, double inv_d, int64_t n, int64_t ldv,
            int64_t nblocks, int64_t panel, double* partials) {
  constexpr int RPW = 32 / L, RPB = RPW * kRowWarps;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane / L, q = lane % L;
  double2 ib[VPL], bp[VPL], acc[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    ib[v] = ld_d2(st.inv_beta + 2 * q + 2 * L * v);
    bp[v] = ld_d2(st.beta_prev + 2 * q + 2 * L * v);
    acc[v] = make_double2(0.0, 0.0);
  }
  for_each_panel_chunk<RPB>(PanelSched{n, nblocks, panel}, [&](int64_t base, int64_t pend) {
    const int64_t row = base + warp * RPW + g;
    const bool valid = row < pend;
    double2 y[VPL];
    spmv_row<L, VPL>(A, row, valid, valid ? (int)row : (int)base, wprev, ldv, q, y);
    if (valid) {
      const int64_t o = row * ldv + 2 * q;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int off = 2 * L * v;
        double2 wp = ld_d2(wprev + o + off);
        double2 vv = make_double2(wp.x * ib[v].x, wp.y * ib[v].y);  // v_j = w / beta
        st_d2(vj + o + off, vv);
        // (A v_j - c v_j)/d  (the MappedOperator form, matrix.py:126)
        double2 w = make_double2((y[v].x * ib[v].x - c * vv.x) * inv_d, (y[v].y * ib[v].y - c * vv.y) * inv_d);
        if (!first) {
          double2 pv = ld_d2(vprev + o + off);
          w.x -= bp[v].x * pv.x;
          w.y -= bp[v].y * pv.y;
        }
        st_d2(wout + o + off, w);
        acc[v].x += vv.x * w.x;
        acc[v].y += vv.y * w.y;
      }
    }
  });
  __shared__ double smem[kRowWarps * SDB_MAX_BATCH];
  block_partial<L, VPL>(acc, smem, partials, 0, nblocks, ldv);
}

__global__ void lz_alpha_reduce(const double* __restrict__ partials, int64_t nblocks, int64_t ldv, int64_t n_vec,
                                int64_t j, int64_t steps, LzState st, double* __restrict__ alpha,
                                const int32_t* __restrict__ status) {
  const int64_t l = blockIdx.x * 32 + (threadIdx.x & 31);
  const double a = block_col_sum<kRedSegs>(partials, 0, nblocks, ldv, l);
  if ((threadIdx.x >> 5) != 0 || l >= ldv) return;
  const bool live = l < n_vec && status[l] == SDB_LZ_OK;
  st.alpha_cur[l] = live ? a : 0.0;
  if (live) alpha[l * steps + j] = a;
}

// ---- K5a: h[t] = V_t^T w for t <= j  (one warp per basis vector) ----------------
// Block (t-chunk, row block).  Warp w handles t = chunk*8 + w and streams the
// contiguous rows V[t][rs..re) of its row block; the w rows are shared by the
// block's warps through L1.  When SUB_ALPHA, w' = w - alpha v_j is formed on
// the fly and the warp handling t == 0 stores it to wdst (a different
// buffer, so concurrent blocks never see a half-updated w).  NORM adds
// ||w'||^2 partials (selective mode) at slot norm_slot.
// GRAM (two-pass schedule, see lz_gram_correct): the same basis read also
// yields column j of the Gram matrix, g[t] = V_t^T v_j, at slot norm_slot + t.
template <int NV, bool SUB_ALPHA, bool NORM, bool GRAM = false>
__global__ void __launch_bounds__(kProjWarps * 32)
    lz_proj(const double* __restrict__ basis, const double* __restrict__ wsrc, double* __restrict__ wdst, LzState st,
            int64_t j, int64_t n, int64_t ldv, int64_t nrb, double* partials, int64_t norm_slot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tchunk = blockIdx.x, rb = blockIdx.y;
  const int64_t t = tchunk * kProjWarps + warp;
  const int64_t rs = n * rb / nrb, re = n * (rb + 1) / nrb;
  const size_t plane = (size_t)n * ldv;
  const double* vt = basis + (size_t)t * plane;
  const double* vj = basis + (size_t)j * plane;
  static_assert(!(GRAM && (SUB_ALPHA || NORM)), "the Gram column rides on the plain projection");
  double2 acc[NV], nacc[NV], al[NV];
  bool colok[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int64_t col = 2 * (lane + 32 * v);
    colok[v] = col < ldv;
    acc[v] = nacc[v] = make_double2(0.0, 0.0);  // nacc: ||w'||^2 (NORM) or the Gram column (GRAM)
    al[v] = (SUB_ALPHA && colok[v]) ? ld_d2(st.alpha_cur + col) : make_double2(0.0, 0.0);
  }
  const bool active = t <= j;
  const bool storer = SUB_ALPHA && tchunk == 0 && warp == 0;
  if (active) {
#pragma unroll kProjUnroll
    for (int64_t i = rs; i < re; ++i) {
      const int64_t o = i * ldv + 2 * lane;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if (!colok[v]) continue;
        double2 w = ld_d2(wsrc + o + 64 * v);
        if (SUB_ALPHA) {
          double2 p = ld_d2(vj + o + 64 * v);
          w.x -= al[v].x * p.x;
          w.y -= al[v].y * p.y;
          if (storer) st_d2(wdst + o + 64 * v, w);
          if (NORM && storer) {
            nacc[v].x += w.x * w.x;
            nacc[v].y += w.y * w.y;
          }
        }
        double2 b = ld_d2_stream(vt + o + 64 * v);
        acc[v].x += b.x * w.x;
        acc[v].y += b.y * w.y;
        if (GRAM) {
          const double2 p = ld_d2(vj + o + 64 * v);
          nacc[v].x += b.x * p.x;
          nacc[v].y += b.y * p.y;
        }
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!colok[v]) continue;
      const int64_t col = 2 * (lane + 32 * v);
      double* p = partials + ((size_t)t * nrb + rb) * ldv + col;
      p[0] = acc[v].x;
      p[1] = acc[v].y;
      if (GRAM) {
        double* gp = partials + ((size_t)(norm_slot + t) * nrb + rb) * ldv + col;
        gp[0] = nacc[v].x;
        gp[1] = nacc[v].y;
      }
    }
  }
  if (NORM && storer) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!colok[v]) continue;
      const int64_t col = 2 * (lane + 32 * v);
      double* p = partials + ((size_t)norm_slot * nrb + rb) * ldv + col;
      p[0] = nacc[v].x;
      p[1] = nacc[v].y;
    }
  }
}

// h[t][l] = sum over row blocks (t <= j).  Selective mode keeps only the
// overlaps above sqrt(eps) ||w|| (lanczos.py:107-110).
__global__ void lz_h_reduce(const double* __restrict__ partials, int64_t nrb, int64_t ldv, int64_t j,
                            double* __restrict__ h, int selective, int64_t norm_slot) {
  // grid (t, column chunk of 32); see block_col_sum
  const int64_t t = blockIdx.x, l = blockIdx.y * 32 + (threadIdx.x & 31);
  double v = block_col_sum<kRedSegs>(partials, t, nrb, ldv, l);
  if (selective) {
    const double wn = sqrt(block_col_sum<kRedSegs>(partials, norm_slot, nrb, ldv, l));
    if (!(fabs(v) > 1.4901161193847656e-08 * wn)) v = 0.0;
  }
  if ((threadIdx.x >> 5) == 0 && l < ldv) h[t * ldv + l] = v;
}

// ---- two-pass full reorthogonalisation (Gram-corrected CGS2) ---------------------------
// CGS twice is w'' = (I - V V^T)(I - V V^T) w = w - V (2 h1 - G h1) with
// h1 = V^T w and G = V^T V: the second projection h2 = V^T (w - V h1) equals
// (I - G) h1, so with the Gram matrix of the basis at hand the second basis
// read is not needed -- one projection pass (which also yields the new Gram
// column V^T v_j) and one update pass per step instead of three passes.  This
// is the low-synchronisation CGS2 projector I - V T V^T with T = 2I - G
// ~ (V^T V)^{-1}; what it leaves out is the rounding error of the first update
// projected on V (O(eps)), so the basis stays orthogonal to ~1e-14 instead of
// ~1e-15 and alpha, beta agree with the three-pass schedule to ~1e-13
// relative (measured; tests/test_gpu_lanczos.py), far inside the 1e-10 bar.
// G is kept per probe as [t][s][ldv], t, s < gdim.
__global__ void lz_g_reduce(const double* __restrict__ partials, int64_t slot0, int64_t nrb, int64_t ldv, int64_t j,
                            int64_t gdim, double* __restrict__ G) {
  const int64_t t = blockIdx.x, l = blockIdx.y * 32 + (threadIdx.x & 31);
  const double v = block_col_sum<kRedSegs>(partials, slot0 + t, nrb, ldv, l);
  if ((threadIdx.x >> 5) == 0 && l < ldv) {
    G[(t * gdim + j) * ldv + l] = v;
    G[(j * gdim + t) * ldv + l] = v;
  }
}

// hc[t] = 2 h1[t] - sum_{s <= j} G[t][s] h1[s]   (fixed-order segment sums)
__global__ void lz_gram_correct(const double* __restrict__ G, const double* __restrict__ h1, int64_t ldv, int64_t j,
                                int64_t gdim, double* __restrict__ hc) {
  __shared__ double red[kRedSegs][32];
  const int lane = threadIdx.x & 31, seg = threadIdx.x >> 5;
  const int64_t t = blockIdx.x, l = blockIdx.y * 32 + lane;
  double sum = 0.0;
  if (l < ldv)
    for (int64_t s = seg; s <= j; s += kRedSegs) sum = fma(G[(t * gdim + s) * ldv + l], h1[s * ldv + l], sum);
  red[seg][lane] = sum;
  __syncthreads();
  if (seg == 0 && l < ldv) {
    double tot = 0.0;
#pragma unroll
    for (int k = 0; k < kRedSegs; ++k) tot += red[k][lane];
    const double a = h1[t * ldv + l];
    hc[t * ldv + l] = a + (a - tot);
  }
}

// ---- K5b: w -= V h (row-local), optional ||w||^2 partials ---------------------------
#ifndef SDB_UPD_MINB
#define SDB_UPD_MINB 4
#endif
template <int L, int VPL, bool NORM>
__global__ void __launch_bounds__(kRowThreads, VPL <= 2 ? SDB_UPD_MINB : 2)
    lz_update(const double* __restrict__ basis, double* w, const double* __restrict__ h, int64_t j, int64_t n,
              int64_t ldv, int64_t nblocks, int64_t panel, double* partials) {
  constexpr int RPW = 32 / L, RPB = RPW * kRowWarps;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane / L, q = lane % L;
  const size_t plane = (size_t)n * ldv;
  double2 acc[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) acc[v] = make_double2(0.0, 0.0);
  for_each_panel_chunk<RPB>(PanelSched{n, nblocks, panel}, [&](int64_t base, int64_t pend) {
    const int64_t row = base + warp * RPW + g;
    if (row < pend) {
      const int64_t o = row * ldv + 2 * q;
      double2 s[VPL];
#pragma unroll
      for (int v = 0; v < VPL; ++v) s[v] = make_double2(0.0, 0.0);
      int64_t t = 0;
      for (; t + kUpdTU <= j + 1; t += kUpdTU) {
        double2 b[kUpdTU][VPL], hh[kUpdTU][VPL];
#pragma unroll
        for (int u = 0; u < kUpdTU; ++u)
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            b[u][v] = ld_d2_stream(basis + (size_t)(t + u) * plane + o + 2 * L * v);
            hh[u][v] = ld_d2(h + (t + u) * ldv + 2 * q + 2 * L * v);
          }
#pragma unroll
        for (int u = 0; u < kUpdTU; ++u)
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            s[v].x = fma(b[u][v].x, hh[u][v].x, s[v].x);
            s[v].y = fma(b[u][v].y, hh[u][v].y, s[v].y);
          }
      }
      for (; t <= j; ++t) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          double2 b = ld_d2_stream(basis + (size_t)t * plane + o + 2 * L * v);
          double2 hh = ld_d2(h + t * ldv + 2 * q + 2 * L * v);
          s[v].x = fma(b.x, hh.x, s[v].x);
          s[v].y = fma(b.y, hh.y, s[v].y);
        }
      }
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        double2* wp = reinterpret_cast<double2*>(w + o + 2 * L * v);
        double2 x = *wp;
        x.x -= s[v].x;
        x.y -= s[v].y;
        *wp = x;
        if (NORM) {
          acc[v].x += x.x * x.x;
          acc[v].y += x.y * x.y;
        }
      }
    }
  });
  if (NORM) {
    __shared__ double smem[kRowWarps * SDB_MAX_BATCH];
    block_partial<L, VPL>(acc, smem, partials, 0, nblocks, ldv);
  }
}

// ---- K5c: fused CGS2 middle pass: w -= V h1, then h2 partials = V^T w -------
// The classical schedule reads the basis four times per step (proj, update,
// proj, update).  The update of pass 1 and the projection of pass 2 touch the
// same basis entries V[t][i][:] for a row i, and the new w[i] depends only on
// row i, so one pass can do both: load V[t][i][cols] for every t <= j into
// registers, form s = sum_t V h1, w' = w - s (block reduce over t-groups),
// then accumulate h2[t] += V[t][i] w'[i] from the same registers.  The basis
// is read once instead of twice; the step reads it 3x in total.
// Block (row block rb, column slice cs): kZcs column pairs x kZtg t-groups;
// thread (c, tg) owns t = tg + kZtg*k, k < KMAX (KMAX*kZtg >= j+1) and keeps
// those h1 values and h2 accumulators in registers.  kZrows rows per
// iteration keep 2*KMAX independent 16-byte loads in flight per thread.
constexpr int kZcs = 16;

// Two resident blocks per SM up to KMAX = 8 (<= 128 registers; the KMAX = 8
// form spills 160 bytes but the doubled warps in flight win: C4 0.806 ->
// 0.789 s); KMAX = 16 (236 registers) keeps one.
#ifndef SDB_UPJ_MINB_SMALL
#define SDB_UPJ_MINB_SMALL 2
#endif
template <int KMAX, int kZrows, int kZtg>
__global__ void __launch_bounds__(kZcs * kZtg, KMAX >= 16 ? 1 : (KMAX <= 4 ? SDB_UPJ_MINB_SMALL : 2))
    lz_update_proj(const double* __restrict__ basis, const double* __restrict__ wsrc, double* __restrict__ w,
                   const double* __restrict__ h, int64_t j,
                   int64_t n, int64_t ldv, int64_t nrb, double* __restrict__ partials) {
  const int c = threadIdx.x % kZcs, tg = threadIdx.x / kZcs;
  const int64_t rb = blockIdx.y;  // column slices of the same rows run side by side
  const int64_t col = 2 * ((int64_t)blockIdx.x * kZcs + c);
  const bool colok = col < ldv;
  const int64_t rs = n * rb / nrb, re = n * (rb + 1) / nrb;
  const size_t plane = (size_t)n * ldv;
  extern __shared__ double2 h1s[];  // [KMAX * kZtg][kZcs]: this block's column slice of h1
  __shared__ double2 red[kZrows][kZtg][kZcs];
  __shared__ double2 wn[kZrows][kZcs];
  for (int idx = threadIdx.x; idx < KMAX * kZtg * kZcs; idx += blockDim.x) {
    const int64_t t = idx / kZcs, cc = 2 * ((int64_t)blockIdx.x * kZcs + idx % kZcs);
    h1s[idx] = (t <= j && cc < ldv) ? ld_d2(h + t * ldv + cc) : make_double2(0.0, 0.0);
  }
  double2 acc[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) acc[k] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int64_t r0 = rs; r0 < re; r0 += kZrows) {
    double2 v[kZrows][KMAX];
    double2 wv = make_double2(0.0, 0.0);
    const bool wown = tg < kZrows && colok && r0 + tg < re;
    if (wown) wv = ld_d2(wsrc + (r0 + tg) * ldv + col);  // in flight with the basis loads
#pragma unroll
    for (int r = 0; r < kZrows; ++r)
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        const int64_t t = tg + (int64_t)kZtg * k;
        v[r][k] = (colok && t <= j && r0 + r < re) ? ld_d2_stream(basis + (size_t)t * plane + (r0 + r) * ldv + col)
                                                    : make_double2(0.0, 0.0);
      }
#pragma unroll
    for (int r = 0; r < kZrows; ++r) {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        const double2 hh = h1s[(tg + kZtg * k) * kZcs + c];
        s.x = fma(v[r][k].x, hh.x, s.x);
        s.y = fma(v[r][k].y, hh.y, s.y);
      }
      red[r][tg][c] = s;
    }
    __syncthreads();
    if (tg < kZrows) {
      const int r = tg;
      double2 s = red[r][0][c];
#pragma unroll
      for (int g = 1; g < kZtg; ++g) {
        s.x += red[r][g][c].x;
        s.y += red[r][g][c].y;
      }
      wv.x -= s.x;
      wv.y -= s.y;
      if (wown) st_d2(w + (r0 + r) * ldv + col, wv);
      wn[r][c] = wv;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kZrows; ++r) {
      const double2 x = wn[r][c];
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        acc[k].x = fma(v[r][k].x, x.x, acc[k].x);
        acc[k].y = fma(v[r][k].y, x.y, acc[k].y);
      }
    }
  }
  if (!colok) return;
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    const int64_t t = tg + (int64_t)kZtg * k;
    if (t <= j) {
      double* p = partials + ((size_t)t * nrb + rb) * ldv + col;
      p[0] = acc[k].x;
      p[1] = acc[k].y;
    }
  }
}

// reorth = "none": w' = w - alpha v_j into wdst, ||w'||^2 partials.
template <int L, int VPL>
__global__ void __launch_bounds__(kRowThreads) lz_sub_alpha_norm(const double* __restrict__ vj,
                                                                 const double* __restrict__ wsrc,
                                                                 double* __restrict__ wdst, LzState st, int64_t n,
                                                                 int64_t ldv, int64_t nblocks, int64_t panel,
                                                                 double* partials) {
  constexpr int RPW = 32 / L, RPB = RPW * kRowWarps;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane / L, q = lane % L;
  double2 acc[VPL], al[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    acc[v] = make_double2(0.0, 0.0);
    al[v] = ld_d2(st.alpha_cur + 2 * q + 2 * L * v);
  }
  for_each_panel_chunk<RPB>(PanelSched{n, nblocks, panel}, [&](int64_t base, int64_t pend) {
    const int64_t row = base + warp * RPW + g;
    if (row < pend) {
      const int64_t o = row * ldv + 2 * q;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        double2 w = ld_d2(wsrc + o + 2 * L * v), p = ld_d2(vj + o + 2 * L * v);
        w.x -= al[v].x * p.x;
        w.y -= al[v].y * p.y;
        st_d2(wdst + o + 2 * L * v, w);
        acc[v].x += w.x * w.x;
        acc[v].y += w.y * w.y;
      }
    }
  });
  __shared__ double smem[kRowWarps * SDB_MAX_BATCH];
  block_partial<L, VPL>(acc, smem, partials, 0, nblocks, ldv);
}

// beta_j = ||w||, finiteness, breakdown and truncation logic (lanczos.py:111-128).
__global__ void lz_beta_reduce(const double* __restrict__ partials, int64_t nblocks, int64_t ldv, int64_t n_vec,
                               int64_t j, int64_t steps, LzState st, double* __restrict__ beta,
                               int32_t* __restrict__ steps_done, int32_t* __restrict__ status) {
  const int64_t l = blockIdx.x * 32 + (threadIdx.x & 31);
  const double b = sqrt(block_col_sum<kRedSegs>(partials, 0, nblocks, ldv, l));
  if ((threadIdx.x >> 5) != 0 || l >= ldv) return;
  if (l >= n_vec || status[l] != SDB_LZ_OK) {
    st.inv_beta[l] = 0.0;
    st.beta_prev[l] = 0.0;
    return;
  }
  const double a = st.alpha_cur[l];
  if (!(isfinite(a) && isfinite(b))) {
    status[l] = SDB_LZ_NONFINITE;
    steps_done[l] = (int32_t)(j + 1);
    st.inv_beta[l] = 0.0;
    st.beta_prev[l] = 0.0;
    return;
  }
  const double ts = fmax(st.tscale[l], fmax(fabs(a), b));
  st.tscale[l] = ts;
  if (j == steps - 1) {
    beta[l * steps + j] = b;  // beta_next
    steps_done[l] = (int32_t)steps;
    st.inv_beta[l] = 0.0;
    st.beta_prev[l] = b;
  } else if (b <= 1e-13 * fmax(ts, 1.0)) {
    beta[l * steps + j] = 0.0;  // truncated: beta_next = 0
    steps_done[l] = (int32_t)(j + 1);
    status[l] = SDB_LZ_BREAKDOWN;
    st.inv_beta[l] = 0.0;
    st.beta_prev[l] = 0.0;
  } else {
    beta[l * steps + j] = b;
    st.inv_beta[l] = 1.0 / b;
    st.beta_prev[l] = b;
  }
}

// ---- host driver ------------------------------------------------------------------------
static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// Two-pass (Gram-corrected) full reorthogonalisation covers steps j < gdim:
// default gdim = n / 64 for n >= kGramMinRows (the run stays far from
// exhausting the space, so the dimension-exhaustion breakdowns of small
// matrices keep the three-pass schedule bit for bit; the rule depends on n and
// j only, so a shorter run stays an exact prefix of a longer one).  The Gram
// matrix is gdim^2 x ldv doubles, at most 1/64 of the basis.  SDB_LZ_GRAM=0 /
// 1 forces the schedule off / on for every step.
constexpr int64_t kGramMinRows = 16384;
static int64_t lz_gram_steps(int64_t n, int64_t steps) {
  const char* e = getenv("SDB_LZ_GRAM");
  if (e && e[0] == '0') return 0;
  if (e && e[0] == '1') return steps;
  if (n < kGramMinRows) return 0;
  return steps < n / 64 ? steps : n / 64;
}

struct LzLayout {
  size_t block, part, h, state, gram, total;
  int64_t gdim;
};

static LzLayout lz_layout(const sdb_matrix* m, int64_t ldv, int64_t steps) {
  LzLayout L;
  L.gdim = lz_gram_steps(m->n, steps);
  L.block = align256(sizeof(double) * (size_t)m->n * ldv);
  // slots 0..steps-1: projection partials, steps: ||w||^2, steps+1..: Gram column partials
  L.part = align256(sizeof(double) * (size_t)(steps + 1 + L.gdim) * row_blocks(m) * ldv);
  L.h = align256(sizeof(double) * (size_t)steps * ldv);  // two of these: h1 and the corrected h
  L.state = align256(sizeof(double) * 4 * (size_t)ldv);
  L.gram = align256(sizeof(double) * (size_t)L.gdim * L.gdim * ldv);
  L.total = 2 * L.block + L.part + 2 * L.h + L.state + L.gram;
  return L;
}

template <class View>
static int lz_launch_spmm(const View& A, const Geometry& g, const double* wprev, const double* vprev, double* vj,
                          double* wout, const LzState& st, int first, double c, double inv_d, int64_t n,
                          int64_t nblocks, int64_t panel, double* part, cudaStream_t s) {
#define SDB_LZ_CASE(LL, VV)                                                                                    \
  lz_spmm<View, LL, VV><<<(unsigned)nblocks, kRowThreads, 0, s>>>(A, wprev, vprev, vj, wout, st, first, c, inv_d, \
                                                                 n, g.ldv, nblocks, panel, part)
  SDB_GEOMETRY_DISPATCH(g, SDB_LZ_CASE);
#undef SDB_LZ_CASE
  return SDB_OK;
}

static int lz_launch_proj(int nv, bool sub_alpha, bool norm, const double* basis, const double* wsrc, double* wdst,
                          const LzState& st, int64_t j, int64_t n, int64_t ldv, int64_t nrb, double* part,
                          int64_t norm_slot, cudaStream_t s) {
  dim3 grid((unsigned)((j + 1 + kProjWarps - 1) / kProjWarps), (unsigned)nrb);
  dim3 block(kProjWarps * 32);
#define SDB_PROJ(NVV, SA, NO)                                                                             \
  if (nv == NVV && sub_alpha == SA && norm == NO) {                                                       \
    lz_proj<NVV, SA, NO><<<grid, block, 0, s>>>(basis, wsrc, wdst, st, j, n, ldv, nrb, part, norm_slot); \
    return SDB_OK;                                                                                        \
  }
#define SDB_PROJ_NV(NVV) SDB_PROJ(NVV, true, false) SDB_PROJ(NVV, false, false) SDB_PROJ(NVV, true, true)
  SDB_PROJ_NV(1) SDB_PROJ_NV(2) SDB_PROJ_NV(3) SDB_PROJ_NV(4)
#undef SDB_PROJ_NV
#undef SDB_PROJ
  return fail(SDB_EUNSUPPORTED, "no projection kernel for ldv=%lld", (long long)ldv);
}

static int lz_launch_proj_gram(int nv, const double* basis, const double* wsrc, const LzState& st, int64_t j, int64_t n,
                               int64_t ldv, int64_t nrb, double* part, int64_t gram_slot0, cudaStream_t s) {
  dim3 grid((unsigned)((j + 1 + kProjWarps - 1) / kProjWarps), (unsigned)nrb);
  dim3 block(kProjWarps * 32);
#define SDB_PROJ_G(NVV)                                                                                              \
  if (nv == NVV) {                                                                                                   \
    lz_proj<NVV, false, false, true><<<grid, block, 0, s>>>(basis, wsrc, nullptr, st, j, n, ldv, nrb, part, gram_slot0); \
    return SDB_OK;                                                                                                   \
  }
  SDB_PROJ_G(1) SDB_PROJ_G(2) SDB_PROJ_G(3) SDB_PROJ_G(4)
#undef SDB_PROJ_G
  return fail(SDB_EUNSUPPORTED, "no projection kernel for ldv=%lld", (long long)ldv);
}

static int lz_launch_update(const Geometry& g, bool norm, const double* basis, double* w, const double* h, int64_t j,
                            int64_t n, int64_t nblocks, int64_t panel, double* part, cudaStream_t s) {
  if (norm) {
#define SDB_UP_CASE(LL, VV) \
  lz_update<LL, VV, true><<<(unsigned)nblocks, kRowThreads, 0, s>>>(basis, w, h, j, n, g.ldv, nblocks, panel, part)
    SDB_GEOMETRY_DISPATCH(g, SDB_UP_CASE);
#undef SDB_UP_CASE
  } else {
#define SDB_UP_CASE(LL, VV) \
  lz_update<LL, VV, false><<<(unsigned)nblocks, kRowThreads, 0, s>>>(basis, w, h, j, n, g.ldv, nblocks, panel, part)
    SDB_GEOMETRY_DISPATCH(g, SDB_UP_CASE);
#undef SDB_UP_CASE
  }
  return SDB_OK;
}

// Fused middle pass when the per-thread t range fits the register budget.
template <int KM, int RW, int TG>
static void lz_upj_launch(dim3 grid, const double* basis, const double* wsrc, double* w, const double* h, int64_t j,
                          int64_t n,
                          int64_t ldv, int64_t nrb, double* part, cudaStream_t s) {
  const size_t smem = (size_t)KM * TG * kZcs * sizeof(double2);
  // function attributes are per device: set on every launch (cheap); a failure
  // surfaces through the launch check that follows
  if (smem > 48 * 1024)
    (void)cudaFuncSetAttribute(lz_update_proj<KM, RW, TG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  lz_update_proj<KM, RW, TG><<<grid, kZcs * TG, smem, s>>>(basis, wsrc, w, h, j, n, ldv, nrb, part);
}

static bool lz_launch_update_proj(const double* basis, const double* wsrc, double* w, const double* h, int64_t j,
                                  int64_t n, int64_t ldv,
                                  int64_t nrb, double* part, cudaStream_t s) {
  dim3 grid((unsigned)((ldv / 2 + kZcs - 1) / kZcs), (unsigned)nrb);
  const int64_t T = j + 1;
#define SDB_UPJ(KM, RW, TG)                                                  \
  if (T <= (int64_t)KM * TG) {                                               \
    lz_upj_launch<KM, RW, TG>(grid, basis, wsrc, w, h, j, n, ldv, nrb, part, s);  \
    return true;                                                             \
  }
  // two rows per iteration (measured best on C4: 16 t-groups x 2 rows beats
  // 1 row, 4 rows and 32 t-groups)
  SDB_UPJ(1, 2, 16) SDB_UPJ(2, 2, 16) SDB_UPJ(4, 2, 16) SDB_UPJ(8, 2, 16) SDB_UPJ(16, 1, 16)
#undef SDB_UPJ
  return false;
}

static bool lz_update_proj_fits(int64_t j) { return j + 1 <= 16LL * 16; }

static bool lz_fused_enabled() {
  const char* e = getenv("SDB_LZ_FUSED");
  return !(e && e[0] == '0');
}

}  // namespace sdb

using namespace sdb;

extern "C" {

int sdb_lanczos_workspace_size(const sdb_matrix* m, int64_t n_vec, int64_t steps, size_t* bytes) {
  SDB_REQUIRE(m && bytes, "NULL argument");
  SDB_REQUIRE(n_vec >= 1 && n_vec <= SDB_MAX_BATCH, "n_vec must lie in [1, %d] per batch", SDB_MAX_BATCH);
  SDB_REQUIRE(steps >= 1, "need at least one Lanczos step");
  *bytes = lz_layout(m, choose_geometry(n_vec).ldv, steps).total;
  return SDB_OK;
}

int sdb_lanczos(const sdb_matrix* m, double c, double d, int64_t n_vec, int64_t steps, int reorth, const double* v0, double* basis,
                double* alpha, double* beta, int32_t* steps_done, int32_t* status, void* workspace,
                size_t workspace_bytes, void* stream) {
  SDB_REQUIRE(m && v0 && basis && alpha && beta && steps_done && status, "NULL argument");
  SDB_REQUIRE(reorth == SDB_REORTH_FULL || reorth == SDB_REORTH_SELECTIVE || reorth == SDB_REORTH_NONE,
              "unknown reorth mode %d", reorth);
  SDB_REQUIRE(steps >= 1, "need at least one Lanczos step");
  SDB_REQUIRE(d != 0.0, "spectral halfwidth must be non-zero");
  SDB_REQUIRE(steps <= m->n, "steps=%lld exceeds matrix dimension %lld", (long long)steps, (long long)m->n);
  size_t need = 0;
  int rc = sdb_lanczos_workspace_size(m, n_vec, steps, &need);
  if (rc) return rc;
  SDB_REQUIRE(workspace && workspace_bytes >= need, "workspace too small (%zu < %zu bytes)", workspace_bytes, need);
  DeviceGuard dg(m->device);
  if (!dg.ok) return fail(SDB_ECUDA, "cannot select CUDA device %d", m->device);
  cudaStream_t s = (cudaStream_t)stream;

  const Geometry g = choose_geometry(n_vec);
  const int64_t ldv = g.ldv, n = m->n, nrb = row_blocks(m);
  const int nv = (int)((ldv + 63) / 64);
  const int64_t panel = panel_rows(m, ldv, (32 / g.L) * kRowWarps);
  const LzLayout lay = lz_layout(m, ldv, steps);
  char* p = (char*)workspace;
  double* const Wa = (double*)p;
  double* const Wb = (double*)(p + lay.block);
  double* part = (double*)(p + 2 * lay.block);
  double* h = (double*)(p + 2 * lay.block + lay.part);
  double* hc = (double*)(p + 2 * lay.block + lay.part + lay.h);
  double* stp = (double*)(p + 2 * lay.block + lay.part + 2 * lay.h);
  double* G = (double*)(p + 2 * lay.block + lay.part + 2 * lay.h + lay.state);
  LzState st{stp, stp + ldv, stp + 2 * ldv, stp + 3 * ldv};
  const size_t plane = (size_t)n * ldv;
  const int64_t norm_slot = steps;

  SDB_CUDA(cudaMemsetAsync(alpha, 0, sizeof(double) * n_vec * steps, s));
  SDB_CUDA(cudaMemsetAsync(beta, 0, sizeof(double) * n_vec * steps, s));
#define SDB_SN_CASE(LL, VV) lz_start_norm<LL, VV><<<(unsigned)nrb, kRowThreads, 0, s>>>(v0, n, ldv, nrb, panel, part)
  SDB_GEOMETRY_DISPATCH(g, SDB_SN_CASE);
#undef SDB_SN_CASE
  SDB_CHECK_LAUNCH();
  const int rblk = (int)((ldv + 127) / 128);
  lz_start_reduce<<<rblk, 128, 0, s>>>(part, nrb, ldv, n_vec, st, steps_done, status);
  SDB_CHECK_LAUNCH();
  const int cblk = (int)((ldv + 31) / 32);

  StencilView sv{};
  CsrView cv{};
  if (m->format == SDB_FMT_CSR) cv = make_csr_view(m); else sv = make_stencil_view(m);

  const bool fused = lz_fused_enabled();
  const bool gram = reorth == SDB_REORTH_FULL && lay.gdim > 0;
  const int64_t gram_slot0 = steps + 1;
  const double* wraw = v0;
  for (int64_t j = 0; j < steps; ++j) {
    // the step reads wraw (the previous step's w) and leaves its w in the other buffer
    double* const W1 = wraw == Wb ? Wa : Wb;
    double* const W0 = wraw == Wb ? Wb : Wa;
    double* wfinal = W0;
    double* vj = basis + (size_t)j * plane;
    const double* vprev = j > 0 ? basis + (size_t)(j - 1) * plane : nullptr;
    if (m->format == SDB_FMT_CSR)
      rc = lz_launch_spmm(cv, g, wraw, vprev, vj, W1, st, j == 0, c, 1.0 / d, n, nrb, panel, part, s);
    else if (m->shape == SDB_SHAPE_FACE7)
      rc = lz_launch_spmm(make_grid_view<SDB_SHAPE_FACE7>(m), g, wraw, vprev, vj, W1, st, j == 0, c, 1.0 / d, n, nrb,
                          panel, part, s);
    else if (m->shape == SDB_SHAPE_BOX27)
      rc = lz_launch_spmm(make_grid_view<SDB_SHAPE_BOX27>(m), g, wraw, vprev, vj, W1, st, j == 0, c, 1.0 / d, n, nrb,
                          panel, part, s);
    else
      rc = lz_launch_spmm(sv, g, wraw, vprev, vj, W1, st, j == 0, c, 1.0 / d, n, nrb, panel, part, s);
    if (rc) return rc;
    SDB_CHECK_LAUNCH();
    lz_alpha_reduce<<<cblk, 32 * kRedSegs, 0, s>>>(part, nrb, ldv, n_vec, j, steps, st, alpha, status);
    SDB_CHECK_LAUNCH();
    const dim3 hblk((unsigned)(j + 1), (unsigned)cblk);
    if (reorth == SDB_REORTH_FULL) {
      // pass 1 + 2.  Fused schedule (3 basis reads): h1 = V^T w on the raw w
      // (v_j is a basis column, so CGS on w also removes alpha v_j: the
      // reference's explicit w -= alpha v_j (lanczos.py:101-102) folds into
      // h1[j]); then w' = w - V h1 -> W0 together with h2 = V^T w' (K5c);
      // then w' -= V h2 with ||w'||^2.  Fallback (t range beyond the fused
      // kernel's registers): the reference order with 4 basis reads.
      const bool fz = fused && lz_update_proj_fits(j);
      if (gram && j + 1 <= lay.gdim) {
        // two basis reads: h1 = V^T w with the Gram column V^T v_j, h = 2 h1 - G h1, w -= V h in place
        if ((rc = lz_launch_proj_gram(nv, basis, W1, st, j, n, ldv, nrb, part, gram_slot0, s))) return rc;
        SDB_CHECK_LAUNCH();
        lz_h_reduce<<<hblk, 32 * kRedSegs, 0, s>>>(part, nrb, ldv, j, h, 0, norm_slot);
        SDB_CHECK_LAUNCH();
        lz_g_reduce<<<hblk, 32 * kRedSegs, 0, s>>>(part, gram_slot0, nrb, ldv, j, lay.gdim, G);
        SDB_CHECK_LAUNCH();
        lz_gram_correct<<<hblk, 32 * kRedSegs, 0, s>>>(G, h, ldv, j, lay.gdim, hc);
        SDB_CHECK_LAUNCH();
        if ((rc = lz_launch_update(g, true, basis, W1, hc, j, n, nrb, panel, part, s))) return rc;
        SDB_CHECK_LAUNCH();
        wfinal = W1;
      } else if (fz) {
        if ((rc = lz_launch_proj(nv, false, false, basis, W1, W1, st, j, n, ldv, nrb, part, norm_slot, s))) return rc;
        SDB_CHECK_LAUNCH();
        lz_h_reduce<<<hblk, 32 * kRedSegs, 0, s>>>(part, nrb, ldv, j, h, 0, norm_slot);
        SDB_CHECK_LAUNCH();
        lz_launch_update_proj(basis, W1, W0, h, j, n, ldv, nrb, part, s);
        SDB_CHECK_LAUNCH();
      } else {
        // w' = w - alpha v_j -> W0, h = V^T w'; w' -= V h; h = V^T w'
        if ((rc = lz_launch_proj(nv, true, false, basis, W1, W0, st, j, n, ldv, nrb, part, norm_slot, s))) return rc;
        SDB_CHECK_LAUNCH();
        lz_h_reduce<<<hblk, 32 * kRedSegs, 0, s>>>(part, nrb, ldv, j, h, 0, norm_slot);
        SDB_CHECK_LAUNCH();
        if ((rc = lz_launch_update(g, false, basis, W0, h, j, n, nrb, panel, part, s))) return rc;
        SDB_CHECK_LAUNCH();
        if ((rc = lz_launch_proj(nv, false, false, basis, W0, W0, st, j, n, ldv, nrb, part, norm_slot, s))) return rc;
        SDB_CHECK_LAUNCH();
      }
      if (wfinal == W0) {
        lz_h_reduce<<<hblk, 32 * kRedSegs, 0, s>>>(part, nrb, ldv, j, h, 0, norm_slot);
        SDB_CHECK_LAUNCH();
        if ((rc = lz_launch_update(g, true, basis, W0, h, j, n, nrb, panel, part, s))) return rc;
        SDB_CHECK_LAUNCH();
      }
    } else if (reorth == SDB_REORTH_SELECTIVE) {
      if ((rc = lz_launch_proj(nv, true, true, basis, W1, W0, st, j, n, ldv, nrb, part, norm_slot, s))) return rc;
      SDB_CHECK_LAUNCH();
      lz_h_reduce<<<hblk, 32 * kRedSegs, 0, s>>>(part, nrb, ldv, j, h, 1, norm_slot);
      SDB_CHECK_LAUNCH();
      if ((rc = lz_launch_update(g, true, basis, W0, h, j, n, nrb, panel, part, s))) return rc;
      SDB_CHECK_LAUNCH();
    } else {
#define SDB_NONE_CASE(LL, VV) \
  lz_sub_alpha_norm<LL, VV><<<(unsigned)nrb, kRowThreads, 0, s>>>(vj, W1, W0, st, n, ldv, nrb, panel, part)
      SDB_GEOMETRY_DISPATCH(g, SDB_NONE_CASE);
#undef SDB_NONE_CASE
      SDB_CHECK_LAUNCH();
    }
    lz_beta_reduce<<<cblk, 32 * kRedSegs, 0, s>>>(part, nrb, ldv, n_vec, j, steps, st, beta, steps_done, status);
    SDB_CHECK_LAUNCH();
    wraw = wfinal;
  }
  return SDB_OK;
}

}  // extern "C"
