// band.cu — probe-sliced band + far Chebyshev step for banded-plus-random CSR
// matrices (BASELINE config 3: a band of half-width 20 plus ~20 random
// off-band entries per row, n = 1e6, 128 probes).
//
// Reference hot loop: kpm.py:96-107 / kpm.py:174-189 with B x = (A x - c x)/d
// (matrix.py:125-126) and A x = csr @ x (matrix.py:101-102, csr_matvec: each
// row summed in storage order).
//
// Why a separate path.  With the probe block row-major (n x 128 fp64, 1 KB per
// row) the ~20 random columns of a row are 20 random 1 KB gathers from a 1 GB
// block that cannot stay in the 126 MB L2: the CSR kernel moves ~27 GB of DRAM
// per step against 3.8 GB of compulsory bytes.  Here
//   * the probe block is slice-major, [ns][rows][16]: one slice of 16 probes
//     is n x 128 B = 128 MB, and the whole grid works through one slice at a
//     time, so the random gathers of a slice mostly hit L2 (measured on B200,
//     tools/mb/c3_probe.cu: 128 B gathers from a 128 MB slice run at
//     ~15 TB/s, from the 1 GB block at ~5 TB/s);
//   * the dense band is split off at upload (band_build): symmetric, so only
//     its upper diagonals are stored (values only, no indices: 8 B per entry
//     for half the band), staged per 128-row tile in shared memory together
//     with the tile's x window (rows r0-pad .. r0+128+pad), and applied with a
//     register sliding window (each thread: 8 rows x 2 probe columns, one new
//     x row per diagonal);
//   * the remaining (far) entries are kept per row as a lower segment
//     (j < i - hb) and an upper segment (j > i + hb), pair-padded, so a row's
//     sum runs lower far -> band (d = -hb..hb) -> upper far: exactly the
//     sorted column order of the CSR, with the same fma chain from 0 -- the
//     band kernel's w is bit-identical to the CSR kernel's (padding terms are
//     fma(0, x, acc) = acc).
// The spectral map, 2 t - w_{k-1} (or the Legendre update) and the moment
// dots are fused into the epilogue as in cheb.cu; dot partials go to
// [(M+1)][grid][ldvb] and are reduced by K2 in fixed order (deterministic:
// the tile schedule is static).
#include <cub/cub.cuh>

#include <cstdlib>
#include <vector>

#include "stepargs.cuh"

namespace sdb {

constexpr int kBandRT = 4;         // rows per thread = SELL chunk height of the far slots
constexpr int kBandThreads = 256;
constexpr int kBandTileAlign = 256; // rows are padded to this (covers every tile height)
constexpr int kBandMaxOff = 64;    // offsets histogrammed for the band search

// Block geometry for a slice of S probe columns: S/2 threads per row group
// (one double2 column pair each), kBandRT consecutive rows per row group.
template <int S>
struct BandGeom {
  static constexpr int TPR = S / 2;
  static constexpr int NG = kBandThreads / TPR;  // row groups per block
  static constexpr int R = NG * kBandRT;         // rows per tile (S=16: 128, S=8: 256)
};

// band half-widths with a kernel instantiation (the detected band is rounded up)
constexpr int kBandWidths[] = {8, 16, 20, 24, 32};

// ---- device helpers -----------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, uint64_t pol) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
// L2 policies: the x slice being gathered is kept (evict_last); everything
// streamed once per slice pass (band diagonals, far slots, w_{k-1}, v0,
// w_{k+1}) is evict_first, so the data streamed per pass does not push the
// slice out of L2 between its ~21 reuses.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_x_keep(const double* p, uint64_t pol) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int4 ld_i4_once(const int4* p, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ double2 ld_d2_nc_once(const double2* p, uint64_t pol) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p), "l"(pol));
  return r;
}

struct BandArgs {
  const double* x;      // slice-major blocks, base of slice 0 (guard row 0)
  const double* prev;
  double* next;
  const double* v0;
  int64_t sstride;      // doubles per slice
  const double* bu;     // [hb+1][ustride]
  int64_t ustride;
  const int32_t* fptr;
  const int32_t* fmid;
  const int4* fcol;
  const double2* fval;
  double c, inv_d;
  int64_t n, ntiles;
  int nslices;
  int64_t ldv;          // partials row width (nslices * S)
  double* partials;
  int64_t nblocks;
  int slotA, slotB, slot0;
  int legendre;
  double la, lb, lc;
  int diag;             // diagnostics (SDB_BAND_DIAG): 1 skip far, 2 far gathers own row, 4 skip band
  int slice0;           // first slice of this launch (per-slice launches)
};

// Bulk L2 prefetch (TMA engine, no registers, no completion): the next
// tile's streamed operands are requested while this tile computes, so the
// far-slot loads of the gather rounds hit L2 instead of waiting on DRAM.
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes, uint64_t pol) {
  if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(pol)
                          : "memory");
}

// Far entries of rows row0 .. row0+3 (one SELL-4 chunk; its lower or upper
// segments), gathered from the L2-resident x slice and accumulated in storage
// order.  A slot holds one entry per row and segments hold an even number of
// slots (padding: own row, weight 0): each round issues two slots' eight
// gathers with no predicates, then loads the next two slots' columns and
// values (L2 hits: bulk-prefetched) while the gathers are in flight.
template <int S, bool LOWER>
__device__ __forceinline__ void band_far(const BandArgs& a, const double* __restrict__ xsl, int64_t row0, int q,
                                         double2 (&acc)[kBandRT], uint64_t keep, uint64_t once) {
  const int c = (int)(row0 / kBandRT);
  int s = LOWER ? __ldg(a.fptr + c) : __ldg(a.fmid + c);
  const int s1 = LOWER ? __ldg(a.fmid + c) : __ldg(a.fptr + c + 1);
  if (s >= s1) return;
  const double* xq = xsl + 2 * q;
  int4 c0 = ld_i4_once(a.fcol + s, once), c1 = ld_i4_once(a.fcol + s + 1, once);
  double2 v0 = ld_d2_nc_once(a.fval + 2 * s, once), v1 = ld_d2_nc_once(a.fval + 2 * s + 1, once),
          v2 = ld_d2_nc_once(a.fval + 2 * s + 2, once), v3 = ld_d2_nc_once(a.fval + 2 * s + 3, once);
  for (;;) {
    const double2 g0 = ld_x_keep(xq + c0.x * S, keep), g1 = ld_x_keep(xq + c0.y * S, keep),
                  g2 = ld_x_keep(xq + c0.z * S, keep), g3 = ld_x_keep(xq + c0.w * S, keep),
                  g4 = ld_x_keep(xq + c1.x * S, keep), g5 = ld_x_keep(xq + c1.y * S, keep),
                  g6 = ld_x_keep(xq + c1.z * S, keep), g7 = ld_x_keep(xq + c1.w * S, keep);
    const double2 w0 = v0, w1 = v1, w2 = v2, w3 = v3;
    s += 2;
    const bool more = s < s1;
    if (more) {
      c0 = ld_i4_once(a.fcol + s, once);
      c1 = ld_i4_once(a.fcol + s + 1, once);
      v0 = ld_d2_nc_once(a.fval + 2 * s, once);
      v1 = ld_d2_nc_once(a.fval + 2 * s + 1, once);
      v2 = ld_d2_nc_once(a.fval + 2 * s + 2, once);
      v3 = ld_d2_nc_once(a.fval + 2 * s + 3, once);
    }
    // slot s-2 (rows 0..3) before slot s-1: per-row storage order
    acc[0].x = fma(w0.x, g0.x, acc[0].x); acc[0].y = fma(w0.x, g0.y, acc[0].y);
    acc[1].x = fma(w0.y, g1.x, acc[1].x); acc[1].y = fma(w0.y, g1.y, acc[1].y);
    acc[2].x = fma(w1.x, g2.x, acc[2].x); acc[2].y = fma(w1.x, g2.y, acc[2].y);
    acc[3].x = fma(w1.y, g3.x, acc[3].x); acc[3].y = fma(w1.y, g3.y, acc[3].y);
    acc[0].x = fma(w2.x, g4.x, acc[0].x); acc[0].y = fma(w2.x, g4.y, acc[0].y);
    acc[1].x = fma(w2.y, g5.x, acc[1].x); acc[1].y = fma(w2.y, g5.y, acc[1].y);
    acc[2].x = fma(w3.x, g6.x, acc[2].x); acc[2].y = fma(w3.x, g6.y, acc[2].y);
    acc[3].x = fma(w3.y, g7.x, acc[3].x); acc[3].y = fma(w3.y, g7.y, acc[3].y);
    if (!more) break;
  }
}

// Band rows rl .. rl+3 of the tile: for d = -HB..HB (increasing column),
// acc[r] += A[i][i+d] x[i+d] with A[i][i+d] = bu[d][i] (d >= 0) or
// bu[-d][i+d] (d < 0, symmetry); x rows come from the staged window through
// a register sliding window (one new row per diagonal).
template <int HB, int S>
__device__ __forceinline__ void band_diag(const double* xs, const double* us, int rl, int q,
                                          double2 (&acc)[kBandRT]) {
  constexpr int P = band_pad(HB), RT = kBandRT, UW = BandGeom<S>::R + P;
  double2 win[RT];
#pragma unroll
  for (int r = 0; r < RT; ++r) win[r] = lds2(xs + (rl + P - HB + r) * S + 2 * q);
#pragma unroll
  for (int d = -HB; d <= HB; ++d) {
    double v[RT];
    const double* vp = d >= 0 ? us + d * UW + P + rl : us + (-d) * UW + P + rl + d;
    if (d >= 0 || (d & 1) == 0) {
#pragma unroll
      for (int r = 0; r < RT; r += 2) {
        const double2 t = lds2(vp + r);
        v[r] = t.x;
        v[r + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int r = 0; r < RT; ++r) v[r] = vp[r];
    }
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      acc[r].x = fma(v[r], win[r].x, acc[r].x);
      acc[r].y = fma(v[r], win[r].y, acc[r].y);
    }
    if (d < HB) {
#pragma unroll
      for (int r = 0; r < RT - 1; ++r) win[r] = win[r + 1];
      win[RT - 1] = lds2(xs + (rl + P + d + RT) * S + 2 * q);
    }
  }
}

template <int HB, int S>
__host__ __device__ constexpr size_t band_smem_doubles() {
  return (size_t)(BandGeom<S>::R + 2 * band_pad(HB)) * S + (size_t)(HB + 1) * (BandGeom<S>::R + band_pad(HB));
}

template <int HB, int S, int MODE, bool FIRST>
__global__ void __launch_bounds__(kBandThreads, 2) cheb_step_band(BandArgs a) {
  using Gm = BandGeom<S>;
  constexpr int P = band_pad(HB), R = Gm::R, RT = kBandRT, TPR = Gm::TPR;
  constexpr int XW = R + 2 * P, UW = R + P;
  extern __shared__ __align__(16) double band_smem[];
  double* xs = band_smem;           // XW x S   x rows r0-P .. r0+R+P
  double* us = band_smem + XW * S;  // (HB+1) x UW   bu[d][r0-P .. r0+R)
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x, g = tid / TPR, q = tid % TPR, rl = g * RT;
  const uint64_t pol = policy_evict_first(), keep = policy_evict_last();
  const int G = gridDim.x, b = blockIdx.x, ntiles = (int)a.ntiles;
  const int warp = tid >> 5, lane = tid & 31;
  for (int s = a.slice0; s < a.slice0 + a.nslices; ++s) {
    const int64_t so = s * a.sstride + (int64_t)P * S;  // row 0 of slice s
    const double* xsl = a.x + so;
    double2 accA = make_double2(0.0, 0.0), accB = accA, accZ = accA;
    // static schedule over the items (slice, tile) in slice-major order
    const int base = (s - a.slice0) * ntiles;
    const int t0 = (int)(((int64_t)b - base) % G + G) % G;
    for (int t = t0; t < ntiles; t += G) {
      const int64_t r0 = (int64_t)t * R;
      // this block's next item, and its far-slot range (loaded now, used below)
      const int tn = t + G;
      const int s_n = s + tn / ntiles;  // G <= ntiles: at most one slice ahead
      const int64_t r0n = (int64_t)(tn % ntiles) * R;
      const bool has_next = s_n < a.slice0 + a.nslices;
      int f_n = 0;
      if (warp == 1 && lane < 2 && has_next) f_n = __ldg(a.fptr + (r0n + lane * R) / kBandRT);
      {  // stage the x window and the band diagonals of this tile
        const double* xw = a.x + s * a.sstride + r0 * S;  // = xsl + (r0 - P) * S
        for (int c = tid; c < XW * S / 2; c += kBandThreads) cp_async16(xs + 2 * c, xw + 2 * c, keep);
        constexpr int UC = UW / 2;
        for (int c = tid; c < (HB + 1) * UC; c += kBandThreads) {
          const int d = c / UC, k = c - d * UC;
          cp_async16(us + d * UW + 2 * k, a.bu + d * a.ustride + r0 + 2 * k, pol);
        }
        cp_async_commit();
      }
      const int64_t row0 = r0 + rl;
      double2 acc[RT];
#pragma unroll
      for (int r = 0; r < RT; ++r) acc[r] = make_double2(0.0, 0.0);
      if (!(a.diag & 1)) band_far<S, true>(a, xsl, row0, q, acc, keep, pol);
      cp_async_wait_all();
      __syncthreads();
      if (!(a.diag & 4)) band_diag<HB, S>(xs, us, rl, q, acc);
      if (has_next && warp <= 1) {  // L2 prefetch of the next item's operands
        if (warp == 0) {
          for (int d = lane; d <= HB; d += 32) l2_prefetch(a.bu + d * a.ustride + r0n, UW * 8, pol);
        } else {
          const int f1 = __shfl_sync(0xffffffffu, f_n, 1), f0 = __shfl_sync(0xffffffffu, f_n, 0);
          const int64_t son = s_n * a.sstride + (int64_t)P * S;
          if (lane == 0) l2_prefetch(a.fcol + f0, (uint32_t)(f1 - f0) * 16u, pol);
          if (lane == 1) l2_prefetch(a.fval + 2 * f0, (uint32_t)(f1 - f0) * 32u, pol);
          if (lane == 2 && !FIRST) l2_prefetch(a.prev + son + r0n * S, R * S * 8, pol);
          if (lane == 3 && MODE == SDB_CHEB_DIRECT && !FIRST) l2_prefetch(a.v0 + son + r0n * S, R * S * 8, pol);
          if (lane == 4) l2_prefetch(a.x + s_n * a.sstride + r0n * S, XW * S * 8, keep);
        }
      }
      if (!(a.diag & 1)) band_far<S, false>(a, xsl, row0, q, acc, keep, pol);
      // epilogue: t = (A x - c x)/d; w+ = t | 2t - w- | Legendre; dots.  The
      // row operands are all requested before the first store.
      double2 wp[RT], p0[RT];
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        const int64_t o = so + (row0 + r) * S + 2 * q;
        wp[r] = p0[r] = make_double2(0.0, 0.0);
        if (row0 + r < a.n) {
          if (!FIRST) wp[r] = ld_d2_once(a.prev + o, pol);
          if (MODE == SDB_CHEB_DIRECT && !FIRST) p0[r] = ld_d2_once(a.v0 + o, pol);
        }
      }
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        const int64_t row = row0 + r;
        if (row < a.n) {
          const double2 xi = lds2(xs + (rl + P + r) * S + 2 * q);
          const int64_t o = so + row * S + 2 * q;
          if (FIRST || MODE != SDB_CHEB_DIRECT) p0[r] = xi;
          const double tx = (acc[r].x - a.c * xi.x) * a.inv_d;
          const double ty = (acc[r].y - a.c * xi.y) * a.inv_d;
          double2 wn;
          if (FIRST) {
            wn = make_double2(tx, ty);
          } else if (MODE == SDB_CHEB_DIRECT && a.legendre) {
            wn.x = (a.la * tx - a.lb * wp[r].x) / a.lc;
            wn.y = (a.la * ty - a.lb * wp[r].y) / a.lc;
          } else {
            wn.x = 2.0 * tx - wp[r].x;
            wn.y = 2.0 * ty - wp[r].y;
          }
          st_d2_once(a.next + o, wn, pol);
          if (MODE == SDB_CHEB_DOUBLING) {
            accA.x += wn.x * wn.x;
            accA.y += wn.y * wn.y;
            accB.x += wn.x * xi.x;
            accB.y += wn.y * xi.y;
          } else {
            accA.x += p0[r].x * wn.x;
            accA.y += p0[r].y * wn.y;
          }
          if (FIRST) {
            accZ.x += xi.x * xi.x;
            accZ.y += xi.y * xi.y;
          }
        }
      }
      __syncthreads();  // the next tile's staging overwrites xs / us
    }
    // per-slice partial rows: sum the row groups in order (deterministic)
    double* red = band_smem;
    auto flush = [&](const double2& acc, int slot) {
      red[g * S + 2 * q] = acc.x;
      red[g * S + 2 * q + 1] = acc.y;
      __syncthreads();
      if (tid < S) {
        double sum = 0.0;
#pragma unroll 8
        for (int gg = 0; gg < Gm::NG; ++gg) sum += red[gg * S + tid];
        a.partials[((int64_t)slot * a.nblocks + b) * a.ldv + s * S + tid] = sum;
      }
      __syncthreads();
    };
    if (a.slotA >= 0) flush(accA, a.slotA);
    if (MODE == SDB_CHEB_DOUBLING && a.slotB >= 0) flush(accB, a.slotB);
    if (FIRST && a.slot0 >= 0) flush(accZ, a.slot0);
  }
}

// ---- probe packing ----------------------------------------------------------------
// probes (n x ldv row-major) -> v0b [ns][rows][S] with zero guard / padding
// rows and columns; the same rows of bufA / bufB are zeroed (never written by
// the step kernel, read through the x windows).
__global__ void band_pack_kernel(const double* __restrict__ in, int64_t n, int64_t ldv, int S, int ns, int64_t rows,
                                 int pad, double* __restrict__ v0b, double* __restrict__ bufA,
                                 double* __restrict__ bufB) {
  const int half = S / 2;
  const int64_t total = (int64_t)ns * rows * half;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c2 = (int)(idx % half);
    const int64_t rr = (idx / half) % rows;
    const int s = (int)(idx / ((int64_t)half * rows));
    const int64_t i = rr - pad;
    const int64_t col = (int64_t)s * S + 2 * c2;
    const bool inside = i >= 0 && i < n;
    double2 v = make_double2(0.0, 0.0);
    if (inside && col < ldv) v = *reinterpret_cast<const double2*>(in + i * ldv + col);
    const int64_t o = ((int64_t)s * rows + rr) * S + 2 * c2;
    *reinterpret_cast<double2*>(v0b + o) = v;
    if (!inside) {
      *reinterpret_cast<double2*>(bufA + o) = make_double2(0.0, 0.0);
      *reinterpret_cast<double2*>(bufB + o) = make_double2(0.0, 0.0);
    }
  }
}

// ---- split construction (one-time, at upload) ---------------------------------------
__global__ void band_hist_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t n,
                                 unsigned long long* __restrict__ hist, int* __restrict__ unsorted) {
  // hist[0..kBandMaxOff]: entries with j - i = d (upper), hist[kBandMaxOff+1+d]: i - j = d (lower)
  __shared__ unsigned int h[2 * (kBandMaxOff + 1)];
  for (int k = threadIdx.x; k < 2 * (kBandMaxOff + 1); k += blockDim.x) h[k] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int prev = -1;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int j = ci[k];
      if (j <= prev) *unsorted = 1;
      prev = j;
      const int64_t d = (int64_t)j - i;
      if (d >= 0 && d <= kBandMaxOff) atomicAdd(&h[d], 1u);
      else if (d < 0 && -d <= kBandMaxOff) atomicAdd(&h[kBandMaxOff + 1 - d], 1u);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 2 * (kBandMaxOff + 1); k += blockDim.x)
    if (h[k]) atomicAdd(&hist[k], (unsigned long long)h[k]);
}

// upper band -> bu; per-chunk far slot counts (max over the chunk's 4 rows of
// the lower / upper off-band counts)
__global__ void band_fill_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 const double* __restrict__ va, int64_t n, int hb, int pad, int64_t ustride,
                                 double* __restrict__ bu, int64_t nchunks, int32_t* __restrict__ cnt,
                                 int32_t* __restrict__ low, unsigned long long* __restrict__ far_nnz) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks; c += (int64_t)gridDim.x * blockDim.x) {
    int ml = 0, mu = 0, tot = 0;
    for (int64_t i = kBandRT * c; i < kBandRT * (c + 1) && i < n; ++i) {
      int nl = 0, nu = 0;
      for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int64_t d = (int64_t)ci[k] - i;
        if (d >= 0 && d <= hb) bu[d * ustride + pad + i] = va[k];
        else if (d < -hb) ++nl;
        else if (d > hb) ++nu;
      }
      ml = nl > ml ? nl : ml;
      mu = nu > mu ? nu : mu;
      tot += nl + nu;
    }
    ml = (ml + 1) & ~1;  // slots are consumed in pairs
    mu = (mu + 1) & ~1;
    low[c] = ml;
    cnt[c] = ml + mu;
    if (tot) atomicAdd(far_nnz, (unsigned long long)tot);
  }
}

// every lower band entry must equal its mirrored upper entry bit for bit
__global__ void band_sym_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double* __restrict__ va, int64_t n, int hb, int pad, int64_t ustride,
                                const double* __restrict__ bu, int* __restrict__ asym) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int64_t j = ci[k], d = i - j;
      if (d >= 1 && d <= hb) {
        const double u = bu[d * ustride + pad + j];
        if (__double_as_longlong(u) != __double_as_longlong(va[k])) *asym = 1;
      }
    }
  }
}

// SELL-4 far slots: chunk c's lower slots then upper slots (even counts),
// row r of the chunk at lane r of every slot, entries in storage (column)
// order, padded with (own row, 0.0)
__global__ void band_far_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double* __restrict__ va, int64_t n, int hb, int64_t nchunks,
                                const int32_t* __restrict__ fptr, const int32_t* __restrict__ low,
                                int32_t* __restrict__ fmid, int32_t* __restrict__ fcol, double* __restrict__ fval) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks; c += (int64_t)gridDim.x * blockDim.x) {
    const int s0 = fptr[c], sm = s0 + low[c], s1 = fptr[c + 1];
    fmid[c] = sm;
    for (int r = 0; r < kBandRT; ++r) {
      const int64_t i = kBandRT * c + r;
      int pl = s0, pu = sm;
      if (i < n) {
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
          const int64_t d = (int64_t)ci[k] - i;
          if (d < -hb) {
            fcol[kBandRT * (int64_t)pl + r] = ci[k];
            fval[kBandRT * (int64_t)pl + r] = va[k];
            ++pl;
          } else if (d > hb) {
            fcol[kBandRT * (int64_t)pu + r] = ci[k];
            fval[kBandRT * (int64_t)pu + r] = va[k];
            ++pu;
          }
        }
      }
      // padding: the row's own x with weight 0 (fma(0, x_i, acc) = acc for
      // finite x_i), so the gather loop needs no predicates
      const int32_t self = (int32_t)(i < n ? i : n - 1);
      for (; pl < sm; ++pl) {
        fcol[kBandRT * (int64_t)pl + r] = self;
        fval[kBandRT * (int64_t)pl + r] = 0.0;
      }
      for (; pu < s1; ++pu) {
        fcol[kBandRT * (int64_t)pu + r] = self;
        fval[kBandRT * (int64_t)pu + r] = 0.0;
      }
    }
  }
}

static bool band_env_enabled() {
  const char* e = getenv("SDB_BAND");
  return !(e && e[0] == '0');
}

int band_build(sdb_matrix* m, cudaStream_t s) {
  if (m->format != SDB_FMT_CSR || m->nnz == 0 || m->n < 2 * kBandTileAlign || !band_env_enabled()) return SDB_OK;
  const int64_t n = m->n;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 4LL * num_sms(m->device));
  unsigned long long* hist = nullptr;
  int* flags = nullptr;  // [0] unsorted/duplicate, [1] asymmetric
  SDB_CUDA(cudaMalloc(&hist, sizeof(unsigned long long) * 2 * (kBandMaxOff + 1)));
  SDB_CUDA(cudaMalloc(&flags, 2 * sizeof(int)));
  struct Free {
    void* p[2];
    ~Free() {
      for (void* x : p)
        if (x) cudaFree(x);
    }
  } fr{{hist, flags}};
  SDB_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * 2 * (kBandMaxOff + 1), s));
  SDB_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), s));
  band_hist_kernel<<<blocks, 256, 0, s>>>(m->rowptr, m->colidx, n, hist, flags);
  SDB_CHECK_LAUNCH();
  std::vector<unsigned long long> h(2 * (kBandMaxOff + 1));
  int hflags[2] = {0, 0};
  SDB_CUDA(cudaMemcpyAsync(h.data(), hist, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, s));
  SDB_CUDA(cudaMemcpyAsync(hflags, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  SDB_CUDA(cudaStreamSynchronize(s));
  if (hflags[0]) return SDB_OK;  // rows must be sorted without duplicates (csr_matvec order = column order)
  // dense band: every off-diagonal d <= hb at least half full
  int hb = 0;
  while (hb < kBandMaxOff && (double)h[hb + 1] >= 0.5 * (double)(n - hb - 1)) ++hb;
  int hbk = 0;
  for (int w : kBandWidths)
    if (w >= hb) {
      hbk = w;
      break;
    }
  if (hb < 4 || hbk == 0) return SDB_OK;
  unsigned long long band_nnz = h[0];
  for (int d = 1; d <= hbk; ++d) {
    if (h[d] != h[kBandMaxOff + 1 + d]) return SDB_OK;  // not structurally symmetric
    band_nnz += 2 * h[d];
  }
  if ((double)band_nnz < 0.25 * (double)m->nnz) return SDB_OK;
  const int pad = band_pad(hbk);
  const int64_t npad = (n + kBandTileAlign - 1) / kBandTileAlign * kBandTileAlign;
  const int64_t ustride = pad + npad;
  const int64_t nchunks = npad / kBandRT;
  double* bu = nullptr;
  int32_t *cnt = nullptr, *low = nullptr, *fptr = nullptr, *fmid = nullptr, *fcol = nullptr;
  double* fval = nullptr;
  void* tmp = nullptr;
  unsigned long long* fnnz_d = hist;  // reuse: the histogram has been read back
  auto release = [&]() {
    for (void* p : {(void*)bu, (void*)cnt, (void*)low, (void*)fptr, (void*)fmid, (void*)fcol, (void*)fval, tmp})
      if (p) cudaFree(p);
  };
  cudaError_t e = cudaMalloc(&bu, sizeof(double) * (hbk + 1) * ustride);
  if (e == cudaSuccess) e = cudaMalloc(&cnt, sizeof(int32_t) * (nchunks + 1));
  if (e == cudaSuccess) e = cudaMalloc(&low, sizeof(int32_t) * nchunks);
  if (e == cudaSuccess) e = cudaMalloc(&fptr, sizeof(int32_t) * (nchunks + 1));
  if (e == cudaSuccess) e = cudaMalloc(&fmid, sizeof(int32_t) * nchunks);
  if (e == cudaSuccess) e = cudaMemsetAsync(bu, 0, sizeof(double) * (hbk + 1) * ustride, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt + nchunks, 0, sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(fnnz_d, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) {
    release();
    return cuda_fail(e, "band split allocation", __FILE__, __LINE__);
  }
  const int cblocks = (int)std::min<int64_t>((nchunks + 255) / 256, 4LL * num_sms(m->device));
  band_fill_kernel<<<cblocks, 256, 0, s>>>(m->rowptr, m->colidx, m->values, n, hbk, pad, ustride, bu, nchunks, cnt,
                                           low, fnnz_d);
  band_sym_kernel<<<blocks, 256, 0, s>>>(m->rowptr, m->colidx, m->values, n, hbk, pad, ustride, bu, flags + 1);
  size_t tmp_bytes = 0;
  e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, fptr, nchunks + 1, s);
  if (e == cudaSuccess) e = cudaMalloc(&tmp, tmp_bytes);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, fptr, nchunks + 1, s);
  int32_t total = 0;
  unsigned long long fnnz = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&total, fptr + nchunks, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&fnnz, fnnz_d, sizeof(fnnz), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hflags, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    release();
    return cuda_fail(e, "band split", __FILE__, __LINE__);
  }
  if (hflags[1]) {  // values not symmetric: keep the plain CSR path
    release();
    return SDB_OK;
  }
  const int64_t fn = kBandRT * (int64_t)(total > 0 ? total : 1);
  e = cudaMalloc(&fcol, sizeof(int32_t) * fn);
  if (e == cudaSuccess) e = cudaMalloc(&fval, sizeof(double) * fn);
  if (e == cudaSuccess) {
    band_far_kernel<<<cblocks, 256, 0, s>>>(m->rowptr, m->colidx, m->values, n, hbk, nchunks, fptr, low, fmid, fcol,
                                            fval);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(cnt);
  cudaFree(low);
  cudaFree(tmp);
  cnt = low = nullptr;
  tmp = nullptr;
  if (e != cudaSuccess) {
    release();
    return cuda_fail(e, "band far entries", __FILE__, __LINE__);
  }
  m->hb = hbk;
  m->ustride = ustride;
  m->bu = bu;
  m->fptr = fptr;
  m->fmid = fmid;
  m->fcol = reinterpret_cast<int4*>(fcol);
  m->fval = reinterpret_cast<double2*>(fval);
  m->fslots = total;
  m->fnnz = (int64_t)fnnz;
  return SDB_OK;
}

// ---- host planning / launch ---------------------------------------------------------
#define SDB_BAND_HB(HBV, CASE) \
  do {                         \
    switch (HBV) {             \
      case 8: CASE(8); break;  \
      case 16: CASE(16); break; \
      case 20: CASE(20); break; \
      case 24: CASE(24); break; \
      case 32: CASE(32); break; \
      default: return fail(SDB_EUNSUPPORTED, "no band kernel for half-width %d", HBV); \
    }                          \
  } while (0)

template <int HB, int S>
static int band_occupancy(int* occ, size_t* smem) {
  *smem = sizeof(double) * band_smem_doubles<HB, S>();
  const void* fns[4] = {(const void*)cheb_step_band<HB, S, SDB_CHEB_DOUBLING, true>,
                        (const void*)cheb_step_band<HB, S, SDB_CHEB_DOUBLING, false>,
                        (const void*)cheb_step_band<HB, S, SDB_CHEB_DIRECT, true>,
                        (const void*)cheb_step_band<HB, S, SDB_CHEB_DIRECT, false>};
  int best = 1 << 20;
  for (const void* f : fns) {
    SDB_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem));
    int o = 0;
    SDB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, f, kBandThreads, *smem));
    best = o < best ? o : best;
  }
  *occ = best < 1 ? 1 : best;
  return SDB_OK;
}

// Slice width: 16 probe columns (128 MB x slice at n = 1e6, 8 matrix passes
// for 128 probes) or 8 (64 MB slice, 16 passes); SDB_BAND_S overrides.
static int band_slice_width() {
  const char* e = getenv("SDB_BAND_S");
  const int v = e ? atoi(e) : 16;
  return v == 8 ? 8 : 16;
}

int band_plan(const sdb_matrix* m, int64_t n_vec, int mode, BandPlan* p) {
  *p = BandPlan{};
  if (m->hb <= 0 || n_vec < 1 || n_vec > SDB_MAX_BATCH) return SDB_OK;
  if (const char* e = getenv("SDB_BAND"))
    if (e[0] == '0') return SDB_OK;
  (void)mode;
  const int S = band_slice_width();
  p->hb = m->hb;
  p->S = S;
  p->R = S == 16 ? BandGeom<16>::R : BandGeom<8>::R;
  p->ns = (int)((n_vec + S - 1) / S);
  p->ldvb = (int64_t)p->ns * S;
  const int pad = band_pad(m->hb);
  const int64_t npad = (m->n + kBandTileAlign - 1) / kBandTileAlign * kBandTileAlign;
  p->rows = npad + 2 * pad;
  p->ntiles = npad / p->R;
  int occ = 1;
  size_t smem = 0;
  {
    DeviceGuard dg(m->device);
#define SDB_BAND_OCC(HBV)                                                                          \
  {                                                                                                \
    int rc = S == 16 ? band_occupancy<HBV, 16>(&occ, &smem) : band_occupancy<HBV, 8>(&occ, &smem); \
    if (rc) return rc;                                                                             \
  }
    SDB_BAND_HB(m->hb, SDB_BAND_OCC);
#undef SDB_BAND_OCC
  }
  if (const char* e = getenv("SDB_BAND_BPS")) {
    const int v = atoi(e);
    if (v > 0 && v < occ) occ = v;
  }
  int64_t grid = (int64_t)occ * num_sms(m->device);
  if (grid > 8LL * num_sms(m->device)) grid = 8LL * num_sms(m->device);  // partials sized for 8 per SM
  if (grid > p->ntiles) grid = p->ntiles;
  p->grid = grid < 1 ? 1 : grid;
  p->smem = smem;
  p->block_bytes = ((size_t)p->ns * p->rows * S * sizeof(double) + 255) & ~(size_t)255;
  p->on = true;
  return SDB_OK;
}

int band_pack(const sdb_matrix* m, const BandPlan& p, const double* probes, int64_t ldv, double* v0b, double* bufA,
              double* bufB, cudaStream_t s) {
  const int64_t total = (int64_t)p.ns * p.rows * (p.S / 2);
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 16LL * num_sms(m->device));
  band_pack_kernel<<<blocks, 256, 0, s>>>(probes, m->n, ldv, p.S, p.ns, p.rows, band_pad(p.hb), v0b, bufA, bufB);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

template <int HB, int S, int MODE, bool FIRST>
static int band_launch_t(const BandPlan& p, BandArgs& ba, cudaStream_t s) {
  void* args[] = {(void*)&ba};
  SDB_CUDA(launch_maybe_pdl((const void*)cheb_step_band<HB, S, MODE, FIRST>, dim3((unsigned)p.grid),
                            dim3(kBandThreads), args, p.smem, s));
  return SDB_OK;
}

template <int HB, int S>
static int band_launch_mode(const BandPlan& p, BandArgs& ba, bool first, int mode, cudaStream_t s) {
  if (mode == SDB_CHEB_DOUBLING)
    return first ? band_launch_t<HB, S, SDB_CHEB_DOUBLING, true>(p, ba, s)
                 : band_launch_t<HB, S, SDB_CHEB_DOUBLING, false>(p, ba, s);
  return first ? band_launch_t<HB, S, SDB_CHEB_DIRECT, true>(p, ba, s)
               : band_launch_t<HB, S, SDB_CHEB_DIRECT, false>(p, ba, s);
}

int band_launch_step(const sdb_matrix* m, const BandPlan& p, const StepArgs& a, bool first, int mode,
                     cudaStream_t s) {
  BandArgs ba{};
  ba.x = a.x;
  ba.prev = a.prev;
  ba.next = a.next;
  ba.v0 = a.v0;
  ba.sstride = p.rows * p.S;
  ba.bu = m->bu;
  ba.ustride = m->ustride;
  ba.fptr = m->fptr;
  ba.fmid = m->fmid;
  ba.fcol = m->fcol;
  ba.fval = m->fval;
  ba.c = a.c;
  ba.inv_d = a.inv_d;
  ba.n = m->n;
  ba.ntiles = p.ntiles;
  ba.nslices = p.ns;
  ba.ldv = p.ldvb;
  ba.partials = a.partials;
  ba.nblocks = p.grid;
  ba.slotA = a.slotA;
  ba.slotB = a.slotB;
  ba.slot0 = a.slot0;
  ba.legendre = a.legendre;
  ba.la = a.la;
  ba.lb = a.lb;
  ba.lc = a.lc;
  if (const char* e = getenv("SDB_BAND_DIAG")) ba.diag = atoi(e);
  // SDB_BAND_PERSLICE=1: one launch per probe slice (the whole grid finishes
  // slice s before any block starts slice s+1)
  const char* ps = getenv("SDB_BAND_PERSLICE");
  const int per_slice = ps && ps[0] == '1';
  for (int s0 = 0; s0 < p.ns; s0 += per_slice ? 1 : p.ns) {
    ba.slice0 = s0;
    ba.nslices = per_slice ? 1 : p.ns;
    int rc = SDB_OK;
#define SDB_BAND_LAUNCH(HBV)                                                                            \
  rc = p.S == 16 ? band_launch_mode<HBV, 16>(p, ba, first, mode, s) : band_launch_mode<HBV, 8>(p, ba, first, mode, s)
    SDB_BAND_HB(m->hb, SDB_BAND_LAUNCH);
#undef SDB_BAND_LAUNCH
    if (rc) return rc;
  }
  return SDB_OK;
}

}  // namespace sdb

using namespace sdb;

extern "C" int sdb_matrix_band_info(const sdb_matrix* m, int32_t* half_width, int64_t* far_entries,
                                    int64_t* bytes_per_pass) {
  SDB_REQUIRE(m != nullptr, "NULL argument");
  if (half_width) *half_width = m->hb;
  if (far_entries) *far_entries = m->hb ? m->fnnz : 0;
  if (bytes_per_pass)
    *bytes_per_pass = m->hb ? (int64_t)(m->hb + 1) * 8 * m->n + 12 * kBandRT * m->fslots + 8 * (m->n / kBandRT + 1) : 0;
  return SDB_OK;
}
