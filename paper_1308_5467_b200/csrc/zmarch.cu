// zmarch.cu — TMA z-marching Chebyshev step for periodic 7-point / 27-point
// grids (both moment modes); used by sdb_cheb_moments (cheb.cu) when it applies.
//
// Why: with 64 probes one grid point of the probe block is 512 B.  The
// row-panel kernel (cheb_step_grid) gathers every neighbour through L2
// (~1.15 GB of L2->SM traffic per C2 step, capped by L2 throughput), and the
// cp.async tile kernel (tile25d.cuh) spends its time issuing 16-byte copies
// and waiting at block barriers.  Here:
//
//  * the recurrence buffers use a ghost-padded layout
//      [nz][ny+4][nx+4][ldv]   (two periodic ghost layers in x and y)
//    so the (TY+2) x (TX+2) halo tile of a plane, CS probe columns wide, is
//    ONE rectangular TMA box (cp.async.bulk.tensor.4d), whatever the tile's
//    position on the torus; the epilogue writes the ghost copies of boundary
//    points (3 % extra stores at 256^2 planes, 13 % at 64^2);
//  * one producer warp streams the planes of the block's z-segment through a
//    ring of R shared-memory slots (mbarrier full/empty pairs, expect_tx), so
//    the consumer warps never execute a block-wide barrier;
//  * each consumer thread owns PPT (x, y) columns x one probe pair and marches
//    z with three rolling register accumulators: plane p is read from shared
//    memory ONCE (9 or 5 loads per point) and contributes its dz = -1 terms to
//    out(p+1), its dz = 0 terms to out(p) and its dz = +1 terms to out(p-1),
//    which is then complete.  Per output point the FMAs therefore run in
//    lexicographic (dz, dy, dx) order -- the same sequence as cheb_step_grid,
//    so both kernels produce bit-identical w_{k+1};
//  * the slot is released right after the loads (values live in registers);
//    w_{k-1}, v_0 and the diagonal of the next plane are prefetched into
//    registers one plane ahead with evict-first loads.
//
// Per point the epilogue is the grid kernel's: (y - c x)/d, 2 t - w_{k-1},
// store, and the moment dots of the step (doubling <w+,w+>, <w+,w>; direct
// <v0,w+>; + <w0,w0> on the first step).  Partials: block b owns the CS
// columns of slice b % slices of partial row b / slices (fixed order).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "stepargs.cuh"
#include "tma.cuh"

namespace sdb {

struct ZmArgs {
  int nx, ny, nz;
  int n_xt, n_yt, n_zs, ZS;   // tiles in x, y; z segments and planes per segment
  int slices;                 // ldv / CS
  int R;                      // ring slots
  int64_t items;              // n_xt * n_yt * n_zs * slices
  int G;                      // ghost width of the padded blocks (1, or 2 with fused pairs)
  int z_lo, z_hi;             // planes computed: [z_lo, z_hi) (row partition: a slab's planes)
  const double* diag;         // n (unpadded)
  int hint;                   // L2 policies on the TMA loads: 1 = w_{k-1} / v0 boxes evict_first, 2 = x boxes evict_last
  int order, gtiles, sw;      // item order (zm_decode): 0 raster; 1 wave groups of gtiles tiles in strips sw tiles wide
  double wc[27];              // weights, lexicographic (dz, dy, dx); centre unused
};

// Streamed rows (w_{k-1}, v0 reads; w_{k+1} writes): cache-streaming hints.
__device__ __forceinline__ double2 ld_d2_cs(const double* p) {
  double2 r;
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_d2_cs(double* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// Item -> (probe slice, tile, z segment).  Order 0: slice fastest, then x tiles,
// y tiles, z segments.  Order 1: the tiles are numbered in column strips `sw`
// tiles wide (a compact patch instead of a few full rows) and cut into groups
// of `gtiles` (= one wave of the persistent grid); a group runs all its z
// segments before the next group starts, so the blocks in flight share halos
// with each other and a segment's first planes were the previous wave's last.
__device__ __forceinline__ void zm_decode(const ZmArgs& t, int64_t item, int& slice, int& xt, int& yt, int& zs) {
  slice = (int)(item % t.slices);
  int64_t sp = item / t.slices;
  if (t.order == 0) {
    xt = (int)(sp % t.n_xt);
    sp /= t.n_xt;
    yt = (int)(sp % t.n_yt);
    zs = (int)(sp / t.n_yt);
    return;
  }
  const int ntiles = t.n_xt * t.n_yt;
  const int64_t per_group = (int64_t)t.gtiles * t.n_zs;
  const int full = ntiles / t.gtiles;
  int group = (int)(sp / per_group), tig = t.gtiles;
  int64_t r = sp - (int64_t)group * per_group;
  if (group >= full) {
    group = full;
    r = sp - (int64_t)full * per_group;
    tig = ntiles - full * t.gtiles;
  }
  zs = (int)(r / tig);
  const int u = group * t.gtiles + (int)(r % tig);
  const int per_strip = t.sw * t.n_yt;
  const int strip = u / per_strip, within = u % per_strip;
  yt = within / t.sw;
  xt = strip * t.sw + within % t.sw;
}

// Which in-plane positions (dy, dx) a shape reads: bit (dy+1)*3 + (dx+1).
template <int SHAPE>
__host__ __device__ constexpr int zm_plane_mask() {
  int m = 0;
  for (int o = 0; o < GridShape<SHAPE>::NT; ++o)
    m |= 1 << ((GridShape<SHAPE>::dy(o) + 1) * 3 + GridShape<SHAPE>::dx(o) + 1);
  return m;
}

template <int CS, int TX, int TY, int PPT>
struct ZmGeom {
  static constexpr int L = CS / 2;                 // lanes per point (one double2 each)
  static constexpr int NT = TX * TY * L / PPT;     // consumer threads
  static constexpr int GROUPS = NT / L;            // points per pass
  static constexpr int PX = TX + 2, PY = TY + 2;   // halo box extent
  static constexpr int BOX = PY * PX * CS;         // doubles per plane box
  static_assert((TX * TY) % GROUPS == 0, "tile must split evenly over the point groups");
  static_assert(PPT == 1 || (PPT == 2 && TY % 2 == 0), "columns per thread: 1, or 2 (a y pair)");
  static_assert(NT % 32 == 0 && NT <= 1024 - 32, "consumer threads");
};

// Ghost width of the padded blocks [nz][ny+2G][nx+2G][ldv]: 1 for single
// steps, 2 when fused pairs run (their halo-2 boxes are single TMA
// rectangles too); the fused kernel is compiled for kZmGhost.
constexpr int kZmGhost = 2;

// Store w at padded offset dst of point (x, y) and at every periodic ghost
// image of it (x within G of an x face, y of a y face, and the corner).
__device__ __forceinline__ void zm_store_ghosted(double* dst, double2 w, int x, int y, int nx, int ny, int64_t ldv,
                                                 int64_t pstride_y, int G) {
  st_d2_cs(dst, w);
  const int gx = x < G ? nx : (x >= nx - G ? -nx : 0);
  const int gy = y < G ? ny : (y >= ny - G ? -ny : 0);
  if (gx) st_d2_cs(dst + (int64_t)gx * ldv, w);
  if (gy) st_d2_cs(dst + (int64_t)gy * pstride_y, w);
  if (gx && gy) st_d2_cs(dst + (int64_t)gx * ldv + (int64_t)gy * pstride_y, w);
}

// Shared-memory ring slot: the halo box of x = w_k (always), then for output
// planes the interior boxes of w_{k-1} (not on the first step), v0 (direct
// mode after the first step) and the diagonal.
template <int CS, int TX, int TY, int MODE, bool FIRST>
struct ZmSlot {
  static constexpr int XB = (TY + 2) * (TX + 2) * CS;                            // x halo box
  static constexpr int PB = FIRST ? 0 : TY * TX * CS;                            // w_{k-1}
  static constexpr int VB = (MODE == SDB_CHEB_DIRECT && !FIRST) ? TY * TX * CS : 0;  // v0
  static constexpr int DB = TY * TX;                                             // diagonal
  static constexpr int X0 = 0, P0 = (XB + 15) / 16 * 16, V0 = P0 + (PB + 15) / 16 * 16,
                       D0 = V0 + (VB + 15) / 16 * 16;
  static constexpr int DOUBLES = D0 + (DB + 15) / 16 * 16;  // 128-byte aligned pieces
  static constexpr uint32_t HALO_BYTES = XB * 8;
  static constexpr uint32_t FULL_BYTES = (XB + PB + VB + DB) * 8;
};

struct ZmMaps {
  CUtensorMap x, prev, v0, diag;
};

template <int SHAPE, int CS, int TX, int TY, int PPT, int MODE, bool FIRST, bool PUSH>
__global__ void __launch_bounds__(ZmGeom<CS, TX, TY, PPT>::NT + 32, 1)
    cheb_step_zmarch(const __grid_constant__ ZmMaps maps, ZmArgs t, StepArgs a) {
  using G = GridShape<SHAPE>;
  using Z = ZmGeom<CS, TX, TY, PPT>;
  using SL = ZmSlot<CS, TX, TY, MODE, FIRST>;
  constexpr int L = Z::L, NT = Z::NT, GROUPS = Z::GROUPS;
  constexpr int PMASK = zm_plane_mask<SHAPE>();
  extern __shared__ __align__(128) double zsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(zsm + (int64_t)t.R * SL::DOUBLES);
  uint64_t* empty = full + t.R;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < t.R; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();

  const int nx = t.nx, ny = t.ny, nz = t.nz;
  const int64_t pstride_y = (int64_t)(nx + 2 * t.G) * a.ldv;  // padded row of points
  const int64_t pplane = (int64_t)(ny + 2 * t.G) * pstride_y;  // padded plane
  const int64_t G_ = gridDim.x;

  if (tid >= NT) {
    // ---- producer warp: one elected lane streams the plane groups ----
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.x) : "memory");
      // w_{k-1} and v0 are read once per step (evict_first); the x boxes overlap
      // their neighbours' (halo rows, z-segment ends), so they may be kept
      uint64_t pol_once, pol_keep;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_once));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
      const bool once = t.hint & 1, keep = t.hint & 2;
      int s = 0;
      uint32_t use = 0;
      for (int64_t item = blockIdx.x; item < t.items; item += G_) {
        int slice, xt, yt, zs;
        zm_decode(t, item, slice, xt, yt, zs);
        const int zbeg = t.z_lo + zs * t.ZS, zend = min(zbeg + t.ZS, t.z_hi);
        const int c0 = slice * CS, x0 = xt * TX, y0 = yt * TY;
        for (int p = zbeg - 1; p <= zend; ++p) {
          if (use > 0) mbar_wait(empty + s, (use - 1) & 1);
          const int zw = p < 0 ? p + nz : (p >= nz ? p - nz : p);
          const bool outp = p >= zbeg && p < zend;
          double* slot = zsm + (int64_t)s * SL::DOUBLES;
          mbar_expect_tx(full + s, outp ? SL::FULL_BYTES : SL::HALO_BYTES);
          if (keep)
            tma_load_4d_hint(slot + SL::X0, &maps.x, full + s, c0, x0 + t.G - 1, y0 + t.G - 1, zw, pol_keep);
          else
            tma_load_4d(slot + SL::X0, &maps.x, full + s, c0, x0 + t.G - 1, y0 + t.G - 1, zw);
          if (outp) {
            if (once) {
              if (SL::PB) tma_load_4d_hint(slot + SL::P0, &maps.prev, full + s, c0, x0 + t.G, y0 + t.G, p, pol_once);
              if (SL::VB) tma_load_4d_hint(slot + SL::V0, &maps.v0, full + s, c0, x0 + t.G, y0 + t.G, p, pol_once);
            } else {
              if (SL::PB) tma_load_4d(slot + SL::P0, &maps.prev, full + s, c0, x0 + t.G, y0 + t.G, p);
              if (SL::VB) tma_load_4d(slot + SL::V0, &maps.v0, full + s, c0, x0 + t.G, y0 + t.G, p);
            }
            tma_load_3d(slot + SL::D0, &maps.diag, full + s, x0, y0, p);
          }
          if (++s == t.R) {
            s = 0;
            ++use;
          } 
        }
      }
    }
    return;
  }

  // ---- consumer threads ----
  const int q = tid % L, g = tid / L;
  double2 accA = make_double2(0.0, 0.0), accB = accA, accZ = accA;
  int s = 0;           // ring slot of the next plane
  uint32_t phase = 0;  // its full-barrier parity
  int pb_row = -1;     // partial row of this block (fixed slice: gridDim % slices == 0)
  int col0 = 0;
  for (int64_t item = blockIdx.x; item < t.items; item += G_) {
    int slice, xt, yt, zs;
    zm_decode(t, item, slice, xt, yt, zs);
    const int zbeg = t.z_lo + zs * t.ZS, zend = min(zbeg + t.ZS, t.z_hi);
    col0 = slice * CS;
    pb_row = (int)(blockIdx.x / t.slices);
    // this thread's columns: point index g + k*GROUPS of the TX x TY tile
    int cx[PPT], cy[PPT], xo[PPT], io[PPT], dio[PPT];
    int64_t cofs[PPT];  // padded block offset of (z = zbeg, y, x) + column
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      // PPT == 2: the two columns are neighbours in y (rows 2j, 2j+1), so their
      // 3x3 neighbourhoods share a 4x3 window of loads; a warp's points stay
      // consecutive in x (conflict-free 16-byte loads for every CS)
      const int pnt = g + k * GROUPS;
      const int px = PPT == 2 ? g % TX : pnt % TX, py = PPT == 2 ? 2 * (g / TX) + k : pnt / TX;
      cx[k] = xt * TX + px;
      cy[k] = yt * TY + py;
      xo[k] = ((py + 1) * (TX + 2) + (px + 1)) * CS + 2 * q;  // centre in the x halo box
      io[k] = (py * TX + px) * CS + 2 * q;                    // in the interior boxes
      dio[k] = py * TX + px;                                  // in the diagonal box
      cofs[k] = (int64_t)zbeg * pplane + (int64_t)(cy[k] + t.G) * pstride_y + (int64_t)(cx[k] + t.G) * a.ldv + col0 +
                2 * q;
    }
    // rolling accumulators: at plane p, accC = out(p), accN = out(p+1), accP = out(p-1)
    double2 accN[PPT], accC[PPT], accP[PPT];
#pragma unroll
    for (int k = 0; k < PPT; ++k) accN[k] = accC[k] = accP[k] = make_double2(0.0, 0.0);
    double* pn = a.next - 2 * pplane;  // output plane p - 1 (+ cofs), for p = zbeg - 1 first
    int sprev = -1;  // slot of plane p - 1 (this item), released after its epilogue
    double2 xcen[PPT], xcen_prev[PPT];  // x at the columns' own points, planes p and p - 1 (PPT == 2)
#pragma unroll
    for (int k = 0; k < PPT; ++k) xcen[k] = xcen_prev[k] = make_double2(0.0, 0.0);
    for (int p = zbeg - 1; p <= zend; ++p) {
      mbar_wait(full + s, phase);
      const double* slot = zsm + (int64_t)s * SL::DOUBLES;
      const bool outp = p >= zbeg && p < zend;
      // plane p: per column, the 3x3 (or star) neighbourhood into registers,
      // then its terms in lexicographic (dz, dy, dx) order
      if constexpr (PPT == 2) {
        // rows py0-1 .. py0+2 of the halo box, x-1 .. x+1: 12 loads (27-point) or
        // 8 (7-point) serve both columns instead of 18 / 10
        double2 nbw[4][3];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const bool need = (r <= 2 && ((PMASK >> (r * 3 + c)) & 1)) || (r >= 1 && ((PMASK >> ((r - 1) * 3 + c)) & 1));
            if (need)
              nbw[r][c] =
                  *reinterpret_cast<const double2*>(slot + SL::X0 + xo[0] + ((r - 1) * (TX + 2) + (c - 1)) * CS);
          }
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const double dg = outp ? slot[SL::D0 + dio[k]] : 0.0;
          xcen_prev[k] = xcen[k];
          xcen[k] = nbw[1 + k][1];
#pragma unroll
          for (int o = 0; o < G::NT; ++o) {
            const double2 v = nbw[G::dy(o) + 1 + k][G::dx(o) + 1];
            const bool centre = G::dx(o) == 0 && G::dy(o) == 0 && G::dz(o) == 0;
            const double w = centre ? dg : t.wc[o];
            double2& y = G::dz(o) < 0 ? accN[k] : (G::dz(o) == 0 ? accC[k] : accP[k]);
            y.x = fma(w, v.x, y.x);
            y.y = fma(w, v.y, y.y);
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const double dg = outp ? slot[SL::D0 + dio[k]] : 0.0;
          double2 nb[9];
#pragma unroll
          for (int e = 0; e < 9; ++e) {
            if (!((PMASK >> e) & 1)) continue;
            const int dy = e / 3 - 1, dx = e % 3 - 1;
            nb[e] = *reinterpret_cast<const double2*>(slot + SL::X0 + xo[k] + (dy * (TX + 2) + dx) * CS);
          }
#pragma unroll
          for (int o = 0; o < G::NT; ++o) {
            const int e = (G::dy(o) + 1) * 3 + G::dx(o) + 1;
            const double2 v = nb[e];
            const bool centre = G::dx(o) == 0 && G::dy(o) == 0 && G::dz(o) == 0;
            const double w = centre ? dg : t.wc[o];
            double2& y = G::dz(o) < 0 ? accN[k] : (G::dz(o) == 0 ? accC[k] : accP[k]);
            y.x = fma(w, v.x, y.x);
            y.y = fma(w, v.y, y.y);
          }
        }
      }
      // out(p-1) is complete: its operands are in the previous slot
      if (p - 1 >= zbeg) {
        const double* ps = zsm + (int64_t)sprev * SL::DOUBLES;
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const double2 xi = PPT == 2 ? xcen_prev[k] : *reinterpret_cast<const double2*>(ps + SL::X0 + xo[k]);
          const double tx = (accP[k].x - a.c * xi.x) * a.inv_d;
          const double ty = (accP[k].y - a.c * xi.y) * a.inv_d;
          double2 wn;
          if (FIRST) {
            wn = make_double2(tx, ty);
          } else {
            const double2 wp = *reinterpret_cast<const double2*>(ps + SL::P0 + io[k]);
            if (MODE == SDB_CHEB_DIRECT && a.legendre)
              wn = make_double2((a.la * tx - a.lb * wp.x) / a.lc, (a.la * ty - a.lb * wp.y) / a.lc);
            else
              wn = make_double2(2.0 * tx - wp.x, 2.0 * ty - wp.y);
          }
          double* dst = pn + cofs[k];
          zm_store_ghosted(dst, wn, cx[k], cy[k], nx, ny, a.ldv, pstride_y, t.G);  // point + its ghost images
          // plane-range push (row partition, sdb_cheb_step_planes_halo): the
          // first / last plane of the range also lands at the same offset in
          // the neighbour slab's full-size block (peer memory over NVLink)
          // (a separate instantiation: the extra address registers cost the
          // plain step ~10 %, measured)
          if constexpr (PUSH) {
            if (a.halo_lo && p - 1 == t.z_lo)
              zm_store_ghosted(a.halo_lo + (dst - a.next), wn, cx[k], cy[k], nx, ny, a.ldv, pstride_y, t.G);
            if (a.halo_hi && p - 1 == t.z_hi - 1)
              zm_store_ghosted(a.halo_hi + (dst - a.next), wn, cx[k], cy[k], nx, ny, a.ldv, pstride_y, t.G);
          }
          if (MODE == SDB_CHEB_DOUBLING) {
            accA.x += wn.x * wn.x;
            accA.y += wn.y * wn.y;
            accB.x += wn.x * xi.x;
            accB.y += wn.y * xi.y;
          } else {
            const double2 p0 = FIRST ? xi : *reinterpret_cast<const double2*>(ps + SL::V0 + io[k]);
            accA.x += p0.x * wn.x;
            accA.y += p0.y * wn.y;
          }
          if (FIRST) {
            accZ.x += xi.x * xi.x;
            accZ.y += xi.y * xi.y;
          }
        }
      }
      if (sprev >= 0) {  // plane p-1 fully consumed
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + sprev);
      }
      sprev = s;
      if (++s == t.R) {
        s = 0;
        phase ^= 1u;
      }
      pn += pplane;
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        accP[k] = accC[k];
        accC[k] = accN[k];
        accN[k] = make_double2(0.0, 0.0);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + sprev);  // the trailing halo plane
  }

  // ---- block partials: threads with equal q hold the same columns; add them
  // in group order through shared memory (consumers only; fixed order) ----
  asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
  double* red = zsm;  // every slot has been consumed: reuse the ring
  auto partial = [&](double2 v, int slot) {
    red[tid * 2] = v.x;
    red[tid * 2 + 1] = v.y;
    asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
    if (tid < CS && pb_row >= 0) {
      const int qq = tid / 2, comp = tid % 2;
      double sum = 0.0;
      for (int gg = 0; gg < GROUPS; ++gg) sum += red[(gg * L + qq) * 2 + comp];
      a.partials[((int64_t)slot * a.nblocks + pb_row) * a.ldv + col0 + tid] = sum;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
  };
  if (a.slotA >= 0) partial(accA, a.slotA);
  if (MODE == SDB_CHEB_DOUBLING && a.slotB >= 0) partial(accB, a.slotB);
  if (FIRST && a.slot0 >= 0) partial(accZ, a.slot0);
}

// ---- fused pair of doubling-mode steps (temporal blocking) -----------------------------
// One launch advances the recurrence by two steps: x = w_k, prev = w_{k-1} in,
// w_{k+1} (next) and w_{k+2} (next2) out, so per two steps the block is read
// twice and written twice instead of read four times and written twice.
//   stage 1: w_{k+1} on the tile plus a one-point halo ((TX+2) x (TY+2), the
//            halo computed redundantly) from x boxes with a two-point halo;
//            the extended w_{k+1} plane goes to a 3-plane shared ring (and the
//            owned points to HBM);
//   stage 2: w_{k+2} = 2 B w_{k+1} - w_k on the tile from that ring, one plane
//            behind, w_k read back from the x box still in the TMA ring.
// Both stages use the register-rolled z terms of the one-step kernel, so each
// point's FMAs run in the same (dz, dy, dx) order: w_{k+1}, w_{k+2} are
// bit-identical to two one-step launches.  Moments: <w+,w+>, <w+,w> (step k)
// and <w++,w++>, <w++,w+> (step k+1) over owned points, + <w0,w0> if FIRST.
template <int CS, int TX, int TY, bool FIRST>
struct ZmSlot2 {
  static constexpr int XB = (TY + 4) * (TX + 4) * CS;        // x, halo 2
  static constexpr int PB = FIRST ? 0 : (TY + 2) * (TX + 2) * CS;  // w_{k-1}, halo 1
  // diagonal, halo 1: the box starts one point further left (the innermost
  // box coordinate must be 16-byte aligned, else the TMA faults with an
  // illegal instruction), rows of DW >= TX + 3 doubles, 64-byte multiples
  static constexpr int DW = ((TX + 3) + 7) / 8 * 8;
  static constexpr int DB = (TY + 2) * DW;
  static constexpr int X0 = 0, P0 = (XB + 15) / 16 * 16, D0 = P0 + (PB + 15) / 16 * 16;
  static constexpr int DOUBLES = D0 + (DB + 15) / 16 * 16;
  static constexpr uint32_t HALO_BYTES = XB * 8;
  static constexpr uint32_t FULL_BYTES = (XB + PB + DB) * 8;
  static constexpr int W1 = (TY + 2) * (TX + 2) * CS;        // one extended w_{k+1} plane
};

template <int SHAPE, int CS, int TX, int TY, int PPT, bool FIRST>
__global__ void __launch_bounds__(ZmGeom<CS, TX, TY, PPT>::NT + 32, 1)
    cheb_step2_zmarch(const __grid_constant__ ZmMaps maps, ZmArgs t, StepArgs a) {
  using G = GridShape<SHAPE>;
  using Z = ZmGeom<CS, TX, TY, PPT>;
  using SL = ZmSlot2<CS, TX, TY, FIRST>;
  constexpr int L = Z::L, NT = Z::NT, GROUPS = Z::GROUPS;
  constexpr int EX = TX + 2, E1 = (TX + 2) * (TY + 2), E2 = TX * TY;
  constexpr int K1 = (E1 + GROUPS - 1) / GROUPS, K2 = E2 / GROUPS;
  static_assert(E2 % GROUPS == 0, "tile must split evenly over the point groups");
  constexpr int PMASK = zm_plane_mask<SHAPE>();
  extern __shared__ __align__(128) double zsm[];
  double* w1ring = zsm + (int64_t)t.R * SL::DOUBLES;
  uint64_t* full = reinterpret_cast<uint64_t*>(w1ring + 3 * SL::W1);
  uint64_t* empty = full + t.R;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < t.R; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();

  const int nx = t.nx, ny = t.ny, nz = t.nz;
  const int64_t pstride_y = (int64_t)(nx + 2 * kZmGhost) * a.ldv;
  const int64_t pplane = (int64_t)(ny + 2 * kZmGhost) * pstride_y;
  const int64_t G_ = gridDim.x;

  if (tid >= NT) {
    // ---- producer: planes zbeg-2 .. zend+1; w_{k-1} and diag for zbeg-1 .. zend ----
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.x) : "memory");
      int s = 0;
      uint32_t use = 0;
      for (int64_t item = blockIdx.x; item < t.items; item += G_) {
        const int slice = (int)(item % t.slices);
        int64_t sp = item / t.slices;
        const int xt = (int)(sp % t.n_xt);
        sp /= t.n_xt;
        const int yt = (int)(sp % t.n_yt);
        const int zs = (int)(sp / t.n_yt);
        const int zbeg = t.z_lo + zs * t.ZS, zend = min(zbeg + t.ZS, t.z_hi);
        const int c0 = slice * CS, x0 = xt * TX, y0 = yt * TY;
        for (int p = zbeg - 2; p <= zend + 1; ++p) {
          if (use > 0) mbar_wait(empty + s, (use - 1) & 1);
          const int zw = (p % nz + nz) % nz;
          const bool ext = p >= zbeg - 1 && p <= zend;
          double* slot = zsm + (int64_t)s * SL::DOUBLES;
          mbar_expect_tx(full + s, ext ? SL::FULL_BYTES : SL::HALO_BYTES);
          tma_load_4d(slot + SL::X0, &maps.x, full + s, c0, x0 + kZmGhost - 2, y0 + kZmGhost - 2, zw);
          if (ext) {
            if (SL::PB) tma_load_4d(slot + SL::P0, &maps.prev, full + s, c0, x0 + kZmGhost - 1, y0 + kZmGhost - 1, zw);
            tma_load_3d(slot + SL::D0, &maps.diag, full + s, x0 + kZmGhost - 2, y0 + kZmGhost - 1, zw);
          }
          if (++s == t.R) {
            s = 0;
            ++use;
          }
        }
      }
    }
    return;
  }

  // ---- consumers ----
  const int q = tid % L, g = tid / L;
  double2 accA1 = make_double2(0.0, 0.0), accB1 = accA1, accA2 = accA1, accB2 = accA1, accZ = accA1;
  int s = 0;
  uint32_t phase = 0;
  int pb_row = -1, col0 = 0;
  // slot index of a plane relative to the current one (ring order)
  auto slot_back = [&](int back) { return (s - back + 2 * t.R) % t.R; };
  for (int64_t item = blockIdx.x; item < t.items; item += G_) {
    const int slice = (int)(item % t.slices);
    int64_t sp = item / t.slices;
    const int xt = (int)(sp % t.n_xt);
    sp /= t.n_xt;
    const int yt = (int)(sp % t.n_yt);
    const int zs = (int)(sp / t.n_yt);
    const int zbeg = t.z_lo + zs * t.ZS, zend = min(zbeg + t.ZS, t.z_hi);
    col0 = slice * CS;
    pb_row = (int)(blockIdx.x / t.slices);
    const int x0 = xt * TX, y0 = yt * TY;
    // stage-1 columns (extended tile) and stage-2 columns (owned tile)
    int e1[K1];
    bool v1[K1], own1[K1];
    int64_t gofs1[K1];
#pragma unroll
    for (int k = 0; k < K1; ++k) {
      const int pe = g + k * GROUPS;
      v1[k] = pe < E1;
      e1[k] = v1[k] ? pe : 0;
      const int ex = e1[k] % EX - 1, ey = e1[k] / EX - 1;
      own1[k] = v1[k] && ex >= 0 && ex < TX && ey >= 0 && ey < TY;
      gofs1[k] = (int64_t)(y0 + ey + kZmGhost) * pstride_y + (int64_t)(x0 + ex + kZmGhost) * a.ldv + col0 + 2 * q;
    }
    int e2[K2];
    int64_t gofs2[K2];
#pragma unroll
    for (int k = 0; k < K2; ++k) {
      const int pi = g + k * GROUPS;
      e2[k] = (pi / TX + 1) * EX + (pi % TX + 1);  // in extended coordinates
      gofs2[k] = (int64_t)(y0 + pi / TX + kZmGhost) * pstride_y + (int64_t)(x0 + pi % TX + kZmGhost) * a.ldv + col0 +
                 2 * q;
    }
    double2 a1N[K1], a1C[K1], a1P[K1], a2N[K2], a2C[K2], a2P[K2];
#pragma unroll
    for (int k = 0; k < K1; ++k) a1N[k] = a1C[k] = a1P[k] = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < K2; ++k) a2N[k] = a2C[k] = a2P[k] = make_double2(0.0, 0.0);

    for (int p = zbeg - 2; p <= zend + 1; ++p) {
      mbar_wait(full + s, phase);
      const double* sx = zsm + (int64_t)s * SL::DOUBLES;  // plane p
      const bool ext = p >= zbeg - 1 && p <= zend;
      // -- stage 1: x plane p into the w_{k+1} accumulators --
#pragma unroll
      for (int k = 0; k < K1; ++k) {
        if (!v1[k]) continue;
        const int ex = e1[k] % EX, ey = e1[k] / EX;  // +1-shifted extended coords
        const double dg = ext ? sx[SL::D0 + ey * SL::DW + ex + 1] : 0.0;
        const int bo = ((ey + 1) * (TX + 4) + (ex + 1)) * CS + 2 * q;  // centre in the x box
        double2 nb[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) {
          if (!((PMASK >> e) & 1)) continue;
          nb[e] = *reinterpret_cast<const double2*>(sx + SL::X0 + bo + ((e / 3 - 1) * (TX + 4) + (e % 3 - 1)) * CS);
        }
#pragma unroll
        for (int o = 0; o < G::NT; ++o) {
          const double2 v = nb[(G::dy(o) + 1) * 3 + G::dx(o) + 1];
          const bool centre = G::dx(o) == 0 && G::dy(o) == 0 && G::dz(o) == 0;
          const double w = centre ? dg : t.wc[o];
          double2& y = G::dz(o) < 0 ? a1N[k] : (G::dz(o) == 0 ? a1C[k] : a1P[k]);
          y.x = fma(w, v.x, y.x);
          y.y = fma(w, v.y, y.y);
        }
      }
      // -- stage 1 epilogue: w_{k+1}(p-1) on the extended tile --
      const int q1 = p - 1;
      const bool fin1 = q1 >= zbeg - 1 && q1 <= zend;
      if (fin1) {
        const double* s1 = zsm + (int64_t)slot_back(1) * SL::DOUBLES;
        double* w1 = w1ring + (int64_t)((q1 + 3) % 3) * SL::W1;
        const bool own_plane = q1 >= zbeg && q1 < zend;
#pragma unroll
        for (int k = 0; k < K1; ++k) {
          if (!v1[k]) continue;
          const int ex = e1[k] % EX, ey = e1[k] / EX;
          const double2 xi =
              *reinterpret_cast<const double2*>(s1 + SL::X0 + ((ey + 1) * (TX + 4) + (ex + 1)) * CS + 2 * q);
          const double tx = (a1P[k].x - a.c * xi.x) * a.inv_d;
          const double ty = (a1P[k].y - a.c * xi.y) * a.inv_d;
          double2 wn;
          if (FIRST) {
            wn = make_double2(tx, ty);
          } else {
            const double2 wp = *reinterpret_cast<const double2*>(s1 + SL::P0 + e1[k] * CS + 2 * q);
            wn = make_double2(2.0 * tx - wp.x, 2.0 * ty - wp.y);
          }
          *reinterpret_cast<double2*>(w1 + e1[k] * CS + 2 * q) = wn;
          if (own_plane && own1[k]) {
            zm_store_ghosted(a.next + (int64_t)q1 * pplane + gofs1[k], wn, x0 + ex - 1, y0 + ey - 1, nx, ny, a.ldv,
                             pstride_y, kZmGhost);
            accA1.x += wn.x * wn.x;
            accA1.y += wn.y * wn.y;
            accB1.x += wn.x * xi.x;
            accB1.y += wn.y * xi.y;
            if (FIRST) {
              accZ.x += xi.x * xi.x;
              accZ.y += xi.y * xi.y;
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < K1; ++k) {
        a1P[k] = a1C[k];
        a1C[k] = a1N[k];
        a1N[k] = make_double2(0.0, 0.0);
      }
      // the extended w_{k+1}(p-1) plane is complete once every consumer is here
      asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
      // -- stage 2: w_{k+1} plane q1 into the w_{k+2} accumulators --
      if (fin1) {
        const double* w1 = w1ring + (int64_t)((q1 + 3) % 3) * SL::W1;
        const double* s1 = zsm + (int64_t)slot_back(1) * SL::DOUBLES;  // diag of plane q1
        const bool dq = q1 >= zbeg && q1 < zend;
#pragma unroll
        for (int k = 0; k < K2; ++k) {
          const double dg = dq ? s1[SL::D0 + (e2[k] / EX) * SL::DW + e2[k] % EX + 1] : 0.0;
          double2 nb[9];
#pragma unroll
          for (int e = 0; e < 9; ++e) {
            if (!((PMASK >> e) & 1)) continue;
            nb[e] = *reinterpret_cast<const double2*>(w1 + (e2[k] + (e / 3 - 1) * EX + (e % 3 - 1)) * CS + 2 * q);
          }
#pragma unroll
          for (int o = 0; o < G::NT; ++o) {
            const double2 v = nb[(G::dy(o) + 1) * 3 + G::dx(o) + 1];
            const bool centre = G::dx(o) == 0 && G::dy(o) == 0 && G::dz(o) == 0;
            const double w = centre ? dg : t.wc[o];
            double2& y = G::dz(o) < 0 ? a2N[k] : (G::dz(o) == 0 ? a2C[k] : a2P[k]);
            y.x = fma(w, v.x, y.x);
            y.y = fma(w, v.y, y.y);
          }
        }
        // -- stage 2 epilogue: w_{k+2}(q1-1) --
        const int q2 = q1 - 1;
        if (q2 >= zbeg && q2 < zend) {
          const double* w1c = w1ring + (int64_t)((q2 + 3) % 3) * SL::W1;
          const double* s2 = zsm + (int64_t)slot_back(2) * SL::DOUBLES;  // x = w_k of plane q2
#pragma unroll
          for (int k = 0; k < K2; ++k) {
            const int ex = e2[k] % EX, ey = e2[k] / EX;
            const double2 wi = *reinterpret_cast<const double2*>(w1c + e2[k] * CS + 2 * q);
            const double2 xk =
                *reinterpret_cast<const double2*>(s2 + SL::X0 + ((ey + 1) * (TX + 4) + (ex + 1)) * CS + 2 * q);
            const double tx = (a2P[k].x - a.c * wi.x) * a.inv_d;
            const double ty = (a2P[k].y - a.c * wi.y) * a.inv_d;
            const double2 wn = make_double2(2.0 * tx - xk.x, 2.0 * ty - xk.y);
            zm_store_ghosted(a.next2 + (int64_t)q2 * pplane + gofs2[k], wn, x0 + ex - 1, y0 + ey - 1, nx, ny, a.ldv,
                             pstride_y, kZmGhost);
            accA2.x += wn.x * wn.x;
            accA2.y += wn.y * wn.y;
            accB2.x += wn.x * wi.x;
            accB2.y += wn.y * wi.y;
          }
        }
#pragma unroll
        for (int k = 0; k < K2; ++k) {
          a2P[k] = a2C[k];
          a2C[k] = a2N[k];
          a2N[k] = make_double2(0.0, 0.0);
        }
      }
      // plane p-2 is no longer needed
      if (p - 2 >= zbeg - 2) {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + slot_back(2));
      }
      if (++s == t.R) {
        s = 0;
        phase ^= 1u;
      }
    }
    // release the item's last two planes (zend, zend+1)
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(empty + slot_back(2));
      mbar_arrive(empty + slot_back(1));
    }
  }

  asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
  double* red = zsm;
  auto partial = [&](double2 v, int slot) {
    red[tid * 2] = v.x;
    red[tid * 2 + 1] = v.y;
    asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
    if (tid < CS && pb_row >= 0) {
      const int qq = tid / 2, comp = tid % 2;
      double sum = 0.0;
      for (int gg = 0; gg < GROUPS; ++gg) sum += red[(gg * L + qq) * 2 + comp];
      a.partials[((int64_t)slot * a.nblocks + pb_row) * a.ldv + col0 + tid] = sum;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
  };
  if (a.slotA >= 0) partial(accA1, a.slotA);
  if (a.slotB >= 0) partial(accB1, a.slotB);
  if (a.slotA2 >= 0) partial(accA2, a.slotA2);
  if (a.slotB2 >= 0) partial(accB2, a.slotB2);
  if (FIRST && a.slot0 >= 0) partial(accZ, a.slot0);
}

// diagonal (n) -> ghost-padded [nz][ny+2G][nx+2G]
__global__ void zm_pad_diag_kernel(const double* __restrict__ src, int nx, int ny, int nz, double* __restrict__ dst) {
  // (fused pairs only: ghost width kZmGhost)
  const int px = nx + 2 * kZmGhost, py = ny + 2 * kZmGhost;
  const int64_t total = (int64_t)nz * py * px;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int xx = (int)(i % px);
    const int64_t r = i / px;
    const int yy = (int)(r % py);
    const int z = (int)(r / py);
    int x = xx - kZmGhost, y = yy - kZmGhost;
    x = x < 0 ? x + nx : (x >= nx ? x - nx : x);
    y = y < 0 ? y + ny : (y >= ny ? y - ny : y);
    dst[i] = src[((int64_t)z * ny + y) * nx + x];
  }
}

// Probe block (n x ldv) -> ghost-padded block [nz][ny+2G][nx+2G][ldv].
__global__ void zm_pad_kernel(const double* __restrict__ src, int nx, int ny, int nz, int64_t ldv, int G,
                              double* __restrict__ dst) {
  const int64_t pts = (int64_t)nz * (ny + 2 * G) * (nx + 2 * G);
  const int64_t h = ldv / 2;  // double2 per point
  const int64_t total = pts * h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % h, pt = i / h;
    const int xx = (int)(pt % (nx + 2 * G));
    const int64_t r = pt / (nx + 2 * G);
    const int yy = (int)(r % (ny + 2 * G));
    const int z = (int)(r / (ny + 2 * G));
    int x = xx - G, y = yy - G;
    x = x < 0 ? x + nx : (x >= nx ? x - nx : x);
    y = y < 0 ? y + ny : (y >= ny ? y - ny : y);
    const int64_t s = (((int64_t)z * ny + y) * nx + x) * ldv + 2 * c;
    reinterpret_cast<double2*>(dst)[i] = *reinterpret_cast<const double2*>(src + s);
  }
}

// ---- host side ---------------------------------------------------------------------
// Tile configurations (CS probe columns, TX x TY points, PPT columns per thread);
// 256 consumer threads (2 columns each) + 1 producer warp: 9 warps leave up
// to 168 registers per thread.
// zm_plan picks the first that fits; SDB_ZM_CFG overrides it (tuning).
struct ZmCfg {
  int CS, TX, TY, PPT;
};
static constexpr ZmCfg kZmCfgs[] = {
    {8, 16, 8, 2},   // 0: 11.5 KB boxes, halo 1.41x
    {4, 32, 8, 2},   // 1: 10.9 KB, 1.33x
    {8, 32, 4, 2},   // 2: 13.1 KB, 1.59x
    {16, 8, 8, 2},   // 3: 12.8 KB, 1.56x
    {4, 16, 16, 2},  // 4: 10.4 KB, 1.27x
    {8, 8, 8, 2},    // 5: 128 consumer threads (small grids)
    {16, 8, 8, 1},   // 6: 512 consumer threads, one column each
};
constexpr int kZmNumCfgs = (int)(sizeof(kZmCfgs) / sizeof(kZmCfgs[0]));

static int zm_env(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

template <int SHAPE, int CFG, int MODE, bool FIRST>
static const void* zm_kernel(bool push) {
  constexpr ZmCfg c = kZmCfgs[CFG];
  return push ? (const void*)cheb_step_zmarch<SHAPE, c.CS, c.TX, c.TY, c.PPT, MODE, FIRST, true>
              : (const void*)cheb_step_zmarch<SHAPE, c.CS, c.TX, c.TY, c.PPT, MODE, FIRST, false>;
}

template <int SHAPE, int CFG>
static const void* zm_kernel_rt(int mode, bool first, bool push) {
  if (mode == SDB_CHEB_DOUBLING)
    return first ? zm_kernel<SHAPE, CFG, SDB_CHEB_DOUBLING, true>(push)
                 : zm_kernel<SHAPE, CFG, SDB_CHEB_DOUBLING, false>(push);
  return first ? zm_kernel<SHAPE, CFG, SDB_CHEB_DIRECT, true>(push) : zm_kernel<SHAPE, CFG, SDB_CHEB_DIRECT, false>(push);
}

static const void* zm_kernel_for(int shape, int cfg, int mode, bool first, bool push) {
#define SDB_ZM_CFG_CASE(C)                                                                      \
  case C:                                                                                       \
    return shape == SDB_SHAPE_FACE7 ? zm_kernel_rt<SDB_SHAPE_FACE7, C>(mode, first, push)       \
                                    : zm_kernel_rt<SDB_SHAPE_BOX27, C>(mode, first, push);
  switch (cfg) {
    SDB_ZM_CFG_CASE(0)
    SDB_ZM_CFG_CASE(1)
    SDB_ZM_CFG_CASE(2)
    SDB_ZM_CFG_CASE(3)
    SDB_ZM_CFG_CASE(4)
    SDB_ZM_CFG_CASE(5)
    SDB_ZM_CFG_CASE(6)
  }
#undef SDB_ZM_CFG_CASE
  return nullptr;
}

// Host mirror of ZmSlot<...>::DOUBLES.
static int64_t zm_slot_doubles(const ZmCfg& c, int mode, bool first) {
  auto al = [](int64_t v) { return (v + 15) / 16 * 16; };
  const int64_t xb = (int64_t)(c.TY + 2) * (c.TX + 2) * c.CS, ib = (int64_t)c.TY * c.TX * c.CS;
  return al(xb) + (first ? 0 : al(ib)) + ((mode == SDB_CHEB_DIRECT && !first) ? al(ib) : 0) + al((int64_t)c.TY * c.TX);
}

template <int SHAPE, int CFG>
static const void* zm_pair_kernel_rt(bool first) {
  constexpr ZmCfg c = kZmCfgs[CFG];
  return first ? (const void*)cheb_step2_zmarch<SHAPE, c.CS, c.TX, c.TY, c.PPT, true>
               : (const void*)cheb_step2_zmarch<SHAPE, c.CS, c.TX, c.TY, c.PPT, false>;
}

static const void* zm_pair_kernel_for(int shape, int cfg, bool first) {
#define SDB_ZM2_CASE(C)                                                                       \
  case C:                                                                                     \
    return shape == SDB_SHAPE_FACE7 ? zm_pair_kernel_rt<SDB_SHAPE_FACE7, C>(first)            \
                                    : zm_pair_kernel_rt<SDB_SHAPE_BOX27, C>(first);
  switch (cfg) {
    SDB_ZM2_CASE(0)
    SDB_ZM2_CASE(2)
    SDB_ZM2_CASE(3)
    SDB_ZM2_CASE(5)
  }
#undef SDB_ZM2_CASE
  return nullptr;
}

// Host mirror of ZmSlot2<...>::DOUBLES and of the w_{k+1} ring.
static int zm_diag_box_width(int TX) { return ((TX + 3) + 7) / 8 * 8; }
static int64_t zm_slot2_doubles(const ZmCfg& c, bool first) {
  auto al = [](int64_t v) { return (v + 15) / 16 * 16; };
  const int64_t xb = (int64_t)(c.TY + 4) * (c.TX + 4) * c.CS, eb = (int64_t)(c.TY + 2) * (c.TX + 2);
  return al(xb) + (first ? 0 : al(eb * c.CS)) + al((int64_t)(c.TY + 2) * zm_diag_box_width(c.TX));
}
static int64_t zm_w1ring_doubles(const ZmCfg& c) { return 3LL * (c.TY + 2) * (c.TX + 2) * c.CS; }

static bool zm_fits(const ZmCfg& c, int nx, int ny, int64_t ldv) {
  return ldv % c.CS == 0 && nx % c.TX == 0 && ny % c.TY == 0;
}

int zm_plan(const sdb_matrix* m, int64_t ldv, int mode, ZmPlan* out) {
  return zm_plan_range(m, ldv, mode, 0, m->format == SDB_FMT_STENCIL ? m->st.nz : 0, out);
}

int zm_plan_range(const sdb_matrix* m, int64_t ldv, int mode, int64_t z_lo, int64_t z_hi, ZmPlan* out) {
  int leg_;
  mode = split_mode(mode, &leg_);
  ZmPlan p;
  *out = p;
  if (m->format != SDB_FMT_STENCIL || m->zghost) return SDB_OK;
  if (m->shape != SDB_SHAPE_FACE7 && m->shape != SDB_SHAPE_BOX27) return SDB_OK;
  if (mode != SDB_CHEB_DIRECT && mode != SDB_CHEB_DOUBLING) return SDB_OK;
  if (!zm_env("SDB_ZMARCH", 1)) return SDB_OK;
  const int nx = (int)m->st.nx, ny = (int)m->st.ny, nz = (int)m->st.nz;
  if (nx < 2 * kZmGhost || ny < 2 * kZmGhost || nz < 3) return SDB_OK;  // ghost images must not overlap
  if (z_lo < 0 || z_hi > nz || z_lo >= z_hi) return SDB_OK;
  const int nzr = (int)(z_hi - z_lo);  // planes this plan computes
  p.z_lo = (int)z_lo;
  p.z_hi = (int)z_hi;
  int cfg = -1;
  const int forced = zm_env("SDB_ZM_CFG", -1);
  if (forced >= 0 && forced < kZmNumCfgs) {
    if (zm_fits(kZmCfgs[forced], nx, ny, ldv)) cfg = forced;
  } else {
    // measured preference (profiles/r01_zmarch_sweep.txt): 16-column slices of
    // 8x8 tiles, then 8-column slices, then the narrow / small-grid shapes
    static const int pref[] = {3, 0, 2, 1, 4, 5};
    for (int i = 0; i < (int)(sizeof(pref) / sizeof(pref[0])) && cfg < 0; ++i)
      if (zm_fits(kZmCfgs[pref[i]], nx, ny, ldv)) cfg = pref[i];
  }
  if (cfg < 0) return SDB_OK;
  const ZmCfg c = kZmCfgs[cfg];
  p.cfg = cfg;
  p.CS = c.CS;
  p.TX = c.TX;
  p.TY = c.TY;
  const int slices = (int)(ldv / c.CS);
  // ring depth from the largest slot (direct mode after the first step): 7 for
  // the 16-column 8x8 tiles.  Measured (C2 doubling, whose slots would allow
  // 10): R = 6 / 7 / 8 / 10 -> 71.3 / 69.9 / 74.8 / 82.2 us per step -- deeper
  // prefetch runs the TMA further ahead of the neighbouring tiles and loses
  const int64_t slot_max = zm_slot_doubles(c, SDB_CHEB_DIRECT, false);
  const size_t budget = 220 * 1024;
  int R = (int)((budget - 256) / (slot_max * sizeof(double)));
  const int rmax = zm_env("SDB_ZM_R", 8);
  if (R > rmax) R = rmax;
  if (R < 3) return SDB_OK;  // plane p and p-1 are held while p+1 streams in
  p.R = R;
  const int nt = c.TX * c.TY * (c.CS / 2) / c.PPT;
  p.smem = (size_t)R * slot_max * sizeof(double) + 2 * R * sizeof(uint64_t);
  if (p.smem < (size_t)nt * 2 * sizeof(double) + 2 * R * sizeof(uint64_t))
    p.smem = (size_t)nt * 2 * sizeof(double) + 2 * R * sizeof(uint64_t);
  // z segments and persistent grid, chosen together: a block's time is its
  // item count x (ZS + 1) plane iterations (the two halo planes of a segment
  // cost about one output plane), so minimise ceil(items / grid) * (ZS + 1)
  // over the segment count (>= 4 planes per segment) and the grid (a multiple
  // of the slice count, at most one block per SM).  C2 (256 items per
  // segment on 148 SMs): 4 segments, 69.9 us/step, against 73.2 us for the
  // former "~4 items per SM" rule (3 segments, 6 vs 5.2 items per block).
  const int sms = num_sms(m->device);
  const int64_t base = (int64_t)(nx / c.TX) * (ny / c.TY) * slices;
  const int nzs_env = zm_env("SDB_ZM_NZS", 0);
  const int nzs_max = nzs_env > 0 ? nzs_env : (nzr / 4 > 0 ? nzr / 4 : 1);
  const int nzs_min = nzs_env > 0 ? nzs_env : 1;
  int64_t best_g = slices, best_cost = -1;
  for (int nzs = nzs_min; nzs <= nzs_max; ++nzs) {
    const int zs_len = (nzr + nzs - 1) / nzs;
    const int64_t items = base * ((nzr + zs_len - 1) / zs_len);
    for (int64_t g = (sms / slices) * slices; g >= slices; g -= slices) {
      if (g > items) continue;
      const int64_t cost = (items + g - 1) / g * (zs_len + 1);
      if (best_cost < 0 || cost < best_cost) {
        best_cost = cost;
        best_g = g;
        p.ZS = zs_len;
      }
    }
  }
  if (best_cost < 0) {  // fewer items than slices cannot happen (base >= slices); keep a sane plan
    p.ZS = nzr;
    best_g = slices;
  }
  p.n_zs = (nzr + p.ZS - 1) / p.ZS;
  p.items = base * p.n_zs;
  const int eg = zm_env("SDB_ZM_GRID", 0);
  if (eg > 0) best_g = (eg / slices) * slices > 0 ? (eg / slices) * slices : slices;
  if (best_g > p.items) best_g = p.items;
  p.grid = best_g;
  p.nbp = p.grid / slices;
  p.name = "cheb_step_zmarch";
  // fused pairs of steps (doubling mode, opt-in with SDB_ZM_FUSE=1): measured
  // 1.8-2.6x SLOWER per step than single steps on C2/C5 (profiles/
  // r01_zmarch_sweep.txt) -- the per-plane stage barrier serialises the 8
  // consumer warps and the halo recompute adds 56 % stage-1 work, while the
  // single-step kernel already streams at ~85 % of HBM peak
  if (nzr == nz && mode == SDB_CHEB_DOUBLING && zm_env("SDB_ZM_FUSE", 0) && (cfg == 0 || cfg == 2 || cfg == 3 || cfg == 5)) {
    const int64_t slot2 = zm_slot2_doubles(c, false);
    const int64_t ring = zm_w1ring_doubles(c);
    int R2 = (int)((int64_t)(budget - 256 - ring * sizeof(double)) / (slot2 * (int64_t)sizeof(double)));
    const int r2max = zm_env("SDB_ZM_R2", 8);
    if (R2 > r2max) R2 = r2max;
    if (R2 >= 4 && nz >= 4) {
      p.fuse = true;
      p.R2 = R2;
      p.smem2 = (size_t)R2 * slot2 * sizeof(double) + ring * sizeof(double) + 2 * R2 * sizeof(uint64_t);
      p.diag_bytes = sizeof(double) * (size_t)nz * (ny + 2 * kZmGhost) * (nx + 2 * kZmGhost);
      p.diag_bytes = (p.diag_bytes + 255) & ~(size_t)255;
      p.name = "cheb_step2_zmarch";
    }
  }
  p.G = p.fuse ? kZmGhost : 1;
  p.block_bytes = sizeof(double) * (size_t)nz * (ny + 2 * p.G) * (nx + 2 * p.G) * (size_t)ldv;
  p.block_bytes = (p.block_bytes + 255) & ~(size_t)255;
  p.on = true;
  *out = p;
  return SDB_OK;
}

int zm_launch_step(const sdb_matrix* m, const ZmPlan& p, const StepArgs& a, bool first, int mode, cudaStream_t s) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SDB_ECUDA, "cuTensorMapEncodeTiled is not available from the driver");
  const int nx = (int)m->st.nx, ny = (int)m->st.ny, nz = (int)m->st.nz;
  const ZmCfg c = kZmCfgs[p.cfg];
  ZmMaps maps;
  auto encode = [&](CUtensorMap* map, const double* base, int bx, int by) -> int {
    const int px = nx + 2 * p.G, py = ny + 2 * p.G;
    cuuint64_t gdim[4] = {(cuuint64_t)a.ldv, (cuuint64_t)px, (cuuint64_t)py, (cuuint64_t)nz};
    cuuint64_t gstr[3] = {(cuuint64_t)a.ldv * 8, (cuuint64_t)px * a.ldv * 8, (cuuint64_t)py * px * a.ldv * 8};
    cuuint32_t box[4] = {(cuuint32_t)c.CS, (cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), gdim, gstr, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? SDB_OK : fail(SDB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  };
  int rc;
  if ((rc = encode(&maps.x, a.x, c.TX + 2, c.TY + 2))) return rc;
  if ((rc = encode(&maps.prev, a.prev ? a.prev : a.x, c.TX, c.TY))) return rc;
  if ((rc = encode(&maps.v0, a.v0 ? a.v0 : a.x, c.TX, c.TY))) return rc;
  {
    cuuint64_t gdim[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    cuuint64_t gstr[2] = {(cuuint64_t)nx * 8, (cuuint64_t)nx * ny * 8};
    cuuint32_t box[3] = {(cuuint32_t)c.TX, (cuuint32_t)c.TY, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&maps.diag, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(m->diag), gdim, gstr, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SDB_ECUDA, "cuTensorMapEncodeTiled (diag) failed (%d)", (int)r);
  }
  ZmArgs t{};
  t.nx = nx;
  t.ny = ny;
  t.nz = nz;
  t.n_xt = nx / c.TX;
  t.n_yt = ny / c.TY;
  t.n_zs = p.n_zs;
  t.ZS = p.ZS;
  t.slices = (int)(a.ldv / c.CS);
  t.R = p.R;
  t.items = p.items;
  t.G = p.G;
  t.z_lo = p.z_lo;
  t.z_hi = p.z_hi;
  t.diag = m->diag;
  t.order = zm_env("SDB_ZM_ORDER", 0);
  t.gtiles = (int)(p.grid / t.slices) > 0 ? (int)(p.grid / t.slices) : 1;
  t.sw = zm_env("SDB_ZM_SW", 8);
  if (t.sw < 1 || t.n_xt % t.sw != 0) t.sw = t.n_xt;
  t.hint = zm_env("SDB_ZM_HINT", 2);  // measured: x boxes evict_last 69.4 -> 68.6 us (C2), 2427 -> 2392 us (C5)
  for (int o = 0; o < 27; ++o) t.wc[o] = o < m->nterms ? m->term_w_host[o] : 0.0;
  StepArgs aa = a;
  aa.nblocks = p.nbp;
  const void* fn = zm_kernel_for(m->shape, p.cfg, mode, first, a.halo_lo != nullptr || a.halo_hi != nullptr);
  if (!fn) return fail(SDB_EUNSUPPORTED, "no z-march kernel for configuration %d", p.cfg);
  size_t smem = (size_t)p.R * zm_slot_doubles(c, mode, first) * sizeof(double) + 2 * p.R * sizeof(uint64_t);
  const int nt = c.TX * c.TY * (c.CS / 2) / c.PPT;
  if (smem < (size_t)nt * 2 * sizeof(double) + 2 * p.R * sizeof(uint64_t))
    smem = (size_t)nt * 2 * sizeof(double) + 2 * p.R * sizeof(uint64_t);
  SDB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* args[] = {(void*)&maps, (void*)&t, (void*)&aa};
  SDB_CUDA(launch_maybe_pdl(fn, dim3((unsigned)p.grid), dim3(nt + 32), args, smem, s));
  return SDB_OK;
}

int zm_launch_pair(const sdb_matrix* m, const ZmPlan& p, const StepArgs& a, const double* diag_padded, bool first,
                   cudaStream_t s) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SDB_ECUDA, "cuTensorMapEncodeTiled is not available from the driver");
  const int nx = (int)m->st.nx, ny = (int)m->st.ny, nz = (int)m->st.nz;
  const int px = nx + 2 * kZmGhost, py = ny + 2 * kZmGhost;
  const ZmCfg c = kZmCfgs[p.cfg];
  ZmMaps maps;
  auto encode4 = [&](CUtensorMap* map, const double* base, int bx, int by) -> int {
    cuuint64_t gdim[4] = {(cuuint64_t)a.ldv, (cuuint64_t)px, (cuuint64_t)py, (cuuint64_t)nz};
    cuuint64_t gstr[3] = {(cuuint64_t)a.ldv * 8, (cuuint64_t)px * a.ldv * 8, (cuuint64_t)py * px * a.ldv * 8};
    cuuint32_t box[4] = {(cuuint32_t)c.CS, (cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), gdim, gstr, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? SDB_OK : fail(SDB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  };
  int rc;
  if ((rc = encode4(&maps.x, a.x, c.TX + 4, c.TY + 4))) return rc;
  if ((rc = encode4(&maps.prev, a.prev ? a.prev : a.x, c.TX + 2, c.TY + 2))) return rc;
  maps.v0 = maps.prev;
  {
    cuuint64_t gdim[3] = {(cuuint64_t)px, (cuuint64_t)py, (cuuint64_t)nz};
    cuuint64_t gstr[2] = {(cuuint64_t)px * 8, (cuuint64_t)px * py * 8};
    cuuint32_t box[3] = {(cuuint32_t)zm_diag_box_width(c.TX), (cuuint32_t)(c.TY + 2), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&maps.diag, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(diag_padded), gdim, gstr,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SDB_ECUDA, "cuTensorMapEncodeTiled (padded diag) failed (%d)", (int)r);
  }
  ZmArgs t{};
  t.nx = nx;
  t.ny = ny;
  t.nz = nz;
  t.n_xt = nx / c.TX;
  t.n_yt = ny / c.TY;
  t.n_zs = p.n_zs;
  t.ZS = p.ZS;
  t.slices = (int)(a.ldv / c.CS);
  t.R = p.R2;
  t.items = p.items;
  t.z_lo = 0;
  t.z_hi = nz;
  t.diag = m->diag;
  for (int o = 0; o < 27; ++o) t.wc[o] = o < m->nterms ? m->term_w_host[o] : 0.0;
  StepArgs aa = a;
  aa.nblocks = p.nbp;
  const void* fn = zm_pair_kernel_for(m->shape, p.cfg, first);
  if (!fn) return fail(SDB_EUNSUPPORTED, "no fused z-march kernel for configuration %d", p.cfg);
  const size_t smem = (size_t)p.R2 * zm_slot2_doubles(c, first) * sizeof(double) +
                      zm_w1ring_doubles(c) * sizeof(double) + 2 * p.R2 * sizeof(uint64_t);
  SDB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int nt = c.TX * c.TY * (c.CS / 2) / c.PPT;
  void* args[] = {(void*)&maps, (void*)&t, (void*)&aa};
  SDB_CUDA(launch_maybe_pdl(fn, dim3((unsigned)p.grid), dim3(nt + 32), args, smem, s));
  return SDB_OK;
}

int zm_pad_diag(const sdb_matrix* m, double* padded, cudaStream_t s) {
  const int nx = (int)m->st.nx, ny = (int)m->st.ny, nz = (int)m->st.nz;
  const int64_t total = (int64_t)nz * (ny + 2 * kZmGhost) * (nx + 2 * kZmGhost);
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = 8LL * num_sms(m->device);
  if (blocks > cap) blocks = cap;
  zm_pad_diag_kernel<<<(unsigned)blocks, 256, 0, s>>>(m->diag, nx, ny, nz, padded);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int zm_pad(const sdb_matrix* m, const ZmPlan& p, const double* probes, int64_t ldv, double* padded, cudaStream_t s) {
  const int nx = (int)m->st.nx, ny = (int)m->st.ny, nz = (int)m->st.nz;
  const int64_t total = (int64_t)nz * (ny + 2 * p.G) * (nx + 2 * p.G) * (ldv / 2);
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = 8LL * num_sms(m->device);
  if (blocks > cap) blocks = cap;
  zm_pad_kernel<<<(unsigned)blocks, 256, 0, s>>>(probes, nx, ny, nz, ldv, p.G, padded);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

}  // namespace sdb
