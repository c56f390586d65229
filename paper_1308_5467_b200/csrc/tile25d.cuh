// tile25d.cuh — 2.5-D blocked Chebyshev step for periodic 7-point / 27-point
// grids (doubling mode), included by cheb.cu after GridShape.
//
// Why: with 64 probes a grid point's row of the block is 512 B, so the +-ny
// and +-nz neighbour lines do not fit in L1 and the row-panel kernel moves
// ~3x the DRAM traffic through L2, capping it at the L2 throughput limit
// (profiles/r01_ncu_grid_face7_c2.txt).  Here each block owns a column
// slice (CS probes) of a TX x TY tile of the (x, y) plane and sweeps z over a
// segment of planes.  The (TY+2) x (TX+2) halo tiles of planes z-1, z, z+1
// sit in a 4-slot shared-memory ring; plane z+2 and w_{k-1} / diag of plane
// z+1 are prefetched with cp.async (LDGSTS) while plane z is computed, so
// every neighbour read is a shared-memory load and each x row crosses L2
// about (TY+2)/TY * (ZS+2)/ZS times.
//
// Arithmetic per point is the grid kernel's: terms in lexicographic (dz,dy,dx)
// order (sorted-column order), then (y - c x)/d, 2 t - w_{k-1}, store, and the
// doubling dots <w+,w+>, <w+,w> (+ <w0,w0> on the first step).
#pragma once
// (included inside namespace sdb)

struct TileArgs {
  int nx, ny, nz;
  int TX;                // tile extent in x (<= kTileMaxX)
  int n_xt, n_yt, n_zs;  // tiles in x, y and z segments
  int ZS;                // planes per z segment
  int slices;            // column slices (ldv / CS)
  int zghost;            // z-slab: no z wrap (ghost planes next to the slab)
  const double* diag;
  double wc[27];         // weights in lexicographic (dz,dy,dx) order; centre unused
};

constexpr int kTileMaxX = 64;
#ifndef SDB_TILE_THREADS
#define SDB_TILE_THREADS 256
#endif
constexpr int kTileThreads = SDB_TILE_THREADS;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16_stream(void* smem, const void* gmem) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Ring of R = 3 + PD plane slots (z-1, z, z+1 in use, PD planes in flight)
// and PD + 1 slots for w_{k-1} / diag.
template <int CS, int TY, int PD>
struct TileSmem {
  static constexpr int PX = kTileMaxX + 2;          // padded tile width
  static constexpr int R = 3 + PD;                  // plane slots
  static constexpr int RP = PD + 1;                 // prev/diag slots
  static constexpr int PLANE = (TY + 2) * PX * CS;  // doubles per plane slot
  static constexpr int PREV = TY * kTileMaxX * CS;  // doubles per prev slot
  static constexpr int DIAG = TY * kTileMaxX;       // doubles per diag slot
  static constexpr size_t bytes = sizeof(double) * (R * PLANE + RP * PREV + RP * DIAG);
};

template <int SHAPE, int CS, int TY, int PD, bool FIRST>
__global__ void __launch_bounds__(kTileThreads, 1) cheb_step_tile(TileArgs t, StepArgs a) {
  using G = GridShape<SHAPE>;
  using SM = TileSmem<CS, TY, PD>;
  constexpr int L = CS / 2;                 // lanes per point (one double2 each)
  constexpr int GROUPS = kTileThreads / L;  // points per block iteration
  constexpr int CH = CS / 2;                // 16-byte chunks per point slice
  extern __shared__ __align__(16) double tsm[];
  double* planes = tsm;
  double* prevb = tsm + SM::R * SM::PLANE;
  double* diagb = prevb + SM::RP * SM::PREV;
  pdl_wait();
  pdl_trigger();

  // slice fastest: the CS-column slices of one tile run side by side, so each
  // x row is fetched from DRAM once and its other slices hit in L2
  const int bid = blockIdx.x / t.slices;
  const int zs = bid % t.n_zs;
  const int rest = bid / t.n_zs;
  const int yt = rest % t.n_yt, xt = rest / t.n_yt;
  const int x0 = xt * t.TX, y0 = yt * TY;
  const int tx_n = min(t.TX, t.nx - x0), ty_n = min(TY, t.ny - y0);
  const int zbeg = zs * t.ZS, zend = min(zbeg + t.ZS, t.nz);
  const int col0 = (blockIdx.x % t.slices) * CS;  // this block's probe columns [col0, col0 + CS)
  const int tid = threadIdx.x;
  const int g = tid / L, q = tid % L;
  const uint64_t pol = policy_evict_first();
  const int nx = t.nx, ny = t.ny, nz = t.nz;

  // Per-thread copy tables, built once: each plane / prev copy is then one
  // address IMAD + one cp.async per 16-byte chunk.
  constexpr int NCH = ((TY + 2) * SM::PX * CH + kTileThreads - 1) / kTileThreads;  // plane chunks / thread
  constexpr int NPC = (TY * kTileMaxX * CH + kTileThreads - 1) / kTileThreads;     // prev chunks / thread
  constexpr int NPT = (TY * kTileMaxX + GROUPS - 1) / GROUPS;                       // points / thread
  const int64_t plane_rows = (int64_t)nx * ny;
  int pl_smem[NCH], pl_row[NCH];
  {
    const int W = tx_n + 2, H = ty_n + 2;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const int i = tid + k * kTileThreads;
      pl_smem[k] = -1;
      pl_row[k] = 0;
      if (i < H * W * CH) {
        const int c = i % CH, p = i / CH;
        const int ix = p % W, iy = p / W;
        int x = x0 - 1 + ix, y = y0 - 1 + iy;
        x = x < 0 ? x + nx : (x >= nx ? x - nx : x);
        y = y < 0 ? y + ny : (y >= ny ? y - ny : y);
        pl_smem[k] = (iy * SM::PX + ix) * CS + 2 * c;
        pl_row[k] = (y * nx + x) * (int)(a.ldv / 2) + c;  // in 16-byte units within the plane
      }
    }
  }
  int pv_smem[NPC], pv_row[NPC];
#pragma unroll
  for (int k = 0; k < NPC; ++k) {
    const int i = tid + k * kTileThreads;
    pv_smem[k] = -1;
    pv_row[k] = 0;
    if (i < ty_n * tx_n * CH) {
      const int c = i % CH, p = i / CH;
      const int ix = p % tx_n, iy = p / tx_n;
      pv_smem[k] = (iy * kTileMaxX + ix) * CS + 2 * c;
      pv_row[k] = ((y0 + iy) * nx + (x0 + ix)) * (int)(a.ldv / 2) + c;
    }
  }
  const double2* xg = reinterpret_cast<const double2*>(a.x + col0);
  const double2* pg = reinterpret_cast<const double2*>(a.prev + col0);
  const int64_t plane_units = plane_rows * (a.ldv / 2);  // 16-byte units per plane
  auto load_plane = [&](int z) {
    const int zs_ = z;  // ring slot follows the unwrapped plane index
    if (!t.zghost) z = z < 0 ? z + nz : (z >= nz ? z - nz : z);
    double* dst = planes + (size_t)(((zs_ % SM::R) + SM::R) % SM::R) * SM::PLANE;
    const double2* src = xg + (int64_t)z * plane_units;
#pragma unroll
    for (int k = 0; k < NCH; ++k)
      if (pl_smem[k] >= 0) cp_async16(dst + pl_smem[k], src + pl_row[k]);
  };
  auto load_prev_diag = [&](int z) {
    const int slot = z % SM::RP;
    double* pd = prevb + (size_t)slot * SM::PREV;
    double* dd = diagb + (size_t)slot * SM::DIAG;
    if (!FIRST) {
      const double2* src = pg + (int64_t)z * plane_units;
#pragma unroll
      for (int k = 0; k < NPC; ++k)
        if (pv_smem[k] >= 0) cp_async16_stream(pd + pv_smem[k], src + pv_row[k]);
    }
    for (int p = tid; p < ty_n * tx_n; p += kTileThreads) {
      const int ix = p % tx_n, iy = p / tx_n;
      cp_async8(dd + iy * kTileMaxX + ix, t.diag + (int64_t)z * plane_rows + (y0 + iy) * nx + (x0 + ix));
    }
  };
  // this thread's points of a plane
  int pt_ix[NPT], pt_iy[NPT];
#pragma unroll
  for (int k = 0; k < NPT; ++k) {
    const int p = g + k * GROUPS;
    pt_ix[k] = -1;
    pt_iy[k] = 0;
    if (p < tx_n * ty_n) {
      pt_ix[k] = p % tx_n;
      pt_iy[k] = p / tx_n;
    }
  }

  double2 accA = make_double2(0.0, 0.0), accB = accA, accZ = accA;
  // prologue: planes zbeg-1 .. zbeg+1 and prev/diag of zbeg (group 0), then
  // PD-1 more groups so PD groups are in flight when plane zbeg is computed
  if (zbeg < zend) {
    load_plane(zbeg - 1);
    load_plane(zbeg);
    load_plane(zbeg + 1);
    load_prev_diag(zbeg);
  }
  cp_async_commit();
  for (int j = 1; j < PD; ++j) {
    if (zbeg + j < zend) {
      load_plane(zbeg + 1 + j);
      load_prev_diag(zbeg + j);
    }
    cp_async_commit();
  }
  for (int z = zbeg; z < zend; ++z) {
    // group for plane z+PD (+1 halo) and prev/diag of plane z+PD
    if (z + PD < zend) {
      load_plane(z + PD + 1);
      load_prev_diag(z + PD);
    }
    cp_async_commit();
    cp_async_wait<PD>();
    __syncthreads();
    const double* pz[3] = {planes + (size_t)((z - 1 + SM::R) % SM::R) * SM::PLANE,
                           planes + (size_t)(z % SM::R) * SM::PLANE, planes + (size_t)((z + 1) % SM::R) * SM::PLANE};
    const double* pd = prevb + (size_t)(z % SM::RP) * SM::PREV;
    const double* dd = diagb + (size_t)(z % SM::RP) * SM::DIAG;
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
      const int ix = pt_ix[k], iy = pt_iy[k];
      if (ix < 0) continue;
      const double dg = dd[iy * kTileMaxX + ix];
      double2 y = make_double2(0.0, 0.0);
#pragma unroll
      for (int o = 0; o < G::NT; ++o) {
        const double* src = pz[G::dz(o) + 1] +
                            ((size_t)(iy + 1 + G::dy(o)) * SM::PX + (ix + 1 + G::dx(o))) * CS + 2 * q;
        const double2 xv = *reinterpret_cast<const double2*>(src);
        const double w = (G::dx(o) == 0 && G::dy(o) == 0 && G::dz(o) == 0) ? dg : t.wc[o];
        y.x = fma(w, xv.x, y.x);
        y.y = fma(w, xv.y, y.y);
      }
      const double2 xi =
          *reinterpret_cast<const double2*>(pz[1] + ((size_t)(iy + 1) * SM::PX + (ix + 1)) * CS + 2 * q);
      const double tx = (y.x - a.c * xi.x) * a.inv_d;
      const double ty = (y.y - a.c * xi.y) * a.inv_d;
      double2 wn;
      if (FIRST) {
        wn = make_double2(tx, ty);
      } else {
        const double2 wp = *reinterpret_cast<const double2*>(pd + ((size_t)iy * kTileMaxX + ix) * CS + 2 * q);
        wn = make_double2(2.0 * tx - wp.x, 2.0 * ty - wp.y);
      }
      const int64_t row = (int64_t)z * plane_rows + (y0 + iy) * nx + (x0 + ix);
      st_d2_once(a.next + row * a.ldv + col0 + 2 * q, wn, pol);
      halo_push(a, row, col0 + 2 * q, wn);
      accA.x += wn.x * wn.x;
      accA.y += wn.y * wn.y;
      accB.x += wn.x * xi.x;
      accB.y += wn.y * xi.y;
      if (FIRST) {
        accZ.x += xi.x * xi.x;
        accZ.y += xi.y * xi.y;
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  // block partials for this block's CS columns: lanes with equal q hold the
  // same columns; sum threads in index order through shared memory.
  __syncthreads();
  double* red = tsm;  // reuse the ring
  auto partial = [&](double2 v, int slot) {
    red[tid * 2] = v.x;
    red[tid * 2 + 1] = v.y;
    __syncthreads();
    if (tid < CS) {
      const int qq = tid / 2, comp = tid % 2;
      double s = 0.0;
      for (int gg = 0; gg < GROUPS; ++gg) s += red[(gg * L + qq) * 2 + comp];
      a.partials[((int64_t)slot * a.nblocks + bid) * a.ldv + col0 + tid] = s;
    }
    __syncthreads();
  };
  if (a.slotA >= 0) partial(accA, a.slotA);
  if (a.slotB >= 0) partial(accB, a.slotB);
  if (FIRST && a.slot0 >= 0) partial(accZ, a.slot0);
}

