// resident.cu — cluster-resident Chebyshev recurrence for small CSR matrices
// (BASELINE config 1: the 100 x 100 Laplacian, n = 1e4, 20 probes).
//
// Reference hot loop: kpm.py:96-107 (direct), kpm.py:174-189 (product formula),
// kpm.py:110-124 (Legendre) with B x = (A x - c x)/d (matrix.py:125-126).
//
// Why a separate path.  A problem this small is latency-bound under one launch
// per recurrence step: each step is a chain of dependent L2 round trips plus a
// kernel boundary, 4.6 us per step with PDL-chained launches, against 0.8 us
// for its 5 MB of traffic.  Here the whole recurrence runs in ONE launch:
//   * a thread-block cluster (up to 16 CTAs, one per SM) owns PC probe columns
//     of the block; CTA r of the cluster owns rows [r R, (r+1) R) and keeps
//     w_k and w_{k-1} (w_{k+1} overwrites it in place; v0 too in direct mode)
//     for them in shared memory, with its slice of the CSR matrix (values and
//     columns pre-translated to (owner CTA, local row));
//   * a gathered x row comes from the CTA's own shared memory or, through
//     distributed shared memory (mapa + ld.shared::cluster), from the owning
//     CTA's; rows accumulate in CSR storage order (csr_matvec order);
//   * one cluster barrier per step (release/acquire) publishes w_{k+1} and
//     retires the reads of w_k; nothing else synchronises: the moment dots are
//     reduced over a warp's rows by shuffles (fixed tree) and each warp stores
//     its partial row to [(M+1)][CL x warps][ldv]; K2 sums them in fixed order.
// Clusters are independent (different probe columns), so the grid is
// (clusters x CL) CTAs with no grid-wide barrier.
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "stepargs.cuh"

namespace sdb {

constexpr int kResThreads = 1024;
constexpr int kResWarps = kResThreads / 32;
constexpr int kResLocalBits = 24;  // packed column: (owner << 24) | local row

struct ResArgs {
  const int32_t* rowptr;
  const int32_t* colidx;
  const double* vals;
  const double* probes;  // n x ldv
  double* partials;      // [(degree+1)][CL * kResWarps][ldv]
  double c, inv_d;
  int64_t n, ldv;
  int R;                 // rows per CTA
  float inv_R;
  int nnz_cap;           // CSR entries staged per CTA
  int steps, degree;
  int legendre;
  int diag;              // timing diagnostics (SDB_RES_DIAG; wrong results): 1 CTA-scope fence + relaxed
                         // barrier, 2 no row loop, 4 no barrier
};

__device__ __forceinline__ uint32_t res_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t res_cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void res_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void res_cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void res_cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void res_cluster_sync_diag(int diag) {
  if (diag & 4) {
    __syncthreads();
  } else if (diag & 1) {
    asm volatile("fence.acq_rel.cta;\n\tbarrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
  } else {
    res_cluster_sync();
  }
}
__device__ __forceinline__ double2 res_ld_remote(uint32_t local_saddr, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_saddr), "r"(rank));
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(ra) : "memory");
  return v;
}

__device__ __forceinline__ double2 res_lds(uint32_t saddr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(saddr) : "memory");
  return v;
}
__device__ __forceinline__ void res_sts(uint32_t saddr, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(saddr), "d"(v.x), "d"(v.y) : "memory");
}

// sum over the lanes of a warp that hold the same column pair (lane % LPR)
template <int LPR>
__device__ __forceinline__ double2 res_warp_sum(double2 v) {
#pragma unroll
  for (int off = 16; off >= LPR; off >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
  }
  return v;
}

// LPR lanes per row (2 probe columns each): the cluster owns PC = 2 LPR columns.
template <int LPR, int MODE>
__global__ void __launch_bounds__(kResThreads, 1) cheb_resident(ResArgs a) {
  constexpr int PC = 2 * LPR;
  constexpr int NBUF = MODE == SDB_CHEB_DIRECT ? 3 : 2;
  extern __shared__ __align__(16) double rsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = tid % LPR, rslot = tid / LPR;
  constexpr int RS = kResThreads / LPR;
  const uint32_t rank = res_cluster_rank(), CL = res_cluster_size();
  const int cluster = blockIdx.x / CL;
  const int64_t col = (int64_t)cluster * PC + 2 * q;
  const bool colok = col < a.ldv;
  const int R = a.R;
  const int64_t row0 = (int64_t)rank * R;
  const int nrows = (int)(a.n - row0 < R ? (a.n - row0 > 0 ? a.n - row0 : 0) : R);
  double* buf0 = rsm;
  double* buf1 = rsm + (size_t)R * PC;
  double* bufv = rsm + 2 * (size_t)R * PC;  // direct mode: v0
  double* svals = rsm + (size_t)NBUF * R * PC;
  int32_t* scols = reinterpret_cast<int32_t*>(svals + a.nnz_cap);
  int32_t* srptr = scols + a.nnz_cap;  // nrows + 1 local offsets

  // ---- stage this CTA's rows: probes, CSR slice with translated columns ----
  const int32_t e0 = nrows > 0 ? a.rowptr[row0] : 0;
  const int32_t e1 = nrows > 0 ? a.rowptr[row0 + nrows] : 0;
  // (the staging loops run once: kept rolled, a cold kernel pays DRAM latency per instruction line)
#pragma unroll 1
  for (int r = tid; r <= nrows; r += kResThreads) srptr[r] = (nrows > 0 ? a.rowptr[row0 + r] : 0) - e0;
#pragma unroll 1
  for (int e = tid; e < e1 - e0; e += kResThreads) {
    const int32_t cj = a.colidx[e0 + e];
    // owner = cj / R by a float estimate, corrected to the exact quotient (cj < 2^24)
    int o = __float2int_rd((float)cj * a.inv_R);
    int l = cj - o * R;
    if (l >= R) {
      ++o;
      l -= R;
    } else if (l < 0) {
      --o;
      l += R;
    }
    scols[e] = (o << kResLocalBits) | l;
    svals[e] = a.vals[e0 + e];
  }
#pragma unroll 1
  for (int r = rslot; r < nrows; r += RS) {
    double2 p = make_double2(0.0, 0.0);
    if (colok) p = *reinterpret_cast<const double2*>(a.probes + (row0 + r) * a.ldv + col);
    *reinterpret_cast<double2*>(buf0 + (size_t)r * PC + 2 * q) = p;
    if (MODE == SDB_CHEB_DIRECT) *reinterpret_cast<double2*>(bufv + (size_t)r * PC + 2 * q) = p;
  }
  res_cluster_sync();

  const int nblocks = (int)CL * kResWarps;
  const int prow = (int)rank * kResWarps + warp;
  auto store_partial = [&](double2 v, int slot) {
    if (slot >= 0 && lane < LPR && colok)
      *reinterpret_cast<double2*>(a.partials + ((size_t)slot * nblocks + prow) * a.ldv + col) = v;
  };
  // A step's warp sums are stored at the top of the NEXT step: the cluster
  // barrier's release fence waits for a thread's outstanding global stores, so
  // stores issued right before it would put their DRAM round trip on the
  // critical path of every step; issued a step early they have drained.
  double2 pendA = make_double2(0.0, 0.0), pendB = pendA;
  int pslotA = -1, pslotB = -1;

  // shared-window addresses of this lane's 16 bytes of row 0 of each buffer
  uint32_t cur_s = (uint32_t)__cvta_generic_to_shared(buf0) + 16u * q;
  uint32_t oth_s = (uint32_t)__cvta_generic_to_shared(buf1) + 16u * q;
  const uint32_t v0_s = (uint32_t)__cvta_generic_to_shared(bufv) + 16u * q;
  constexpr uint32_t ROWB = PC * 8;
  for (int k = 0; k < a.steps; ++k) {
    store_partial(pendA, pslotA);  // the previous step's sums
    store_partial(pendB, pslotB);
    double2 accA = make_double2(0.0, 0.0), accB = accA, accZ = accA;
    const double la = (double)(2 * k + 1), lb = (double)k, lc = (double)k + 1.0;
    // two rows per iteration (r, r + RS): independent gather chains in flight
#pragma unroll 1
    for (int r0 = rslot; r0 < ((a.diag & 2) ? 0 : nrows); r0 += 2 * RS) {
      const int r1 = r0 + RS;
      const bool ok1 = r1 < nrows;
      const int eb0 = srptr[r0], n0 = srptr[r0 + 1] - eb0;
      const int eb1 = ok1 ? srptr[r1] : 0, n1 = ok1 ? srptr[r1 + 1] - eb1 : 0;
      double2 y0 = make_double2(0.0, 0.0), y1 = y0;
      const int nmax = n0 > n1 ? n0 : n1;
#pragma unroll 2
      for (int i = 0; i < nmax; ++i) {
        if (i < n0) {
          const int32_t pc = scols[eb0 + i];
          const double av = svals[eb0 + i];
          const uint32_t o = (uint32_t)pc >> kResLocalBits, l = (uint32_t)pc & ((1u << kResLocalBits) - 1);
          const double2 xv = o == rank ? res_lds(cur_s + l * ROWB) : res_ld_remote(cur_s + l * ROWB, o);
          y0.x = fma(av, xv.x, y0.x);
          y0.y = fma(av, xv.y, y0.y);
        }
        if (i < n1) {
          const int32_t pc = scols[eb1 + i];
          const double av = svals[eb1 + i];
          const uint32_t o = (uint32_t)pc >> kResLocalBits, l = (uint32_t)pc & ((1u << kResLocalBits) - 1);
          const double2 xv = o == rank ? res_lds(cur_s + l * ROWB) : res_ld_remote(cur_s + l * ROWB, o);
          y1.x = fma(av, xv.x, y1.x);
          y1.y = fma(av, xv.y, y1.y);
        }
      }
      auto finish = [&](int r, double2 y) {
        const double2 xi = res_lds(cur_s + (uint32_t)r * ROWB);
        // t = (A x - c x)/d (matrix.py:126); w+ = t (k = 0), 2 t - w- (kpm.py:105) or the Legendre update
        const double tx = (y.x - a.c * xi.x) * a.inv_d, ty = (y.y - a.c * xi.y) * a.inv_d;
        const uint32_t wslot = oth_s + (uint32_t)r * ROWB;
        double2 wn;
        if (k == 0) {
          wn = make_double2(tx, ty);
        } else {
          const double2 wp = res_lds(wslot);
          if (MODE == SDB_CHEB_DIRECT && a.legendre)
            wn = make_double2((la * tx - lb * wp.x) / lc, (la * ty - lb * wp.y) / lc);
          else
            wn = make_double2(2.0 * tx - wp.x, 2.0 * ty - wp.y);
        }
        res_sts(wslot, wn);
        if (MODE == SDB_CHEB_DOUBLING) {
          accA.x += wn.x * wn.x;
          accA.y += wn.y * wn.y;
          accB.x += wn.x * xi.x;
          accB.y += wn.y * xi.y;
        } else {
          const double2 p0 = k == 0 ? xi : res_lds(v0_s + (uint32_t)r * ROWB);
          accA.x += p0.x * wn.x;
          accA.y += p0.y * wn.y;
        }
        if (k == 0) {
          accZ.x += xi.x * xi.x;
          accZ.y += xi.y * xi.y;
        }
      };
      finish(r0, y0);
      if (ok1) finish(r1, y1);
    }
    // w_{k+1} complete everywhere, every remote read of w_k retired: arrive now,
    // sum the step's dots (registers only) while the other CTAs arrive, then wait
    if (a.diag)
      res_cluster_sync_diag(a.diag);
    else
      res_cluster_arrive();
    accA = res_warp_sum<LPR>(accA);
    if (MODE == SDB_CHEB_DOUBLING) accB = res_warp_sum<LPR>(accB);
    if (k == 0) store_partial(res_warp_sum<LPR>(accZ), 0);
    pendA = accA;
    pendB = accB;
    if (MODE == SDB_CHEB_DOUBLING) {
      pslotA = 2 * k + 2 <= a.degree ? 2 * k + 2 : -1;
      pslotB = 2 * k + 1 <= a.degree ? 2 * k + 1 : -1;
    } else {
      pslotA = k + 1;
    }
    if (!a.diag) res_cluster_wait();
    const uint32_t t = cur_s;
    cur_s = oth_s;
    oth_s = t;
  }
  store_partial(pendA, pslotA);
  store_partial(pendB, pslotB);
}

static bool res_env_enabled() {
  const char* e = getenv("SDB_RESIDENT");
  return !(e && e[0] == '0');
}

template <int MODE>
static const void* res_kernel(int lpr) {
  switch (lpr) {
    case 1: return (const void*)cheb_resident<1, MODE>;
    case 2: return (const void*)cheb_resident<2, MODE>;
    case 4: return (const void*)cheb_resident<4, MODE>;
    case 8: return (const void*)cheb_resident<8, MODE>;
  }
  return nullptr;
}
static const void* res_kernel_for(int lpr, int mode) {
  return mode == SDB_CHEB_DOUBLING ? res_kernel<SDB_CHEB_DOUBLING>(lpr) : res_kernel<SDB_CHEB_DIRECT>(lpr);
}

static size_t res_smem(int nbuf, int R, int pc, int nnz_cap) {
  return (size_t)nbuf * R * pc * sizeof(double) + (size_t)nnz_cap * (sizeof(double) + sizeof(int32_t)) +
         (size_t)(R + 1) * sizeof(int32_t) + 16;
}

// Function attributes are per device and sticky: raise them when a
// configuration needs more than what is already set (never on every launch:
// the calls would sit between the caller's work and a ~100 us kernel).
static cudaError_t res_ensure_attrs(int device, const void* fn, size_t smem, bool nonportable) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, std::pair<size_t, bool>> set;
  std::lock_guard<std::mutex> lock(mu);
  auto& st = set[std::make_pair(device, fn)];
  cudaError_t e = cudaSuccess;
  if (smem > st.first) {
    if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess) return e;
    st.first = smem;
  }
  if (nonportable && !st.second) {
    if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess) return e;
    st.second = true;
  }
  return e;
}

// Can a cluster of CL such CTAs be co-scheduled?  (cached per configuration)
static bool res_schedulable(int device, int lpr, int mode, int CL, int64_t clusters, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, size_t>, bool> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(device, lpr, mode, CL, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  bool ok = false;
  const void* fn = res_kernel_for(lpr, mode);
  if (res_ensure_attrs(device, fn, smem, CL > 8) == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(clusters * CL));
    cfg.blockDim = dim3(kResThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int active = 0;
    ok = cudaOccupancyMaxActiveClusters(&active, fn, &cfg) == cudaSuccess && active >= 1;
  }
  if (!ok) cudaGetLastError();
  cache[key] = ok;
  return ok;
}

int res_plan(const sdb_matrix* m, int64_t n_vec, int mode, ResPlan* p) {
  *p = ResPlan{};
  if (!res_env_enabled()) return SDB_OK;
  if (m->format != SDB_FMT_CSR || m->hb > 0 || m->res_cap[0] < 0) return SDB_OK;
  if (m->n >= (1LL << kResLocalBits) || n_vec < 1 || n_vec > SDB_MAX_BATCH) return SDB_OK;
  if (mode != SDB_CHEB_DOUBLING && mode != SDB_CHEB_DIRECT) return SDB_OK;
  const int64_t ldv = choose_geometry(n_vec).ldv;
  const int nbuf = mode == SDB_CHEB_DIRECT ? 3 : 2;
  const int sms = num_sms(m->device);
  const size_t budget = 220 * 1024;
  const int cls[] = {16, 8};
  const char* cl_env = getenv("SDB_RES_CL");  // tuning: 8 skips the 16-CTA (non-portable) clusters
  for (int ci = (cl_env && atoi(cl_env) == 8) ? 1 : 0; ci < 2; ++ci) {
    const int CL = cls[ci];
    const int R = (int)((m->n + CL - 1) / CL);
    if (R < 1) continue;
    int nnz_cap = m->res_cap[ci] > 0 ? m->res_cap[ci] : 1;
    nnz_cap = (nnz_cap + 3) & ~3;  // keeps the int32 arrays behind it 16-byte aligned
    // fewest columns per cluster (most SMs busy) that still fits one wave of the GPU
    for (int lpr = 1; lpr <= 8; lpr *= 2) {
      const int pc = 2 * lpr;
      const int64_t clusters = (ldv + pc - 1) / pc;
      if (clusters * CL > sms) continue;
      const size_t smem = res_smem(nbuf, R, pc, nnz_cap);
      if (smem > budget) continue;
      if (!res_schedulable(m->device, lpr, mode, CL, clusters, smem)) continue;
      p->on = true;
      p->CL = CL;
      p->lpr = lpr;
      p->R = R;
      p->nnz_cap = nnz_cap;
      p->clusters = clusters;
      p->smem = smem;
      p->nblocks = (int64_t)CL * kResWarps;
      return SDB_OK;
    }
  }
  return SDB_OK;
}

int res_launch(const sdb_matrix* m, const ResPlan& p, const StepArgs& a, int64_t degree, int mode,
               const double* probes, double* partials, cudaStream_t s) {
  ResArgs ra{};
  ra.rowptr = m->rowptr;
  ra.colidx = m->colidx;
  ra.vals = m->values;
  ra.probes = probes;
  ra.partials = partials;
  ra.c = a.c;
  ra.inv_d = a.inv_d;
  ra.n = m->n;
  ra.ldv = a.ldv;
  ra.R = p.R;
  ra.inv_R = 1.0f / (float)p.R;
  ra.nnz_cap = p.nnz_cap;
  ra.degree = (int)degree;
  ra.steps = (int)(mode == SDB_CHEB_DOUBLING ? (degree + 1) / 2 : degree);
  ra.legendre = a.legendre;
  if (const char* e = getenv("SDB_RES_DIAG")) ra.diag = atoi(e);
  const void* fn = res_kernel_for(p.lpr, mode);
  SDB_CUDA(res_ensure_attrs(m->device, fn, p.smem, p.CL > 8));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p.clusters * p.CL));
  cfg.blockDim = dim3(kResThreads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)p.CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  void* args[] = {(void*)&ra};
  SDB_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
  return SDB_OK;
}

}  // namespace sdb
