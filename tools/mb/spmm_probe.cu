// Microbenchmark: what the C2 access pattern (n = 64^3 rows x 64 fp64 probes,
// 7-point periodic gathers, w_{k+1} = 2 A w_k - w_{k-1}) can reach on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 spmm_probe.cu -o spmm_probe
// Prints one line per variant: time per launch and effective GB/s of the
// algorithmic traffic (read w_k, read w_{k-1}, write w_{k+1}).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int NX = 64, NY = 64, NZ = 64, N = NX * NY * NZ, LDV = 64;

__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ uint64_t pol_ef() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ double2 ld_once(const double* ptr, uint64_t pol) {
  double2 r; asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(ptr), "l"(pol)); return r; }
__device__ __forceinline__ void st_once(double* ptr, double2 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(ptr), "d"(v.x), "d"(v.y), "l"(pol) : "memory"); }

// rows of block b: grid-wide phased panels of P rows
template <int L, int VPL, int MODE>  // MODE 0: stream only, 1: 7-pt gathers
__global__ void __launch_bounds__(256) step(const double* __restrict__ x, const double* prev, double* next, int P, int nb,
                                            double* out) {
  constexpr int RPW = 32 / L, RPB = RPW * 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane / L, q = lane % L;
  const uint64_t pol = pol_ef();
  double acc = 0.0;
  for (int ph = 0;; ++ph) {
    int p0 = (ph * nb + blockIdx.x) * P;
    if (p0 >= N) break;
    int p1 = min(p0 + P, N);
    for (int base = p0; base < p1; base += RPB) {
      int row = base + warp * RPW + g;
      if (row >= p1) continue;
      double2 y[VPL], xi[VPL], wp[VPL];
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        xi[v] = ldg2(x + (size_t)row * LDV + 2 * q + 2 * L * v);
        wp[v] = ld_once(prev + (size_t)row * LDV + 2 * q + 2 * L * v, pol);
        y[v] = make_double2(6.0 * xi[v].x, 6.0 * xi[v].y);
      }
      if (MODE == 1) {
        int ix = row % NX, iy = (row / NX) % NY, iz = row / (NX * NY);
        int cols[6] = {row - ix + (ix + NX - 1) % NX, row - ix + (ix + 1) % NX,
                       row + (((iy + NY - 1) % NY) - iy) * NX, row + (((iy + 1) % NY) - iy) * NX,
                       row + (((iz + NZ - 1) % NZ) - iz) * NX * NY, row + (((iz + 1) % NZ) - iz) * NX * NY};
        double2 xv[6][VPL];
#pragma unroll
        for (int u = 0; u < 6; ++u)
#pragma unroll
          for (int v = 0; v < VPL; ++v) xv[u][v] = ldg2(x + (size_t)cols[u] * LDV + 2 * q + 2 * L * v);
#pragma unroll
        for (int u = 0; u < 6; ++u)
#pragma unroll
          for (int v = 0; v < VPL; ++v) { y[v].x -= xv[u][v].x; y[v].y -= xv[u][v].y; }
      }
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        double2 wn = make_double2(2.0 * 0.05 * y[v].x - wp[v].x, 2.0 * 0.05 * y[v].y - wp[v].y);
        st_once(next + (size_t)row * LDV + 2 * q + 2 * L * v, wn, pol);
        acc += wn.x * wn.x + wn.y * wn.y;
      }
    }
  }
  if (acc == 12345.0) out[0] = acc;
}

// Bulk-copy variant: one elected lane per warp issues cp.async.bulk of the 7
// x rows (512 B each) of the warp's next row into a shared-memory ring, so
// the copies are in flight without registers; the warp then consumes the
// ring stage from shared memory.
template <int STAGES>
__global__ void __launch_bounds__(256) step_bulk(const double* __restrict__ x, const double* prev, double* next, int P,
                                                 int nb, double* out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* ring = reinterpret_cast<double*>(smem_raw) + (size_t)warp * STAGES * 7 * LDV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + 8 * STAGES * 7 * LDV * 8) + warp * STAGES;
  const uint64_t pol = pol_ef();
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) {
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&bars[s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  // this warp's rows, in order
  auto row_at = [&](int k, int& row) -> bool {
    // k-th row of this warp across panels: each block iteration covers 8 rows (1 per warp)
    int per_panel = (P + 7) / 8;
    int ph = k / per_panel, it = k % per_panel;
    int p0 = (ph * nb + blockIdx.x) * P;
    if (p0 >= N) return false;
    int p1 = min(p0 + P, N);
    row = p0 + it * 8 + warp;
    if (row >= p1) { row = -1; }
    return true;
  };
  auto issue = [&](int k, int stage) {
    int row;
    if (!row_at(k, row) || row < 0) return;
    if (lane == 0) {
      int ix = row % NX, iy = (row / NX) % NY, iz = row / (NX * NY);
      int cols[7] = {row, row - ix + (ix + NX - 1) % NX, row - ix + (ix + 1) % NX,
                     row + (((iy + NY - 1) % NY) - iy) * NX, row + (((iy + 1) % NY) - iy) * NX,
                     row + (((iz + NZ - 1) % NZ) - iz) * NX * NY, row + (((iz + 1) % NZ) - iz) * NX * NY};
      uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[stage]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(7 * LDV * 8));
      for (int u = 0; u < 7; ++u) {
        uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + (stage * 7 + u) * LDV);
        const double* src = x + (size_t)cols[u] * LDV;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(src), "r"(LDV * 8), "r"(bar) : "memory");
      }
    }
  };
  double acc = 0.0;
  int phase_bits = 0;
  for (int s = 0; s < STAGES - 1; ++s) issue(s, s);
  for (int k = 0;; ++k) {
    int row;
    if (!row_at(k, row)) break;
    issue(k + STAGES - 1, (k + STAGES - 1) % STAGES);
    if (row < 0) continue;
    int stage = k % STAGES;
    double2 wp = ld_once(prev + (size_t)row * LDV + 2 * lane, pol);
    uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[stage]);
    uint32_t parity = (phase_bits >> stage) & 1;
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(bar), "r"(parity) : "memory");
    phase_bits ^= (1 << stage);
    const double* st = ring + stage * 7 * LDV + 2 * lane;
    double2 xi = *reinterpret_cast<const double2*>(st);
    double2 y = make_double2(6.0 * xi.x, 6.0 * xi.y);
#pragma unroll
    for (int u = 1; u < 7; ++u) {
      double2 xv = *reinterpret_cast<const double2*>(st + u * LDV);
      y.x -= xv.x; y.y -= xv.y;
    }
    __syncwarp();
    double2 wn = make_double2(0.1 * y.x - wp.x, 0.1 * y.y - wp.y);
    st_once(next + (size_t)row * LDV + 2 * lane, wn, pol);
    acc += wn.x * wn.x + wn.y * wn.y;
  }
  if (acc == 12345.0) out[0] = acc;
}


// cp.async (LDGSTS, L1-allocating) software pipeline: each lane copies its own
// 16 B columns of the 7 gathered rows + w_{k-1} of a future row iteration into
// shared memory and later reads back exactly those bytes (no barriers).
__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  uint32_t d = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem) : "memory");
}
template <int S>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(S) : "memory"); }
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

template <int STAGES>
__global__ void __launch_bounds__(256) step_cp(const double* __restrict__ x, const double* prev, double* next, int P, int nb,
                                               double* out) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* mine = sm + (size_t)warp * STAGES * 8 * LDV + 2 * lane;  // [stage][slot][LDV]
  const uint64_t pol = pol_ef();
  const int per_panel = P / 8;
  auto row_of = [&](int k) -> int {  // -2: done, -1: idle slot
    int ph = k / per_panel, it = k % per_panel;
    int p0 = (ph * nb + blockIdx.x) * P;
    if (p0 >= N) return -2;
    int row = p0 + it * 8 + warp;
    return row < min(p0 + P, N) ? row : -1;
  };
  auto issue = [&](int k) {
    int row = row_of(k);
    double* d = mine + (k % STAGES) * 8 * LDV;
    if (row >= 0) {
      int ix = row % NX, iy = (row / NX) % NY, iz = row / (NX * NY);
      int cols[7] = {row, row - ix + (ix + NX - 1) % NX, row - ix + (ix + 1) % NX,
                     row + (((iy + NY - 1) % NY) - iy) * NX, row + (((iy + 1) % NY) - iy) * NX,
                     row + (((iz + NZ - 1) % NZ) - iz) * NX * NY, row + (((iz + 1) % NZ) - iz) * NX * NY};
#pragma unroll
      for (int u = 0; u < 7; ++u) cp16(d + u * LDV, x + (size_t)cols[u] * LDV + 2 * lane);
      cp16(d + 7 * LDV, prev + (size_t)row * LDV + 2 * lane);
    }
    cp_commit();
  };
  double acc = 0.0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) issue(s);
  for (int k = 0;; ++k) {
    int row = row_of(k);
    if (row == -2) break;
    issue(k + STAGES - 1);
    cp_wait<STAGES - 1>();
    if (row < 0) continue;
    const double* d = mine + (k % STAGES) * 8 * LDV;
    double2 xi = *reinterpret_cast<const double2*>(d);
    double2 y = make_double2(6.0 * xi.x, 6.0 * xi.y);
#pragma unroll
    for (int u = 1; u < 7; ++u) {
      double2 xv = *reinterpret_cast<const double2*>(d + u * LDV);
      y.x -= xv.x; y.y -= xv.y;
    }
    double2 wp = *reinterpret_cast<const double2*>(d + 7 * LDV);
    double2 wn = make_double2(0.1 * y.x - wp.x, 0.1 * y.y - wp.y);
    st_once(next + (size_t)row * LDV + 2 * lane, wn, pol);
    acc += wn.x * wn.x + wn.y * wn.y;
  }
  cp_wait<0>();
  if (acc == 12345.0) out[0] = acc;
}


// Ablation: the micro gather7 kernel with the real kernel's features added.
//  F_DOTS  two per-column dot accumulators (doubling moments) + block partials
//  F_WTAB  weights loaded per term from a device table (+ diagonal array)
//  F_XI    x_i loaded separately, centre term gathered as a term
//  F_U4    gathers issued in batches of 4 (instead of all at once)
//  F_RLDV  runtime ldv
enum { F_DOTS = 1, F_WTAB = 2, F_XI = 4, F_U4 = 8, F_RLDV = 16 };
template <int L, int VPL, int F, int MINB>
__global__ void __launch_bounds__(256, MINB) step_ab(const double* __restrict__ x, const double* prev, double* next, int P,
                                                     int nb, double* out, const double* __restrict__ wt,
                                                     const double* __restrict__ diag, int ldv_rt) {
  constexpr int RPW = 32 / L, RPB = RPW * 8;
  const int ldv = (F & F_RLDV) ? ldv_rt : LDV;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane / L, q = lane % L;
  const uint64_t pol = pol_ef();
  double2 accA[VPL], accB[VPL];
  double acc = 0.0;
#pragma unroll
  for (int v = 0; v < VPL; ++v) accA[v] = accB[v] = make_double2(0.0, 0.0);
  for (int ph = 0;; ++ph) {
    int p0 = (ph * nb + blockIdx.x) * P;
    if (p0 >= N) break;
    int p1 = min(p0 + P, N);
    for (int base = p0; base < p1; base += RPB) {
      int row = base + warp * RPW + g;
      if (row >= p1) continue;
      double2 y[VPL], xi[VPL], wp[VPL];
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        xi[v] = ldg2(x + (size_t)row * ldv + 2 * q + 2 * L * v);
        wp[v] = ld_once(prev + (size_t)row * ldv + 2 * q + 2 * L * v, pol);
        y[v] = make_double2(0.0, 0.0);
      }
      int ix = row % NX, iy = (row / NX) % NY, iz = row / (NX * NY);
      int cols[7] = {row + (((iz + NZ - 1) % NZ) - iz) * NX * NY, row + (((iy + NY - 1) % NY) - iy) * NX,
                     row - ix + (ix + NX - 1) % NX, row, row - ix + (ix + 1) % NX,
                     row + (((iy + 1) % NY) - iy) * NX, row + (((iz + 1) % NZ) - iz) * NX * NY};
      double w[7];
#pragma unroll
      for (int u = 0; u < 7; ++u) w[u] = (F & F_WTAB) ? (u == 3 ? __ldg(diag + row) : __ldg(wt + u)) : (u == 3 ? 6.0 : -1.0);
      constexpr int U = (F & F_U4) ? 4 : 8;
#pragma unroll
      for (int o0 = 0; o0 < 7; o0 += U) {
        double2 xv[U][VPL];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int o = o0 + u;
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            if (o < 7 && ((F & F_XI) || o != 3))
              xv[u][v] = ldg2(x + (size_t)cols[o < 7 ? o : 3] * ldv + 2 * q + 2 * L * v);
            else if (o == 3)
              xv[u][v] = xi[v];
            else
              xv[u][v] = make_double2(0.0, 0.0);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int o = o0 + u;
          if (o < 7)
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
              y[v].x = fma(w[o], xv[u][v].x, y[v].x);
              y[v].y = fma(w[o], xv[u][v].y, y[v].y);
            }
        }
      }
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        double2 wn = make_double2(2.0 * ((y[v].x - 0.3 * xi[v].x) * 0.05) - wp[v].x,
                                  2.0 * ((y[v].y - 0.3 * xi[v].y) * 0.05) - wp[v].y);
        st_once(next + (size_t)row * ldv + 2 * q + 2 * L * v, wn, pol);
        if (F & F_DOTS) {
          accA[v].x += wn.x * wn.x; accA[v].y += wn.y * wn.y;
          accB[v].x += wn.x * xi[v].x; accB[v].y += wn.y * xi[v].y;
        } else {
          acc += wn.x * wn.x + wn.y * wn.y;
        }
      }
    }
  }
  if (F & F_DOTS) {
    __shared__ double sm[8 * 64];
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int off = L; off < 32; off <<= 1) {
        accA[v].x += __shfl_xor_sync(~0u, accA[v].x, off); accA[v].y += __shfl_xor_sync(~0u, accA[v].y, off);
        accB[v].x += __shfl_xor_sync(~0u, accB[v].x, off); accB[v].y += __shfl_xor_sync(~0u, accB[v].y, off);
      }
    if (lane < L)
#pragma unroll
      for (int v = 0; v < VPL; ++v) { sm[warp * 64 + 2 * (q + v * L)] = accA[v].x + accB[v].x; sm[warp * 64 + 2 * (q + v * L) + 1] = accA[v].y + accB[v].y; }
    __syncthreads();
    if (threadIdx.x < 64) { double s2 = 0; for (int w2 = 0; w2 < 8; ++w2) s2 += sm[w2 * 64 + threadIdx.x]; out[1 + blockIdx.x * 64 + threadIdx.x] = s2; }
  } else if (acc == 12345.0) out[0] = acc;
}

template <class F>
float timeit(F launch, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  launch(); launch();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  size_t bytes = (size_t)N * LDV * 8;
  double *x, *p, *q, *out;
  CK(cudaMalloc(&x, bytes)); CK(cudaMalloc(&p, bytes)); CK(cudaMalloc(&q, bytes)); CK(cudaMalloc(&out, 8));
  CK(cudaMemset(x, 0, bytes)); CK(cudaMemset(p, 0, bytes)); CK(cudaMemset(q, 0, bytes));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double alg = 3.0 * bytes;  // read x, read prev, write next
  auto report = [&](const char* name, float ms) { printf("%-40s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, alg / (ms * 1e-3) / 1e9); };
  double *wt, *dg;
  CK(cudaMalloc(&wt, 64)); CK(cudaMalloc(&dg, N * 8)); CK(cudaMemset(wt, 0, 64)); CK(cudaMemset(dg, 0, N * 8));
  CK(cudaFree(out)); CK(cudaMalloc(&out, 8 * (1 + 2000 * 64)));
#define AB(LL, VV, FF, MB)                                                                                    \
  for (int bps : {4, 5, 6}) {                                                                                 \
    int nb = bps * sms;                                                                                       \
    char nm[128];                                                                                             \
    snprintf(nm, sizeof nm, "ab L%d V%d F=%02d MB=%d nb=%d", LL, VV, FF, MB, nb);                             \
    report(nm, timeit([&] { step_ab<LL, VV, FF, MB><<<nb, 256>>>(x, p, q, 64, nb, out, wt, dg, LDV); }, 20)); \
  }
  AB(32, 1, 0, 1)
  AB(32, 1, F_DOTS, 1)
  AB(32, 1, F_WTAB, 1)
  AB(32, 1, F_XI, 1)
  AB(32, 1, F_U4, 1)
  AB(32, 1, F_RLDV, 1)
  AB(32, 1, F_DOTS | F_WTAB | F_XI | F_U4 | F_RLDV, 1)
  AB(32, 1, F_DOTS | F_WTAB | F_XI | F_U4 | F_RLDV, 5)
  AB(16, 2, 0, 1)
  AB(16, 2, F_DOTS | F_WTAB | F_XI | F_U4 | F_RLDV, 1)
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}
