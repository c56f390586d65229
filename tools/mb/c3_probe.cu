// Microbenchmark for the C3 (n = 1e6, band + ~20 random off-band entries per
// row, 128 fp64 probes) step design on B200:
//   * random row gathers of G bytes from an x slice of B bytes (L2-resident
//     or not), with and without an L2 persisting access-policy window, with
//     and without concurrent evict-first streaming traffic;
//   * fp64 FMA issue rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 c3_probe.cu -o /tmp/c3_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA %s at %d: %s\n", cudaGetErrorString(e), __LINE__, #x);           \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ uint64_t pol_ef() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_once(const double* ptr, uint64_t pol) {
  double2 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y)
               : "l"(ptr), "l"(pol));
  return r;
}

// Each group of LPR lanes gathers one random row of G = 16*LPR bytes from
// buf (rows of G bytes); U gathers in flight per lane.  STREAM: every
// iteration also streams SB double2 per lane from a large buffer (evict-first).
template <int LPR, int U, int STREAM>
__global__ void __launch_bounds__(256) gather(const double* __restrict__ buf, int64_t rows, int64_t total_gathers,
                                              const double* __restrict__ sbuf, int64_t sdoubles, double* out) {
  constexpr int GPW = 32 / LPR;  // gathers per warp per u
  const int lane = threadIdx.x & 31, q = lane % LPR, g = lane / LPR;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol = pol_ef();
  double acc = 0.0;
  int64_t spos = warp * 32 * 2 + lane * 2;
  for (int64_t base = warp * GPW * U; base < total_gathers; base += nwarps * GPW * U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t id = (uint32_t)(base + u * GPW + g);
      const int64_t r = hash32(id) % (uint32_t)rows;
      v[u] = __ldg(reinterpret_cast<const double2*>(buf + r * (2 * LPR) + 2 * q));
    }
    if (STREAM) {
#pragma unroll
      for (int s = 0; s < STREAM; ++s) {
        double2 t = ld_once(sbuf + spos, pol);
        acc += t.x;
        spos += nwarps * 64;
        if (spos >= sdoubles) spos -= sdoubles;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x * v[u].y;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void __launch_bounds__(256) dfma_kernel(double* out, int iters, double b, double c) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

template <int LPR, int U, int STREAM>
static int run_gather(const char* tag, double* buf, int64_t bytes, double* sbuf, int64_t sbytes, double* out,
                      cudaStream_t st, int sms) {
  const int64_t G = 16 * LPR;
  const int64_t rows = bytes / G;
  const int64_t total = 160000000LL * 128 / G;  // the same gathered bytes for every G (20.5 GB)
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int grid = sms * 8;
  for (int w = 0; w < 2; ++w) gather<LPR, U, STREAM><<<grid, 256, 0, st>>>(buf, rows, total, sbuf, sbytes / 8, out);
  CK(cudaEventRecord(e0, st));
  const int reps = 3;
  for (int r = 0; r < reps; ++r) gather<LPR, U, STREAM><<<grid, 256, 0, st>>>(buf, rows, total, sbuf, sbytes / 8, out);
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  ms /= reps;
  const double gbytes = (double)total * G;
  const double sbytes_moved = STREAM ? (double)total / (32 / LPR) / U * 32 * 16 * STREAM : 0.0;
  printf("%-10s G=%4lld B x-slice=%6.0f MB U=%d stream=%d: %8.3f ms  gather %7.0f GB/s  stream %6.0f GB/s\n", tag,
         (long long)G, bytes / 1048576.0, U, STREAM, ms, gbytes / ms / 1e6, sbytes_moved / ms / 1e6);
  return 0;
}

int main() {
  int dev = 0, sms = 0, l2 = 0, maxpersist = 0, maxwin = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&maxpersist, cudaDevAttrMaxPersistingL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, dev));
  printf("SMs %d  L2 %d B  max persisting L2 %d B  max window %d B\n", sms, l2, maxpersist, maxwin);
  const int64_t big = 1LL << 30;
  double *buf, *sbuf, *out;
  CK(cudaMalloc(&buf, big));
  CK(cudaMalloc(&sbuf, 2 * big));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(buf, 0, big));
  CK(cudaMemset(sbuf, 0, 2 * big));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));

  // fp64 FMA rate
  {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int iters = 1 << 14, grid = sms * 8;
    dfma_kernel<<<grid, 256, 0, st>>>(out, iters, 0.999, 1e-3);
    CK(cudaEventRecord(e0, st));
    dfma_kernel<<<grid, 256, 0, st>>>(out, iters, 0.999, 1e-3);
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double fmas = (double)grid * 256 * iters * 8;
    printf("DFMA: %.3f ms  %.2f TFMA/s = %.2f TFLOP/s fp64\n", ms, fmas / ms / 1e9, 2 * fmas / ms / 1e9);
  }

  const int64_t sizes_mb[] = {32, 48, 64, 96, 128, 192, 256, 512, 1024};
  for (int64_t mb : sizes_mb) {
    const int64_t bytes = mb << 20;
    run_gather<4, 4, 0>("plain", buf, bytes, sbuf, 2 * big, out, st, sms);
    run_gather<8, 4, 0>("plain", buf, bytes, sbuf, 2 * big, out, st, sms);
    run_gather<16, 4, 0>("plain", buf, bytes, sbuf, 2 * big, out, st, sms);
  }
  // with concurrent streaming (evict-first) traffic
  for (int64_t mb : {64, 128, 256}) {
    const int64_t bytes = mb << 20;
    run_gather<8, 4, 1>("stream", buf, bytes, sbuf, 2 * big, out, st, sms);
    run_gather<16, 4, 1>("stream", buf, bytes, sbuf, 2 * big, out, st, sms);
  }
  // persisting window on the slice
  if (maxpersist > 0) {
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxpersist));
    for (int64_t mb : {64, 96, 128, 256}) {
      const int64_t bytes = mb << 20;
      cudaStreamAttrValue v{};
      v.accessPolicyWindow.base_ptr = buf;
      v.accessPolicyWindow.num_bytes = bytes < maxwin ? bytes : maxwin;
      v.accessPolicyWindow.hitRatio = (float)((double)maxpersist / (double)v.accessPolicyWindow.num_bytes);
      if (v.accessPolicyWindow.hitRatio > 1.f) v.accessPolicyWindow.hitRatio = 1.f;
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v));
      run_gather<8, 4, 0>("persist", buf, bytes, sbuf, 2 * big, out, st, sms);
      run_gather<16, 4, 0>("persist", buf, bytes, sbuf, 2 * big, out, st, sms);
      run_gather<8, 4, 1>("persist+s", buf, bytes, sbuf, 2 * big, out, st, sms);
      run_gather<16, 4, 1>("persist+s", buf, bytes, sbuf, 2 * big, out, st, sms);
      v.accessPolicyWindow.num_bytes = 0;
      CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v));
      CK(cudaCtxResetPersistingL2Cache());
    }
  }
  return 0;
}
