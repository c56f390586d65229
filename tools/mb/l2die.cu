// Microbenchmark: is B200's L2 effectively per die for data every SM reads?
// One "pass" gathers random 128 B rows of a fresh W-byte buffer, each row ~20
// times (the C3 band kernel's far-gather pattern).  Run under ncu for DRAM
// bytes; the printed time is the kernel time.  Modes:
//   0: every SM gathers;  1: only SMs with smid < nsm/2;  2: only even smids;
//   3: SMs of die A (per the latency probe below) gather.
// A per-SM latency probe classifies SMs by which half of a set of lines is
// "near" (lower latency), printing the smid -> group map.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 l2die.cu -o l2die
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// per-SM gather pass: active blocks gather total/active rows each
__global__ void gather(const double* __restrict__ buf, int64_t rows, int64_t per_block, int mode, int nsm,
                       const int* __restrict__ group, double* out) {
  const unsigned sm = smid();
  bool active = true;
  if (mode == 1) active = sm < (unsigned)(nsm / 2);
  if (mode == 2) active = (sm & 1) == 0;
  if (mode == 3) active = group[sm] == 0;
  if (!active) return;
  const int lane = threadIdx.x & 31, q = lane & 7, g = lane >> 3;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  double acc = 0.0;
  for (int64_t k = 0; k < per_block; k += 4 * 4) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t r = hash32((uint32_t)(warp * 977 + k + 4 * u + g) * 2654435761u) % (uint32_t)rows;
      v[u] = __ldg(reinterpret_cast<const double2*>(buf + r * 16 + 2 * q));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x * v[u].y;
  }
  if (acc == 12345.678) out[0] = acc;
}

// latency probe: one thread per block chases 64 lines (stride 4 KB apart) and
// records per-line latency; lines are on one die or the other
__global__ void probe(const double* buf, int nlines, unsigned* lat, unsigned* sm_of_block) {
  if (threadIdx.x) return;
  sm_of_block[blockIdx.x] = smid();
  volatile const double* b = buf;
  for (int l = 0; l < nlines; ++l) {
    const volatile double* p = b + (int64_t)l * 512;  // 4 KB apart
    double t = *p;  // warm (into L2)
    (void)t;
    long long t0 = clock64();
    double v = *p;
    long long t1 = clock64();
    if (v == 1234.5) lat[0] = 0;
    lat[blockIdx.x * nlines + l] = (unsigned)(t1 - t0);
  }
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int64_t maxbytes = 256LL << 20;
  double *buf, *out;
  CK(cudaMalloc(&buf, maxbytes * 8));  // 8 fresh regions
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(buf, 0, maxbytes * 8));
  // latency probe: 148 blocks (one per SM with a big smem request to spread them)
  const int nl = 64;
  unsigned *lat, *smb;
  int* group;
  CK(cudaMalloc(&lat, sizeof(unsigned) * nsm * nl));
  CK(cudaMalloc(&smb, sizeof(unsigned) * nsm));
  CK(cudaMalloc(&group, sizeof(int) * 1024));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  probe<<<nsm, 32, 200 * 1024>>>(buf, nl, lat, smb);
  CK(cudaDeviceSynchronize());
  std::vector<unsigned> hl(nsm * nl), hs(nsm);
  CK(cudaMemcpy(hl.data(), lat, sizeof(unsigned) * nsm * nl, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hs.data(), smb, sizeof(unsigned) * nsm, cudaMemcpyDeviceToHost));
  // reference pattern: SM of block 0's near/far lines; group = agreement
  std::vector<int> gsm(1024, -1);
  std::vector<int> near0(nl);
  double med0 = 0;
  for (int l = 0; l < nl; ++l) med0 += hl[l];
  med0 /= nl;
  for (int l = 0; l < nl; ++l) near0[l] = hl[l] < med0;
  int ga = 0, gb = 0;
  for (int b = 0; b < nsm; ++b) {
    double med = 0;
    for (int l = 0; l < nl; ++l) med += hl[b * nl + l];
    med /= nl;
    int agree = 0;
    for (int l = 0; l < nl; ++l) agree += ((hl[b * nl + l] < med) == near0[l]);
    gsm[hs[b]] = agree > nl / 2 ? 0 : 1;
    (gsm[hs[b]] == 0 ? ga : gb)++;
  }
  printf("latency groups: %d / %d SMs\nsmid->group:", ga, gb);
  for (int s = 0; s < nsm; ++s) printf("%d", gsm[s] < 0 ? 9 : gsm[s]);
  printf("\n");
  CK(cudaMemcpy(group, gsm.data(), sizeof(int) * 1024, cudaMemcpyHostToDevice));

  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  int region = 0;
  for (int64_t mb : {32, 64, 96, 128}) {
    for (int mode = 0; mode < 4; ++mode) {
      const int64_t bytes = mb << 20, rows = bytes / 128;
      const int64_t gathers = 20 * rows;  // each row ~20 times per pass
      const int blocks = nsm * 4;
      const int64_t per_block_warp = gathers / (blocks * 8);  // rows per warp
      const double* b = buf + (int64_t)(region++ % 8) * (maxbytes / 8);
      CK(cudaEventRecord(e0));
      gather<<<blocks, 256>>>(b, rows, per_block_warp * ((mode == 0) ? 1 : 2), mode, nsm, group, out);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("W=%4lld MB mode=%d: %.3f ms  (%.0f GB/s gathered)\n", (long long)mb, mode, ms,
             gathers * 128.0 / ms / 1e6);
    }
  }
  return 0;
}
