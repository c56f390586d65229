// Microbenchmark / semantics probe: cp.async.bulk.tensor.2d tile::gather4 on sm_100a.
// A [rows][16] fp64 tensor (row r holds the value r), box {16, 1}; one thread gathers four
// rows (in-bounds and out-of-bounds) into shared memory and waits on an mbarrier with a
// bounded spin, printing the transaction-byte behaviour.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 gather4.cu -o gather4 -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap map, int r0, int r1, int r2, int r3, uint32_t expect,
                  double* out, int* info) {
  __shared__ __align__(128) double buf[4 * 16];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 64; ++i) buf[i] = -7.0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(expect) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4, %5, %6}], [%7];" ::"r"(su32(buf)),
        "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(&bar))
        : "memory");
    int done = 0, spins = 0;
    for (; spins < 2000000 && !done; ++spins) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.s32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(su32(&bar))
          : "memory");
    }
    info[0] = done;
    info[1] = spins;
    for (int i = 0; i < 64; ++i) out[i] = buf[i];
  }
}

int main() {
  const int rows = 64;
  double* d;
  cudaMalloc(&d, rows * 16 * 8);
  double h[rows * 16];
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < 16; ++c) h[r * 16 + c] = r + 0.01 * c;
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
  for (int boxrows = 1; boxrows <= 4; boxrows += 3) {
    CUtensorMap map;
    cuuint64_t gdim[2] = {16, (cuuint64_t)rows};
    cuuint64_t gstr[1] = {128};
    cuuint32_t box[2] = {16, (cuuint32_t)boxrows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("box rows %d: encode -> %d\n", boxrows, (int)r);
    if (r != CUDA_SUCCESS) continue;
    double* out;
    int* info;
    cudaMalloc(&out, 64 * 8);
    cudaMalloc(&info, 8);
    const int cases[3][4] = {{3, 10, 20, 63}, {3, -1, 20, 63}, {3, 64, 20, 1000}};
    for (int c = 0; c < 3; ++c)
      for (uint32_t expect : {512u}) {
        cudaMemset(info, 0, 8);
        k<<<1, 32>>>(map, cases[c][0], cases[c][1], cases[c][2], cases[c][3], expect, out, info);
        cudaError_t e = cudaDeviceSynchronize();
        double ho[64];
        int hi[2] = {0, 0};
        cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
        cudaMemcpy(hi, info, 8, cudaMemcpyDeviceToHost);
        printf("  rows {%d,%d,%d,%d} expect %u: %s done=%d spins=%d  got rows [%.2f %.2f %.2f %.2f] (col 1: %.2f)\n",
               cases[c][0], cases[c][1], cases[c][2], cases[c][3], expect, cudaGetErrorString(e), hi[0], hi[1], ho[0],
               ho[16], ho[32], ho[48], ho[1]);
        if (e != cudaSuccess) return 0;
      }
  }
  return 0;
}
