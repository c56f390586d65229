// Microbenchmark: which setmaxnreg patterns are legal on sm_100a for a 640-thread block
// (warpgroup 0 raises its register count, warpgroups 1..4 lower theirs), with and
// without griddepcontrol (PDL) instructions before it, large dynamic shared memory,
// a full grid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 setmaxnreg.cu -o setmaxnreg
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int INC, int DEC, int THREADS, int PDL>
__global__ void __launch_bounds__(THREADS, 1) k(int* out) {
  extern __shared__ char sm[];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) sm[0] = 1;
  __syncthreads();
  if (PDL & 1) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (PDL & 2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp < 4) {
    if (INC) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(INC ? INC : 24));
    out[threadIdx.x] = 1 + sm[0];
    return;
  }
  if (DEC) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(DEC ? DEC : 24));
  out[threadIdx.x] = 2;
}

template <int INC, int DEC, int THREADS, int PDL>
void run(const char* tag, int* out, int grid, int smem) {
  cudaFuncSetAttribute(k<INC, DEC, THREADS, PDL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<INC, DEC, THREADS, PDL><<<grid, THREADS, smem>>>(out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%-28s threads=%d grid=%d smem=%d pdl=%d inc=%d dec=%d -> %s\n", tag, THREADS, grid, smem, PDL, INC, DEC,
         cudaGetErrorString(e));
  fflush(stdout);
  if (e != cudaSuccess) exit(0);
}

int main() {
  int* out;
  cudaMalloc(&out, 4096);
  run<168, 64, 640, 0>("plain", out, 1, 1024);
  run<168, 64, 640, 0>("grid 148", out, 148, 1024);
  run<168, 64, 640, 0>("smem 221K", out, 148, 226368);
  run<168, 64, 640, 1>("griddep wait", out, 148, 226368);
  run<168, 64, 640, 3>("griddep wait+launch", out, 148, 226368);
  return 0;
}
