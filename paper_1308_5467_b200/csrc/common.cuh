// common.cuh — shared plumbing for the specdens_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/specdens_b200.h"

namespace sdb {

// stencil shapes with compile-time term order (cheb.cu)
#define SDB_SHAPE_GENERIC 0
#define SDB_SHAPE_FACE7 1
#define SDB_SHAPE_BOX27 2

// ---- error reporting (thread-local message, status codes) ----------------
void set_error(const std::string& msg);
int fail(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define SDB_CUDA(call)                                                         \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) return ::sdb::cuda_fail(_e, #call, __FILE__, __LINE__); \
  } while (0)

#define SDB_CHECK_LAUNCH() SDB_CUDA(cudaGetLastError())

#define SDB_REQUIRE(cond, ...)                                                 \
  do {                                                                         \
    if (!(cond)) return ::sdb::fail(SDB_EINVAL, __VA_ARGS__);                 \
  } while (0)

// Switch the calling thread to `device` for the lifetime of the guard.
struct DeviceGuard {
  int prev = -1;
  int ok = 0;
  explicit DeviceGuard(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = (cudaSetDevice(device) == cudaSuccess);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int num_sms(int device);

// Band + far split of a freshly uploaded CSR matrix (band.cu).  Leaves the
// matrix unsplit (hb = 0) when it has no dense symmetric band; returns an
// error code only on CUDA failures.
}  // namespace sdb
struct sdb_matrix;
namespace sdb {
int band_build(sdb_matrix* m, cudaStream_t s);
// zero guard rows/diagonal entries before and after the band data
__host__ __device__ constexpr int band_pad(int hb) { return (hb + 7) & ~7; }

// ---- matrix handle ---------------------------------------------------------
struct StencilDev {
  int64_t nx, ny, nz;
  int32_t n_off;
  int32_t off[26][3];
  double w[26];
};

}  // namespace sdb

struct sdb_matrix {
  int device = 0;
  int format = SDB_FMT_CSR;
  int64_t n = 0;
  int64_t nnz = 0;
  // CSR (int32 row pointers and column indices: nnz < 2^31)
  int32_t* rowptr = nullptr;
  int32_t* colidx = nullptr;
  double* values = nullptr;
  // stencil
  sdb::StencilDev st{};
  double* diag = nullptr;
  int4* terms = nullptr;      // (dx, dy, dz, interior column delta), sorted by delta
  double* term_w = nullptr;   // weight per term (diagonal slot unused)
  double term_w_host[27] = {};
  int nterms = 0, center_pos = 0, mx = 0, my = 0, mz = 0;
  int shape = 0;              // SDB_SHAPE_*: specialised grid kernel available
  int zghost = 0;             // z-slab of a row partition (no z wrap, ghost planes)
  // band + far split of a CSR matrix (band.cu): the dense band |i-j| <= hb as
  // symmetric upper diagonals, the rest (far entries) as SELL-4-sigma streams
  int hb = 0;                 // 0: no split
  int64_t ustride = 0;        // doubles per diagonal of bu
  double* bu = nullptr;       // [hb+1][ustride]: bu[d*ustride + band_pad(hb) + i] = A[i][i+d]
  // far entries: per 128-row tile the rows are sorted by far count (sigma =
  // 128), cut into 4-row chunks (C = 4) and dealt to 16 streams; a stream is a
  // run of 208-byte batch records (4 slots x 4 rows: columns, values, chunk /
  // tile end flags, the chunk's local row ids), see band.cu
  int2* fhdr = nullptr;       // [ntiles][16]: (first record, records) of a stream
  uint4* frec = nullptr;      // records, 13 x 16 B each
  int64_t frecs = 0;          // stored records
  int64_t fnnz = 0;           // far entries (without padding)
  // cluster-resident recurrence (resident.cu): most CSR entries in one row
  // block when the rows are cut into 16 / 8 equal blocks (-1: not computed)
  int32_t res_cap[2] = {-1, -1};
};

namespace sdb {

// ---- programmatic dependent launch (PDL) between recurrence steps -----------
// Inside sdb_cheb_moments every step kernel is launched with programmatic
// stream serialisation: step k+1 is launched while step k runs, its blocks
// take SMs as step k's blocks retire, and they wait in griddepcontrol.wait
// until step k has completed and flushed.  So launch latency and block
// start-up overlap the previous step's tail instead of sitting between the
// steps.  Kernels launched without the attribute pass griddepcontrol.wait
// immediately, so the same kernels serve every other entry point unchanged.
// Every step kernel calls pdl_wait() before touching global memory.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Set for the duration of one sdb_cheb_moments step loop (thread-local): the
// step launchers then add the PDL attribute.  SDB_PDL=0 disables it.
struct PdlScope {
  PdlScope();
  ~PdlScope();
};
bool pdl_active();
cudaError_t launch_maybe_pdl(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t s);

// Rows per panel of the phased-panel schedule (rowgroup.cuh) for a block
// width of ldv doubles and RPB rows per block iteration.  SDB_PANEL_ROWS
// overrides it (tuning).
int64_t panel_rows(const sdb_matrix* m, int64_t ldv, int rpb);

// Blocks of the persistent row-range kernels.  Depends on n and the SM count
// only, so the reduction tree (and hence every bit of the result) is fixed for
// a given matrix on a given GPU model.
int64_t row_blocks(const sdb_matrix* m);

// Row group geometry: L lanes per row (power of two <= 32), each lane holding
// VPL double2 values; ldv = 2 * L * VPL.
struct Geometry {
  int L;
  int VPL;
  int64_t ldv;
};
Geometry choose_geometry(int64_t n_vec);

// ---- device helpers ---------------------------------------------------------
__device__ __forceinline__ double2 ld_d2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}
// Streaming load of data touched once per pass (do not keep in L1).
__device__ __forceinline__ double2 ld_d2_stream(const double* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_d2(double* p, double2 v) {
  *reinterpret_cast<double2*>(p) = v;
}

}  // namespace sdb
