// matrix.cu — library plumbing and the sparse-matrix layer.
//
// Reference: SparseSymmetricMatrix (matrix.py:35-109) stores a SciPy CSR with
// both triangles; its matvec is `csr @ x` (matrix.py:101-102), i.e. SciPy
// csr_matvec: y_i = sum over the row's entries in storage order.  We keep the
// CSR exactly as given (row order and in-row order) so the per-row sums run in
// the same order, narrowed to int32 indices on the device.
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"

namespace sdb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  cudaGetLastError();  // clear sticky-free errors
  const char* base = strrchr(file, '/');
  return fail(e == cudaErrorMemoryAllocation ? SDB_ENOMEM : SDB_ECUDA, "CUDA error %s (%s) in %s at %s:%d",
              cudaGetErrorName(e), cudaGetErrorString(e), what, base ? base + 1 : file, line);
}

int num_sms(int device) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0) device = 0;
  if ((int)cache.size() <= device) cache.resize(device + 1, 0);
  if (cache[device] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0) v = 148;
    cache[device] = v;
  }
  return cache[device];
}

static thread_local int g_pdl_depth = 0;
static bool pdl_env_enabled() {
  static const bool on = [] {
    const char* e = getenv("SDB_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
PdlScope::PdlScope() { ++g_pdl_depth; }
PdlScope::~PdlScope() { --g_pdl_depth; }
bool pdl_active() { return g_pdl_depth > 0 && pdl_env_enabled(); }

cudaError_t launch_maybe_pdl(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_active() ? 1 : 0;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

int64_t row_blocks(const sdb_matrix* m) {
  // 4 resident row-range blocks per SM; never fewer rows than one block
  // iteration per block for small matrices.
  int64_t b = 4LL * num_sms(m->device);
  int64_t by_rows = (m->n + 63) / 64;
  if (by_rows < b) b = by_rows;
  return b < 1 ? 1 : b;
}

int64_t panel_rows(const sdb_matrix* m, int64_t ldv, int rpb) {
  int64_t p = 0;
  if (const char* env = getenv("SDB_PANEL_ROWS")) p = atoll(env);
  const int64_t B = row_blocks(m);
  (void)B;
  (void)ldv;
  // 64-row panels: short enough that the far neighbours of a row are gathered
  // by other blocks within a few microseconds (L2 hits), long enough for the
  // +-1 / +-nx neighbours to be L1 hits (measured, tools/mb/spmm_probe.cu)
  if (p <= 0) p = 64;
  p = (p + rpb - 1) / rpb * rpb;
  return p < rpb ? rpb : p;
}

Geometry choose_geometry(int64_t n_vec) {
  // Wide blocks: one warp per row, VPL double2 per lane.
  if (n_vec > 64) {
    int vpl = (int)((n_vec + 63) / 64);
    return Geometry{32, vpl, 64LL * vpl};
  }
  // Narrow blocks: pick the padded width 2*L*VPL (VPL <= 4) with the least
  // padding, preferring more lanes per row (fewer rows per warp).
  Geometry best{1, 1, 1LL << 40};
  for (int L = 32; L >= 1; L >>= 1) {
    for (int vpl = 1; vpl <= 4; ++vpl) {
      int64_t ldv = 2LL * L * vpl;
      if (ldv < n_vec) continue;
      if (ldv < best.ldv) best = Geometry{L, vpl, ldv};
      break;
    }
  }
  // tuning override: same ldv, different lanes per row
  if (const char* env = getenv("SDB_LANES")) {
    int L = atoi(env);
    if (L >= 1 && L <= 32 && (L & (L - 1)) == 0 && best.ldv % (2 * L) == 0 && best.ldv / (2 * L) <= 4)
      best = Geometry{L, (int)(best.ldv / (2 * L)), best.ldv};
  }
  return best;
}

}  // namespace sdb

using namespace sdb;

namespace {

__global__ void narrow_i64_kernel(const int64_t* __restrict__ src, int32_t* __restrict__ dst, int64_t count,
                                  int64_t limit, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = src[i];
    if (v < 0 || v >= limit) atomicExch(bad, 1);
    dst[i] = (int32_t)v;
  }
}

__global__ void check_i32_kernel(const int32_t* __restrict__ src, int64_t count, int64_t limit, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = src[i];
    if (v < 0 || v >= limit) atomicExch(bad, 1);
  }
}

__global__ void pack_kernel(const double* __restrict__ pt, int64_t n_vec, int64_t n, int64_t ldv,
                            double* __restrict__ block) {
  // pt: n_vec x n ; block: n x ldv.  32x32 tiles through shared memory.
  __shared__ double tile[32][33];
  int64_t r0 = (int64_t)blockIdx.x * 32;  // row of block (= index into n)
  int64_t c0 = (int64_t)blockIdx.y * 32;  // column of block (= probe)
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    int64_t l = c0 + j, i = r0 + threadIdx.x;
    tile[j][threadIdx.x] = (l < n_vec && i < n) ? pt[l * n + i] : 0.0;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    int64_t i = r0 + j, l = c0 + threadIdx.x;
    if (i < n && l < ldv) block[i * ldv + l] = tile[threadIdx.x][j];
  }
}

__global__ void unpack_kernel(const double* __restrict__ block, int64_t n, int64_t ldv, int64_t n_vec,
                              double* __restrict__ pt) {
  __shared__ double tile[32][33];
  int64_t r0 = (int64_t)blockIdx.x * 32;
  int64_t c0 = (int64_t)blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    int64_t i = r0 + j, l = c0 + threadIdx.x;
    tile[j][threadIdx.x] = (i < n && l < n_vec) ? block[i * ldv + l] : 0.0;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    int64_t l = c0 + j, i = r0 + threadIdx.x;
    if (l < n_vec && i < n) pt[l * n + i] = tile[threadIdx.x][j];
  }
}

// one thread per (row, 2 columns): coalesced double2 stores into the block
__global__ void unpack_signs_kernel(const uint8_t* __restrict__ bits, int64_t n_vec, int64_t n, int64_t ldv,
                                    double* __restrict__ block) {
  const int64_t nbytes = (n + 7) / 8;
  const int64_t half = ldv / 2;
  const int64_t total = n * half;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / half, c = 2 * (idx % half);
    double v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t l = c + u;
      v[u] = 0.0;
      if (l < n_vec) v[u] = ((bits[l * nbytes + (i >> 3)] >> (i & 7)) & 1) ? 1.0 : -1.0;
    }
    *reinterpret_cast<double2*>(block + i * ldv + c) = make_double2(v[0], v[1]);
  }
}

}  // namespace

extern "C" {

const char* sdb_last_error(void) { return g_last_error.c_str(); }

int sdb_version(void) { return 1; }

int64_t sdb_block_ldv(int64_t n_vec) {
  if (n_vec < 1 || n_vec > SDB_MAX_BATCH) return -1;
  return choose_geometry(n_vec).ldv;
}

int sdb_matrix_create_csr(int device, int64_t n, int64_t nnz, const int64_t* indptr, const void* indices,
                          int index_bits, const double* values, void* stream, sdb_matrix** out) {
  SDB_REQUIRE(out != nullptr, "out must not be NULL");
  *out = nullptr;
  SDB_REQUIRE(n >= 1, "matrix dimension must be positive (got %lld)", (long long)n);
  SDB_REQUIRE(nnz >= 0, "nnz must be non-negative");
  SDB_REQUIRE(nnz < (1LL << 31) && n < (1LL << 31), "matrix too large for int32 CSR (n=%lld, nnz=%lld)",
              (long long)n, (long long)nnz);
  SDB_REQUIRE(index_bits == 32 || index_bits == 64, "index_bits must be 32 or 64");
  SDB_REQUIRE(indptr != nullptr, "indptr must not be NULL");
  SDB_REQUIRE(nnz == 0 || (indices != nullptr && values != nullptr), "indices/values must not be NULL");
  // host-side structural checks on the row pointer (n+1 entries, cheap)
  SDB_REQUIRE(indptr[0] == 0 && indptr[n] == nnz, "indptr must start at 0 and end at nnz");
  std::vector<int32_t> rp((size_t)n + 1);
  for (int64_t i = 0; i <= n; ++i) {
    if (i > 0 && indptr[i] < indptr[i - 1]) return fail(SDB_EINVAL, "indptr must be non-decreasing");
    rp[(size_t)i] = (int32_t)indptr[i];
  }
  DeviceGuard g(device);
  if (!g.ok) return fail(SDB_ECUDA, "cannot select CUDA device %d", device);
  cudaStream_t s = (cudaStream_t)stream;

  sdb_matrix* m = new sdb_matrix();
  m->device = device;
  m->format = SDB_FMT_CSR;
  m->n = n;
  m->nnz = nnz;
  for (int i = 0; i < 2; ++i) {  // row-block entry counts for the cluster-resident path
    const int64_t CL = i == 0 ? 16 : 8, R = (n + CL - 1) / CL;
    int32_t cap = 0;
    for (int64_t r = 0; r < CL; ++r) {
      const int64_t lo = r * R < n ? r * R : n, hi = (r + 1) * R < n ? (r + 1) * R : n;
      const int32_t cnt = rp[(size_t)hi] - rp[(size_t)lo];
      if (cnt > cap) cap = cnt;
    }
    m->res_cap[i] = cap;
  }
  auto cleanup = [&](int code) {
    sdb_matrix_destroy(m);
    return code;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&m->rowptr, sizeof(int32_t) * (n + 1))) != cudaSuccess)
    return cleanup(cuda_fail(e, "cudaMalloc(rowptr)", __FILE__, __LINE__));
  size_t nz = (size_t)(nnz > 0 ? nnz : 1);
  if ((e = cudaMalloc(&m->colidx, sizeof(int32_t) * nz)) != cudaSuccess)
    return cleanup(cuda_fail(e, "cudaMalloc(colidx)", __FILE__, __LINE__));
  if ((e = cudaMalloc(&m->values, sizeof(double) * nz)) != cudaSuccess)
    return cleanup(cuda_fail(e, "cudaMalloc(values)", __FILE__, __LINE__));
  if ((e = cudaMemcpyAsync(m->rowptr, rp.data(), sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, s)) !=
      cudaSuccess)
    return cleanup(cuda_fail(e, "upload rowptr", __FILE__, __LINE__));
  if (nnz > 0) {
    if ((e = cudaMemcpyAsync(m->values, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return cleanup(cuda_fail(e, "upload values", __FILE__, __LINE__));
    int* bad = nullptr;
    if ((e = cudaMalloc(&bad, sizeof(int))) != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc", __FILE__, __LINE__));
    cudaMemsetAsync(bad, 0, sizeof(int), s);
    if (index_bits == 32) {
      e = cudaMemcpyAsync(m->colidx, indices, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) {
        check_i32_kernel<<<1024, 256, 0, s>>>(m->colidx, nnz, n, bad);
        e = cudaGetLastError();
      }
    } else {
      // stage int64 indices in chunks and narrow on the device
      const int64_t chunk = 1LL << 26;
      int64_t* tmp = nullptr;
      int64_t cn = nnz < chunk ? nnz : chunk;
      e = cudaMalloc(&tmp, sizeof(int64_t) * cn);
      for (int64_t off = 0; e == cudaSuccess && off < nnz; off += chunk) {
        int64_t cnt = (nnz - off) < chunk ? (nnz - off) : chunk;
        e = cudaMemcpyAsync(tmp, (const int64_t*)indices + off, sizeof(int64_t) * cnt, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) {
          narrow_i64_kernel<<<1024, 256, 0, s>>>(tmp, m->colidx + off, cnt, n, bad);
          e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // tmp is reused
      }
      if (tmp) cudaFree(tmp);
    }
    int hbad = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(bad);
    if (e != cudaSuccess) return cleanup(cuda_fail(e, "upload indices", __FILE__, __LINE__));
    if (hbad) return cleanup(fail(SDB_EINVAL, "column index out of range [0, %lld)", (long long)n));
  } else {
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cleanup(cuda_fail(e, "sync", __FILE__, __LINE__));
  }
  // dense-band + far split for the probe-sliced band kernel (band.cu); a
  // matrix without a dense symmetric band keeps the plain CSR path
  int brc = band_build(m, s);
  if (brc) return cleanup(brc);
  *out = m;
  return SDB_OK;
}

int sdb_matrix_create_stencil(int device, const sdb_stencil_desc* desc, const double* diag, void* stream,
                              sdb_matrix** out) {
  SDB_REQUIRE(out != nullptr && desc != nullptr && diag != nullptr, "NULL argument");
  *out = nullptr;
  SDB_REQUIRE(desc->nx >= 1 && desc->ny >= 1 && desc->nz >= 1, "stencil grid dims must be positive");
  SDB_REQUIRE(desc->n_offsets >= 0 && desc->n_offsets <= 26, "stencil supports at most 26 off-centre points");
  int64_t n = desc->nx * desc->ny * desc->nz;
  SDB_REQUIRE(n < (1LL << 31), "stencil grid too large");
  for (int o = 0; o < desc->n_offsets; ++o)
    for (int a = 0; a < 3; ++a)
      SDB_REQUIRE(desc->offsets[o][a] >= -1 && desc->offsets[o][a] <= 1, "stencil offsets must lie in [-1,1]");
  DeviceGuard g(device);
  if (!g.ok) return fail(SDB_ECUDA, "cannot select CUDA device %d", device);
  cudaStream_t s = (cudaStream_t)stream;
  sdb_matrix* m = new sdb_matrix();
  m->device = device;
  m->format = SDB_FMT_STENCIL;
  m->n = n;
  m->nnz = n * (desc->n_offsets + 1);
  m->st.nx = desc->nx;
  m->st.ny = desc->ny;
  m->st.nz = desc->nz;
  m->st.n_off = desc->n_offsets;
  memcpy(m->st.off, desc->offsets, sizeof(m->st.off));
  memcpy(m->st.w, desc->weights, sizeof(m->st.w));
  // term table: off-centre points + the diagonal, sorted by the column offset
  // dz*nx*ny + dy*nx + dx they produce for an interior point
  const int nt = desc->n_offsets + 1;
  std::vector<int4> terms(nt);
  std::vector<double> tw(nt, 0.0);
  std::vector<int> idx(nt);
  auto flat = [&](int o) -> int64_t {
    if (o == nt - 1) return 0;
    return (int64_t)desc->offsets[o][2] * desc->nx * desc->ny + (int64_t)desc->offsets[o][1] * desc->nx +
           desc->offsets[o][0];
  };
  for (int o = 0; o < nt; ++o) idx[o] = o;
  for (int i = 1; i < nt; ++i)
    for (int j = i; j > 0 && flat(idx[j]) < flat(idx[j - 1]); --j) std::swap(idx[j], idx[j - 1]);
  for (int o = 0; o < nt; ++o) {
    const int k = idx[o];
    if (k == nt - 1) {
      terms[o] = make_int4(0, 0, 0, 0);
      m->center_pos = o;
    } else {
      terms[o] = make_int4(desc->offsets[k][0], desc->offsets[k][1], desc->offsets[k][2], (int)flat(k));
      tw[o] = desc->weights[k];
      m->mx |= desc->offsets[k][0] != 0;
      m->my |= desc->offsets[k][1] != 0;
      m->mz |= desc->offsets[k][2] != 0;
    }
  }
  m->nterms = nt;
  m->zghost = desc->z_ghost ? 1 : 0;
  for (int o = 0; o < nt; ++o) m->term_w_host[o] = tw[o];
  // shape detection: 6 face neighbours or the full 3x3x3 box, with every
  // extent >= 3 so the lexicographic term order is the sorted one
  {
    bool dims_ok = desc->nx >= 3 && desc->ny >= 3 && (desc->nz >= 3 || desc->z_ghost);
    auto has = [&](int dx, int dy, int dz) {
      for (int o = 0; o < desc->n_offsets; ++o)
        if (desc->offsets[o][0] == dx && desc->offsets[o][1] == dy && desc->offsets[o][2] == dz) return true;
      return false;
    };
    bool face = desc->n_offsets == 6 && has(-1, 0, 0) && has(1, 0, 0) && has(0, -1, 0) && has(0, 1, 0) &&
                has(0, 0, -1) && has(0, 0, 1);
    bool box = desc->n_offsets == 26;
    for (int dz = -1; box && dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx)
          if ((dx || dy || dz) && !has(dx, dy, dz)) box = false;
    m->shape = !dims_ok ? SDB_SHAPE_GENERIC : (face ? SDB_SHAPE_FACE7 : (box ? SDB_SHAPE_BOX27 : SDB_SHAPE_GENERIC));
    if (const char* env = getenv("SDB_STENCIL_GENERIC"))
      if (atoi(env)) m->shape = SDB_SHAPE_GENERIC;
  }
  cudaError_t e = cudaMalloc(&m->diag, sizeof(double) * n);
  if (e == cudaSuccess) e = cudaMalloc(&m->terms, sizeof(int4) * nt);
  if (e == cudaSuccess) e = cudaMalloc(&m->term_w, sizeof(double) * nt);
  if (e == cudaSuccess) e = cudaMemcpyAsync(m->diag, diag, sizeof(double) * n, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(m->terms, terms.data(), sizeof(int4) * nt, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(m->term_w, tw.data(), sizeof(double) * nt, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    int code = cuda_fail(e, "upload stencil", __FILE__, __LINE__);
    sdb_matrix_destroy(m);
    return code;
  }
  *out = m;
  return SDB_OK;
}

int sdb_matrix_get_info(const sdb_matrix* m, sdb_matrix_info* info) {
  SDB_REQUIRE(m != nullptr && info != nullptr, "NULL argument");
  info->n = m->n;
  info->nnz = m->nnz;
  info->format = m->format;
  info->device = m->device;
  if (m->format == SDB_FMT_CSR)
    info->bytes = 12 * m->nnz + 4 * (m->n + 1);
  else
    info->bytes = 8 * m->n;
  return SDB_OK;
}

void sdb_matrix_destroy(sdb_matrix* m) {
  if (!m) return;
  DeviceGuard g(m->device);
  if (m->rowptr) cudaFree(m->rowptr);
  if (m->colidx) cudaFree(m->colidx);
  if (m->values) cudaFree(m->values);
  if (m->diag) cudaFree(m->diag);
  if (m->terms) cudaFree(m->terms);
  if (m->term_w) cudaFree(m->term_w);
  if (m->bu) cudaFree(m->bu);
  if (m->fhdr) cudaFree(m->fhdr);
  if (m->frec) cudaFree(m->frec);
  delete m;
}

int sdb_pack_probes(const double* probes_t, int64_t n_vec, int64_t n, int64_t ldv, double* block, void* stream) {
  SDB_REQUIRE(probes_t && block, "NULL argument");
  SDB_REQUIRE(n_vec >= 1 && n >= 1 && ldv >= n_vec, "bad pack shape");
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((ldv + 31) / 32));
  pack_kernel<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>(probes_t, n_vec, n, ldv, block);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int sdb_unpack_signs(const uint8_t* bits, int64_t n_vec, int64_t n, int64_t ldv, double* block, void* stream) {
  SDB_REQUIRE(bits && block, "NULL argument");
  SDB_REQUIRE(n_vec >= 1 && n >= 1 && ldv >= n_vec && ldv % 2 == 0, "bad unpack shape");
  const int64_t total = n * (ldv / 2);
  int blocks = (int)((total + 255) / 256);
  if (blocks > 65535 * 4) blocks = 65535 * 4;
  unpack_signs_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(bits, n_vec, n, ldv, block);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

int sdb_unpack_block(const double* block, int64_t n, int64_t ldv, int64_t n_vec, double* out_t, void* stream) {
  SDB_REQUIRE(out_t && block, "NULL argument");
  SDB_REQUIRE(n_vec >= 1 && n >= 1 && ldv >= n_vec, "bad unpack shape");
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((n_vec + 31) / 32));
  unpack_kernel<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>(block, n, ldv, n_vec, out_t);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

}  // extern "C"

extern "C" int sdb_enable_peer_access(int device, int peer) {
  if (device == peer) return SDB_OK;
  int can = 0;
  SDB_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) return sdb::fail(SDB_EUNSUPPORTED, "device %d cannot access peer %d", device, peer);
  sdb::DeviceGuard dg(device);
  if (!dg.ok) return sdb::fail(SDB_ECUDA, "cannot select CUDA device %d", device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    (void)cudaGetLastError();
    return SDB_OK;
  }
  if (e != cudaSuccess) return sdb::cuda_fail(e, "cudaDeviceEnablePeerAccess", __FILE__, __LINE__);
  return SDB_OK;
}
