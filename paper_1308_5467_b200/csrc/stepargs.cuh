// stepargs.cuh — step-kernel argument block and compile-time grid shapes,
// shared by cheb.cu (row-panel / tile kernels) and zmarch.cu (TMA z-march).
#pragma once
#include "rowgroup.cuh"

namespace sdb {

struct StepArgs {
  const double* x;     // w_k                      (gathered)
  const double* prev;  // w_{k-1}                  (row-local; may alias next)
  double* next;        // w_{k+1}
  const double* v0;    // probes (direct mode dots)
  double c;            // spectral centre
  double inv_d;        // 1/halfwidth
  int64_t n;
  int64_t ldv;
  int64_t nblocks;
  int64_t panel;       // rows per panel of the phased schedule
  double* partials;    // [(M+1)][nblocks][ldv]
  int slotA;           // doubling: <w+,w+>, direct: <v0,w+>   (-1: none)
  int slotB;           // doubling: <w+,w>                       (-1: none)
  int slot0;           // step 0: <w0,w0>                        (-1: none)
  int slices;          // column slices per panel (grid kernel; 1 = whole rows)
  // Legendre recurrence (kpm.py:110-124), direct-mode kernels after step 0:
  // w_{k+1} = (la t - lb w_{k-1}) / lc with la = 2k+1, lb = k, lc = k+1
  int legendre;
  double la, lb, lc;
  // row partition (z-slabs): the step also stores its first / last own plane
  // of w_{k+1} into the neighbouring slabs' ghost planes (peer memory over
  // NVLink, or the same device); NULL: no push
  double* halo_lo;     // lower neighbour's upper ghost plane (nxy x ldv)
  double* halo_hi;     // upper neighbour's lower ghost plane
  int64_t halo_rows;   // rows per plane (nx*ny)
  int64_t last_row0;   // first row of the last own plane
  // fused two-step z-march (zmarch.cu): w_{k+2} and its moment slots
  double* next2;
  int slotA2;          // <w++,w++>  (-1: none)
  int slotB2;          // <w++,w+>   (-1: none)
};

// SDB_LEGENDRE runs the direct-mode kernels with the Legendre update.
inline int split_mode(int mode, int* legendre) {
  *legendre = mode == SDB_LEGENDRE;
  return mode == SDB_LEGENDRE ? SDB_CHEB_DIRECT : mode;
}
// Halo push of one stored double2 (row-local offset o = row*ldv + column).
__device__ __forceinline__ void halo_push(const StepArgs& a, int64_t row, int64_t col_ofs, double2 w) {
  if (a.halo_lo && row < a.halo_rows)
    *reinterpret_cast<double2*>(a.halo_lo + row * a.ldv + col_ofs) = w;
  if (a.halo_hi && row >= a.last_row0)
    *reinterpret_cast<double2*>(a.halo_hi + (row - a.last_row0) * a.ldv + col_ofs) = w;
}

inline void set_step_scalars(StepArgs& a, int64_t k) {
  a.la = (double)(2 * k + 1);
  a.lb = (double)k;
  a.lc = (double)k + 1.0;
}

// Structured-grid term order (7-point faces, 27-point box): lexicographic in
// (dz, dy, dx), which is the sorted-column order of the stencil's CSR form for
// nx, ny >= 3.
template <int SHAPE>
struct GridShape;
template <>
struct GridShape<SDB_SHAPE_FACE7> {
  static constexpr int NT = 7;
  __host__ __device__ static constexpr int dx(int o) { return o == 2 ? -1 : (o == 4 ? 1 : 0); }
  __host__ __device__ static constexpr int dy(int o) { return o == 1 ? -1 : (o == 5 ? 1 : 0); }
  __host__ __device__ static constexpr int dz(int o) { return o == 0 ? -1 : (o == 6 ? 1 : 0); }
};
template <>
struct GridShape<SDB_SHAPE_BOX27> {
  static constexpr int NT = 27;
  __host__ __device__ static constexpr int dx(int o) { return o % 3 - 1; }
  __host__ __device__ static constexpr int dy(int o) { return (o / 3) % 3 - 1; }
  __host__ __device__ static constexpr int dz(int o) { return o / 9 - 1; }
};


// ---- TMA z-march path (zmarch.cu) ------------------------------------------------
// Plan for sdb_cheb_moments on a periodic 7/27-point grid: the recurrence
// buffers are ghost-padded blocks [nz][ny+2G][nx+2G][ldv] (block_bytes each).
struct ZmPlan {
  bool on = false;
  int cfg = -1;          // tile configuration (CS, TX, TY, PPT)
  int CS = 0, TX = 0, TY = 0;
  int R = 0;             // ring slots
  int ZS = 0, n_zs = 0;  // planes per z segment, segments
  int64_t items = 0;     // work items (tile x slice x z segment)
  int64_t grid = 0;      // persistent blocks (multiple of the slice count)
  int64_t nbp = 0;       // partial rows = grid / slices
  size_t smem = 0;
  size_t block_bytes = 0;
  size_t diag_bytes = 0;   // padded diagonal (fused pairs)
  bool fuse = false;       // fused two-step launches (doubling mode)
  size_t smem2 = 0;        // their dynamic shared memory
  int R2 = 0;              // and ring depth
  int G = 1;               // ghost width of the padded blocks (2 with fused pairs)
  int z_lo = 0, z_hi = 0;  // planes computed per launch
  const char* name = "";
};
int zm_plan(const sdb_matrix* m, int64_t ldv, int mode, ZmPlan* p);
// Plan for the planes [z_lo, z_hi) only (row partition on full-size padded
// blocks: the other planes are neither read, except the two neighbour
// planes, nor written).  Off (p->on false) when the range is empty.
int zm_plan_range(const sdb_matrix* m, int64_t ldv, int mode, int64_t z_lo, int64_t z_hi, ZmPlan* p);
// w_{k+1} = step(x = w_k, prev = w_{k-1}) on padded blocks; partial rows p.nbp.
int zm_launch_step(const sdb_matrix* m, const ZmPlan& p, const StepArgs& a, bool first, int mode, cudaStream_t s);
// Fused pair of doubling-mode steps k, k+1: x = w_k, prev = w_{k-1} (unused
// when first) -> next = w_{k+1}, next2 = w_{k+2} (padded blocks distinct from
// x and prev); diag_padded from zm_pad_diag.
int zm_launch_pair(const sdb_matrix* m, const ZmPlan& p, const StepArgs& a, const double* diag_padded, bool first,
                   cudaStream_t s);
// diagonal (n) -> ghost-padded [nz][ny+4][nx+4]
int zm_pad_diag(const sdb_matrix* m, double* padded, cudaStream_t s);

// ---- probe-sliced band + far path (band.cu) --------------------------------------
// Plan for sdb_cheb_moments on a CSR matrix with a dense symmetric band: the
// recurrence buffers are slice-major blocks [ns][rows][S] (S probes per
// slice, `pad` zero guard rows before and after the n_pad tile rows).
struct BandPlan {
  bool on = false;
  int hb = 0;              // band half-width (kernel instantiation)
  int S = 16;              // probe columns per slice (8 or 16)
  int R = 128;             // rows per tile
  int ns = 0;              // probe slices
  int64_t ldvb = 0;        // ns * S: partials row width
  int64_t rows = 0;        // rows per slice incl. guards
  int64_t ntiles = 0;      // 128-row tiles per slice
  int64_t grid = 0;        // persistent blocks (= partial rows)
  size_t smem = 0;
  size_t block_bytes = 0;  // one slice-major block
};
int band_plan(const sdb_matrix* m, int64_t n_vec, int mode, BandPlan* p);
// probes (n x ldv row-major) -> slice-major v0b; zero the guard rows of bufA/bufB
int band_pack(const sdb_matrix* m, const BandPlan& p, const double* probes, int64_t ldv, double* v0b, double* bufA,
              double* bufB, cudaStream_t s);
int band_launch_step(const sdb_matrix* m, const BandPlan& p, const StepArgs& a, bool first, int mode, cudaStream_t s);
// ---- cluster-resident recurrence for small CSR matrices (resident.cu) ---------------
// The whole recurrence in one launch: clusters of CL CTAs own column groups,
// each CTA keeps its rows of w_k / w_{k-1} and its CSR slice in shared memory.
struct ResPlan {
  bool on = false;
  int CL = 0;              // CTAs per cluster (row blocks)
  int lpr = 0;             // lanes per row: 2 * lpr probe columns per cluster
  int R = 0;               // rows per CTA
  int nnz_cap = 0;         // CSR entries staged per CTA
  int64_t clusters = 0;
  int64_t nblocks = 0;     // partial rows (CL * warps per CTA)
  size_t smem = 0;
};
int res_plan(const sdb_matrix* m, int64_t n_vec, int mode, ResPlan* p);
// all steps of the moment run; partials [(degree+1)][p.nblocks][ldv]
int res_launch(const sdb_matrix* m, const ResPlan& p, const StepArgs& a, int64_t degree, int mode,
               const double* probes, double* partials, cudaStream_t s);
// probes (n x ldv) -> padded block
int zm_pad(const sdb_matrix* m, const ZmPlan& p, const double* probes, int64_t ldv, double* padded, cudaStream_t s);

}  // namespace sdb
