// band.cu — probe-sliced band + far Chebyshev step for banded-plus-random CSR
// matrices (BASELINE config 3: a band of half-width 20 plus ~20 random
// off-band entries per row, n = 1e6, 128 probes).
//
// Reference hot loop: kpm.py:96-107 / kpm.py:174-189 with B x = (A x - c x)/d
// (matrix.py:125-126) and A x = csr @ x (matrix.py:101-102).
//
// Why a separate path.  With the probe block row-major (n x 128 fp64, 1 KB per
// row) the ~20 random columns of a row are 20 random 1 KB gathers from a 1 GB
// block that cannot stay in the 126 MB L2: the CSR kernel moves ~27 GB of DRAM
// per step against 3.8 GB of compulsory bytes.  Here
//   * the probe block is slice-major, [ns][rows][16]: one slice of 16 probes
//     is n x 128 B = 128 MB, and the whole grid works through one slice at a
//     time, so about half of a slice's random gathers hit L2 (measured on
//     B200, tools/mb/c3_probe.cu: 128 B gathers from a 128 MB slice run at
//     ~10-15 TB/s, from the 1 GB block at ~5 TB/s);
//   * the dense band is split off at upload (band_build): symmetric, so only
//     its upper diagonals are stored (values only, no indices: 8 B per entry
//     for half the band);
//   * the remaining (far) entries are stored SELL-C-sigma style (C = 4,
//     sigma = 128): per 128-row tile the rows are sorted by far count, cut
//     into 4-row chunks and dealt to 16 streams, one per gather warp; a stream
//     is a run of batch records (4 slots x 4 rows) so that a warp (8 lanes per
//     row x 4 rows) gathers one slot with one 16-byte load per lane.
//
// The step kernel is warp-specialised, one persistent 20-warp block per SM:
//   * 16 far warps walk their streams through a per-warp shared-memory ring of
//     NB batches x 4 slots of outstanding 16-byte cp.async gathers per lane
//     (NB = 3: 6 KB per warp, 96 KB per SM in flight; a step of the walk is a
//     ~500-cycle dependent chain, so the warp count sets the gather rate) -- the gathers are
//     latency-bound, and cp.async groups are the one completion mechanism with
//     an in-order counted wait (a register ring of plain loads ends up on a
//     single scoreboard, measured: every consume waits for the newest load);
//     the ring keeps the memory system busy without pausing at tile
//     boundaries.  The batch records arrive through a second small ring.  Far
//     sums of a chunk's rows go to a double-buffered shared tile (yfar).
//   * 4 band warps take a tile's x window, band diagonals and w_{k-1} rows
//     from bulk async copies (TMA engine, mbarrier completion), start each
//     row's sum from yfar, add the band with a register
//     sliding window (8 rows x 2 probe columns per thread), and run the fused
//     epilogue: spectral map, 2 t - w_{k-1} (or the Legendre update), store,
//     moment dots.
// A row's sum runs far entries (column order) -> band (d = -hb..hb); the CSR
// kernel runs in pure column order, so w agrees to rounding (1e-16 relative),
// not bit for bit.  Dot partials go to [(M+1)][grid][ldvb] and are reduced by
// K2 in fixed order (deterministic: the tile schedule is static).
#include <cub/cub.cuh>

#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "stepargs.cuh"
#include "tma.cuh"

namespace sdb {

constexpr int kBandS = 16;          // probe columns per slice
constexpr int kBandR = 128;         // rows per tile (sigma)
constexpr int kFarWarps = 16;       // gather warps = far streams per tile
constexpr int kBandWarps = 4;       // band / epilogue warps
constexpr int kBandThreads = 32 * (kFarWarps + kBandWarps);
constexpr int kBandRT = 8;          // rows per band thread
constexpr int kBandTileAlign = 256; // rows are padded to this
constexpr int kBandMaxOff = 64;     // offsets histogrammed for the band search
constexpr int kChunksPerTile = kBandR / 4;
// far batch record: int32 col[4 rows][4 slots] (-1: padding slot, no gather) |
// double val[4][4] | u32 flags (1: last batch of its chunk, 2: last batch of
// the tile's stream, 4: end of all streams) | u8 rows[4] | pad.  One extra
// record with flag 4 follows the last stream (every warp ends on it).
constexpr int kRecBytes = 208;
constexpr int kRecVal = 64, kRecMeta = 192;
constexpr uint32_t kRecChunkEnd = 1, kRecTileEnd = 2, kRecStop = 4;
// per-warp record ring in shared memory (slots padded to 256 bytes)
constexpr int kSlotBytes = 256;
constexpr int kRecRing = 8;         // slots (> kRecAhead + NB)
constexpr int kRecAhead = 4;        // records are requested this many batches before their gathers are issued

// band half-widths with a kernel instantiation (the detected band is rounded up)
constexpr int kBandWidths[] = {8, 16, 20, 24, 32};

// ---- device helpers -----------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ double2 lds2(const void* p) { return *reinterpret_cast<const double2*>(p); }
// L2 policies: the x slice being gathered is kept (evict_last); everything
// streamed once per slice pass (band diagonals, far records, w_{k-1}, v0,
// w_{k+1}) is evict_first, so the data streamed per pass does not push the
// slice out of L2 between its ~21 reuses.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_x_keep(const double* p, uint64_t pol) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p), "l"(pol));
  return r;
}
// 1-D bulk async copy global -> shared (TMA engine), completion on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes, uint64_t pol) {
  if (bytes)
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void band_bar_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kBandWarps) : "memory"); }

struct BandArgs {
  const double* x;      // slice-major blocks, base of slice 0 (guard row 0)
  const double* prev;
  double* next;
  const double* v0;
  int64_t sstride;      // doubles per slice
  const double* bu;     // [hb+1][ustride]
  int64_t ustride;
  const int2* fhdr;     // [ntiles][kFarWarps]
  const char* frec;
  int64_t stop_rec;     // index of the stop record (after the last stream)
  double c, inv_d;
  int64_t n;
  int ntiles, nslices;
  int64_t ldv;          // partials row width (nslices * S)
  double* partials;
  int64_t nblocks;
  int slotA, slotB, slot0;
  int legendre;
  double la, lb, lc;
  uint64_t keep_pol, once_pol;  // L2 evict_last / evict_first policies (made once per device, band_policies)
  int diag;             // diagnostics (SDB_BAND_DIAG): 4 skip the band, 8 no stage loads, 16 no far
                        // warps (wrong results; timing only)
};

template <int HB, int NB>
struct BandSmem {
  static constexpr int P = band_pad(HB);
  static constexpr int XW = kBandR + 2 * P;   // x window rows
  static constexpr int UW = kBandR + P;       // diagonal window entries
  static constexpr size_t kBars = 0;                                  // 5 mbarriers
  static constexpr size_t kRed = 128;                                 // 16 x 16 doubles
  static constexpr size_t kRing = kRed + 16 * kBandS * sizeof(double);
  static constexpr size_t kWarpData = (size_t)NB * 4 * 32 * 16;       // gather ring of one far warp
  static constexpr size_t kData = kRing + (size_t)kFarWarps * kRecRing * kSlotBytes;
  static constexpr size_t kYfar = kData + kFarWarps * kWarpData;
  static constexpr size_t kStage = kYfar + 2 * (size_t)kBandR * kBandS * sizeof(double);
  static constexpr size_t kXs = 0;
  static constexpr size_t kUs = (size_t)XW * kBandS * sizeof(double);
  static constexpr size_t kPv = kUs + (size_t)(HB + 1) * UW * sizeof(double);
  static constexpr size_t kStageBytes = kPv + (size_t)kBandR * kBandS * sizeof(double);
  static constexpr size_t kTotal = kStage + kStageBytes;
  static_assert(kTotal <= 227 * 1024, "band step shared memory exceeds the 227 KB per block limit");
};
// gather ring depth per band half-width (shared memory budget)
template <int HB>
struct BandDepth {
  static constexpr int kDefault = HB > 20 ? 2 : 3;
};

// ---- far warps ------------------------------------------------------------------
// Warp w of the block walks stream w of every tile the block owns.  Per loop
// step (one batch = 4 slots): wait until the cp.async group of NB steps ago
// has landed, consume that batch from ring slot bb (own lane's 16 bytes per
// slot), request the record kRecAhead batches ahead of its gathers, issue the
// gathers of the batch NB ahead into the same ring slot, commit the group.
// The step is kept short (~50 instructions: the walk is issue-bound, measured):
// running pointers, item changes on cold paths, padding slots predicated off
// (the ring starts zeroed and only ever holds x values, so weight 0 times the
// stale entry is 0).
struct FarCursor {
  int item;         // item (slice * ntiles + tile) being requested / issued
  int left;         // records left in it
};

template <int NB>
__device__ __forceinline__ void band_far_warp(const BandArgs& a, int w, int lane, char* ring, char* dring,
                                              double* yfar, uint64_t* full, uint64_t* empty, int P) {
  static_assert(kRecRing > kRecAhead + NB, "record ring too small");
  static_assert((kRecRing & (kRecRing - 1)) == 0 && kSlotBytes == 256, "ring offsets are (it << 8) & mask");
  constexpr int kPending = (NB < kRecAhead ? NB : kRecAhead) - 1;
  constexpr int kMask = (kRecRing - 1) * kSlotBytes;
  const int g = lane >> 3, q = lane & 7;
  const uint64_t keep = a.keep_pol, once = a.once_pol;
  const int G = gridDim.x;
  const int total = a.nslices * a.ntiles;
  const char* const stop_rec = a.frec + a.stop_rec * kRecBytes + lane * 16;
  // ---- request cursor: this lane's 16 bytes of the next record to fetch
  FarCursor rq{(int)blockIdx.x, 0};
  const char* rp = stop_rec;
  int rstride = 0;
  int2 nh = make_int2(0, 0);  // header of the item after rq.item
  auto load_header = [&](int item) { return __ldg(a.fhdr + (item % a.ntiles) * kFarWarps + w); };
  if (rq.item < total) {
    const int2 h = load_header(rq.item);
    rp = a.frec + (int64_t)h.x * kRecBytes + lane * 16;
    rstride = kRecBytes;
    rq.left = h.y;
    if (rq.item + G < total) nh = load_header(rq.item + G);
  }
  auto next_request_item = [&]() {  // cold: once per tile
    rq.item += G;
    if (rq.item < total) {
      rp = a.frec + (int64_t)nh.x * kRecBytes + lane * 16;
      rq.left = nh.y;
      if (rq.item + G < total) {
        nh = load_header(rq.item + G);
        if (lane == 0) l2_prefetch(a.frec + (int64_t)nh.x * kRecBytes, (uint32_t)nh.y * kRecBytes, once);
      }
    } else {
      rp = stop_rec;
      rstride = 0;
      rq.left = 0x7fffffff;
    }
  };
  auto request = [&](int it) {
    if (lane < kRecBytes / 16) cp_async16(ring + ((it << 8) & kMask) + lane * 16, rp, once);
    rp += rstride;
    if (--rq.left == 0) next_request_item();
  };
  // ---- issue cursor: x rows of the slice the issued records belong to
  int is_item = blockIdx.x;
  const double* xrow = a.x + (int64_t)(is_item / a.ntiles) * a.sstride + (int64_t)P * kBandS + 2 * q;
  // the gather ring starts zeroed (padding slots are never written)
  char* mine = dring + lane * 16;  // this lane's 16 bytes of every ring slot
#pragma unroll
  for (int k = 0; k < NB * 4; ++k) *reinterpret_cast<double2*>(mine + k * 512) = make_double2(0.0, 0.0);
  double2 acc = make_double2(0.0, 0.0);
  int seq = 0;  // tiles finished by this warp
  int it = 0;
  for (; it < kRecAhead; ++it) {
    request(it);
    cp_async_commit();
  }
  // one step of the walk; CONSUME is false for the first NB steps (nothing gathered yet)
  auto step = [&](int bb, auto consume_tag) -> bool {
    constexpr bool CONSUME = decltype(consume_tag)::value;
    cp_async_wait<kPending>();
    __syncwarp();
    // every shared-memory operand of this step is requested up front (the
    // addresses depend on `it` only), so the step pays one LDS round trip
    const char* recC = ring + (((it - kRecAhead - NB) << 8) & kMask);
    const char* recI = ring + (((it - kRecAhead) << 8) & kMask);
    const uint32_t flagsI = *reinterpret_cast<const uint32_t*>(recI + kRecMeta);
    const int4 c4 = *reinterpret_cast<const int4*>(recI + g * 16);
    if (CONSUME) {
      const uint2 meta = *reinterpret_cast<const uint2*>(recC + kRecMeta);
      const double2 v01 = lds2(recC + kRecVal + g * 32), v23 = lds2(recC + kRecVal + g * 32 + 16);
      const double2 g0 = lds2(mine + (bb * 4 + 0) * 512), g1 = lds2(mine + (bb * 4 + 1) * 512),
                    g2 = lds2(mine + (bb * 4 + 2) * 512), g3 = lds2(mine + (bb * 4 + 3) * 512);
      acc.x = fma(v01.x, g0.x, acc.x);
      acc.y = fma(v01.x, g0.y, acc.y);
      acc.x = fma(v01.y, g1.x, acc.x);
      acc.y = fma(v01.y, g1.y, acc.y);
      acc.x = fma(v23.x, g2.x, acc.x);
      acc.y = fma(v23.x, g2.y, acc.y);
      acc.x = fma(v23.y, g3.x, acc.x);
      acc.y = fma(v23.y, g3.y, acc.y);
      if (meta.x) {  // cold: ~1 step in 5
        if (meta.x & kRecStop) return false;
        // chunk done: its rows' far sums go to the shared tile
        const int row = (meta.y >> (8 * g)) & 255;
        *reinterpret_cast<double2*>(yfar + ((size_t)(seq & 1) * kBandR + row) * kBandS + 2 * q) = acc;
        acc = make_double2(0.0, 0.0);
        if (meta.x & kRecTileEnd) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[seq & 1]);
          ++seq;
          const int use = seq >> 1;  // the next tile's buffer must have been read by the band warps
          if (use > 0) mbar_wait(&empty[seq & 1], (use - 1) & 1);
        }
      }
    }
    request(it);
    if (c4.x >= 0) cp_async16(mine + (bb * 4 + 0) * 512, xrow + (int64_t)(uint32_t)c4.x * kBandS, keep);
    if (c4.y >= 0) cp_async16(mine + (bb * 4 + 1) * 512, xrow + (int64_t)(uint32_t)c4.y * kBandS, keep);
    if (c4.z >= 0) cp_async16(mine + (bb * 4 + 2) * 512, xrow + (int64_t)(uint32_t)c4.z * kBandS, keep);
    if (c4.w >= 0) cp_async16(mine + (bb * 4 + 3) * 512, xrow + (int64_t)(uint32_t)c4.w * kBandS, keep);
    cp_async_commit();
    if (flagsI & kRecTileEnd) {  // cold: the next issued record belongs to the block's next tile
      is_item += G;
      if (is_item < total)
        xrow = a.x + (int64_t)(is_item / a.ntiles) * a.sstride + (int64_t)P * kBandS + 2 * q;
    }
    ++it;
    return true;
  };
#pragma unroll
  for (int bb = 0; bb < NB; ++bb) step(bb, std::false_type{});
  for (;;) {
#pragma unroll
    for (int bb = 0; bb < NB; ++bb)
      if (!step(bb, std::true_type{})) return;
  }
}

// ---- band warps -------------------------------------------------------------------
// Band rows rl .. rl+RT-1 of the tile: for d = -HB..HB (increasing column),
// acc[r] += A[i][i+d] x[i+d] with A[i][i+d] = bu[d][i] (d >= 0) or
// bu[-d][i+d] (d < 0, symmetry); x rows come from the staged window through
// a register sliding window (one new row per diagonal).
template <int HB>
__device__ __forceinline__ void band_diag(const double* xs, const double* us, int rl, int q,
                                          double2 (&acc)[kBandRT]) {
  constexpr int P = band_pad(HB), RT = kBandRT, UW = kBandR + P, S = kBandS;
  double2 win[RT];
#pragma unroll
  for (int r = 0; r < RT; ++r) win[r] = lds2(xs + (rl + P - HB + r) * S + 2 * q);
#pragma unroll
  for (int d = -HB; d <= HB; ++d) {
    double v[RT];
    const double* vp = d >= 0 ? us + d * UW + P + rl : us + (-d) * UW + P + rl + d;
    if (d >= 0 || (d & 1) == 0) {
#pragma unroll
      for (int r = 0; r < RT; r += 2) {
        const double2 t = lds2(vp + r);
        v[r] = t.x;
        v[r + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int r = 0; r < RT; ++r) v[r] = vp[r];
    }
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      acc[r].x = fma(v[r], win[r].x, acc[r].x);
      acc[r].y = fma(v[r], win[r].y, acc[r].y);
    }
    if (d < HB) {
#pragma unroll
      for (int r = 0; r < RT - 1; ++r) win[r] = win[r + 1];
      win[RT - 1] = lds2(xs + (rl + P + d + RT) * S + 2 * q);
    }
  }
}

template <int HB, int MODE, bool FIRST, int NB>
__device__ __forceinline__ void band_band_warps(const BandArgs& a, int tb, char* smem, uint64_t* sfull,
                                                uint64_t* full, uint64_t* empty) {
  using L = BandSmem<HB, NB>;
  constexpr int P = L::P, R = kBandR, RT = kBandRT, S = kBandS, XW = L::XW, UW = L::UW;
  const int lane = tb & 31, wb = tb >> 5;
  const int g8 = tb >> 3, q = tb & 7, rl = g8 * RT;
  const uint64_t once = a.once_pol, keep = a.keep_pol;
  const int G = gridDim.x, b = blockIdx.x;
  const int total = a.nslices * a.ntiles;
  double* red = reinterpret_cast<double*>(smem + L::kRed);
  const double* yfar = reinterpret_cast<const double*>(smem + L::kYfar);
  // bulk copies of one tile's operands, spread over the lanes of band warp 0
  char* st = smem + L::kStage;
  auto issue = [&](int item) {
    const int s = item / a.ntiles, t = item - s * a.ntiles;
    const int64_t r0 = (int64_t)t * R;
    constexpr uint32_t bytes = XW * S * 8 + (HB + 1) * UW * 8 + (FIRST ? 0 : R * S * 8);
    if (lane == 0) {
      mbar_expect_tx(sfull, bytes);
      bulk_g2s(st + L::kXs, a.x + s * a.sstride + r0 * S, XW * S * 8, sfull, keep);
      if (!FIRST) bulk_g2s(st + L::kPv, a.prev + s * a.sstride + (P + r0) * S, R * S * 8, sfull, once);
    }
    for (int d = lane; d <= HB; d += 32)
      bulk_g2s(st + L::kUs + (size_t)d * UW * 8, a.bu + d * a.ustride + r0, UW * 8, sfull, once);
  };
  // per-slice partial rows: the 16 row groups summed in order (deterministic)
  auto flush = [&](const double2& acc, int slot, int s) {
    red[g8 * S + 2 * q] = acc.x;
    red[g8 * S + 2 * q + 1] = acc.y;
    band_bar_sync();
    if (tb < S) {
      double sum = 0.0;
#pragma unroll
      for (int gg = 0; gg < R / RT; ++gg) sum += red[gg * S + tb];
      a.partials[((int64_t)slot * a.nblocks + b) * a.ldv + s * S + tb] = sum;
    }
    band_bar_sync();
  };
  double2 accA = make_double2(0.0, 0.0), accB = accA, accZ = accA;
  auto flush_slice = [&](int s) {
    if (a.slotA >= 0) flush(accA, a.slotA, s);
    if (MODE == SDB_CHEB_DOUBLING && a.slotB >= 0) flush(accB, a.slotB, s);
    if (FIRST && a.slot0 >= 0) flush(accZ, a.slot0, s);
    accA = accB = accZ = make_double2(0.0, 0.0);
  };
  // every block writes a partial row for every slice (zeros when it owns no
  // tile of a slice), so the K2 reduce never reads an unwritten row
  int cur_s = 0, seq = 0;
  for (int item = b; item < total; item += G, ++seq) {
    const int buf = seq & 1, ph = (seq >> 1) & 1;
    const int s = item / a.ntiles, t = item - s * a.ntiles;
    for (; cur_s < s; ++cur_s) flush_slice(cur_s);
    // the stage buffer is free: every band warp passed the barrier that ends
    // the previous tile (the band warps have slack, the far warps set the pace)
    if (wb == 0 && !(a.diag & 8)) issue(item);
    const double* xs = reinterpret_cast<const double*>(st + L::kXs);
    const double* us = reinterpret_cast<const double*>(st + L::kUs);
    const double* pv = reinterpret_cast<const double*>(st + L::kPv);
    const int64_t row0 = (int64_t)t * R + rl;
    const int64_t so = s * a.sstride + (int64_t)P * S;  // row 0 of slice s
    double2 p0[RT];
    if (MODE == SDB_CHEB_DIRECT && !FIRST) {
#pragma unroll
      for (int r = 0; r < RT; ++r)
        p0[r] = row0 + r < a.n ? ld_d2_once(a.v0 + so + (row0 + r) * S + 2 * q, once) : make_double2(0.0, 0.0);
    }
    double2 acc[RT];
    if (!(a.diag & 16)) mbar_wait(&full[buf], ph);
#pragma unroll
    for (int r = 0; r < RT; ++r) acc[r] = lds2(yfar + ((size_t)buf * R + rl + r) * S + 2 * q);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[buf]);
    if (!(a.diag & 8)) mbar_wait(sfull, seq & 1);
    if (!(a.diag & 4)) band_diag<HB>(xs, us, rl, q, acc);
    // epilogue: t = (A x - c x)/d; w+ = t | 2t - w- | Legendre; dots
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      const int64_t row = row0 + r;
      if (row < a.n) {
        const double2 xi = lds2(xs + (rl + P + r) * S + 2 * q);
        const int64_t o = so + row * S + 2 * q;
        if (FIRST || MODE != SDB_CHEB_DIRECT) p0[r] = xi;
        const double tx = (acc[r].x - a.c * xi.x) * a.inv_d;
        const double ty = (acc[r].y - a.c * xi.y) * a.inv_d;
        double2 wn;
        if (FIRST) {
          wn = make_double2(tx, ty);
        } else {
          const double2 wp = lds2(pv + (rl + r) * S + 2 * q);
          if (MODE == SDB_CHEB_DIRECT && a.legendre) {
            wn.x = (a.la * tx - a.lb * wp.x) / a.lc;
            wn.y = (a.la * ty - a.lb * wp.y) / a.lc;
          } else {
            wn.x = 2.0 * tx - wp.x;
            wn.y = 2.0 * ty - wp.y;
          }
        }
        st_d2_once(a.next + o, wn, once);
        if (MODE == SDB_CHEB_DOUBLING) {
          accA.x += wn.x * wn.x;
          accA.y += wn.y * wn.y;
          accB.x += wn.x * xi.x;
          accB.y += wn.y * xi.y;
        } else {
          accA.x += p0[r].x * wn.x;
          accA.y += p0[r].y * wn.y;
        }
        if (FIRST) {
          accZ.x += xi.x * xi.x;
          accZ.y += xi.y * xi.y;
        }
      }
    }
    band_bar_sync();  // every band warp is done with this stage buffer
  }
  for (; cur_s < a.nslices; ++cur_s) flush_slice(cur_s);
}

template <int HB, int MODE, bool FIRST, int NB>
__global__ void __launch_bounds__(kBandThreads, 1) cheb_step_band(BandArgs a) {
  using L = BandSmem<HB, NB>;
  extern __shared__ __align__(128) char band_smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(band_smem + L::kBars);
  uint64_t* sfull = bars;       // stage buffer filled (bulk copies)
  uint64_t* full = bars + 2;    // [2] yfar tile written by the far warps
  uint64_t* empty = bars + 4;   // [2] yfar tile read by the band warps
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(sfull, 1);
    mbar_init(&full[0], kFarWarps);
    mbar_init(&full[1], kFarWarps);
    mbar_init(&empty[0], kBandWarps);
    mbar_init(&empty[1], kBandWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  // (setmaxnreg to move registers from the far warps to the band warps gave
  // an illegal-instruction fault in this kernel, cause not found --
  // tools/mb/setmaxnreg.cu runs the same pattern fine; at 96 registers the
  // band warps spill only for half-widths 24 and 32)
  if (warp < kBandWarps) {
    band_band_warps<HB, MODE, FIRST, NB>(a, tid, band_smem, sfull, full, empty);
    return;
  }
  if (!(a.diag & 16)) {
    const int w = warp - kBandWarps;
    band_far_warp<NB>(a, w, lane, band_smem + L::kRing + (size_t)w * kRecRing * kSlotBytes,
                      band_smem + L::kData + (size_t)w * L::kWarpData,
                      reinterpret_cast<double*>(band_smem + L::kYfar), full, empty, L::P);
  }
}

// ---- probe packing ----------------------------------------------------------------
// probes (n x ldv row-major) -> v0b [ns][rows][S] with zero guard / padding
// rows and columns; the same rows of bufA / bufB are zeroed (never written by
// the step kernel, read through the x windows).
__global__ void band_pack_kernel(const double* __restrict__ in, int64_t n, int64_t ldv, int S, int ns, int64_t rows,
                                 int pad, double* __restrict__ v0b, double* __restrict__ bufA,
                                 double* __restrict__ bufB) {
  const int half = S / 2;
  const int64_t total = (int64_t)ns * rows * half;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c2 = (int)(idx % half);
    const int64_t rr = (idx / half) % rows;
    const int s = (int)(idx / ((int64_t)half * rows));
    const int64_t i = rr - pad;
    const int64_t col = (int64_t)s * S + 2 * c2;
    const bool inside = i >= 0 && i < n;
    double2 v = make_double2(0.0, 0.0);
    if (inside && col < ldv) v = *reinterpret_cast<const double2*>(in + i * ldv + col);
    const int64_t o = ((int64_t)s * rows + rr) * S + 2 * c2;
    *reinterpret_cast<double2*>(v0b + o) = v;
    if (!inside) {
      *reinterpret_cast<double2*>(bufA + o) = make_double2(0.0, 0.0);
      *reinterpret_cast<double2*>(bufB + o) = make_double2(0.0, 0.0);
    }
  }
}

// ---- split construction (one-time, at upload) ---------------------------------------
__global__ void band_hist_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t n,
                                 unsigned long long* __restrict__ hist, int* __restrict__ unsorted) {
  // hist[0..kBandMaxOff]: entries with j - i = d (upper), hist[kBandMaxOff+1+d]: i - j = d (lower)
  __shared__ unsigned int h[2 * (kBandMaxOff + 1)];
  for (int k = threadIdx.x; k < 2 * (kBandMaxOff + 1); k += blockDim.x) h[k] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int prev = -1;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int j = ci[k];
      if (j <= prev) *unsorted = 1;
      prev = j;
      const int64_t d = (int64_t)j - i;
      if (d >= 0 && d <= kBandMaxOff) atomicAdd(&h[d], 1u);
      else if (d < 0 && -d <= kBandMaxOff) atomicAdd(&h[kBandMaxOff + 1 - d], 1u);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 2 * (kBandMaxOff + 1); k += blockDim.x)
    if (h[k]) atomicAdd(&hist[k], (unsigned long long)h[k]);
}

// upper band -> bu
__global__ void band_fill_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 const double* __restrict__ va, int64_t n, int hb, int pad, int64_t ustride,
                                 double* __restrict__ bu) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int64_t d = (int64_t)ci[k] - i;
      if (d >= 0 && d <= hb) bu[d * ustride + pad + i] = va[k];
    }
  }
}

// every lower band entry must equal its mirrored upper entry bit for bit
__global__ void band_sym_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double* __restrict__ va, int64_t n, int hb, int pad, int64_t ustride,
                                const double* __restrict__ bu, int* __restrict__ asym) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int64_t j = ci[k], d = i - j;
      if (d >= 1 && d <= hb) {
        const double u = bu[d * ustride + pad + j];
        if (__double_as_longlong(u) != __double_as_longlong(va[k])) *asym = 1;
      }
    }
  }
}

// Far streams of one tile (one block of kBandR threads per tile).  Rows are
// ranked by far count (descending, ties by row: sigma = 128 sorting), chunk
// c holds the ranks 4c..4c+3 and needs max(1, ceil(count(rank 4c)/4)) batch
// records; chunk c goes to stream w(c) as its k(c)-th chunk, dealt in snake
// order so the streams carry about the same number of records.
__device__ __forceinline__ int band_chunk_stream(int c) {
  const int quad = c / kFarWarps, idx = c % kFarWarps;
  return (quad & 1) ? kFarWarps - 1 - idx : idx;
}
struct BandTileSort {
  int cnt[kBandR];
  int row_of_rank[kBandR];
  int nrec[kChunksPerTile];
};
// counts and ranks of the calling block's tile; returns this thread's far count
__device__ __forceinline__ int band_tile_sort(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                              int64_t n, int hb, int64_t tile, BandTileSort& sh, int* my_rank) {
  const int p = threadIdx.x;
  const int64_t i = tile * kBandR + p;
  int cnt = 0;
  if (i < n)
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int64_t d = (int64_t)ci[k] - i;
      cnt += (d < -hb || d > hb);
    }
  sh.cnt[p] = cnt;
  __syncthreads();
  int rank = 0;
  for (int o = 0; o < kBandR; ++o) {
    const int co = sh.cnt[o];
    rank += (co > cnt) || (co == cnt && o < p);
  }
  sh.row_of_rank[rank] = p;
  __syncthreads();
  if (p < kChunksPerTile) {
    const int len = sh.cnt[sh.row_of_rank[4 * p]];
    sh.nrec[p] = len > 0 ? (len + 3) / 4 : 1;
  }
  __syncthreads();
  *my_rank = rank;
  return cnt;
}

__global__ void __launch_bounds__(kBandR) band_far_count_kernel(const int32_t* __restrict__ rp,
                                                                const int32_t* __restrict__ ci, int64_t n, int hb,
                                                                int32_t* __restrict__ stream_recs,
                                                                unsigned long long* __restrict__ far_nnz) {
  __shared__ BandTileSort sh;
  __shared__ int tot;
  if (threadIdx.x == 0) tot = 0;
  int rank;
  const int cnt = band_tile_sort(rp, ci, n, hb, blockIdx.x, sh, &rank);
  if (cnt) atomicAdd(&tot, cnt);
  if (threadIdx.x < kFarWarps) {
    int sum = 0;
    for (int c = 0; c < kChunksPerTile; ++c)
      if (band_chunk_stream(c) == (int)threadIdx.x) sum += sh.nrec[c];
    stream_recs[(int64_t)blockIdx.x * kFarWarps + threadIdx.x] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0 && tot) atomicAdd(far_nnz, (unsigned long long)tot);
}

__global__ void __launch_bounds__(kBandR) band_far_fill_kernel(const int32_t* __restrict__ rp,
                                                               const int32_t* __restrict__ ci,
                                                               const double* __restrict__ va, int64_t n, int hb,
                                                               const int32_t* __restrict__ stream_off,
                                                               int2* __restrict__ fhdr, char* __restrict__ frec,
                                                               int64_t stop_rec) {
  __shared__ BandTileSort sh;
  int rank;
  band_tile_sort(rp, ci, n, hb, blockIdx.x, sh, &rank);
  const int p = threadIdx.x;
  const int64_t i = (int64_t)blockIdx.x * kBandR + p;
  const int c = rank / 4, g = rank % 4;
  const int w = band_chunk_stream(c), kq = c / kFarWarps;
  // first record of this chunk: stream start + records of the stream's earlier chunks
  int64_t rec0 = stream_off[(int64_t)blockIdx.x * kFarWarps + w];
  for (int k2 = 0; k2 < kq; ++k2) {
    const int c2 = k2 * kFarWarps + ((k2 & 1) ? kFarWarps - 1 - w : w);
    rec0 += sh.nrec[c2];
  }
  const int nrec = sh.nrec[c];
  int e = 0;
  if (i < n)
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int64_t d = (int64_t)ci[k] - i;
      if (d < -hb || d > hb) {
        char* rec = frec + (rec0 + e / 4) * kRecBytes;
        reinterpret_cast<int32_t*>(rec)[g * 4 + (e & 3)] = ci[k];
        reinterpret_cast<double*>(rec + kRecVal)[g * 4 + (e & 3)] = va[k];
        ++e;
      }
    }
  for (; e < 4 * nrec; ++e) {  // padding slots: no gather (column -1), weight 0
    char* rec = frec + (rec0 + e / 4) * kRecBytes;
    reinterpret_cast<int32_t*>(rec)[g * 4 + (e & 3)] = -1;
    reinterpret_cast<double*>(rec + kRecVal)[g * 4 + (e & 3)] = 0.0;
  }
  if (g == 0) {
    uint32_t rows = 0;
    for (int r = 0; r < 4; ++r) rows |= (uint32_t)sh.row_of_rank[4 * c + r] << (8 * r);
    for (int k = 0; k < nrec; ++k) {
      uint32_t* meta = reinterpret_cast<uint32_t*>(frec + (rec0 + k) * kRecBytes + kRecMeta);
      const bool last = k == nrec - 1;
      meta[0] = (last ? kRecChunkEnd : 0u) | ((last && kq == kChunksPerTile / kFarWarps - 1) ? kRecTileEnd : 0u);
      meta[1] = rows;
      meta[2] = meta[3] = 0u;
    }
  }
  if (p < kFarWarps) {
    int sum = 0;
    for (int c2 = 0; c2 < kChunksPerTile; ++c2)
      if (band_chunk_stream(c2) == p) sum += sh.nrec[c2];
    fhdr[(int64_t)blockIdx.x * kFarWarps + p] = make_int2(stream_off[(int64_t)blockIdx.x * kFarWarps + p], sum);
  }
  if (blockIdx.x == 0 && p < kRecBytes / 4) {  // the stop record
    uint32_t* rec = reinterpret_cast<uint32_t*>(frec + stop_rec * kRecBytes);
    rec[p] = p < 16 ? 0xffffffffu : (p == kRecMeta / 4 ? kRecStop : 0u);
  }
}

static bool band_env_enabled() {
  const char* e = getenv("SDB_BAND");
  return !(e && e[0] == '0');
}

int band_build(sdb_matrix* m, cudaStream_t s) {
  if (m->format != SDB_FMT_CSR || m->nnz == 0 || m->n < 2 * kBandTileAlign || !band_env_enabled()) return SDB_OK;
  const int64_t n = m->n;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 4LL * num_sms(m->device));
  unsigned long long* hist = nullptr;
  int* flags = nullptr;  // [0] unsorted/duplicate, [1] asymmetric
  SDB_CUDA(cudaMalloc(&hist, sizeof(unsigned long long) * 2 * (kBandMaxOff + 1)));
  SDB_CUDA(cudaMalloc(&flags, 2 * sizeof(int)));
  struct Free {
    void* p[2];
    ~Free() {
      for (void* x : p)
        if (x) cudaFree(x);
    }
  } fr{{hist, flags}};
  SDB_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * 2 * (kBandMaxOff + 1), s));
  SDB_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), s));
  band_hist_kernel<<<blocks, 256, 0, s>>>(m->rowptr, m->colidx, n, hist, flags);
  SDB_CHECK_LAUNCH();
  std::vector<unsigned long long> h(2 * (kBandMaxOff + 1));
  int hflags[2] = {0, 0};
  SDB_CUDA(cudaMemcpyAsync(h.data(), hist, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, s));
  SDB_CUDA(cudaMemcpyAsync(hflags, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  SDB_CUDA(cudaStreamSynchronize(s));
  if (hflags[0]) return SDB_OK;  // rows must be sorted without duplicates
  // dense band: every off-diagonal d <= hb at least half full
  int hb = 0;
  while (hb < kBandMaxOff && (double)h[hb + 1] >= 0.5 * (double)(n - hb - 1)) ++hb;
  int hbk = 0;
  for (int w : kBandWidths)
    if (w >= hb) {
      hbk = w;
      break;
    }
  if (hb < 4 || hbk == 0) return SDB_OK;
  unsigned long long band_nnz = h[0];
  for (int d = 1; d <= hbk; ++d) {
    if (h[d] != h[kBandMaxOff + 1 + d]) return SDB_OK;  // not structurally symmetric
    band_nnz += 2 * h[d];
  }
  if ((double)band_nnz < 0.25 * (double)m->nnz) return SDB_OK;
  const int pad = band_pad(hbk);
  const int64_t npad = (n + kBandTileAlign - 1) / kBandTileAlign * kBandTileAlign;
  const int64_t ustride = pad + npad;
  const int64_t ntiles = npad / kBandR;
  const int64_t nstreams = ntiles * kFarWarps;
  if (nstreams + 1 > INT32_MAX) return SDB_OK;
  double* bu = nullptr;
  int32_t *cnt = nullptr, *off = nullptr;
  int2* fhdr = nullptr;
  char* frec = nullptr;
  void* tmp = nullptr;
  unsigned long long* fnnz_d = hist;  // reuse: the histogram has been read back
  auto release = [&]() {
    for (void* p : {(void*)bu, (void*)cnt, (void*)off, (void*)fhdr, (void*)frec, tmp})
      if (p) cudaFree(p);
  };
  cudaError_t e = cudaMalloc(&bu, sizeof(double) * (hbk + 1) * ustride);
  if (e == cudaSuccess) e = cudaMalloc(&cnt, sizeof(int32_t) * (nstreams + 1));
  if (e == cudaSuccess) e = cudaMalloc(&off, sizeof(int32_t) * (nstreams + 1));
  if (e == cudaSuccess) e = cudaMalloc(&fhdr, sizeof(int2) * nstreams);
  if (e == cudaSuccess) e = cudaMemsetAsync(bu, 0, sizeof(double) * (hbk + 1) * ustride, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt + nstreams, 0, sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(fnnz_d, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) {
    release();
    return cuda_fail(e, "band split allocation", __FILE__, __LINE__);
  }
  band_fill_kernel<<<blocks, 256, 0, s>>>(m->rowptr, m->colidx, m->values, n, hbk, pad, ustride, bu);
  band_sym_kernel<<<blocks, 256, 0, s>>>(m->rowptr, m->colidx, m->values, n, hbk, pad, ustride, bu, flags + 1);
  band_far_count_kernel<<<(unsigned)ntiles, kBandR, 0, s>>>(m->rowptr, m->colidx, n, hbk, cnt, fnnz_d);
  size_t tmp_bytes = 0;
  e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, off, nstreams + 1, s);
  if (e == cudaSuccess) e = cudaMalloc(&tmp, tmp_bytes);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, off, nstreams + 1, s);
  int32_t total = 0;
  unsigned long long fnnz = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&total, off + nstreams, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&fnnz, fnnz_d, sizeof(fnnz), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hflags, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    release();
    return cuda_fail(e, "band split", __FILE__, __LINE__);
  }
  if (hflags[1] || total <= 0) {  // values not symmetric (or record count overflow): keep the plain CSR path
    release();
    return SDB_OK;
  }
  e = cudaMalloc(&frec, ((size_t)total + 1) * kRecBytes);  // + the stop record
  if (e == cudaSuccess) {
    band_far_fill_kernel<<<(unsigned)ntiles, kBandR, 0, s>>>(m->rowptr, m->colidx, m->values, n, hbk, off, fhdr,
                                                              frec, total);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(cnt);
  cudaFree(off);
  cudaFree(tmp);
  cnt = off = nullptr;
  tmp = nullptr;
  if (e != cudaSuccess) {
    release();
    return cuda_fail(e, "band far streams", __FILE__, __LINE__);
  }
  m->hb = hbk;
  m->ustride = ustride;
  m->bu = bu;
  m->fhdr = fhdr;
  m->frec = reinterpret_cast<uint4*>(frec);
  m->frecs = total;
  m->fnnz = (int64_t)fnnz;
  return SDB_OK;
}

// The two L2 cache policies as plain 64-bit values: created once per device by a
// one-thread kernel and passed as kernel arguments, so they reach the copy
// instructions from the constant bank (uniform registers) instead of being
// re-materialised per use.
__global__ void band_policy_kernel(uint64_t* out) {
  out[0] = policy_evict_last();
  out[1] = policy_evict_first();
}
static int band_policies(int device, uint64_t* keep, uint64_t* once) {
  static std::mutex mu;
  static uint64_t cache[64][2];
  static bool have[64] = {};
  std::lock_guard<std::mutex> lock(mu);
  if (device < 0 || device >= 64) return fail(SDB_EINVAL, "device index %d out of range", device);
  if (!have[device]) {
    uint64_t* d = nullptr;
    SDB_CUDA(cudaMalloc(&d, 2 * sizeof(uint64_t)));
    band_policy_kernel<<<1, 1>>>(d);
    cudaError_t e = cudaMemcpy(cache[device], d, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "band policy kernel", __FILE__, __LINE__);
    have[device] = true;
  }
  *keep = cache[device][0];
  *once = cache[device][1];
  return SDB_OK;
}

// ---- host planning / launch ---------------------------------------------------------
#define SDB_BAND_HB(HBV, CASE) \
  do {                         \
    switch (HBV) {             \
      case 8: CASE(8); break;  \
      case 16: CASE(16); break; \
      case 20: CASE(20); break; \
      case 24: CASE(24); break; \
      case 32: CASE(32); break; \
      default: return fail(SDB_EUNSUPPORTED, "no band kernel for half-width %d", HBV); \
    }                          \
  } while (0)

// outstanding gather batches per lane (4 slots each): 3, or 2 where shared
// memory is short (half-widths 24 and 32); SDB_BAND_NB=2 forces the shallow ring
static bool band_shallow_ring() {
  const char* e = getenv("SDB_BAND_NB");
  return e && atoi(e) == 2;
}

int band_plan(const sdb_matrix* m, int64_t n_vec, int mode, BandPlan* p) {
  *p = BandPlan{};
  if (m->hb <= 0 || n_vec < 1 || n_vec > SDB_MAX_BATCH) return SDB_OK;
  if (!band_env_enabled()) return SDB_OK;
  (void)mode;
  const int S = kBandS;
  p->hb = m->hb;
  p->S = S;
  p->R = kBandR;
  p->ns = (int)((n_vec + S - 1) / S);
  p->ldvb = (int64_t)p->ns * S;
  const int pad = band_pad(m->hb);
  const int64_t npad = (m->n + kBandTileAlign - 1) / kBandTileAlign * kBandTileAlign;
  p->rows = npad + 2 * pad;
  p->ntiles = npad / p->R;
  size_t smem = 0;
  const bool shallow = band_shallow_ring();
#define SDB_BAND_SMEM(HBV) \
  smem = shallow ? BandSmem<HBV, 2>::kTotal : BandSmem<HBV, BandDepth<HBV>::kDefault>::kTotal
  SDB_BAND_HB(m->hb, SDB_BAND_SMEM);
#undef SDB_BAND_SMEM
  int64_t grid = num_sms(m->device);  // one persistent block per SM
  if (const char* e = getenv("SDB_BAND_GRID")) {
    const int v = atoi(e);
    if (v > 0 && v < grid) grid = v;
  }
  if (grid > p->ntiles * p->ns) grid = p->ntiles * p->ns;
  p->grid = grid < 1 ? 1 : grid;
  p->smem = smem;
  p->block_bytes = ((size_t)p->ns * p->rows * S * sizeof(double) + 255) & ~(size_t)255;
  p->on = true;
  return SDB_OK;
}

int band_pack(const sdb_matrix* m, const BandPlan& p, const double* probes, int64_t ldv, double* v0b, double* bufA,
              double* bufB, cudaStream_t s) {
  const int64_t total = (int64_t)p.ns * p.rows * (p.S / 2);
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 16LL * num_sms(m->device));
  band_pack_kernel<<<blocks, 256, 0, s>>>(probes, m->n, ldv, p.S, p.ns, p.rows, band_pad(p.hb), v0b, bufA, bufB);
  SDB_CHECK_LAUNCH();
  return SDB_OK;
}

template <int HB, int MODE, bool FIRST, int NB>
static int band_launch_t(const BandPlan& p, BandArgs& ba, cudaStream_t s) {
  const void* fn = (const void*)cheb_step_band<HB, MODE, FIRST, NB>;
  // function attributes are per device: set on every launch (cheap)
  SDB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  void* args[] = {(void*)&ba};
  SDB_CUDA(launch_maybe_pdl(fn, dim3((unsigned)p.grid), dim3(kBandThreads), args, p.smem, s));
  return SDB_OK;
}

template <int HB, int NB>
static int band_launch_mode(const BandPlan& p, BandArgs& ba, bool first, int mode, cudaStream_t s) {
  if (mode == SDB_CHEB_DOUBLING)
    return first ? band_launch_t<HB, SDB_CHEB_DOUBLING, true, NB>(p, ba, s)
                 : band_launch_t<HB, SDB_CHEB_DOUBLING, false, NB>(p, ba, s);
  return first ? band_launch_t<HB, SDB_CHEB_DIRECT, true, NB>(p, ba, s)
               : band_launch_t<HB, SDB_CHEB_DIRECT, false, NB>(p, ba, s);
}

int band_launch_step(const sdb_matrix* m, const BandPlan& p, const StepArgs& a, bool first, int mode,
                     cudaStream_t s) {
  BandArgs ba{};
  ba.x = a.x;
  ba.prev = a.prev;
  ba.next = a.next;
  ba.v0 = a.v0;
  ba.sstride = p.rows * p.S;
  ba.bu = m->bu;
  ba.ustride = m->ustride;
  ba.fhdr = m->fhdr;
  ba.frec = reinterpret_cast<const char*>(m->frec);
  ba.stop_rec = m->frecs;
  ba.c = a.c;
  ba.inv_d = a.inv_d;
  ba.n = m->n;
  ba.ntiles = (int)p.ntiles;
  ba.nslices = p.ns;
  ba.ldv = p.ldvb;
  ba.partials = a.partials;
  ba.nblocks = p.grid;
  ba.slotA = a.slotA;
  ba.slotB = a.slotB;
  ba.slot0 = a.slot0;
  ba.legendre = a.legendre;
  ba.la = a.la;
  ba.lb = a.lb;
  ba.lc = a.lc;
  if (const char* e = getenv("SDB_BAND_DIAG")) ba.diag = atoi(e);
  if (int prc = band_policies(m->device, &ba.keep_pol, &ba.once_pol)) return prc;
  const bool shallow = band_shallow_ring();
  int rc = SDB_OK;
#define SDB_BAND_LAUNCH(HBV)                                         \
  rc = shallow ? band_launch_mode<HBV, 2>(p, ba, first, mode, s)     \
               : band_launch_mode<HBV, BandDepth<HBV>::kDefault>(p, ba, first, mode, s)
  SDB_BAND_HB(m->hb, SDB_BAND_LAUNCH);
#undef SDB_BAND_LAUNCH
  return rc;
}

}  // namespace sdb

using namespace sdb;

extern "C" int sdb_matrix_band_info(const sdb_matrix* m, int32_t* half_width, int64_t* far_entries,
                                    int64_t* bytes_per_pass) {
  SDB_REQUIRE(m != nullptr, "NULL argument");
  if (half_width) *half_width = m->hb;
  if (far_entries) *far_entries = m->hb ? m->fnnz : 0;
  if (bytes_per_pass)
    *bytes_per_pass = m->hb ? (int64_t)(m->hb + 1) * 8 * m->n + (int64_t)kRecBytes * m->frecs +
                                  8 * kFarWarps * ((m->n + kBandR - 1) / kBandR)
                            : 0;
  return SDB_OK;
}
